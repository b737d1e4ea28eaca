// Offline preprocessing API of the drop-in (reference include/trijoin/mesh.hpp:65-73 and
// index.hpp:48): thin host layer over the GPU kernels of csrc/preprocess.cu (tj_facet_hd_batch,
// tj_facet_ph_batch, tj_voxelize_batch). Meshes are packed into the C-ABI's mesh-set form.
#include <cmath>
#include <stdexcept>

#include "packed.hpp"
#include "trijoin/index.hpp"
#include "trijoin/mesh.hpp"

namespace trijoin {

namespace {

// Packed mesh set (tj_capi.h "offline preprocessing" layout).
struct MeshSet {
    std::vector<uint64_t> vo{0}, fo{0};
    std::vector<double> v;
    std::vector<uint32_t> f;
    void add(const Mesh& m) {
        for (const Point3& p : m.vertices) v.insert(v.end(), {p.x, p.y, p.z});
        for (const auto& t : m.facets) f.insert(f.end(), {t[0], t[1], t[2]});
        vo.push_back(vo.back() + m.vertices.size());
        fo.push_back(fo.back() + m.facets.size());
    }
    uint32_t n() const { return (uint32_t)(vo.size() - 1); }
};

void push_tri(std::vector<double>& out, const Triangle& t) {
    out.insert(out.end(), {t.v0.x, t.v0.y, t.v0.z, t.v1.x, t.v1.y, t.v1.z, t.v2.x, t.v2.y, t.v2.z});
}

tj_ctx* ctx0() { return detail::device_context(detail::join_devices()[0]); }

} // namespace

double hd_covering_radius(const Triangle& f_prime, int grid_level) {
    return (2.0 / 3.0) * f_prime.longest_edge() / static_cast<double>(grid_level);
}

std::vector<double> compute_facet_hd(const Mesh& lod, const Mesh& original, int grid_level) {
    MeshSet ms;
    ms.add(original);
    std::vector<double> q;
    q.reserve(9 * lod.facets.size());
    for (size_t f = 0; f < lod.facets.size(); ++f) push_tri(q, lod.triangle(f));
    const uint64_t qo[2] = {0, lod.facets.size()};
    std::vector<double> hd(lod.facets.size());
    tj_ctx* ctx = ctx0();
    detail::check(tj_facet_hd_batch(ctx, 1, ms.vo.data(), ms.v.data(), ms.fo.data(), ms.f.data(), qo, q.data(),
                                    grid_level, hd.data()),
                  ctx);
    return hd;
}

double compute_facet_hd(const Triangle& f_prime, const Mesh& original, int grid_level) {
    MeshSet ms;
    ms.add(original);
    std::vector<double> q;
    push_tri(q, f_prime);
    const uint64_t qo[2] = {0, 1};
    double hd = 0;
    tj_ctx* ctx = ctx0();
    detail::check(tj_facet_hd_batch(ctx, 1, ms.vo.data(), ms.v.data(), ms.fo.data(), ms.f.data(), qo, q.data(),
                                    grid_level, &hd),
                  ctx);
    return hd;
}

double compute_facet_ph(uint32_t f_prime_id, const LodMesh& lod, const Mesh& original) {
    if (f_prime_id >= lod.mesh.facets.size()) throw std::invalid_argument("compute_facet_ph: facet id out of range");
    if (lod.ancestor_of_original.size() != original.facets.size())
        throw std::invalid_argument("compute_facet_ph: ancestor map does not match the original mesh");
    // only the originals mapped to f_prime matter: a one-facet LOD set keeps the transfer small
    Mesh sub;
    sub.vertices = original.vertices;
    std::vector<uint32_t> anc;
    for (uint32_t o = 0; o < original.facets.size(); ++o)
        if (lod.ancestor_of_original[o] == f_prime_id) {
            sub.facets.push_back(original.facets[o]);
            anc.push_back(0);
        }
    if (sub.facets.empty()) return 0.0;
    MeshSet ms;
    ms.add(sub);
    std::vector<double> t;
    push_tri(t, lod.mesh.triangle(f_prime_id));
    const uint64_t lo[2] = {0, 1};
    double ph = 0;
    tj_ctx* ctx = ctx0();
    detail::check(tj_facet_ph_batch(ctx, 1, ms.vo.data(), ms.v.data(), ms.fo.data(), ms.f.data(), anc.data(), lo,
                                    t.data(), &ph),
                  ctx);
    return ph;
}

void fill_ladder_paddings(std::span<LodLadder* const> ladders, std::span<const Mesh* const> originals, int hd_grid) {
    if (ladders.size() != originals.size()) throw std::invalid_argument("fill_ladder_paddings: size mismatch");
    // hd: one mesh-set entry per ladder (its original mesh, one tree), queried by the facets of
    // all its coarse levels; ph: one entry per (ladder, coarse level) with that level's ancestors
    MeshSet hd_set, ph_set;
    std::vector<uint64_t> hq{0}, pq{0};
    std::vector<double> q;
    std::vector<uint32_t> anc;
    std::vector<std::pair<size_t, size_t>> slots; // (ladder, level) in query order
    for (size_t i = 0; i < ladders.size(); ++i) {
        LodLadder& L = *ladders[i];
        const Mesh& orig = *originals[i];
        size_t coarse = 0;
        for (size_t li = 0; li < L.levels.size(); ++li) {
            LodMesh& lod = L.levels[li];
            const size_t nf = lod.mesh.facets.size();
            if (li + 1 == L.levels.size()) { // level 100: identically 0 (include/trijoin/mesh.hpp:57)
                lod.hd.assign(nf, 0.0);
                lod.ph.assign(nf, 0.0);
                continue;
            }
            if (lod.ancestor_of_original.size() != orig.facets.size())
                throw std::invalid_argument("fill_ladder_paddings: ancestor map does not match the original mesh");
            for (uint32_t a : lod.ancestor_of_original)
                if (a >= nf) throw std::invalid_argument("fill_ladder_paddings: ancestor id out of range");
            for (size_t f = 0; f < nf; ++f) push_tri(q, lod.mesh.triangle(f));
            ph_set.add(orig);
            pq.push_back(pq.back() + nf);
            anc.insert(anc.end(), lod.ancestor_of_original.begin(), lod.ancestor_of_original.end());
            slots.emplace_back(i, li);
            coarse += nf;
        }
        if (coarse) {
            hd_set.add(orig);
            hq.push_back(hq.back() + coarse);
        }
    }
    if (slots.empty()) return;
    std::vector<double> hd(pq.back()), ph(pq.back());
    tj_ctx* ctx = ctx0();
    detail::check(tj_facet_hd_batch(ctx, hd_set.n(), hd_set.vo.data(), hd_set.v.data(), hd_set.fo.data(),
                                    hd_set.f.data(), hq.data(), q.data(), hd_grid, hd.data()),
                  ctx);
    detail::check(tj_facet_ph_batch(ctx, ph_set.n(), ph_set.vo.data(), ph_set.v.data(), ph_set.fo.data(),
                                    ph_set.f.data(), anc.data(), pq.data(), q.data(), ph.data()),
                  ctx);
    for (size_t k = 0; k < slots.size(); ++k) {
        LodMesh& lod = ladders[slots[k].first]->levels[slots[k].second];
        lod.hd.assign(hd.begin() + (ptrdiff_t)pq[k], hd.begin() + (ptrdiff_t)pq[k + 1]);
        lod.ph.assign(ph.begin() + (ptrdiff_t)pq[k], ph.begin() + (ptrdiff_t)pq[k + 1]);
    }
}

void fill_ladder_paddings(LodLadder& ladder, const Mesh& original, int hd_grid) {
    LodLadder* l = &ladder;
    const Mesh* o = &original;
    fill_ladder_paddings(std::span<LodLadder* const>(&l, 1), std::span<const Mesh* const>(&o, 1), hd_grid);
}

std::vector<std::vector<uint32_t>> voxelize_batch(std::span<const LodMesh* const> coarsest,
                                                  std::span<const uint32_t> k, std::span<const uint64_t> seeds) {
    if (coarsest.size() != k.size() || k.size() != seeds.size())
        throw std::invalid_argument("voxelize: size mismatch");
    for (uint32_t kk : k)
        if (kk == 0) throw std::invalid_argument("voxelize: k must be >= 1");
    MeshSet ms;
    for (const LodMesh* l : coarsest) ms.add(l->mesh);
    std::vector<uint32_t> labels(ms.fo.back());
    tj_ctx* ctx = ctx0();
    detail::check(tj_voxelize_batch(ctx, ms.n(), ms.vo.data(), ms.v.data(), ms.fo.data(), ms.f.data(), k.data(),
                                    seeds.data(), labels.data()),
                  ctx);
    std::vector<std::vector<uint32_t>> out(coarsest.size());
    for (size_t i = 0; i < coarsest.size(); ++i)
        out[i].assign(labels.begin() + (ptrdiff_t)ms.fo[i], labels.begin() + (ptrdiff_t)ms.fo[i + 1]);
    return out;
}

std::vector<uint32_t> voxelize(const LodMesh& coarsest, uint32_t k, uint64_t seed) {
    if (k == 0) throw std::invalid_argument("voxelize: k must be >= 1");
    const LodMesh* c = &coarsest;
    return voxelize_batch(std::span<const LodMesh* const>(&c, 1), std::span<const uint32_t>(&k, 1),
                          std::span<const uint64_t>(&seed, 1))[0];
}

} // namespace trijoin
