// C++ drop-in preprocessing API (include/trijoin/mesh.hpp, index.hpp) against the reference's
// own outputs for one mesh (tests/golden/preprocess_m1.bin, written by make_preprocess.py from
// proj/src/simplify.cpp build_lod_ladder and proj/src/voxelize.cpp): fill_ladder_paddings,
// compute_facet_hd / compute_facet_ph (single-facet forms), hd_covering_radius and voxelize,
// all bitwise. Run by tests/test_gpu_preprocess.py on a B200.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "trijoin/index.hpp"
#include "trijoin/mesh.hpp"

using namespace trijoin;

namespace {
int g_fail = 0, g_checks = 0;
void check(bool ok, const std::string& what) {
    ++g_checks;
    if (!ok) {
        ++g_fail;
        std::printf("FAIL %s\n", what.c_str());
    }
}
bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

struct Reader {
    std::vector<char> b;
    size_t o = 0;
    template <class T>
    T get() {
        T v;
        std::memcpy(&v, b.data() + o, sizeof(T));
        o += sizeof(T);
        return v;
    }
    Mesh mesh(uint64_t nv, uint64_t nf) {
        Mesh m;
        for (uint64_t i = 0; i < nv; ++i) {
            const double x = get<double>(), y = get<double>(), z = get<double>();
            m.vertices.push_back({x, y, z});
        }
        for (uint64_t f = 0; f < nf; ++f) {
            const uint32_t a = get<uint32_t>(), c = get<uint32_t>(), d = get<uint32_t>();
            m.facets.push_back({a, c, d});
        }
        return m;
    }
};
} // namespace

int main(int argc, char** argv) {
    const std::string path = argc > 1 ? argv[1] : "tests/golden/preprocess_m1.bin";
    std::ifstream in(path, std::ios::binary);
    if (!in) {
        std::printf("cannot open %s\n", path.c_str());
        return 2;
    }
    Reader r{std::vector<char>(std::istreambuf_iterator<char>(in), {})};
    const uint64_t nv = r.get<uint64_t>(), nf = r.get<uint64_t>();
    const Mesh orig = r.mesh(nv, nf);
    const uint32_t nl = r.get<uint32_t>();
    LodLadder want, got;
    for (uint32_t li = 0; li < nl; ++li) {
        LodMesh l;
        l.level = r.get<int32_t>();
        const uint64_t lnv = r.get<uint64_t>(), lnf = r.get<uint64_t>();
        l.mesh = r.mesh(lnv, lnf);
        for (uint64_t f = 0; f < lnf; ++f) l.hd.push_back(r.get<double>());
        for (uint64_t f = 0; f < lnf; ++f) l.ph.push_back(r.get<double>());
        for (uint64_t o = 0; o < nf; ++o) l.ancestor_of_original.push_back(r.get<uint32_t>());
        want.levels.push_back(l);
        l.hd.clear();
        l.ph.clear();
        got.levels.push_back(l);
    }
    const uint32_t k = r.get<uint32_t>();
    const uint64_t seed = r.get<uint64_t>();
    std::vector<uint32_t> labels(want.levels[0].mesh.facets.size());
    for (auto& x : labels) x = r.get<uint32_t>();

    // the whole ladder's paddings in one GPU pass (src/simplify.cpp:229-252)
    fill_ladder_paddings(got, orig, 8);
    for (uint32_t li = 0; li < nl; ++li) {
        const LodMesh &a = got.levels[li], &b = want.levels[li];
        bool ok = a.hd.size() == b.hd.size() && a.ph.size() == b.ph.size();
        for (size_t f = 0; ok && f < a.hd.size(); ++f) ok = same_bits(a.hd[f], b.hd[f]) && same_bits(a.ph[f], b.ph[f]);
        check(ok, "fill_ladder_paddings level " + std::to_string(b.level));
    }
    // batched hd of one level and the single-facet forms
    const LodMesh& c = want.levels[0];
    const std::vector<double> hd = compute_facet_hd(c.mesh, orig, 8);
    bool ok = hd.size() == c.hd.size();
    for (size_t f = 0; ok && f < hd.size(); ++f) ok = same_bits(hd[f], c.hd[f]);
    check(ok, "compute_facet_hd(lod, original)");
    for (uint32_t f : {0u, 7u, (uint32_t)c.mesh.facets.size() - 1}) {
        check(same_bits(compute_facet_hd(c.mesh.triangle(f), orig, 8), c.hd[f]), "compute_facet_hd facet " + std::to_string(f));
        check(same_bits(compute_facet_ph(f, c, orig), c.ph[f]), "compute_facet_ph facet " + std::to_string(f));
    }
    const Triangle t = c.mesh.triangle(3);
    check(same_bits(hd_covering_radius(t, 8), (2.0 / 3.0) * t.longest_edge() / 8.0), "hd_covering_radius");
    // k-means voxelisation of the coarsest level (src/voxelize.cpp:27-79)
    check(voxelize(c, k, seed) == labels, "voxelize");
    bool threw = false;
    try {
        voxelize(c, 0, seed);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    check(threw, "voxelize k = 0 throws std::invalid_argument");
    std::printf("test_preprocess: %d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
