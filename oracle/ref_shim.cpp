// TEST INFRASTRUCTURE ONLY. extern "C" probes into the reference trijoin core
// (compiled from /root/reference/proj/src by oracle/Makefile). Used by tests/
// and tests/golden/make_golden.py to produce golden vectors; never linked into
// the product. Every probe calls the reference's own functions unchanged.
#include <cstdint>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "helpers.hpp"  // reference tests' fixtures (mini_dataset, random_triangle)
#include "trijoin/engine.hpp"
#include "trijoin/filter.hpp"
#include "trijoin/geom.hpp"
#include "trijoin/index.hpp"
#include "trijoin/knn.hpp"
#include "trijoin/mesh.hpp"
#include "trijoin/bvh.hpp"
#include "trijoin/refine.hpp"

using namespace trijoin;

namespace {
thread_local std::string g_err;

Triangle tri_from(const double* p) {
    return {{p[0], p[1], p[2]}, {p[3], p[4], p[5]}, {p[6], p[7], p[8]}};
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const EngineError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}
Mesh mesh_from(const double* verts, uint64_t nv, const uint32_t* facets, uint64_t nf) {
    Mesh m;
    m.vertices.resize(nv);
    for (uint64_t i = 0; i < nv; ++i) m.vertices[i] = {verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]};
    m.facets.resize(nf);
    for (uint64_t f = 0; f < nf; ++f) m.facets[f] = {facets[3 * f], facets[3 * f + 1], facets[3 * f + 2]};
    return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// proj/src/geom.cpp:152-183
void ref_tri_tri_batch(uint64_t n, const double* a9, const double* b9, double* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = tri_tri_distance(tri_from(a9 + 9 * i), tri_from(b9 + 9 * i));
}

// proj/src/geom.cpp:18-24 (a: points [3], b: segments [6])
void ref_point_segment_batch(uint64_t n, const double* a3, const double* b6, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const double* p = a3 + 3 * i;
        const double* q = b6 + 6 * i;
        out[i] = point_segment_distance({p[0], p[1], p[2]}, {q[0], q[1], q[2]}, {q[3], q[4], q[5]});
    }
}

// proj/src/geom.cpp:39-80 (a: points [3], b: triangles [9])
void ref_point_triangle_batch(uint64_t n, const double* a3, const double* b9, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const double* p = a3 + 3 * i;
        out[i] = point_triangle_distance({p[0], p[1], p[2]}, tri_from(b9 + 9 * i));
    }
}

// proj/src/geom.cpp:82-113 (a, b: segments [6])
void ref_segment_segment_batch(uint64_t n, const double* a6, const double* b6, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const double* p = a6 + 6 * i;
        const double* q = b6 + 6 * i;
        out[i] = segment_segment_distance({p[0], p[1], p[2]}, {p[3], p[4], p[5]}, {q[0], q[1], q[2]},
                                          {q[3], q[4], q[5]});
    }
}

// proj/src/geom.cpp:11-16
void ref_mindist_aabb_batch(uint64_t n, const double* a6, const double* b6, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        Aabb a{{a6[6 * i], a6[6 * i + 1], a6[6 * i + 2]}, {a6[6 * i + 3], a6[6 * i + 4], a6[6 * i + 5]}};
        Aabb b{{b6[6 * i], b6[6 * i + 1], b6[6 * i + 2]}, {b6[6 * i + 3], b6[6 * i + 4], b6[6 * i + 5]}};
        out[i] = mindist_aabb(a, b);
    }
}

// proj/tests/helpers.hpp:35-38 random_triangle over SplitMix64 (proj/include/trijoin/rng.hpp)
void ref_random_tri_pairs(uint64_t seed, uint64_t n, double lo, double hi, double size, double* a9,
                          double* b9) {
    SplitMix64 rng(seed);
    for (uint64_t i = 0; i < n; ++i) {
        const Triangle a = testing::random_triangle(rng, lo, hi, size);
        const Triangle b = testing::random_triangle(rng, lo, hi, size);
        std::memcpy(a9 + 9 * i, &a, sizeof(double) * 9);
        std::memcpy(b9 + 9 * i, &b, sizeof(double) * 9);
    }
}

// proj/src/refine.cpp:63-84 on a caller-provided batch
int ref_refine_kernel(uint64_t n_tris, const double* tris9, const double* hd, const double* ph,
                      uint64_t n_descs, const uint64_t* r_off, const uint64_t* s_off,
                      const uint32_t* r_len, const uint32_t* s_len, double* vp_lb, double* vp_ub,
                      unsigned workers) {
    return guarded([&] {
        VoxelPairBatch b;
        b.tris.resize(n_tris);
        std::memcpy(b.tris.data(), tris9, sizeof(double) * 9 * n_tris);
        b.hd.assign(hd, hd + n_tris);
        b.ph.assign(ph, ph + n_tris);
        for (uint64_t d = 0; d < n_descs; ++d) b.descs.push_back({r_off[d], s_off[d], r_len[d], s_len[d], 0});
        ThreadPool pool(workers);
        std::vector<double> lb, ub;
        refine_kernel(b, pool, lb, ub);
        std::memcpy(vp_lb, lb.data(), sizeof(double) * n_descs);
        std::memcpy(vp_ub, ub.data(), sizeof(double) * n_descs);
    });
}

// proj/tests/helpers.hpp:69-87 mini_dataset -> 3DPJ1 file
int ref_mini_dataset(uint32_t count, double spacing, uint64_t seed, uint32_t facets,
                     double voxel_ratio, const char* out_path) {
    return guarded([&] {
        const PreparedDataset ds = testing::mini_dataset(count, spacing, seed, facets, voxel_ratio);
        save_index(ds, out_path);
    });
}

// Staged reference run (proj/tests/test_refine.cpp:21-39 staged_within + active_of):
// MBB filter + chunked voxel filter at tau, then per listed level the gathered
// batch and refine_kernel outputs for the full active set. Binary dump:
//   u64 n_cands; per cand: u32 r, u32 s, f64 lb, f64 ub, u8 status, i16 decided_at
//   u64 n_active; per active: u32 op, u32 vr, u32 vs
//   u32 n_levels; per level: u32 level, u64 facet_pairs; f64 lb[n_active]; f64 ub[n_active]
int ref_staged_dump(const char* r_path, const char* s_path, double tau, const uint32_t* levels,
                    uint32_t n_levels, const char* out_path) {
    return guarded([&] {
        const PreparedDataset R = load_index(r_path);
        PreparedDataset s_store;
        const PreparedDataset* S = &R;
        if (s_path && *s_path && std::string(s_path) != r_path) {
            s_store = load_index(s_path);
            S = &s_store;
        }
        ThreadPool pool(2);
        const RTree tree = build_rtree(S->objects);
        CandidateSet cands = mbb_filter_within(R, *S, tree, tau, pool);
        const VoxelPairList vpl = chunked_filter(cands, R, *S, UINT64_MAX, tau, false, pool);
        std::vector<ActiveVp> active;
        for (uint32_t op = 0; op < cands.size(); ++op) {
            if (cands.status[op] != PairStatus::Undecided) continue;
            for (uint64_t i = vpl.op_offsets[op]; i < vpl.op_offsets[op + 1]; ++i)
                active.push_back({op, vpl.vpairs[i].first, vpl.vpairs[i].second});
        }
        FILE* f = std::fopen(out_path, "wb");
        if (!f) throw std::runtime_error("cannot open dump");
        auto put = [&](const void* p, size_t n) { std::fwrite(p, 1, n, f); };
        uint64_t nc = cands.size();
        put(&nc, 8);
        for (uint64_t i = 0; i < nc; ++i) {
            put(&cands.pairs[i].first, 4);
            put(&cands.pairs[i].second, 4);
            put(&cands.intervals[i].lb, 8);
            put(&cands.intervals[i].ub, 8);
            uint8_t st = static_cast<uint8_t>(cands.status[i]);
            put(&st, 1);
            put(&cands.decided_at[i], 2);
        }
        uint64_t na = active.size();
        put(&na, 8);
        for (const ActiveVp& a : active) {
            put(&a.op, 4);
            put(&a.vr, 4);
            put(&a.vs, 4);
        }
        put(&n_levels, 4);
        for (uint32_t li = 0; li < n_levels; ++li) {
            const VoxelPairBatch batch = gather_facet_data(active, levels[li], R, *S, cands);
            std::vector<double> lb, ub;
            refine_kernel(batch, pool, lb, ub);
            uint64_t fp = 0;
            for (const VpDesc& d : batch.descs) fp += uint64_t(d.r_len) * d.s_len;
            put(&levels[li], 4);
            put(&fp, 8);
            put(lb.data(), 8 * lb.size());
            put(ub.data(), 8 * ub.size());
        }
        std::fclose(f);
    });
}

// The reference's own run_join (src/engine.cpp:122-237) timed at its own boundary: both
// indexes are loaded first (untimed), then `repeats` joins run on ThreadPool(workers).
// out[0] = best wall ms, out[1] = candidate pairs entering the voxel stage
// (stats stages["voxel"].pairs_in), out[2] = sum of facet_pairs, out[3] = results,
// out[4] = pool size, out[5] = total candidate pairs.
int ref_join_timed_records(const char* r_path, const char* s_path, int type, double tau, uint32_t k,
                           const uint32_t* lods, uint32_t n_lods, unsigned workers, uint32_t repeats,
                           double* out, const char* records_path);
int ref_join_timed(const char* r_path, const char* s_path, int type, double tau, uint32_t k,
                   const uint32_t* lods, uint32_t n_lods, unsigned workers, uint32_t repeats,
                   double* out) {
    return ref_join_timed_records(r_path, s_path, type, tau, k, lods, n_lods, workers, repeats, out, nullptr);
}

// Same, and the last join's records (JoinResultRecord, include/trijoin/engine.hpp:36-41, in
// the reference's own order) are written to `records_path` (when non-NULL) as packed
// 32-byte rows: u32 r, u32 s, f64 lb, f64 ub, i16 decided_at, i16 0, u32 rank.
int ref_join_timed_records(const char* r_path, const char* s_path, int type, double tau, uint32_t k,
                           const uint32_t* lods, uint32_t n_lods, unsigned workers, uint32_t repeats,
                           double* out, const char* records_path) {
    return guarded([&] {
        const PreparedDataset R = load_index(r_path);
        PreparedDataset s_store;
        const PreparedDataset* S = &R;
        if (s_path && *s_path && std::string(s_path) != r_path) {
            s_store = load_index(s_path);
            S = &s_store;
        }
        JoinSpec spec;
        spec.type = type == 0 ? JoinType::Within : type == 1 ? JoinType::Intersect : JoinType::Knn;
        spec.tau = tau;
        spec.k = k;
        spec.lods.assign(lods, lods + n_lods);
        ThreadPool pool(workers);
        double best = 1e300;
        JoinOutput jo;
        for (uint32_t i = 0; i < (repeats ? repeats : 1); ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            jo = run_join(R, *S, spec, pool);
            const double ms =
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            best = std::min(best, ms);
        }
        uint64_t fp = 0;
        for (const auto& st : jo.stats.stages) fp += st.facet_pairs;
        out[0] = best;
        out[1] = jo.stats.stages.size() > 1 ? static_cast<double>(jo.stats.stages[1].pairs_in) : 0.0;
        out[2] = static_cast<double>(fp);
        out[3] = static_cast<double>(jo.stats.results);
        out[4] = pool.size();
        out[5] = jo.stats.stages.empty()
                     ? 0.0
                     : static_cast<double>(jo.stats.stages[0].pairs_in - jo.stats.stages[0].removed);
        if (records_path && *records_path) {
            std::FILE* f = std::fopen(records_path, "wb");
            if (!f) throw std::runtime_error(std::string("cannot write ") + records_path);
            for (const JoinResultRecord& rec : jo.records) {
                unsigned char row[32] = {};
                const int16_t pad = 0;
                std::memcpy(row, &rec.r, 4);
                std::memcpy(row + 4, &rec.s, 4);
                std::memcpy(row + 8, &rec.lb, 8);
                std::memcpy(row + 16, &rec.ub, 8);
                std::memcpy(row + 24, &rec.decided_at, 2);
                std::memcpy(row + 26, &pad, 2);
                std::memcpy(row + 28, &rec.rank, 4);
                std::fwrite(row, 1, 32, f);
            }
            std::fclose(f);
        }
    });
}


// ---- offline preprocessing ----
// proj/src/simplify.cpp build_lod_ladder (incl. hd / ph, :229-251). Binary dump to out_path:
//   u32 n_levels; per level: i32 level, u8 clamped, u64 nv, u64 nf, f64 verts[3 nv],
//   u32 facets[3 nf], f64 hd[nf or 0 at level 100: u64 count first], f64 ph[same],
//   u64 n_orig, u32 ancestor_of_original[n_orig]
int ref_build_ladder(const double* verts, uint64_t nv, const uint32_t* facets, uint64_t nf, const int32_t* lods,
                     uint32_t n_lods, int32_t hd_grid, const char* out_path) {
    return guarded([&] {
        const Mesh m = mesh_from(verts, nv, facets, nf);
        const LodLadder L = build_lod_ladder(m, std::vector<int>(lods, lods + n_lods), hd_grid);
        FILE* f = std::fopen(out_path, "wb");
        if (!f) throw std::runtime_error("cannot write ladder dump");
        auto w = [&](const void* p, size_t n) { std::fwrite(p, 1, n, f); };
        const uint32_t nl = (uint32_t)L.levels.size();
        w(&nl, 4);
        for (const LodMesh& lod : L.levels) {
            const int32_t lv = lod.level;
            const uint8_t cl = lod.clamped ? 1 : 0;
            const uint64_t lnv = lod.mesh.vertices.size(), lnf = lod.mesh.facets.size();
            w(&lv, 4);
            w(&cl, 1);
            w(&lnv, 8);
            w(&lnf, 8);
            for (const Point3& v : lod.mesh.vertices) { const double t[3] = {v.x, v.y, v.z}; w(t, 24); }
            for (const auto& t : lod.mesh.facets) w(t.data(), 12);
            const uint64_t nh = lod.hd.size(), np = lod.ph.size();
            w(&nh, 8);
            w(lod.hd.data(), 8 * nh);
            w(&np, 8);
            w(lod.ph.data(), 8 * np);
            const uint64_t na = lod.ancestor_of_original.size();
            w(&na, 8);
            w(lod.ancestor_of_original.data(), 4 * na);
        }
        std::fclose(f);
    });
}

// proj/src/hausdorff.cpp:15-33 compute_facet_hd (Mesh overload) for n query triangles
int ref_facet_hd(const double* verts, uint64_t nv, const uint32_t* facets, uint64_t nf, uint64_t n,
                 const double* tris9, int32_t grid, double* out) {
    return guarded([&] {
        const Mesh m = mesh_from(verts, nv, facets, nf);
        const TriBvh bvh(m);
        for (uint64_t i = 0; i < n; ++i) out[i] = compute_facet_hd(tri_from(tris9 + 9 * i), bvh, grid);
    });
}

// proj/src/voxelize.cpp:27-79 voxelize on a mesh given as its coarsest level
int ref_voxelize(const double* verts, uint64_t nv, const uint32_t* facets, uint64_t nf, uint32_t k, uint64_t seed,
                 uint32_t* labels) {
    return guarded([&] {
        LodMesh lod;
        lod.level = 20;
        lod.mesh = mesh_from(verts, nv, facets, nf);
        const std::vector<uint32_t> l = voxelize(lod, k, seed);
        std::memcpy(labels, l.data(), 4 * l.size());
    });
}

}  // extern "C"
