// Shared declarations of the device join pipeline (filter, knn, refine-loop stages).
#pragma once
#include <cstdint>
#include <memory>
#include <vector>

#include "tj_internal.cuh"

namespace tjx {

// First soundness failure seen on the device (EngineError tripwires).
struct DevError {
    int code;      // 0 or TJ_EENGINE
    uint32_t op;   // lowest failing candidate (UINT32_MAX = none)
    double lb, ub; // its crossing interval (intersect_interval message)
    int kind;      // 0 bound crossing, 1 knn confirmed count exceeds k
};

// Device view of the candidate set (reference CandidateSet, include/trijoin/filter.hpp:38-48).
struct CandDev {
    uint32_t* pair_r;
    uint32_t* pair_s;
    double* lb;
    double* ub;
    uint8_t* status;
    int16_t* decided_at;
    uint32_t* num_confirmed;
    const uint64_t* r2op;
};

struct CandDevStore {
    DevBuf<uint32_t> pair_r, pair_s, num_confirmed;
    DevBuf<double> lb, ub;
    DevBuf<uint8_t> status;
    DevBuf<int16_t> decided_at;
    DevBuf<uint64_t> r2op;
    uint64_t n = 0;
    uint32_t nq = 0;
    void resize(uint64_t n_cands, uint32_t n_queries) {
        n = n_cands;
        nq = n_queries;
        const uint64_t m = n_cands ? n_cands : 1;
        pair_r.reserve(m);
        pair_s.reserve(m);
        lb.reserve(m);
        ub.reserve(m);
        status.reserve(m);
        decided_at.reserve(m);
        num_confirmed.reserve(n_queries ? n_queries : 1);
    }
    CandDev view() {
        return {pair_r.p, pair_s.p, lb.p, ub.p, status.p, decided_at.p, num_confirmed.p, r2op.p};
    }
};

// One side's on-demand expansion of a compact-resident level (materialize_level): the active
// voxels' facet records, their FP32 screening records and segment aggregates, grow-only.
struct LevelMat {
    DevBuf<uint8_t> flag;       // [nv] voxel touched by the chunk's active voxel pairs
    DevBuf<uint64_t> cnt, off;  // [nv] facets of touched voxels; [nv+1] their exclusive scan
    DevBuf<double> facets;      // [total * TJ_FACET_STRIDE]
    DevBuf<float4> screen, seg; // [total * kScreenRecF4], [3 nv]
    DevBuf<unsigned> agg;       // [3] level aggregates of the expanded records
    uint64_t total = 0;
};

struct Workspace {
    int num_sms = 148;
    LevelMat mat[2];            // compact-resident datasets: R side, S side
    uint64_t workset_budget = 0; // bytes for materialized levels (0 = not yet chosen)
    DevBuf<unsigned char> temp;
    DevBuf<uint64_t> u64a;
    std::unique_ptr<RefineQueueStore> queue; // refinement pair queues, grow-only, per context
    DevBuf<float4> screen_r, screen_s;       // per-level FP32 screening records, grow-only
    DevBuf<unsigned> level_agg;              // per-level record aggregates (RefineSource::agg)
    DevBuf<float4> seg_r, seg_s;             // per-level voxel segment aggregates, grow-only
    DevBuf<ActiveVpDev> active;              // the join's active voxel pairs (tj_join), grow-only: a
                                             // per-join allocation of GBs (D, E) stalled on pool growth
    DevBuf<ActiveVpDev> active_alt;          // compaction scratch of the active list, grow-only
    DevBuf<int64_t> nsel;
    void release() {
        temp.release();
        u64a.release();
        queue.reset();
        screen_r.release();
        screen_s.release();
        level_agg.release();
        seg_r.release();
        seg_s.release();
        active.release();
        active_alt.release();
        nsel.release();
        for (auto& m : mat) m = LevelMat{};
    }
};

struct SortedS {
    DevBuf<uint32_t> order; // S indices sorted by mbb.min.x
    DevBuf<double> mbb;     // S mbbs in that order
    DevBuf<float4> yz;      // their y / z extents outward-rounded to FP32: (y lo, y hi, z lo, z hi)
    double max_ext = 0.0;   // max over S of mbb.max.x - mbb.min.x
};

struct MbbArgs {
    const double* r_mbb;
    const double* r_anchor;
    const double* s_mbb;
    const double* s_anchor;
    const double* s_sorted_mbb;
    const float4* s_sorted_yz; // optional FP32 y / z pre-rejection (SortedS::yz)
    const uint32_t* s_order;
    uint32_t nr, ns;
    double tau;              // within threshold
    const double* tau_per_r; // k-NN: u_k(r) per query (nullptr = scalar tau)
    double max_ext;
    int confirm_at_mbb;      // within: ub <= tau confirms at the MBB stage
    uint32_t shard_index, shard_count, shard_block;
};

struct VoxelArgs {
    uint64_t n_cands;
    const uint64_t* r_voff;
    const uint64_t* s_voff;
    const double* r_vbox;
    const double* s_vbox;
    const double* r_vanc;
    const double* s_vanc;
    int prune;  // within: prune at the voxel stage
    double tau;
    DevError* err;
};

struct PrunedVp {
    uint32_t op, vr, vs; // object-local voxel ids
    double lb;
};

struct VoxelOut {
    uint64_t vp_generated, vp_pruned, survivors;
};

uint64_t scan_counts(Workspace& ws, const uint32_t* counts, uint64_t n, DevBuf<uint64_t>& offsets, cudaStream_t st);
void mbb_prepare_s(Workspace& ws, const DatasetDev& S, SortedS& out, cudaStream_t st);
void knn_kth_anchor(Workspace& ws, const MbbArgs& a, uint32_t k, DevBuf<double>& u_k, cudaStream_t st);
uint64_t mbb_candidates(Workspace& ws, const MbbArgs& a, CandDevStore& cs, cudaStream_t st);
VoxelOut voxel_filter(Workspace& ws, const VoxelArgs& a, CandDevStore& cs, DevBuf<ActiveVpDev>& active,
                      bool want_trace, std::vector<PrunedVp>* pruned_host, std::vector<uint8_t>* touched_host,
                      cudaStream_t st);

// knn.cu
// k-NN pruning rounds to a fixpoint for every query (knn_prune_to_fixpoint, src/knn.cpp:82-91).
uint64_t knn_fixpoint(Workspace& ws, CandDevStore& cs, uint32_t k, int16_t stage, DevError* err, cudaStream_t st);
// One pruning round, deltas only (knn_prune_round, src/knn.cpp:19-63); returns the count.
uint64_t knn_round_dev(Workspace& ws, CandDevStore& cs, uint32_t k, DevBuf<uint8_t>& delta, DevError* err,
                       cudaStream_t st);
// knn_finalize (src/knn.cpp:93-118).
void knn_finalize_dev(Workspace& ws, CandDevStore& cs, uint32_t k, cudaStream_t st);

// refine_loop.cu
struct LevelStats {
    uint32_t level;
    uint64_t vps, facet_pairs, evaluated, tested, screened, verified, vps_skipped, facets_dropped;
    double ms, kernel_ms, wait_ms;
    double screen_ms = 0.0; // k_screen launches only (CUDA events)
};
struct RefineLoopOut {
    std::vector<LevelStats> levels;
    uint64_t chunks = 0;
    uint32_t queue_reruns = 0; // levels re-run after an exact-queue overflow
    uint64_t mat_chunks = 0;   // compact-resident datasets: materialized chunks over all levels
};
struct TraceSink; // host-side trace forwarding (engine.cu)
RefineLoopOut refine_loop_dev(Workspace& ws, const DatasetDev& R, const DatasetDev& S, CandDevStore& cs,
                              DevBuf<ActiveVpDev>& active, uint64_t n_active, const tj_join_spec& spec, bool knn,
                              double tau, bool decision, DevError* err, TraceSink* trace, cudaStream_t st);
// --exact: confirmed intervals become [d, d], d the level-100 mesh distance (src/engine.cpp:96-118).
void exact_recompute_dev(Workspace& ws, const DatasetDev& R, const DatasetDev& S, CandDevStore& cs, cudaStream_t st);

} // namespace tjx
