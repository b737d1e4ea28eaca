// Device-resident progressive refinement (reference refine_loop / run_level /
// aggregate_object_bounds, src/refine.cpp:86-122, :136-314; paper Alg. 4-5).
//
// The active voxel-pair list lives in HBM for the whole loop. Per LOD level:
//   1. the reference facet-pair count sum(r_len * s_len) is reduced from the CSR offsets;
//   2. refine kernel launches (launch size = max(refine_chunk, 16Mi) voxel pairs: the
//      reference's refine_chunk bounds host memory, the device has room for a whole level,
//      and every launch boundary costs a drain + an exact-evaluation launch (config B:
//      500k -> 81.5 ms, 2M -> 76.4, 8M -> 74.8); the outcome is independent of it) fold each voxel pair's exact minima into per-op
//      minima with 64-bit atomicMin on the IEEE bit patterns (order-free and exact for
//      non-negative doubles);
//   3. one thread per op applies aggregate_object_bounds (skip ops whose minima stayed
//      +inf, intersect_interval with the 1e-9 crossing tripwire) and, for within-tau,
//      prune_within at this level's stage code; k-NN runs its pruning fixpoint;
//   4. voxel pairs of decided ops are dropped by a stable compaction
//      (erase_if, src/refine.cpp:299-301).
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "filter.cuh"
#include "scan.cuh"
#include "trace_sink.h"

namespace tjx {

namespace {

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000ll); }

__global__ void k_fill_u64(unsigned long long* p, uint64_t n, unsigned long long v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_copy_agg(const unsigned* __restrict__ r, const unsigned* __restrict__ s, unsigned* agg) {
    if (threadIdx.x < 3) agg[threadIdx.x] = r[threadIdx.x];
    else if (threadIdx.x < 6) agg[threadIdx.x] = s[threadIdx.x - 3];
}

__global__ void k_facet_pairs(const ActiveVpDev* __restrict__ act, uint64_t n, const uint64_t* __restrict__ rf,
                              const uint64_t* __restrict__ sf, unsigned long long* out) {
    unsigned long long acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const ActiveVpDev a = act[i];
        acc += (rf[a.gvr + 1] - rf[a.gvr]) * (sf[a.gvs + 1] - sf[a.gvs]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

__global__ void k_aggregate(CandDev c, uint64_t n, const unsigned long long* __restrict__ lbb,
                            const unsigned long long* __restrict__ ubb, int prune, double tau, int16_t stage,
                            int decision, uint32_t exact_mask, uint8_t* __restrict__ updated, DevError* err) {
    for (uint64_t op = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; op < n; op += (uint64_t)gridDim.x * blockDim.x) {
        if (updated) updated[op] = 0;
        if (c.status[op] != TJ_UNDECIDED) continue;
        const double mlb = __longlong_as_double((long long)lbb[op]);
        const double mub = __longlong_as_double((long long)ubb[op]);
        if (!(mlb < dinf())) continue; // every voxel pair empty at this level (or op not active)
        double lb = c.lb[op], ub = c.ub[op];
        ub = (mub < ub) ? mub : ub;
        // decision mode: a positive mlb is only known to be positive (pairs that could lower
        // it were skipped); clamping it to ub keeps "lb > 0" and never trips the crossing check
        // (except the sampled ops that keep exact intervals: their crossing check is the reference's)
        const double mlb_d = (decision && !exact_op(exact_mask, (uint32_t)op) && mlb > 0.0 && ub < mlb) ? ub : mlb;
        lb = (lb < mlb_d) ? mlb_d : lb;
        if (lb > ub) {
            if (lb - ub > 1e-9) {
                atomicMin(&err->op, (uint32_t)op);
                err->lb = lb;
                err->ub = ub;
                err->kind = 0;
                atomicExch(&err->code, (int)TJ_EENGINE);
            }
            const double mid = 0.5 * (lb + ub);
            lb = ub = mid;
        }
        c.lb[op] = lb;
        c.ub[op] = ub;
        if (updated) updated[op] = 1;
        if (prune) { // prune_within (src/filter.cpp:241-263)
            if (ub <= tau) {
                c.status[op] = TJ_CONFIRMED;
                c.decided_at[op] = stage;
                atomicAdd(c.num_confirmed + c.pair_r[op], 1u);
            } else if (lb > tau) {
                c.status[op] = TJ_REMOVED;
                c.decided_at[op] = stage;
            }
        }
    }
}


inline int grid_for(uint64_t items, int per_block, int num_sms) {
    const uint64_t g = (items + per_block - 1) / per_block;
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(g, (uint64_t)num_sms * 32));
}

int level_slot(const DatasetDev& d, uint32_t level) {
    for (size_t i = 0; i < d.levels.size(); ++i)
        if (d.levels[i] == (int32_t)level) return (int)i;
    return -1;
}

void check_error(DevError* err, cudaStream_t st) {
    DevError h;
    TJ_CUDA(cudaMemcpyAsync(&h, err, sizeof(DevError), cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    if (h.code == 0) return;
    if (h.kind == 1) throw Error(TJ_EENGINE, "knn_apply_deltas: confirmed count exceeds k");
    throw Error(TJ_EENGINE, "bound crossing: lb " + std::to_string(h.lb) + " > ub " + std::to_string(h.ub));
}

// ---- on-demand expansion of compact-resident levels (TJ_DATASET_COMPACT) ----

struct ReadU64 {
    const uint64_t* p;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return p[i]; }
};

__global__ void k_mark_voxels(const ActiveVpDev* __restrict__ act, uint64_t b, uint64_t e, uint8_t* __restrict__ fr,
                              uint8_t* __restrict__ fs) {
    for (uint64_t i = b + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e; i += (uint64_t)gridDim.x * blockDim.x) {
        const ActiveVpDev a = act[i];
        if (fr) fr[a.gvr] = 1;
        if (fs) fs[a.gvs] = 1;
    }
}

__global__ void k_flag_counts(const uint8_t* __restrict__ flag, const uint64_t* __restrict__ foff, uint64_t nv,
                              uint64_t* __restrict__ cnt) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * blockDim.x)
        cnt[v] = flag[v] ? foff[v + 1] - foff[v] : 0;
}

// Records needed to expand the voxels flagged in m (m.flag set by k_mark_voxels): m.off, m.total.
void mat_count(Workspace& ws, const DatasetDev& D, int slot, LevelMat& m, cudaStream_t st) {
    const uint64_t nv = D.n_voxels;
    m.cnt.reserve(std::max<uint64_t>(nv, 1));
    m.off.reserve(nv + 1);
    TJ_CUDA(cudaMemsetAsync(m.off.p, 0, 8, st));
    m.total = 0;
    if (!nv) return;
    count_launch();
    k_flag_counts<<<grid_for(nv, 256, ws.num_sms), 256, 0, st>>>(m.flag.p, D.facet_offsets[slot].p, nv, m.cnt.p);
    m.total = device_scan(ReadU64{m.cnt.p}, nv, m.off.p, ws.u64a, ws.num_sms, st);
}

// Expands the counted voxels and derives their screening records / segment aggregates.
void mat_expand(Workspace& ws, const DatasetDev& D, int slot, LevelMat& m, int zero_pad, cudaStream_t st) {
    const uint64_t n = m.total;
    m.facets.reserve(std::max<uint64_t>(n, 1) * TJ_FACET_STRIDE);
    m.screen.reserve(std::max<uint64_t>(n * kScreenRecF4, 1));
    m.seg.reserve(std::max<uint64_t>(3 * D.n_voxels, 1));
    m.agg.reserve(3);
    const unsigned init[3] = {0x7f800000u, 0u, 0u};
    TJ_CUDA(cudaMemcpyAsync(m.agg.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    expand_compact_level(D, (uint32_t)slot, m.off.p, m.facets.p, ws.num_sms, st);
    refine_prep(m.facets.p, n, m.screen.p, m.agg.p, ws.num_sms, st, zero_pad);
    refine_seg_prep(m.screen.p, m.off.p, D.n_voxels, m.seg.p, ws.num_sms, st);
    stream_sync(st); // the init above is a pageable-host copy
}

// Working-set budget for materialized levels: $TRIJOIN_WORKSET_MB, else 70 % of the device
// memory free when first needed (per context).
uint64_t workset_budget(Workspace& ws) {
    if (const char* e = std::getenv("TRIJOIN_WORKSET_MB"); e && *e)
        return std::max<uint64_t>(1, uint64_t(std::stod(e) * 1048576.0));
    if (ws.workset_budget) return ws.workset_budget;
    size_t free_b = 0, total_b = 0;
    TJ_CUDA(cudaMemGetInfo(&free_b, &total_b));
    return ws.workset_budget = std::max<uint64_t>(free_b / 10 * 7, 64ull << 20);
}

// Bytes a materialized record costs (FP64 record + FP32 screening record).
constexpr uint64_t kMatBytes = TJ_FACET_STRIDE * 8 + kScreenRecF4 * 16;

// The level arrays one side of a refinement pass reads: resident (expanded at upload) or
// materialized for the chunk of active voxel pairs [b, e).
struct SideLevel {
    const uint64_t* foff;
    const double* facets;
    const float4* box;
    const float4* geo;
    const float4* seg;
    const unsigned* agg;
};

SideLevel resident_side(const DatasetDev& D, int slot) {
    const uint64_t n = D.level_entries[slot];
    return {D.facet_offsets[slot].p, D.facets[slot].p, D.screen[slot].p, D.screen[slot].p + 3 * n, D.seg[slot].p,
            D.agg.p + 3 * slot};
}

SideLevel mat_side(const LevelMat& m) {
    return {m.off.p, m.facets.p, m.screen.p, m.screen.p + 3 * m.total, m.seg.p, m.agg.p};
}

// Splits the active voxel pairs [b, e) into chunks whose materialized records fit the
// working-set budget, materializing each in turn: fn(chunk begin, chunk end, R side, S side).
// Resident (non-compact) sides are used as they are.
template <class F>
void for_mat_chunks(Workspace& ws, const DatasetDev& R, int sr, const DatasetDev& S, int ss,
                    const ActiveVpDev* active, uint64_t b, uint64_t e, int zero_pad, cudaStream_t st, F&& fn) {
    const bool same = &R == &S;
    std::vector<std::pair<uint64_t, uint64_t>> todo{{b, e}};
    const uint64_t budget = workset_budget(ws);
    while (!todo.empty()) {
        const auto [cb, ce] = todo.back();
        todo.pop_back();
        if (ce <= cb) continue;
        LevelMat& mr = ws.mat[0];
        LevelMat& ms = same ? ws.mat[0] : ws.mat[1];
        if (R.compact) {
            mr.flag.reserve(std::max<uint64_t>(R.n_voxels, 1));
            TJ_CUDA(cudaMemsetAsync(mr.flag.p, 0, std::max<uint64_t>(R.n_voxels, 1), st));
        }
        if (S.compact && !same) {
            ms.flag.reserve(std::max<uint64_t>(S.n_voxels, 1));
            TJ_CUDA(cudaMemsetAsync(ms.flag.p, 0, std::max<uint64_t>(S.n_voxels, 1), st));
        }
        count_launch();
        k_mark_voxels<<<grid_for(ce - cb, 256, ws.num_sms), 256, 0, st>>>(active, cb, ce, R.compact ? mr.flag.p : nullptr,
                                                                          S.compact ? ms.flag.p : nullptr);
        TJ_CUDA(cudaGetLastError());
        uint64_t need = 0;
        if (R.compact) {
            mat_count(ws, R, sr, mr, st);
            need += mr.total;
        }
        if (S.compact && !same) {
            mat_count(ws, S, ss, ms, st);
            need += ms.total;
        }
        if (need * kMatBytes > budget && ce - cb > 1) { // too large: halves, first half first
            const uint64_t mid = cb + (ce - cb) / 2;
            todo.emplace_back(mid, ce);
            todo.emplace_back(cb, mid);
            continue;
        }
        if (R.compact) mat_expand(ws, R, sr, mr, zero_pad, st);
        if (S.compact && !same) mat_expand(ws, S, ss, ms, zero_pad, st);
        const SideLevel rs = R.compact ? mat_side(mr) : resident_side(R, sr);
        const SideLevel ss_ = S.compact ? mat_side(ms) : resident_side(S, ss);
        fn(cb, ce, rs, ss_);
    }
}

} // namespace

uint32_t tripwire_mask() {
    const char* e = std::getenv("TRIJOIN_TRIPWIRE_SAMPLE");
    const long v = e && *e ? std::atol(e) : 1024;
    if (v <= 0) return 0xffffffffu; // none
    uint32_t p = 1;
    while (p < (uint32_t)v && p < (1u << 30)) p <<= 1;
    return p - 1;
}

// erase_if of the decided ops' voxel pairs (src/refine.cpp:299-301): stable compaction of the
// active list (scan.cuh) into the workspace, copied back.
struct ActiveKeep {
    const ActiveVpDev* a;
    const uint8_t* status;
    __device__ __forceinline__ bool operator()(uint64_t i) const { return status[a[i].op] == TJ_UNDECIDED; }
};
struct ActiveEmit {
    const ActiveVpDev* a;
    ActiveVpDev* out;
    __device__ __forceinline__ void operator()(uint64_t i, uint64_t k) const { out[k] = a[i]; }
};

uint64_t compact_active(Workspace& ws, const CandDevStore& cs, DevBuf<ActiveVpDev>& active, uint64_t n,
                        cudaStream_t st) {
    if (n == 0) return 0;
    // scratch from the workspace (grow-only: no allocation between the levels of a join,
    // where a pool growth stalled the host for tens of milliseconds), result copied back
    ws.active_alt.reserve(n);
    const uint64_t h = device_select(ActiveKeep{active.p, cs.status.p}, ActiveEmit{active.p, ws.active_alt.p}, n,
                                     ws.u64a, st);
    if (h > 0)
        TJ_CUDA(cudaMemcpyAsync(active.p, ws.active_alt.p, (size_t)h * sizeof(ActiveVpDev), cudaMemcpyDeviceToDevice, st));
    return h;
}

// First active voxel pair (op order) whose op belongs to a query >= obj (ops are query-major:
// r2op[r] = the first op of query r).
__global__ void k_active_lower_bound(const ActiveVpDev* __restrict__ active, uint64_t n, const uint64_t* __restrict__ r2op,
                                     uint32_t nq, uint32_t obj, uint64_t* out) {
    if (threadIdx.x || blockIdx.x) return;
    if (obj >= nq) {
        *out = n;
        return;
    }
    const uint64_t op = r2op[obj];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (active[mid].op < op) lo = mid + 1;
        else hi = mid;
    }
    *out = lo;
}

RefineLoopOut refine_loop_dev(Workspace& ws, const DatasetDev& R, const DatasetDev& S, CandDevStore& cs,
                              DevBuf<ActiveVpDev>& active, uint64_t n_active, const tj_join_spec& spec, bool knn,
                              double tau, bool decision, DevError* err, TraceSink* trace, cudaStream_t st) {
    using Clock = std::chrono::steady_clock;
    RefineLoopOut out;
    const uint64_t n = cs.n;
    DevBuf<unsigned long long> lbb(std::max<uint64_t>(n, 1)), ubb(std::max<uint64_t>(n, 1));
    DevBuf<unsigned long long> counters(kNumCounters), work(1), dbg;
    DevBuf<uint64_t> piece_b(1);
    // k_screen launch timing (level stats screen_ms: bench.py's dominant-kernel roofline)
    std::vector<cudaEvent_t> sev_pool;
    size_t sev_used = 0;
    auto sev = [&]() -> cudaEvent_t* {
        if (sev_used + 2 > sev_pool.size())
            for (int k = 0; k < 2; ++k) {
                cudaEvent_t e;
                TJ_CUDA(cudaEventCreate(&e));
                sev_pool.push_back(e);
            }
        cudaEvent_t* p = sev_pool.data() + sev_used;
        sev_used += 2;
        return p;
    };
    Clock::time_point tdbg[4];
    static const bool dbg_timing = std::getenv("TRIJOIN_DEBUG_TIMING") != nullptr;
    if (const char* e = std::getenv("TRIJOIN_DEBUG_OPSTATS"); e && *e && *e != '0') dbg.alloc(std::max<uint64_t>(n, 1));
    if (!ws.queue) ws.queue = std::make_unique<RefineQueueStore>();
    RefineQueueStore& queue = *ws.queue;
    DevBuf<uint8_t> updated;
    if (trace && trace->on_interval) updated.alloc(std::max<uint64_t>(n, 1));
    cudaEvent_t e0, e1;
    TJ_CUDA(cudaEventCreate(&e0));
    TJ_CUDA(cudaEventCreate(&e1));
    // $TRIJOIN_DEBUG_TIMELINE: per level, device time the join stream waited for the level's data
    // (streamed datasets) and spent on it, printed to stderr (diagnostics)
    static const bool dbg_tl = std::getenv("TRIJOIN_DEBUG_TIMELINE") != nullptr;
    std::vector<cudaEvent_t> tl_ev;
    auto tl_mark = [&] {
        if (!dbg_tl) return;
        cudaEvent_t e;
        TJ_CUDA(cudaEventCreate(&e));
        TJ_CUDA(cudaEventRecord(e, st));
        tl_ev.push_back(e);
    };
    tl_mark();
    const unsigned long long kInfBits = 0x7ff0000000000000ull;
    const uint64_t launch = std::max<uint64_t>(spec.refine_chunk, 1ull << 24);
    uint64_t test_queue_cap = 0;
    if (const char* e = std::getenv("TRIJOIN_TEST_QUEUE_CAP"); e && *e) test_queue_cap = std::strtoull(e, nullptr, 10);
    try {
        for (uint32_t li = 0; li < spec.n_lods; ++li) {
            if (n_active == 0) break;
            const uint32_t level = spec.lods[li];
            const int sr = level_slot(R, level), ss = level_slot(S, level);
            const auto t0 = Clock::now();
            LevelStats ls{};
            ls.level = level;
            ls.vps = n_active;
            // streamed datasets: this level's facets may still be in flight
            tl_mark(); // level start (previous level done)
            // R's level arriving in object-range pieces (run_join's last level): S whole first,
            // then each query range's voxel pairs as soon as its piece is on the device
            const bool mat = R.compact || S.compact;
            const bool pieced = !mat && &S != &R && level_pieced(R, sr);
            ls.wait_ms = pieced ? 0.0 : level_ready(R, sr, st);
            if (&S != &R) ls.wait_ms += level_ready(S, ss, st);
            tl_mark(); // this level's data on the device
            RefineSource src{};
            src.active = active.p;
            src.exact_mask = decision ? tripwire_mask() : 0u;
            src.n_ops = (uint32_t)n;
            src.cand_lb = cs.lb.p;
            src.cand_ub = cs.ub.p;
            ws.level_agg.reserve(8);
            src.agg = ws.level_agg.p;
            {
                const uint64_t nr = R.level_entries[sr], ns = S.level_entries[ss];
                const double mr = R.n_voxels ? double(nr) / double(R.n_voxels) : 0.0;
                const double ms = S.n_voxels ? double(ns) / double(S.n_voxels) : 0.0;
                src.mean_seg = float(0.5 * (mr + ms));
            }
            // the level arrays of both sides: FP32 screening records, voxel segment aggregates
            // and level aggregates (derived once per dataset at upload: DatasetDev::screen / seg
            // / agg), or for compact-resident datasets expanded here for the voxels in use
            auto bind = [&](const SideLevel& rs, const SideLevel& ss_) {
                src.r_foff = rs.foff;
                src.s_foff = ss_.foff;
                src.r_facets = rs.facets;
                src.s_facets = ss_.facets;
                src.r_box = rs.box;
                src.r_geo = rs.geo;
                src.r_seg = rs.seg;
                src.s_box = ss_.box;
                src.s_geo = ss_.geo;
                src.s_seg = ss_.seg;
                count_launch();
                k_copy_agg<<<1, 32, 0, st>>>(rs.agg, ss_.agg, ws.level_agg.p);
            };
            if (!mat) bind(resident_side(R, sr), resident_side(S, ss));
            // 0: every facet pair; 1: exact-preserving culling; 2: decision-mode culling
            const int cull = (spec.flags & TJ_FLAG_NO_CULL) ? 0 : decision ? 2 : 1;
            unsigned long long hc[kNumCounters];
            if (dbg.n) {
                TJ_CUDA(cudaMemsetAsync(dbg.p, 0, n * 8, st));
                refine_debug_op_tested(dbg.p);
            }
            queue.cap = test_queue_cap;
            for (;;) {
                sev_used = 0;
                count_launch();
                k_fill_u64<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(lbb.p, n, kInfBits);
                count_launch();
                k_fill_u64<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(ubb.p, n, kInfBits);
                TJ_CUDA(cudaMemsetAsync(counters.p, 0, kNumCounters * 8, st));
                queue.reset(st);
                count_launch();
                k_facet_pairs<<<grid_for(n_active, 256, ws.num_sms), 256, 0, st>>>(
                    active.p, n_active, R.facet_offsets[sr].p, S.facet_offsets[ss].p, counters.p + 2);
                TJ_CUDA(cudaEventRecord(e0, st));
                if (pieced) {
                    // per piece: its queries' voxel pairs, seeds then screens (an op's voxel
                    // pairs all belong to its query, hence to one piece)
                    // Pieces are taken in batches: at least the next one (host-blocking until it
                    // is queued), plus every later one already queued; the batch's active-list
                    // boundaries cost one round trip, then its pieces' passes queue back to back
                    // (each behind its own piece's event), so the join stream never drains
                    // between pieces that were shipped together.
                    uint64_t a = 0;
                    for (size_t k = 0;;) {
                        std::vector<std::pair<uint32_t, cudaEvent_t>> batch;
                        uint32_t obj_end = 0;
                        const auto tw = Clock::now();
                        const cudaEvent_t pev = level_piece(R, sr, k, &obj_end);
                        ls.wait_ms += std::chrono::duration<double, std::milli>(Clock::now() - tw).count();
                        if (!pev) break;
                        batch.emplace_back(obj_end, pev);
                        for (;;) {
                            uint32_t oe = 0;
                            const cudaEvent_t e = level_piece_try(R, sr, k + batch.size(), &oe);
                            if (!e) break;
                            batch.emplace_back(oe, e);
                        }
                        piece_b.reserve(batch.size());
                        for (size_t i = 0; i < batch.size(); ++i) {
                            count_launch();
                            k_active_lower_bound<<<1, 32, 0, st>>>(active.p, n_active, cs.r2op.p, cs.nq, batch[i].first,
                                                                   piece_b.p + i);
                        }
                        std::vector<uint64_t> bnd(batch.size());
                        TJ_CUDA(cudaMemcpyAsync(bnd.data(), piece_b.p, batch.size() * 8, cudaMemcpyDeviceToHost, st));
                        stream_sync(st);
                        for (size_t i = 0; i < batch.size(); ++i) {
                            const uint64_t b = bnd[i];
                            TJ_CUDA(cudaStreamWaitEvent(st, batch[i].second, 0));
                            // R's level aggregates so far (pieces 0..i at least, k_prep's running
                            // min / max): a conservative bound for this piece's facets
                            count_launch();
                            k_copy_agg<<<1, 32, 0, st>>>(resident_side(R, sr).agg, resident_side(S, ss).agg,
                                                         ws.level_agg.p);
                            for (uint64_t c0 = a; cull && c0 < b; c0 += launch)
                                refine_pass(src, c0, std::min(b, c0 + launch), true, lbb.p, ubb.p, cull, queue, work.p,
                                            counters.p, ws.num_sms, st);
                            for (uint64_t c0 = a; c0 < b; c0 += launch)
                                refine_pass(src, c0, std::min(b, c0 + launch), false, lbb.p, ubb.p, cull, queue, work.p,
                                            counters.p, ws.num_sms, st, sev());
                            a = b;
                        }
                        k += batch.size();
                    }
                    if (a != n_active) throw Error(TJ_EINVAL, "join: the pieces of a level do not cover its queries");
                    level_ready(R, sr, st);
                } else if (!mat) {
                    // seeds for every voxel pair first (op thresholds), then the screened passes
                    if (cull)
                        for (uint64_t c0 = 0; c0 < n_active; c0 += launch)
                            refine_pass(src, c0, std::min(n_active, c0 + launch), true, lbb.p, ubb.p, cull, queue,
                                        work.p, counters.p, ws.num_sms, st);
                    for (uint64_t c0 = 0; c0 < n_active; c0 += launch)
                        refine_pass(src, c0, std::min(n_active, c0 + launch), false, lbb.p, ubb.p, cull, queue,
                                    work.p, counters.p, ws.num_sms, st, sev());
                } else {
                    // per materialized chunk: its seeds, then its screened pass (the op minima
                    // only tighten; a chunk screened before another's seeds skips fewer pairs,
                    // never a pair that matters)
                    for_mat_chunks(ws, R, sr, S, ss, active.p, 0, n_active, 0, st,
                                   [&](uint64_t cb, uint64_t ce, const SideLevel& rs, const SideLevel& ss_) {
                                       bind(rs, ss_);
                                       ++out.mat_chunks;
                                       for (uint64_t c0 = cb; c0 < ce; c0 += launch) {
                                           const uint64_t c1 = std::min(ce, c0 + launch);
                                           if (cull)
                                               refine_pass(src, c0, c1, true, lbb.p, ubb.p, cull, queue, work.p,
                                                           counters.p, ws.num_sms, st);
                                           refine_pass(src, c0, c1, false, lbb.p, ubb.p, cull, queue, work.p,
                                                       counters.p, ws.num_sms, st, sev());
                                       }
                                   });
                }
                TJ_CUDA(cudaEventRecord(e1, st));
                TJ_CUDA(cudaMemcpyAsync(hc, counters.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
                tdbg[0] = Clock::now();
                // an exact-evaluation (or stage-2 candidate) queue overflowed somewhere in the
                // level: grow it and redo the level (the screen is deterministic given the same
                // evaluations)
                const bool rerun = queue.grow_if_overflowed(st);
                tdbg[1] = Clock::now();
                if (!rerun) break;
                ++out.queue_reruns;
            }
            out.chunks += (n_active + spec.refine_chunk - 1) / spec.refine_chunk;
            if (dbg.n) refine_debug_op_tested(nullptr);
            count_launch();
            k_aggregate<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(cs.view(), n, lbb.p, ubb.p, knn ? 0 : 1, tau,
                                                                      (int16_t)level, cull == 2 ? 1 : 0,
                                                                      src.exact_mask, updated.p,
                                                                      err);
            TJ_CUDA(cudaGetLastError());
            check_error(err, st);
            tdbg[2] = Clock::now();
            if (trace && trace->on_interval) trace->emit_updated(cs, updated, (int16_t)level, st);
            if (knn) {
                knn_fixpoint(ws, cs, spec.k, (int16_t)level, err, st);
                check_error(err, st);
            }
            if (dbg.n) { // tested pairs by the op's outcome at this level
                std::vector<unsigned long long> t(n);
                std::vector<uint8_t> sts(n);
                std::vector<int16_t> at(n);
                TJ_CUDA(cudaMemcpyAsync(t.data(), dbg.p, n * 8, cudaMemcpyDeviceToHost, st));
                TJ_CUDA(cudaMemcpyAsync(sts.data(), cs.status.p, n, cudaMemcpyDeviceToHost, st));
                TJ_CUDA(cudaMemcpyAsync(at.data(), cs.decided_at.p, n * 2, cudaMemcpyDeviceToHost, st));
                stream_sync(st);
                unsigned long long conf = 0, rem = 0, und = 0, nconf = 0, nrem = 0, nund = 0;
                for (uint64_t op = 0; op < n; ++op) {
                    if (!t[op]) continue;
                    if (sts[op] == TJ_UNDECIDED) { und += t[op]; ++nund; }
                    else if (at[op] == (int16_t)level && sts[op] == TJ_CONFIRMED) { conf += t[op]; ++nconf; }
                    else if (at[op] == (int16_t)level) { rem += t[op]; ++nrem; }
                }
                std::fprintf(stderr, "[opstats] lod %u tested: confirmed-here %llu (%llu ops) removed-here %llu (%llu ops) undecided %llu (%llu ops)\n",
                             level, conf, nconf, rem, nrem, und, nund);
            }
            float kms = 0.f;
            TJ_CUDA(cudaEventElapsedTime(&kms, e0, e1));
            ls.tested = hc[0];
            ls.evaluated = hc[1];
            ls.facet_pairs = hc[2];
            ls.screened = hc[3];
            ls.verified = hc[4];
            ls.vps_skipped = hc[5];
            ls.facets_dropped = hc[6];
            ls.kernel_ms = kms;
            for (size_t k = 0; k + 1 < sev_used; k += 2) {
                float m = 0.f;
                TJ_CUDA(cudaEventElapsedTime(&m, sev_pool[k], sev_pool[k + 1]));
                ls.screen_ms += m;
            }
            tdbg[3] = Clock::now();
            n_active = compact_active(ws, cs, active, n_active, st);
            if (dbg_timing) {
                const auto ms = [](Clock::time_point a, Clock::time_point b) {
                    return std::chrono::duration<double, std::milli>(b - a).count();
                };
                std::fprintf(stderr, "[timing] lod %u: to-sync %.1f sync %.1f agg %.1f mid %.1f compact %.1f\n", level,
                             ms(t0, tdbg[0]), ms(tdbg[0], tdbg[1]), ms(tdbg[1], tdbg[2]), ms(tdbg[2], tdbg[3]),
                             ms(tdbg[3], Clock::now()));
            }

            ls.ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
            out.levels.push_back(ls);
        }
    } catch (...) {
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        throw;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (cudaEvent_t e : sev_pool) cudaEventDestroy(e);
    if (dbg_tl && !tl_ev.empty()) {
        tl_mark();
        TJ_CUDA(cudaEventSynchronize(tl_ev.back()));
        std::string line = "[timeline] refine from t0 (ms):";
        for (size_t i = 1; i < tl_ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tl_ev[0], tl_ev[i]);
            char b[32];
            std::snprintf(b, sizeof(b), " %.2f", ms);
            line += b;
        }
        std::fprintf(stderr, "%s\n", line.c_str());
        std::string cl = "[timeline] copy streams from t0 (ms):";
        for (auto& [what, e] : take_copy_marks()) {
            float ms = 0.f;
            if (cudaEventSynchronize(e) == cudaSuccess && cudaEventElapsedTime(&ms, tl_ev[0], e) == cudaSuccess) {
                char b[64];
                std::snprintf(b, sizeof(b), " %s=%.2f", what.c_str(), ms);
                cl += b;
            }
            cudaEventDestroy(e);
        }
        std::fprintf(stderr, "%s\n", cl.c_str());
        for (cudaEvent_t e : tl_ev) cudaEventDestroy(e);
    }
    return out;
}

namespace {

__global__ void k_exact_counts(CandDev c, uint64_t n, const uint64_t* __restrict__ r_voff,
                               const uint64_t* __restrict__ s_voff, uint32_t* __restrict__ counts) {
    for (uint64_t op = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; op < n; op += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t cnt = 0;
        if (c.status[op] == TJ_CONFIRMED) {
            const uint32_t r = c.pair_r[op], s = c.pair_s[op];
            cnt = (uint32_t)((r_voff[r + 1] - r_voff[r]) * (s_voff[s + 1] - s_voff[s]));
        }
        counts[op] = cnt;
    }
}

// Warp per confirmed op: every voxel pair (i, j) of its two objects.
__global__ void k_exact_emit(CandDev c, uint64_t n, const uint64_t* __restrict__ offsets,
                             const uint64_t* __restrict__ r_voff, const uint64_t* __restrict__ s_voff,
                             ActiveVpDev* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    for (uint64_t op = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; op < n; op += warps) {
        if (c.status[op] != TJ_CONFIRMED) continue;
        const uint32_t r = c.pair_r[op], s = c.pair_s[op];
        const uint64_t vr0 = r_voff[r], vs0 = s_voff[s], ns = s_voff[s + 1] - vs0;
        const uint64_t total = (r_voff[r + 1] - vr0) * ns, base = offsets[op];
        for (uint64_t t = lane; t < total; t += 32)
            out[base + t] = {(uint32_t)op, (uint32_t)(vr0 + t / ns), (uint32_t)(vs0 + t % ns)};
    }
}

__global__ void k_exact_store(CandDev c, uint64_t n, const unsigned long long* __restrict__ dbits) {
    for (uint64_t op = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; op < n; op += (uint64_t)gridDim.x * blockDim.x) {
        if (c.status[op] != TJ_CONFIRMED) continue;
        const double d = __longlong_as_double((long long)dbits[op]);
        c.lb[op] = d;
        c.ub[op] = d;
    }
}

} // namespace

// --exact (reference recompute_exact, src/engine.cpp:96-118): for every confirmed pair the
// minimum tri_tri_distance over all facet pairs of the two level-100 meshes (TriBvh::
// pair_distance is that minimum). On the device it is one more level-100 pass over every
// voxel pair of the confirmed pairs (the level-100 voxel lists partition the mesh facets),
// with the paddings ignored and the same exact-preserving culling against the op minima.
void exact_recompute_dev(Workspace& ws, const DatasetDev& R, const DatasetDev& S, CandDevStore& cs, cudaStream_t st) {
    const uint64_t n = cs.n;
    if (n == 0) return;
    const int sr = level_slot(R, 100), ss = level_slot(S, 100);
    if (sr < 0 || ss < 0) throw Error(TJ_EENGINE, "refine: level 100 is not in the dataset's lod schedule");
    level_ready(R, sr, st);
    if (&S != &R) level_ready(S, ss, st);
    DevBuf<uint32_t> counts(n);
    count_launch();
    k_exact_counts<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(cs.view(), n, R.voxel_offsets.p, S.voxel_offsets.p,
                                                                 counts.p);
    DevBuf<uint64_t> offsets;
    const uint64_t total = scan_counts(ws, counts.p, n, offsets, st);
    if (total == 0) return;
    DevBuf<ActiveVpDev> active(total);
    count_launch();
    k_exact_emit<<<grid_for(n * 32, 256, ws.num_sms), 256, 0, st>>>(cs.view(), n, offsets.p, R.voxel_offsets.p,
                                                                     S.voxel_offsets.p, active.p);
    DevBuf<double> iv_lb(n), iv_ub(n);
    DevBuf<unsigned long long> lbb(n), ubb(n), counters(kNumCounters), work(1);
    const unsigned long long kInfBits = 0x7ff0000000000000ull;
    TJ_CUDA(cudaMemsetAsync(iv_lb.p, 0, n * 8, st));
    count_launch();
    k_fill_u64<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(reinterpret_cast<unsigned long long*>(iv_ub.p), n,
                                                              kInfBits);
    RefineSource src{};
    src.active = active.p;
    src.cand_lb = iv_lb.p;
    src.cand_ub = iv_ub.p;
    src.zero_pad = 1;
    if (!ws.queue) ws.queue = std::make_unique<RefineQueueStore>();
    RefineQueueStore& queue = *ws.queue;
    queue.cap = 0;
    if (const char* e = std::getenv("TRIJOIN_TEST_QUEUE_CAP"); e && *e) queue.cap = std::strtoull(e, nullptr, 10);
    const uint64_t launch = 1ull << 20;
    auto passes = [&](uint64_t b, uint64_t e) {
        for (uint64_t c0 = b; c0 < e; c0 += launch)
            refine_pass(src, c0, std::min(e, c0 + launch), true, lbb.p, ubb.p, 1, queue, work.p, counters.p,
                        ws.num_sms, st);
        for (uint64_t c0 = b; c0 < e; c0 += launch)
            refine_pass(src, c0, std::min(e, c0 + launch), false, lbb.p, ubb.p, 1, queue, work.p, counters.p,
                        ws.num_sms, st);
    };
    const bool mat = R.compact || S.compact;
    if (!mat) {
        src.r_foff = R.facet_offsets[sr].p;
        src.s_foff = S.facet_offsets[ss].p;
        src.r_facets = R.facets[sr].p;
        src.s_facets = S.facets[ss].p;
        const uint64_t nr = R.level_entries[sr], ns = S.level_entries[ss];
        ws.screen_r.reserve(std::max<uint64_t>(nr * kScreenRecF4, 1));
        refine_prep(R.facets[sr].p, nr, ws.screen_r.p, nullptr, ws.num_sms, st, 1);
        src.r_box = ws.screen_r.p;
        src.r_geo = ws.screen_r.p + 3 * nr;
        ws.seg_r.reserve(std::max<uint64_t>(3 * R.n_voxels, 1));
        refine_seg_prep(src.r_box, R.facet_offsets[sr].p, R.n_voxels, ws.seg_r.p, ws.num_sms, st);
        src.r_seg = ws.seg_r.p;
        if (S.facets[ss].p == R.facets[sr].p) {
            src.s_box = src.r_box;
            src.s_geo = src.r_geo;
            src.s_seg = src.r_seg;
        } else {
            ws.screen_s.reserve(std::max<uint64_t>(ns * kScreenRecF4, 1));
            refine_prep(S.facets[ss].p, ns, ws.screen_s.p, nullptr, ws.num_sms, st, 1);
            src.s_box = ws.screen_s.p;
            src.s_geo = ws.screen_s.p + 3 * ns;
            ws.seg_s.reserve(std::max<uint64_t>(3 * S.n_voxels, 1));
            refine_seg_prep(src.s_box, S.facet_offsets[ss].p, S.n_voxels, ws.seg_s.p, ws.num_sms, st);
            src.s_seg = ws.seg_s.p;
        }
    }
    for (;;) {
        count_launch();
        k_fill_u64<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(lbb.p, n, kInfBits);
        count_launch();
        k_fill_u64<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(ubb.p, n, kInfBits);
        queue.reset(st);
        if (!mat) {
            passes(0, total);
        } else { // compact-resident: expand the level-100 voxels of the confirmed pairs chunk by chunk
            for_mat_chunks(ws, R, sr, S, ss, active.p, 0, total, 1, st,
                           [&](uint64_t cb, uint64_t ce, const SideLevel& rs, const SideLevel& ss_) {
                               src.r_foff = rs.foff;
                               src.s_foff = ss_.foff;
                               src.r_facets = rs.facets;
                               src.s_facets = ss_.facets;
                               src.r_box = rs.box;
                               src.r_geo = rs.geo;
                               src.r_seg = rs.seg;
                               src.s_box = ss_.box;
                               src.s_geo = ss_.geo;
                               src.s_seg = ss_.seg;
                               passes(cb, ce);
                           });
        }
        if (!queue.grow_if_overflowed(st)) break;
    }
    count_launch();
    k_exact_store<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(cs.view(), n, lbb.p);
    TJ_CUDA(cudaGetLastError());
}

} // namespace tjx
