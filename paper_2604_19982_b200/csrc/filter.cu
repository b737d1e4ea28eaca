// Filter stages on sm_100a.
//
//  * MBB object filter (reference mbb_filter_within / mbb_filter_knn,
//    src/filter.cpp:88-190 + finalize_candidate_set :48-84). The reference walks an
//    STR R-tree; its pruning is exact (node boxes contain their entries and the FP gap
//    is monotone), so its output is exactly {s : mindist(mbb_r, mbb_s) <= tau}. Here
//    S is sorted by mbb.min.x once and each query scans the x-window that can contain
//    such s, applying the reference's exact FP64 mindist test. For k-NN the reference's
//    best-first search returns exactly {s : mindist <= u_k(r)} with u_k(r) the k-th
//    smallest anchor distance over all of S; u_k is a warp-level
//    k-selection, then the same window scan runs with a per-query threshold.
//  * Voxel-pair filter (reference voxel_pair_bounds / prune_within / voxel_pair_compact /
//    chunked_filter, src/filter.cpp:199-448, paper Alg. 1-3), fused: one warp per
//    candidate computes the n_r x n_s box/anchor bounds, their minima, the interval
//    intersection and the within-tau prune, and counts survivors; a scan gives offsets;
//    a second pass recomputes the (cheap) box bound and scatters survivors stably in the
//    reference's (op, i, j) row-major order. The per-voxel-pair arrays the reference
//    materialises are never written: recomputation is cheaper than the HBM round trip.
#include <cub/cub.cuh>

#include "filter.cuh"
#include "scan.cuh"
#include "geom_exact.cuh"

namespace tjx {

namespace {

__device__ __forceinline__ bool participates(uint32_t r, uint32_t idx, uint32_t cnt, uint32_t blk) {
    return cnt <= 1 || (r / blk) % cnt == idx;
}

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000ll); }

__global__ void k_minx_keys(const double* __restrict__ mbb, uint32_t n, double* keys, uint32_t* vals) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        keys[i] = mbb[6 * i];
        vals[i] = i;
    }
}

__global__ void k_gather_sorted(const double* __restrict__ mbb, const uint32_t* __restrict__ order, uint32_t n,
                                double* __restrict__ out, float4* __restrict__ yz, unsigned long long* max_ext_bits) {
    unsigned long long local = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double* m = mbb + 6 * (size_t)order[i];
#pragma unroll
        for (int k = 0; k < 6; ++k) out[6 * (size_t)i + k] = m[k];
        yz[i] = make_float4(__double2float_rd(m[1]), __double2float_ru(m[4]), __double2float_rd(m[2]),
                            __double2float_ru(m[5]));
        const double ext = m[3] - m[0];
        const unsigned long long b = (unsigned long long)__double_as_longlong(ext > 0.0 ? ext : 0.0);
        local = b > local ? b : local;
    }
    atomicMax(max_ext_bits, local);
}

// First index i in [0, n) with pred(i) false, for a monotone (true...false) predicate.
template <class P>
__device__ __forceinline__ uint32_t partition_point(uint32_t n, P pred) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (pred(mid)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct Window {
    uint32_t lo, hi;
};

// x-window of sorted S that may hold s with mindist(mbb_r, mbb_s) <= tau.
__device__ __forceinline__ Window mbb_window(const double* rb, double tau, const double* __restrict__ smbb, uint32_t ns,
                                             double max_ext) {
    if (!(tau < dinf())) return {0u, ns};
    // gx >= fl(s.min.x - r.max.x), and mindist >= gx whenever gx > 1e-150 (no underflow in
    // gx*gx, sqrt(fl(x*x)) == |x|): s beyond hi have gx > tau' >= tau, hence mindist > tau.
    const double taup = tau > 1e-150 ? tau : 1e-150;
    const double rmaxx = rb[3];
    const uint32_t hi = partition_point(ns, [&](uint32_t i) { return (smbb[6 * (size_t)i] - rmaxx) <= taup; });
    // s below lo have s.max.x <= s.min.x + max_ext < r.min.x - tau', so gx > tau'.
    const double margin = 1e-9 * (1.0 + fabs(rb[0]) + max_ext + taup);
    const double lim = rb[0] - taup - max_ext - margin;
    const uint32_t lo = partition_point(hi, [&](uint32_t i) { return smbb[6 * (size_t)i] < lim; });
    return {lo, hi};
}

__device__ __forceinline__ double query_tau(const MbbArgs& a, uint32_t r) {
    return a.tau_per_r ? a.tau_per_r[r] : a.tau;
}

// FP32 pre-rejection of sorted S entries on their y / z gaps to a query box (the x window
// is mbb_window's). Rejects only if a rounded-down gap exceeds tau (1 + 2^-20) (rounded up,
// at least 1e-30): the true gap then exceeds tau, so does its FP64 rounding, and mindist_box
// (>= that rounded gap: sqrt(fl(g*g)) == g without underflow) cannot be <= tau.
struct YzReject {
    float ylo, yhi, zlo, zhi, t;
    bool on;
    __device__ YzReject(const MbbArgs& a, const double* rb, double tau) {
        on = a.s_sorted_yz != nullptr;
        ylo = __double2float_rd(rb[1]);
        yhi = __double2float_ru(rb[4]);
        zlo = __double2float_rd(rb[2]);
        zhi = __double2float_ru(rb[5]);
        t = fmaxf(__double2float_ru(tau * (1.0 + 0x1p-20)), 1e-30f);
    }
    __device__ __forceinline__ bool operator()(const MbbArgs& a, uint32_t i) const {
        if (!on) return false;
        const float4 s = __ldg(a.s_sorted_yz + i);
        const float gy = fmaxf(__fsub_rd(s.x, yhi), __fsub_rd(ylo, s.y));
        const float gz = fmaxf(__fsub_rd(s.z, zhi), __fsub_rd(zlo, s.w));
        return gy > t || gz > t;
    }
};

__global__ void k_mbb_count(MbbArgs a, uint32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.nr; r += warps) {
        uint32_t c = 0;
        if (participates(r, a.shard_index, a.shard_count, a.shard_block) && a.ns > 0) {
            const double* rb = a.r_mbb + 6 * (size_t)r;
            const double tau = query_tau(a, r);
            const Window w = mbb_window(rb, tau, a.s_sorted_mbb, a.ns, a.max_ext);
            const YzReject reject(a, rb, tau);
            for (uint32_t i = w.lo + lane; i < w.hi; i += 32)
                if (!reject(a, i)) c += mindist_box(rb, a.s_sorted_mbb + 6 * (size_t)i) <= tau ? 1u : 0u;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) counts[r] = c;
    }
}

__global__ void k_mbb_fill(MbbArgs a, const uint64_t* __restrict__ offsets, uint32_t* __restrict__ pair_r,
                           uint32_t* __restrict__ pair_s) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.nr; r += warps) {
        uint64_t pos = offsets[r];
        if (offsets[r + 1] == pos) continue;
        const double* rb = a.r_mbb + 6 * (size_t)r;
        const double tau = query_tau(a, r);
        const Window w = mbb_window(rb, tau, a.s_sorted_mbb, a.ns, a.max_ext);
        const YzReject reject(a, rb, tau);
        for (uint32_t base = w.lo; base < w.hi; base += 32) {
            const uint32_t i = base + lane;
            const bool keep = i < w.hi && !reject(a, i) && mindist_box(rb, a.s_sorted_mbb + 6 * (size_t)i) <= tau;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint64_t o = pos + __popc(bal & ((1u << lane) - 1u));
                pair_r[o] = r;
                pair_s[o] = a.s_order[i];
            }
            pos += __popc(bal);
        }
    }
}

__global__ void k_mbb_finalize(MbbArgs a, uint64_t n, const uint32_t* __restrict__ pair_r,
                               const uint32_t* __restrict__ pair_s, CandDev c) {
    for (uint64_t op = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; op < n; op += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = pair_r[op], s = pair_s[op];
        const double lb = mindist_box(a.r_mbb + 6 * (size_t)r, a.s_mbb + 6 * (size_t)s);
        const double ub = point_dist(a.r_anchor + 3 * (size_t)r, a.s_anchor + 3 * (size_t)s);
        c.lb[op] = lb;
        c.ub[op] = ub;
        c.pair_r[op] = r;
        c.pair_s[op] = s;
        uint8_t st = TJ_UNDECIDED;
        int16_t at = TJ_STAGE_NONE;
        if (a.confirm_at_mbb && ub <= a.tau) { // within: ub <= tau confirms (src/filter.cpp:112)
            st = TJ_CONFIRMED;
            at = TJ_STAGE_MBB;
            atomicAdd(c.num_confirmed + r, 1u);
        }
        c.status[op] = st;
        c.decided_at[op] = at;
    }
}

// k-th smallest anchor distance over all of S for each participating query (k-NN).
// One warp per query; candidates below the running threshold accumulate in a shared
// buffer that is bitonic-sorted and truncated to k whenever it fills.
__global__ void k_knn_kth(MbbArgs a, uint32_t k, uint32_t cap, double* __restrict__ u_k) {
    extern __shared__ double kbuf_all[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    double* buf = kbuf_all + (size_t)wib * cap;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.nr; r += warps) {
        if (!participates(r, a.shard_index, a.shard_count, a.shard_block)) {
            if (lane == 0) u_k[r] = 0.0;
            continue;
        }
        const double* ra = a.r_anchor + 3 * (size_t)r;
        double theta = dinf();
        uint32_t cnt = 0;
        auto sort_truncate = [&]() {
            for (uint32_t i = cnt + lane; i < cap; i += 32) buf[i] = dinf();
            __syncwarp();
            for (uint32_t size = 2; size <= cap; size <<= 1) {
                for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                    for (uint32_t i = lane; i < cap; i += 32) {
                        const uint32_t j = i ^ stride;
                        if (j > i) {
                            const bool up = (i & size) == 0;
                            const double x = buf[i], y = buf[j];
                            if ((x > y) == up) { buf[i] = y; buf[j] = x; }
                        }
                    }
                    __syncwarp();
                }
            }
            if (cnt >= k) {
                theta = buf[k - 1];
                cnt = k;
            }
        };
        for (uint32_t base = 0; base < a.ns; base += 32) {
            const uint32_t s = base + lane;
            double d = dinf();
            if (s < a.ns) d = point_dist(ra, a.s_anchor + 3 * (size_t)s);
            const bool keep = s < a.ns && d < theta;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (cnt + 32 > cap) {
                sort_truncate();
            }
            if (keep) buf[cnt + __popc(bal & ((1u << lane) - 1u))] = d;
            cnt += __popc(bal);
            __syncwarp();
        }
        sort_truncate();
        if (lane == 0) u_k[r] = (a.ns >= k) ? buf[k - 1] : dinf();
        __syncwarp();
    }
}

// ---- voxel-pair filter ----

__device__ __forceinline__ void intersect_dev(double& lb, double& ub, double nlb, double nub, uint32_t op,
                                              DevError* err) {
    // intersect_interval (src/filter.cpp:22-32)
    lb = (lb < nlb) ? nlb : lb;
    ub = (nub < ub) ? nub : ub;
    if (lb > ub) {
        if (lb - ub > 1e-9) {
            if (atomicMin(&err->op, op) > op) {
                err->lb = lb; // best effort: the lowest op's values win most races
                err->ub = ub;
            }
            err->kind = 0;
            atomicExch(&err->code, (int)TJ_EENGINE);
        }
        const double mid = 0.5 * (lb + ub);
        lb = ub = mid;
    }
}

__global__ void k_vf_bounds(VoxelArgs a, CandDev c, uint32_t* __restrict__ surv, unsigned long long* __restrict__ stats,
                            uint8_t* __restrict__ touched) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long gen = 0, pruned = 0;
    for (uint64_t op = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; op < a.n_cands; op += warps) {
        uint32_t cnt = 0;
        if (c.status[op] == TJ_UNDECIDED) {
            const uint32_t r = c.pair_r[op], s = c.pair_s[op];
            const uint64_t vr0 = a.r_voff[r], nr = a.r_voff[r + 1] - vr0;
            const uint64_t vs0 = a.s_voff[s], ns = a.s_voff[s + 1] - vs0;
            const uint64_t total = nr * ns;
            double mlb = dinf(), mub = dinf();
            for (uint64_t t = lane; t < total; t += 32) {
                const uint64_t i = t / ns, j = t - i * ns; // decode_pair (parcore.hpp:23-25)
                const double lb = mindist_box(a.r_vbox + 6 * (vr0 + i), a.s_vbox + 6 * (vs0 + j));
                const double ub = point_dist(a.r_vanc + 3 * (vr0 + i), a.s_vanc + 3 * (vs0 + j));
                mlb = (lb < mlb) ? lb : mlb;
                mub = (ub < mub) ? ub : mub;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double x = __shfl_xor_sync(0xffffffffu, mlb, o);
                const double y = __shfl_xor_sync(0xffffffffu, mub, o);
                mlb = (x < mlb) ? x : mlb;
                mub = (y < mub) ? y : mub;
            }
            double lb = c.lb[op], ub = c.ub[op];
            intersect_dev(lb, ub, mlb, mub, (uint32_t)op, a.err);
            uint8_t st = TJ_UNDECIDED;
            if (a.prune) { // prune_within (src/filter.cpp:241-263) at stage voxel
                if (ub <= a.tau) st = TJ_CONFIRMED;
                else if (lb > a.tau) st = TJ_REMOVED;
            }
            if (st == TJ_UNDECIDED) {
                for (uint64_t t = lane; t < total; t += 32) {
                    const uint64_t i = t / ns, j = t - i * ns;
                    cnt += mindist_box(a.r_vbox + 6 * (vr0 + i), a.s_vbox + 6 * (vs0 + j)) <= ub ? 1u : 0u;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            }
            if (lane == 0) {
                c.lb[op] = lb;
                c.ub[op] = ub;
                if (touched) touched[op] = 1;
                if (st != TJ_UNDECIDED) {
                    c.status[op] = st;
                    c.decided_at[op] = TJ_STAGE_VOXEL;
                    if (st == TJ_CONFIRMED) atomicAdd(c.num_confirmed + r, 1u);
                }
                gen += total;
                if (st == TJ_UNDECIDED) pruned += total - cnt;
            }
        }
        if (lane == 0) surv[op] = cnt;
    }
    if (lane == 0) {
        atomicAdd(stats + 0, gen);
        atomicAdd(stats + 1, pruned);
    }
}

// Stable scatter of surviving voxel pairs in (op, i, j) order. keep_pruned selects the
// complement (trace slow path, reference on_vp_pruned order).
template <bool kPruned>
__global__ void k_vf_scatter(VoxelArgs a, CandDev c, const uint64_t* __restrict__ offsets, ActiveVpDev* __restrict__ out,
                             double* __restrict__ out_lb) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    for (uint64_t op = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; op < a.n_cands; op += warps) {
        uint64_t pos = offsets[op];
        if (offsets[op + 1] == pos) continue;
        const uint32_t r = c.pair_r[op], s = c.pair_s[op];
        const uint64_t vr0 = a.r_voff[r], nr = a.r_voff[r + 1] - vr0;
        const uint64_t vs0 = a.s_voff[s], ns = a.s_voff[s + 1] - vs0;
        const uint64_t total = nr * ns;
        const double ub = c.ub[op];
        for (uint64_t base = 0; base < total; base += 32) {
            const uint64_t t = base + lane;
            bool keep = false;
            double lbv = 0.0;
            uint64_t i = 0, j = 0;
            if (t < total) {
                i = t / ns;
                j = t - i * ns;
                lbv = mindist_box(a.r_vbox + 6 * (vr0 + i), a.s_vbox + 6 * (vs0 + j));
                keep = kPruned ? !(lbv <= ub) : (lbv <= ub);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint64_t o = pos + __popc(bal & ((1u << lane) - 1u));
                if (kPruned) {
                    out[o] = {(uint32_t)op, (uint32_t)i, (uint32_t)j};
                    out_lb[o] = lbv;
                } else {
                    out[o] = {(uint32_t)op, (uint32_t)(vr0 + i), (uint32_t)(vs0 + j)};
                }
            }
            pos += __popc(bal);
        }
    }
}

__global__ void k_pruned_count(VoxelArgs a, CandDev c, const uint8_t* __restrict__ touched,
                               const uint32_t* __restrict__ surv, uint32_t* __restrict__ out) {
    for (uint64_t op = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; op < a.n_cands;
         op += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t n = 0;
        if (touched[op] && c.status[op] == TJ_UNDECIDED) {
            const uint32_t r = c.pair_r[op], s = c.pair_s[op];
            const uint64_t nr = a.r_voff[r + 1] - a.r_voff[r], ns = a.s_voff[s + 1] - a.s_voff[s];
            n = (uint32_t)(nr * ns) - surv[op];
        }
        out[op] = n;
    }
}

template <class T>
__global__ void k_widen(const T* __restrict__ in, uint64_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

inline int grid_for(uint64_t items, int per_block, int num_sms) {
    const uint64_t g = (items + per_block - 1) / per_block;
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(g, (uint64_t)num_sms * 32));
}

} // namespace

struct ReadU32 {
    const uint32_t* p;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return p[i]; }
};

// Exclusive scan of n u32 counts into n+1 u64 offsets (offsets[n] = total): scan.cuh.
uint64_t scan_counts(Workspace& ws, const uint32_t* counts, uint64_t n, DevBuf<uint64_t>& offsets, cudaStream_t st) {
    offsets.reserve(n + 1);
    return device_scan(ReadU32{counts}, n, offsets.p, ws.u64a, ws.num_sms, st);
}

void mbb_prepare_s(Workspace& ws, const DatasetDev& S, SortedS& out, cudaStream_t st) {
    const uint32_t ns = S.n_objects;
    out.order.reserve(std::max<uint32_t>(ns, 1));
    out.mbb.reserve(std::max<uint64_t>(6ull * ns, 1));
    out.max_ext = 0.0;
    if (ns == 0) return;
    DevBuf<double> keys(ns), keys_out(ns);
    DevBuf<uint32_t> vals(ns);
    count_launch();
    k_minx_keys<<<grid_for(ns, 256, ws.num_sms), 256, 0, st>>>(S.mbb.p, ns, keys.p, vals.p);
    size_t bytes = 0;
    TJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys_out.p, vals.p, out.order.p, (int)ns, 0, 64, st));
    ws.temp.reserve(bytes);
    TJ_CUDA(cub::DeviceRadixSort::SortPairs(ws.temp.p, bytes, keys.p, keys_out.p, vals.p, out.order.p, (int)ns, 0, 64, st));
    DevBuf<unsigned long long> ext(1);
    TJ_CUDA(cudaMemsetAsync(ext.p, 0, sizeof(unsigned long long), st));
    count_launch();
    out.yz.reserve(ns);
    k_gather_sorted<<<grid_for(ns, 256, ws.num_sms), 256, 0, st>>>(S.mbb.p, out.order.p, ns, out.mbb.p, out.yz.p, ext.p);
    unsigned long long bits = 0;
    TJ_CUDA(cudaMemcpyAsync(&bits, ext.p, 8, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    double e;
    memcpy(&e, &bits, 8);
    out.max_ext = e;
}

void knn_kth_anchor(Workspace& ws, const MbbArgs& a, uint32_t k, DevBuf<double>& u_k, cudaStream_t st) {
    u_k.reserve(std::max<uint32_t>(a.nr, 1));
    if (a.nr == 0) return;
    uint32_t cap = 64;
    while (cap < 2 * k + 32) cap <<= 1;
    const int warps_per_block = cap <= 512 ? 4 : 1;
    const size_t smem = (size_t)cap * sizeof(double) * warps_per_block;
    if (smem > 48 * 1024)
        TJ_CUDA(cudaFuncSetAttribute(k_knn_kth, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = grid_for((uint64_t)a.nr * 32, 32 * warps_per_block, ws.num_sms);
    count_launch();
    k_knn_kth<<<grid, 32 * warps_per_block, smem, st>>>(a, k, cap, u_k.p);
    TJ_CUDA(cudaGetLastError());
}

uint64_t mbb_candidates(Workspace& ws, const MbbArgs& a, CandDevStore& cs, cudaStream_t st) {
    const uint32_t nr = a.nr;
    DevBuf<uint32_t> counts(std::max<uint32_t>(nr, 1));
    count_launch();
    k_mbb_count<<<grid_for((uint64_t)nr * 32, 256, ws.num_sms), 256, 0, st>>>(a, counts.p);
    TJ_CUDA(cudaGetLastError());
    const uint64_t n = scan_counts(ws, counts.p, nr, cs.r2op, st);
    cs.resize(n, nr);
    DevBuf<uint32_t> pr(std::max<uint64_t>(n, 1)), ps(std::max<uint64_t>(n, 1));
    if (n > 0) {
        count_launch();
        k_mbb_fill<<<grid_for((uint64_t)nr * 32, 256, ws.num_sms), 256, 0, st>>>(a, cs.r2op.p, pr.p, ps.p);
        TJ_CUDA(cudaGetLastError());
        // sort each query's candidates by s (finalize_candidate_set, src/filter.cpp:65-66)
        DevBuf<uint32_t> ps_sorted(n);
        size_t bytes = 0;
        TJ_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, ps.p, ps_sorted.p, (int64_t)n, (int64_t)nr,
                                                   cs.r2op.p, cs.r2op.p + 1, st));
        ws.temp.reserve(bytes);
        TJ_CUDA(cub::DeviceSegmentedSort::SortKeys(ws.temp.p, bytes, ps.p, ps_sorted.p, (int64_t)n, (int64_t)nr,
                                                   cs.r2op.p, cs.r2op.p + 1, st));
        TJ_CUDA(cudaMemsetAsync(cs.num_confirmed.p, 0, sizeof(uint32_t) * std::max<uint32_t>(nr, 1), st));
        count_launch();
        k_mbb_finalize<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(a, n, pr.p, ps_sorted.p, cs.view());
        TJ_CUDA(cudaGetLastError());
    } else {
        TJ_CUDA(cudaMemsetAsync(cs.num_confirmed.p, 0, sizeof(uint32_t) * std::max<uint32_t>(nr, 1), st));
    }
    stream_sync(st);
    return n;
}

VoxelOut voxel_filter(Workspace& ws, const VoxelArgs& a, CandDevStore& cs, DevBuf<ActiveVpDev>& active,
                      bool want_trace, std::vector<PrunedVp>* pruned_host, std::vector<uint8_t>* touched_host,
                      cudaStream_t st) {
    VoxelOut out{};
    const uint64_t n = a.n_cands;
    DevBuf<uint32_t> surv(std::max<uint64_t>(n, 1));
    DevBuf<unsigned long long> stats(2);
    TJ_CUDA(cudaMemsetAsync(stats.p, 0, 16, st));
    DevBuf<uint8_t> touched;
    if (want_trace) {
        touched.alloc(std::max<uint64_t>(n, 1));
        TJ_CUDA(cudaMemsetAsync(touched.p, 0, touched.n, st));
    }
    if (n > 0) {
        count_launch();
        k_vf_bounds<<<grid_for(n * 32, 256, ws.num_sms), 256, 0, st>>>(a, cs.view(), surv.p, stats.p,
                                                                        want_trace ? touched.p : nullptr);
        TJ_CUDA(cudaGetLastError());
    }
    unsigned long long hs[2] = {0, 0};
    TJ_CUDA(cudaMemcpyAsync(hs, stats.p, 16, cudaMemcpyDeviceToHost, st));
    DevBuf<uint64_t> offsets;
    const uint64_t total = scan_counts(ws, surv.p, n, offsets, st);
    out.vp_generated = hs[0];
    out.vp_pruned = hs[1];
    out.survivors = total;
    active.reserve(std::max<uint64_t>(total, 1));
    if (total > 0) {
        count_launch();
        k_vf_scatter<false><<<grid_for(n * 32, 256, ws.num_sms), 256, 0, st>>>(a, cs.view(), offsets.p, active.p,
                                                                               nullptr);
        TJ_CUDA(cudaGetLastError());
    }
    if (want_trace) {
        touched_host->resize(n);
        if (n) TJ_CUDA(cudaMemcpyAsync(touched_host->data(), touched.p, n, cudaMemcpyDeviceToHost, st));
        DevBuf<uint32_t> pc(std::max<uint64_t>(n, 1));
        count_launch();
        if (n) k_pruned_count<<<grid_for(n, 256, ws.num_sms), 256, 0, st>>>(a, cs.view(), touched.p, surv.p, pc.p);
        DevBuf<uint64_t> poff;
        const uint64_t np = scan_counts(ws, pc.p, n, poff, st);
        DevBuf<ActiveVpDev> pv(std::max<uint64_t>(np, 1));
        DevBuf<double> plb(std::max<uint64_t>(np, 1));
        count_launch();
        if (np) k_vf_scatter<true><<<grid_for(n * 32, 256, ws.num_sms), 256, 0, st>>>(a, cs.view(), poff.p, pv.p, plb.p);
        std::vector<ActiveVpDev> hv(np);
        std::vector<double> hl(np);
        if (np) {
            TJ_CUDA(cudaMemcpyAsync(hv.data(), pv.p, np * sizeof(ActiveVpDev), cudaMemcpyDeviceToHost, st));
            TJ_CUDA(cudaMemcpyAsync(hl.data(), plb.p, np * sizeof(double), cudaMemcpyDeviceToHost, st));
        }
        stream_sync(st);
        pruned_host->resize(np);
        for (uint64_t i = 0; i < np; ++i) (*pruned_host)[i] = {hv[i].op, hv[i].gvr, hv[i].gvs, hl[i]};
    }
    stream_sync(st);
    return out;
}

} // namespace tjx
