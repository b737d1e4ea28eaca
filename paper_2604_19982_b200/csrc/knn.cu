// k-NN progressive pruning on sm_100a (reference src/knn.cpp, paper Alg. 6 as revised by
// the reference: strict comparisons, N = |U| - 1, rounds to a fixpoint).
//
// One warp per query r. A round evaluates, against the state at round start, for every
// undecided candidate m of r:
//     farther(m) = |{n in U : lb(n) > ub(m)}|      closer(m) = |{n in U : ub(n) < lb(m)}|
//     CONFIRMED  if (|U| - 1) - farther(m) < kLeft;   else REMOVED if closer(m) >= kLeft
// (knn_prune_round, src/knn.cpp:19-63; the reference's sorted-array binary searches count
// exactly these sets, and m never counts itself because lb(m) <= ub(m)). The deltas are then
// applied (knn_apply_deltas :65-80) and rounds repeat until none change. A query's rounds
// depend only on its own candidates, so per-query fixpoints equal the reference's global
// round loop (:82-91).
#include "filter.cuh"

namespace tjx {

namespace {

__device__ __forceinline__ void flag_knn_error(DevError* err, uint32_t op) {
    atomicMin(&err->op, op);
    err->kind = 1;
    atomicExch(&err->code, (int)TJ_EENGINE);
}

__global__ void k_knn_fixpoint(CandDev c, uint32_t nq, uint32_t k, int16_t stage, uint8_t* __restrict__ delta,
                               DevError* err, unsigned long long* decided_total, int apply) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    unsigned long long decided = 0;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nq; r += warps) {
        const uint64_t b = c.r2op[r], e = c.r2op[r + 1];
        for (;;) {
            // |U|
            uint32_t u = 0;
            for (uint64_t op = b + lane; op < e; op += 32) u += c.status[op] == TJ_UNDECIDED;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
            if (u == 0) break;
            const int64_t k_left = (int64_t)k - (int64_t)c.num_confirmed[r];
            if (k_left < 0) {
                if (lane == 0) flag_knn_error(err, (uint32_t)b);
                break;
            }
            uint32_t changes = 0, confirms = 0;
            for (uint64_t m = b + lane; m < e; m += 32) {
                uint8_t d = 0;
                if (c.status[m] == TJ_UNDECIDED) {
                    const double lbm = c.lb[m], ubm = c.ub[m];
                    int64_t farther = 0, closer = 0;
                    for (uint64_t n = b; n < e; ++n) {
                        if (c.status[n] != TJ_UNDECIDED) continue;
                        farther += c.lb[n] > ubm;
                        closer += c.ub[n] < lbm;
                    }
                    if (((int64_t)u - 1) - farther < k_left) d = TJ_CONFIRMED;
                    else if (closer >= k_left) d = TJ_REMOVED;
                }
                delta[m] = d;
                if (!apply) changes += d != 0;
            }
            __syncwarp();
            if (!apply) { // one round, deltas only (knn_prune_round)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) changes += __shfl_xor_sync(0xffffffffu, changes, o);
                decided += changes;
                break;
            }
            for (uint64_t m = b + lane; m < e; m += 32) {
                const uint8_t d = delta[m];
                if (d) {
                    c.status[m] = d;
                    c.decided_at[m] = stage;
                    ++changes;
                    confirms += d == TJ_CONFIRMED;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                changes += __shfl_xor_sync(0xffffffffu, changes, o);
                confirms += __shfl_xor_sync(0xffffffffu, confirms, o);
            }
            __syncwarp();
            if (changes == 0) break;
            if (lane == 0) {
                const uint32_t nc = c.num_confirmed[r] + confirms;
                c.num_confirmed[r] = nc;
                if (nc > k) flag_knn_error(err, (uint32_t)b);
            }
            decided += changes;
            __syncwarp();
            if (c.num_confirmed[r] > k) break;
        }
    }
    if (lane == 0 && decided) atomicAdd(decided_total, decided);
}

// knn_finalize: fill the remaining slots per query in (lb, s) order, remove the rest.
__global__ void k_knn_finalize(CandDev c, uint32_t nq, uint32_t k, uint8_t* __restrict__ delta) {
    const int lane = threadIdx.x & 31;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nq; r += warps) {
        const uint64_t b = c.r2op[r], e = c.r2op[r + 1];
        const uint32_t nc = c.num_confirmed[r];
        const uint32_t k_left = k > nc ? k - nc : 0;
        for (uint64_t m = b + lane; m < e; m += 32) {
            uint8_t d = 0;
            if (c.status[m] == TJ_UNDECIDED) {
                const double lbm = c.lb[m];
                const uint32_t sm = c.pair_s[m];
                uint32_t rank = 0; // position in the reference's std::sort by (lb, s)
                for (uint64_t n = b; n < e; ++n) {
                    if (n == m || c.status[n] != TJ_UNDECIDED) continue;
                    const double lbn = c.lb[n];
                    rank += (lbn < lbm) || (!(lbn != lbm) && c.pair_s[n] < sm);
                }
                d = rank < k_left ? TJ_CONFIRMED : TJ_REMOVED;
            }
            delta[m] = d;
        }
        __syncwarp();
        uint32_t confirms = 0;
        for (uint64_t m = b + lane; m < e; m += 32) {
            const uint8_t d = delta[m];
            if (d) {
                c.status[m] = d;
                c.decided_at[m] = 100;
                confirms += d == TJ_CONFIRMED;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) confirms += __shfl_xor_sync(0xffffffffu, confirms, o);
        if (lane == 0) c.num_confirmed[r] = nc + confirms;
        __syncwarp();
    }
}

} // namespace

uint64_t knn_fixpoint(Workspace& ws, CandDevStore& cs, uint32_t k, int16_t stage, DevError* err, cudaStream_t st) {
    if (cs.n == 0 || cs.nq == 0) return 0;
    DevBuf<uint8_t> delta(cs.n);
    DevBuf<unsigned long long> total(1);
    TJ_CUDA(cudaMemsetAsync(total.p, 0, 8, st));
    const uint64_t threads = (uint64_t)cs.nq * 32;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((threads + 255) / 256, (uint64_t)ws.num_sms * 16));
    count_launch();
    k_knn_fixpoint<<<grid, 256, 0, st>>>(cs.view(), cs.nq, k, stage, delta.p, err, total.p, 1);
    TJ_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    TJ_CUDA(cudaMemcpyAsync(&h, total.p, 8, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    return h;
}

uint64_t knn_round_dev(Workspace& ws, CandDevStore& cs, uint32_t k, DevBuf<uint8_t>& delta, DevError* err,
                       cudaStream_t st) {
    if (cs.n == 0) return 0;
    TJ_CUDA(cudaMemsetAsync(delta.p, 0, cs.n, st));
    if (cs.nq == 0) return 0;
    DevBuf<unsigned long long> total(1);
    TJ_CUDA(cudaMemsetAsync(total.p, 0, 8, st));
    const uint64_t threads = (uint64_t)cs.nq * 32;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((threads + 255) / 256, (uint64_t)ws.num_sms * 16));
    count_launch();
    k_knn_fixpoint<<<grid, 256, 0, st>>>(cs.view(), cs.nq, k, 0, delta.p, err, total.p, 0);
    TJ_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    TJ_CUDA(cudaMemcpyAsync(&h, total.p, 8, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    return h;
}

} // namespace tjx

namespace tjx {
void knn_finalize_dev(Workspace& ws, CandDevStore& cs, uint32_t k, cudaStream_t st) {
    if (cs.n == 0 || cs.nq == 0) return;
    DevBuf<uint8_t> delta(cs.n);
    const uint64_t threads = (uint64_t)cs.nq * 32;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((threads + 255) / 256, (uint64_t)ws.num_sms * 16));
    count_launch();
    k_knn_finalize<<<grid, 256, 0, st>>>(cs.view(), cs.nq, k, delta.p);
    TJ_CUDA(cudaGetLastError());
    stream_sync(st);
}
} // namespace tjx
