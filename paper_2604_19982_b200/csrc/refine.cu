// Refinement kernels (reference refine_kernel, src/refine.cpp:63-84) and the exact
// geometry batch entry points. Compiled with --fmad=false as a second line of defence;
// the geometry itself uses non-contractible __d*_rn intrinsics.
#include <cuda_runtime.h>

#include "refine_kernel.cuh"
#include "tj_internal.cuh"

namespace tjx {

namespace {

constexpr int kThreads = kWarps * 32;

__device__ __forceinline__ void flush_counters(unsigned long long tested, unsigned long long evaluated,
                                               unsigned long long* counters) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tested += __shfl_xor_sync(0xffffffffu, tested, o);
        evaluated += __shfl_xor_sync(0xffffffffu, evaluated, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(counters + 0, tested);
        atomicAdd(counters + 1, evaluated);
    }
}

__global__ void __launch_bounds__(kThreads, 4) refine_join_kernel(RefineJoinArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    unsigned long long tested = 0, evaluated = 0;
    for (;;) {
        unsigned long long vp = 0;
        if (lane == 0) vp = atomicAdd(a.work, 1ull);
        vp = __shfl_sync(0xffffffffu, vp, 0);
        if (vp >= a.n_vp) break;
        const ActiveVpDev av = a.active[vp];
        const uint64_t r0 = a.r_foff[av.gvr], r1 = a.r_foff[av.gvr + 1];
        const uint64_t s0 = a.s_foff[av.gvs], s1 = a.s_foff[av.gvs + 1];
        double lb, ub;
        // op-level cull thresholds unless exact per-voxel-pair outputs were requested
        const OpMin om{a.vp_lb ? nullptr : a.op_lb_bits, a.vp_lb ? nullptr : a.op_ub_bits, av.op};
        refine_voxel_pair(sm, a.r_facets + r0 * 12, (uint32_t)(r1 - r0), a.s_facets + s0 * 12,
                          (uint32_t)(s1 - s0), a.cull != 0, om, lb, ub, tested, evaluated);
        if (lane == 0) {
            if (a.vp_lb) {
                a.vp_lb[vp] = lb;
                a.vp_ub[vp] = ub;
            }
            // empty voxel pairs are (+inf, +inf) and leave the op minima untouched
            if (lb != __longlong_as_double(0x7ff0000000000000ll)) {
                atomicMin(a.op_lb_bits + av.op, (unsigned long long)__double_as_longlong(lb));
                atomicMin(a.op_ub_bits + av.op, (unsigned long long)__double_as_longlong(ub));
            }
        }
    }
    flush_counters(tested, evaluated, a.counters);
}

__global__ void __launch_bounds__(kThreads, 4) refine_batch_kernel(RefineBatchArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    unsigned long long tested = 0, evaluated = 0;
    for (;;) {
        unsigned long long vp = 0;
        if (lane == 0) vp = atomicAdd(a.work, 1ull);
        vp = __shfl_sync(0xffffffffu, vp, 0);
        if (vp >= a.n_vp) break;
        double lb, ub;
        const OpMin om{nullptr, nullptr, 0};
        refine_voxel_pair(sm, a.facets + a.r_off[vp] * 12, a.r_len[vp], a.facets + a.s_off[vp] * 12, a.s_len[vp],
                          a.cull != 0, om, lb, ub, tested, evaluated);
        if (lane == 0) {
            a.vp_lb[vp] = lb;
            a.vp_ub[vp] = ub;
        }
    }
    flush_counters(tested, evaluated, a.counters);
}

__device__ __noinline__ double tri_tri_call(uint32_t a, uint32_t b) { return tri_tri(a, b); }

__global__ void __launch_bounds__(128) tri_tri_batch_kernel(uint64_t n, const double* __restrict__ a9,
                                                            const double* __restrict__ b9, double* __restrict__ out) {
    __shared__ double rec[128][2][kFacetWords];
    const uint32_t ta = smem_addr(&rec[threadIdx.x][0][0]), tb = smem_addr(&rec[threadIdx.x][1][0]);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        double n2, s2;
        stage_exact(a9 + 9 * i, 0.0, 0.0, ta, &n2, &s2);
        stage_exact(b9 + 9 * i, 0.0, 0.0, tb, &n2, &s2);
        out[i] = tri_tri_call(ta, tb);
    }
}

__global__ void mindist_batch_kernel(uint64_t n, const double* __restrict__ a6, const double* __restrict__ b6,
                                     double* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = mindist_box(a6 + 6 * i, b6 + 6 * i);
}

size_t refine_smem_bytes() { return sizeof(WarpSmem) * kWarps; }

} // namespace

void launch_refine_join(const RefineJoinArgs& a, int num_sms, cudaStream_t st) {
    if (a.n_vp == 0) return;
    static bool attr = false;
    if (!attr) {
        TJ_CUDA(cudaFuncSetAttribute(refine_join_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)refine_smem_bytes()));
        attr = true;
    }
    const uint64_t want = (a.n_vp + kWarps - 1) / kWarps;
    const int grid = (int)std::min<uint64_t>(want, (uint64_t)num_sms * 4);
    count_launch();
    refine_join_kernel<<<grid, kThreads, refine_smem_bytes(), st>>>(a);
    TJ_CUDA(cudaGetLastError());
}

void launch_refine_batch(const RefineBatchArgs& a, int num_sms, cudaStream_t st) {
    if (a.n_vp == 0) return;
    static bool attr = false;
    if (!attr) {
        TJ_CUDA(cudaFuncSetAttribute(refine_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)refine_smem_bytes()));
        attr = true;
    }
    const uint64_t want = (a.n_vp + kWarps - 1) / kWarps;
    const int grid = (int)std::min<uint64_t>(want, (uint64_t)num_sms * 4);
    count_launch();
    refine_batch_kernel<<<grid, kThreads, refine_smem_bytes(), st>>>(a);
    TJ_CUDA(cudaGetLastError());
}

void launch_tri_tri_batch(uint64_t n, const double* a9, const double* b9, double* out, cudaStream_t st) {
    if (!n) return;
    const int grid = (int)std::min<uint64_t>((n + 127) / 128, 148 * 8);
    count_launch();
    tri_tri_batch_kernel<<<grid, 128, 0, st>>>(n, a9, b9, out);
    TJ_CUDA(cudaGetLastError());
}

void launch_mindist_batch(uint64_t n, const double* a6, const double* b6, double* out, cudaStream_t st) {
    if (!n) return;
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, 148 * 8);
    count_launch();
    mindist_batch_kernel<<<grid, 256, 0, st>>>(n, a6, b6, out);
    TJ_CUDA(cudaGetLastError());
}

} // namespace tjx
