// Refinement kernels (reference refine_kernel, src/refine.cpp:63-84) and the exact geometry
// batch entry points; design and exactness argument in refine_kernel.cuh. Compiled with
// --fmad=false as a second line of defence (the FP64 geometry uses non-contractible
// __d*_rn intrinsics).
#include <cuda_runtime.h>

#include "refine_kernel.cuh"
#include "tj_internal.cuh"

namespace tjx {

namespace {

struct VpDescDev {
    uint32_t op;
    uint64_t r0, s0; // first facet (record index) of each segment
    uint32_t rn, sn;
    double iv_lb, iv_ub;
};

__device__ __forceinline__ VpDescDev get_vp(const RefineSource& src, uint64_t vp) {
    VpDescDev d;
    if (src.active) { // join mode
        const ActiveVpDev av = src.active[vp];
        d.op = av.op;
        d.r0 = src.r_foff[av.gvr];
        d.rn = (uint32_t)(src.r_foff[av.gvr + 1] - d.r0);
        d.s0 = src.s_foff[av.gvs];
        d.sn = (uint32_t)(src.s_foff[av.gvs + 1] - d.s0);
        d.iv_lb = src.cand_lb[av.op];
        d.iv_ub = src.cand_ub[av.op];
    } else { // batch mode: every voxel pair is its own op, interval [0, +inf]
        d.op = (uint32_t)vp;
        d.r0 = src.r_off[vp];
        d.rn = src.r_len[vp];
        d.s0 = src.s_off[vp];
        d.sn = src.s_len[vp];
        d.iv_lb = 0.0;
        d.iv_ub = __longlong_as_double(0x7ff0000000000000ll);
    }
    return d;
}

// Warp-aggregated append of one pair per lane with `want` set; entries beyond the capacity
// are dropped but counted (the host re-runs the pass with a larger queue).
__device__ __forceinline__ void queue_push(const RefineQueue& q, bool want, uint32_t op, uint32_t fr, uint32_t fs,
                                           uint32_t mask = 0) {
    const unsigned bal = __ballot_sync(0xffffffffu, want);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(q.count, (unsigned long long)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (want) {
        const unsigned long long pos = base + __popc(bal & ((1u << lane) - 1u));
        if (pos < q.capacity) q.items[pos] = {op, fr, fs, mask};
    }
}

// Seed pass: the 2 facet pairs of smallest box gap of every voxel pair are queued.
// Screen pass: every facet pair not provably irrelevant (refine_kernel.cuh) is queued.
template <bool kSeed>
__global__ void __launch_bounds__(256) k_screen(RefineSource src, uint64_t vp_begin, uint64_t vp_end,
                                                const unsigned long long* __restrict__ op_lb_bits,
                                                const unsigned long long* __restrict__ op_ub_bits, int cull,
                                                RefineQueue q, RefineQueue qv, unsigned long long* work,
                                                unsigned long long* counters) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScreenSmem& sm = reinterpret_cast<ScreenSmem*>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    unsigned long long tested = 0, sat_tests = 0;
    const float kInfF = __int_as_float(0x7f800000);
    for (;;) {
        unsigned long long vp = 0;
        if (lane == 0) vp = atomicAdd(work, 1ull);
        vp = __shfl_sync(0xffffffffu, vp, 0) + vp_begin;
        if (vp >= vp_end) break;
        const VpDescDev d = get_vp(src, vp);
        if (d.rn == 0 || d.sn == 0) continue;
        Thresh th{kInfF, kInfF, false};
        if (!kSeed) {
            const double tlb = bits_to_double(__ldcg(op_lb_bits + d.op));
            double tub = bits_to_double(__ldcg(op_ub_bits + d.op));
            tub = tub < d.iv_ub ? tub : d.iv_ub;
            th.lb_sat = tlb <= d.iv_lb;
            th.lb_u = ru(tlb);
            th.ub_u = ru(tub);
            // nothing can change lb' or ub': the whole voxel pair is irrelevant
            if (cull && (th.lb_sat || th.lb_u == 0.f) && th.ub_u == 0.f) continue;
        }
        const double* rbase = src.r_facets + d.r0 * 12;
        const double* sbase = src.s_facets + d.s0 * 12;
        const double origin[3] = {__ldg(rbase), __ldg(rbase + 1), __ldg(rbase + 2)};
        // seed candidates (lane-local best two): box gap and global facet indices
        float b1 = kInfF, b2 = kInfF;
        uint32_t f1r = 0, f1s = 0, f2r = 0, f2s = 0;
        for (uint32_t r0 = 0; r0 < d.rn; r0 += kRT) {
            const int rcnt = (int)min((uint32_t)kRT, d.rn - r0);
            __syncwarp();
            if (lane < rcnt) stage_screen(rbase + (size_t)(r0 + lane) * 12, origin, sm.rc + lane * kCS);
            for (uint32_t s0 = 0; s0 < d.sn; s0 += kST) {
                const int scnt = (int)min((uint32_t)kST, d.sn - s0);
                __syncwarp();
                if (lane < scnt) stage_screen(sbase + (size_t)(s0 + lane) * 12, origin, sm.sc + lane * kCS);
                __syncwarp();
                const int npairs = rcnt * scnt;
                const int step_i = 32 / scnt, step_j = 32 - (32 / scnt) * scnt; // t += 32 in (i, j)
                int bi = lane / scnt, bj = lane - (lane / scnt) * scnt;
                int nq = 0;
                auto sat_round = [&](int n) { // screen sm.q[0, n) with the separating-axis bound
                    __syncwarp();
                    bool need = false, verify = false;
                    int i = 0, j = 0, mask = 0;
                    if (lane < n) {
                        const int e = sm.q[lane];
                        i = e >> 5;
                        j = e & 31;
                        const float* a = sm.rc + i * kCS;
                        const float* b = sm.sc + j * kCS;
                        const float B = fmaxf(box_gap_lb(a, b), sat_lower_bound(a, b));
                        mask = cannot_improve(B, a, b, th) ? skip_mask(B, a, b) : -1;
                        need = mask < 0;
                        verify = mask > 0;
                        ++sat_tests;
                    }
                    const uint32_t fr = (uint32_t)(d.r0 + r0 + i), fs = (uint32_t)(d.s0 + s0 + j);
                    queue_push(q, need, d.op, fr, fs);
                    queue_push(qv, verify, d.op, fr, fs, (uint32_t)mask);
                };
                for (int t0 = 0; t0 < npairs; t0 += 32) {
                    const int t = t0 + lane;
                    if (kSeed) {
                        if (t < npairs) {
                            const float B = box_gap_lb(sm.rc + bi * kCS, sm.sc + bj * kCS);
                            const uint32_t fr = (uint32_t)(d.r0 + r0 + bi), fs = (uint32_t)(d.s0 + s0 + bj);
                            if (B < b1) {
                                b2 = b1; f2r = f1r; f2s = f1s;
                                b1 = B; f1r = fr; f1s = fs;
                            } else if (B < b2) {
                                b2 = B; f2r = fr; f2s = fs;
                            }
                        }
                    } else {
                        bool need = false;
                        if (t < npairs) {
                            const float* a = sm.rc + bi * kCS;
                            const float* b = sm.sc + bj * kCS;
                            const float B = box_gap_lb(a, b);
                            need = !cull || !(cannot_improve(B, a, b, th) && skip_mask(B, a, b) == 0);
                            ++tested;
                        }
                        if (!cull) {
                            queue_push(q, need, d.op, (uint32_t)(d.r0 + r0 + bi), (uint32_t)(d.s0 + s0 + bj));
                        } else {
                            const unsigned bal = __ballot_sync(0xffffffffu, need);
                            if (need) sm.q[nq + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)((bi << 5) | bj);
                            nq += __popc(bal);
                            if (nq >= 32) {
                                sat_round(32);
                                __syncwarp();
                                if (lane < nq - 32) sm.q[lane] = sm.q[32 + lane];
                                nq -= 32;
                            }
                        }
                    }
                    bj += step_j;
                    bi += step_i;
                    if (bj >= scnt) { bj -= scnt; ++bi; }
                }
                if (!kSeed && nq > 0) sat_round(nq);
            }
        }
        if (kSeed) {
            // warp top-2 by box gap (ties: lowest lane)
            float best = b1;
            int wl = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int ol = __shfl_xor_sync(0xffffffffu, wl, o);
                if (ob < best || (ob == best && ol < wl)) { best = ob; wl = ol; }
            }
            const bool first = lane == wl && b1 < kInfF;
            float cand = lane == wl ? b2 : b1;
            int cl = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ob = __shfl_xor_sync(0xffffffffu, cand, o);
                const int ol = __shfl_xor_sync(0xffffffffu, cl, o);
                if (ob < cand || (ob == cand && ol < cl)) { cand = ob; cl = ol; }
            }
            const bool second = lane == cl && cand < kInfF;
            const uint32_t sr = lane == wl ? f2r : f1r, ss = lane == wl ? f2s : f1s;
            queue_push(q, first, d.op, f1r, f1s);
            queue_push(q, second, d.op, sr, ss);
        }
    }
    if (counters) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            tested += __shfl_xor_sync(0xffffffffu, tested, o);
            sat_tests += __shfl_xor_sync(0xffffffffu, sat_tests, o);
        }
        if (lane == 0) {
            atomicAdd(counters + 0, tested);
            atomicAdd(counters + 3, sat_tests);
        }
    }
}

// Exact evaluation of the queued facet pairs: thread per pair, records staged in the
// thread's own shared-memory slots, minima folded into the op bits with atomicMin.
__global__ void __launch_bounds__(128) k_eval(RefineSource src, RefineQueue q, unsigned long long* __restrict__ lb_bits,
                                              unsigned long long* __restrict__ ub_bits, unsigned long long* counters) {
    __shared__ double rec[128][2][kFacetWords];
    const uint32_t ra = smem_addr(&rec[threadIdx.x][0][0]), sb = smem_addr(&rec[threadIdx.x][1][0]);
    unsigned long long n = *q.count;
    if (n > q.capacity) n = q.capacity;
    unsigned long long done = 0;
    for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
         k += (unsigned long long)gridDim.x * blockDim.x) {
        const PairRef p = q.items[k];
        double c[12];
        double n2, s2;
        load_facet(src.r_facets + (size_t)p.fr * 12, c);
        stage_exact(c, c[9], c[10], ra, &n2, &s2);
        load_facet(src.s_facets + (size_t)p.fs * 12, c);
        stage_exact(c, c[9], c[10], sb, &n2, &s2);
        const double2 v = eval_pair(ra, sb);
        const unsigned long long lbv = (unsigned long long)__double_as_longlong(v.x);
        const unsigned long long ubv = (unsigned long long)__double_as_longlong(v.y);
        if (lbv < __ldcg(lb_bits + p.op)) atomicMin(lb_bits + p.op, lbv);
        if (ubv < __ldcg(ub_bits + p.op)) atomicMin(ub_bits + p.op, ubv);
        ++done;
    }
    if (counters) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) done += __shfl_xor_sync(0xffffffffu, done, o);
        if ((threadIdx.x & 31) == 0 && done) atomicAdd(counters + 1, done);
    }
}

// Piercing verification of skip candidates with ill-conditioned edge/plane combinations:
// thread per entry; entries whose reference piercing test fires go to the exact queue.
__global__ void __launch_bounds__(128) k_verify(RefineSource src, RefineQueue qv, RefineQueue q) {
    __shared__ double rec[128][2][kFacetWords];
    const uint32_t ra = smem_addr(&rec[threadIdx.x][0][0]), sb = smem_addr(&rec[threadIdx.x][1][0]);
    unsigned long long n = *qv.count;
    if (n > qv.capacity) n = qv.capacity;
    const unsigned long long n_round = (n + 31) & ~31ull; // whole warps iterate together
    for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n_round;
         k += (unsigned long long)gridDim.x * blockDim.x) {
        bool need = false;
        PairRef p{0, 0, 0, 0};
        if (k < n) {
            p = qv.items[k];
            double c[12];
            double n2, s2;
            load_facet(src.r_facets + (size_t)p.fr * 12, c);
            stage_exact(c, c[9], c[10], ra, &n2, &s2);
            load_facet(src.s_facets + (size_t)p.fs * 12, c);
            stage_exact(c, c[9], c[10], sb, &n2, &s2);
            need = !pierce_clear((int)p.mask, ra, sb);
        }
        queue_push(q, need, p.op, p.fr, p.fs);
    }
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

constexpr int kScreenThreads = 256;
constexpr size_t kScreenSmem = sizeof(ScreenSmem) * (kScreenThreads / 32);

template <bool kSeed>
void launch_screen(const RefineSource& src, uint64_t b, uint64_t e, const unsigned long long* lbb,
                   const unsigned long long* ubb, int cull, const RefineQueue& q, const RefineQueue& qv,
                   unsigned long long* work, unsigned long long* counters, int num_sms, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        TJ_CUDA(cudaFuncSetAttribute(k_screen<kSeed>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScreenSmem));
        attr = true;
    }
    const uint64_t warps = e - b;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, (uint64_t)num_sms * 3));
    TJ_CUDA(cudaMemsetAsync(work, 0, 8, st));
    count_launch();
    k_screen<kSeed><<<grid, kScreenThreads, kScreenSmem, st>>>(src, b, e, lbb, ubb, cull, q, qv, work, counters);
    TJ_CUDA(cudaGetLastError());
}

} // namespace

void refine_pass(const RefineSource& src, uint64_t vp_begin, uint64_t vp_end, bool seed, unsigned long long* lb_bits,
                 unsigned long long* ub_bits, int cull, RefineQueueStore& qs, unsigned long long* work,
                 unsigned long long* counters, int num_sms, cudaStream_t st) {
    if (vp_end <= vp_begin) return;
    for (int attempt = 0; attempt < 3; ++attempt) {
        TJ_CUDA(cudaMemsetAsync(qs.count.p, 0, 16, st));
        const RefineQueue q = qs.view(), qv = qs.verify_view();
        if (seed)
            launch_screen<true>(src, vp_begin, vp_end, lb_bits, ub_bits, cull, q, qv, work,
                                attempt ? nullptr : counters, num_sms, st);
        else
            launch_screen<false>(src, vp_begin, vp_end, lb_bits, ub_bits, cull, q, qv, work,
                                 attempt ? nullptr : counters, num_sms, st);
        unsigned long long n[2] = {0, 0};
        TJ_CUDA(cudaMemcpyAsync(n, qs.count.p, 16, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaStreamSynchronize(st));
        // the verify pass can move every verify entry to the exact queue: reserve for both
        const unsigned long long need_q = n[0] + n[1], need_v = n[1];
        if (need_q <= qs.items.n && need_v <= qs.vitems.n) break;
        // queue overflow: grow and re-run the (deterministic) pass; nothing was evaluated yet
        if (need_q > qs.items.n) qs.items.alloc(need_q + need_q / 4);
        if (need_v > qs.vitems.n) qs.vitems.alloc(need_v + need_v / 4);
    }
    const int grid = num_sms * 8;
    count_launch();
    k_verify<<<grid, 128, 0, st>>>(src, qs.verify_view(), qs.view());
    TJ_CUDA(cudaGetLastError());
    count_launch();
    k_eval<<<grid, 128, 0, st>>>(src, qs.view(), lb_bits, ub_bits, counters);
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
