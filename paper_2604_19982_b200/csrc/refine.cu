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

// Warp-aggregated append of one pair per lane with `want` set (all lanes must call);
// entries beyond the capacity are dropped but counted (the host re-runs with a larger queue).
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

__device__ __forceinline__ void load_rec(const float4* __restrict__ g, float* dst) {
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const float4 v = __ldg(g + k);
        dst[4 * k] = v.x;
        dst[4 * k + 1] = v.y;
        dst[4 * k + 2] = v.z;
        dst[4 * k + 3] = v.w;
    }
}

// Cooperative copy of n records (7 float4 each) into shared memory.
__device__ __forceinline__ void copy_recs(const float4* __restrict__ g, uint64_t first, int n, float* dst) {
    const int lane = threadIdx.x & 31;
    float4* d4 = reinterpret_cast<float4*>(dst);
    const float4* s4 = g + first * 7;
    for (int k = lane; k < 7 * n; k += 32) d4[k] = __ldg(s4 + k);
}

// Warp argmin (ties: lowest index) of (value, index).
__device__ __forceinline__ void warp_argmin(float& v, uint32_t& idx) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov < v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
}

__global__ void k_prep(const double* __restrict__ facets, uint64_t n, float4* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float r[kCS];
        make_screen(facets + i * 12, r);
#pragma unroll
        for (int k = 0; k < 7; ++k) out[i * 7 + k] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
    }
}

// Seed pass, warp per voxel pair, O(r + s): i* = the r facet closest (box gap) to the s
// segment's box, j* symmetrically; then j' = the s facet closest to i* and i' the r facet
// closest to j*. Queues (i*, j') and (i', j*).
__global__ void __launch_bounds__(256) k_seed(RefineSource src, uint64_t vp_begin, uint64_t vp_end, RefineQueue q,
                                              unsigned long long* work) {
    const int lane = threadIdx.x & 31;
    const float kInfF = __int_as_float(0x7f800000);
    for (;;) {
        unsigned long long vp = 0;
        if (lane == 0) vp = atomicAdd(work, 1ull);
        vp = __shfl_sync(0xffffffffu, vp, 0) + vp_begin;
        if (vp >= vp_end) break;
        const VpDescDev d = get_vp(src, vp);
        if (d.rn == 0 || d.sn == 0) continue;
        const float4* R = src.r_screen + d.r0 * 7;
        const float4* S = src.s_screen + d.s0 * 7;
        // segment boxes (lo at [0..2], hi at [4..6], as in a record)
        float br[8] = {kInfF, kInfF, kInfF, 0.f, -kInfF, -kInfF, -kInfF, 0.f};
        float bs[8] = {kInfF, kInfF, kInfF, 0.f, -kInfF, -kInfF, -kInfF, 0.f};
        for (uint32_t i = lane; i < d.rn; i += 32) {
            const float4 lo = __ldg(R + i * 7), hi = __ldg(R + i * 7 + 1);
            br[0] = fminf(br[0], lo.x); br[1] = fminf(br[1], lo.y); br[2] = fminf(br[2], lo.z);
            br[4] = fmaxf(br[4], hi.x); br[5] = fmaxf(br[5], hi.y); br[6] = fmaxf(br[6], hi.z);
        }
        for (uint32_t j = lane; j < d.sn; j += 32) {
            const float4 lo = __ldg(S + j * 7), hi = __ldg(S + j * 7 + 1);
            bs[0] = fminf(bs[0], lo.x); bs[1] = fminf(bs[1], lo.y); bs[2] = fminf(bs[2], lo.z);
            bs[4] = fmaxf(bs[4], hi.x); bs[5] = fmaxf(bs[5], hi.y); bs[6] = fmaxf(bs[6], hi.z);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                br[k] = fminf(br[k], __shfl_xor_sync(0xffffffffu, br[k], o));
                bs[k] = fminf(bs[k], __shfl_xor_sync(0xffffffffu, bs[k], o));
                br[4 + k] = fmaxf(br[4 + k], __shfl_xor_sync(0xffffffffu, br[4 + k], o));
                bs[4 + k] = fmaxf(bs[4 + k], __shfl_xor_sync(0xffffffffu, bs[4 + k], o));
            }
        }
        // argmin of (box gap, then centre distance): among facets touching the other box,
        // prefer the one nearest its centre (deepest overlap)
        auto closest = [&](const float4* set, uint32_t n, const float* box) {
            const float cx = 0.5f * (box[0] + box[4]), cy = 0.5f * (box[1] + box[5]), cz = 0.5f * (box[2] + box[6]);
            float best = kInfF;
            uint32_t bi = 0xffffffffu;
            for (uint32_t i = lane; i < n; i += 32) {
                const float4 lo = __ldg(set + i * 7), hi = __ldg(set + i * 7 + 1);
                const float rec[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
                const float g = box_gap_lb(rec, box);
                const float dx = 0.5f * (lo.x + hi.x) - cx, dy = 0.5f * (lo.y + hi.y) - cy, dz = 0.5f * (lo.z + hi.z) - cz;
                // gap dominates; the centre distance only orders near-ties (scaled to stay below gaps)
                const float key = g + 1e-3f * sqrtf(dx * dx + dy * dy + dz * dz);
                if (key < best || (key == best && i < bi)) { best = key; bi = i; }
            }
            warp_argmin(best, bi);
            return bi;
        };
        const uint32_t ist = closest(R, d.rn, bs);
        const uint32_t jst = closest(S, d.sn, br);
        float bi_box[8], bj_box[8];
        {
            const float4 lo = __ldg(R + ist * 7), hi = __ldg(R + ist * 7 + 1);
            bi_box[0] = lo.x; bi_box[1] = lo.y; bi_box[2] = lo.z; bi_box[4] = hi.x; bi_box[5] = hi.y; bi_box[6] = hi.z;
            const float4 lo2 = __ldg(S + jst * 7), hi2 = __ldg(S + jst * 7 + 1);
            bj_box[0] = lo2.x; bj_box[1] = lo2.y; bj_box[2] = lo2.z; bj_box[4] = hi2.x; bj_box[5] = hi2.y; bj_box[6] = hi2.z;
        }
        const uint32_t jp = closest(S, d.sn, bi_box);
        const uint32_t ip = closest(R, d.rn, bj_box);
        queue_push(q, lane == 0, d.op, (uint32_t)(d.r0 + ist), (uint32_t)(d.s0 + jp));
        queue_push(q, lane == 0 && !(ip == ist && jst == jp), d.op, (uint32_t)(d.r0 + ip), (uint32_t)(d.s0 + jst));
    }
}

// The reference's FP64 piercing test for the masked edge/plane combinations of two facet
// records (global memory): true iff none fires (both facets are well shaped, hence not
// degenerate, so the reference would run every one of these tests).
__device__ __noinline__ bool pierce_clear(int mask, const double* __restrict__ pa, const double* __restrict__ pb) {
    double a[9], b[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        a[k] = __ldg(pa + k);
        b[k] = __ldg(pb + k);
    }
    const V3 A[3] = {{a[0], a[1], a[2]}, {a[3], a[4], a[5]}, {a[6], a[7], a[8]}};
    const V3 B[3] = {{b[0], b[1], b[2]}, {b[3], b[4], b[5]}, {b[6], b[7], b[8]}};
#pragma unroll 1
    for (int c = 0; c < 6; ++c) {
        if (!(mask & (1 << c))) continue;
        const int e = c < 3 ? c : c - 3, e1 = e == 2 ? 0 : e + 1;
        const bool hit = c < 3 ? pierces_ref(A[e], A[e1], B[0], B[1], B[2]) : pierces_ref(B[e], B[e1], A[0], A[1], A[2]);
        if (hit) return false;
    }
    return true;
}

// Screen pass: every facet pair not provably irrelevant (refine_kernel.cuh) is queued; skip
// candidates with ill-conditioned edge/plane combinations are first checked with the
// reference's own FP64 piercing test (pierce_clear).
__global__ void __launch_bounds__(256) k_screen(RefineSource src, uint64_t vp_begin, uint64_t vp_end,
                                                const unsigned long long* __restrict__ op_lb_bits,
                                                const unsigned long long* __restrict__ op_ub_bits, int cull,
                                                RefineQueue q, unsigned long long* work,
                                                unsigned long long* counters) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScreenSmem& sm = reinterpret_cast<ScreenSmem*>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    unsigned long long tested = 0, sat_tests = 0;
    for (;;) {
        unsigned long long vp = 0;
        if (lane == 0) vp = atomicAdd(work, 1ull);
        vp = __shfl_sync(0xffffffffu, vp, 0) + vp_begin;
        if (vp >= vp_end) break;
        const VpDescDev d = get_vp(src, vp);
        if (d.rn == 0 || d.sn == 0) continue;
        const double tlb = bits_to_double(__ldcg(op_lb_bits + d.op));
        double tub = bits_to_double(__ldcg(op_ub_bits + d.op));
        tub = tub < d.iv_ub ? tub : d.iv_ub;
        const Thresh th{ru(tlb), ru(tub), tlb <= d.iv_lb};
        // nothing can change lb' or ub': the whole voxel pair is irrelevant
        if (cull && (th.lb_sat || th.lb_u == 0.f) && th.ub_u == 0.f) continue;
        for (uint32_t r0 = 0; r0 < d.rn; r0 += kRT) {
            const int rcnt = (int)min((uint32_t)kRT, d.rn - r0);
            __syncwarp();
            copy_recs(src.r_screen, d.r0 + r0, rcnt, sm.rc);
            for (uint32_t s0 = 0; s0 < d.sn; s0 += kST) {
                const int scnt = (int)min((uint32_t)kST, d.sn - s0);
                __syncwarp();
                copy_recs(src.s_screen, d.s0 + s0, scnt, sm.sc);
                __syncwarp();
                const int npairs = rcnt * scnt;
                const int step_i = 32 / scnt, step_j = 32 - (32 / scnt) * scnt; // t += 32 in (i, j)
                int bi = lane / scnt, bj = lane - (lane / scnt) * scnt;
                int nq = 0;
                {   // per-row thresholds for the stage-1 test (box_cannot_improve)
                    float Lm = 0.f, Mm = 0.f;
                    if (lane < rcnt) { Lm = fabsf(sm.rc[lane * kCS + 3]); Mm = sm.rc[lane * kCS + 27]; }
                    if (lane < scnt) {
                        Lm = fmaxf(Lm, fabsf(sm.sc[lane * kCS + 3]));
                        Mm = fmaxf(Mm, sm.sc[lane * kCS + 27]);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        Lm = fmaxf(Lm, __shfl_xor_sync(0xffffffffu, Lm, o));
                        Mm = fmaxf(Mm, __shfl_xor_sync(0xffffffffu, Mm, o));
                    }
                    const float delta0 = __fadd_ru(__fmul_ru(2e-5f, Lm), __fmul_ru(2e-12f, Mm));
                    if (lane < rcnt) {
                        const float ninf = __int_as_float(0xff800000);
                        const bool lb_settled = th.lb_sat || th.lb_u == 0.f;
                        sm.row_lb[lane] = lb_settled ? ninf : __fadd_ru(__fadd_ru(th.lb_u, delta0), sm.rc[lane * kCS + 11]);
                        sm.row_ub[lane] = th.ub_u == 0.f ? ninf : __fsub_ru(__fadd_ru(th.ub_u, delta0), sm.rc[lane * kCS + 7]);
                    }
                    __syncwarp();
                }
                auto sat_round = [&](int n) { // screen sm.q[0, n) with the separating-axis bound
                    __syncwarp();
                    bool need = false;
                    int i = 0, j = 0, mask = 0;
                    uint32_t fr = 0, fs = 0;
                    if (lane < n) {
                        const int e = sm.q[lane];
                        i = e >> 5;
                        j = e & 31;
                        fr = (uint32_t)(d.r0 + r0 + i);
                        fs = (uint32_t)(d.s0 + s0 + j);
                        const float* a = sm.rc + i * kCS;
                        const float* b = sm.sc + j * kCS;
                        const double* va = src.r_facets + (size_t)fr * 12;
                        const double* vb = src.s_facets + (size_t)fs * 12;
                        const float off[3] = {(float)(__ldg(vb) - __ldg(va)), (float)(__ldg(vb + 1) - __ldg(va + 1)),
                                              (float)(__ldg(vb + 2) - __ldg(va + 2))};
                        const float B = fmaxf(box_gap_lb(a, b), sat_lower_bound(a, b, off));
                        mask = cannot_improve(B, a, b, th) ? skip_mask(B, a, b) : -1;
                        need = mask < 0;
                        if (mask > 0) need = !pierce_clear(mask, va, vb); // reference piercing test
                        ++sat_tests;
                    }
                    queue_push(q, need, d.op, fr, fs);
                };
                for (int t0 = 0; t0 < npairs; t0 += 32) {
                    const int t = t0 + lane;
                    bool need = false;
                    if (t < npairs) {
                        const float* a = sm.rc + bi * kCS;
                        const float* b = sm.sc + bj * kCS;
                        const float g2 = box_gap2_lb(a, b);
                        need = !cull || !box_cannot_improve(g2, sm.row_lb[bi], sm.row_ub[bi], b) ||
                               skip_mask(__fmul_rd(sqrtf(g2), 1.0f - 0x1p-20f), a, b) != 0;
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
                    bj += step_j;
                    bi += step_i;
                    if (bj >= scnt) { bj -= scnt; ++bi; }
                }
                if (nq > 0) sat_round(nq);
            }
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

inline int warp_grid(uint64_t warps, int num_sms, int per_sm) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, (uint64_t)num_sms * per_sm));
}

} // namespace

void refine_prep(const double* facets, uint64_t n, float4* out, int num_sms, cudaStream_t st) {
    if (!n) return;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 16));
    count_launch();
    k_prep<<<grid, 256, 0, st>>>(facets, n, out);
    TJ_CUDA(cudaGetLastError());
}

void refine_pass(const RefineSource& src, uint64_t vp_begin, uint64_t vp_end, bool seed, unsigned long long* lb_bits,
                 unsigned long long* ub_bits, int cull, RefineQueueStore& qs, unsigned long long* work,
                 unsigned long long* counters, int num_sms, cudaStream_t st) {
    if (vp_end <= vp_begin) return;
    static bool attr = false;
    if (!attr) {
        TJ_CUDA(cudaFuncSetAttribute(k_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScreenSmem));
        attr = true;
    }
    const int grid = num_sms * 8;
    if (seed) {
        // 2 entries per voxel pair at most
        if (2 * (vp_end - vp_begin) > qs.items.n) qs.items.alloc(2 * (vp_end - vp_begin));
        TJ_CUDA(cudaMemsetAsync(qs.count.p, 0, 16, st));
        TJ_CUDA(cudaMemsetAsync(work, 0, 8, st));
        count_launch();
        k_seed<<<warp_grid(vp_end - vp_begin, num_sms, 4), 256, 0, st>>>(src, vp_begin, vp_end, qs.view(), work);
        TJ_CUDA(cudaGetLastError());
    } else {
        for (int attempt = 0; attempt < 3; ++attempt) {
            TJ_CUDA(cudaMemsetAsync(qs.count.p, 0, 16, st));
            TJ_CUDA(cudaMemsetAsync(work, 0, 8, st));
            count_launch();
            k_screen<<<warp_grid(vp_end - vp_begin, num_sms, 3), kScreenThreads, kScreenSmem, st>>>(
                src, vp_begin, vp_end, lb_bits, ub_bits, cull, qs.view(), work,
                attempt ? nullptr : counters);
            TJ_CUDA(cudaGetLastError());
            unsigned long long n[2] = {0, 0};
            TJ_CUDA(cudaMemcpyAsync(n, qs.count.p, 16, cudaMemcpyDeviceToHost, st));
            TJ_CUDA(cudaStreamSynchronize(st));
            if (n[0] <= qs.items.n) break;
            // queue overflow: grow and re-run the (deterministic) pass; nothing was evaluated yet
            qs.items.alloc(n[0] + n[0] / 4);
        }
    }
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
