// Refinement kernels (reference refine_kernel, src/refine.cpp:63-84) and the exact geometry
// batch entry points; design and exactness argument in refine_kernel.cuh. Compiled with
// --fmad=false as a second line of defence (the FP64 geometry uses non-contractible
// __d*_rn intrinsics).
#include <cuda_runtime.h>
#include <cstdlib>
#include <mutex>
#include <map>
#include <set>
#include <type_traits>

#include "refine_kernel.cuh"
#include "tj_internal.cuh"

namespace tjx {

namespace {

// TRIJOIN_DEBUG_OPSTATS diagnostics (per-op counters only in a -DTJ_DEBUG_OPSTATS build)
__device__ unsigned long long* g_dbg_op_tested = nullptr;


// k_screen launch shape: 8 warps per block, 2 blocks per SM (16 warps, 128 registers; 4 x 5 was
// slower: the 102-register bound spills the stage-2 code)
#ifndef TJ_S1_UNROLL
#define TJ_S1_UNROLL 1 // stage-1 inner loop unroll (B: 1 = 2 = 63.6 ms, 4: 67.4; C: 1: 191, 2: 198, 4: 216 ms)
#endif

#ifndef TJ_ROWS_SINGLE_MIN
#define TJ_ROWS_SINGLE_MIN 27
#endif
#ifndef TJ_ROWS_SINGLE
#define TJ_ROWS_SINGLE 1 // measured: B 44.95 -> 44.46 ms (LOD 60 13.3 -> 13.0), C within noise
#endif
constexpr int kScreenThreads = 256;
constexpr int kScreenBlocks = 2;

struct VpDescDev {
    uint32_t op;
    uint32_t gvr, gvs; // global voxel ids (join mode)
    uint32_t r0, s0; // first facet (record index) of each segment (a level's records: < 2^32, like the queues')
    uint32_t rn, sn;
    double iv_lb, iv_ub;
};

__device__ __forceinline__ VpDescDev get_vp(const RefineSource& src, uint64_t vp) {
    VpDescDev d;
    if (src.active) { // join mode
        const ActiveVpDev av = src.active[vp];
        d.op = av.op;
        d.gvr = av.gvr;
        d.gvs = av.gvs;
        const uint64_t rf = src.r_foff[av.gvr];
        d.r0 = (uint32_t)rf;
        d.rn = (uint32_t)(src.r_foff[av.gvr + 1] - rf);
        const uint64_t sf = src.s_foff[av.gvs];
        d.s0 = (uint32_t)sf;
        d.sn = (uint32_t)(src.s_foff[av.gvs + 1] - sf);
        d.iv_lb = src.cand_lb[av.op];
        d.iv_ub = src.cand_ub[av.op];
    } else { // batch mode: every voxel pair is its own op, interval [0, +inf]
        d.op = (uint32_t)vp;
        d.gvr = d.gvs = 0;
        d.r0 = (uint32_t)src.r_off[vp];
        d.rn = src.r_len[vp];
        d.s0 = (uint32_t)src.s_off[vp];
        d.sn = src.s_len[vp];
        d.iv_lb = 0.0;
        d.iv_ub = __longlong_as_double(0x7ff0000000000000ll);
    }
    return d;
}

// Segment aggregates of a voxel pair: precomputed per voxel (join mode) or reduced here.
__device__ __forceinline__ SegAgg seg_r_of(const RefineSource& src, const VpDescDev& d) {
    return src.r_seg ? seg_load(src.r_seg + 3ull * d.gvr) : seg_reduce(src.r_box, d.r0, d.rn);
}
__device__ __forceinline__ SegAgg seg_s_of(const RefineSource& src, const VpDescDev& d) {
    return src.s_seg ? seg_load(src.s_seg + 3ull * d.gvs) : seg_reduce(src.s_box, d.s0, d.sn);
}

__global__ void k_seg_prep(const float4* __restrict__ box, const uint64_t* __restrict__ foff, uint64_t n_voxels,
                           float4* __restrict__ seg) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t v = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); v < n_voxels; v += warps) {
        const uint64_t f0 = foff[v];
        const SegAgg g = seg_reduce(box, f0, (uint32_t)(foff[v + 1] - f0));
        if (lane == 0) seg_store(seg + 3 * v, g);
    }
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

// Cooperative gather of up to 32 screening records (facets first + list[k]) into shared
// memory: box part from `box`, geometry part from `geo` (kRecF4 float4 per record, rows
// kCS floats apart).
__device__ __forceinline__ void gather_recs(const float4* __restrict__ box, const float4* __restrict__ geo,
                                            const double* __restrict__ facets, uint64_t first, const uint16_t* list,
                                            int n, float* dst) {
    // cp.async: every 16-B piece is in flight at once (a load -> store loop serialises one
    // global latency per iteration and lane).
    constexpr int kParts = kRecF4, kStride4 = kCS / 4;
    const int lane = threadIdx.x & 31;
    float4* d4 = reinterpret_cast<float4*>(dst);
#if TJ_GATHER_FIXED_PART
    // kParts = 8: lane copies part (lane & 7) of records lane / 8, + 4, ...; the part's source
    // array, stride and the shared-memory column are loop-invariant per lane
    static_assert(kParts == 8, "gather: 8 parts per record");
    const int part = lane & 7;
    const char* src = part < kBoxF4 ? reinterpret_cast<const char*>(box + part)
                                    : reinterpret_cast<const char*>(geo + (part - kBoxF4));
    const uint32_t stride = part < kBoxF4 ? kBoxF4 * 16u : kGeoF4 * 16u;
    uint32_t sa = smem_addr(d4 + (lane >> 3) * kStride4 + part);
    const uint32_t f0 = (uint32_t)first; // facet indices of a level are 32-bit
#pragma unroll 4
    for (int rec = lane >> 3; rec < n; rec += 4, sa += 4 * kCS * 4) {
        const char* g = src + (uint64_t)(f0 + list[rec]) * stride;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
    }
#else
    for (int k = lane; k < kParts * n; k += 32) {
        const int rec = k / kParts, part = k % kParts;
        const uint64_t f = first + list[rec];
        const float4* g = part < kBoxF4 ? box + f * kBoxF4 + part : geo + f * kGeoF4 + (part - kBoxF4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(d4 + rec * kStride4 + part)),
                     "l"(g)
                     : "memory");
    }
#endif
    if (lane < n) { // the facet's FP64 v0 (16 + 8 B)
        const double* v = facets + (first + list[lane]) * 12;
        float* r = dst + lane * kCS + kV0Off;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(r)), "l"(v) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr(r + 4)), "l"(v + 2) : "memory");
    }
}
__device__ __forceinline__ void gather_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// TMA bulk staging of a tile (-DTJ_TILE_BULK=1; off by default): lane k < n copies record k
// with three cp.async.bulk transfers (48-B box part, 80-B geometry part, the facet's first 32 B
// of FP64 coordinates = v0 + v1.x) completing on the warp's mbarrier (160 B of transactions per
// record). Correct (the GPU suite passes with it) but measured slower than the per-lane
// cp.async gather: config B 57.9 -> 71.1 ms, C 192.8 -> 224.5 ms — ~200 small bulk copies per
// tile pair from 16 warps queue on the SM's TMA unit, where LDGSTS spreads them over the LSU.
#ifndef TJ_TILE_BULK
#define TJ_TILE_BULK 0
#endif
constexpr uint32_t kTileRecBytes = 48 + 80 + 32;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void gather_bulk(const float4* __restrict__ box, const float4* __restrict__ geo,
                                            const double* __restrict__ facets, uint64_t first, const uint16_t* list,
                                            int n, float* dst, uint32_t bar) {
    const int lane = threadIdx.x & 31;
    if (lane < n) {
        const uint64_t f = first + list[lane];
        const uint32_t d = smem_addr(dst + lane * kCS);
        bulk_g2s(d, box + f * kBoxF4, 16 * kBoxF4, bar);
        bulk_g2s(d + 16 * kBoxF4, geo + f * kGeoF4, 16 * kGeoF4, bar);
        bulk_g2s(d + 4 * kV0Off, facets + f * 12, 32, bar);
    }
}
// Before the warp's lanes let the async proxy overwrite tiles they have read: all prior
// (generic-proxy) accesses ordered before the copies; lane 0 then arms the barrier for `bytes`.
__device__ __forceinline__ void tile_arm(uint32_t bar, uint32_t bytes) {
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    if ((threadIdx.x & 31) == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
    __syncwarp();
}
__device__ __forceinline__ void tile_wait(uint32_t bar, uint32_t& phase) {
    asm volatile(
        "{\n .reg .pred p;\n TJ_TILE_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra TJ_TILE_WAIT_%=;\n}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
    phase ^= 1u;
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

// Records [0, n) of a level of n records, or with rng (voxel range [rng[0], rng[1]) of the CSR
// foff) the records of those voxels only (a level arriving in object-range pieces).
__global__ void k_prep(const double* __restrict__ facets, uint64_t n, float4* __restrict__ out, unsigned* agg,
                       int zero_pad, const uint64_t* __restrict__ foff, uint64_t v_begin, uint64_t v_end) {
    float4* box = out;
    float4* geo = out + kBoxF4 * n;
    float hdmin = __int_as_float(0x7f800000), lmax = 0.f, mmax = 0.f;
    const uint64_t i0 = foff ? foff[v_begin] : 0, i1 = foff ? foff[v_end] : n;
    for (uint64_t i = i0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < i1; i += (uint64_t)gridDim.x * blockDim.x) {
        float r[kCS];
        make_screen(facets + i * 12, r);
        if (zero_pad) r[7] = r[11] = 0.f; // hd, ph
        hdmin = fminf(hdmin, r[7]);
        lmax = fmaxf(lmax, fabsf(r[3]));
        mmax = fmaxf(mmax, r[27]);
#pragma unroll
        for (int k = 0; k < kBoxF4; ++k) box[i * kBoxF4 + k] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
#pragma unroll
        for (int k = 0; k < kGeoF4; ++k)
            geo[i * kGeoF4 + k] = make_float4(r[12 + 4 * k], r[13 + 4 * k], r[14 + 4 * k], r[15 + 4 * k]);
    }
    if (agg) { // non-negative floats order like their bit patterns
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            hdmin = fminf(hdmin, __shfl_xor_sync(0xffffffffu, hdmin, o));
            lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
            mmax = fmaxf(mmax, __shfl_xor_sync(0xffffffffu, mmax, o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(agg, __float_as_uint(fmaxf(hdmin, 0.f)));
            atomicMax(agg + 1, __float_as_uint(lmax));
            atomicMax(agg + 2, __float_as_uint(mmax));
        }
    }
}

// Seed ordering key (a heuristic; exactness never depends on it) of a facet box (a: lo.xyz
// L, b: hi.xyz hd) against box (lo, hi): squared gap + 1e-6 x squared centre distance, so
// the gap dominates and the centre distance orders near-ties (deepest overlap first).
__device__ __forceinline__ float seed_key(float4 a, float4 b, const float* lo, const float* hi) {
    const float gx = fmaxf(0.f, fmaxf(lo[0] - b.x, a.x - hi[0]));
    const float gy = fmaxf(0.f, fmaxf(lo[1] - b.y, a.y - hi[1]));
    const float gz = fmaxf(0.f, fmaxf(lo[2] - b.z, a.z - hi[2]));
    const float cx = (a.x + b.x) - (lo[0] + hi[0]), cy = (a.y + b.y) - (lo[1] + hi[1]), cz = (a.z + b.z) - (lo[2] + hi[2]);
    const float g2 = __fmaf_rn(gx, gx, __fmaf_rn(gy, gy, __fmul_rn(gz, gz)));
    const float c2 = __fmaf_rn(cx, cx, __fmaf_rn(cy, cy, __fmul_rn(cz, cz)));
    return __fmaf_rn(0.25e-6f, c2, g2);
}

// Warp argmin of a non-negative key held by lanes [0, 32) (lane = index): the key's low 5
// bits are replaced by the lane, so one integer min-reduction returns the winner (ties, and
// keys within 2^-18 relative, resolve to the lowest lane; a heuristic order only).
__device__ __forceinline__ uint32_t warp_argmin_lane(float key) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned packed = (__float_as_uint(key) & ~31u) | lane;
    return __reduce_min_sync(0xffffffffu, packed) & 31u;
}

// Facets i* of r closest (seed_key) to box sb and j* of s closest to box rb, in one sweep.
__device__ __forceinline__ void closest_pair(const float4* __restrict__ rset, uint64_t r0, uint32_t rn,
                                             const float4* __restrict__ sset, uint64_t s0, uint32_t sn,
                                             const SegAgg& rb, const SegAgg& sb, uint32_t& ist, uint32_t& jst) {
    const int lane = threadIdx.x & 31;
    const float kInfF = __int_as_float(0x7f800000);
    float br = kInfF, bs = kInfF;
    uint32_t ir = 0xffffffffu, is = 0xffffffffu;
    for (uint32_t i = lane; i < max(rn, sn); i += 32) {
        if (i < rn) {
            const float k = seed_key(__ldg(rset + (r0 + i) * kBoxF4), __ldg(rset + (r0 + i) * kBoxF4 + 1), sb.lo, sb.hi);
            if (k < br) { br = k; ir = i; }
        }
        if (i < sn) {
            const float k = seed_key(__ldg(sset + (s0 + i) * kBoxF4), __ldg(sset + (s0 + i) * kBoxF4 + 1), rb.lo, rb.hi);
            if (k < bs) { bs = k; is = i; }
        }
    }
    warp_argmin(br, ir);
    warp_argmin(bs, is);
    ist = ir;
    jst = is;
}

// Decision mode: when every facet pair has hd_i + hd_j > 1e-5 (L_i + L_j) + 1e-12 (M_i + M_j),
// no ub_ij can be 0 at this level (B + hd_i + hd_j >= tiny + delta for every pair), so the ub
// side of every op is settled (the level's aggregates, k_prep).
__device__ __forceinline__ bool level_ub_settled(const RefineSource& src, int cull) {
    if (cull != 2 || !src.agg) return false;
    const float hd2 = __fadd_rd(__uint_as_float(src.agg[0]), __uint_as_float(src.agg[3]));
    const float l2 = __fadd_ru(__uint_as_float(src.agg[1]), __uint_as_float(src.agg[4]));
    const float m2 = __fadd_ru(__uint_as_float(src.agg[2]), __uint_as_float(src.agg[5]));
    return hd2 > __fadd_ru(__fadd_ru(__fmul_ru(1e-5f, l2), __fmul_ru(1e-12f, m2)), 1e-30f);
}

// Decision mode, a voxel pair whose segments can hold a zero bound (segment gap <= ph_max(r) +
// ph_max(s)): only those are seeded.
__device__ __forceinline__ bool seedable_dm(const SegAgg& ar, const SegAgg& as) {
    const float arec[8] = {ar.lo[0], ar.lo[1], ar.lo[2], 0.f, ar.hi[0], ar.hi[1], ar.hi[2], 0.f};
    const float brec[8] = {as.lo[0], as.lo[1], as.lo[2], 0.f, as.hi[0], as.hi[1], as.hi[2], 0.f};
    return !(box_gap_lb(arec, brec) > __fadd_ru(as.phmax, ar.phmax));
}

#ifndef TJ_SEED2_OVERLAP
#define TJ_SEED2_OVERLAP 0 // phase-2 seeds only for voxel pairs whose segment boxes overlap
#endif
__device__ __forceinline__ bool seg_boxes_overlap(const SegAgg& a, const SegAgg& b) {
    return a.lo[0] <= b.hi[0] && b.lo[0] <= a.hi[0] && a.lo[1] <= b.hi[1] && b.lo[1] <= a.hi[1] &&
           a.lo[2] <= b.hi[2] && b.lo[2] <= a.hi[2];
}

// Decision-mode seeding in two phases (refine_pass): one op needs a single zero-bound facet
// pair to settle, so each op's most promising voxel pair (segment boxes by decreasing overlap
// volume, then by increasing squared gap; ties to the lowest index) is seeded and evaluated
// first, and the op's other voxel pairs are seeded only if the op is still open. A heuristic
// order only: exactness rests on the screen, which tests every pair of every open op.
// pick[op] = min over the op's seedable voxel pairs of (key << 32 | voxel pair - vp_begin).
__global__ void k_seed_pick(RefineSource src, uint64_t vp_begin, uint64_t vp_end, unsigned long long* pick) {
    for (uint64_t vp = vp_begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; vp < vp_end;
         vp += (uint64_t)gridDim.x * blockDim.x) {
        const VpDescDev d = get_vp(src, vp);
        if (d.rn == 0 || d.sn == 0) continue;
        const SegAgg ar = seg_r_of(src, d), as = seg_s_of(src, d);
        if (!seedable_dm(ar, as)) continue;
        float g2 = 0.f, vol = 1.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float e = fminf(ar.hi[k], as.hi[k]) - fmaxf(ar.lo[k], as.lo[k]);
            g2 += e < 0.f ? e * e : 0.f;
            vol *= fmaxf(e, 0.f);
        }
        const uint32_t key = g2 > 0.f ? 0x80000000u + __float_as_uint(g2) : 0x7fffffffu - __float_as_uint(vol);
        atomicMin(pick + d.op, (unsigned long long)key << 32 | (uint32_t)(vp - vp_begin));
    }
}

// Seed pass, warp per voxel pair, O(r + s): i* = the r facet closest (box gap) to the s
// segment's box, j* symmetrically; then j' = the s facet closest to i* and i' the r facet
// closest to j*; queues (i*, j') and (i', j*). In decision mode only voxel pairs that can
// hold a zero bound are seeded (segment gap <= ph_max(r) + ph_max(s)).
#ifndef SEED_BATCH
#define SEED_BATCH 32
#endif
__device__ __forceinline__ unsigned seed_batch() { return SEED_BATCH; }
__global__ void __launch_bounds__(256, 4) k_seed(RefineSource src, uint64_t vp_begin, uint64_t vp_end, RefineQueue q,
                                              int cull, int phase, const unsigned long long* __restrict__ pick,
                                              const unsigned long long* __restrict__ lb_bits,
                                              const unsigned long long* __restrict__ ub_bits) {
    // per warp: the voxel pairs of the current batch that need seeds (segments + boxes)
    struct SeedVp {
        uint64_t r0, s0;
        uint32_t op, rn, sn, pad;
        float alo[3], ahi[3], blo[3], bhi[3];
    };
    __shared__ SeedVp sv[8][32];
    const int lane = threadIdx.x & 31;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t gw = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    PairRef pref{0u, 0u, 0u, 0u}; // this lane's buffered seed
    int pend = 0;
    // decision mode: only voxel pairs that can hold a zero bound
    auto seedable = [&](const SegAgg& ar, const SegAgg& as) { return cull != 2 || seedable_dm(ar, as); };
    // two-phase decision-mode seeding (k_seed_pick): phase 1 the ops' primary voxel pairs, phase 2
    // the others of the ops still open (k_eval's settled test); phase 0 every voxel pair
    const bool ub_settled = level_ub_settled(src, cull);
    auto wanted = [&](uint64_t vp, uint32_t op) {
        if (phase == 0) return true;
        const bool prim = (uint32_t)__ldcg(pick + op) == (uint32_t)(vp - vp_begin);
        if (phase == 1 || prim) return prim;
        return exact_op(src.exact_mask, op) || !(bits_to_double(__ldcg(lb_bits + op)) == 0.0 &&
                                                 (ub_settled || bits_to_double(__ldcg(ub_bits + op)) == 0.0));
    };
    // buffer the seeds (i*, j') and (i', j*) of a voxel pair in lanes (pend = entries held),
    // one queue append per 30+ seeds; arguments warp-uniform
    auto emit = [&](uint32_t op, uint64_t r0, uint64_t s0, uint32_t ist, uint32_t jst, uint32_t ip, uint32_t jp) {
        const bool two = !(ip == ist && jp == jst);
        if (lane == pend) pref = {op, (uint32_t)(r0 + ist), (uint32_t)(s0 + jp), 0u};
        if (two && lane == pend + 1) pref = {op, (uint32_t)(r0 + ip), (uint32_t)(s0 + jst), 0u};
        pend += two ? 2 : 1;
        if (pend >= 31) {
            queue_push(q, lane < pend, pref.op, pref.fr, pref.fs);
            pend = 0;
        }
    };
    auto seed_vp = [&](const VpDescDev& d, const SegAgg& ar, const SegAgg& as) {
        uint32_t ist, jst, ip, jp;
        if (d.rn <= 32 && d.sn <= 32) {
            // both segments fit the warp: each lane keeps its r and s facet boxes in registers
            const float kInfF = __int_as_float(0x7f800000);
            float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, s0 = r0, s1 = r0;
            if (lane < (int)d.rn) { r0 = __ldg(src.r_box + ((size_t)d.r0 + lane) * kBoxF4); r1 = __ldg(src.r_box + ((size_t)d.r0 + lane) * kBoxF4 + 1); }
            if (lane < (int)d.sn) { s0 = __ldg(src.s_box + ((size_t)d.s0 + lane) * kBoxF4); s1 = __ldg(src.s_box + ((size_t)d.s0 + lane) * kBoxF4 + 1); }
            ist = warp_argmin_lane(lane < (int)d.rn ? seed_key(r0, r1, as.lo, as.hi) : kInfF);
            jst = warp_argmin_lane(lane < (int)d.sn ? seed_key(s0, s1, ar.lo, ar.hi) : kInfF);
            // second round against the single facets i*, j* (their boxes by shuffle)
            const float fil[3] = {__shfl_sync(~0u, r0.x, ist), __shfl_sync(~0u, r0.y, ist), __shfl_sync(~0u, r0.z, ist)};
            const float fih[3] = {__shfl_sync(~0u, r1.x, ist), __shfl_sync(~0u, r1.y, ist), __shfl_sync(~0u, r1.z, ist)};
            const float fjl[3] = {__shfl_sync(~0u, s0.x, jst), __shfl_sync(~0u, s0.y, jst), __shfl_sync(~0u, s0.z, jst)};
            const float fjh[3] = {__shfl_sync(~0u, s1.x, jst), __shfl_sync(~0u, s1.y, jst), __shfl_sync(~0u, s1.z, jst)};
            ip = warp_argmin_lane(lane < (int)d.rn ? seed_key(r0, r1, fjl, fjh) : kInfF);
            jp = warp_argmin_lane(lane < (int)d.sn ? seed_key(s0, s1, fil, fih) : kInfF);
        } else if (d.rn <= 64 && d.sn <= 64) {
            // two facets per lane and side (lane, lane + 32) in registers; argmin over 64
            // indices (6 low key bits)
            const float kInfF = __int_as_float(0x7f800000);
            float4 ra0 = make_float4(0.f, 0.f, 0.f, 0.f), ra1 = ra0, rb0 = ra0, rb1 = ra0;
            float4 sa0 = ra0, sa1 = ra0, sb0 = ra0, sb1 = ra0;
            const int l2 = lane + 32;
            if (lane < (int)d.rn) { ra0 = __ldg(src.r_box + ((size_t)d.r0 + lane) * kBoxF4); ra1 = __ldg(src.r_box + ((size_t)d.r0 + lane) * kBoxF4 + 1); }
            if (l2 < (int)d.rn) { rb0 = __ldg(src.r_box + ((size_t)d.r0 + l2) * kBoxF4); rb1 = __ldg(src.r_box + ((size_t)d.r0 + l2) * kBoxF4 + 1); }
            if (lane < (int)d.sn) { sa0 = __ldg(src.s_box + ((size_t)d.s0 + lane) * kBoxF4); sa1 = __ldg(src.s_box + ((size_t)d.s0 + lane) * kBoxF4 + 1); }
            if (l2 < (int)d.sn) { sb0 = __ldg(src.s_box + ((size_t)d.s0 + l2) * kBoxF4); sb1 = __ldg(src.s_box + ((size_t)d.s0 + l2) * kBoxF4 + 1); }
            auto argmin64 = [&](float ka, float kb) -> uint32_t {
                const unsigned pa = (__float_as_uint(ka) & ~63u) | (unsigned)lane;
                const unsigned pb = (__float_as_uint(kb) & ~63u) | (unsigned)l2;
                return __reduce_min_sync(0xffffffffu, min(pa, pb)) & 63u;
            };
            ist = argmin64(lane < (int)d.rn ? seed_key(ra0, ra1, as.lo, as.hi) : kInfF,
                           l2 < (int)d.rn ? seed_key(rb0, rb1, as.lo, as.hi) : kInfF);
            jst = argmin64(lane < (int)d.sn ? seed_key(sa0, sa1, ar.lo, ar.hi) : kInfF,
                           l2 < (int)d.sn ? seed_key(sb0, sb1, ar.lo, ar.hi) : kInfF);
            const bool ih = ist >= 32, jh = jst >= 32;
            const int il = ist & 31, jl = jst & 31;
            const float fil[3] = {__shfl_sync(~0u, ih ? rb0.x : ra0.x, il), __shfl_sync(~0u, ih ? rb0.y : ra0.y, il),
                                  __shfl_sync(~0u, ih ? rb0.z : ra0.z, il)};
            const float fih[3] = {__shfl_sync(~0u, ih ? rb1.x : ra1.x, il), __shfl_sync(~0u, ih ? rb1.y : ra1.y, il),
                                  __shfl_sync(~0u, ih ? rb1.z : ra1.z, il)};
            const float fjl[3] = {__shfl_sync(~0u, jh ? sb0.x : sa0.x, jl), __shfl_sync(~0u, jh ? sb0.y : sa0.y, jl),
                                  __shfl_sync(~0u, jh ? sb0.z : sa0.z, jl)};
            const float fjh[3] = {__shfl_sync(~0u, jh ? sb1.x : sa1.x, jl), __shfl_sync(~0u, jh ? sb1.y : sa1.y, jl),
                                  __shfl_sync(~0u, jh ? sb1.z : sa1.z, jl)};
            ip = argmin64(lane < (int)d.rn ? seed_key(ra0, ra1, fjl, fjh) : kInfF,
                          l2 < (int)d.rn ? seed_key(rb0, rb1, fjl, fjh) : kInfF);
            jp = argmin64(lane < (int)d.sn ? seed_key(sa0, sa1, fil, fih) : kInfF,
                          l2 < (int)d.sn ? seed_key(sb0, sb1, fil, fih) : kInfF);
        } else {
            closest_pair(src.r_box, d.r0, d.rn, src.s_box, d.s0, d.sn, ar, as, ist, jst);
            SegAgg fi = ar, fj = as; // only lo / hi are read
            {
                const float4 a = __ldg(src.r_box + ((size_t)d.r0 + ist) * kBoxF4), b = __ldg(src.r_box + ((size_t)d.r0 + ist) * kBoxF4 + 1);
                fi.lo[0] = a.x; fi.lo[1] = a.y; fi.lo[2] = a.z; fi.hi[0] = b.x; fi.hi[1] = b.y; fi.hi[2] = b.z;
                const float4 c = __ldg(src.s_box + ((size_t)d.s0 + jst) * kBoxF4), e = __ldg(src.s_box + ((size_t)d.s0 + jst) * kBoxF4 + 1);
                fj.lo[0] = c.x; fj.lo[1] = c.y; fj.lo[2] = c.z; fj.hi[0] = e.x; fj.hi[1] = e.y; fj.hi[2] = e.z;
            }
            closest_pair(src.r_box, d.r0, d.rn, src.s_box, d.s0, d.sn, fi, fj, ip, jp);
        }
        emit(d.op, d.r0, d.s0, ist, jst, ip, jp);
    };
    if (src.r_seg && src.s_seg) {
        // precomputed segment aggregates: batches of 32 voxel pairs, one per lane for the
        // descriptor / aggregate lookups and the decision-mode test (independent latency
        // chains), then the warp seeds the survivors
        SeedVp* mine = sv[threadIdx.x >> 5];
        const unsigned nb = seed_batch();
        // phase 1 walks the ops (their primary voxel pairs, pick[op]) instead of every voxel pair
        const bool by_op = phase == 1;
        const uint64_t it_begin = by_op ? 0 : vp_begin, it_end = by_op ? src.n_ops : vp_end;
        for (uint64_t base = it_begin + gw * nb; base < it_end; base += nw * nb) {
            bool live = false;
            __syncwarp();
            uint64_t vp = base + lane;
            bool have = lane < nb && vp < it_end;
            if (have && by_op) {
                const unsigned long long pk = __ldcg(pick + vp);
                have = pk != ~0ull;
                vp = vp_begin + (uint32_t)pk;
            }
            if (have) {
                const VpDescDev d = get_vp(src, vp);
                if (d.rn != 0 && d.sn != 0) {
                    const SegAgg ar = seg_r_of(src, d), as = seg_s_of(src, d);
                    live = seedable(ar, as) && wanted(vp, d.op) && (phase != 2 || !TJ_SEED2_OVERLAP ||
                                                                     seg_boxes_overlap(ar, as));
                    if (live)
                        mine[lane] = {d.r0, d.s0, d.op, d.rn, d.sn, 0u,
                                      {ar.lo[0], ar.lo[1], ar.lo[2]}, {ar.hi[0], ar.hi[1], ar.hi[2]},
                                      {as.lo[0], as.lo[1], as.lo[2]}, {as.hi[0], as.hi[1], as.hi[2]}};
                }
            }
            // voxel pairs with both segments <= 8 (<= 16) facets are seeded four (two) at a
            // time, one per 8-lane (16-lane) group; the others one per warp
            auto run_groups = [&](auto gsize, unsigned set) {
                constexpr int G = decltype(gsize)::value, NG = 32 / G;
                while (set) {
                    const int grp = lane / G, sub = lane % G, gl = lane - sub;
                    int sel = -1; // the batch lane whose voxel pair this group seeds
#pragma unroll
                    for (int k = 0; k < NG; ++k) {
                        const int v = set ? __ffs(set) - 1 : -1;
                        if (set) set &= set - 1;
                        if (k == grp) sel = v;
                    }
                    const bool on = sel >= 0;
                    const SeedVp& e = mine[on ? sel : 0];
                    const uint32_t rn = on ? e.rn : 0u, sn = on ? e.sn : 0u;
                    const float kInfF = __int_as_float(0x7f800000);
                    float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, s0 = r0, s1 = r0;
                    if (sub < (int)rn) { r0 = __ldg(src.r_box + (e.r0 + sub) * kBoxF4); r1 = __ldg(src.r_box + (e.r0 + sub) * kBoxF4 + 1); }
                    if (sub < (int)sn) { s0 = __ldg(src.s_box + (e.s0 + sub) * kBoxF4); s1 = __ldg(src.s_box + (e.s0 + sub) * kBoxF4 + 1); }
                    // argmin within the group (key bits with the lane in the low 5 bits)
                    auto group_argmin = [&](float key) -> uint32_t {
                        unsigned p = (__float_as_uint(key) & ~31u) | (unsigned)lane;
#pragma unroll
                        for (int o = G / 2; o > 0; o >>= 1) p = min(p, __shfl_xor_sync(0xffffffffu, p, o));
                        return (p & 31u) - (unsigned)gl;
                    };
                    const uint32_t ist = group_argmin(sub < (int)rn ? seed_key(r0, r1, e.blo, e.bhi) : kInfF);
                    const uint32_t jst = group_argmin(sub < (int)sn ? seed_key(s0, s1, e.alo, e.ahi) : kInfF);
                    const float fil[3] = {__shfl_sync(~0u, r0.x, gl + ist), __shfl_sync(~0u, r0.y, gl + ist), __shfl_sync(~0u, r0.z, gl + ist)};
                    const float fih[3] = {__shfl_sync(~0u, r1.x, gl + ist), __shfl_sync(~0u, r1.y, gl + ist), __shfl_sync(~0u, r1.z, gl + ist)};
                    const float fjl[3] = {__shfl_sync(~0u, s0.x, gl + jst), __shfl_sync(~0u, s0.y, gl + jst), __shfl_sync(~0u, s0.z, gl + jst)};
                    const float fjh[3] = {__shfl_sync(~0u, s1.x, gl + jst), __shfl_sync(~0u, s1.y, gl + jst), __shfl_sync(~0u, s1.z, gl + jst)};
                    const uint32_t ip = group_argmin(sub < (int)rn ? seed_key(r0, r1, fjl, fjh) : kInfF);
                    const uint32_t jp = group_argmin(sub < (int)sn ? seed_key(s0, s1, fil, fih) : kInfF);
                    // the groups' seeds into the lane buffer, group by group (groups fill in order)
#pragma unroll
                    for (int k = 0; k < NG; ++k) {
                        const int src_lane = G * k;
                        if (!__shfl_sync(0xffffffffu, (int)on, src_lane)) break;
                        const uint32_t op = __shfl_sync(0xffffffffu, on ? e.op : 0u, src_lane);
                        const uint64_t gr0 = __shfl_sync(0xffffffffu, on ? e.r0 : 0ull, src_lane);
                        const uint64_t gs0 = __shfl_sync(0xffffffffu, on ? e.s0 : 0ull, src_lane);
                        emit(op, gr0, gs0, __shfl_sync(0xffffffffu, ist, src_lane), __shfl_sync(0xffffffffu, jst, src_lane),
                             __shfl_sync(0xffffffffu, ip, src_lane), __shfl_sync(0xffffffffu, jp, src_lane));
                    }
                }
            };
            const unsigned all = __ballot_sync(0xffffffffu, live);
            const unsigned le8 = __ballot_sync(0xffffffffu, live && mine[lane].rn <= 8 && mine[lane].sn <= 8);
            const unsigned le16 = __ballot_sync(0xffffffffu, live && mine[lane].rn <= 16 && mine[lane].sn <= 16) & ~le8;
            unsigned pending = all & ~le8 & ~le16;
            __syncwarp();
            run_groups(std::integral_constant<int, 8>{}, le8);
            run_groups(std::integral_constant<int, 16>{}, le16);
            while (pending) {
                const int lv = __ffs(pending) - 1;
                pending &= pending - 1;
                const SeedVp& e = mine[lv];
                VpDescDev d{};
                d.op = e.op;
                d.r0 = e.r0;
                d.s0 = e.s0;
                d.rn = e.rn;
                d.sn = e.sn;
                SegAgg ar{}, as{}; // only lo / hi are read by the seeding
                for (int k = 0; k < 3; ++k) {
                    ar.lo[k] = e.alo[k];
                    ar.hi[k] = e.ahi[k];
                    as.lo[k] = e.blo[k];
                    as.hi[k] = e.bhi[k];
                }
                seed_vp(d, ar, as);
            }
        }
    } else {
        for (uint64_t vp = vp_begin + gw; vp < vp_end; vp += nw) {
            const VpDescDev d = get_vp(src, vp);
            if (d.rn == 0 || d.sn == 0) continue;
            const SegAgg ar = seg_r_of(src, d);
            const SegAgg as = seg_s_of(src, d);
            if (!seedable(ar, as) || !wanted(vp, d.op) || (phase == 2 && TJ_SEED2_OVERLAP && !seg_boxes_overlap(ar, as)))
                continue;
            seed_vp(d, ar, as);
        }
    }
    queue_push(q, lane < pend, pref.op, pref.fr, pref.fs);
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

// Second-stage screen of one queued facet pair (a, b: shared records): true iff the pair
// must be evaluated exactly. Separating-axis bound in two stages (face normals, then the
// 9 edge-edge axes); skip candidates with ill-conditioned edge/plane combinations are
// checked with the reference's own FP64 piercing test (pierce_clear). Returns bit 0: needed,
// bit 1: a piercing verification ran (one call site).
__device__ __forceinline__ int sat_needed(const float* a, const float* b, const double* va, const double* vb, Thresh th) {
    const float B0 = box_gap_lb(a, b);
    int mask = cannot_improve(B0, a, b, th) ? skip_mask(B0, a, b) : -1;
    if (mask == 0) return 0;
    // b.v0 - a.v0 from the staged FP64 vertices, rounded once
    const double* sa = reinterpret_cast<const double*>(a + kV0Off);
    const double* sb = reinterpret_cast<const double*>(b + kV0Off);
    const float off[3] = {(float)(sb[0] - sa[0]), (float)(sb[1] - sa[1]), (float)(sb[2] - sa[2])};
    const SatFrame f = sat_frame(a, b, off);
    if (mask > 0) { // the box gap already rules the pair out up to conditioning: plane sides first
        mask = plane_clear(mask, f, a, b);
        if (mask == 0) return 0;
    }
    float B = fmaxf(B0, sat_faces(f, a, b));
    mask = cannot_improve(B, a, b, th) ? skip_mask(B, a, b) : -1;
    if (mask != 0) {
        // The 9 edge axes can only raise B towards the distance. Skip them where they cannot
        // change the outcome (shapes outside the skip argument) or are very unlikely to (the
        // bound needed for a skip is over twice the face bound): the pair is then evaluated,
        // which is always exact.
        if (a[3] < 0.f || b[3] < 0.f) return 1;
        const float need_lb = (th.lb_sat || th.lb_u == 0.f) ? 0.f : th.lb_u + a[11] + b[11];
        const float need_ub = th.ub_u == 0.f ? 0.f : th.ub_u - a[7] - b[7];
        if (B < 0.5f * fmaxf(need_lb, need_ub)) return 1;
        B = fmaxf(B, sat_edges(f, a, b));
        mask = cannot_improve(B, a, b, th) ? skip_mask(B, a, b) : -1;
    }
    if (mask < 0) return 1;
    if (mask > 0) mask = plane_clear(mask, f, a, b);
    if (mask == 0) return 0;
    return pierce_clear(mask, va, vb) ? 2 : 3; // reference piercing test
}

// Builds the list of facets of [first, first + n) (n <= kCap) that survive the row/column
// screen against the partner segment `o` (offsets relative to first); returns the count.
__device__ __forceinline__ int build_list(const float4* __restrict__ box, uint64_t first, uint32_t n, const SegAgg& o,
                                          float delta0, const Thresh& th, bool cull, uint16_t* list,
                                          uint32_t* dropped) {
    const int lane = threadIdx.x & 31;
    int cnt = 0;
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        bool keep = false;
        if (i < n) {
            keep = true;
            if (cull && o.ok) {
                const float4 a = __ldg(box + (first + i) * kBoxF4), b = __ldg(box + (first + i) * kBoxF4 + 1);
                const float ph = __ldg(box + (first + i) * kBoxF4 + 2).w;
                const float lo[3] = {a.x, a.y, a.z}, hi[3] = {b.x, b.y, b.z};
                if (a.w >= 0.f)
                    keep = !agg_skip(lo, hi, o.lo, o.hi, a.w + o.Lmax, fminf(a.w, o.Lmin), __fadd_ru(ph, o.phmax),
                                     __fadd_rd(b.w, o.hdmin), delta0, th);
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (cull && o.ok && lane == 0) *dropped += (uint32_t)min(32u, n - i0) - __popc(bal);
        if (keep) list[cnt + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)i;
        cnt += __popc(bal);
    }
    __syncwarp();
    return cnt;
}

// Screen pass, warp per voxel pair, hierarchical: (1) the whole voxel pair against the op
// thresholds (segment aggregates); (2) each r facet against the s segment and each s facet
// against the r segment (row / column screens, O(r + s)); (3) the surviving facets in
// 32 x 32 shared-memory tiles, every pair tested on its facet-AABB gap; (4) box survivors
// through the separating-axis stage (sat_needed). Pairs that may still change the op's
// bounds go to the exact queue (refine_kernel.cuh has the exactness argument).
// voxel pairs with fewer facet pairs skip the row / column screens (TRIJOIN_HIER_MIN: tuning)
uint32_t hier_min_pairs() {
    static const uint32_t v = [] {
        const char* e = getenv("TRIJOIN_HIER_MIN");
        return e ? (uint32_t)atoi(e) : kHierMinPairs;
    }();
    return v;
}

// Voxel pairs per work grab of k_screen: inversely proportional to the expected work of a
// voxel pair (mean segment length m, work ~ m^2 facet pairs): kGrabWork / m^2 clamped to
// [4, 32] — large grabs where most voxel pairs are cheap or settled (fewer work-counter
// atomics), small ones where heavy voxel pairs cluster (load balance). kGrabWork = 32768: with
// the cheaper per-pair screen the grab overhead weighs more (8192 / 16384 / 32768 / 65536: B 44.5
// / 43.7 / 43.7 / 44.0 ms, C 179.9 / 178.9 / 176.6 / 177.4, E 294.5 / 293.6 / 294.9 / 295.9, D
// 1358 / - / 1354 / -; round 1 had chosen 8192 over 16384 at B 66.0 vs 65.7, C 201 vs 197).
// TRIJOIN_SCREEN_BATCH (1..32) / TRIJOIN_SCREEN_GRAB_WORK override (tuning).
unsigned screen_batch(float mean_seg, uint64_t n_vps, uint64_t warps) {
    static const int forced = [] {
        const char* e = getenv("TRIJOIN_SCREEN_BATCH");
        const int v = e ? atoi(e) : 0;
        return v >= 1 && v <= 32 ? v : 0;
    }();
    static const float work = [] {
        const char* e = getenv("TRIJOIN_SCREEN_GRAB_WORK");
        return e ? (float)atof(e) : 32768.f;
    }();
    if (forced) return (unsigned)forced;
    if (!(mean_seg > 0.f)) return 4u;
    float b = work / (mean_seg * mean_seg);
    // at least ~8 grabs per warp: a small launch is spread over the whole grid
    const float cap = float(n_vps) / float(8 * (warps ? warps : 1));
    b = fminf(b, cap);
    return b >= 32.f ? 32u : b <= 4.f ? 4u : (unsigned)b;
}

// kBF: the stage-1 DP4A pre-test branch-free, two pairs per iteration (stage1_row); chosen for
// decision mode, whose tested pairs are mostly near (separate kernels keep each one's code lean:
// with both loop variants in one kernel config C lost 4 %).
template <bool kBF>
__global__ void __launch_bounds__(kScreenThreads, kScreenBlocks)
    k_screen(RefineSource src, uint64_t vp_begin, uint64_t vp_end, const unsigned long long* __restrict__ op_lb_bits,
             const unsigned long long* __restrict__ op_ub_bits, int cull, RefineQueue q, unsigned long long* work,
             unsigned long long* counters, unsigned batch, uint32_t hier_min) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SM = ScreenSmem;
    constexpr int CS = kCS, QO = kQOff, MO = kMOff;
    SM& sm = reinterpret_cast<SM*>(smem_raw)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    if (lane < 5) sm.cnt[lane] = 0;
    const uint32_t bar = smem_addr(&sm.bar);
    uint32_t bar_phase = 0;
    if (TJ_TILE_BULK && lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncwarp();
    const bool ub_level_settled = level_ub_settled(src, cull);
    // The op thresholds of a voxel pair (decision mode, intersection with tau = 0: only "is the
    // minimum 0?" matters on either side; a pair surely positive on a side cannot change it).
    auto thresholds = [&](const VpDescDev& d) {
        const double tlb = bits_to_double(__ldcg(op_lb_bits + d.op));
        double tub = bits_to_double(__ldcg(op_ub_bits + d.op));
        tub = tub < d.iv_ub ? tub : d.iv_ub;
        Thresh th{ru(tlb), ru(tub), tlb <= d.iv_lb};
        if (cull == 2 && !exact_op(src.exact_mask, d.op)) {
            constexpr float kTiny = 1e-30f;
            th.lb_sat = tlb == 0.0;
            th.lb_u = th.lb_sat ? 0.f : kTiny;
            th.ub_u = tub == 0.0 || ub_level_settled ? 0.f : kTiny;
        }
        return th;
    };
    // nothing can change lb' or ub': the whole voxel pair is irrelevant
    auto settled = [&](const Thresh& th) { return cull && (th.lb_sat || th.lb_u == 0.f) && th.ub_u == 0.f; };
    // Work in batches of `batch` voxel pairs per work-counter atomic (screen_batch): lane i
    // looks up voxel pair i of the batch and its op thresholds (independent latency chains),
    // the warp then screens only the voxel pairs whose op can still change.
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(work, (unsigned long long)batch);
        base = __shfl_sync(0xffffffffu, base, 0) + vp_begin;
        if (base >= vp_end) break;
        // whole-voxel-pair screen on the segment aggregates; d0 >= 1e-5 (L_i + L_j) + 1e-12
        // (M_i + M_j) for every facet pair of the voxel pair
        auto vp_screen = [&](const VpDescDev& d, const Thresh& th, float& d0, SegAgg& ar, SegAgg& as) {
            ar = seg_r_of(src, d);
            as = seg_s_of(src, d);
            d0 = __fadd_ru(__fmul_ru(2e-5f, fmaxf(ar.Lmax, as.Lmax)), __fmul_ru(2e-12f, fmaxf(seg_m(ar), seg_m(as))));
            return ar.ok && as.ok &&
                   agg_skip(ar.lo, ar.hi, as.lo, as.hi, ar.Lmax + as.Lmax, fminf(ar.Lmin, as.Lmin),
                            __fadd_ru(ar.phmax, as.phmax), __fadd_rd(ar.hdmin, as.hdmin), d0, th);
        };
        // with precomputed segment aggregates (join mode) the voxel-pair screen runs here too,
        // one voxel pair per lane
        const bool pre_seg = cull && src.r_seg && src.s_seg;
        bool live = false, agg_skipped = false;
        __syncwarp();
        if (lane < batch && base + lane < vp_end) {
            const VpDescDev dl = get_vp(src, base + lane);
            const Thresh tl = thresholds(dl);
            live = dl.rn != 0 && dl.sn != 0 && !settled(tl);
            int flags = tl.lb_sat ? 1 : 0;
            float d0 = 0.f;
            if (live && pre_seg) {
                SegAgg ar, as;
                agg_skipped = vp_screen(dl, tl, d0, ar, as);
                live = !agg_skipped;
                if (shapes_settled(ar, as)) flags |= 2;
            }
            if (live) sm.vpd[lane] = {dl.r0, dl.s0, dl.op, dl.gvr, dl.gvs, dl.rn, dl.sn, tl.lb_u, tl.ub_u, d0, flags};
        }
        if (pre_seg) {
            const unsigned n_agg = __popc(__ballot_sync(0xffffffffu, agg_skipped));
            if (lane == 0) sm.cnt[3] += n_agg;
        }
        unsigned pending = __ballot_sync(0xffffffffu, live);
        __syncwarp(); // sm.vpd visible to the warp
        while (pending) {
        const int lv = __ffs(pending) - 1;
        pending &= pending - 1;
        VpDescDev d;
        Thresh th;
        {
            const typename SM::BatchVp& b = sm.vpd[lv];
            d.op = b.op;
            d.gvr = b.gvr;
            d.gvs = b.gvs;
            d.r0 = b.r0;
            d.s0 = b.s0;
            d.rn = b.rn;
            d.sn = b.sn;
            th.lb_u = b.lb_u;
            th.ub_u = b.ub_u;
            th.lb_sat = (b.flags & 1) != 0;
        }
        const bool shapes_ok = (sm.vpd[lv].flags & 2) != 0;
        // hierarchical screens: the whole voxel pair (always when the segment aggregates are
        // precomputed), then rows / columns where that can pay off
        const bool hier = cull && d.rn * d.sn >= hier_min;
        // delta0 >= 1e-5 (L_i + L_j) + 1e-12 (M_i + M_j) for every facet pair: the voxel pair's (from
        // its segment aggregates) when known, else each tile pair computes its own
        float delta0 = sm.vpd[lv].d0;
        if (hier || (cull && !pre_seg && src.r_seg)) {
            float d0;
            SegAgg ar, as;
            const bool skip = vp_screen(d, th, d0, ar, as);
            if (!pre_seg && skip) {
                if (lane == 0) ++sm.cnt[3];
                continue;
            }
            if (hier) {
                delta0 = d0;
                __syncwarp();
                if (lane == 0) {
                    sm.seg_r = ar;
                    sm.seg_s = as;
                }
                __syncwarp();
            }
        }
        // per s record of a staged tile: its ph and hd pre-scaled for stage1_box (pad floats 32, 33)
        auto scale_s_tile = [&](int scnt) {
            if (lane < scnt) {
                float* r = sm.sc + lane * CS;
                r[32] = __fmul_ru(r[11], kInvC);
                r[33] = __fmul_rd(r[7], kInvC);
            }
            __syncwarp();
        };
        for (uint32_t rc0 = 0; rc0 < d.rn; rc0 += kCap) {
            const int nrl = build_list(src.r_box, d.r0 + rc0, min((uint32_t)kCap, d.rn - rc0), sm.seg_s, delta0, th, hier,
                                       sm.rl, &sm.cnt[4]);
            for (uint32_t sc0 = 0; nrl > 0 && sc0 < d.sn; sc0 += kCap) {
                const int nsl = build_list(src.s_box, d.s0 + sc0, min((uint32_t)kCap, d.sn - sc0), sm.seg_r, delta0, th,
                                           hier, sm.sl, &sm.cnt[4]);
                for (int rt0 = 0; nsl > 0 && rt0 < nrl; rt0 += kRT) {
                    const int rcnt = min(kRT, nrl - rt0);
                    // the r tile and the first s tile in flight together
                    if (TJ_TILE_BULK) {
                        tile_arm(bar, kTileRecBytes * (uint32_t)(rcnt + min(kST, nsl)));
                        gather_bulk(src.r_box, src.r_geo, src.r_facets, d.r0 + rc0, sm.rl + rt0, rcnt, sm.rc, bar);
                        gather_bulk(src.s_box, src.s_geo, src.s_facets, d.s0 + sc0, sm.sl, min(kST, nsl), sm.sc, bar);
                        tile_wait(bar, bar_phase);
                    } else {
                        __syncwarp();
                        gather_recs(src.r_box, src.r_geo, src.r_facets, d.r0 + rc0, sm.rl + rt0, rcnt, sm.rc);
                        gather_recs(src.s_box, src.s_geo, src.s_facets, d.s0 + sc0, sm.sl, min(kST, nsl), sm.sc);
                        gather_wait();
                    }
                    __syncwarp();
                    scale_s_tile(min(kST, nsl));
                    for (int st0 = 0; st0 < nsl; st0 += kST) {
                        const int scnt = min(kST, nsl - st0);
                        if (st0 > 0) {
                            if (TJ_TILE_BULK) {
                                tile_arm(bar, kTileRecBytes * (uint32_t)scnt);
                                gather_bulk(src.s_box, src.s_geo, src.s_facets, d.s0 + sc0, sm.sl + st0, scnt, sm.sc, bar);
                                tile_wait(bar, bar_phase);
                            } else {
                                __syncwarp();
                                gather_recs(src.s_box, src.s_geo, src.s_facets, d.s0 + sc0, sm.sl + st0, scnt, sm.sc);
                                gather_wait();
                            }
                            __syncwarp();
                            scale_s_tile(scnt);
                        }
                        float dl = delta0;
                        if (!(dl > 0.f)) { // tile-pair delta0 >= 1e-5 (L_i + L_j) + 1e-12 (M_i + M_j)
                            float Lm = 0.f, Mm = 0.f;
                            if (lane < rcnt) { Lm = fabsf(sm.rc[lane * CS + 3]); Mm = sm.rc[lane * CS + MO]; }
                            if (lane < scnt) {
                                Lm = fmaxf(Lm, fabsf(sm.sc[lane * CS + 3]));
                                Mm = fmaxf(Mm, sm.sc[lane * CS + MO]);
                            }
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) {
                                Lm = fmaxf(Lm, __shfl_xor_sync(0xffffffffu, Lm, o));
                                Mm = fmaxf(Mm, __shfl_xor_sync(0xffffffffu, Mm, o));
                            }
                            dl = __fadd_ru(__fmul_ru(2e-5f, Lm), __fmul_ru(2e-12f, Mm));
                        }
                        // Stage 1, register-blocked: lane -> r facet i (its record in registers)
                        // and s facets j = jj, jj + P, ... (shared-memory reads that the P-lane
                        // groups share as broadcasts); P = lanes per r facet.
                        const bool lb_settled = th.lb_sat || th.lb_u == 0.f;
                        const float ninf = __int_as_float(0xff800000);
                        if (lane == 0) sm.cnt[0] += (uint32_t)(rcnt * scnt);
#ifdef TJ_DEBUG_OPSTATS
                        if (lane == 0 && g_dbg_op_tested) atomicAdd(g_dbg_op_tested + d.op, (unsigned long long)(rcnt * scnt));
#endif
                        if (!cull) { // every pair to the exact queue
                            const int P = rcnt >= 32 ? 1 : 32 / rcnt;
                            const int bi = min(lane / P, rcnt - 1), jj = lane - (lane / P) * P;
                            const bool row_on = lane / P < rcnt;
                            const int iters = (scnt - jj + P - 1) / P, max_iters = (scnt + P - 1) / P;
                            for (int t = 0; t < max_iters; ++t) {
                                const bool nn = row_on && t < iters;
                                queue_push(q, nn, d.op, (uint32_t)(d.r0 + rc0 + sm.rl[rt0 + bi]),
                                           (uint32_t)(d.s0 + sc0 + sm.sl[st0 + (nn ? jj + t * P : 0)]));
                            }
                            continue;
                        }
                        // Stage 1, register-blocked, in row passes: a pass takes `rows` r facets
                        // (32, 16 or the rest) with P = 32 / rows lanes per r facet, so a 24-row
                        // tile runs as 16 + 8 rows on all 32 lanes instead of 24 lanes.
                        int nq = 0, qh = 0; // the warp's stage-2 ring: nq entries from sm.q[qh]
                        for (int rp0 = 0; rp0 < rcnt;) {
                            const int left = rcnt - rp0;
                            // (TJ_ROWS_SINGLE: TJ_ROWS_SINGLE_MIN..31 rows in one pass at P = 1: one pass fewer
                            // for the same iterations)
                            const int rows = left >= 32 ? 32 : (TJ_ROWS_SINGLE && left >= TJ_ROWS_SINGLE_MIN) ? left : left > 16 ? 16 : left;
                            const bool final_pass = rp0 + rows >= rcnt;
                            // small-integer quotients by float reciprocal (x / P for 0 <= x < 64,
                            // P <= 32: the + 0.5 keeps the product >= 1/64 away from integers, far
                            // beyond the reciprocal's rounding)
                            const int P = (int)__fdividef(32.5f, (float)rows);
                            const float rP = __fdividef(1.f, (float)P);
                            const int lq = (int)(((float)lane + 0.5f) * rP);
                            const int bi = rp0 + min(lq, rows - 1), jj = lane - lq * P;
                            const bool row_on = lq < rows;
                            rp0 += rows;
                            const RowRec ar = load_row(sm.rc + bi * CS, QO);
                            // per-row thresholds of the stage-1 pair test, pre-scaled by 1 / c (stage1_box)
                            const float rlb = lb_settled ? ninf : __fadd_ru(__fadd_ru(th.lb_u, dl), ar.ph);
                            const float rub = th.ub_u == 0.f ? ninf : __fsub_ru(__fadd_ru(th.ub_u, dl), ar.hd);
                            const float rlbc = __fmul_ru(rlb, kInvC), rubc = __fmul_ru(rub, kInvC);
                            const int iters = (int)(((float)(scnt - jj + P - 1) + 0.5f) * rP); // this lane's s facets
                            // The lane's s facets (jj + t P) into bit masks: bit t of `nmask` = the
                            // pair goes to stage 2; of `fmask` = a near pair whose DP4A conditioning
                            // pre-test failed (its FP32 test runs at the flush, 32 pairs at a time).
                            uint32_t nmask = 0, fmask = 0;
                            if (row_on) {
                                const float* bp0 = sm.sc + jj * CS;
                                if (TJ_S1_UBSPEC && shapes_ok && th.ub_u == 0.f)
                                    stage1_row<false, kBF, false>(ar, bp0, P * CS, iters, rlbc, rubc, nmask, fmask);
                                else if (shapes_ok)
                                    stage1_row<false, kBF>(ar, bp0, P * CS, iters, rlbc, rubc, nmask, fmask);
                                else
                                    stage1_row<true, kBF>(ar, bp0, P * CS, iters, rlbc, rubc, nmask, fmask);
                            }
                            // compact the masks into the warp queue one entry per lane and round;
                            // stage 2 runs whenever 32 entries are queued (and on the rest after
                            // the final pass: the entries index this tile's records)
                            for (;;) {
                                bool more, last;
                                if constexpr ((kBF && TJ_QUEUE_SCAN) || TJ_QUEUE_SCAN == 2) {
                                // every lane's entries at once, placed by a warp prefix sum of the
                                // mask counts (as many as the ring has room for; the rest next round)
                                more = false;
                                if (__ballot_sync(0xffffffffu, nmask != 0)) {
                                    const int c = __popc(nmask);
                                    int x = c;
#pragma unroll
                                    for (int o = 1; o < 32; o <<= 1) {
                                        const int y = __shfl_up_sync(0xffffffffu, x, o);
                                        if (lane >= o) x += y;
                                    }
                                    const int total = __shfl_sync(0xffffffffu, x, 31);
                                    const int room = kQueue - nq;
                                    int pos = x - c;
                                    while (nmask != 0 && pos < room) {
                                        const int t = __ffs(nmask) - 1;
                                        nmask &= nmask - 1;
                                        sm.q[(qh + nq + pos) & (kQueue - 1)] =
                                            (uint16_t)(((fmask >> t) & 1u ? 0x8000 : 0) | (bi << 5) | (jj + t * P));
                                        ++pos;
                                    }
                                    nq += min(total, room);
                                    more = total > room;
                                }
                                last = !more && final_pass;
                                } else {
                                const bool has = nmask != 0;
                                const unsigned bal = __ballot_sync(0xffffffffu, has);
                                if (has) {
                                    const int t = __ffs(nmask) - 1;
                                    nmask &= nmask - 1;
                                    sm.q[(qh + nq + __popc(bal & ((1u << lane) - 1u))) & (kQueue - 1)] =
                                        (uint16_t)(((fmask >> t) & 1u ? 0x8000 : 0) | (bi << 5) | (jj + t * P));
                                }
                                nq += __popc(bal);
                                more = bal != 0;
                                last = !more && final_pass;
                                }
                                while (nq >= 32 || (last && nq > 0)) { // second stage on up to 32 queued pairs
                                    const int n = min(nq, 32);
                                    __syncwarp();
                                    bool need = false;
                                    uint32_t fr = 0, fs = 0;
                                    bool go = false, ver = false;
                                    if (lane < n) {
                                        const int e = sm.q[(qh + lane) & (kQueue - 1)];
                                        const int i = (e >> 5) & 31, j = e & 31;
                                        const float* ra = sm.rc + i * kCS;
                                        const float* sb = sm.sc + j * kCS;
                                        // a flagged entry is a near pair stage 1 found skippable by its box
                                        // (so cannot_improve and the shape / range terms hold) whose DP4A
                                        // pre-test failed: its ill-conditioned combinations only, and where
                                        // the plane sides clear them all (sat_needed's first exit) no more
                                        bool full = !(e & 0x8000);
                                        if (!full) {
                                            const int m = TJ_FLAG_QMASK ? ill_mask_q(ra, sb) : ill_mask_fp32(ra, sb);
                                            if (m) {
                                                go = true;
                                                const double* va = reinterpret_cast<const double*>(ra + kV0Off);
                                                const double* vb = reinterpret_cast<const double*>(sb + kV0Off);
                                                const float off[3] = {(float)(vb[0] - va[0]), (float)(vb[1] - va[1]),
                                                                      (float)(vb[2] - va[2])};
                                                full = plane_clear(m, sat_frame(ra, sb, off), ra, sb) != 0;
                                            }
                                        } else {
                                            go = true;
                                        }
                                        if (full) {
                                            fr = (uint32_t)(d.r0 + rc0 + sm.rl[rt0 + i]);
                                            fs = (uint32_t)(d.s0 + sc0 + sm.sl[st0 + j]);
                                            const int r = sat_needed(ra, sb, src.r_facets + (size_t)fr * 12,
                                                                     src.s_facets + (size_t)fs * 12, th);
                                            need = r & 1;
                                            ver = r >> 1;
                                        }
                                    }
#if TJ_FLAG_QMASK
                                    // every entry goes on (a flagged entry's DP4A mask is never empty);
                                    // verifications are rare: shared-memory atomics by their lanes
                                    (void)go;
                                    if (lane == 0) sm.cnt[1] += (uint32_t)n;
                                    if (ver) atomicAdd(&sm.cnt[2], 1u);
#else
                                    const unsigned ngo = __popc(__ballot_sync(0xffffffffu, go));
                                    const unsigned nver = __popc(__ballot_sync(0xffffffffu, ver));
                                    if (lane == 0) {
                                        sm.cnt[1] += ngo;
                                        sm.cnt[2] += nver;
                                    }
#endif
                                    queue_push(q, need, d.op, fr, fs);
                                    __syncwarp();
                                    qh = (qh + n) & (kQueue - 1);
                                    nq -= n;
                                }
                                if (!more) break;
                            }
                        }
                    }
                }
            }
        }
        }
    }
    if (counters) {
        __syncwarp();
        if (lane == 0) {
            atomicAdd(counters + 0, (unsigned long long)sm.cnt[0]);
            atomicAdd(counters + 3, (unsigned long long)sm.cnt[1]);
            atomicAdd(counters + 4, (unsigned long long)sm.cnt[2]);
            atomicAdd(counters + 5, (unsigned long long)sm.cnt[3]);
            atomicAdd(counters + 6, (unsigned long long)sm.cnt[4]);
        }
    }
}

// Exact evaluation of the queued facet pairs: thread per pair, records staged in the
// thread's own shared-memory slots, minima folded into the op bits with atomicMin.
#ifndef TJ_EVAL_MINB
#define TJ_EVAL_MINB 1
#endif
__global__ void __launch_bounds__(128, TJ_EVAL_MINB) k_eval(RefineSource src, RefineQueue q, unsigned long long* __restrict__ lb_bits,
                                              unsigned long long* __restrict__ ub_bits, unsigned long long* counters,
                                              int cull) {
    __shared__ double rec[128][2][kFacetWords];
    // decision mode: a pair of an op whose answer is already settled on both sides (min lb 0;
    // min ub 0 or impossible at this level) cannot change the op's outcome
    const bool ub_settled = level_ub_settled(src, cull);
    const uint32_t ra = smem_addr(&rec[threadIdx.x][0][0]), sb = smem_addr(&rec[threadIdx.x][1][0]);
    unsigned long long n = *q.count;
    if (blockIdx.x == 0 && threadIdx.x == 0 && n > q.capacity) atomicMax(q.count + 1, n); // overflow record
    if (n > q.capacity) n = q.capacity;
    unsigned long long done = 0;
    for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
         k += (unsigned long long)gridDim.x * blockDim.x) {
        const PairRef p = q.items[k];
        if (cull == 2 && !exact_op(src.exact_mask, p.op) && bits_to_double(__ldcg(lb_bits + p.op)) == 0.0 &&
            (ub_settled || bits_to_double(__ldcg(ub_bits + p.op)) == 0.0))
            continue;
        double c[12];
        double n2, s2;
        load_facet(src.r_facets + (size_t)p.fr * 12, c);
        stage_exact(c, src.zero_pad ? 0.0 : c[9], src.zero_pad ? 0.0 : c[10], ra, &n2, &s2);
        load_facet(src.s_facets + (size_t)p.fs * 12, c);
        stage_exact(c, src.zero_pad ? 0.0 : c[9], src.zero_pad ? 0.0 : c[10], sb, &n2, &s2);
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

constexpr size_t kScreenSmem = sizeof(ScreenSmem) * (kScreenThreads / 32);

inline int warp_grid(uint64_t warps, int num_sms, int per_sm, int warps_per_block = 8) {
    return (int)std::max<uint64_t>(
        1, std::min<uint64_t>((warps + warps_per_block - 1) / warps_per_block, (uint64_t)num_sms * per_sm));
}

} // namespace

void refine_prep(const double* facets, uint64_t n, float4* out, unsigned* agg, int num_sms, cudaStream_t st,
                 int zero_pad) {
    if (!n) return;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 16));
    count_launch();
    k_prep<<<grid, 256, 0, st>>>(facets, n, out, agg, zero_pad, nullptr, 0, 0);
    TJ_CUDA(cudaGetLastError());
}

void RefineQueueStore::reset(cudaStream_t st) {
    TJ_CUDA(cudaMemsetAsync(count.p, 0, 16, st));
}

bool RefineQueueStore::grow_if_overflowed(cudaStream_t st) {
    unsigned long long h = 0;
    TJ_CUDA(cudaMemcpyAsync(&h, count.p + 1, 8, cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    if (!h) return false;
    if (h + h / 4 > items.n) items.alloc(h + h / 4);
    cap = 0;
    return true;
}

void refine_debug_op_tested(unsigned long long* p) {
    TJ_CUDA(cudaMemcpyToSymbol(g_dbg_op_tested, &p, sizeof(p)));
}

__global__ void k_init_level_agg(unsigned* agg) {
    if (threadIdx.x < 3) agg[threadIdx.x] = threadIdx.x == 0 ? 0x7f800000u : 0u;
}

namespace {
void derive_alloc(DatasetDev& d, uint32_t li, cudaStream_t st) {
    const uint64_t n = d.level_entries[li];
    if (d.screen.size() <= li) d.screen.resize(li + 1);
    if (d.seg.size() <= li) d.seg.resize(li + 1);
    if (d.screen[li].n < std::max<uint64_t>(n * kScreenRecF4, 1)) d.screen[li].alloc(std::max<uint64_t>(n * kScreenRecF4, 1));
    if (d.seg[li].n < std::max<uint64_t>(3 * d.n_voxels, 1)) d.seg[li].alloc(std::max<uint64_t>(3 * d.n_voxels, 1));
    if (d.agg.n < 3 * d.levels.size()) d.agg.alloc(3 * d.levels.size());
    count_launch();
    k_init_level_agg<<<1, 32, 0, st>>>(d.agg.p + 3 * li);
    d.bytes += n * kScreenRecF4 * 16 + 3 * d.n_voxels * 16;
}
} // namespace

void derive_level(DatasetDev& d, uint32_t li, int num_sms, cudaStream_t st) {
    derive_alloc(d, li, st);
    refine_prep(d.facets[li].p, d.level_entries[li], d.screen[li].p, d.agg.p + 3 * li, num_sms, st);
    refine_seg_prep(d.screen[li].p, d.facet_offsets[li].p, d.n_voxels, d.seg[li].p, num_sms, st);
}

void derive_level_range(DatasetDev& d, uint32_t li, uint64_t v_begin, uint64_t v_end, bool first, int num_sms,
                        cudaStream_t st) {
    if (first) derive_alloc(d, li, st);
    if (v_end <= v_begin) return;
    const uint64_t n = d.level_entries[li];
    const uint64_t per = n / std::max<uint64_t>(d.n_voxels, 1) + 1; // records per voxel, for the grid size
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(((v_end - v_begin) * per + 255) / 256,
                                                                    (uint64_t)num_sms * 16));
    count_launch();
    k_prep<<<grid, 256, 0, st>>>(d.facets[li].p, n, d.screen[li].p, d.agg.p + 3 * li, 0, d.facet_offsets[li].p,
                                 v_begin, v_end);
    TJ_CUDA(cudaGetLastError());
    refine_seg_prep(d.screen[li].p, d.facet_offsets[li].p + v_begin, v_end - v_begin, d.seg[li].p + 3 * v_begin,
                    num_sms, st);
}

void refine_seg_prep(const float4* box, const uint64_t* foff, uint64_t n_voxels, float4* seg, int num_sms,
                     cudaStream_t st) {
    if (!n_voxels) return;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n_voxels + 7) / 8, (uint64_t)num_sms * 16));
    count_launch();
    k_seg_prep<<<grid, 256, 0, st>>>(box, foff, n_voxels, seg);
    TJ_CUDA(cudaGetLastError());
}

namespace {
int eval_blocks_per_sm() {
    static std::mutex mu;
    static std::map<int, int> per_dev;
    int dev = 0;
    TJ_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_dev.find(dev);
    if (it != per_dev.end()) return it->second;
    int b = 0;
    TJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_eval, 128, 0));
    return per_dev[dev] = std::max(1, b);
}

// $TRIJOIN_SEED_ONEPASS=1: decision mode seeds every voxel pair in one pass; =2: the ops'
// primary voxel pairs only (tuning / A-B)
int seed_mode() {
    static const int v = [] {
        const char* e = getenv("TRIJOIN_SEED_ONEPASS");
        return e ? atoi(e) : 0;
    }();
    return v;
}
bool two_phase_seeds() { return seed_mode() != 1; }
} // namespace

void refine_pass(const RefineSource& src, uint64_t vp_begin, uint64_t vp_end, bool seed, unsigned long long* lb_bits,
                 unsigned long long* ub_bits, int cull, RefineQueueStore& qs, unsigned long long* work,
                 unsigned long long* counters, int num_sms, cudaStream_t st, cudaEvent_t* screen_ev) {
    if (vp_end <= vp_begin) return;
    // the dynamic shared-memory opt-in is per device: set once per device this process uses
    // (several host threads may drive several GPUs, run_join's shard threads)
    {
        static std::mutex mu;
        static std::set<int> done;
        int dev = 0;
        TJ_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (!done.count(dev)) {
            TJ_CUDA(cudaFuncSetAttribute(k_screen<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kScreenSmem));
            TJ_CUDA(cudaFuncSetAttribute(k_screen<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kScreenSmem));
            done.insert(dev);
        }
    }
    // k_eval: exactly the resident blocks (a grid-stride kernel with even per-block work: a grid
    // beyond one wave would run its surplus blocks in a second, mostly empty wave)
    const int grid = num_sms * eval_blocks_per_sm();
    if (seed) {
        // 2 entries per voxel pair at most
        if (2 * (vp_end - vp_begin) > qs.items.n) qs.items.alloc(2 * (vp_end - vp_begin));
        const int sg = warp_grid(vp_end - vp_begin, num_sms, 4);
        if (cull == 2 && src.active && src.r_seg && src.s_seg && src.n_ops && two_phase_seeds()) {
            // decision mode: the ops' primary voxel pairs seeded and evaluated first, then the
            // other voxel pairs of the ops still open (k_seed_pick)
            qs.pick.reserve(src.n_ops);
            TJ_CUDA(cudaMemsetAsync(qs.pick.p, 0xff, (size_t)src.n_ops * 8, st));
            count_launch();
            k_seed_pick<<<(int)std::min<uint64_t>((vp_end - vp_begin + 255) / 256, (uint64_t)num_sms * 8), 256, 0, st>>>(
                src, vp_begin, vp_end, qs.pick.p);
            TJ_CUDA(cudaMemsetAsync(qs.count.p, 0, 8, st));
            count_launch();
            k_seed<<<sg, 256, 0, st>>>(src, vp_begin, vp_end, qs.view(), cull, 1, qs.pick.p, lb_bits, ub_bits);
            count_launch();
            k_eval<<<grid, 128, 0, st>>>(src, qs.view(), lb_bits, ub_bits, counters, cull);
            TJ_CUDA(cudaMemsetAsync(qs.count.p, 0, 8, st));
            count_launch();
            if (seed_mode() != 2)
                k_seed<<<sg, 256, 0, st>>>(src, vp_begin, vp_end, qs.view(), cull, 2, qs.pick.p, lb_bits, ub_bits);
        } else {
            TJ_CUDA(cudaMemsetAsync(qs.count.p, 0, 8, st));
            count_launch();
            k_seed<<<sg, 256, 0, st>>>(src, vp_begin, vp_end, qs.view(), cull, 0, nullptr, lb_bits, ub_bits);
        }
        TJ_CUDA(cudaGetLastError());
    } else {
        // No host round trip: a queue overflow only drops entries, k_eval records the largest
        // count in count[1] and the caller re-runs the whole level with a larger queue.
        TJ_CUDA(cudaMemsetAsync(qs.count.p, 0, 8, st));
        TJ_CUDA(cudaMemsetAsync(work, 0, 8, st));
        const int sgrid = warp_grid(vp_end - vp_begin, num_sms, kScreenBlocks, kScreenThreads / 32);
        const unsigned batch = screen_batch(src.mean_seg, vp_end - vp_begin, (uint64_t)sgrid * (kScreenThreads / 32));
        count_launch();
        auto* screen = cull == 2 ? k_screen<true> : k_screen<false>;
        if (screen_ev) TJ_CUDA(cudaEventRecord(screen_ev[0], st));
        screen<<<sgrid, kScreenThreads, kScreenSmem, st>>>(src, vp_begin, vp_end, lb_bits, ub_bits, cull, qs.view(), work,
                                                            counters, batch, hier_min_pairs());
        if (screen_ev) TJ_CUDA(cudaEventRecord(screen_ev[1], st));
        TJ_CUDA(cudaGetLastError());
    }
    count_launch();
    k_eval<<<grid, 128, 0, st>>>(src, qs.view(), lb_bits, ub_bits, counters, cull);
    TJ_CUDA(cudaGetLastError());
}

} // namespace tjx
