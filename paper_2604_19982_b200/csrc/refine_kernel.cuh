// Multi-LOD facet refinement on sm_100a (reference refine_kernel, src/refine.cpp:63-84,
// paper Alg. 4): per candidate pair (op), the exact minima over all facet pairs (i, j) of all
// its voxel pairs of
//     lb_ij = max(0, d_ij - ph_i - ph_j)      ub_ij = d_ij + hd_i + hd_j
// with d_ij the reference tri_tri_distance (geom_exact.cuh), bit-identical to the CPU.
//
// Phase-separated design (each phase a tight, converged loop; kernels in refine.cu):
//   prep   : thread per facet of the level; FP32 screening record (7 x float4) computed once;
//   seed   : warp per voxel pair; O(r + s) choice of 2 promising facet pairs (facet box vs the
//            partner segment's box, then the best partner facet) -> exact queue;
//   eval   : thread per queued pair; exact FP64 tri_tri; 64-bit atomicMin of the IEEE bits of
//            lb_ij / ub_ij into the op minima (order-free, exact for non-negative doubles);
//   screen : warp per voxel pair, 32 x 32 facet tiles copied into shared memory; every facet
//            pair is tested in FP32 against the op's thresholds (stage 1: facet-AABB gap;
//            stage 2, box survivors through a per-warp queue: separating-axis bound);
//            survivors -> exact queue, skip candidates with ill-conditioned edge/plane
//            combinations -> verify queue;
//   verify : thread per entry; the reference's FP64 piercing test for those combinations;
//            a firing test sends the pair to the exact queue; then eval runs again.
//
// Exact-preserving screening. The join consumes only
//     lb' = max(iv_lb, min lb_ij)      ub' = min(iv_ub, min ub_ij)      (intersect_interval)
// with [iv_lb, iv_ub] the op's interval before the level. A facet pair is skipped only if it
// provably cannot change lb' or ub', with B_ij a rigorous lower bound of the exact triangle
// distance (outward-rounded facet-AABB gap, or the separating-axis bound minus its rounding
// error bound) and T_lb / T_ub the op minima after the seeds:
//     lb side:  T_lb <= iv_lb (lb' is already iv_lb), or T_lb == 0, or B - ph_i - ph_j >= T_lb + delta
//     ub side:  T_ub == 0, or B + hd_i + hd_j >= min(T_ub, iv_ub) + delta
// (per-voxel-pair outputs, tj_refine_batch: each voxel pair is its own op, iv = [0, +inf]).
// The reference's computed d_ij is the distance between two points on the triangles up to
// rounding (clamped Ericson parameters), except (a) the interior case of point_triangle on
// sliver triangles and (b) a spurious edge-piercing "0" on nearly parallel edge/plane
// configurations. (a): both facets must be well shaped (all angles with sin >= 1e-2) and
// B <= 1e3 * min(L_i, L_j). (b): a computed piercing through a well-conditioned combination
// (|cos(edge, normal)| >= 1e-3) needs the segment within ~1e-10 of the triangle, i.e. B below
// delta, where a reference value of 0 is still >= B - delta; pairs with an ill-conditioned
// combination are skipped only after the reference's FP64 piercing test for that combination
// came out negative (verify). delta = 1e-5 (B + L_i + L_j) + 1e-12 |coords| dwarfs the FP64
// rounding in that regime. Skipped pairs cannot lower any minimum that matters, so the op's
// lb' and ub' are bit-identical to the exhaustive loop.
#pragma once
#include <cstdint>

#include "geom_exact.cuh"
#include "tj_internal.cuh"

namespace tjx {

constexpr int kRT = 32;    // r facets per screening tile
constexpr int kST = 32;    // s facets per screening tile
// Shared-memory stride of a staged screening record (floats): 0-31 the record, 32-33 (s tiles)
// ph and hd pre-scaled for stage 1, 36-41 the facet's v0 in FP64 (the separating-axis frame
// offset), the rest padding; 44 floats = 176 B keeps the per-lane 16-B row loads conflict-free
// (12 i mod 32 over 8 lanes).
constexpr int kCS = 44;
constexpr int kV0Off = 36; // FP64 v0 in a staged record (float index; 16-B aligned)
constexpr int kRecF4 = kScreenRecF4; // float4 per screening record (floats 0-31)
constexpr int kBoxF4 = 3;  // box part of a record (floats 0-11), its own array: 3 float4 per facet
constexpr int kGeoF4 = 5;  // geometry part (floats 12-31): 5 float4 per facet
#ifndef TJ_GATHER_FIXED_PART
#define TJ_GATHER_FIXED_PART 0 // gather_recs: one record part per lane (measured slower: B 50.9 -> 59.6 ms)
#endif
#ifndef TJ_FLAG_QMASK
#define TJ_FLAG_QMASK 1 // flagged stage-2 entries: DP4A per-combination mask instead of FP32 dots
#endif
#ifndef TJ_S1_UBSPEC
#define TJ_S1_UBSPEC 0 // stage 1: a loop variant for ub-settled voxel pairs (measured: B 48.9 vs 49.2 ms, C no gain)
#endif
#ifndef TJ_QUEUE_SCAN
#define TJ_QUEUE_SCAN 1 // decision mode (k_screen<true>): stage-2 queue fill by a warp prefix sum
                        // of the lanes' mask counts (B 50.9 -> 49.6 ms; k-NN C 178.8 -> 182.5, so not there)
#endif

// per-warp stage-2 queue: < 32 pending + 32 new per compaction round, or (TJ_QUEUE_SCAN) a
// whole row pass's entries at once when they fit
constexpr int kQueue = TJ_QUEUE_SCAN ? 256 : 64;
constexpr int kCap = 128;  // per-warp survivor lists: facets per raw segment chunk
// voxel pairs with fewer facet pairs skip the row / column screens (B: 1024 -> 85.9 ms,
// 2048 -> 83.0, 8192 -> 81.3, never -> 81.3; C within 1 %)
constexpr uint32_t kHierMinPairs = 8192;

// Aggregate of a facet segment (or of one facet) for the hierarchical screen: the union of
// the outward-rounded facet boxes and the extreme per-facet quantities the pair tests use.
struct SegAgg {
    float lo[3], hi[3];
    float Lmax;  // max facet L
    float Lmin;  // min facet L
    float phmax; // max ph (rounded up)
    float hdmin; // min hd (rounded down)
    bool ok;     // every facet well shaped
};

// Screening record (floats), one per facet of a level, computed once by k_prep and stored
// as two arrays: the box part (floats 0-11, read by the seed pass and the row/column
// screens) and the geometry part (floats 12-27, only for facets that survive them):
//  0-2 lo (rd)   3 L (ru facet AABB diagonal; negative if the facet is not well shaped)
//  4-6 hi (ru)   7 hd (rd)
//  8-10 unit normal   11 ph (ru)
//  12-20 unit edge directions (v1-v0, v2-v1, v0-v2)
//  21-23 v1 - v0   24-26 v2 - v0   (FP64 differences rounded to FP32)   27 M (max |coordinate|)
//  28-31 (int bits) the unit normal and the 3 unit edge directions quantised to int8x3
//        (round(127 x), 4th byte 0) for the DP4A conditioning pre-test (well_cond_q)
constexpr int kQOff = 28;  // quantised directions in a record
constexpr int kMOff = 27;  // M in a record

struct __align__(16) ScreenSmem {
    float rc[kRT * kCS];
    float sc[kST * kCS];
    uint16_t q[kQueue];
    uint16_t rl[kCap]; // surviving r facets of the current raw chunk (offsets in the chunk)
    uint16_t sl[kCap]; // surviving s facets
    SegAgg seg_r, seg_s; // aggregates of the current voxel pair's segments
    // the current work batch: per voxel pair (lane) its segments, op and thresholds
    struct BatchVp {
        uint32_t r0, s0;
        uint32_t op, gvr, gvs, rn, sn;
        float lb_u, ub_u;
        float d0;  // delta0 of the whole voxel pair (vp_screen; 0: none, the tiles compute their own)
        int flags; // bit 0: lb side settled; bit 1: every facet pair meets the shape / range terms (shapes_settled)
    } vpd[32];
    // the warp's counters (lane 0 writes; kept out of registers: the stage-1 loop is at the
    // register limit): tested, separating-axis tests, verified, voxel pairs skipped, dropped
    uint32_t cnt[5];
    uint64_t bar; // the warp's tile mbarrier (TMA bulk staging)
};

__device__ __forceinline__ float rd(double x) { return __double2float_rd(x); }
__device__ __forceinline__ float ru(double x) { return __double2float_ru(x); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void load_facet(const double* __restrict__ g, double* c) {
    const double2* g2 = reinterpret_cast<const double2*>(g);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 t = __ldg(g2 + k);
        c[2 * k] = t.x;
        c[2 * k + 1] = t.y;
    }
}

// int8x3 quantisation of an FP32 unit vector: round(127 x) per component, 4th byte 0.
__device__ __forceinline__ int quant_dir(const float* u) {
    int q = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) q |= (__float2int_rn(127.f * fminf(1.f, fmaxf(-1.f, u[k]))) & 0xff) << (8 * k);
    return q;
}

// Screening record of one facet record (TJ_FACET_STRIDE doubles).
__device__ __forceinline__ void make_screen(const double* __restrict__ g, float* cr) {
    double c[12];
    load_facet(g, c);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        cr[d] = rd(fmin(fmin(c[d], c[3 + d]), c[6 + d]));
        cr[4 + d] = ru(fmax(fmax(c[d], c[3 + d]), c[6 + d]));
    }
    const float dx = __fsub_ru(cr[4], cr[0]), dy = __fsub_ru(cr[5], cr[1]), dz = __fsub_ru(cr[6], cr[2]);
    // facet AABB diagonal, rounded up (hardware sqrt is within 2 ulp; 1 + 2^-20 covers it)
    const float L = __fmul_ru(sqrtf(__fadd_ru(__fadd_ru(__fmul_ru(dx, dx), __fmul_ru(dy, dy)), __fmul_ru(dz, dz))),
                              1.0f + 0x1p-20f);
    const V3 v0 = {c[0], c[1], c[2]}, v1 = {c[3], c[4], c[5]}, v2 = {c[6], c[7], c[8]};
    double n2, s2;
    const bool degen = tri_degenerate(v0, v1, v2, &n2, &s2);
    const bool ok = !degen && n2 >= TJ_MUL(TJ_MUL(1e-4, s2), s2);
    cr[3] = ok ? L : -(L + 1e-30f); // strictly negative: not well shaped
    cr[7] = rd(c[9]);
    cr[11] = ru(c[10]);
    const V3 e01 = vsub(v1, v0), e12 = vsub(v2, v1), e20 = vsub(v0, v2), e02 = vsub(v2, v0);
    const V3 es[4] = {vcross(e01, e02), e01, e12, e20};
    const int at[4] = {8, 12, 15, 18};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double l2 = vnorm2(es[k]);
        const double inv = l2 > 0.0 ? rsqrt(l2) : 0.0;
        cr[at[k]] = (float)(es[k].x * inv);
        cr[at[k] + 1] = (float)(es[k].y * inv);
        cr[at[k] + 2] = (float)(es[k].z * inv);
    }
    cr[21] = (float)e01.x;
    cr[22] = (float)e01.y;
    cr[23] = (float)e01.z;
    cr[24] = (float)e02.x;
    cr[25] = (float)e02.y;
    cr[26] = (float)e02.z;
    cr[27] = fmaxf(fmaxf(fmaxf(fabsf(cr[0]), fabsf(cr[1])), fmaxf(fabsf(cr[2]), fabsf(cr[4]))),
                   fmaxf(fabsf(cr[5]), fabsf(cr[6]))); // M: max |coordinate|
#pragma unroll
    for (int k = 0; k < 4; ++k) cr[28 + k] = __int_as_float(quant_dir(cr + at[k]));
}

// Rigorous lower bound of the gap between two outward-rounded boxes (lo at b+0, hi at b+4).
__device__ __forceinline__ float box_gap_lb(const float* a, const float* b) {
    float s = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const float g = fmaxf(0.f, fmaxf(__fsub_rd(b[d], a[4 + d]), __fsub_rd(a[d], b[4 + d])));
        s = __fadd_rd(s, __fmul_rd(g, g));
    }
    // lower bound of sqrt(s): hardware sqrt (<= 2 ulp error) scaled down by 1 - 2^-20
    return __fmul_rd(sqrtf(s), 1.0f - 0x1p-20f);
}

// 1 / c with c = 1 - 1e-5 (stage1_box, agg_skip), rounded up
constexpr float kInvC = 1.0f / (1.0f - 1e-5f) * (1.0f + 0x1p-20f);

// Screening thresholds (warp-uniform, rounded up); lb_sat: lb' can no longer change.
struct Thresh {
    float lb_u, ub_u;
    bool lb_sat;
};

// True iff a pair with distance lower bound B can change neither lb' nor ub'.
__device__ __forceinline__ bool cannot_improve(float B, const float* a, const float* b, const Thresh& t) {
    const float La = fabsf(a[3]), Lb = fabsf(b[3]);
    const float M = __fadd_ru(a[27], b[27]);
    const float delta = __fadd_ru(__fmul_ru(1e-5f, __fadd_ru(__fadd_ru(B, La), Lb)), __fmul_ru(1e-12f, M));
    const float lbs = __fsub_rd(__fsub_rd(B, a[11]), b[11]);
    const float ubs = __fadd_rd(__fadd_rd(B, a[7]), b[7]);
    // a minimum of exactly 0 is the floor (lb_ij, ub_ij >= 0): that side needs no test
    const bool lb_ok = t.lb_sat || t.lb_u == 0.f || lbs >= __fadd_ru(t.lb_u, delta);
    const bool ub_ok = t.ub_u == 0.f || ubs >= __fadd_ru(t.ub_u, delta);
    return lb_ok && ub_ok;
}

// Warp reduction of the box parts of facets [first, first + n) (all lanes call).
__device__ __forceinline__ SegAgg seg_reduce(const float4* __restrict__ box, uint64_t first, uint32_t n) {
    const float kInfF = __int_as_float(0x7f800000);
    SegAgg g;
    g.lo[0] = g.lo[1] = g.lo[2] = kInfF;
    g.hi[0] = g.hi[1] = g.hi[2] = -kInfF;
    g.Lmax = 0.f;
    g.Lmin = kInfF;
    g.phmax = 0.f;
    g.hdmin = kInfF;
    bool ok = true;
    const int lane = threadIdx.x & 31;
    for (uint32_t i = lane; i < n; i += 32) {
        const float4* f = box + (first + i) * kBoxF4;
        const float4 a = __ldg(f), b = __ldg(f + 1), c = __ldg(f + 2);
        g.lo[0] = fminf(g.lo[0], a.x); g.lo[1] = fminf(g.lo[1], a.y); g.lo[2] = fminf(g.lo[2], a.z);
        g.hi[0] = fmaxf(g.hi[0], b.x); g.hi[1] = fmaxf(g.hi[1], b.y); g.hi[2] = fmaxf(g.hi[2], b.z);
        ok = ok && a.w >= 0.f;
        g.Lmax = fmaxf(g.Lmax, fabsf(a.w));
        g.Lmin = fminf(g.Lmin, fabsf(a.w));
        g.hdmin = fminf(g.hdmin, b.w);
        g.phmax = fmaxf(g.phmax, c.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            g.lo[k] = fminf(g.lo[k], __shfl_xor_sync(0xffffffffu, g.lo[k], o));
            g.hi[k] = fmaxf(g.hi[k], __shfl_xor_sync(0xffffffffu, g.hi[k], o));
        }
        g.Lmax = fmaxf(g.Lmax, __shfl_xor_sync(0xffffffffu, g.Lmax, o));
        g.Lmin = fminf(g.Lmin, __shfl_xor_sync(0xffffffffu, g.Lmin, o));
        g.hdmin = fminf(g.hdmin, __shfl_xor_sync(0xffffffffu, g.hdmin, o));
        g.phmax = fmaxf(g.phmax, __shfl_xor_sync(0xffffffffu, g.phmax, o));
    }
    g.ok = __all_sync(0xffffffffu, ok);
    return g;
}

// Segment aggregates stored per voxel (3 float4: lo.xyz Lmax | hi.xyz Lmin | phmax hdmin ok 0).
__device__ __forceinline__ void seg_store(float4* dst, const SegAgg& g) {
    dst[0] = make_float4(g.lo[0], g.lo[1], g.lo[2], g.Lmax);
    dst[1] = make_float4(g.hi[0], g.hi[1], g.hi[2], g.Lmin);
    dst[2] = make_float4(g.phmax, g.hdmin, g.ok ? 1.f : 0.f, 0.f);
}
__device__ __forceinline__ SegAgg seg_load(const float4* __restrict__ src) {
    const float4 a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2);
    SegAgg g;
    g.lo[0] = a.x; g.lo[1] = a.y; g.lo[2] = a.z; g.Lmax = a.w;
    g.hi[0] = b.x; g.hi[1] = b.y; g.hi[2] = b.z; g.Lmin = b.w;
    g.phmax = c.x;
    g.hdmin = c.y;
    g.ok = c.z != 0.f;
    return g;
}

// Max |coordinate| of a segment (bounds every facet's M).
__device__ __forceinline__ float seg_m(const SegAgg& g) {
    return fmaxf(fmaxf(fmaxf(fabsf(g.lo[0]), fabsf(g.lo[1])), fmaxf(fabsf(g.lo[2]), fabsf(g.hi[0]))),
                 fmaxf(fabsf(g.hi[1]), fabsf(g.hi[2])));
}

// Aggregated skip test (hierarchical screen): true only if EVERY facet pair (x, y) with x's
// box inside box a and y's box inside box b passes the pair screen's skip conditions, i.e.
// the stage-1 box condition (stage1_box) and skip_mask == 0 (far branch), given
//   lsum  >= L_x + L_y,  lmin <= min(L_x, L_y)   (all facets well shaped),
//   phsum >= ph_x + ph_y (rounded up),   hdsum <= hd_x + hd_y (rounded down),
//   delta0 >= 1e-5 (L_x + L_y) + 1e-12 (M_x + M_y).
// Every quantity is monotone in the right direction: the union-box gap lower-bounds each
// pair's box gap (directed rounding), and the farthest-point distance Bmax (rounded up)
// upper-bounds it.
__device__ __forceinline__ bool agg_skip(const float* alo, const float* ahi, const float* blo, const float* bhi,
                                         float lsum, float lmin, float phsum, float hdsum, float delta0,
                                         const Thresh& t) {
    float g2 = 0.f, m2 = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const float g = fmaxf(0.f, fmaxf(__fsub_rd(blo[d], ahi[d]), __fsub_rd(alo[d], bhi[d])));
        g2 = __fadd_rd(g2, __fmul_rd(g, g));
        const float m = fmaxf(__fsub_ru(bhi[d], alo[d]), __fsub_ru(ahi[d], blo[d]));
        m2 = __fadd_ru(m2, __fmul_ru(m, m));
    }
    const bool lb_settled = t.lb_sat || t.lb_u == 0.f;
    const float xl = __fadd_ru(__fadd_ru(t.lb_u, delta0), phsum);
    const float yu = __fsub_ru(__fadd_ru(t.ub_u, delta0), hdsum);
    const float xs = __fmul_ru(xl, kInvC), ys = __fmul_ru(yu, kInvC);
    const bool lb_ok = lb_settled || xl <= 0.f || g2 >= __fmul_ru(xs, xs);
    const bool ub_ok = t.ub_u == 0.f || yu <= 0.f || g2 >= __fmul_ru(ys, ys);
    const float B = __fmul_rd(sqrtf(g2), 1.0f - 0x1p-20f);
    const bool far = B > 2.f * lsum;                   // skip_mask's far branch for every pair
    const bool near = __fsqrt_ru(m2) <= 1e3f * lmin;   // no pair beyond skip_mask's 1e3 L range
    return lb_ok && ub_ok && far && near;
}

// The r-side part of the register-blocked stage-1 loop (floats 0-7, 11 and the quantised
// directions 28-31 of a screening record, held in registers by the lane owning the r facet).
struct RowRec {
    float lo[3], hi[3], L, hd, ph;
    int q[4];
};

__device__ __forceinline__ RowRec load_row(const float* a, int qoff = kQOff) {
    RowRec r;
    const float4 p0 = *reinterpret_cast<const float4*>(a), p1 = *reinterpret_cast<const float4*>(a + 4);
    const int4 pq = *reinterpret_cast<const int4*>(a + qoff);
    r.lo[0] = p0.x; r.lo[1] = p0.y; r.lo[2] = p0.z; r.L = p0.w;
    r.hi[0] = p1.x; r.hi[1] = p1.y; r.hi[2] = p1.z; r.hd = p1.w;
    r.ph = a[11];
    r.q[0] = pq.x; r.q[1] = pq.y; r.q[2] = pq.z; r.q[3] = pq.w;
    return r;
}

// |u . v| < 1e-3 for unit vectors (a conditioning cutoff; FMA only sharpens the dot).
__device__ __forceinline__ bool ill_cond(float ux, float uy, float uz, float vx, float vy, float vz) {
    return fabsf(__fmaf_rn(ux, vx, __fmaf_rn(uy, vy, __fmul_rn(uz, vz)))) < 1e-3f;
}

// DP4A pre-test of the 6 edge / normal combinations: true only if every |e . n| of the FP32
// unit vectors exceeds 1e-3. With q = round(127 x) per component, |q_u . q_v / 127^2 - u . v|
// <= 2 * sqrt(3) * 0.5 / 127 + 3 (0.5 / 127)^2 < 0.01370, so |q_u . q_v| > 16129 * 0.01470
// (= 237.1) implies |u . v| > 1e-3.
__device__ __forceinline__ bool well_cond_q(const int* aq, int4 bq) {
    constexpr unsigned kT = 238;
    const int d0 = __dp4a(aq[1], bq.x, 0), d1 = __dp4a(aq[2], bq.x, 0), d2 = __dp4a(aq[3], bq.x, 0);
    const int d3 = __dp4a(bq.y, aq[0], 0), d4 = __dp4a(bq.z, aq[0], 0), d5 = __dp4a(bq.w, aq[0], 0);
    // (unsigned)(d + T) > 2 T  <=>  |d| > T
    return (unsigned)(d0 + (int)kT) > 2 * kT && (unsigned)(d1 + (int)kT) > 2 * kT &&
           (unsigned)(d2 + (int)kT) > 2 * kT && (unsigned)(d3 + (int)kT) > 2 * kT &&
           (unsigned)(d4 + (int)kT) > 2 * kT && (unsigned)(d5 + (int)kT) > 2 * kT;
}

// Box part of stage 1 for one pair, branch-free: 1 = the pair must go to stage 2 (it may
// change a minimum, or it is out of the skip argument's shape / range), 2 = skippable by its
// box gap but near (the edge / plane conditioning decides), 0 = skippable (far apart).
// The box condition uses the squared box gap g2 = B^2 against the row thresholds
// rlb = T_lb + delta0 + ph_i, rub = T_ub + delta0 - hd_i: with c = 1 - 1e-5 and
// delta0 >= 1e-5 (L_i + L_j) + 1e-12 (M_i + M_j),
//   lb side: c B >= T_lb + delta0 + ph_i + ph_j   implies  B - ph_i - ph_j >= T_lb + delta(B)
//   ub side: c B >= T_ub + delta0 - hd_i - hd_j   implies  B + hd_i + hd_j >= T_ub + delta(B)
// i.e. cannot_improve with a (larger) tile-wide delta. Everything is pre-scaled by 1 / c with
// upward rounding: rlbc >= rlb / c and phc >= ph_j / c per row / s record (hdc <= hd_j / c),
// so xs = rlbc + phc >= (rlb + ph_j) / c and ys = rubc - hdc >= (rub - hd_j) / c; both sides
// hold iff max(xs, ys) <= 0 or g2 >= max(xs, ys)^2 (squares of non-negative values compared,
// directed rounding; the FMAs round once, downwards, so g2 stays a lower bound).
// kShapes = false when the voxel pair is known to meet the shape / range terms for every
// facet pair (shapes_settled); kUb = false when the voxel pair's ub side is settled (rubc = -inf,
// so z is the lb side's term alone).
template <bool kShapes, bool kUb = true>
__device__ __forceinline__ int stage1_box(const RowRec& a, float4 b0, float4 b1, float2 pc, float rlbc, float rubc) {
    const float gx = fmaxf(0.f, fmaxf(__fsub_rd(b0.x, a.hi[0]), __fsub_rd(a.lo[0], b1.x)));
    const float gy = fmaxf(0.f, fmaxf(__fsub_rd(b0.y, a.hi[1]), __fsub_rd(a.lo[1], b1.y)));
    const float gz = fmaxf(0.f, fmaxf(__fsub_rd(b0.z, a.hi[2]), __fsub_rd(a.lo[2], b1.z)));
    const float g2 = __fmaf_rd(gz, gz, __fmaf_rd(gy, gy, __fmul_rd(gx, gx)));
    const float z = kUb ? fmaxf(__fadd_ru(rlbc, pc.x), __fsub_ru(rubc, pc.y)) : __fadd_ru(rlbc, pc.x);
    bool skip = z <= 0.f || g2 >= __fmul_ru(z, z);
    if constexpr (kShapes) {
        const float m = 1e3f * fminf(a.L, b0.w);
        skip = skip && a.L >= 0.f && b0.w >= 0.f && g2 <= m * m;
    }
    const float f = 2.f * (a.L + b0.w);
    return skip ? (g2 > f * f ? 0 : 2) : 1;
}

// Stage 1 of one lane's row (r facet `a` in registers) against its s facets of the staged tile
// (`bp`: the first, `step` floats apart; `iters` of them): bit t of `nmask` = pair t goes to
// stage 2, of `fmask` = a near pair whose DP4A conditioning pre-test failed.
// kBF: the DP4A pre-test runs for every pair, branch-free, two pairs per iteration (faster when
// most tested pairs are near, as in decision mode: config B 60.5 -> 58.1 ms); otherwise behind
// a branch (faster when most are far: config C 199 -> 192 ms).
template <bool kShapes, bool kBF, bool kUb>
__device__ __forceinline__ void stage1_pair(const RowRec& a, const float* bp, float rlbc, float rubc, uint32_t bit,
                                            uint32_t& nmask, uint32_t& fmask) {
    const float4 b0 = *reinterpret_cast<const float4*>(bp), b1 = *reinterpret_cast<const float4*>(bp + 4);
    const float2 pc = *reinterpret_cast<const float2*>(bp + 32);
    const int sb = stage1_box<kShapes, kUb>(a, b0, b1, pc, rlbc, rubc);
    bool f;
    if constexpr (!kBF) {
        f = sb == 2 && !well_cond_q(a.q, *reinterpret_cast<const int4*>(bp + kQOff));
    } else {
        const bool wc = well_cond_q(a.q, *reinterpret_cast<const int4*>(bp + kQOff));
        f = (sb == 2) & !wc;
    }
    nmask |= ((sb == 1) | f) ? bit : 0u;
    fmask |= f ? bit : 0u;
}

template <bool kShapes, bool kBF, bool kUb = true>
__device__ __forceinline__ void stage1_row(const RowRec& a, const float* bp, int step, int iters, float rlbc, float rubc,
                                           uint32_t& nmask, uint32_t& fmask) {
    uint32_t bit = 1u;
    int t = 0;
    if constexpr (kBF) {
#pragma unroll 1
        for (; t + 1 < iters; t += 2, bp += 2 * step, bit <<= 2) {
            stage1_pair<kShapes, kBF, kUb>(a, bp, rlbc, rubc, bit, nmask, fmask);
            stage1_pair<kShapes, kBF, kUb>(a, bp + step, rlbc, rubc, bit << 1, nmask, fmask);
        }
    }
#pragma unroll 1
    for (; t < iters; ++t, bp += step, bit <<= 1) stage1_pair<kShapes, kBF, kUb>(a, bp, rlbc, rubc, bit, nmask, fmask);
}

// True if every facet pair (x, y) of the two segments meets the shape / range terms of the
// stage-1 skip (both facets well shaped, box gap <= 1e3 min(L_x, L_y)): the segments are
// well shaped and their union boxes' farthest distance (rounded up) is within 1e3 L_min.
__device__ __forceinline__ bool shapes_settled(const SegAgg& a, const SegAgg& b) {
    if (!a.ok || !b.ok) return false;
    float m2 = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const float m = fmaxf(__fsub_ru(b.hi[d], a.lo[d]), __fsub_ru(a.hi[d], b.lo[d]));
        m2 = __fadd_ru(m2, __fmul_ru(m, m));
    }
    const float lim = __fmul_rd(1e3f, fminf(a.Lmin, b.Lmin));
    return m2 <= __fmul_rd(lim, lim);
}

// The ill-conditioned edge / plane combinations of a near, box-skippable pair whose DP4A
// pre-test failed (FP32 dots, |cos| < 1e-3), as a mask in skip_mask's bit order: bit k = edge k of a vs the plane of b, bit 3 + k = edge k of b vs the
// plane of a).
__device__ __forceinline__ int ill_mask_fp32(const float* as, const float* b) {
    const float4 b2 = *reinterpret_cast<const float4*>(b + 8);
    const float4 b3 = *reinterpret_cast<const float4*>(b + 12), b4 = *reinterpret_cast<const float4*>(b + 16);
    const float b20 = b[20];
    const float4 a2 = *reinterpret_cast<const float4*>(as + 8), a3 = *reinterpret_cast<const float4*>(as + 12);
    const float4 a4 = *reinterpret_cast<const float4*>(as + 16);
    const float a20 = as[20];
    return (int)ill_cond(a3.x, a3.y, a3.z, b2.x, b2.y, b2.z) | (int)ill_cond(a3.w, a4.x, a4.y, b2.x, b2.y, b2.z) << 1 |
           (int)ill_cond(a4.z, a4.w, a20, b2.x, b2.y, b2.z) << 2 | (int)ill_cond(b3.x, b3.y, b3.z, a2.x, a2.y, a2.z) << 3 |
           (int)ill_cond(b3.w, b4.x, b4.y, a2.x, a2.y, a2.z) << 4 | (int)ill_cond(b4.z, b4.w, b20, a2.x, a2.y, a2.z) << 5;
}

// The same combinations from the quantised directions (well_cond_q's six DP4A dots, same bit
// order): bit set where |q_u . q_v| <= 238, i.e. wherever the pre-test cannot certify
// |u . v| > 1e-3. A superset of the FP32 mask: every combination the pre-test certifies is
// one whose conditioning the skip argument accepts (stage 1 skips on that certificate alone),
// so clearing this mask's bits by the plane sides is sufficient for a skip.
__device__ __forceinline__ int ill_mask_q(const float* as, const float* b) {
    constexpr int kT = 238;
    const int4 aq = *reinterpret_cast<const int4*>(as + kQOff), bq = *reinterpret_cast<const int4*>(b + kQOff);
    const int d[6] = {__dp4a(aq.y, bq.x, 0), __dp4a(aq.z, bq.x, 0), __dp4a(aq.w, bq.x, 0),
                      __dp4a(bq.y, aq.x, 0), __dp4a(bq.z, aq.x, 0), __dp4a(bq.w, aq.x, 0)};
    int m = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) m |= ((unsigned)(d[k] + kT) <= 2u * kT) ? 1 << k : 0;
    return m;
}

// Shape / range eligibility for a skip and the mask of ill-conditioned edge/plane
// combinations (bit k < 3: edge k of a vs the plane of b; bit 3 + k: edge k of b vs the
// plane of a; |cos(edge, normal)| < 1e-3). Returns -1 if the pair may never be skipped; a
// non-zero mask means the skip additionally needs the reference's own piercing test to be
// negative for those combinations (verify).
__device__ __forceinline__ int skip_mask(float B, const float* a, const float* b) {
    if (a[3] < 0.f || b[3] < 0.f) return -1;
    if (B > 1e3f * fminf(a[3], b[3])) return -1;
    // Far apart (B > 2 (L_a + L_b)): no computed piercing can fire for any conditioning that
    // passes the reference's |det| > 1e-14 scale test (its u, v, t errors are then below ~6%
    // of the vertex-to-triangle distance, which needs the segment within 0.44 (L_a + L_b)).
    if (B > 2.f * (a[3] + b[3])) return 0;
    int mask = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (fabsf(a[12 + 3 * k] * b[8] + a[13 + 3 * k] * b[9] + a[14 + 3 * k] * b[10]) < 1e-3f) mask |= 1 << k;
        if (fabsf(b[12 + 3 * k] * a[8] + b[13 + 3 * k] * a[9] + b[14 + 3 * k] * a[10]) < 1e-3f) mask |= 8 << k;
    }
    return mask;
}

// Separating-axis lower bound of the distance between the two triangles (FP32; a's v0 is the
// origin, `off` = b.v0 - a.v0 rounded from FP64): max over the candidate axes u of the
// projection gap / |u|, minus a bound on its rounding error (projections: <= 3 ulp of |u|*R
// each; vertex rounding to FP32: <= 2^-24 R per coordinate (+ 2^-24 |off| for b); rsqrt:
// 2^-22). Two stages: the 2 face normals (sat_faces), then the 9 edge-edge cross products
// (sat_edges); each result alone is a rigorous lower bound.
struct SatFrame {
    float av[9], bv[9];
    float R;
};

__device__ __forceinline__ SatFrame sat_frame(const float* a, const float* b, const float* off) {
    SatFrame f;
    f.av[0] = f.av[1] = f.av[2] = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        f.av[3 + k] = a[21 + k];
        f.av[6 + k] = a[24 + k];
        f.bv[k] = off[k];
        f.bv[3 + k] = off[k] + b[21 + k];
        f.bv[6 + k] = off[k] + b[24 + k];
    }
    f.R = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) f.R = fmaxf(f.R, fmaxf(fabsf(f.av[k]), fabsf(f.bv[k])));
    return f;
}

__device__ __forceinline__ float sat_axis(const SatFrame& f, float ux, float uy, float uz) {
    const float u2 = __fmaf_rn(ux, ux, __fmaf_rn(uy, uy, __fmul_rn(uz, uz)));
    if (!(u2 > 1e-30f)) return 0.f;
    float amin = 3.4e38f, amax = -3.4e38f, bmin = 3.4e38f, bmax = -3.4e38f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float pa = __fmaf_rn(ux, f.av[3 * k], __fmaf_rn(uy, f.av[3 * k + 1], __fmul_rn(uz, f.av[3 * k + 2])));
        const float pb = __fmaf_rn(ux, f.bv[3 * k], __fmaf_rn(uy, f.bv[3 * k + 1], __fmul_rn(uz, f.bv[3 * k + 2])));
        amin = fminf(amin, pa);
        amax = fmaxf(amax, pa);
        bmin = fminf(bmin, pb);
        bmax = fmaxf(bmax, pb);
    }
    const float gap = fmaxf(bmin - amax, amin - bmax);
    return gap > 0.f ? gap * rsqrtf(u2) : 0.f;
}

// rounding margin: 8e-6 R absolute (>= 16x the analysed bound) + 1e-5 relative
__device__ __forceinline__ float sat_margin(float best, const SatFrame& f) {
    return fmaxf(0.f, best * (1.0f - 1e-5f) - 8e-6f * f.R);
}

__device__ __forceinline__ float sat_faces(const SatFrame& f, const float* a, const float* b) {
    return sat_margin(fmaxf(sat_axis(f, a[8], a[9], a[10]), sat_axis(f, b[8], b[9], b[10])), f);
}

__device__ __forceinline__ float sat_edges(const SatFrame& f, const float* a, const float* b) {
    float best = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float* e = a + 12 + 3 * i;
            const float* g = b + 12 + 3 * j;
            best = fmaxf(best, sat_axis(f, e[1] * g[2] - e[2] * g[1], e[2] * g[0] - e[0] * g[2],
                                        e[0] * g[1] - e[1] * g[0]));
        }
    }
    return sat_margin(best, f);
}

// Clears the bits of an ill-conditioned-combination mask (skip_mask) whose edge lies
// robustly on one side of the other triangle's plane. The reference's piercing test for
// edge (p, q) against triangle (v0, v1, v2) (src/geom.cpp:120-136) computes
//     tt = (e2 . ((p - v0) x e1)) / (e1 . ((q - p) x e2)) = h_p / (h_p - h_q),
// h_x = (x - v0) . (e1 x e2); with both h_p, h_q of one sign and |h| above the FP64
// rounding of numerator and denominator (<= ~8 eps (|p - v0| + |q - p|) |e1| |e2|, i.e. a
// clearance of ~1e-13 R for a well-shaped triangle, sin(angle) >= 1e-2), the computed tt
// cannot land in [0, 1]: no piercing can be reported, whatever the conditioning. Here the
// clearance is the FP32 signed distance to the plane (unit normal; error <= ~2e-6 R in the
// local frame of radius R), required to exceed 3.2e-5 R.
__device__ __forceinline__ int plane_clear(int mask, const SatFrame& f, const float* a, const float* b) {
    const float m = 3.2e-5f * f.R;
    float sa[3], sb[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        // a's vertices against b's plane (through bv[0..2]); b's vertices against a's (origin)
        // FMA dots (one rounding per term: within the analysed error bound)
        sa[k] = __fmaf_rn(b[8], f.av[3 * k] - f.bv[0],
                          __fmaf_rn(b[9], f.av[3 * k + 1] - f.bv[1], __fmul_rn(b[10], f.av[3 * k + 2] - f.bv[2])));
        sb[k] = __fmaf_rn(a[8], f.bv[3 * k], __fmaf_rn(a[9], f.bv[3 * k + 1], __fmul_rn(a[10], f.bv[3 * k + 2])));
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int k1 = k == 2 ? 0 : k + 1;
        if ((sa[k] > m && sa[k1] > m) || (sa[k] < -m && sa[k1] < -m)) mask &= ~(1 << k);
        if ((sb[k] > m && sb[k1] > m) || (sb[k] < -m && sb[k1] < -m)) mask &= ~(8 << k);
    }
    return mask;
}

// The reference's FP64 piercing test (segment_pierces_triangle, src/geom.cpp:120-136) for
// edge (p, q) of one triangle against triangle (v0, v1, v2), with a pre-test: when
// det^2 <= 1e-28 (1 - 1e-12) |dir|^2 |e1|^2 |e2|^2 (same det and squared norms as the
// reference) the reference's |det| <= 1e-14 * norm*norm*norm test is certain to reject, and
// the sqrt-based remainder is skipped. Otherwise the reference test runs unchanged.
__device__ __forceinline__ bool pierces_ref(const V3& p, const V3& q, const V3& v0, const V3& v1, const V3& v2) {
    const V3 dir = vsub(q, p);
    const V3 e1 = vsub(v1, v0), e2 = vsub(v2, v0);
    const V3 pv = vcross(dir, e2);
    const double det = vdot(e1, pv);
    const double n2d = vnorm2(dir), n2a = vnorm2(e1), n2b = vnorm2(e2);
    if (det * det <= 1e-28 * (1.0 - 1e-12) * (n2d * n2a * n2b)) return false;
    const double scale = TJ_MUL(TJ_MUL(TJ_SQRT(n2d), TJ_SQRT(n2a)), TJ_SQRT(n2b));
    if (fabs(det) <= TJ_MUL(1e-14, scale)) return false;
    const double inv = TJ_DIV(1.0, det);
    const V3 tv = vsub(p, v0);
    const double u = TJ_MUL(vdot(tv, pv), inv);
    if (u < 0.0 || u > 1.0) return false;
    const V3 qv = vcross(tv, e1);
    const double v = TJ_MUL(vdot(dir, qv), inv);
    if (v < 0.0 || TJ_ADD(u, v) > 1.0) return false;
    const double tt = TJ_MUL(vdot(e2, qv), inv);
    return tt >= 0.0 && tt <= 1.0;
}

// Exact evaluation of one facet pair from two staged exact records (shared addresses):
// returns (max(0, d - ph_r - ph_s), d + hd_r + hd_s)  (src/refine.cpp:77-79). Not inlined:
// one copy of the geometry serves every call site (instruction-cache footprint).
__device__ __noinline__ double2 eval_pair(uint32_t ra, uint32_t sb) {
    staged_read_barrier();
    const double d = tri_tri(ra, sb);
    const double lbp = smax(0.0, TJ_SUB(TJ_SUB(d, ldw(ra, 10)), ldw(sb, 10)));
    const double ubp = TJ_ADD(TJ_ADD(d, ldw(ra, 9)), ldw(sb, 9));
    return make_double2(lbp, ubp);
}

__device__ __forceinline__ double bits_to_double(unsigned long long b) { return __longlong_as_double((long long)b); }

} // namespace tjx
