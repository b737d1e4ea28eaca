// Multi-LOD facet refinement on sm_100a (reference refine_kernel, src/refine.cpp:63-84,
// paper Alg. 4): per candidate pair (op), the exact minima over all facet pairs (i, j) of all
// its voxel pairs of
//     lb_ij = max(0, d_ij - ph_i - ph_j)      ub_ij = d_ij + hd_i + hd_j
// with d_ij the reference tri_tri_distance (geom_exact.cuh), bit-identical to the CPU.
//
// Phase-separated design (each phase a tight, converged loop; see refine.cu):
//   seed   : warp per voxel pair; the pairs of smallest facet-AABB gap are queued;
//   eval   : thread per queued pair; exact FP64 tri_tri; 64-bit atomicMin of the IEEE bits of
//            lb_ij / ub_ij into the op minima (order-free, exact for non-negative doubles);
//   screen : warp per voxel pair; every facet pair is tested in FP32 against the op's
//            thresholds (stage 1: facet-AABB gap; stage 2, box survivors through a per-warp
//            queue: separating-axis bound); survivors are queued for a second eval.
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
// came out negative (k_verify). delta = 1e-5 (B + L_i + L_j) + 1e-12 |coords| dwarfs the
// FP64 rounding in that regime. Skipped pairs cannot lower any minimum that matters, so the
// op's lb' and ub' are bit-identical to the exhaustive loop.
#pragma once
#include <cstdint>

#include "geom_exact.cuh"

namespace tjx {

constexpr int kRT = 32;    // r facets per screening tile
constexpr int kST = 32;    // s facets per screening tile
constexpr int kCS = 36;    // floats per screening record
constexpr int kQueue = 64; // per-warp SAT queue (< 32 pending + 32 new)

// Screening record layout (floats):
//  0-2 lo (rd)  3-5 hi (ru)  6 L (ru, facet AABB diagonal)  7 M (ru, max |coord|)
//  8 hd (rd)  9 ph (ru)  10 ok (well shaped and non-degenerate)  11 pad
//  12-20 unit edge directions (v1-v0, v2-v1, v0-v2)  21-23 unit normal
//  24-32 v0 v1 v2 relative to the voxel pair's origin  33-35 pad
struct ScreenSmem {
    float rc[kRT * kCS];
    float sc[kST * kCS];
    uint16_t q[kQueue];
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

// Build the FP32 screening record of one facet record (TJ_FACET_STRIDE doubles).
__device__ __forceinline__ void stage_screen(const double* __restrict__ g, const double* o, float* cr) {
    double c[12];
    load_facet(g, c);
    float M = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double lo = fmin(fmin(c[d], c[3 + d]), c[6 + d]);
        const double hi = fmax(fmax(c[d], c[3 + d]), c[6 + d]);
        cr[d] = rd(lo);
        cr[3 + d] = ru(hi);
        M = fmaxf(M, fmaxf(fabsf(cr[d]), fabsf(cr[3 + d])));
    }
    const float dx = __fsub_ru(cr[3], cr[0]), dy = __fsub_ru(cr[4], cr[1]), dz = __fsub_ru(cr[5], cr[2]);
    // facet AABB diagonal, rounded up (hardware sqrt is within 2 ulp; 1 + 2^-20 covers it)
    cr[6] = __fmul_ru(sqrtf(__fadd_ru(__fadd_ru(__fmul_ru(dx, dx), __fmul_ru(dy, dy)), __fmul_ru(dz, dz))),
                      1.0f + 0x1p-20f);
    cr[7] = M;
    cr[8] = rd(c[9]);
    cr[9] = ru(c[10]);
    const V3 v0 = {c[0], c[1], c[2]}, v1 = {c[3], c[4], c[5]}, v2 = {c[6], c[7], c[8]};
    double n2, s2;
    const bool degen = tri_degenerate(v0, v1, v2, &n2, &s2);
    cr[10] = (!degen && n2 >= TJ_MUL(TJ_MUL(1e-4, s2), s2)) ? 1.f : 0.f;
    cr[11] = 0.f;
    const V3 es[4] = {vsub(v1, v0), vsub(v2, v1), vsub(v0, v2), vcross(vsub(v1, v0), vsub(v2, v0))};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double l2 = vnorm2(es[k]);
        const double inv = l2 > 0.0 ? rsqrt(l2) : 0.0;
        cr[12 + 3 * k] = (float)(es[k].x * inv);
        cr[13 + 3 * k] = (float)(es[k].y * inv);
        cr[14 + 3 * k] = (float)(es[k].z * inv);
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) cr[24 + k] = (float)(c[k] - o[k % 3]);
    cr[33] = cr[34] = cr[35] = 0.f;
}

// Rigorous lower bound of the AABB gap (outward-rounded boxes, round-down arithmetic).
__device__ __forceinline__ float box_gap_lb(const float* a, const float* b) {
    float s = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const float g = fmaxf(0.f, fmaxf(__fsub_rd(b[d], a[3 + d]), __fsub_rd(a[d], b[3 + d])));
        s = __fadd_rd(s, __fmul_rd(g, g));
    }
    // lower bound of sqrt(s): hardware sqrt (<= 2 ulp error) scaled down by 1 - 2^-20
    return __fmul_rd(sqrtf(s), 1.0f - 0x1p-20f);
}

// Screening thresholds (warp-uniform, rounded up); lb_sat: lb' can no longer change.
struct Thresh {
    float lb_u, ub_u;
    bool lb_sat;
};

// True iff a pair with distance lower bound B can change neither lb' nor ub'.
__device__ __forceinline__ bool cannot_improve(float B, const float* a, const float* b, const Thresh& t) {
    const float delta =
        __fadd_ru(__fmul_ru(1e-5f, __fadd_ru(__fadd_ru(B, a[6]), b[6])), __fmul_ru(1e-12f, __fadd_ru(a[7], b[7])));
    const float lbs = __fsub_rd(__fsub_rd(B, a[9]), b[9]);
    const float ubs = __fadd_rd(__fadd_rd(B, a[8]), b[8]);
    // a minimum of exactly 0 is the floor (lb_ij, ub_ij >= 0): that side needs no test
    const bool lb_ok = t.lb_sat || t.lb_u == 0.f || lbs >= __fadd_ru(t.lb_u, delta);
    const bool ub_ok = t.ub_u == 0.f || ubs >= __fadd_ru(t.ub_u, delta);
    return lb_ok && ub_ok;
}

// Shape / range eligibility for a skip and the mask of ill-conditioned edge/plane
// combinations (bit k < 3: edge k of a vs the plane of b; bit 3 + k: edge k of b vs the
// plane of a; |cos(edge, normal)| < 1e-3). Returns -1 if the pair may never be skipped; a
// non-zero mask means the skip additionally needs the reference's own piercing test to be
// negative for those combinations (k_verify).
__device__ __forceinline__ int skip_mask(float B, const float* a, const float* b) {
    if (a[10] == 0.f || b[10] == 0.f) return -1;
    if (B > 1e3f * fminf(a[6], b[6])) return -1;
    int mask = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (fabsf(a[12 + 3 * k] * b[21] + a[13 + 3 * k] * b[22] + a[14 + 3 * k] * b[23]) < 1e-3f) mask |= 1 << k;
        if (fabsf(b[12 + 3 * k] * a[21] + b[13 + 3 * k] * a[22] + b[14 + 3 * k] * a[23]) < 1e-3f) mask |= 8 << k;
    }
    return mask;
}

// The reference's FP64 piercing test (segment_pierces_triangle, src/geom.cpp:120-136) for the
// combinations in `mask` on two staged exact records: true iff none fires, i.e. the pair's
// reference distance cannot be a (spurious) piercing 0.
__device__ __noinline__ bool pierce_clear(int mask, uint32_t ra, uint32_t sb) {
#pragma unroll 1
    for (int k = 0; k < 6; ++k) {
        if (!(mask & (1 << k))) continue;
        const uint32_t src = k < 3 ? ra : sb, tri = k < 3 ? sb : ra;
        if (ldw(tri, 14) != 0.0) continue; // degenerate target: the reference never tests it
        const int e = k < 3 ? k : k - 3, e1 = e == 2 ? 0 : e + 1;
        if (segment_pierces(ldv(src, e), ldv(src, e1), ldw(src, 11 + e), tri)) return false;
    }
    return true;
}

// Separating-axis lower bound of the distance between the two triangles (FP32, coordinates
// relative to the voxel pair's origin): max over the 2 face normals and 9 edge-edge cross
// products u of the projection gap / |u|, minus a bound on its rounding error (projections:
// <= 3 ulp of |u|*R each; vertex rounding to FP32: <= 2^-24 * R per coordinate; rsqrt: 2^-22).
__device__ __forceinline__ float sat_lower_bound(const float* a, const float* b) {
    const float* av = a + 24;
    const float* bv = b + 24;
    float R = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) R = fmaxf(R, fmaxf(fabsf(av[k]), fabsf(bv[k])));
    float best = 0.f;
    auto axis = [&](float ux, float uy, float uz) {
        const float u2 = ux * ux + uy * uy + uz * uz;
        if (!(u2 > 1e-30f)) return;
        float amin = 3.4e38f, amax = -3.4e38f, bmin = 3.4e38f, bmax = -3.4e38f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float pa = ux * av[3 * k] + uy * av[3 * k + 1] + uz * av[3 * k + 2];
            const float pb = ux * bv[3 * k] + uy * bv[3 * k + 1] + uz * bv[3 * k + 2];
            amin = fminf(amin, pa);
            amax = fmaxf(amax, pa);
            bmin = fminf(bmin, pb);
            bmax = fmaxf(bmax, pb);
        }
        const float gap = fmaxf(bmin - amax, amin - bmax);
        if (gap > 0.f) best = fmaxf(best, gap * rsqrtf(u2));
    };
    axis(a[21], a[22], a[23]);
    axis(b[21], b[22], b[23]);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float* e = a + 12 + 3 * i;
            const float* f = b + 12 + 3 * j;
            axis(e[1] * f[2] - e[2] * f[1], e[2] * f[0] - e[0] * f[2], e[0] * f[1] - e[1] * f[0]);
        }
    }
    // rounding margin: 8e-6 R absolute (>= 16x the analysed bound) + 1e-5 relative
    return fmaxf(0.f, best * (1.0f - 1e-5f) - 8e-6f * R);
}

// Exact evaluation of one facet pair from two staged exact records (shared addresses):
// returns (max(0, d - ph_r - ph_s), d + hd_r + hd_s)  (src/refine.cpp:77-79). Not inlined:
// one copy of the geometry serves every call site (instruction-cache footprint).
__device__ __noinline__ double2 eval_pair(uint32_t ra, uint32_t sb) {
    const double d = tri_tri(ra, sb);
    const double lbp = smax(0.0, TJ_SUB(TJ_SUB(d, ldw(ra, 10)), ldw(sb, 10)));
    const double ubp = TJ_ADD(TJ_ADD(d, ldw(ra, 9)), ldw(sb, 9));
    return make_double2(lbp, ubp);
}

__device__ __forceinline__ double bits_to_double(unsigned long long b) { return __longlong_as_double((long long)b); }

} // namespace tjx
