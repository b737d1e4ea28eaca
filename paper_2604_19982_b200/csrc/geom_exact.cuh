// Bit-exact FP64 triangle geometry for sm_100a.
//
// Restates the reference primitives (paths relative to /root/reference/proj):
//   mindist_aabb             src/geom.cpp:11-16
//   point_segment_distance   src/geom.cpp:18-24
//   triangle_degenerate      src/geom.cpp:29-35
//   point_triangle_distance  src/geom.cpp:39-80   (Ericson closest point)
//   segment_segment_distance src/geom.cpp:82-113  (Ericson clamped)
//   segment_pierces_triangle src/geom.cpp:120-136
//   triangle_less            src/geom.cpp:140-148
//   tri_tri_distance         src/geom.cpp:152-183
//
// Every add/sub/mul/div/sqrt goes through the IEEE round-to-nearest intrinsics
// (__dadd_rn & co.), which the compiler never contracts into FMA, in the same
// association order as the reference's C++ expressions. Results are therefore
// bit-identical to the reference built without FMA contraction (x86-64, no -march;
// SURVEY.md §0 trap 1) independent of nvcc's --fmad setting.
//
// Two exact re-formulations make the GPU version cheap and nearly divergence-free:
//  * sqrt is monotone under correct rounding, so min_k sqrt(x_k) == sqrt(min_k x_k)
//    bitwise: all 15 candidates are carried as squared distances and one sqrt is
//    taken at the end (the reference takes 33 per call).
//  * each branchy region test in point_triangle / segment_segment is evaluated as
//    pure predicates and the final closest point is selected, so a warp executes one
//    path instead of the union of seven. Every selected formula is the reference's.
// The triangle-order canonicalisation only affects the 9 segment-segment calls (the
// 6 point-triangle calls and the 6 piercing tests form order-free sets), so the
// canonical order is applied there only.
#pragma once
#include <cstdint>

namespace tjx {

#define TJ_ADD(a, b) __dadd_rn((a), (b))
#define TJ_SUB(a, b) __dsub_rn((a), (b))
#define TJ_MUL(a, b) __dmul_rn((a), (b))
#define TJ_DIV(a, b) __ddiv_rn((a), (b))
#define TJ_SQRT(a) __dsqrt_rn(a)

struct V3 {
    double x, y, z;
};

__device__ __forceinline__ V3 vsub(const V3& a, const V3& b) {
    return {TJ_SUB(a.x, b.x), TJ_SUB(a.y, b.y), TJ_SUB(a.z, b.z)};
}
__device__ __forceinline__ V3 vadd(const V3& a, const V3& b) {
    return {TJ_ADD(a.x, b.x), TJ_ADD(a.y, b.y), TJ_ADD(a.z, b.z)};
}
__device__ __forceinline__ V3 vmul(const V3& a, double s) {
    return {TJ_MUL(a.x, s), TJ_MUL(a.y, s), TJ_MUL(a.z, s)};
}
// dot(a,b) = (ax*bx + ay*by) + az*bz   (proj/include/trijoin/geom.hpp:24)
__device__ __forceinline__ double vdot(const V3& a, const V3& b) {
    return TJ_ADD(TJ_ADD(TJ_MUL(a.x, b.x), TJ_MUL(a.y, b.y)), TJ_MUL(a.z, b.z));
}
// proj/include/trijoin/geom.hpp:25-27
__device__ __forceinline__ V3 vcross(const V3& a, const V3& b) {
    return {TJ_SUB(TJ_MUL(a.y, b.z), TJ_MUL(a.z, b.y)), TJ_SUB(TJ_MUL(a.z, b.x), TJ_MUL(a.x, b.z)),
            TJ_SUB(TJ_MUL(a.x, b.y), TJ_MUL(a.y, b.x))};
}
__device__ __forceinline__ double vnorm2(const V3& a) { return vdot(a, a); }
__device__ __forceinline__ V3 vsel(bool c, const V3& a, const V3& b) {
    return {c ? a.x : b.x, c ? a.y : b.y, c ? a.z : b.z};
}

// std::min(best, x) == (x < best) ? x : best ; std::max(a, b) == (a < b) ? b : a
__device__ __forceinline__ double smin(double best, double x) { return (x < best) ? x : best; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
// std::clamp(v, 0.0, 1.0) (libstdc++: min(max(v, lo), hi))
__device__ __forceinline__ double sclamp01(double v) {
    const double m = (v < 0.0) ? 0.0 : v;
    return (1.0 < m) ? 1.0 : m;
}

// mindist_aabb (src/geom.cpp:11-16). std::max({0, p, q}) keeps the first largest.
__device__ __forceinline__ double mindist_box(const double* a, const double* b) {
    double g[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double m = 0.0;
        const double p = TJ_SUB(a[d], b[3 + d]);
        const double q = TJ_SUB(b[d], a[3 + d]);
        if (m < p) m = p;
        if (m < q) m = q;
        g[d] = m;
    }
    return TJ_SQRT(TJ_ADD(TJ_ADD(TJ_MUL(g[0], g[0]), TJ_MUL(g[1], g[1])), TJ_MUL(g[2], g[2])));
}

// distance(a, b) (proj/include/trijoin/geom.hpp:29-30)
__device__ __forceinline__ double point_dist(const double* a, const double* b) {
    const V3 d = {TJ_SUB(a[0], b[0]), TJ_SUB(a[1], b[1]), TJ_SUB(a[2], b[2])};
    return TJ_SQRT(vnorm2(d));
}

// ---------------------------------------------------------------------------------------
// Triangles in shared memory. A staged facet record is kFacetWords doubles:
//   [0..8] v0 v1 v2   [9] hd   [10] ph   [11] |v1-v0|   [12] |v2-v1|   [13] |v2-v0| (== |v0-v2|)
//   [14] 1.0 if triangle_degenerate (src/geom.cpp:29-35) else 0.0
// Records are addressed by 32-bit shared-window addresses; the geometry below loops over
// vertices/edges with runtime indices into these records, so each formula exists once in
// the binary (the fully unrolled form was 19k SASS instructions and starved the warps on
// instruction fetch). Hoisting the per-triangle quantities is bit-exact: each is the
// reference's own formula evaluated on the same inputs.
constexpr int kFacetWords = 15;

// Geometry entry points that read a staged record (lds below: asm loads the compiler does not
// see as memory reads) begin with this barrier: it gives the out-of-line call a side effect,
// so two calls on the same slot are never merged into one (e.g. by loop unrolling) although
// the record was re-staged between them.
__device__ __forceinline__ void staged_read_barrier() { asm volatile("" ::: "memory"); }

__device__ __forceinline__ double lds(uint32_t a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ V3 ldv(uint32_t t, int i) {
    const uint32_t a = t + 24u * (uint32_t)i;
    return {lds(a), lds(a + 8), lds(a + 16)};
}
__device__ __forceinline__ double ldw(uint32_t t, int w) { return lds(t + 8u * (uint32_t)w); }

// triangle_degenerate, also returning n2 and scale2 (used by the culling shape test).
__device__ __forceinline__ bool tri_degenerate(const V3& v0, const V3& v1, const V3& v2, double* n2_out,
                                               double* scale2_out) {
    const V3 ab = vsub(v1, v0), ac = vsub(v2, v0), bc = vsub(v2, v1);
    double s2 = vnorm2(ab); // std::max({norm2(ab), norm2(ac), norm2(bc)})
    const double n_ac = vnorm2(ac), n_bc = vnorm2(bc);
    if (s2 < n_ac) s2 = n_ac;
    if (s2 < n_bc) s2 = n_bc;
    const double n2 = vnorm2(vcross(ab, ac));
    if (n2_out) *n2_out = n2;
    if (scale2_out) *scale2_out = s2;
    return n2 <= TJ_MUL(TJ_MUL(1e-24, s2), s2);
}

// point_segment_distance squared (src/geom.cpp:18-24)
__device__ __forceinline__ double point_segment_d2(const V3& p, const V3& a, const V3& b) {
    const V3 d = vsub(b, a);
    const double dd = vnorm2(d);
    if (dd <= 0.0) return vnorm2(vsub(p, a));
    const double t = sclamp01(TJ_DIV(vdot(vsub(p, a), d), dd));
    return vnorm2(vsub(p, vadd(a, vmul(d, t))));
}

// point_triangle_distance squared (src/geom.cpp:39-80) of triangle (a, b, c) whose degenerate
// flag (triangle_degenerate, src/geom.cpp:29-35) is `degen`.
__device__ __forceinline__ double point_triangle_d2(const V3& p, const V3& a, const V3& b, const V3& c, bool degen) {
    if (degen) {
        // std::min({psd(v0,v1), psd(v1,v2), psd(v2,v0)}) keeps the first smallest
        double m = point_segment_d2(p, a, b);
        const double m1 = point_segment_d2(p, b, c);
        const double m2 = point_segment_d2(p, c, a);
        if (m1 < m) m = m1;
        if (m2 < m) m = m2;
        return m;
    }
    const V3 ab = vsub(b, a), ac = vsub(c, a), ap = vsub(p, a);
    const double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
    const V3 bp = vsub(p, b);
    const double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
    const double vc = TJ_SUB(TJ_MUL(d1, d4), TJ_MUL(d3, d2));
    const V3 cp = vsub(p, c);
    const double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
    const double vb = TJ_SUB(TJ_MUL(d5, d2), TJ_MUL(d1, d6));
    const double va = TJ_SUB(TJ_MUL(d3, d6), TJ_MUL(d5, d4));
    const double d43 = TJ_SUB(d4, d3), d56 = TJ_SUB(d5, d6);

    // Region predicates in the reference's order; the first true one wins.
    int reg = 6; // interior
    if (va <= 0.0 && d43 >= 0.0 && d56 >= 0.0) reg = 5;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) reg = 4;
    if (d6 >= 0.0 && d5 <= d6) reg = 3;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) reg = 2;
    if (d3 >= 0.0 && d4 <= d3) reg = 1;
    if (d1 <= 0.0 && d2 <= 0.0) reg = 0;

    // One division: the region's own quotient (interior: denom = 1/(va+vb+vc)); vertex
    // regions divide nothing (0/1 keeps the unused quotient off the slow path).
    double num = 0.0, den = 1.0;
    if (reg == 6) { num = 1.0; den = TJ_ADD(TJ_ADD(va, vb), vc); }
    if (reg == 2) { num = d1; den = TJ_SUB(d1, d3); }
    if (reg == 4) { num = d2; den = TJ_SUB(d2, d6); }
    if (reg == 5) { num = d43; den = TJ_ADD(d43, d56); }
    const double q = TJ_DIV(num, den);

    // Closest point X, each candidate with the reference's formula:
    // a+ab*v | a+ac*w | b+(c-b)*w | (a+ab*v)+ac*w.
    const V3 bc = vsub(c, b);
    const V3 base = (reg == 5) ? b : a;
    const V3 e1 = (reg == 4) ? ac : ((reg == 5) ? bc : ab);
    const double s1 = (reg == 6) ? TJ_MUL(vb, q) : q;
    V3 x = vadd(base, vmul(e1, s1));
    if (reg == 6) x = vadd(x, vmul(ac, TJ_MUL(vc, q)));
    if (reg == 0) x = a;
    if (reg == 1) x = b;
    if (reg == 3) x = c;
    return vnorm2(vsub(p, x));
}
// ... of a staged record t.
__device__ __forceinline__ double point_triangle_d2(const V3& p, uint32_t t) {
    return point_triangle_d2(p, ldv(t, 0), ldv(t, 1), ldv(t, 2), ldw(t, 14) != 0.0);
}

// segment_segment_distance squared (src/geom.cpp:82-113).
__device__ __forceinline__ double segment_segment_d2(const V3& p1, const V3& q1, const V3& p2, const V3& q2) {
    const V3 d1 = vsub(q1, p1), d2 = vsub(q2, p2), r = vsub(p1, p2);
    const double a = vnorm2(d1), e = vnorm2(d2), f = vdot(d2, r);
    double s = 0.0, t = 0.0;
    if (a <= 0.0 || e <= 0.0) { // point-degenerate segments (rare)
        if (a <= 0.0 && e <= 0.0) return vnorm2(vsub(p1, p2));
        if (a <= 0.0) {
            t = sclamp01(TJ_DIV(f, e));
        } else {
            const double c = vdot(d1, r);
            s = sclamp01(TJ_DIV(-c, a));
        }
    } else {
        const double c = vdot(d1, r);
        const double b = vdot(d1, d2);
        const double denom = TJ_SUB(TJ_MUL(a, e), TJ_MUL(b, b));
        // parallel segments (denom <= 0) use s = 0 and never read the quotient: divide by
        // 1 instead of 0 so the unused division stays on the fast path
        const double sq = sclamp01(TJ_DIV(TJ_SUB(TJ_MUL(b, f), TJ_MUL(c, e)), denom > 0.0 ? denom : 1.0));
        const double s0 = (denom > 0.0) ? sq : 0.0;
        const double t0 = TJ_DIV(TJ_ADD(TJ_MUL(b, s0), f), e);
        const bool tneg = t0 < 0.0;
        const bool tbig = !tneg && t0 > 1.0;
        const double s1 = sclamp01(TJ_DIV(tneg ? -c : TJ_SUB(b, c), a));
        s = (tneg || tbig) ? s1 : s0;
        t = tneg ? 0.0 : (tbig ? 1.0 : t0);
    }
    return vnorm2(vsub(vadd(p1, vmul(d1, s)), vadd(p2, vmul(d2, t))));
}

// segment_pierces_triangle (src/geom.cpp:120-136) with the three norms hoisted.
__device__ __forceinline__ bool segment_pierces(const V3& p, const V3& q, double ndir, uint32_t t) {
    const V3 v0 = ldv(t, 0), v1 = ldv(t, 1), v2 = ldv(t, 2);
    const V3 dir = vsub(q, p);
    const V3 e1 = vsub(v1, v0), e2 = vsub(v2, v0);
    const V3 pv = vcross(dir, e2);
    const double det = vdot(e1, pv);
    const double scale = TJ_MUL(TJ_MUL(ndir, ldw(t, 11)), ldw(t, 13));
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

// triangle_less (src/geom.cpp:140-148): lexicographic over the 9 coordinates.
__device__ __forceinline__ bool tri_less(uint32_t a, uint32_t b) {
#pragma unroll 1
    for (int i = 0; i < 9; ++i) {
        const double x = ldw(a, i), y = ldw(b, i);
        if (x < y) return true;
        if (x > y) return false;
    }
    return false;
}

// tri_tri_distance (src/geom.cpp:152-183) on two staged records.
__device__ __forceinline__ double tri_tri(uint32_t A, uint32_t B) {
    double best2 = __longlong_as_double(0x7ff0000000000000ll); // +inf
    // 6 vertex-triangle candidates: {A's vertices -> B} U {B's vertices -> A}, an order-free set.
#pragma unroll 1
    for (int k = 0; k < 6; ++k) {
        const uint32_t src = (k & 1) ? B : A, dst = (k & 1) ? A : B;
        best2 = smin(best2, point_triangle_d2(ldv(src, k >> 1), dst));
    }
    // 9 edge-edge candidates with t1 = the lexicographically smaller triangle.
    const bool swap = tri_less(B, A);
    const uint32_t t1 = swap ? B : A, t2 = swap ? A : B;
#pragma unroll 1
    for (int m = 0; m < 9; ++m) {
        const int i = m / 3, j = m - 3 * (m / 3);
        const int i1 = i == 2 ? 0 : i + 1, j1 = j == 2 ? 0 : j + 1;
        best2 = smin(best2, segment_segment_d2(ldv(t1, i), ldv(t1, i1), ldv(t2, j), ldv(t2, j1)));
    }
    const double best = TJ_SQRT(best2);
    if (best > 0.0) {
        // edges of A through B (if B is not degenerate) and of B through A: an order-free OR
#pragma unroll 1
        for (int k = 0; k < 6; ++k) {
            const uint32_t src = k < 3 ? A : B, tri = k < 3 ? B : A;
            const int e = k < 3 ? k : k - 3;
            if (ldw(tri, 14) != 0.0) continue;
            const int e1 = e == 2 ? 0 : e + 1;
            if (segment_pierces(ldv(src, e), ldv(src, e1), ldw(src, 11 + e), tri)) return 0.0;
        }
    }
    return best;
}

// Stage the 9 coordinates (+ hd, ph) into a record at shared address t. Returns the
// degenerate flag; n2/scale2 feed the culling shape test.
__device__ __forceinline__ void sts(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v)); }

__device__ __forceinline__ bool stage_exact(const double* c, double hd, double ph, uint32_t t, double* n2,
                                            double* s2) {
    const V3 v0 = {c[0], c[1], c[2]}, v1 = {c[3], c[4], c[5]}, v2 = {c[6], c[7], c[8]};
#pragma unroll
    for (int k = 0; k < 9; ++k) sts(t + 8u * k, c[k]);
    sts(t + 72, hd);
    sts(t + 80, ph);
    sts(t + 88, TJ_SQRT(vnorm2(vsub(v1, v0))));
    sts(t + 96, TJ_SQRT(vnorm2(vsub(v2, v1))));
    sts(t + 104, TJ_SQRT(vnorm2(vsub(v2, v0))));
    const bool degen = tri_degenerate(v0, v1, v2, n2, s2);
    sts(t + 112, degen ? 1.0 : 0.0);
    return degen;
}

} // namespace tjx
