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

// A triangle as it sits in shared memory during refinement: vertices plus the
// per-triangle quantities the reference recomputes inside every call. Each
// derived value uses the reference's exact formula, so hoisting is bit-exact.
struct TriRef {
    V3 v0, v1, v2;
    double lab, lbc, lac; // norm(v1-v0), norm(v2-v1), norm(v2-v0) == norm(v0-v2)
    bool degenerate;      // triangle_degenerate (src/geom.cpp:29-35)
};

// triangle_degenerate, returning also the shape flag used by the culling logic.
__device__ __forceinline__ bool tri_degenerate(const V3& v0, const V3& v1, const V3& v2,
                                               double* n2_out, double* scale2_out) {
    const V3 ab = vsub(v1, v0), ac = vsub(v2, v0), bc = vsub(v2, v1);
    double s2 = vnorm2(ab);  // std::max({norm2(ab), norm2(ac), norm2(bc)})
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

// point_triangle_distance squared (src/geom.cpp:39-80).
__device__ __forceinline__ double point_triangle_d2(const V3& p, const TriRef& t) {
    if (t.degenerate) {
        // std::min({psd(v0,v1), psd(v1,v2), psd(v2,v0)}) keeps the first smallest
        double m = point_segment_d2(p, t.v0, t.v1);
        const double m1 = point_segment_d2(p, t.v1, t.v2);
        const double m2 = point_segment_d2(p, t.v2, t.v0);
        if (m1 < m) m = m1;
        if (m2 < m) m = m2;
        return m;
    }
    const V3& a = t.v0;
    const V3& b = t.v1;
    const V3& c = t.v2;
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
    const bool r0 = d1 <= 0.0 && d2 <= 0.0;
    const bool r1 = d3 >= 0.0 && d4 <= d3;
    const bool r2 = vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0;
    const bool r3 = d6 >= 0.0 && d5 <= d6;
    const bool r4 = vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0;
    const bool r5 = va <= 0.0 && d43 >= 0.0 && d56 >= 0.0;
    // region id 0..6 (6 = interior)
    int reg = 6;
    if (r5) reg = 5;
    if (r4) reg = 4;
    if (r3) reg = 3;
    if (r2) reg = 2;
    if (r1) reg = 1;
    if (r0) reg = 0;

    // One division: the region's own quotient.
    double num = 1.0, den = TJ_ADD(TJ_ADD(va, vb), vc); // interior: denom = 1/(va+vb+vc)
    if (reg == 2) { num = d1; den = TJ_SUB(d1, d3); }
    if (reg == 4) { num = d2; den = TJ_SUB(d2, d6); }
    if (reg == 5) { num = d43; den = TJ_ADD(d43, d56); }
    const double q = TJ_DIV(num, den);

    // Closest point X, each candidate with the reference's formula.
    const V3 bc = vsub(c, b);
    const V3 base = (reg == 5) ? b : a;
    const V3 e1 = (reg == 4) ? ac : ((reg == 5) ? bc : ab);
    const double s1 = (reg == 6) ? TJ_MUL(vb, q) : q;
    V3 x = vadd(base, vmul(e1, s1)); // a+ab*v | a+ac*w | b+(c-b)*w | a+ab*v (interior, 1st term)
    if (reg == 6) x = vadd(x, vmul(ac, TJ_MUL(vc, q)));
    if (reg == 0) x = a;
    if (reg == 1) x = b;
    if (reg == 3) x = c;
    return vnorm2(vsub(p, x));
}

// segment_segment_distance squared (src/geom.cpp:82-113).
__device__ __forceinline__ double segment_segment_d2(const V3& p1, const V3& q1, const V3& p2,
                                                     const V3& q2) {
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
        const double sq = sclamp01(TJ_DIV(TJ_SUB(TJ_MUL(b, f), TJ_MUL(c, e)), denom));
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
__device__ __forceinline__ bool segment_pierces(const V3& p, const V3& q, double ndir,
                                                const TriRef& t) {
    const V3 dir = vsub(q, p);
    const V3 e1 = vsub(t.v1, t.v0), e2 = vsub(t.v2, t.v0);
    const V3 pv = vcross(dir, e2);
    const double det = vdot(e1, pv);
    const double scale = TJ_MUL(TJ_MUL(ndir, t.lab), t.lac);
    const bool ok_det = !(fabs(det) <= TJ_MUL(1e-14, scale));
    const double inv = TJ_DIV(1.0, det);
    const V3 tv = vsub(p, t.v0);
    const double u = TJ_MUL(vdot(tv, pv), inv);
    const V3 qv = vcross(tv, e1);
    const double v = TJ_MUL(vdot(dir, qv), inv);
    const double tt = TJ_MUL(vdot(e2, qv), inv);
    return ok_det && !(u < 0.0 || u > 1.0) && !(v < 0.0 || TJ_ADD(u, v) > 1.0) && tt >= 0.0 &&
           tt <= 1.0;
}

// triangle_less (src/geom.cpp:140-148): lexicographic over the 9 coordinates.
__device__ __forceinline__ bool tri_less(const TriRef& a, const TriRef& b) {
    const double pa[9] = {a.v0.x, a.v0.y, a.v0.z, a.v1.x, a.v1.y, a.v1.z, a.v2.x, a.v2.y, a.v2.z};
    const double pb[9] = {b.v0.x, b.v0.y, b.v0.z, b.v1.x, b.v1.y, b.v1.z, b.v2.x, b.v2.y, b.v2.z};
    int res = 0; // 0 undecided, 1 less, 2 greater
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        if (res == 0 && pa[i] < pb[i]) res = 1;
        if (res == 0 && pa[i] > pb[i]) res = 2;
    }
    return res == 1;
}

// tri_tri_distance (src/geom.cpp:152-183).
__device__ __forceinline__ double tri_tri(const TriRef& A, const TriRef& B) {
    double best2 = __longlong_as_double(0x7ff0000000000000ll); // +inf
    // 6 vertex-triangle candidates: an order-free set under canonicalisation.
    best2 = smin(best2, point_triangle_d2(A.v0, B));
    best2 = smin(best2, point_triangle_d2(B.v0, A));
    best2 = smin(best2, point_triangle_d2(A.v1, B));
    best2 = smin(best2, point_triangle_d2(B.v1, A));
    best2 = smin(best2, point_triangle_d2(A.v2, B));
    best2 = smin(best2, point_triangle_d2(B.v2, A));
    // 9 edge-edge candidates with t1 = the lexicographically smaller triangle.
    const bool swap = tri_less(B, A);
    const TriRef& t1 = swap ? B : A;
    const TriRef& t2 = swap ? A : B;
    const V3 a[3] = {t1.v0, t1.v1, t1.v2};
    const V3 b[3] = {t2.v0, t2.v1, t2.v2};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            best2 = smin(best2, segment_segment_d2(a[i], a[(i + 1) % 3], b[j], b[(j + 1) % 3]));
        }
    }
    const double best = TJ_SQRT(best2);
    if (best > 0.0) {
        // edges of A through B (if B is not degenerate), edges of B through A: order-free OR
        bool hit = false;
        if (!B.degenerate) {
            hit = hit || segment_pierces(A.v0, A.v1, A.lab, B);
            hit = hit || segment_pierces(A.v1, A.v2, A.lbc, B);
            hit = hit || segment_pierces(A.v2, A.v0, A.lac, B);
        }
        if (!A.degenerate) {
            hit = hit || segment_pierces(B.v0, B.v1, B.lab, A);
            hit = hit || segment_pierces(B.v1, B.v2, B.lbc, A);
            hit = hit || segment_pierces(B.v2, B.v0, B.lac, A);
        }
        if (hit) return 0.0;
    }
    return best;
}

// Build the hoisted per-triangle data from the 9 coordinates.
__device__ __forceinline__ TriRef make_tri(const double* c, double* n2_out = nullptr,
                                           double* scale2_out = nullptr) {
    TriRef t;
    t.v0 = {c[0], c[1], c[2]};
    t.v1 = {c[3], c[4], c[5]};
    t.v2 = {c[6], c[7], c[8]};
    t.lab = TJ_SQRT(vnorm2(vsub(t.v1, t.v0)));
    t.lbc = TJ_SQRT(vnorm2(vsub(t.v2, t.v1)));
    t.lac = TJ_SQRT(vnorm2(vsub(t.v2, t.v0)));
    t.degenerate = tri_degenerate(t.v0, t.v1, t.v2, n2_out, scale2_out);
    return t;
}

} // namespace tjx
