// Multi-LOD facet refinement on sm_100a (reference refine_kernel, src/refine.cpp:63-84,
// paper Alg. 4): per voxel pair, the exact minima over all facet pairs (i, j) of
//     lb_ij = max(0, d_ij - ph_i - ph_j)      ub_ij = d_ij + hd_i + hd_j
// with d_ij the reference tri_tri_distance (geom_exact.cuh), bit-identical to the CPU.
//
// Work decomposition (one warp per voxel pair, dynamic work counter):
//   * the r-voxel's facets are staged 32 at a time into shared memory, one per lane
//     (each lane also keeps its facet's FP32 culling record in registers);
//   * the s-voxel's facets are staged 64 at a time into shared memory and read as
//     warp-wide broadcasts;
//   * every (i, j) first goes through a cheap FP32 test (exact-preserving cull,
//     below); survivors are pushed into a per-warp queue and evaluated exactly in
//     FP64 32 at a time, so the expensive path always runs with a converged warp;
//   * running minima are warp-reduced after each evaluation round.
//
// Exact-preserving culling: pair (i, j) is skipped
// only if it provably cannot lower either running minimum, i.e. with B_ij a rigorous
// lower bound of the exact triangle distance (facet-AABB gap, FP32 with directed
// rounding on outward-rounded boxes):
//     B - ph_i - ph_j >= min_lb + delta   and   B + hd_i + hd_j >= min_ub + delta.
// The reference's computed d_ij is the distance between two points on the triangles
// (clamped Ericson parameters) up to rounding, except for (a) the interior case of
// point_triangle on sliver triangles and (b) a spurious edge-piercing "0" on nearly
// parallel edge/plane configurations. Pairs where either is possible are never culled:
// both facets must be well shaped (all angles with sin >= 1e-2), every edge/plane
// combination must satisfy |cos| >= 1e-3, and B <= 1e3 * min(L_i, L_j). delta adds a
// 1e-5 relative and 1e-12 * |coords| absolute margin, orders of magnitude above the
// rounding error bounds in that regime. Skipping a pair that cannot change a minimum
// leaves both minima bit-identical to the exhaustive loop.
#pragma once
#include <cstdint>

#include "geom_exact.cuh"

namespace tjx {

constexpr int kRT = 32;      // r facets per tile (one per lane)
constexpr int kST = 32;      // s facets per tile
constexpr int kFS = 15;      // doubles per staged facet: v[9] hd ph lab lbc lac flags
constexpr int kCS = 24;      // floats per culling record
constexpr int kWarps = 4;    // warps per CTA
constexpr int kQueue = 64;

struct WarpSmem {
    double rf[kRT * kFS];
    double sf[kST * kFS];
    float rc[kRT * kCS];
    float sc[kST * kCS];
    uint32_t queue[kQueue];
};

// Culling record layout (floats):
//  0-2 lo (rd)  3-5 hi (ru)  6 L (ru, facet AABB diagonal)  7 M (ru, max |coord|)
//  8 hd (rd)    9 ph (ru)    10 ok (1 = well shaped and non-degenerate)
//  11-13 unit(v1-v0)  14-16 unit(v2-v1)  17-19 unit(v0-v2)  20-22 unit normal  23 pad
struct CullRec {
    float f[kCS];
};

struct RefineCounters {
    unsigned long long tested;    // FP32 culling tests
    unsigned long long evaluated; // exact FP64 tri_tri evaluations
};

__device__ __forceinline__ float rd(double x) { return __double2float_rd(x); }
__device__ __forceinline__ float ru(double x) { return __double2float_ru(x); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Stage one facet record (TJ_FACET_STRIDE doubles: v[9] hd ph pad) into shared memory:
// the exact record (geom_exact.cuh layout) at `sm` and the FP32 culling record at `cr`.
__device__ __forceinline__ void stage_facet(const double* __restrict__ g, double* sm, float* cr) {
    const double2* g2 = reinterpret_cast<const double2*>(g);
    double c[12];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const double2 t = __ldg(g2 + k);
        c[2 * k] = t.x;
        c[2 * k + 1] = t.y;
    }
    double n2, s2;
    const bool degen = stage_exact(c, c[9], c[10], smem_addr(sm), &n2, &s2);
    const bool shaped = n2 >= TJ_MUL(TJ_MUL(1e-4, s2), s2);
    const bool ok = !degen && shaped;

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
    cr[10] = ok ? 1.f : 0.f;
    // unit edge directions and unit normal (conditioning estimates only)
    const V3 v0 = {c[0], c[1], c[2]}, v1 = {c[3], c[4], c[5]}, v2 = {c[6], c[7], c[8]};
    const V3 es[4] = {vsub(v1, v0), vsub(v2, v1), vsub(v0, v2), vcross(vsub(v1, v0), vsub(v2, v0))};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double l2 = vnorm2(es[k]);
        const double inv = l2 > 0.0 ? rsqrt(l2) : 0.0;
        cr[11 + 3 * k] = (float)(es[k].x * inv);
        cr[12 + 3 * k] = (float)(es[k].y * inv);
        cr[13 + 3 * k] = (float)(es[k].z * inv);
    }
    cr[23] = 0.f;
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

__device__ __forceinline__ float absdot3(const float* u, const float* v) {
    return fabsf(u[0] * v[0] + u[1] * v[1] + u[2] * v[2]);
}

// True iff (a, b) provably cannot lower min_lb or min_ub (both given rounded up).
__device__ __forceinline__ bool cullable(const float* a, const float* b, float mlb_u, float mub_u) {
    const float B = box_gap_lb(a, b);
    const float delta =
        __fadd_ru(__fmul_ru(1e-5f, __fadd_ru(__fadd_ru(B, a[6]), b[6])), __fmul_ru(1e-12f, __fadd_ru(a[7], b[7])));
    const float lbs = __fsub_rd(__fsub_rd(B, a[9]), b[9]);
    const float ubs = __fadd_rd(__fadd_rd(B, a[8]), b[8]);
    // A running minimum of exactly 0 is the floor (lb_ij, ub_ij >= 0): that side needs no test.
    const bool lb_ok = mlb_u == 0.f || lbs >= __fadd_ru(mlb_u, delta);
    const bool ub_ok = mub_u == 0.f || ubs >= __fadd_ru(mub_u, delta);
    if (!(lb_ok && ub_ok)) return false;
    if (a[10] == 0.f || b[10] == 0.f) return false;
    if (B > 1e3f * fminf(a[6], b[6])) return false;
    const float kC = 1e-3f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (absdot3(a + 11 + 3 * k, b + 20) < kC) return false;
        if (absdot3(b + 11 + 3 * k, a + 20) < kC) return false;
    }
    return true;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = (w < v) ? w : v;
    }
    return v;
}

// Exact evaluation of one facet pair (staged records at shared addresses ra, sb):
// returns (max(0, d - ph_r - ph_s), d + hd_r + hd_s)  (src/refine.cpp:77-79). Not inlined:
// one copy of the geometry serves every call site (instruction-cache footprint).
__device__ __noinline__ double2 eval_pair(uint32_t ra, uint32_t sb) {
    const double d = tri_tri(ra, sb);
    const double lbp = smax(0.0, TJ_SUB(TJ_SUB(d, ldw(ra, 10)), ldw(sb, 10)));
    const double ubp = TJ_ADD(TJ_ADD(d, ldw(ra, 9)), ldw(sb, 9));
    return make_double2(lbp, ubp);
}

__device__ __forceinline__ void fold(double2 v, double& mlb, double& mub) {
    mlb = smin(mlb, v.x);
    mub = smin(mub, v.y);
}

// Op-level running minima shared by all warps refining voxel pairs of the same candidate
// (join mode). A pair that cannot lower the *op* minimum cannot change the aggregated
// object bounds (aggregate_object_bounds folds the minimum over the op's voxel pairs), so
// culling against min(vp-local, op-global) is exact for the join. Per-voxel-pair outputs
// (refine_kernel / tj_refine_batch) use op == nullptr: vp-local minima only.
struct OpMin {
    unsigned long long* lb_bits; // nullptr = no op-level sharing
    unsigned long long* ub_bits;
    uint32_t op;
};

__device__ __forceinline__ double load_min(const unsigned long long* p) {
    return __longlong_as_double((long long)__ldcg(reinterpret_cast<const unsigned long long*>(p)));
}

// One voxel pair: facets [r_base, r_base + r_len) x [s_base, s_base + s_len), each
// record TJ_FACET_STRIDE (12) doubles. Returns the exact vp-local minima (warp-uniform).
// Tile pairs (32 r x 32 s facets) are flattened so lane l tests pairs t = l, l + 32, ...
// of the tile (i = t / scnt, j = t % scnt): small voxels keep all lanes busy.
__device__ __forceinline__ void refine_voxel_pair(WarpSmem& sm, const double* __restrict__ r_base, uint32_t r_len,
                                                  const double* __restrict__ s_base, uint32_t s_len, bool cull,
                                                  const OpMin& om, double& out_lb, double& out_ub,
                                                  unsigned long long& tested, unsigned long long& evaluated) {
    const int lane = threadIdx.x & 31;
    const double kInf = __longlong_as_double(0x7ff0000000000000ll);
    double mlb = kInf, mub = kInf; // vp-local minima, warp-uniform after every reduction
    const uint32_t rbase = smem_addr(sm.rf), sbase = smem_addr(sm.sf);
    constexpr uint32_t kRec = kFS * 8;
    // culling thresholds: min(vp-local, op-global)
    double tlb = kInf, tub = kInf;
    auto refresh = [&]() {
        tlb = mlb;
        tub = mub;
        if (om.lb_bits) {
            // one lane reads, all lanes use the same value: every branch on tlb/tub must
            // stay warp-uniform (the warp-synchronous queue relies on it)
            double glb = 0.0, gub = 0.0;
            if (lane == 0) {
                glb = load_min(om.lb_bits + om.op);
                gub = load_min(om.ub_bits + om.op);
            }
            glb = __shfl_sync(0xffffffffu, glb, 0);
            gub = __shfl_sync(0xffffffffu, gub, 0);
            tlb = smin(tlb, glb);
            tub = smin(tub, gub);
        }
    };
    auto publish = [&]() {
        if (om.lb_bits && lane == 0 && mlb < kInf) {
            atomicMin(om.lb_bits + om.op, (unsigned long long)__double_as_longlong(mlb));
            atomicMin(om.ub_bits + om.op, (unsigned long long)__double_as_longlong(mub));
        }
    };
    refresh();
    if (cull && tlb == 0.0 && tub == 0.0) { // op already at the floor: nothing can lower it
        out_lb = mlb;
        out_ub = mub;
        return;
    }
    bool done = false;
    for (uint32_t r0 = 0; r0 < r_len && !done; r0 += kRT) {
        const int rcnt = (int)min((uint32_t)kRT, r_len - r0);
        __syncwarp();
        if (lane < rcnt) stage_facet(r_base + (size_t)(r0 + lane) * 12, sm.rf + lane * kFS, sm.rc + lane * kCS);
        for (uint32_t s0 = 0; s0 < s_len && !done; s0 += kST) {
            const int scnt = (int)min((uint32_t)kST, s_len - s0);
            __syncwarp();
            for (int l = lane; l < scnt; l += 32)
                stage_facet(s_base + (size_t)(s0 + l) * 12, sm.sf + l * kFS, sm.sc + l * kCS);
            __syncwarp();
            const int npairs = rcnt * scnt;

            double llb = mlb, lub = mub; // lane-local minima
            int seed_t = -1;
            if (cull && tlb == kInf) {
                // Seed: each lane evaluates its pair of smallest box gap.
                float bestB = __int_as_float(0x7f800000);
                for (int t = lane; t < npairs; t += 32) {
                    const int i = t / scnt, j = t - i * scnt;
                    const float B = box_gap_lb(sm.rc + i * kCS, sm.sc + j * kCS);
                    if (B < bestB) { bestB = B; seed_t = t; }
                }
                if (seed_t >= 0) {
                    const int i = seed_t / scnt, j = seed_t - i * scnt;
                    fold(eval_pair(rbase + i * kRec, sbase + j * kRec), llb, lub);
                    ++evaluated;
                }
                mlb = warp_min(llb);
                mub = warp_min(lub);
                publish();
                refresh();
            }
            int qn = 0;
            float tlb_u = ru(tlb), tub_u = ru(tub);
            for (int t0 = 0; t0 < npairs; t0 += 32) {
                const int t = t0 + lane;
                bool need = false;
                if (t < npairs && t != seed_t) {
                    const int i = t / scnt, j = t - i * scnt;
                    need = !cull || !cullable(sm.rc + i * kCS, sm.sc + j * kCS, tlb_u, tub_u);
                    ++tested;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, need);
                if (need) sm.queue[qn + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)t;
                qn += __popc(bal);
                if (qn >= 32) {
                    __syncwarp();
                    const int e = (int)sm.queue[lane];
                    const int i = e / scnt, j = e - i * scnt;
                    fold(eval_pair(rbase + i * kRec, sbase + j * kRec), llb, lub);
                    ++evaluated;
                    __syncwarp();
                    if (lane < qn - 32) sm.queue[lane] = sm.queue[32 + lane];
                    __syncwarp();
                    qn -= 32;
                    mlb = warp_min(llb);
                    mub = warp_min(lub);
                    publish();
                    refresh();
                    tlb_u = ru(tlb);
                    tub_u = ru(tub);
                    if (cull && tlb == 0.0 && tub == 0.0) { done = true; break; }
                }
            }
            if (!done && qn > 0) {
                __syncwarp();
                if (lane < qn) {
                    const int e = (int)sm.queue[lane];
                    const int i = e / scnt, j = e - i * scnt;
                    fold(eval_pair(rbase + i * kRec, sbase + j * kRec), llb, lub);
                    ++evaluated;
                }
                mlb = warp_min(llb);
                mub = warp_min(lub);
                publish();
                refresh();
                if (cull && tlb == 0.0 && tub == 0.0) done = true;
            }
        }
    }
    out_lb = mlb;
    out_ub = mub;
}

} // namespace tjx
