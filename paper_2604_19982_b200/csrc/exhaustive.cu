// Exhaustive exact join on the device: the drop-in for the reference's run_oracle
// (proj/include/trijoin/engine.hpp:77-80, proj/src/oracle.cpp:87-186). Like the reference it
// works on the level-100 (original-resolution) triangles only and shares nothing with the
// engine's bound machinery (object / voxel boxes, LOD paddings, culling thresholds) except
// the exact FP64 geometric primitives (geom_exact.cuh):
//
//   k_facet_boxes / k_object_boxes  facet boxes and per-object facet-bounds boxes (the
//                                   OracleTree root box, oracle.cpp:40-44: exact min / max)
//   k_box_pairs                     brute force over all |R| x |S| object pairs: thread per r,
//                                   S boxes streamed through shared memory; keeps (r, s) iff
//                                   mindist_aabb <= tau (oracle.cpp:147), in (r, s) order
//   k_pair_distance                 CTA per object pair: d = min over all facet pairs of
//                                   tri_tri_distance (oracle_pair_distance, oracle.cpp:95-124).
//                                   Seeded by every thread's closest facet-box pair, then every
//                                   facet pair whose box gap is below the running minimum is
//                                   evaluated; stops at d = 0. The minimum is exact whatever
//                                   the visiting order, like the reference's best-first search.
//   k-NN (oracle.cpp:152-166)       pass 1: per r the k S objects of smallest box gap; their
//                                   exact distances bound the k-th distance by U(r). Pass 2:
//                                   every s with box gap <= U(r), exact distances, a stable
//                                   segmented sort by (d, s) per r, the first k.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <vector>

#include "filter.cuh"
#include "geom_exact.cuh"
#include "scan.cuh"

struct tj_ctx_view {
    int device;
    cudaStream_t stream;
    tjx::Workspace* ws;
};

namespace tjx {
tj_ctx_view ctx_view(tj_ctx* ctx);
int guarded_call(tj_ctx* ctx, void (*fn)(void*), void* arg);
} // namespace tjx

using namespace tjx;

namespace {

constexpr int kBoxThreads = 256;
constexpr int kPairThreads = 128;
constexpr uint32_t kNoObject = 0xffffffffu;
constexpr int kMaxSeedK = 32; // k-NN pass 1 keeps up to this many nearest boxes per r (else U = inf)

__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7ff0000000000000ll); }

// Aabb::expand over v0 v1 v2 (proj/include/trijoin/geom.hpp): exact per-axis min / max.
__global__ void k_facet_boxes(const double* __restrict__ tris, uint64_t n, double* __restrict__ box) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double* t = tris + 9 * i;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double lo = t[d], hi = t[d];
            lo = (t[3 + d] < lo) ? t[3 + d] : lo;
            hi = (hi < t[3 + d]) ? t[3 + d] : hi;
            lo = (t[6 + d] < lo) ? t[6 + d] : lo;
            hi = (hi < t[6 + d]) ? t[6 + d] : hi;
            box[6 * i + d] = lo;
            box[6 * i + 3 + d] = hi;
        }
    }
}

// Warp per object: union of its facet boxes (Aabb::empty() for an object without facets).
__global__ void k_object_boxes(const uint64_t* __restrict__ off, const double* __restrict__ fbox, uint32_t n,
                               double* __restrict__ obox) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t o = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; o < n;
         o += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        double b[6];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            b[d] = inf_d();
            b[3 + d] = -inf_d();
        }
        for (uint64_t f = off[o] + lane; f < off[o + 1]; f += 32) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                b[d] = fmin(b[d], fbox[6 * f + d]);
                b[3 + d] = fmax(b[3 + d], fbox[6 * f + 3 + d]);
            }
        }
#pragma unroll
        for (int s = 16; s > 0; s >>= 1)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                b[d] = fmin(b[d], __shfl_xor_sync(0xffffffffu, b[d], s));
                b[3 + d] = fmax(b[3 + d], __shfl_xor_sync(0xffffffffu, b[3 + d], s));
            }
        if (lane < 6) obox[6 * o + lane] = b[lane];
    }
}

// mindist_aabb(a, b) <= t, exactly as the reference decides it. A per-axis gap g > t already
// implies mindist > t (sqrt(RN(g^2)) == g for normal g^2, and adding non-negative squares
// cannot decrease the rounded sum), which skips the sqrt for almost every pair.
__device__ __forceinline__ bool box_within(const double* a, const double* b, double t) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double p = TJ_SUB(a[d], b[3 + d]), q = TJ_SUB(b[d], a[3 + d]);
        const double g = p < q ? q : p;
        if (g > t && g > 1e-140) return false;
    }
    return mindist_box(a, b) <= t;
}

// Thread per r; S boxes through shared memory in tiles. kFill = false: counts[r] = number of
// s with mindist <= tau_r; kFill = true: their ids in ascending s at out_s[offsets[r] ...].
template <bool kFill>
__global__ void __launch_bounds__(kBoxThreads) k_box_pairs(const double* __restrict__ rbox, uint32_t nr,
                                                           const double* __restrict__ sbox, uint32_t ns, double tau,
                                                           const double* __restrict__ tau_r, uint64_t* counts,
                                                           const uint64_t* __restrict__ offsets, uint32_t* out_s) {
    __shared__ double tile[kBoxThreads * 6];
    const uint32_t r = blockIdx.x * kBoxThreads + threadIdx.x;
    double rb[6];
    double t = 0.0;
    uint64_t pos = 0, c = 0;
    if (r < nr) {
#pragma unroll
        for (int d = 0; d < 6; ++d) rb[d] = rbox[6 * (uint64_t)r + d];
        t = tau_r ? tau_r[r] : tau;
        if (kFill) pos = offsets[r];
    }
    for (uint32_t s0 = 0; s0 < ns; s0 += kBoxThreads) {
        const uint32_t m = min((uint32_t)kBoxThreads, ns - s0);
        __syncthreads();
        for (uint32_t x = threadIdx.x; x < 6 * m; x += kBoxThreads) tile[x] = sbox[6 * (uint64_t)s0 + x];
        __syncthreads();
        if (r < nr) {
            for (uint32_t j = 0; j < m; ++j) {
                if (!box_within(rb, tile + 6 * j, t)) continue;
                if (kFill)
                    out_s[pos++] = s0 + j;
                else
                    ++c;
            }
        }
    }
    if (!kFill && r < nr) counts[r] = c;
}

// k-NN pass 1: per r the (up to) k S objects of smallest box gap, ties to the smaller s.
__global__ void __launch_bounds__(kBoxThreads) k_knn_seed(const double* __restrict__ rbox, uint32_t nr,
                                                          const double* __restrict__ sbox, uint32_t ns, uint32_t k,
                                                          uint32_t* __restrict__ seed_s) {
    __shared__ double tile[kBoxThreads * 6];
    const uint32_t r = blockIdx.x * kBoxThreads + threadIdx.x;
    double rb[6];
    double gap[kMaxSeedK];
    uint32_t id[kMaxSeedK];
    uint32_t n = 0;
    if (r < nr) {
#pragma unroll
        for (int d = 0; d < 6; ++d) rb[d] = rbox[6 * (uint64_t)r + d];
    }
    for (uint32_t s0 = 0; s0 < ns; s0 += kBoxThreads) {
        const uint32_t m = min((uint32_t)kBoxThreads, ns - s0);
        __syncthreads();
        for (uint32_t x = threadIdx.x; x < 6 * m; x += kBoxThreads) tile[x] = sbox[6 * (uint64_t)s0 + x];
        __syncthreads();
        if (r >= nr) continue;
        for (uint32_t j = 0; j < m; ++j) {
            if (n == k && !box_within(rb, tile + 6 * j, gap[k - 1])) continue;
            const double g = mindist_box(rb, tile + 6 * j);
            if (n == k && !(g < gap[k - 1])) continue;
            uint32_t p = n < k ? n++ : k - 1; // insertion (later s never precede equal gaps)
            while (p > 0 && g < gap[p - 1]) {
                gap[p] = gap[p - 1];
                id[p] = id[p - 1];
                --p;
            }
            gap[p] = g;
            id[p] = s0 + j;
        }
    }
    if (r < nr)
        for (uint32_t i = 0; i < k; ++i) seed_s[(uint64_t)r * k + i] = i < n ? id[i] : kNoObject;
}

__device__ __noinline__ double tri_tri_exh(uint32_t a, uint32_t b) {
    staged_read_barrier();
    return tri_tri(a, b); }

__device__ __forceinline__ double gap2(const double* a, const double* b) {
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double p = TJ_SUB(a[d], b[3 + d]), q = TJ_SUB(b[d], a[3 + d]);
        double g = p < q ? q : p;
        g = g < 0.0 ? 0.0 : g;
        s = TJ_ADD(s, TJ_MUL(g, g));
    }
    return s;
}

// CTA per object pair (work counter): exact min over all facet pairs of tri_tri_distance.
__global__ void __launch_bounds__(kPairThreads) k_pair_distance(
    const uint32_t* __restrict__ pr, const uint32_t* __restrict__ ps, uint64_t n, const uint64_t* __restrict__ roff,
    const double* __restrict__ rtris, const double* __restrict__ rfbox, const uint64_t* __restrict__ soff,
    const double* __restrict__ stris, const double* __restrict__ sfbox, double* __restrict__ out,
    unsigned long long* work, unsigned long long* evaluated) {
    __shared__ double rec[kPairThreads][2][kFacetWords];
    __shared__ unsigned long long best_bits;
    __shared__ unsigned long long item;
    const uint32_t ta = static_cast<uint32_t>(__cvta_generic_to_shared(&rec[threadIdx.x][0][0]));
    const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(&rec[threadIdx.x][1][0]));
    unsigned long long evals = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            item = atomicAdd(work, 1ull);
            best_bits = 0x7ff0000000000000ull;
        }
        __syncthreads();
        const uint64_t it = item;
        if (it >= n) break;
        const uint32_t r = pr[it], s = ps[it];
        uint64_t na = 0, nb = 0, r0 = 0, s0 = 0;
        if (s != kNoObject) {
            r0 = roff[r];
            na = roff[r + 1] - r0;
            s0 = soff[s];
            nb = soff[s + 1] - s0;
        }
        const uint64_t np = na * nb;
        // phase A: this thread's facet pair of smallest box gap (a seed upper bound)
        uint64_t i = 0, j = threadIdx.x;
        while (j >= nb && i < na) {
            j -= nb;
            ++i;
        }
        double g_best = inf_d();
        uint64_t bi = 0, bj = 0;
        bool have = false;
        {
            uint64_t ii = i, jj = j;
            for (uint64_t t = threadIdx.x; t < np; t += kPairThreads) {
                const double g = gap2(rfbox + 6 * (r0 + ii), sfbox + 6 * (s0 + jj));
                if (!have || g < g_best) {
                    g_best = g;
                    bi = ii;
                    bj = jj;
                    have = true;
                }
                jj += kPairThreads;
                while (jj >= nb) {
                    jj -= nb;
                    ++ii;
                }
            }
        }
        double n2, sc2;
        if (have) {
            stage_exact(rtris + 9 * (r0 + bi), 0.0, 0.0, ta, &n2, &sc2);
            stage_exact(stris + 9 * (s0 + bj), 0.0, 0.0, tb, &n2, &sc2);
            const double d = tri_tri_exh(ta, tb);
            ++evals;
            atomicMin(&best_bits, (unsigned long long)__double_as_longlong(d));
        }
        __syncthreads();
        // phase B: every facet pair whose box gap is below the running minimum
        {
            uint64_t ii = i, jj = j;
            for (uint64_t t = threadIdx.x; t < np; t += kPairThreads) {
                const double best = __longlong_as_double((long long)*(volatile unsigned long long*)&best_bits);
                if (best == 0.0) break;
                if (!(ii == bi && jj == bj)) {
                    // skip only when the squared box gap clearly exceeds best^2 (conservative:
                    // more pairs are evaluated than a box-gap >= best test would keep)
                    const double g = gap2(rfbox + 6 * (r0 + ii), sfbox + 6 * (s0 + jj));
                    if (!(g > best * best * (1.0 + 1e-9))) {
                        stage_exact(rtris + 9 * (r0 + ii), 0.0, 0.0, ta, &n2, &sc2);
                        stage_exact(stris + 9 * (s0 + jj), 0.0, 0.0, tb, &n2, &sc2);
                        const double d = tri_tri_exh(ta, tb);
                        ++evals;
                        if (d < best) atomicMin(&best_bits, (unsigned long long)__double_as_longlong(d));
                    }
                }
                jj += kPairThreads;
                while (jj >= nb) {
                    jj -= nb;
                    ++ii;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) out[it] = s == kNoObject ? -1.0 : __longlong_as_double((long long)best_bits);
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
    if ((threadIdx.x & 31) == 0 && evals) atomicAdd(evaluated, evals);
}

// k-NN: U(r) = the largest exact distance among r's k seeds (+inf with fewer than k seeds).
__global__ void k_knn_bound(const double* __restrict__ d, const uint32_t* __restrict__ seed_s, uint32_t nr,
                            uint32_t k, double* __restrict__ u) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nr; r += (uint64_t)gridDim.x * blockDim.x) {
        double m = 0.0;
        for (uint32_t i = 0; i < k; ++i) {
            if (seed_s[r * k + i] == kNoObject) {
                m = inf_d();
                break;
            }
            const double x = d[r * k + i];
            m = x > m ? x : m;
        }
        u[r] = m;
    }
}

__global__ void k_expand_r(const uint64_t* __restrict__ offsets, uint32_t nr, uint32_t* __restrict__ pr) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nr; r += (uint64_t)gridDim.x * blockDim.x)
        for (uint64_t x = offsets[r]; x < offsets[r + 1]; ++x) pr[x] = (uint32_t)r;
}

__global__ void k_seed_pairs(uint32_t nr, uint32_t k, uint32_t* __restrict__ pr) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < (uint64_t)nr * k;
         x += (uint64_t)gridDim.x * blockDim.x)
        pr[x] = (uint32_t)(x / k);
}

__global__ void k_to_bits(const double* __restrict__ d, uint64_t n, unsigned long long* __restrict__ bits) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x)
        bits[x] = (unsigned long long)__double_as_longlong(d[x]); // d >= 0: IEEE bits order as unsigned
}

struct ReadU64 {
    const uint64_t* p;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return p[i]; }
};

struct MeshSetDev {
    uint32_t n = 0;
    uint64_t n_tris = 0;
    DevBuf<uint64_t> off;
    DevBuf<double> tris, fbox, obox;
};

inline int grid_for(uint64_t n, int threads, int num_sms, int per_sm = 16) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + threads - 1) / threads, (uint64_t)num_sms * per_sm));
}

void upload_meshes(MeshSetDev& m, const tj_mesh_set_view* v, int num_sms, cudaStream_t st) {
    if (!v || !v->tri_offsets) throw Error(TJ_EINVAL, "tj_exhaustive_join: null mesh set");
    m.n = v->n_objects;
    m.n_tris = v->tri_offsets[m.n];
    if (m.n_tris && !v->tris) throw Error(TJ_EINVAL, "tj_exhaustive_join: null triangles");
    for (uint32_t o = 0; o < m.n; ++o)
        if (v->tri_offsets[o + 1] < v->tri_offsets[o])
            throw Error(TJ_EINVAL, "tj_exhaustive_join: tri_offsets not ascending");
    m.off.alloc(m.n + 1);
    TJ_CUDA(cudaMemcpyAsync(m.off.p, v->tri_offsets, (m.n + 1) * 8, cudaMemcpyHostToDevice, st));
    m.tris.alloc(std::max<uint64_t>(9 * m.n_tris, 1));
    m.fbox.alloc(std::max<uint64_t>(6 * m.n_tris, 1));
    m.obox.alloc(std::max<uint64_t>(6 * (uint64_t)m.n, 1));
    if (m.n_tris) {
        TJ_CUDA(cudaMemcpyAsync(m.tris.p, v->tris, 9 * m.n_tris * 8, cudaMemcpyHostToDevice, st));
        count_launch();
        k_facet_boxes<<<grid_for(m.n_tris, 256, num_sms), 256, 0, st>>>(m.tris.p, m.n_tris, m.fbox.p);
        TJ_CUDA(cudaGetLastError());
    }
    if (m.n) {
        count_launch();
        k_object_boxes<<<grid_for(32ull * m.n, 256, num_sms), 256, 0, st>>>(m.off.p, m.fbox.p, m.n, m.obox.p);
        TJ_CUDA(cudaGetLastError());
    }
}

// Exact distances of pairs (pr[x], ps[x]) into d[x] (-1 for ps[x] == kNoObject).
void pair_distances(const MeshSetDev& R, const MeshSetDev& S, const uint32_t* pr, const uint32_t* ps, uint64_t n,
                    double* d, unsigned long long* counters, int num_sms, cudaStream_t st) {
    if (!n) return;
    TJ_CUDA(cudaMemsetAsync(counters, 0, 8, st));
    count_launch();
    k_pair_distance<<<(int)std::min<uint64_t>(n, (uint64_t)num_sms * 8), kPairThreads, 0, st>>>(
        pr, ps, n, R.off.p, R.tris.p, R.fbox.p, S.off.p, S.tris.p, S.fbox.p, d, counters, counters + 1);
    TJ_CUDA(cudaGetLastError());
}

// Candidate pairs {(r, s) : mindist(box_r, box_s) <= tau_r (or tau)} in (r, s) order.
uint64_t box_pairs(const MeshSetDev& R, const MeshSetDev& S, double tau, const double* tau_r, DevBuf<uint64_t>& offsets,
                   DevBuf<uint32_t>& pr, DevBuf<uint32_t>& ps, Workspace& ws, cudaStream_t st) {
    const uint32_t nr = R.n;
    DevBuf<uint64_t> counts(std::max<uint32_t>(nr, 1));
    offsets.alloc(nr + 1);
    TJ_CUDA(cudaMemsetAsync(offsets.p, 0, 8, st));
    if (!nr) return 0;
    const int grid = (int)((nr + kBoxThreads - 1) / kBoxThreads);
    count_launch();
    k_box_pairs<false><<<grid, kBoxThreads, 0, st>>>(R.obox.p, nr, S.obox.p, S.n, tau, tau_r, counts.p, nullptr,
                                                     nullptr);
    TJ_CUDA(cudaGetLastError());
    const uint64_t total = device_scan(ReadU64{counts.p}, nr, offsets.p, ws.u64a, ws.num_sms, st);
    pr.alloc(std::max<uint64_t>(total, 1));
    ps.alloc(std::max<uint64_t>(total, 1));
    if (!total) return 0;
    count_launch();
    k_box_pairs<true><<<grid, kBoxThreads, 0, st>>>(R.obox.p, nr, S.obox.p, S.n, tau, tau_r, nullptr, offsets.p,
                                                    ps.p);
    TJ_CUDA(cudaGetLastError());
    count_launch();
    k_expand_r<<<grid_for(nr, 256, ws.num_sms), 256, 0, st>>>(offsets.p, nr, pr.p);
    TJ_CUDA(cudaGetLastError());
    return total;
}

template <class T>
T* host_copy(const DevBuf<T>& src, uint64_t n, cudaStream_t st) {
    T* p = static_cast<T*>(std::malloc(std::max<uint64_t>(n, 1) * sizeof(T)));
    if (!p) throw std::bad_alloc();
    if (n) TJ_CUDA(cudaMemcpyAsync(p, src.p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    return p;
}

template <class F>
int run(tj_ctx* ctx, F&& f) {
    struct Box {
        F* f;
        static void call(void* p) { (*static_cast<Box*>(p)->f)(); }
    } box{&f};
    return guarded_call(ctx, &Box::call, &box);
}

} // namespace

extern "C" int tj_exhaustive_join(tj_ctx* ctx, const tj_mesh_set_view* Rv, const tj_mesh_set_view* Sv, int32_t type,
                                  double tau, uint32_t k, tj_exhaustive_result* out) {
    if (!ctx || !out) return TJ_EINVAL;
    std::memset(out, 0, sizeof(*out));
    return run(ctx, [&] {
        const auto t0 = std::chrono::steady_clock::now();
        if (type == TJ_KNN) {
            if (k == 0) throw Error(TJ_EINVAL, "join: k must be >= 1");
        } else if (type == TJ_WITHIN || type == TJ_INTERSECT) {
            if (!(tau >= 0)) throw Error(TJ_EINVAL, "join: tau must be >= 0");
            if (type == TJ_INTERSECT) tau = 0.0;
        } else {
            throw Error(TJ_EINVAL, "join: unknown join type");
        }
        const tj_ctx_view cv = ctx_view(ctx);
        cudaStream_t st = cv.stream;
        Workspace& ws = *cv.ws;
        MeshSetDev R, Sstore;
        upload_meshes(R, Rv, ws.num_sms, st);
        const MeshSetDev* S = &R;
        if (Sv && Sv != Rv) {
            upload_meshes(Sstore, Sv, ws.num_sms, st);
            S = &Sstore;
        }
        DevBuf<unsigned long long> counters(2);
        unsigned long long evaluated = 0, ev_h[2];
        DevBuf<uint64_t> offsets;
        DevBuf<uint32_t> pr, ps;
        uint64_t n_pairs = 0;
        DevBuf<double> d;
        if (type != TJ_KNN) {
            n_pairs = box_pairs(R, *S, tau, nullptr, offsets, pr, ps, ws, st);
            d.alloc(std::max<uint64_t>(n_pairs, 1));
            pair_distances(R, *S, pr.p, ps.p, n_pairs, d.p, counters.p, ws.num_sms, st);
            uint32_t* hr = host_copy(pr, n_pairs, st);
            uint32_t* hs = host_copy(ps, n_pairs, st);
            double* hd = host_copy(d, n_pairs, st);
            if (n_pairs) {
                TJ_CUDA(cudaMemcpyAsync(ev_h, counters.p, 16, cudaMemcpyDeviceToHost, st));
            } else {
                ev_h[1] = 0;
            }
            stream_sync(st);
            evaluated = ev_h[1];
            // records: (r, s, d, d, 100, 0) for d <= tau, in (r, s) order (oracle.cpp:148-149)
            uint64_t m = 0;
            for (uint64_t x = 0; x < n_pairs; ++x)
                if (hd[x] <= tau) {
                    hr[m] = hr[x];
                    hs[m] = hs[x];
                    hd[m] = hd[x];
                    ++m;
                }
            out->n_records = m;
            out->r = hr;
            out->s = hs;
            out->d = hd;
            out->rank = static_cast<uint32_t*>(std::calloc(std::max<uint64_t>(m, 1), sizeof(uint32_t)));
            if (!out->rank) throw std::bad_alloc();
        } else {
            const uint32_t nr = R.n;
            DevBuf<double> u(std::max<uint32_t>(nr, 1));
            if (k <= (uint32_t)kMaxSeedK && nr) {
                // pass 1: U(r) from the exact distances of the k nearest boxes
                DevBuf<uint32_t> seed_s((uint64_t)nr * k), seed_r((uint64_t)nr * k);
                DevBuf<double> seed_d((uint64_t)nr * k);
                count_launch();
                k_knn_seed<<<(nr + kBoxThreads - 1) / kBoxThreads, kBoxThreads, 0, st>>>(R.obox.p, nr, S->obox.p,
                                                                                        S->n, k, seed_s.p);
                TJ_CUDA(cudaGetLastError());
                count_launch();
                k_seed_pairs<<<grid_for((uint64_t)nr * k, 256, ws.num_sms), 256, 0, st>>>(nr, k, seed_r.p);
                TJ_CUDA(cudaGetLastError());
                pair_distances(R, *S, seed_r.p, seed_s.p, (uint64_t)nr * k, seed_d.p, counters.p, ws.num_sms, st);
                TJ_CUDA(cudaMemcpyAsync(ev_h, counters.p, 16, cudaMemcpyDeviceToHost, st));
                stream_sync(st);
                evaluated += ev_h[1];
                count_launch();
                k_knn_bound<<<grid_for(nr, 256, ws.num_sms), 256, 0, st>>>(seed_d.p, seed_s.p, nr, k, u.p);
                TJ_CUDA(cudaGetLastError());
            } else if (nr) {
                const double inf = std::numeric_limits<double>::infinity();
                std::vector<double> hu(nr, inf);
                TJ_CUDA(cudaMemcpyAsync(u.p, hu.data(), nr * 8, cudaMemcpyHostToDevice, st));
                stream_sync(st);
            }
            // pass 2: every s within U(r), exact distances, per-r stable sort by (d, s)
            n_pairs = box_pairs(R, *S, 0.0, u.p, offsets, pr, ps, ws, st);
            d.alloc(std::max<uint64_t>(n_pairs, 1));
            pair_distances(R, *S, pr.p, ps.p, n_pairs, d.p, counters.p, ws.num_sms, st);
            DevBuf<unsigned long long> keys(std::max<uint64_t>(n_pairs, 1)), keys_out(std::max<uint64_t>(n_pairs, 1));
            DevBuf<uint32_t> vals_out(std::max<uint64_t>(n_pairs, 1));
            if (n_pairs) {
                count_launch();
                k_to_bits<<<grid_for(n_pairs, 256, ws.num_sms), 256, 0, st>>>(d.p, n_pairs, keys.p);
                TJ_CUDA(cudaGetLastError());
                size_t bytes = 0;
                TJ_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, bytes, keys.p, keys_out.p, ps.p, vals_out.p,
                                                                  (int64_t)n_pairs, (int64_t)nr, offsets.p,
                                                                  offsets.p + 1, st));
                ws.temp.reserve(bytes);
                TJ_CUDA(cub::DeviceSegmentedSort::StableSortPairs(ws.temp.p, bytes, keys.p, keys_out.p, ps.p,
                                                                  vals_out.p, (int64_t)n_pairs, (int64_t)nr,
                                                                  offsets.p, offsets.p + 1, st));
                TJ_CUDA(cudaMemcpyAsync(ev_h, counters.p, 16, cudaMemcpyDeviceToHost, st));
            } else {
                ev_h[1] = 0;
            }
            std::vector<uint64_t> hoff(nr + 1);
            TJ_CUDA(cudaMemcpyAsync(hoff.data(), offsets.p, (nr + 1) * 8, cudaMemcpyDeviceToHost, st));
            unsigned long long* hk = host_copy(keys_out, n_pairs, st);
            uint32_t* hv = host_copy(vals_out, n_pairs, st);
            stream_sync(st);
            evaluated += ev_h[1];
            uint64_t m = 0;
            for (uint32_t r = 0; r < nr; ++r) m += std::min<uint64_t>(k, hoff[r + 1] - hoff[r]);
            out->r = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(m, 1) * 4));
            out->s = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(m, 1) * 4));
            out->d = static_cast<double*>(std::malloc(std::max<uint64_t>(m, 1) * 8));
            out->rank = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(m, 1) * 4));
            if (!out->r || !out->s || !out->d || !out->rank) throw std::bad_alloc();
            uint64_t w = 0;
            for (uint32_t r = 0; r < nr; ++r) {
                const uint64_t c = std::min<uint64_t>(k, hoff[r + 1] - hoff[r]);
                for (uint64_t x = 0; x < c; ++x, ++w) {
                    out->r[w] = r;
                    out->s[w] = hv[hoff[r] + x];
                    std::memcpy(&out->d[w], &hk[hoff[r] + x], 8);
                    out->rank[w] = (uint32_t)(x + 1);
                }
            }
            std::free(hk);
            std::free(hv);
            out->n_records = m;
        }
        out->object_pairs = n_pairs;
        out->facet_pairs_evaluated = evaluated;
        out->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

extern "C" void tj_exhaustive_result_free(tj_exhaustive_result* res) {
    if (!res) return;
    std::free(res->r);
    std::free(res->s);
    std::free(res->d);
    std::free(res->rank);
    std::memset(res, 0, sizeof(*res));
}
