// Offline preprocessing on the GPU: the per-facet Hausdorff paddings
// hd (reference compute_facet_hd, src/hausdorff.cpp:15-27: 45 point-to-mesh queries per facet
// at grid 8) and ph (src/simplify.cpp:238-252 / :256-267), and the k-means voxelisation of the
// coarsest level (src/voxelize.cpp:27-79). Bit-exact with the reference:
//   * point-to-mesh distance = the reference TriBvh::point_distance (src/bvh.cpp:86-112): the
//     same tree (median split on the longest axis with the (centroid, id) total order of
//     src/bvh.cpp:51-80 — the leaf *sets* and node boxes are determined by that order, the
//     order inside a leaf is not and does not matter to a minimum) traversed by the same
//     stack discipline, so even its pruning ties resolve identically; point_triangle_distance
//     is geom_exact.cuh's bit-exact restatement;
//   * every max / min is of non-negative doubles (order-free); every sum is evaluated in the
//     reference's association order (k-means centre sums run per cluster in facet order).
// The edge-collapse simplifier itself is sequential and stays a CPU tool.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "filter.cuh"
#include "geom_exact.cuh"
#include "tj_internal.cuh"
#include "host/bvh_build.hpp"

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
using tjx::bvh::BvhNode;
using tjx::bvh::HostBvh;
using tjx::bvh::TriSoup;
using tjx::bvh::build_bvh;

namespace {

constexpr int kPreThreads = 128;

// ---------------------------------------------------------------- device
__device__ __forceinline__ double point_box_distance(const V3& p, const BvhNode& n) { // src/bvh.cpp:11-16
    double g[3];
    const double pv[3] = {p.x, p.y, p.z};
#pragma unroll
    for (int d = 0; d < 3; ++d) { // std::max({0.0, lo - p, p - hi}): the first largest
        double m = 0.0;
        const double a = TJ_SUB(n.lo[d], pv[d]), b = TJ_SUB(pv[d], n.hi[d]);
        if (m < a) m = a;
        if (m < b) m = b;
        g[d] = m;
    }
    return TJ_SQRT(TJ_ADD(TJ_ADD(TJ_MUL(g[0], g[0]), TJ_MUL(g[1], g[1])), TJ_MUL(g[2], g[2])));
}

__device__ __forceinline__ BvhNode load_node(const BvhNode* __restrict__ nodes, uint32_t i) {
    BvhNode n;
    const double2* s = reinterpret_cast<const double2*>(nodes + i);
    const double2 a = __ldg(s), b = __ldg(s + 1), c = __ldg(s + 2);
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(s + 3));
    n.lo[0] = a.x; n.lo[1] = a.y; n.lo[2] = b.x;
    n.hi[0] = b.y; n.hi[1] = c.x; n.hi[2] = c.y;
    n.left = u.x; n.count = u.y; n.right = u.z; n.pad = 0;
    return n;
}

// Leaf-ordered triangles for the point queries: kTriWords doubles each (the 9 coordinates, the
// triangle_degenerate flag, 2 pad), read straight into registers by the traversal.
constexpr int kTriWords = 12;
__global__ void k_stage_soup(const double* __restrict__ verts, const uint32_t* __restrict__ facets,
                             const uint32_t* __restrict__ order, const uint64_t* __restrict__ mesh_of_tri,
                             const uint64_t* __restrict__ vert_off, const uint64_t* __restrict__ facet_off,
                             uint64_t n, double* __restrict__ recs) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t m = mesh_of_tri[i];
        const uint64_t f = facet_off[m] + order[i];
        const double* v = verts + 3 * vert_off[m];
        double c[9];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint32_t vid = facets[3 * f + k];
            c[3 * k] = v[3 * (size_t)vid];
            c[3 * k + 1] = v[3 * (size_t)vid + 1];
            c[3 * k + 2] = v[3 * (size_t)vid + 2];
        }
        const V3 v0 = {c[0], c[1], c[2]}, v1 = {c[3], c[4], c[5]}, v2 = {c[6], c[7], c[8]};
        double* r = recs + i * kTriWords;
#pragma unroll
        for (int k = 0; k < 9; ++k) r[k] = c[k];
        r[9] = tri_degenerate(v0, v1, v2, nullptr, nullptr) ? 1.0 : 0.0;
        r[10] = r[11] = 0.0;
    }
}


__device__ __forceinline__ double leaf_tri_distance(const V3& p, const double* __restrict__ r) {
    const double2* r2 = reinterpret_cast<const double2*>(r);
    const double2 x0 = __ldg(r2), x1 = __ldg(r2 + 1), x2 = __ldg(r2 + 2), x3 = __ldg(r2 + 3), x4 = __ldg(r2 + 4);
    const V3 a = {x0.x, x0.y, x1.x}, b = {x1.y, x2.x, x2.y}, c = {x3.x, x3.y, x4.x};
    return TJ_SQRT(point_triangle_d2(p, a, b, c, x4.y != 0.0));
}

// TriBvh::point_distance (src/bvh.cpp:86-112).
__device__ double bvh_point_distance(const V3& p, const BvhNode* __restrict__ nodes, const double* __restrict__ recs) {
    double best = __longlong_as_double(0x7ff0000000000000ll);
    uint32_t stack[64];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        const BvhNode n = load_node(nodes, stack[--top]);
        if (point_box_distance(p, n) >= best) continue;
        if (n.count > 0) {
            for (uint32_t i = 0; i < n.count; ++i) best = smin(best, leaf_tri_distance(p, recs + (size_t)(n.left + i) * kTriWords));
            continue;
        }
        const double dl = point_box_distance(p, load_node(nodes, n.left));
        const double dr = point_box_distance(p, load_node(nodes, n.right));
        if (dl < dr) {
            if (dr < best && top < 63) stack[top++] = n.right;
            if (dl < best && top < 63) stack[top++] = n.left;
        } else {
            if (dl < best && top < 63) stack[top++] = n.left;
            if (dr < best && top < 63) stack[top++] = n.right;
        }
    }
    return best;
}

// compute_facet_hd: thread per (query facet, sample); the facet's maximum over its samples is
// folded into hd_bits with a 64-bit atomicMax on the IEEE bits (non-negative doubles order
// like their bit patterns; +inf for an empty original mesh).
__global__ void __launch_bounds__(kPreThreads) k_facet_hd(const double* __restrict__ qtris, const uint32_t* __restrict__ q_mesh,
                                                          uint64_t nq, int grid, const uint64_t* __restrict__ node_off,
                                                          const BvhNode* __restrict__ nodes, const uint64_t* __restrict__ rec_off,
                                                          const double* __restrict__ recs,
                                                          unsigned long long* __restrict__ hd_bits) {
    const uint32_t ns = (uint32_t)((grid + 1) * (grid + 2) / 2);
    const double inv = TJ_DIV(1.0, (double)grid);
    const uint64_t total = nq * ns;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < total; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = w / ns;
        uint32_t s = (uint32_t)(w - q * ns);
        // sample s -> (i, j) with j + i <= grid, i-major (src/hausdorff.cpp:19-20)
        int i = 0;
        while (s > (uint32_t)(grid - i)) {
            s -= (uint32_t)(grid - i + 1);
            ++i;
        }
        const int j = (int)s;
        const double* t = qtris + 9 * q;
        const V3 v0 = {t[0], t[1], t[2]}, v1 = {t[3], t[4], t[5]}, v2 = {t[6], t[7], t[8]};
        const V3 e1 = vsub(v1, v0), e2 = vsub(v2, v0);
        const V3 p = vadd(vadd(v0, vmul(e1, TJ_MUL((double)i, inv))), vmul(e2, TJ_MUL((double)j, inv)));
        const uint32_t m = q_mesh[q];
        const uint64_t n0 = node_off[m];
        double d = __longlong_as_double(0x7ff0000000000000ll);
        if (node_off[m + 1] > n0) d = bvh_point_distance(p, nodes + n0, recs + rec_off[m] * kTriWords);
        const unsigned long long b = (unsigned long long)__double_as_longlong(d);
        if (b > __ldcg(hd_bits + q)) atomicMax(hd_bits + q, b);
    }
}

// worst + hd_covering_radius (src/hausdorff.cpp:11-13): (2/3) * longest_edge / grid
__global__ void k_hd_finish(const double* __restrict__ qtris, uint64_t nq, int grid,
                            const unsigned long long* __restrict__ hd_bits, double* __restrict__ hd) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq; q += (uint64_t)gridDim.x * blockDim.x) {
        const double* t = qtris + 9 * q;
        const V3 v0 = {t[0], t[1], t[2]}, v1 = {t[3], t[4], t[5]}, v2 = {t[6], t[7], t[8]};
        double m = vnorm2(vsub(v1, v0)); // std::max({norm2(v1 - v0), norm2(v2 - v1), norm2(v0 - v2)})
        const double b = vnorm2(vsub(v2, v1)), c = vnorm2(vsub(v0, v2));
        if (m < b) m = b;
        if (m < c) m = c;
        const double r = TJ_DIV(TJ_MUL(2.0 / 3.0, TJ_SQRT(m)), (double)grid);
        hd[q] = TJ_ADD(__longlong_as_double((long long)hd_bits[q]), r);
    }
}

// compute_facet_ph: thread per original facet; max over its 3 vertices of the distance to its
// ancestor facet, folded per LOD facet with atomicMax on the bits (initial 0.0).
__global__ void __launch_bounds__(kPreThreads) k_facet_ph(const double* __restrict__ verts, const uint32_t* __restrict__ facets,
                                                          const uint64_t* __restrict__ vert_off,
                                                          const uint64_t* __restrict__ facet_off,
                                                          const uint32_t* __restrict__ facet_mesh, uint64_t n_orig,
                                                          const uint32_t* __restrict__ ancestor,
                                                          const uint64_t* __restrict__ lod_off, const double* __restrict__ lod_tris,
                                                          unsigned long long* __restrict__ ph_bits) {
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < n_orig; o += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = facet_mesh[o];
        const uint64_t lf = lod_off[m] + ancestor[o];
        const double* c = lod_tris + 9 * lf;
        const V3 t0 = {c[0], c[1], c[2]}, t1 = {c[3], c[4], c[5]}, t2 = {c[6], c[7], c[8]};
        const bool degen = tri_degenerate(t0, t1, t2, nullptr, nullptr);
        const double* v = verts + 3 * vert_off[m];
        double best = 0.0;
#pragma unroll 1
        for (int k = 0; k < 3; ++k) {
            const uint32_t vid = facets[3 * o + k];
            const V3 p = {v[3 * (size_t)vid], v[3 * (size_t)vid + 1], v[3 * (size_t)vid + 2]};
            best = smax(best, TJ_SQRT(point_triangle_d2(p, t0, t1, t2, degen)));
        }
        const unsigned long long b = (unsigned long long)__double_as_longlong(best);
        if (b > __ldcg(ph_bits + lf)) atomicMax(ph_bits + lf, b);
    }
}

// ---- k-means (src/voxelize.cpp:27-79) over many objects at once
__global__ void k_centroids(const double* __restrict__ verts, const uint32_t* __restrict__ facets,
                            const uint64_t* __restrict__ vert_off, const uint32_t* __restrict__ facet_obj, uint64_t nf,
                            double* __restrict__ cen) {
    for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < nf; f += (uint64_t)gridDim.x * blockDim.x) {
        const double* v = verts + 3 * vert_off[facet_obj[f]];
        const uint32_t a = facets[3 * f], b = facets[3 * f + 1], c = facets[3 * f + 2];
#pragma unroll
        for (int d = 0; d < 3; ++d) // (v0 + v1 + v2) * (1 / 3)
            cen[3 * f + d] = TJ_MUL(TJ_ADD(TJ_ADD(v[3 * (size_t)a + d], v[3 * (size_t)b + d]), v[3 * (size_t)c + d]),
                                    1.0 / 3.0);
    }
}

// nearest_center: strict <, the first smallest wins (src/voxelize.cpp:12-23)
__global__ void k_assign(const double* __restrict__ cen, const uint32_t* __restrict__ facet_obj, uint64_t nf,
                         const uint64_t* __restrict__ center_off, const double* __restrict__ centers,
                         uint32_t* __restrict__ labels) {
    for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < nf; f += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = facet_obj[f];
        const V3 p = {cen[3 * f], cen[3 * f + 1], cen[3 * f + 2]};
        const uint64_t c0 = center_off[o], c1 = center_off[o + 1];
        double best = __longlong_as_double(0x7ff0000000000000ll);
        uint32_t bc = 0;
        for (uint64_t c = c0; c < c1; ++c) {
            const V3 q = {__ldg(centers + 3 * c), __ldg(centers + 3 * c + 1), __ldg(centers + 3 * c + 2)};
            const double d = vnorm2(vsub(p, q));
            if (d < best) {
                best = d;
                bc = (uint32_t)(c - c0);
            }
        }
        labels[f] = bc;
    }
}

// One Lloyd update: thread per (object, cluster), summing the cluster's centroids in facet
// order (the reference's sequential `sums[labels[f]] += centroids[f]`).
__global__ void k_update(const double* __restrict__ cen, const uint32_t* __restrict__ labels,
                         const uint64_t* __restrict__ facet_off, const uint32_t* __restrict__ center_obj,
                         const uint64_t* __restrict__ center_off, uint64_t n_centers, double* __restrict__ centers) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < n_centers; c += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = center_obj[c];
        const uint32_t lc = (uint32_t)(c - center_off[o]);
        double sx = 0.0, sy = 0.0, sz = 0.0;
        uint64_t cnt = 0;
        for (uint64_t f = facet_off[o]; f < facet_off[o + 1]; ++f) {
            if (labels[f] != lc) continue;
            sx = TJ_ADD(sx, cen[3 * f]);
            sy = TJ_ADD(sy, cen[3 * f + 1]);
            sz = TJ_ADD(sz, cen[3 * f + 2]);
            ++cnt;
        }
        if (cnt > 0) {
            const double s = TJ_DIV(1.0, (double)cnt);
            centers[3 * c] = TJ_MUL(sx, s);
            centers[3 * c + 1] = TJ_MUL(sy, s);
            centers[3 * c + 2] = TJ_MUL(sz, s);
        }
    }
}

// SplitMix64 (include/trijoin/rng.hpp): the published generator and its unbiased next_below.
struct SplitMix64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    uint64_t next_below(uint64_t n) {
        if (n <= 1) return 0;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t v = next();
        while (v >= limit) v = next();
        return v % n;
    }
};

inline int grid_for(uint64_t n, int threads, int num_sms) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + threads - 1) / threads, (uint64_t)num_sms * 16));
}

template <class T>
void to_dev(DevBuf<T>& d, const T* h, size_t n, cudaStream_t st) {
    d.alloc(std::max<size_t>(n, 1));
    if (n) TJ_CUDA(cudaMemcpyAsync(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

// Validates a packed mesh set (offsets non-decreasing, vertex ids in range).
void check_meshes(uint32_t n, const uint64_t* vo, const uint64_t* fo, const uint32_t* facets, const char* what) {
    if (n && (!vo || !fo)) throw Error(TJ_EINVAL, std::string(what) + ": null offsets");
    for (uint32_t m = 0; m < n; ++m) {
        if (vo[m + 1] < vo[m] || fo[m + 1] < fo[m]) throw Error(TJ_EINVAL, std::string(what) + ": offsets decrease");
        const uint64_t nv = vo[m + 1] - vo[m];
        for (uint64_t i = 3 * fo[m]; i < 3 * fo[m + 1]; ++i)
            if (facets[i] >= nv) throw Error(TJ_EINVAL, std::string(what) + ": facet vertex id out of range");
    }
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

extern "C" int tj_facet_hd_batch(tj_ctx* ctx, uint32_t n_meshes, const uint64_t* vert_off, const double* verts,
                                 const uint64_t* facet_off, const uint32_t* facets, const uint64_t* query_off,
                                 const double* query_tris9, int32_t grid, double* hd_out) {
    if (!ctx) return TJ_EINVAL;
    return run(ctx, [&] {
        if (grid < 1) throw Error(TJ_EINVAL, "compute_facet_hd: grid_level must be >= 1");
        check_meshes(n_meshes, vert_off, facet_off, facets, "compute_facet_hd");
        if (n_meshes && !query_off) throw Error(TJ_EINVAL, "compute_facet_hd: null query offsets");
        const uint64_t nq = n_meshes ? query_off[n_meshes] : 0;
        if (!nq) return;
        if (!query_tris9 || !hd_out) throw Error(TJ_EINVAL, "compute_facet_hd: null buffer");
        const tj_ctx_view cv = ctx_view(ctx);
        cudaStream_t st = cv.stream;
        // trees on the host (O(n log n) per mesh), leaf-ordered triangles staged on the device
        std::vector<uint64_t> node_off(n_meshes + 1, 0), rec_off(n_meshes + 1, 0);
        std::vector<BvhNode> nodes;
        std::vector<uint32_t> order;
        std::vector<uint64_t> tri_mesh;
        std::vector<HostBvh> trees(n_meshes);
        {
            std::atomic<uint32_t> next{0};
            auto work = [&] {
                for (uint32_t m; (m = next.fetch_add(1)) < n_meshes;)
                    trees[m] = build_bvh(TriSoup{verts + 3 * vert_off[m], facets + 3 * facet_off[m]},
                                         (uint32_t)(facet_off[m + 1] - facet_off[m]));
            };
            const unsigned nt = std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), n_meshes);
            std::vector<std::thread> pool;
            for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
            work();
            for (auto& t : pool) t.join();
        }
        for (uint32_t m = 0; m < n_meshes; ++m) {
            const HostBvh& h = trees[m];
            node_off[m] = nodes.size();
            rec_off[m] = order.size();
            nodes.insert(nodes.end(), h.nodes.begin(), h.nodes.end());
            order.insert(order.end(), h.order.begin(), h.order.end());
            tri_mesh.insert(tri_mesh.end(), h.order.size(), (uint64_t)m);
        }
        node_off[n_meshes] = nodes.size();
        rec_off[n_meshes] = order.size();
        std::vector<uint32_t> q_mesh(nq);
        for (uint32_t m = 0; m < n_meshes; ++m)
            for (uint64_t q = query_off[m]; q < query_off[m + 1]; ++q) q_mesh[q] = m;
        const uint64_t nv = vert_off[n_meshes], nfa = facet_off[n_meshes];
        DevBuf<double> d_verts, d_recs, d_q, d_hd;
        DevBuf<uint32_t> d_fac, d_order, d_qm;
        DevBuf<uint64_t> d_vo, d_fo, d_tm, d_no, d_ro;
        DevBuf<BvhNode> d_nodes;
        DevBuf<unsigned long long> d_bits;
        to_dev(d_verts, verts, 3 * nv, st);
        to_dev(d_fac, facets, 3 * nfa, st);
        to_dev(d_vo, vert_off, n_meshes + 1, st);
        to_dev(d_fo, facet_off, n_meshes + 1, st);
        to_dev(d_order, order.data(), order.size(), st);
        to_dev(d_tm, tri_mesh.data(), tri_mesh.size(), st);
        to_dev(d_nodes, nodes.data(), nodes.size(), st);
        to_dev(d_no, node_off.data(), node_off.size(), st);
        to_dev(d_ro, rec_off.data(), rec_off.size(), st);
        to_dev(d_q, query_tris9, 9 * nq, st);
        to_dev(d_qm, q_mesh.data(), nq, st);
        d_recs.alloc(std::max<size_t>(order.size() * kTriWords, 1));
        d_bits.alloc(nq);
        d_hd.alloc(nq);
        TJ_CUDA(cudaMemsetAsync(d_bits.p, 0, nq * sizeof(unsigned long long), st));
        const int sms = cv.ws->num_sms;
        if (!order.empty()) {
            count_launch();
            k_stage_soup<<<grid_for(order.size(), kPreThreads, sms), kPreThreads, 0, st>>>(
                d_verts.p, d_fac.p, d_order.p, d_tm.p, d_vo.p, d_fo.p, order.size(), d_recs.p);
            TJ_CUDA(cudaGetLastError());
        }
        const uint64_t work = nq * (uint64_t)((grid + 1) * (grid + 2) / 2);
        count_launch();
        k_facet_hd<<<grid_for(work, kPreThreads, sms), kPreThreads, 0, st>>>(d_q.p, d_qm.p, nq, grid, d_no.p, d_nodes.p,
                                                                           d_ro.p, d_recs.p, d_bits.p);
        TJ_CUDA(cudaGetLastError());
        count_launch();
        k_hd_finish<<<grid_for(nq, 256, sms), 256, 0, st>>>(d_q.p, nq, grid, d_bits.p, d_hd.p);
        TJ_CUDA(cudaGetLastError());
        TJ_CUDA(cudaMemcpyAsync(hd_out, d_hd.p, nq * sizeof(double), cudaMemcpyDeviceToHost, st));
        stream_sync(st);
    });
}

extern "C" int tj_facet_ph_batch(tj_ctx* ctx, uint32_t n_meshes, const uint64_t* vert_off, const double* verts,
                                 const uint64_t* facet_off, const uint32_t* facets, const uint32_t* ancestor,
                                 const uint64_t* lod_off, const double* lod_tris9, double* ph_out) {
    if (!ctx) return TJ_EINVAL;
    return run(ctx, [&] {
        check_meshes(n_meshes, vert_off, facet_off, facets, "compute_facet_ph");
        if (n_meshes && !lod_off) throw Error(TJ_EINVAL, "compute_facet_ph: null LOD offsets");
        const uint64_t nl = n_meshes ? lod_off[n_meshes] : 0, no = n_meshes ? facet_off[n_meshes] : 0;
        if (!nl) return;
        if (!lod_tris9 || !ph_out || (no && !ancestor)) throw Error(TJ_EINVAL, "compute_facet_ph: null buffer");
        std::vector<uint32_t> fmesh(no);
        for (uint32_t m = 0; m < n_meshes; ++m) {
            const uint64_t n_lod = lod_off[m + 1] - lod_off[m];
            for (uint64_t o = facet_off[m]; o < facet_off[m + 1]; ++o) {
                if (ancestor[o] >= n_lod) throw Error(TJ_EINVAL, "compute_facet_ph: ancestor id out of range");
                fmesh[o] = m;
            }
        }
        const tj_ctx_view cv = ctx_view(ctx);
        cudaStream_t st = cv.stream;
        DevBuf<double> d_verts, d_lod, d_ph;
        DevBuf<uint32_t> d_fac, d_fm, d_anc;
        DevBuf<uint64_t> d_vo, d_fo, d_lo;
        DevBuf<unsigned long long> d_bits;
        to_dev(d_verts, verts, 3 * vert_off[n_meshes], st);
        to_dev(d_fac, facets, 3 * no, st);
        to_dev(d_vo, vert_off, n_meshes + 1, st);
        to_dev(d_fo, facet_off, n_meshes + 1, st);
        to_dev(d_fm, fmesh.data(), no, st);
        to_dev(d_anc, ancestor, no, st);
        to_dev(d_lo, lod_off, n_meshes + 1, st);
        to_dev(d_lod, lod_tris9, 9 * nl, st);
        d_bits.alloc(nl);
        TJ_CUDA(cudaMemsetAsync(d_bits.p, 0, nl * sizeof(unsigned long long), st));
        if (no) {
            count_launch();
            k_facet_ph<<<grid_for(no, kPreThreads, cv.ws->num_sms), kPreThreads, 0, st>>>(
                d_verts.p, d_fac.p, d_vo.p, d_fo.p, d_fm.p, no, d_anc.p, d_lo.p, d_lod.p, d_bits.p);
            TJ_CUDA(cudaGetLastError());
        }
        static_assert(sizeof(unsigned long long) == sizeof(double), "bit copy");
        TJ_CUDA(cudaMemcpyAsync(ph_out, d_bits.p, nl * sizeof(double), cudaMemcpyDeviceToHost, st));
        stream_sync(st);
    });
}

extern "C" int tj_voxelize_batch(tj_ctx* ctx, uint32_t n_objects, const uint64_t* vert_off, const double* verts,
                                 const uint64_t* facet_off, const uint32_t* facets, const uint32_t* k,
                                 const uint64_t* seeds, uint32_t* labels_out) {
    if (!ctx) return TJ_EINVAL;
    return run(ctx, [&] {
        check_meshes(n_objects, vert_off, facet_off, facets, "voxelize");
        if (n_objects && (!k || !seeds)) throw Error(TJ_EINVAL, "voxelize: null k / seeds");
        const uint64_t nf = n_objects ? facet_off[n_objects] : 0;
        // initial centres (src/voxelize.cpp:36-50): a draw of vertices without replacement
        std::vector<uint64_t> center_off(n_objects + 1, 0);
        std::vector<double> centers;
        std::vector<uint32_t> center_obj, facet_obj(nf);
        for (uint32_t o = 0; o < n_objects; ++o) {
            if (k[o] == 0) throw Error(TJ_EINVAL, "voxelize: k must be >= 1");
            const uint64_t nfo = facet_off[o + 1] - facet_off[o], nv = vert_off[o + 1] - vert_off[o];
            const uint32_t ko = (uint32_t)std::min<uint64_t>(k[o], nfo);
            center_off[o] = center_obj.size();
            std::fill(facet_obj.begin() + facet_off[o], facet_obj.begin() + facet_off[o + 1], o);
            if (ko && !nv) throw Error(TJ_EINVAL, "voxelize: facets without vertices");
            SplitMix64 rng{seeds[o]};
            std::vector<uint32_t> vids(nv);
            std::iota(vids.begin(), vids.end(), 0u);
            const double* v = verts + 3 * vert_off[o];
            for (uint32_t c = 0; c < ko; ++c) {
                uint32_t vid;
                if (c < nv) {
                    const size_t j = c + (size_t)rng.next_below(nv - c);
                    std::swap(vids[c], vids[j]);
                    vid = vids[c];
                } else {
                    vid = (uint32_t)rng.next_below(nv);
                }
                centers.insert(centers.end(), {v[3 * (size_t)vid], v[3 * (size_t)vid + 1], v[3 * (size_t)vid + 2]});
                center_obj.push_back(o);
            }
        }
        center_off[n_objects] = center_obj.size();
        if (!nf) return;
        if (!labels_out) throw Error(TJ_EINVAL, "voxelize: null buffer");
        const tj_ctx_view cv = ctx_view(ctx);
        cudaStream_t st = cv.stream;
        const int sms = cv.ws->num_sms;
        DevBuf<double> d_verts, d_cen, d_centers;
        DevBuf<uint32_t> d_fac, d_fobj, d_cobj, d_lab;
        DevBuf<uint64_t> d_vo, d_fo, d_co;
        to_dev(d_verts, verts, 3 * vert_off[n_objects], st);
        to_dev(d_fac, facets, 3 * nf, st);
        to_dev(d_vo, vert_off, n_objects + 1, st);
        to_dev(d_fo, facet_off, n_objects + 1, st);
        to_dev(d_fobj, facet_obj.data(), nf, st);
        to_dev(d_cobj, center_obj.data(), center_obj.size(), st);
        to_dev(d_co, center_off.data(), center_off.size(), st);
        to_dev(d_centers, centers.data(), centers.size(), st);
        d_cen.alloc(3 * nf);
        d_lab.alloc(nf);
        count_launch();
        k_centroids<<<grid_for(nf, 256, sms), 256, 0, st>>>(d_verts.p, d_fac.p, d_vo.p, d_fobj.p, nf, d_cen.p);
        TJ_CUDA(cudaGetLastError());
        for (int round = 0; round <= 2; ++round) { // assign, then two (update, assign) rounds
            if (round > 0) {
                count_launch();
                k_update<<<grid_for(center_obj.size(), 128, sms), 128, 0, st>>>(d_cen.p, d_lab.p, d_fo.p, d_cobj.p, d_co.p,
                                                                               center_obj.size(), d_centers.p);
                TJ_CUDA(cudaGetLastError());
            }
            count_launch();
            k_assign<<<grid_for(nf, 128, sms), 128, 0, st>>>(d_cen.p, d_fobj.p, nf, d_co.p, d_centers.p, d_lab.p);
            TJ_CUDA(cudaGetLastError());
        }
        TJ_CUDA(cudaMemcpyAsync(labels_out, d_lab.p, nf * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        stream_sync(st);
        // drop empty clusters, relabel contiguously in cluster order (src/voxelize.cpp:69-77)
        for (uint32_t o = 0; o < n_objects; ++o) {
            const uint64_t kc = center_off[o + 1] - center_off[o];
            std::vector<uint32_t> remap(kc, UINT32_MAX);
            for (uint64_t f = facet_off[o]; f < facet_off[o + 1]; ++f) remap[labels_out[f]] = 0;
            uint32_t next = 0;
            for (uint64_t c = 0; c < kc; ++c)
                if (remap[c] != UINT32_MAX) remap[c] = next++;
            for (uint64_t f = facet_off[o]; f < facet_off[o + 1]; ++f) labels_out[f] = remap[labels_out[f]];
        }
    });
}
