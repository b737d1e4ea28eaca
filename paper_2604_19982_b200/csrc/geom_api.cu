// Geometric primitives of the reference's public geometry API on the device
// (proj/include/trijoin/geom.hpp:60-79, proj/src/geom.cpp:11-183): mindist_aabb,
// point_segment_distance, point_triangle_distance, segment_segment_distance and
// tri_tri_distance over n independent inputs, bit-identical to the reference's non-FMA
// FP64 arithmetic (csrc/geom_exact.cuh). The reference's geometry tests and tools call the
// scalar forms one pair at a time, so small calls skip every allocation and copy: the
// inputs go into a page-locked, device-mapped mailbox of the calling thread that the
// kernel reads and writes over PCIe directly (one launch + one stream wait per call).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "filter.cuh"
#include "geom_exact.cuh"

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

constexpr int kGeoThreads = 128;

// doubles per input of each operation: {a, b}
__host__ __device__ constexpr int width_a(int op) {
    return op == TJ_GEOM_MINDIST ? 6 : op == TJ_GEOM_TRI_TRI ? 9 : op == TJ_GEOM_SEGMENT_SEGMENT ? 6 : 3;
}
__host__ __device__ constexpr int width_b(int op) {
    return op == TJ_GEOM_MINDIST ? 6 : op == TJ_GEOM_POINT_SEGMENT ? 6 : op == TJ_GEOM_SEGMENT_SEGMENT ? 6 : 9;
}

__device__ __forceinline__ V3 ld3(const double* p) { return {p[0], p[1], p[2]}; }

__device__ __noinline__ double tri_tri_geo(uint32_t a, uint32_t b) {
    staged_read_barrier();
    return tri_tri(a, b); }
__device__ __noinline__ double point_tri_geo(const V3& p, uint32_t t) {
    staged_read_barrier();
    return point_triangle_d2(p, t); }

__global__ void __launch_bounds__(kGeoThreads) k_geom(int op, uint64_t n, const double* __restrict__ a,
                                                      const double* __restrict__ b, double* __restrict__ out) {
    __shared__ double rec[kGeoThreads][2][kFacetWords];
    const uint32_t ta = static_cast<uint32_t>(__cvta_generic_to_shared(&rec[threadIdx.x][0][0]));
    const uint32_t tb = static_cast<uint32_t>(__cvta_generic_to_shared(&rec[threadIdx.x][1][0]));
    const int wa = width_a(op), wb = width_b(op);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double* x = a + wa * i;
        const double* y = b + wb * i;
        double n2, s2, r;
        switch (op) {
        case TJ_GEOM_MINDIST: // src/geom.cpp:11-16
            r = mindist_box(x, y);
            break;
        case TJ_GEOM_POINT_SEGMENT: // src/geom.cpp:18-24 (distance == sqrt(norm2), one rounding each)
            r = TJ_SQRT(point_segment_d2(ld3(x), ld3(y), ld3(y + 3)));
            break;
        case TJ_GEOM_POINT_TRIANGLE: // src/geom.cpp:39-80
            stage_exact(y, 0.0, 0.0, tb, &n2, &s2);
            r = TJ_SQRT(point_tri_geo(ld3(x), tb));
            break;
        case TJ_GEOM_SEGMENT_SEGMENT: // src/geom.cpp:82-113
            r = TJ_SQRT(segment_segment_d2(ld3(x), ld3(x + 3), ld3(y), ld3(y + 3)));
            break;
        default: // TJ_GEOM_TRI_TRI, src/geom.cpp:152-183
            stage_exact(x, 0.0, 0.0, ta, &n2, &s2);
            stage_exact(y, 0.0, 0.0, tb, &n2, &s2);
            r = tri_tri_geo(ta, tb);
            break;
        }
        out[i] = r;
    }
}

// Calling thread's mapped mailbox (portable: usable with every device's context).
struct Mailbox {
    double* p = nullptr;
    size_t cap = 0; // doubles
    ~Mailbox() {
        if (p) cudaFreeHost(p);
    }
    double* get(size_t n) {
        if (n > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            TJ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), n * sizeof(double),
                                  cudaHostAllocMapped | cudaHostAllocPortable));
            cap = n;
        }
        return p;
    }
};
constexpr size_t kMailboxPairs = 256; // calls up to this size use the mailbox

template <class F>
int run(tj_ctx* ctx, F&& f) {
    struct Box {
        F* f;
        static void call(void* p) { (*static_cast<Box*>(p)->f)(); }
    } box{&f};
    return guarded_call(ctx, &Box::call, &box);
}

void launch_geom(int op, uint64_t n, const double* a, const double* b, double* out, int num_sms, cudaStream_t st) {
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + kGeoThreads - 1) / kGeoThreads,
                                                                   (uint64_t)num_sms * 8));
    count_launch();
    k_geom<<<grid, kGeoThreads, 0, st>>>(op, n, a, b, out);
    TJ_CUDA(cudaGetLastError());
}

} // namespace

extern "C" int tj_geom_batch(tj_ctx* ctx, int32_t op, uint64_t n, const double* a, const double* b, double* out) {
    if (!ctx) return TJ_EINVAL;
    return run(ctx, [&] {
        if (op < TJ_GEOM_MINDIST || op > TJ_GEOM_TRI_TRI) throw Error(TJ_EINVAL, "tj_geom_batch: unknown operation");
        if (!n) return;
        if (!a || !b || !out) throw Error(TJ_EINVAL, "tj_geom_batch: null buffer");
        const tj_ctx_view cv = ctx_view(ctx);
        const size_t wa = width_a(op), wb = width_b(op);
        if (n <= kMailboxPairs) {
            static thread_local Mailbox box;
            double* m = box.get(kMailboxPairs * (9 + 9 + 1));
            std::memcpy(m, a, n * wa * sizeof(double));
            std::memcpy(m + n * wa, b, n * wb * sizeof(double));
            double* mo = m + n * (wa + wb);
            launch_geom(op, n, m, m + n * wa, mo, cv.ws->num_sms, cv.stream);
            stream_sync(cv.stream);
            std::memcpy(out, mo, n * sizeof(double));
            return;
        }
        DevBuf<double> da(n * wa), db(n * wb), dout(n);
        TJ_CUDA(cudaMemcpyAsync(da.p, a, n * wa * sizeof(double), cudaMemcpyHostToDevice, cv.stream));
        TJ_CUDA(cudaMemcpyAsync(db.p, b, n * wb * sizeof(double), cudaMemcpyHostToDevice, cv.stream));
        launch_geom(op, n, da.p, db.p, dout.p, cv.ws->num_sms, cv.stream);
        TJ_CUDA(cudaMemcpyAsync(out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost, cv.stream));
        stream_sync(cv.stream);
    });
}

extern "C" int tj_tri_tri_batch(tj_ctx* ctx, uint64_t n, const double* a9, const double* b9, double* out) {
    return tj_geom_batch(ctx, TJ_GEOM_TRI_TRI, n, a9, b9, out);
}

extern "C" int tj_mindist_batch(tj_ctx* ctx, uint64_t n, const double* a6, const double* b6, double* out) {
    return tj_geom_batch(ctx, TJ_GEOM_MINDIST, n, a6, b6, out);
}
