// Internal device-side types shared by the kernels and the C-ABI implementation.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tj_capi.h"

namespace tjx {

// Process-wide count of this library's own kernel launches (tj_kernel_launches()).
unsigned long long& launch_counter_ref();
inline void count_launch() { __atomic_fetch_add(&launch_counter_ref(), 1ull, __ATOMIC_RELAXED); }

// Error carried through the C-ABI boundary as a status code.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TJ_CUDA(call)                                                                         \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            throw ::tjx::Error(e_ == cudaErrorMemoryAllocation ? TJ_ENOMEM : TJ_ECUDA,        \
                               std::string(#call) + ": " + cudaGetErrorString(e_));           \
    } while (0)

// Minimal owning device buffer.
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) TJ_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    // grow-only reallocation (contents not preserved)
    void reserve(size_t count) { if (count > n) alloc(count); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// A prepared dataset resident in HBM (the device image of reference PreparedDataset).
struct DatasetDev {
    uint32_t n_objects = 0;
    uint64_t n_voxels = 0;
    std::vector<int32_t> levels;          // host copy of the lod schedule
    DevBuf<double> mbb, anchor;           // [n_obj*6], [n_obj*3]
    DevBuf<uint64_t> voxel_offsets;       // [n_obj+1]
    std::vector<uint64_t> voxel_offsets_h;
    DevBuf<double> voxel_box, voxel_anchor; // [nv*6], [nv*3]
    std::vector<DevBuf<uint64_t>> facet_offsets; // per level [nv+1]
    std::vector<DevBuf<double>> facets;          // per level [entries*12]
    uint64_t bytes = 0;
};

// Active voxel pair during refinement: candidate op + global voxel ids.
struct ActiveVpDev {
    uint32_t op, gvr, gvs;
};

// Arguments of a refinement launch in join mode.
struct RefineJoinArgs {
    const ActiveVpDev* active;
    uint64_t n_vp;
    const uint64_t* r_foff; // R facet offsets of this level, by global voxel
    const double* r_facets;
    const uint64_t* s_foff;
    const double* s_facets;
    unsigned long long* op_lb_bits; // atomicMin targets (non-negative doubles as u64)
    unsigned long long* op_ub_bits;
    double* vp_lb; // optional per-vp outputs (nullptr = off)
    double* vp_ub;
    unsigned long long* work; // dynamic work counter
    unsigned long long* counters; // [2]: tested, evaluated
    int cull;
};

struct RefineBatchArgs {
    const double* facets; // [n_tris*12]
    const uint64_t* r_off;
    const uint64_t* s_off;
    const uint32_t* r_len;
    const uint32_t* s_len;
    uint64_t n_vp;
    double* vp_lb;
    double* vp_ub;
    unsigned long long* work;
    unsigned long long* counters;
    int cull;
};

// kernels (refine.cu)
void launch_refine_join(const RefineJoinArgs& a, int num_sms, cudaStream_t st);
void launch_refine_batch(const RefineBatchArgs& a, int num_sms, cudaStream_t st);
void launch_tri_tri_batch(uint64_t n, const double* a9, const double* b9, double* out, cudaStream_t st);
void launch_mindist_batch(uint64_t n, const double* a6, const double* b6, double* out, cudaStream_t st);

} // namespace tjx
