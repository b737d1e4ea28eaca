// C-ABI implementation (include/tj_capi.h): contexts, HBM-resident datasets, the full
// device join pipeline (reference run_join, src/engine.cpp:122-237) and the primitive
// batch entry points. No CPU compute path exists behind any of these functions.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "filter.cuh"
#include "trace_sink.h"

using namespace tjx;

struct tj_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    Workspace ws;
    std::mutex err_mu; // tj_dataset_put_level may fail on another thread than tj_join
    std::string last_error;
};

struct tj_dataset {
    tj_ctx* ctx = nullptr;
    DatasetDev d;
};

namespace {

std::mutex g_err_mu;
std::string g_err;

void set_global_error(const std::string& m) {
    std::lock_guard<std::mutex> lk(g_err_mu);
    g_err = m;
}

void set_ctx_error(tj_ctx* ctx, const char* m) {
    if (ctx) {
        std::lock_guard<std::mutex> lk(ctx->err_mu);
        ctx->last_error = m;
    }
    set_global_error(m);
}

// Restores the thread's allocation stream on scope exit.
struct AllocStreamScope {
    cudaStream_t saved;
    explicit AllocStreamScope(cudaStream_t s) : saved(alloc_stream()) { alloc_stream() = s; }
    ~AllocStreamScope() { alloc_stream() = saved; }
};

template <class F>
int guarded(tj_ctx* ctx, F&& f) {
    try {
        if (ctx) TJ_CUDA(cudaSetDevice(ctx->device));
        AllocStreamScope scope(ctx ? ctx->stream : nullptr);
        f();
        return TJ_OK;
    } catch (const Error& e) {
        set_ctx_error(ctx, e.what());
        return e.code;
    } catch (const std::bad_alloc& e) {
        set_ctx_error(ctx, "host allocation failed");
        return TJ_ENOMEM;
    } catch (const std::exception& e) {
        set_ctx_error(ctx, e.what());
        return TJ_ECUDA;
    }
}

template <class T>
void upload(DevBuf<T>& dst, const T* src, size_t n, cudaStream_t st) {
    dst.alloc(n ? n : 1);
    if (n) TJ_CUDA(cudaMemcpyAsync(dst.p, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

void validate_spec(const tj_join_spec& s) {
    // validate(JoinSpec) (src/engine.cpp:38-56)
    if (s.type == TJ_KNN) {
        if (s.k == 0) throw Error(TJ_EINVAL, "join: k must be >= 1");
    } else if (s.type == TJ_WITHIN || s.type == TJ_INTERSECT) {
        if (!(s.tau >= 0)) throw Error(TJ_EINVAL, "join: tau must be >= 0");
        if (s.type == TJ_INTERSECT && s.tau != 0.0) throw Error(TJ_EINVAL, "join: intersection requires tau == 0");
    } else {
        throw Error(TJ_EINVAL, "join: unknown join type");
    }
    if (s.filter_chunk == 0) throw Error(TJ_EINVAL, "join: filter chunk must be >= 1");
    if (s.refine_chunk == 0) throw Error(TJ_EINVAL, "join: refine chunk must be >= 1");
    if (s.n_lods == 0 || !s.lods || s.lods[s.n_lods - 1] != 100)
        throw Error(TJ_EINVAL, "join: lod schedule must end at 100");
    if (s.n_lods > TJ_MAX_LODS) throw Error(TJ_EINVAL, "join: at most 16 lod levels are supported");
    for (uint32_t i = 0; i < s.n_lods; ++i) {
        if (s.lods[i] == 0 || s.lods[i] > 100) throw Error(TJ_EINVAL, "join: lod levels must be in (0, 100]");
        if (i > 0 && s.lods[i] <= s.lods[i - 1]) throw Error(TJ_EINVAL, "join: lod schedule must be ascending");
    }
}

void check_levels(const DatasetDev& d, const tj_join_spec& s) {
    // level_index_of (src/refine.cpp:16-21) throws EngineError
    for (uint32_t i = 0; i < s.n_lods; ++i) {
        bool found = false;
        for (int32_t l : d.levels) found = found || l == (int32_t)s.lods[i];
        if (!found)
            throw Error(TJ_EENGINE,
                        "refine: level " + std::to_string(s.lods[i]) + " is not in the dataset's lod schedule");
    }
}

void check_dev_error(DevError* err, cudaStream_t st) {
    DevError h;
    TJ_CUDA(cudaMemcpyAsync(&h, err, sizeof(DevError), cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    if (h.code == 0) return;
    if (h.kind == 1) throw Error(TJ_EENGINE, "knn_apply_deltas: confirmed count exceeds k");
    throw Error(TJ_EENGINE, "bound crossing: lb " + std::to_string(h.lb) + " > ub " + std::to_string(h.ub));
}

template <class T>
T* host_copy(const DevBuf<T>& src, uint64_t n, cudaStream_t st) {
    T* p = static_cast<T*>(std::malloc(std::max<uint64_t>(n, 1) * sizeof(T)));
    if (!p) throw std::bad_alloc();
    if (n) TJ_CUDA(cudaMemcpyAsync(p, src.p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    return p;
}


// Byte layout of one level's compact arrays in a dataset's staging area (256-B aligned parts).
struct StageLayout {
    uint64_t verts, tris, hd, ph, vf, total;
};
StageLayout stage_layout(uint64_t nvert, uint64_t nfac, uint64_t entries) {
    auto up = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
    StageLayout L;
    L.verts = 0;
    L.tris = up(nvert * 24);
    L.hd = L.tris + up(nfac * 12);
    L.ph = L.hd + up(nfac * 8);
    L.vf = L.ph + up(nfac * 8);
    L.total = L.vf + up(entries * 4);
    return L;
}

// Object and voxel arrays of a dataset view (shared by tj_dataset_upload / _begin).
void upload_objects(DatasetDev& d, const tj_dataset_view* v, cudaStream_t st) {
    if (v->n_levels == 0 || v->n_levels > TJ_MAX_LODS)
        throw Error(TJ_EINVAL, "tj_dataset_upload: n_levels must be in [1, 16]");
    const uint32_t no = v->n_objects;
    if (!v->levels || !v->voxel_offsets || (no && (!v->mbb || !v->anchor)))
        throw Error(TJ_EINVAL, "tj_dataset_upload: null object arrays");
    d.n_objects = no;
    d.levels.assign(v->levels, v->levels + v->n_levels);
    d.voxel_offsets_h.assign(v->voxel_offsets, v->voxel_offsets + no + 1);
    d.n_voxels = d.voxel_offsets_h.back();
    for (uint32_t o = 0; o < no; ++o)
        if (d.voxel_offsets_h[o + 1] < d.voxel_offsets_h[o])
            throw Error(TJ_EINVAL, "tj_dataset_upload: voxel_offsets not monotone");
    if (d.n_voxels && (!v->voxel_box || !v->voxel_anchor)) throw Error(TJ_EINVAL, "tj_dataset_upload: null voxel arrays");
    upload(d.mbb, v->mbb, 6ull * no, st);
    upload(d.anchor, v->anchor, 3ull * no, st);
    upload(d.voxel_offsets, v->voxel_offsets, no + 1ull, st);
    upload(d.voxel_box, v->voxel_box, 6ull * d.n_voxels, st);
    upload(d.voxel_anchor, v->voxel_anchor, 3ull * d.n_voxels, st);
    d.facet_offsets.resize(v->n_levels);
    d.facets.resize(v->n_levels);
    d.bytes = (9ull * no + 9ull * d.n_voxels) * 8 + (no + 1ull) * 8;
}

// Expansion of one level's compact mesh form into the resident record layout, warp per
// voxel: entry e of voxel v (object o) gets (v0, v1, v2, hd, ph, 0) of o's facet
// voxel_facets[e] (the record the reference's gather_facet_data builds per chunk,
// src/refine.cpp:25-61). Object-local ids are rebased here and range-checked against the
// object's counts; an out-of-range id is clamped (never read out of bounds) and flagged.
template <class Id>
__global__ void k_expand_level(const double* __restrict__ verts, const Id* __restrict__ tris,
                               const double* __restrict__ hd, const double* __restrict__ ph,
                               const Id* __restrict__ vf, const uint64_t* __restrict__ foff,
                               const uint32_t* __restrict__ vox_obj, const uint64_t* __restrict__ vb,
                               const uint64_t* __restrict__ fb, uint64_t n_voxels, double* __restrict__ out,
                               int* __restrict__ err, const uint64_t* __restrict__ act, uint64_t v_begin = 0) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t v = v_begin + blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); v < n_voxels; v += warps) {
        const uint64_t e0 = foff[v], e1 = foff[v + 1];
        // act (on-demand expansion of a compact-resident level): only the flagged voxels, packed
        uint64_t w0 = e0;
        if (act) {
            const uint64_t a0 = act[v];
            if (act[v + 1] == a0) continue;
            w0 = a0;
        }
        const uint32_t o = vox_obj[v];
        const uint64_t v_lo = vb[o], nv = vb[o + 1] - v_lo;
        const uint64_t f_lo = fb[o], nf = fb[o + 1] - f_lo;
        bool bad = false;
        for (uint64_t e = e0 + lane; e < e1; e += 32) {
            uint64_t f = __ldg(vf + e);
            if (f >= nf) { bad = true; f = 0; }
            f += f_lo;
            uint64_t t[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                t[k] = nf ? __ldg(tris + 3 * f + k) : 0;
                if (t[k] >= nv) { bad = true; t[k] = 0; }
                t[k] += v_lo;
            }
            double r[12];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double* p = verts + 3 * t[k];
                const bool ok = nv != 0;
                r[3 * k] = ok ? __ldg(p) : 0.0;
                r[3 * k + 1] = ok ? __ldg(p + 1) : 0.0;
                r[3 * k + 2] = ok ? __ldg(p + 2) : 0.0;
            }
            r[9] = nf && hd ? __ldg(hd + f) : 0.0; // hd / ph NULL: the level's paddings are all 0
            r[10] = nf && ph ? __ldg(ph + f) : 0.0;
            r[11] = 0.0;
            if (out) { // out == nullptr: validation only (compact-resident level at arrival)
                double2* d = reinterpret_cast<double2*>(out + (w0 + (e - e0)) * TJ_FACET_STRIDE);
#pragma unroll
                for (int k = 0; k < 6; ++k) d[k] = make_double2(r[2 * k], r[2 * k + 1]);
            }
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(err, 1);
    }
}

__global__ void k_voxel_owner(const uint64_t* __restrict__ voff, uint32_t n_objects, uint32_t* __restrict__ vox_obj) {
    for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < n_objects; o += gridDim.x * blockDim.x)
        for (uint64_t v = voff[o]; v < voff[o + 1]; ++v) vox_obj[v] = o;
}

} // namespace

namespace tjx {
LevelGate::~LevelGate() {
    cudaSetDevice(device);
    for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : copied)
        if (e) cudaEventDestroy(e);
    for (auto& v : pieces)
        for (auto& pe : v)
            if (pe.second) cudaEventDestroy(pe.second);
    if (expanded) cudaEventDestroy(expanded);
    if (copy) cudaStreamDestroy(copy);
    if (expand) cudaStreamDestroy(expand);
}

void expand_compact_level(const DatasetDev& d, uint32_t slot, const uint64_t* act, double* out, int num_sms,
                          cudaStream_t st) {
    if (!d.compact || !d.n_voxels) return;
    const StageLayout L = stage_layout(d.level_vertices[slot], d.level_facets[slot], d.level_entries[slot]);
    const unsigned char* base = d.cmp[slot].p;
    const uint32_t flags = d.cmp_flags[slot];
    const bool pads = flags & TJ_LEVEL_PADS;
    const double* verts = reinterpret_cast<const double*>(base + L.verts);
    const double* hd = pads && d.level_facets[slot] ? reinterpret_cast<const double*>(base + L.hd) : nullptr;
    const double* ph = pads && d.level_facets[slot] ? reinterpret_cast<const double*>(base + L.ph) : nullptr;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((d.n_voxels + 7) / 8, (uint64_t)num_sms * 16));
    count_launch();
    if (flags & TJ_LEVEL_NARROW)
        k_expand_level<<<grid, 256, 0, st>>>(verts, reinterpret_cast<const uint16_t*>(base + L.tris), hd, ph,
                                             reinterpret_cast<const uint16_t*>(base + L.vf), d.facet_offsets[slot].p,
                                             d.vox_obj.p, d.vert_base[slot].p, d.facet_base[slot].p, d.n_voxels, out,
                                             d.stream_err.p, act);
    else
        k_expand_level<<<grid, 256, 0, st>>>(verts, reinterpret_cast<const uint32_t*>(base + L.tris), hd, ph,
                                             reinterpret_cast<const uint32_t*>(base + L.vf), d.facet_offsets[slot].p,
                                             d.vox_obj.p, d.vert_base[slot].p, d.facet_base[slot].p, d.n_voxels, out,
                                             d.stream_err.p, act);
    TJ_CUDA(cudaGetLastError());
}

static std::mutex g_cm_mu;
static std::vector<std::pair<std::string, cudaEvent_t>> g_cm;
static bool copy_marks_on() {
    static const bool v = std::getenv("TRIJOIN_DEBUG_TIMELINE") != nullptr;
    return v;
}

void copy_mark(const char* what, int level, cudaStream_t st) {
    if (!copy_marks_on()) return;
    cudaEvent_t e;
    TJ_CUDA(cudaEventCreate(&e));
    TJ_CUDA(cudaEventRecord(e, st));
    std::lock_guard<std::mutex> lk(g_cm_mu);
    g_cm.emplace_back(std::string(what) + std::to_string(level) + "@" + std::to_string((uintptr_t)st % 997), e);
}

std::vector<std::pair<std::string, cudaEvent_t>> take_copy_marks() {
    std::lock_guard<std::mutex> lk(g_cm_mu);
    return std::move(g_cm);
}

double level_ready(const DatasetDev& d, int slot, cudaStream_t st) {
    if (!d.gate) return 0.0;
    LevelGate& g = *d.gate;
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_lock<std::mutex> lk(g.mu);
    g.cv.wait(lk, [&] { return g.state[slot] != LevelGate::kPending; });
    if (g.state[slot] == LevelGate::kFailed)
        throw Error(TJ_EINVAL, "join: level " + std::to_string(d.levels[slot]) + " of a streamed dataset was not delivered");
    TJ_CUDA(cudaStreamWaitEvent(st, g.ev[slot], 0));
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

bool level_pieced(const DatasetDev& d, int slot) {
    return d.gate && slot >= 0 && (size_t)slot < d.gate->pieced.size() && d.gate->pieced[slot];
}

cudaEvent_t level_piece_try(const DatasetDev& d, int slot, size_t k, uint32_t* obj_end) {
    LevelGate& g = *d.gate;
    std::lock_guard<std::mutex> lk(g.mu);
    if (g.pieces[slot].size() <= k) return nullptr; // not finished yet (or none left)
    *obj_end = g.pieces[slot][k].first;
    return g.pieces[slot][k].second;
}

cudaEvent_t level_piece(const DatasetDev& d, int slot, size_t k, uint32_t* obj_end) {
    LevelGate& g = *d.gate;
    std::unique_lock<std::mutex> lk(g.mu);
    g.cv.wait(lk, [&] { return g.pieces[slot].size() > k || g.state[slot] != LevelGate::kPending; });
    if (g.state[slot] == LevelGate::kFailed)
        throw Error(TJ_EINVAL, "join: level " + std::to_string(d.levels[slot]) + " of a streamed dataset was not delivered");
    if (g.pieces[slot].size() <= k) return nullptr; // finished: every piece delivered
    *obj_end = g.pieces[slot][k].first;
    return g.pieces[slot][k].second;
}

void stream_sync(cudaStream_t st) {
    // Spin by default: blocking-sync waits (TRIJOIN_BLOCKING_SYNC=1) free the core but were
    // measured to wake up hundreds of milliseconds late now and then on the B200 hosts.
    static const bool blocking = [] {
        const char* e = std::getenv("TRIJOIN_BLOCKING_SYNC");
        return e && *e && *e != '0';
    }();
    if (!blocking) {
        TJ_CUDA(cudaStreamSynchronize(st));
        return;
    }
    struct Events {
        cudaEvent_t ev[64] = {};
        ~Events() {
            for (cudaEvent_t e : ev)
                if (e) cudaEventDestroy(e);
        }
    };
    static thread_local Events evs;
    int dev = 0;
    TJ_CUDA(cudaGetDevice(&dev));
    cudaEvent_t& e = evs.ev[dev & 63];
    if (!e) TJ_CUDA(cudaEventCreateWithFlags(&e, cudaEventBlockingSync | cudaEventDisableTiming));
    TJ_CUDA(cudaEventRecord(e, st));
    TJ_CUDA(cudaEventSynchronize(e));
}

} // namespace tjx
// Accessors for the stage entry points (stages.cu).
struct tj_ctx_view {
    int device;
    cudaStream_t stream;
    tjx::Workspace* ws;
};
namespace tjx {
tj_ctx_view ctx_view(tj_ctx* ctx) { return {ctx->device, ctx->stream, &ctx->ws}; }
const DatasetDev& dataset_dev(const tj_dataset* ds) { return ds->d; }
int guarded_call(tj_ctx* ctx, void (*fn)(void*), void* arg) {
    return guarded(ctx, [&] { fn(arg); });
}

unsigned long long& launch_counter_ref() {
    static unsigned long long n = 0;
    return n;
}
uint64_t compact_active(Workspace& ws, const CandDevStore& cs, DevBuf<ActiveVpDev>& active, uint64_t n,
                        cudaStream_t st);
}

extern "C" {

const char* tj_last_error(const tj_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

const char* tj_global_last_error(void) {
    static thread_local std::string copy;
    std::lock_guard<std::mutex> lk(g_err_mu);
    copy = g_err;
    return copy.c_str();
}

uint64_t tj_kernel_launches(void) { return __atomic_load_n(&launch_counter_ref(), __ATOMIC_RELAXED); }

int tj_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int tj_ctx_create(int device, tj_ctx** out) {
    if (!out) return TJ_EINVAL;
    *out = nullptr;
    auto ctx = std::make_unique<tj_ctx>();
    ctx->device = device;
    const int rc = guarded(ctx.get(), [&] {
        int n = 0;
        TJ_CUDA(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) throw Error(TJ_EINVAL, "tj_ctx_create: no CUDA device " + std::to_string(device));
        TJ_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        TJ_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            throw Error(TJ_ECUDA, std::string("tj_ctx_create: built for sm_100a (B200), found ") + prop.name);
        ctx->ws.num_sms = prop.multiProcessorCount;
        TJ_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        // keep freed pool memory cached for reuse by later joins (stream-ordered allocation)
        cudaMemPool_t pool;
        TJ_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t threshold = UINT64_MAX;
        TJ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    });
    if (rc == TJ_OK) *out = ctx.release();
    return rc;
}

void tj_ctx_destroy(tj_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    {
        AllocStreamScope scope(ctx->stream);
        ctx->ws.release();
    }
    if (ctx->stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
    }
    delete ctx;
}

int tj_dataset_upload(tj_ctx* ctx, const tj_dataset_view* v, tj_dataset** out) {
    if (!ctx || !v || !out) return TJ_EINVAL;
    *out = nullptr;
    auto ds = std::make_unique<tj_dataset>();
    ds->ctx = ctx;
    const int rc = guarded(ctx, [&] {
        DatasetDev& d = ds->d;
        cudaStream_t st = ctx->stream;
        upload_objects(d, v, st);
        if (!v->facet_offsets || !v->facets) throw Error(TJ_EINVAL, "tj_dataset_upload: null facet arrays");
        for (uint32_t li = 0; li < v->n_levels; ++li) {
            const uint64_t* fo = v->facet_offsets[li];
            const uint64_t entries = fo[d.n_voxels];
            for (uint64_t x = 0; x < d.n_voxels; ++x)
                if (fo[x + 1] < fo[x]) throw Error(TJ_EINVAL, "tj_dataset_upload: facet_offsets not monotone");
            upload(d.facet_offsets[li], fo, d.n_voxels + 1, st);
            upload(d.facets[li], v->facets[li], entries * TJ_FACET_STRIDE, st);
            d.level_entries.push_back(entries);
            d.bytes += (d.n_voxels + 1) * 8 + entries * TJ_FACET_STRIDE * 8;
        }
        for (uint32_t li = 0; li < v->n_levels; ++li) derive_level(d, li, ctx->ws.num_sms, st);
        stream_sync(st);
    });
    if (rc == TJ_OK) *out = ds.release();
    return rc;
}

void tj_dataset_free(tj_dataset* ds) {
    if (!ds) return;
    cudaSetDevice(ds->ctx->device);
    if (ds->d.gate && ds->d.gate->copy) cudaStreamSynchronize(ds->d.gate->copy);
    if (ds->d.gate && ds->d.gate->expand) cudaStreamSynchronize(ds->d.gate->expand);
    AllocStreamScope scope(ds->ctx->stream);
    delete ds;
}

int tj_dataset_begin(tj_ctx* ctx, const tj_dataset_view* v, const uint64_t* const* vert_base,
                     const uint64_t* const* facet_base, tj_dataset** out) {
    return tj_dataset_begin_ex(ctx, v, vert_base, facet_base, 0u, out);
}

int tj_dataset_begin_ex(tj_ctx* ctx, const tj_dataset_view* v, const uint64_t* const* vert_base,
                        const uint64_t* const* facet_base, uint32_t flags, tj_dataset** out) {
    if (!ctx || !v || !out || !vert_base || !facet_base || (flags & ~TJ_DATASET_COMPACT)) return TJ_EINVAL;
    *out = nullptr;
    auto ds = std::make_unique<tj_dataset>();
    ds->ctx = ctx;
    const auto t_begin = std::chrono::steady_clock::now();
    const int rc = guarded(ctx, [&] {
        DatasetDev& d = ds->d;
        d.compact = (flags & TJ_DATASET_COMPACT) != 0;
        auto gate = std::make_shared<LevelGate>();
        gate->device = ctx->device;
        TJ_CUDA(cudaStreamCreateWithFlags(&gate->copy, cudaStreamNonBlocking));
        {
            int lo = 0, hi = 0;
            TJ_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            TJ_CUDA(cudaStreamCreateWithPriority(&gate->expand, cudaStreamNonBlocking, hi));
            TJ_CUDA(cudaEventCreateWithFlags(&gate->expanded, cudaEventDisableTiming));
            TJ_CUDA(cudaEventRecord(gate->expanded, gate->expand));
        }
        // everything on the dataset's own copy stream: a begin may run while a join occupies
        // the context's stream (the next R chunk of the out-of-core path)
        cudaStream_t st = gate->copy;
        AllocStreamScope scope(st);
        upload_objects(d, v, st);
        const uint32_t no = d.n_objects;
        gate->state.assign(v->n_levels, LevelGate::kPending);
        gate->ev.assign(v->n_levels, nullptr);
        gate->pieced.assign(v->n_levels, 0);
        gate->pieces.resize(v->n_levels);
        gate->copied.assign(v->n_levels, nullptr);
        gate->started.assign(v->n_levels, 0);
        gate->after.assign(v->n_levels, {nullptr, -1});
        gate->after_done.assign(v->n_levels, 0);
        d.vert_base.resize(v->n_levels);
        d.facet_base.resize(v->n_levels);
        for (uint32_t li = 0; li < v->n_levels; ++li) {
            TJ_CUDA(cudaEventCreateWithFlags(&gate->ev[li], cudaEventDisableTiming));
            TJ_CUDA(cudaEventCreateWithFlags(&gate->copied[li], cudaEventDisableTiming));
            const uint64_t* fo = v->facet_offsets ? v->facet_offsets[li] : nullptr;
            const uint64_t* vb = vert_base[li];
            const uint64_t* fb = facet_base[li];
            if (!fo || !vb || !fb) throw Error(TJ_EINVAL, "tj_dataset_begin: null level offsets");
            const uint64_t entries = fo[d.n_voxels];
            for (uint64_t x = 0; x < d.n_voxels; ++x)
                if (fo[x + 1] < fo[x]) throw Error(TJ_EINVAL, "tj_dataset_begin: facet_offsets not monotone");
            if (vb[0] != 0 || fb[0] != 0) throw Error(TJ_EINVAL, "tj_dataset_begin: object bases must start at 0");
            for (uint32_t o = 0; o < no; ++o)
                if (vb[o + 1] < vb[o] || fb[o + 1] < fb[o])
                    throw Error(TJ_EINVAL, "tj_dataset_begin: object bases not monotone");
            if (vb[no] >> 32 || fb[no] >> 32)
                throw Error(TJ_EINVAL, "tj_dataset_begin: more than 2^32 vertices or facets in one level");
            upload(d.facet_offsets[li], fo, d.n_voxels + 1, st);
            upload(d.vert_base[li], vb, no + 1ull, st);
            upload(d.facet_base[li], fb, no + 1ull, st);
            if (!d.compact) d.facets[li].alloc(std::max<uint64_t>(entries, 1) * TJ_FACET_STRIDE);
            d.level_entries.push_back(entries);
            d.level_vertices.push_back(vb[no]);
            d.level_facets.push_back(fb[no]);
            d.bytes += (d.n_voxels + 1) * 8 + (d.compact ? 0 : entries * TJ_FACET_STRIDE * 8);
        }
        d.screen.resize(v->n_levels);
        d.seg.resize(v->n_levels);
        if (d.compact) { // every level keeps its own compact storage
            d.cmp.resize(v->n_levels);
            d.cmp_flags.assign(v->n_levels, 0u);
            for (uint32_t li = 0; li < v->n_levels; ++li) {
                const uint64_t b = stage_layout(d.level_vertices[li], d.level_facets[li], d.level_entries[li]).total;
                d.cmp[li].alloc(std::max<uint64_t>(b, 256));
                d.bytes += b;
            }
        } else {
            uint64_t stage_bytes = 256;
            for (uint32_t li = 0; li < v->n_levels; ++li)
                stage_bytes = std::max(stage_bytes,
                                       stage_layout(d.level_vertices[li], d.level_facets[li], d.level_entries[li]).total);
            d.stage.alloc(stage_bytes);
            // derived screening data, reserved here (a put never allocates while a join runs)
            for (uint32_t li = 0; li < v->n_levels; ++li) {
                d.screen[li].alloc(std::max<uint64_t>(d.level_entries[li] * kScreenRecF4, 1));
                d.seg[li].alloc(std::max<uint64_t>(3 * d.n_voxels, 1));
            }
        }
        d.agg.alloc(3 * v->n_levels);
        d.vox_obj.alloc(std::max<uint64_t>(d.n_voxels, 1));
        if (no) {
            count_launch();
            k_voxel_owner<<<(no + 255) / 256, 256, 0, st>>>(d.voxel_offsets.p, no, d.vox_obj.p);
            TJ_CUDA(cudaGetLastError());
        }
        d.stream_err.alloc(1);
        TJ_CUDA(cudaMemsetAsync(d.stream_err.p, 0, sizeof(int), st));
        d.gate = std::move(gate);
        static const bool dbg = std::getenv("TRIJOIN_DEBUG_BEGIN") != nullptr;
        const auto ts = std::chrono::steady_clock::now();
        stream_sync(st);
        if (dbg)
            std::fprintf(stderr, "[begin] %u objects: %.2f ms, of which the final sync %.2f ms\n", no,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts).count());
    });
    if (rc == TJ_OK) *out = ds.release();
    return rc;
}

int tj_dataset_put_level_part(tj_dataset* ds, uint32_t slot, const tj_level_mesh_view* lv, uint64_t vert_begin,
                              uint64_t vert_end, uint64_t facet_begin, uint64_t facet_end, uint64_t entry_begin,
                              uint64_t entry_end) {
    if (!ds || !ds->d.gate || slot >= ds->d.levels.size() || !lv) return TJ_EINVAL;
    LevelGate& g = *ds->d.gate;
    tj_ctx* ctx = ds->ctx;
    const int rc = guarded(nullptr, [&] {
        TJ_CUDA(cudaSetDevice(ctx->device));
        DatasetDev& d = ds->d;
        const uint64_t nvert = d.level_vertices[slot], nfac = d.level_facets[slot], used = d.level_entries[slot];
        if (vert_begin > vert_end || vert_end > nvert || facet_begin > facet_end || facet_end > nfac ||
            entry_begin > entry_end || entry_end > used)
            throw Error(TJ_EINVAL, "tj_dataset_put_level_part: row range outside the level");
        const bool narrow = lv->tris16 != nullptr;
        if (narrow != (lv->voxel_facets16 != nullptr))
            throw Error(TJ_EINVAL, "tj_dataset_put_level: tris16 and voxel_facets16 go together");
        const void* tris = narrow ? static_cast<const void*>(lv->tris16) : lv->tris;
        const void* vfs = narrow ? static_cast<const void*>(lv->voxel_facets16) : lv->voxel_facets;
        if ((vert_end > vert_begin && !lv->vertices) || (facet_end > facet_begin && (!tris || !lv->hd != !lv->ph)) ||
            (entry_end > entry_begin && !vfs))
            throw Error(TJ_EINVAL, "tj_dataset_put_level: null level arrays");
        // into the dataset's staging area (reserved at tj_dataset_begin: no allocation here, so
        // a put never waits on the memory pool while a join runs); the copy stream orders the
        // reuse of the area across levels
        const StageLayout L = stage_layout(nvert, nfac, used);
        unsigned char* base = d.compact ? d.cmp[slot].p : d.stage.p;
        // copy order (tj_dataset_copy_after): the first put of the slot waits for the other
        // dataset's level to be fully put, then orders the copy stream after its copies
        if (!g.after_done[slot] && g.after[slot].first) {
            LevelGate& bg = *g.after[slot].first;
            const int bs = g.after[slot].second;
            bool ok = false;
            {
                std::unique_lock<std::mutex> lk(bg.mu);
                bg.cv.wait(lk, [&] { return bg.state[bs] != LevelGate::kPending; });
                ok = bg.state[bs] == LevelGate::kQueued;
            }
            if (ok) TJ_CUDA(cudaStreamWaitEvent(g.copy, bg.copied[bs], 0));
            g.after_done[slot] = 1;
        }
        // the staging area is reused level after level: a level's first copy waits for every
        // expansion queued so far (the pieces of one level fill disjoint rows)
        if (!g.started[slot]) {
            if (!d.compact) TJ_CUDA(cudaStreamWaitEvent(g.copy, g.expanded, 0));
            g.started[slot] = 1;
        }
        auto put = [&](uint64_t off, const void* src, uint64_t b0, uint64_t b1, size_t row) {
            if (b1 > b0)
                TJ_CUDA(cudaMemcpyAsync(base + off + b0 * row, static_cast<const unsigned char*>(src) + b0 * row,
                                        (b1 - b0) * row, cudaMemcpyHostToDevice, g.copy));
        };
        put(L.verts, lv->vertices, vert_begin, vert_end, 24);
        put(L.tris, tris, facet_begin, facet_end, narrow ? 6 : 12);
        if (lv->hd) {
            put(L.hd, lv->hd, facet_begin, facet_end, 8);
            put(L.ph, lv->ph, facet_begin, facet_end, 8);
        }
        put(L.vf, vfs, entry_begin, entry_end, narrow ? 2 : 4);
        TJ_CUDA(cudaEventRecord(g.copied[slot], g.copy));
        copy_mark("put", d.levels[slot], g.copy);
    });
    if (rc != TJ_OK) {
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.state[slot] = LevelGate::kFailed;
        }
        g.cv.notify_all();
        set_ctx_error(ctx, tj_global_last_error());
    }
    return rc;
}

int tj_dataset_finish_level(tj_dataset* ds, uint32_t slot, uint32_t flags) {
    if (!ds || !ds->d.gate || slot >= ds->d.levels.size()) return TJ_EINVAL;
    LevelGate& g = *ds->d.gate;
    tj_ctx* ctx = ds->ctx;
    const int rc = guarded(nullptr, [&] {
        TJ_CUDA(cudaSetDevice(ctx->device));
        AllocStreamScope scope(g.expand);
        TJ_CUDA(cudaStreamWaitEvent(g.expand, g.copied[slot], 0)); // the level's rows have landed
        DatasetDev& d = ds->d;
        const uint64_t nvert = d.level_vertices[slot], nfac = d.level_facets[slot], used = d.level_entries[slot];
        const StageLayout L = stage_layout(nvert, nfac, used);
        unsigned char* base = d.compact ? d.cmp[slot].p : d.stage.p;
        const bool pads = flags & TJ_LEVEL_PADS;
        if (d.compact) d.cmp_flags[slot] = flags;
        double* out = d.compact ? nullptr : d.facets[slot].p; // compact: validate only
        const double* verts = reinterpret_cast<const double*>(base + L.verts);
        const double* hd = pads && nfac ? reinterpret_cast<const double*>(base + L.hd) : nullptr;
        const double* ph = pads && nfac ? reinterpret_cast<const double*>(base + L.ph) : nullptr;
        const bool done = flags & TJ_LEVEL_PIECES; // expanded and derived piece by piece
        if (done && (d.compact || g.pieces[slot].empty()))
            throw Error(TJ_EINVAL, "tj_dataset_finish_level: TJ_LEVEL_PIECES without finished pieces");
        if (d.n_voxels && !done) {
            const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((d.n_voxels + 7) / 8, (uint64_t)ctx->ws.num_sms * 16));
            count_launch();
            if (flags & TJ_LEVEL_NARROW)
                k_expand_level<<<grid, 256, 0, g.expand>>>(verts, reinterpret_cast<const uint16_t*>(base + L.tris), hd, ph,
                                                          reinterpret_cast<const uint16_t*>(base + L.vf),
                                                          d.facet_offsets[slot].p, d.vox_obj.p, d.vert_base[slot].p,
                                                          d.facet_base[slot].p, d.n_voxels, out, d.stream_err.p,
                                                          nullptr);
            else
                k_expand_level<<<grid, 256, 0, g.expand>>>(verts, reinterpret_cast<const uint32_t*>(base + L.tris), hd, ph,
                                                          reinterpret_cast<const uint32_t*>(base + L.vf),
                                                          d.facet_offsets[slot].p, d.vox_obj.p, d.vert_base[slot].p,
                                                          d.facet_base[slot].p, d.n_voxels, out, d.stream_err.p,
                                                          nullptr);
            TJ_CUDA(cudaGetLastError());
        }
        copy_mark("expand", d.levels[slot], g.expand);
        if (!d.compact && !done) derive_level(d, slot, ctx->ws.num_sms, g.expand);
        copy_mark("ready", d.levels[slot], g.expand);
        TJ_CUDA(cudaEventRecord(g.ev[slot], g.expand));
        TJ_CUDA(cudaEventRecord(g.expanded, g.expand));
    });
    {
        std::lock_guard<std::mutex> lk(g.mu);
        g.state[slot] = rc == TJ_OK ? LevelGate::kQueued : LevelGate::kFailed;
    }
    g.cv.notify_all();
    if (rc != TJ_OK) set_ctx_error(ctx, tj_global_last_error());
    return rc;
}

int tj_dataset_set_pieced(tj_dataset* ds, uint32_t slot) {
    if (!ds || !ds->d.gate || slot >= ds->d.levels.size() || ds->d.compact) return TJ_EINVAL;
    std::lock_guard<std::mutex> lk(ds->d.gate->mu);
    ds->d.gate->pieced[slot] = 1;
    return TJ_OK;
}

int tj_dataset_finish_level_part(tj_dataset* ds, uint32_t slot, uint32_t obj_begin, uint32_t obj_end, uint32_t flags) {
    if (!ds || !ds->d.gate || slot >= ds->d.levels.size()) return TJ_EINVAL;
    LevelGate& g = *ds->d.gate;
    tj_ctx* ctx = ds->ctx;
    cudaEvent_t ev = nullptr;
    const int rc = guarded(nullptr, [&] {
        TJ_CUDA(cudaSetDevice(ctx->device));
        AllocStreamScope scope(g.expand);
        DatasetDev& d = ds->d;
        if (d.compact || !g.pieced[slot]) throw Error(TJ_EINVAL, "tj_dataset_finish_level_part: level not set pieced");
        const uint32_t prev = g.pieces[slot].empty() ? 0u : g.pieces[slot].back().first;
        if (obj_begin != prev || obj_end < obj_begin || obj_end > d.n_objects)
            throw Error(TJ_EINVAL, "tj_dataset_finish_level_part: pieces must cover the objects in order");
        const uint64_t nvert = d.level_vertices[slot], nfac = d.level_facets[slot], used = d.level_entries[slot];
        const StageLayout L = stage_layout(nvert, nfac, used);
        unsigned char* base = d.stage.p;
        const bool pads = flags & TJ_LEVEL_PADS;
        const double* verts = reinterpret_cast<const double*>(base + L.verts);
        const double* hd = pads && nfac ? reinterpret_cast<const double*>(base + L.hd) : nullptr;
        const double* ph = pads && nfac ? reinterpret_cast<const double*>(base + L.ph) : nullptr;
        const uint64_t v0 = d.voxel_offsets_h[obj_begin], v1 = d.voxel_offsets_h[obj_end];
        TJ_CUDA(cudaStreamWaitEvent(g.expand, g.copied[slot], 0)); // the piece's rows have landed
        if (v1 > v0) {
            const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((v1 - v0 + 7) / 8, (uint64_t)ctx->ws.num_sms * 16));
            count_launch();
            if (flags & TJ_LEVEL_NARROW)
                k_expand_level<<<grid, 256, 0, g.expand>>>(verts, reinterpret_cast<const uint16_t*>(base + L.tris), hd, ph,
                                                          reinterpret_cast<const uint16_t*>(base + L.vf),
                                                          d.facet_offsets[slot].p, d.vox_obj.p, d.vert_base[slot].p,
                                                          d.facet_base[slot].p, v1, d.facets[slot].p, d.stream_err.p,
                                                          nullptr, v0);
            else
                k_expand_level<<<grid, 256, 0, g.expand>>>(verts, reinterpret_cast<const uint32_t*>(base + L.tris), hd, ph,
                                                          reinterpret_cast<const uint32_t*>(base + L.vf),
                                                          d.facet_offsets[slot].p, d.vox_obj.p, d.vert_base[slot].p,
                                                          d.facet_base[slot].p, v1, d.facets[slot].p, d.stream_err.p,
                                                          nullptr, v0);
            TJ_CUDA(cudaGetLastError());
        }
        derive_level_range(d, slot, v0, v1, g.pieces[slot].empty(), ctx->ws.num_sms, g.expand);
        TJ_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        TJ_CUDA(cudaEventRecord(ev, g.expand));
        TJ_CUDA(cudaEventRecord(g.expanded, g.expand));
    });
    {
        std::lock_guard<std::mutex> lk(g.mu);
        if (rc == TJ_OK)
            g.pieces[slot].emplace_back(obj_end, ev);
        else
            g.state[slot] = LevelGate::kFailed;
    }
    g.cv.notify_all();
    if (rc != TJ_OK) set_ctx_error(ctx, tj_global_last_error());
    return rc;
}

int tj_dataset_copy_after(tj_dataset* ds, uint32_t slot, tj_dataset* before, uint32_t before_slot) {
    if (!ds || !ds->d.gate || slot >= ds->d.levels.size() || !before || before == ds || !before->d.gate ||
        before_slot >= before->d.levels.size() || before->ctx->device != ds->ctx->device)
        return TJ_EINVAL;
    LevelGate& g = *ds->d.gate;
    std::lock_guard<std::mutex> lk(g.mu);
    if (g.state[slot] != LevelGate::kPending || g.after_done[slot]) return TJ_EINVAL; // already being put
    g.after[slot] = {before->d.gate.get(), (int)before_slot};
    return TJ_OK;
}

int tj_dataset_level_wait(tj_dataset* ds, uint32_t slot) {
    if (!ds || !ds->d.gate || slot >= ds->d.levels.size()) return TJ_EINVAL;
    LevelGate& g = *ds->d.gate;
    return guarded(nullptr, [&] {
        {
            std::unique_lock<std::mutex> lk(g.mu);
            g.cv.wait(lk, [&] { return g.state[slot] != LevelGate::kPending; });
            if (g.state[slot] == LevelGate::kFailed) throw Error(TJ_EINVAL, "tj_dataset_level_wait: level failed");
        }
        TJ_CUDA(cudaSetDevice(ds->ctx->device));
        TJ_CUDA(cudaEventSynchronize(g.ev[slot]));
    });
}

int tj_dataset_put_level(tj_dataset* ds, uint32_t slot, const tj_level_mesh_view* lv) {
    if (!ds || !ds->d.gate || slot >= ds->d.levels.size()) return TJ_EINVAL;
    if (!lv) {
        LevelGate& g = *ds->d.gate;
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.state[slot] = LevelGate::kFailed;
        }
        g.cv.notify_all();
        return TJ_OK;
    }
    const DatasetDev& d = ds->d;
    const int rc = tj_dataset_put_level_part(ds, slot, lv, 0, d.level_vertices[slot], 0, d.level_facets[slot], 0,
                                             d.level_entries[slot]);
    if (rc != TJ_OK) return rc;
    return tj_dataset_finish_level(ds, slot, (lv->hd ? TJ_LEVEL_PADS : 0u) | (lv->tris16 ? TJ_LEVEL_NARROW : 0u));
}

int tj_dataset_sync(tj_dataset* ds) {
    if (!ds) return TJ_EINVAL;
    if (!ds->d.gate) return TJ_OK;
    return guarded(nullptr, [&] {
        TJ_CUDA(cudaSetDevice(ds->ctx->device));
        TJ_CUDA(cudaStreamSynchronize(ds->d.gate->copy));
        TJ_CUDA(cudaStreamSynchronize(ds->d.gate->expand));
    });
}

uint64_t tj_dataset_device_bytes(const tj_dataset* ds) { return ds ? ds->d.bytes : 0; }

void tj_join_result_free(tj_join_result* r) {
    if (!r) return;
    std::free(r->pair_r);
    std::free(r->pair_s);
    std::free(r->lb);
    std::free(r->ub);
    std::free(r->status);
    std::free(r->decided_at);
    std::free(r->r2op_offsets);
    std::free(r->num_confirmed);
    std::memset(r, 0, sizeof(*r));
}

int tj_join(tj_ctx* ctx, const tj_dataset* Rh, const tj_dataset* Sh, const tj_join_spec* spec, const tj_trace* trace,
            tj_join_result* out) {
    if (!ctx || !Rh || !Sh || !spec || !out) return TJ_EINVAL;
    std::memset(out, 0, sizeof(*out));
    return guarded(ctx, [&] {
        using Clock = std::chrono::steady_clock;
        const auto t_total = Clock::now();
        const tj_join_spec& sp = *spec;
        validate_spec(sp);
        const DatasetDev& R = Rh->d;
        const DatasetDev& S = Sh->d;
        cudaStream_t st = ctx->stream;
        Workspace& ws = ctx->ws;
        const bool knn = sp.type == TJ_KNN;
        const double tau = sp.type == TJ_INTERSECT ? 0.0 : sp.tau;

        TraceSink sink;
        TraceSink* tsink = nullptr;
        if (trace && (trace->on_interval || trace->on_vp_pruned)) {
            sink.user = trace->user;
            sink.on_interval = trace->on_interval;
            sink.on_vp_pruned = trace->on_vp_pruned;
            tsink = &sink;
        }

        DevBuf<DevError> err(1);
        DevError init{0, 0xffffffffu, 0.0, 0.0, 0};
        TJ_CUDA(cudaMemcpyAsync(err.p, &init, sizeof(init), cudaMemcpyHostToDevice, st));

        // ---- MBB filter ----
        auto t0 = Clock::now();
        SortedS sorted;
        mbb_prepare_s(ws, S, sorted, st);
        MbbArgs ma{};
        ma.r_mbb = R.mbb.p;
        ma.r_anchor = R.anchor.p;
        ma.s_mbb = S.mbb.p;
        ma.s_anchor = S.anchor.p;
        ma.s_sorted_mbb = sorted.mbb.p;
        ma.s_sorted_yz = sorted.yz.p;
        ma.s_order = sorted.order.p;
        ma.nr = R.n_objects;
        ma.ns = S.n_objects;
        ma.max_ext = sorted.max_ext;
        ma.shard_index = sp.shard_index;
        ma.shard_count = sp.shard_count;
        ma.shard_block = sp.shard_block ? sp.shard_block : 1024;
        DevBuf<double> u_k;
        if (knn) {
            knn_kth_anchor(ws, ma, sp.k, u_k, st);
            ma.tau_per_r = u_k.p;
            ma.tau = 0.0;
            ma.confirm_at_mbb = 0;
        } else {
            ma.tau = tau;
            ma.tau_per_r = nullptr;
            ma.confirm_at_mbb = 1;
        }
        CandDevStore cs;
        mbb_candidates(ws, ma, cs, st);
        if (tsink && tsink->on_interval) tsink->emit_flagged(cs, {}, TJ_STAGE_MBB, st);
        if (knn) {
            knn_fixpoint(ws, cs, sp.k, TJ_STAGE_MBB, err.p, st);
            check_dev_error(err.p, st);
        }
        out->mbb_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();

        // ---- voxel-pair filter ----
        t0 = Clock::now();
        VoxelArgs va{};
        va.n_cands = cs.n;
        va.r_voff = R.voxel_offsets.p;
        va.s_voff = S.voxel_offsets.p;
        va.r_vbox = R.voxel_box.p;
        va.s_vbox = S.voxel_box.p;
        va.r_vanc = R.voxel_anchor.p;
        va.s_vanc = S.voxel_anchor.p;
        va.prune = knn ? 0 : 1;
        va.tau = tau;
        va.err = err.p;
        DevBuf<ActiveVpDev>& active = ctx->ws.active;
        std::vector<PrunedVp> pruned;
        std::vector<uint8_t> touched;
        const VoxelOut vo = voxel_filter(ws, va, cs, active, tsink != nullptr, &pruned, &touched, st);
        check_dev_error(err.p, st);
        out->vp_generated = vo.vp_generated;
        out->vp_pruned = vo.vp_pruned;
        if (tsink) {
            if (tsink->on_interval) tsink->emit_flagged(cs, touched, TJ_STAGE_VOXEL, st);
            if (tsink->on_vp_pruned && !pruned.empty()) {
                std::vector<double> ub(cs.n);
                TJ_CUDA(cudaMemcpyAsync(ub.data(), cs.ub.p, cs.n * 8, cudaMemcpyDeviceToHost, st));
                stream_sync(st);
                for (const PrunedVp& p : pruned) tsink->on_vp_pruned(tsink->user, p.op, p.vr, p.vs, p.lb, ub[p.op]);
            }
        }
        if (knn) {
            knn_fixpoint(ws, cs, sp.k, TJ_STAGE_VOXEL, err.p, st);
            check_dev_error(err.p, st);
        }
        out->voxel_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();

        // ---- multi-LOD refinement ----
        t0 = Clock::now();
        check_levels(R, sp);
        check_levels(S, sp);
        uint64_t n_active = compact_active(ws, cs, active, vo.survivors, st);
        const bool decision = sp.type == TJ_INTERSECT && !tsink && !(sp.flags & TJ_FLAG_EXACT_INTERVALS);
        out->decision_mode = decision ? 1 : 0;
        RefineLoopOut ro = refine_loop_dev(ws, R, S, cs, active, n_active, sp, knn, tau, decision, err.p, tsink, st);
        if (knn) {
            knn_finalize_dev(ws, cs, sp.k, st);
        } else {
            std::vector<uint8_t> stv(cs.n);
            if (cs.n) TJ_CUDA(cudaMemcpyAsync(stv.data(), cs.status.p, cs.n, cudaMemcpyDeviceToHost, st));
            stream_sync(st);
            for (uint8_t s : stv)
                if (s == TJ_UNDECIDED)
                    throw Error(TJ_EENGINE, "refine_loop: candidates left undecided after the exact level");
        }
        out->refine_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        out->n_levels_run = (uint32_t)ro.levels.size();
        for (size_t i = 0; i < ro.levels.size() && i < TJ_MAX_LODS; ++i) {
            out->level[i] = ro.levels[i].level;
            out->level_vps[i] = ro.levels[i].vps;
            out->level_facet_pairs[i] = ro.levels[i].facet_pairs;
            out->level_pairs_evaluated[i] = ro.levels[i].evaluated;
            out->level_pairs_tested[i] = ro.levels[i].tested;
            out->level_pairs_screened[i] = ro.levels[i].screened;
            out->level_pairs_verified[i] = ro.levels[i].verified;
            out->level_vps_skipped[i] = ro.levels[i].vps_skipped;
            out->level_facets_dropped[i] = ro.levels[i].facets_dropped;
            out->level_ms[i] = ro.levels[i].ms;
            out->level_kernel_ms[i] = ro.levels[i].kernel_ms;
            out->level_screen_ms[i] = ro.levels[i].screen_ms;
            out->level_wait_ms[i] = ro.levels[i].wait_ms;
        }
        out->refine_chunks = ro.chunks;
        out->queue_reruns = ro.queue_reruns;
        out->mat_chunks = ro.mat_chunks;

        if (sp.flags & TJ_FLAG_EXACT_RECOMPUTE) exact_recompute_dev(ws, R, S, cs, st);

        // streamed datasets: the device-side validation of every level the join asked for
        // (levels the refinement never reached included: the join stream first waits on each
        // level's arrival event, so the flag does not depend on how early refinement ended)
        for (const DatasetDev* D : {&R, &S}) {
            if (!D->gate) continue;
            for (uint32_t li = 0; li < sp.n_lods; ++li)
                for (size_t slot = 0; slot < D->levels.size(); ++slot)
                    if (D->levels[slot] == (int32_t)sp.lods[li]) level_ready(*D, (int)slot, st);
            int bad = 0;
            TJ_CUDA(cudaMemcpyAsync(&bad, D->stream_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
            stream_sync(st);
            if (bad) throw Error(TJ_EINVAL, "trijoin: voxel facet id or facet vertex id out of range");
        }

        // ---- results ----
        out->n_cands = cs.n;
        out->n_queries = R.n_objects;
        out->pair_r = host_copy(cs.pair_r, cs.n, st);
        out->pair_s = host_copy(cs.pair_s, cs.n, st);
        out->lb = host_copy(cs.lb, cs.n, st);
        out->ub = host_copy(cs.ub, cs.n, st);
        out->status = host_copy(cs.status, cs.n, st);
        out->decided_at = host_copy(cs.decided_at, cs.n, st);
        out->r2op_offsets = host_copy(cs.r2op, (uint64_t)R.n_objects + 1, st);
        out->num_confirmed = host_copy(cs.num_confirmed, R.n_objects, st);
        stream_sync(st);
        out->total_ms = std::chrono::duration<double, std::milli>(Clock::now() - t_total).count();
    });
}

int tj_refine_batch(tj_ctx* ctx, uint64_t n_tris, const double* tris, const double* hd, const double* ph,
                    uint64_t n_descs, const uint64_t* r_off, const uint64_t* s_off, const uint32_t* r_len,
                    const uint32_t* s_len, uint32_t flags, double* vp_lb, double* vp_ub) {
    if (!ctx) return TJ_EINVAL;
    return guarded(ctx, [&] {
        cudaStream_t st = ctx->stream;
        if (n_descs == 0) return;
        for (uint64_t d = 0; d < n_descs; ++d)
            if ((r_len[d] && r_off[d] + r_len[d] > n_tris) || (s_len[d] && s_off[d] + s_len[d] > n_tris))
                throw Error(TJ_EINVAL, "tj_refine_batch: descriptor out of range");
        std::vector<double> rec(std::max<uint64_t>(n_tris, 1) * TJ_FACET_STRIDE, 0.0);
        for (uint64_t i = 0; i < n_tris; ++i) {
            std::memcpy(&rec[i * TJ_FACET_STRIDE], tris + 9 * i, 9 * sizeof(double));
            rec[i * TJ_FACET_STRIDE + 9] = hd[i];
            rec[i * TJ_FACET_STRIDE + 10] = ph[i];
        }
        DevBuf<double> f;
        upload(f, rec.data(), rec.size(), st);
        DevBuf<uint64_t> ro, so;
        DevBuf<uint32_t> rl, sl;
        upload(ro, r_off, n_descs, st);
        upload(so, s_off, n_descs, st);
        upload(rl, r_len, n_descs, st);
        upload(sl, s_len, n_descs, st);
        // every descriptor is its own op: per-voxel-pair minima, exact (refine_kernel.cuh)
        DevBuf<unsigned long long> lbb(n_descs), ubb(n_descs), work(1), counters(kNumCounters);
        std::vector<unsigned long long> inf(n_descs, 0x7ff0000000000000ull);
        RefineSource src{};
        src.r_off = ro.p;
        src.s_off = so.p;
        src.r_len = rl.p;
        src.s_len = sl.p;
        src.r_facets = f.p;
        src.s_facets = f.p;
        DevBuf<float4> scr(std::max<uint64_t>(n_tris, 1) * kScreenRecF4);
        refine_prep(f.p, n_tris, scr.p, nullptr, ctx->ws.num_sms, st);
        src.r_box = src.s_box = scr.p;
        src.r_geo = src.s_geo = scr.p + 3 * n_tris;
        const int cull = (flags & TJ_FLAG_NO_CULL) ? 0 : 1;
        RefineQueueStore queue;
        for (;;) { // re-run with a larger exact-evaluation queue if it overflowed
            TJ_CUDA(cudaMemcpyAsync(lbb.p, inf.data(), n_descs * 8, cudaMemcpyHostToDevice, st));
            TJ_CUDA(cudaMemcpyAsync(ubb.p, inf.data(), n_descs * 8, cudaMemcpyHostToDevice, st));
            TJ_CUDA(cudaMemsetAsync(counters.p, 0, kNumCounters * 8, st));
            queue.reset(st);
            if (cull)
                refine_pass(src, 0, n_descs, true, lbb.p, ubb.p, cull, queue, work.p, counters.p, ctx->ws.num_sms, st);
            refine_pass(src, 0, n_descs, false, lbb.p, ubb.p, cull, queue, work.p, counters.p, ctx->ws.num_sms, st);
            if (!queue.grow_if_overflowed(st)) break;
        }
        TJ_CUDA(cudaMemcpyAsync(vp_lb, lbb.p, n_descs * 8, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaMemcpyAsync(vp_ub, ubb.p, n_descs * 8, cudaMemcpyDeviceToHost, st));
        stream_sync(st);
    });
}

} // extern "C"
