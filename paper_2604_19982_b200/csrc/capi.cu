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
        if (ctx) ctx->last_error = e.what();
        set_global_error(e.what());
        return e.code;
    } catch (const std::bad_alloc& e) {
        if (ctx) ctx->last_error = "host allocation failed";
        set_global_error("host allocation failed");
        return TJ_ENOMEM;
    } catch (const std::exception& e) {
        if (ctx) ctx->last_error = e.what();
        set_global_error(e.what());
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
    TJ_CUDA(cudaStreamSynchronize(st));
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

} // namespace

namespace tjx {
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
        if (v->n_levels == 0 || v->n_levels > TJ_MAX_LODS)
            throw Error(TJ_EINVAL, "tj_dataset_upload: n_levels must be in [1, 16]");
        const uint32_t no = v->n_objects;
        if (no && (!v->mbb || !v->anchor || !v->voxel_offsets))
            throw Error(TJ_EINVAL, "tj_dataset_upload: null object arrays");
        d.n_objects = no;
        d.levels.assign(v->levels, v->levels + v->n_levels);
        d.voxel_offsets_h.assign(v->voxel_offsets, v->voxel_offsets + no + 1);
        d.n_voxels = d.voxel_offsets_h.back();
        for (uint32_t o = 0; o < no; ++o)
            if (d.voxel_offsets_h[o + 1] < d.voxel_offsets_h[o])
                throw Error(TJ_EINVAL, "tj_dataset_upload: voxel_offsets not monotone");
        upload(d.mbb, v->mbb, 6ull * no, st);
        upload(d.anchor, v->anchor, 3ull * no, st);
        upload(d.voxel_offsets, v->voxel_offsets, no + 1ull, st);
        upload(d.voxel_box, v->voxel_box, 6ull * d.n_voxels, st);
        upload(d.voxel_anchor, v->voxel_anchor, 3ull * d.n_voxels, st);
        d.facet_offsets.resize(v->n_levels);
        d.facets.resize(v->n_levels);
        d.bytes = (9ull * no + 9ull * d.n_voxels) * 8 + (no + 1ull) * 8;
        for (uint32_t li = 0; li < v->n_levels; ++li) {
            const uint64_t* fo = v->facet_offsets[li];
            const uint64_t entries = fo[d.n_voxels];
            for (uint64_t x = 0; x < d.n_voxels; ++x)
                if (fo[x + 1] < fo[x]) throw Error(TJ_EINVAL, "tj_dataset_upload: facet_offsets not monotone");
            upload(d.facet_offsets[li], fo, d.n_voxels + 1, st);
            upload(d.facets[li], v->facets[li], entries * TJ_FACET_STRIDE, st);
            d.bytes += (d.n_voxels + 1) * 8 + entries * TJ_FACET_STRIDE * 8;
        }
        TJ_CUDA(cudaStreamSynchronize(st));
    });
    if (rc == TJ_OK) *out = ds.release();
    return rc;
}

void tj_dataset_free(tj_dataset* ds) {
    if (!ds) return;
    cudaSetDevice(ds->ctx->device);
    AllocStreamScope scope(ds->ctx->stream);
    delete ds;
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
        DevBuf<ActiveVpDev> active;
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
                TJ_CUDA(cudaStreamSynchronize(st));
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
        RefineLoopOut ro = refine_loop_dev(ws, R, S, cs, active, n_active, sp, knn, tau, err.p, tsink, st);
        if (knn) {
            knn_finalize_dev(ws, cs, sp.k, st);
        } else {
            std::vector<uint8_t> stv(cs.n);
            if (cs.n) TJ_CUDA(cudaMemcpyAsync(stv.data(), cs.status.p, cs.n, cudaMemcpyDeviceToHost, st));
            TJ_CUDA(cudaStreamSynchronize(st));
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
        }
        out->refine_chunks = ro.chunks;

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
        TJ_CUDA(cudaStreamSynchronize(st));
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
        TJ_CUDA(cudaMemcpyAsync(lbb.p, inf.data(), n_descs * 8, cudaMemcpyHostToDevice, st));
        TJ_CUDA(cudaMemcpyAsync(ubb.p, inf.data(), n_descs * 8, cudaMemcpyHostToDevice, st));
        TJ_CUDA(cudaMemsetAsync(counters.p, 0, kNumCounters * 8, st));
        RefineSource src{};
        src.r_off = ro.p;
        src.s_off = so.p;
        src.r_len = rl.p;
        src.s_len = sl.p;
        src.r_facets = f.p;
        src.s_facets = f.p;
        DevBuf<float4> scr(std::max<uint64_t>(n_tris, 1) * 7);
        refine_prep(f.p, n_tris, scr.p, ctx->ws.num_sms, st);
        src.r_box = src.s_box = scr.p;
        src.r_geo = src.s_geo = scr.p + 3 * n_tris;
        const int cull = (flags & TJ_FLAG_NO_CULL) ? 0 : 1;
        RefineQueueStore queue;
        if (cull) refine_pass(src, 0, n_descs, true, lbb.p, ubb.p, cull, queue, work.p, counters.p, ctx->ws.num_sms, st);
        refine_pass(src, 0, n_descs, false, lbb.p, ubb.p, cull, queue, work.p, counters.p, ctx->ws.num_sms, st);
        TJ_CUDA(cudaMemcpyAsync(vp_lb, lbb.p, n_descs * 8, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaMemcpyAsync(vp_ub, ubb.p, n_descs * 8, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaStreamSynchronize(st));
    });
}

int tj_tri_tri_batch(tj_ctx* ctx, uint64_t n, const double* a9, const double* b9, double* out) {
    if (!ctx) return TJ_EINVAL;
    return guarded(ctx, [&] {
        cudaStream_t st = ctx->stream;
        if (!n) return;
        DevBuf<double> a, b, o(n);
        upload(a, a9, 9 * n, st);
        upload(b, b9, 9 * n, st);
        launch_tri_tri_batch(n, a.p, b.p, o.p, st);
        TJ_CUDA(cudaMemcpyAsync(out, o.p, n * 8, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaStreamSynchronize(st));
    });
}

int tj_mindist_batch(tj_ctx* ctx, uint64_t n, const double* a6, const double* b6, double* out) {
    if (!ctx) return TJ_EINVAL;
    return guarded(ctx, [&] {
        cudaStream_t st = ctx->stream;
        if (!n) return;
        DevBuf<double> a, b, o(n);
        upload(a, a6, 6 * n, st);
        upload(b, b6, 6 * n, st);
        launch_mindist_batch(n, a.p, b.p, o.p, st);
        TJ_CUDA(cudaMemcpyAsync(out, o.p, n * 8, cudaMemcpyDeviceToHost, st));
        TJ_CUDA(cudaStreamSynchronize(st));
    });
}

} // extern "C"
