// Stage-level C-ABI (include/tj_capi.h "stage entry points"): the reference's stage functions
// that its own tests and tools call directly (proj/include/trijoin/filter.hpp:62-117,
// refine.hpp:57-87, knn.hpp:19-54), each run on the device over a caller-owned host
// candidate set. tj_join chains the same device stages without the host round trips.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "filter.cuh"
#include "geom_exact.cuh"
#include "scan.cuh"
#include "trace_sink.h"

// Shared with capi.cu (same translation-unit-independent definitions).
struct tj_ctx_view {
    int device;
    cudaStream_t stream;
    tjx::Workspace* ws;
};

namespace tjx {
// capi.cu
tj_ctx_view ctx_view(tj_ctx* ctx);
const DatasetDev& dataset_dev(const tj_dataset* ds);
int guarded_call(tj_ctx* ctx, void (*fn)(void*), void* arg);
uint64_t compact_active(Workspace& ws, const CandDevStore& cs, DevBuf<ActiveVpDev>& active, uint64_t n,
                        cudaStream_t st);
}

using namespace tjx;

namespace {

template <class T>
void to_dev(DevBuf<T>& dst, const T* src, uint64_t n, cudaStream_t st) {
    dst.alloc(std::max<uint64_t>(n, 1));
    if (n) TJ_CUDA(cudaMemcpyAsync(dst.p, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
}
template <class T>
void to_host(T* dst, const DevBuf<T>& src, uint64_t n, cudaStream_t st) {
    if (n) TJ_CUDA(cudaMemcpyAsync(dst, src.p, n * sizeof(T), cudaMemcpyDeviceToHost, st));
}
template <class T>
T* host_alloc(uint64_t n) {
    T* p = static_cast<T*>(std::malloc(std::max<uint64_t>(n, 1) * sizeof(T)));
    if (!p) throw std::bad_alloc();
    return p;
}

void check_cands(const tj_cand_view* c) {
    if (!c) throw Error(TJ_EINVAL, "stage: null candidate set");
    if (c->n_cands && (!c->pair_r || !c->pair_s || !c->lb || !c->ub || !c->status || !c->decided_at))
        throw Error(TJ_EINVAL, "stage: null candidate arrays");
    if (!c->r2op_offsets || (c->n_queries && !c->num_confirmed)) throw Error(TJ_EINVAL, "stage: null query arrays");
    if (c->r2op_offsets[c->n_queries] != c->n_cands)
        throw Error(TJ_EINVAL, "stage: r2op_offsets do not cover the candidate set");
}

void upload_cands(const tj_cand_view* c, CandDevStore& cs, cudaStream_t st) {
    cs.resize(c->n_cands, c->n_queries);
    to_dev(cs.pair_r, c->pair_r, c->n_cands, st);
    to_dev(cs.pair_s, c->pair_s, c->n_cands, st);
    to_dev(cs.lb, c->lb, c->n_cands, st);
    to_dev(cs.ub, c->ub, c->n_cands, st);
    to_dev(cs.status, c->status, c->n_cands, st);
    to_dev(cs.decided_at, c->decided_at, c->n_cands, st);
    to_dev(cs.r2op, c->r2op_offsets, (uint64_t)c->n_queries + 1, st);
    to_dev(cs.num_confirmed, c->num_confirmed, c->n_queries, st);
}

void download_cands(tj_cand_view* c, CandDevStore& cs, cudaStream_t st) {
    to_host(c->lb, cs.lb, c->n_cands, st);
    to_host(c->ub, cs.ub, c->n_cands, st);
    to_host(c->status, cs.status, c->n_cands, st);
    to_host(c->decided_at, cs.decided_at, c->n_cands, st);
    to_host(c->num_confirmed, cs.num_confirmed, c->n_queries, st);
    stream_sync(st);
}

void validate_pairs(const tj_cand_view* c, const DatasetDev& R, const DatasetDev& S) {
    for (uint64_t op = 0; op < c->n_cands; ++op)
        if (c->pair_r[op] >= R.n_objects || c->pair_s[op] >= S.n_objects)
            throw Error(TJ_EINVAL, "stage: candidate pair out of range");
}

TraceSink make_sink(const tj_trace* t) {
    TraceSink s;
    if (t) {
        s.user = t->user;
        s.on_interval = t->on_interval;
        s.on_vp_pruned = t->on_vp_pruned;
    }
    return s;
}

void check_err(DevError* err, cudaStream_t st) {
    DevError h;
    TJ_CUDA(cudaMemcpyAsync(&h, err, sizeof(DevError), cudaMemcpyDeviceToHost, st));
    stream_sync(st);
    if (h.code == 0) return;
    if (h.kind == 1) throw Error(TJ_EENGINE, "knn_apply_deltas: confirmed count exceeds k");
    throw Error(TJ_EENGINE, "bound crossing: lb " + std::to_string(h.lb) + " > ub " + std::to_string(h.ub));
}

struct ErrBuf {
    DevBuf<DevError> e;
    explicit ErrBuf(cudaStream_t st) : e(1) {
        const DevError init{0, 0xffffffffu, 0.0, 0.0, 0};
        TJ_CUDA(cudaMemcpyAsync(e.p, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    }
};

// ---- voxel_pair_bounds: materialised per-voxel-pair bounds of one filter chunk ----
// Thread per flattened voxel pair t of the chunk: (i, j) = decode_pair(t - vp_offsets[ci],
// n_s) (proj/include/trijoin/parcore.hpp:23-25); vp_lb = mindist_aabb of the voxel boxes,
// vp_ub = distance of the voxel anchors (src/filter.cpp:199-239); op minima by 64-bit
// atomicMin on the IEEE bits (non-negative doubles: exact and order-free).
__global__ void k_vox_bounds(const uint32_t* __restrict__ ops, const uint64_t* __restrict__ vp_off, uint64_t n_ops,
                             const uint32_t* __restrict__ pair_r, const uint32_t* __restrict__ pair_s,
                             const uint64_t* __restrict__ r_voff, const uint64_t* __restrict__ s_voff,
                             const double* __restrict__ r_vbox, const double* __restrict__ s_vbox,
                             const double* __restrict__ r_vanc, const double* __restrict__ s_vanc,
                             double* __restrict__ vp_lb, double* __restrict__ vp_ub, unsigned long long* op_lb,
                             unsigned long long* op_ub) {
    const uint64_t total = vp_off[n_ops];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = n_ops; // largest ci with vp_off[ci] <= t
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (vp_off[mid] <= t) lo = mid; else hi = mid;
        }
        const uint64_t ci = lo;
        const uint32_t op = ops[ci];
        const uint32_t r = pair_r[op], s = pair_s[op];
        const uint64_t vr0 = r_voff[r], vs0 = s_voff[s], ns = s_voff[s + 1] - vs0;
        const uint64_t u = t - vp_off[ci];
        const uint64_t i = u / ns, j = u - i * ns;
        const double lb = mindist_box(r_vbox + 6 * (vr0 + i), s_vbox + 6 * (vs0 + j));
        const double ub = point_dist(r_vanc + 3 * (vr0 + i), s_vanc + 3 * (vs0 + j));
        vp_lb[t] = lb;
        vp_ub[t] = ub;
        atomicMin(op_lb + ci, (unsigned long long)__double_as_longlong(lb));
        atomicMin(op_ub + ci, (unsigned long long)__double_as_longlong(ub));
    }
}

__global__ void k_fill(unsigned long long* p, uint64_t n, unsigned long long v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

struct IndexEmit {
    uint64_t* out;
    __device__ __forceinline__ void operator()(uint64_t i, uint64_t k) const { out[k] = i; }
};

// ---- voxel_pair_compact: stable survivors (op, i, j) of one chunk ----
struct Survives {
    const uint32_t* ops;
    const uint64_t* vp_off;
    uint64_t n_ops;
    const uint8_t* status;
    const double* ub;
    const double* vp_lb;
    __device__ __forceinline__ uint64_t slot(uint64_t t) const {
        uint64_t lo = 0, hi = n_ops;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (vp_off[mid] <= t) lo = mid; else hi = mid;
        }
        return lo;
    }
    __device__ __forceinline__ bool operator()(uint64_t t) const {
        const uint32_t op = ops[slot(t)];
        return status[op] == TJ_UNDECIDED && vp_lb[t] <= ub[op];
    }
};

__global__ void k_decode_survivors(Survives sv, const uint64_t* __restrict__ ts, uint64_t n,
                                   const uint32_t* __restrict__ pair_s, const uint64_t* __restrict__ s_voff,
                                   uint32_t* __restrict__ out_op, uint32_t* __restrict__ out_i,
                                   uint32_t* __restrict__ out_j) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = ts[k];
        const uint64_t ci = sv.slot(t);
        const uint32_t op = sv.ops[ci];
        const uint32_t s = pair_s[op];
        const uint64_t ns = s_voff[s + 1] - s_voff[s];
        const uint64_t u = t - sv.vp_off[ci];
        out_op[k] = op;
        out_i[k] = (uint32_t)(u / ns);
        out_j[k] = (uint32_t)(u - (u / ns) * ns);
    }
}

// ---- refine_loop input: active voxel pairs of the undecided ops, global voxel ids ----
__global__ void k_active_from_list(const uint64_t* __restrict__ op_off, uint64_t n_ops, const uint32_t* __restrict__ vr,
                                   const uint32_t* __restrict__ vs, const uint32_t* __restrict__ pair_r,
                                   const uint32_t* __restrict__ pair_s, const uint64_t* __restrict__ r_voff,
                                   const uint64_t* __restrict__ s_voff, ActiveVpDev* __restrict__ out, int* bad) {
    const uint64_t total = op_off[n_ops];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = n_ops;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (op_off[mid] <= t) lo = mid; else hi = mid;
        }
        const uint32_t op = (uint32_t)lo;
        const uint32_t r = pair_r[op], s = pair_s[op];
        const uint64_t nr = r_voff[r + 1] - r_voff[r], ns = s_voff[s + 1] - s_voff[s];
        uint32_t i = vr[t], j = vs[t];
        if (i >= nr || j >= ns) {
            atomicExch(bad, 1);
            i = j = 0;
        }
        out[t] = {op, (uint32_t)(r_voff[r] + i), (uint32_t)(s_voff[s] + j)};
    }
}

inline int grid_of(uint64_t n, int num_sms) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 32));
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

extern "C" {

void tj_vp_list_free(tj_vp_list* l) {
    if (!l) return;
    std::free(l->op_offsets);
    std::free(l->op);
    std::free(l->vr);
    std::free(l->vs);
    std::memset(l, 0, sizeof(*l));
}

int tj_mbb_filter(tj_ctx* ctx, const tj_dataset* Rh, const tj_dataset* Sh, int32_t type, double tau, uint32_t k,
                  const tj_trace* trace, tj_join_result* out) {
    if (!ctx || !Rh || !Sh || !out) return TJ_EINVAL;
    std::memset(out, 0, sizeof(*out));
    return run(ctx, [&] {
        const tj_ctx_view cv = ctx_view(ctx);
        Workspace& ws = *cv.ws;
        cudaStream_t st = cv.stream;
        const DatasetDev& R = dataset_dev(Rh);
        const DatasetDev& S = dataset_dev(Sh);
        const bool knn = type == TJ_KNN;
        if (knn && k == 0) throw Error(TJ_EINVAL, "mbb_filter_knn: k must be >= 1");
        if (!knn && !(tau >= 0)) throw Error(TJ_EINVAL, "mbb_filter_within: tau must be >= 0");
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
        ma.shard_block = 1024;
        DevBuf<double> u_k;
        if (knn) {
            knn_kth_anchor(ws, ma, k, u_k, st);
            ma.tau_per_r = u_k.p;
        } else {
            ma.tau = tau;
            ma.confirm_at_mbb = 1;
        }
        CandDevStore cs;
        mbb_candidates(ws, ma, cs, st);
        TraceSink sink = make_sink(trace);
        if (sink.on_interval) sink.emit_flagged(cs, {}, TJ_STAGE_MBB, st);
        out->n_cands = cs.n;
        out->n_queries = R.n_objects;
        auto copy = [&](auto*& dst, auto& src, uint64_t n) {
            using T = std::remove_reference_t<decltype(*src.p)>;
            dst = host_alloc<T>(n);
            to_host(dst, src, n, st);
        };
        copy(out->pair_r, cs.pair_r, cs.n);
        copy(out->pair_s, cs.pair_s, cs.n);
        copy(out->lb, cs.lb, cs.n);
        copy(out->ub, cs.ub, cs.n);
        copy(out->status, cs.status, cs.n);
        copy(out->decided_at, cs.decided_at, cs.n);
        copy(out->r2op_offsets, cs.r2op, (uint64_t)R.n_objects + 1);
        copy(out->num_confirmed, cs.num_confirmed, R.n_objects);
        stream_sync(st);
    });
}

int tj_voxel_filter(tj_ctx* ctx, const tj_dataset* Rh, const tj_dataset* Sh, tj_cand_view* cands, int prune,
                    double tau, const tj_trace* trace, tj_vp_list* out, uint64_t* vp_generated, uint64_t* vp_pruned) {
    if (!ctx || !Rh || !Sh || !cands || !out) return TJ_EINVAL;
    std::memset(out, 0, sizeof(*out));
    return run(ctx, [&] {
        const tj_ctx_view cv = ctx_view(ctx);
        Workspace& ws = *cv.ws;
        cudaStream_t st = cv.stream;
        const DatasetDev& R = dataset_dev(Rh);
        const DatasetDev& S = dataset_dev(Sh);
        check_cands(cands);
        validate_pairs(cands, R, S);
        CandDevStore cs;
        upload_cands(cands, cs, st);
        ErrBuf err(st);
        VoxelArgs va{};
        va.n_cands = cs.n;
        va.r_voff = R.voxel_offsets.p;
        va.s_voff = S.voxel_offsets.p;
        va.r_vbox = R.voxel_box.p;
        va.s_vbox = S.voxel_box.p;
        va.r_vanc = R.voxel_anchor.p;
        va.s_vanc = S.voxel_anchor.p;
        va.prune = prune ? 1 : 0;
        va.tau = tau;
        va.err = err.e.p;
        TraceSink sink = make_sink(trace);
        const bool want = sink.on_interval || sink.on_vp_pruned;
        DevBuf<ActiveVpDev> active;
        std::vector<PrunedVp> pruned;
        std::vector<uint8_t> touched;
        const VoxelOut vo = voxel_filter(ws, va, cs, active, want, &pruned, &touched, st);
        check_err(err.e.p, st);
        if (vp_generated) *vp_generated = vo.vp_generated;
        if (vp_pruned) *vp_pruned = vo.vp_pruned;
        if (sink.on_interval) sink.emit_flagged(cs, touched, TJ_STAGE_VOXEL, st);
        if (sink.on_vp_pruned && !pruned.empty()) {
            std::vector<double> ub(cs.n);
            to_host(ub.data(), cs.ub, cs.n, st);
            stream_sync(st);
            for (const PrunedVp& p : pruned) sink.on_vp_pruned(sink.user, p.op, p.vr, p.vs, p.lb, ub[p.op]);
        }
        // survivors (op, i, j) in op order -> VoxelPairList with object-local voxel ids
        const uint64_t n = vo.survivors;
        std::vector<ActiveVpDev> h(n);
        if (n) TJ_CUDA(cudaMemcpyAsync(h.data(), active.p, n * sizeof(ActiveVpDev), cudaMemcpyDeviceToHost, st));
        download_cands(cands, cs, st);
        out->n_vps = n;
        out->n_ops = cands->n_cands;
        out->op_offsets = host_alloc<uint64_t>(cands->n_cands + 1);
        out->op = host_alloc<uint32_t>(n);
        out->vr = host_alloc<uint32_t>(n);
        out->vs = host_alloc<uint32_t>(n);
        std::fill(out->op_offsets, out->op_offsets + cands->n_cands + 1, 0);
        for (uint64_t t = 0; t < n; ++t) {
            const ActiveVpDev& a = h[t];
            out->op[t] = a.op;
            out->vr[t] = (uint32_t)(a.gvr - R.voxel_offsets_h[cands->pair_r[a.op]]);
            out->vs[t] = (uint32_t)(a.gvs - S.voxel_offsets_h[cands->pair_s[a.op]]);
            ++out->op_offsets[a.op + 1];
        }
        for (uint64_t op = 0; op < cands->n_cands; ++op) out->op_offsets[op + 1] += out->op_offsets[op];
    });
}

int tj_voxel_bounds(tj_ctx* ctx, const tj_dataset* Rh, const tj_dataset* Sh, const tj_cand_view* cands, uint64_t n_ops,
                    const uint32_t* ops, const uint64_t* vp_offsets, double* vp_lb, double* vp_ub, double* op_lb,
                    double* op_ub) {
    if (!ctx || !Rh || !Sh || !cands || (n_ops && (!ops || !op_lb || !op_ub)) || !vp_offsets) return TJ_EINVAL;
    return run(ctx, [&] {
        const tj_ctx_view cv = ctx_view(ctx);
        cudaStream_t st = cv.stream;
        const DatasetDev& R = dataset_dev(Rh);
        const DatasetDev& S = dataset_dev(Sh);
        check_cands(cands);
        validate_pairs(cands, R, S);
        for (uint64_t ci = 0; ci < n_ops; ++ci) {
            if (ops[ci] >= cands->n_cands) throw Error(TJ_EINVAL, "voxel_pair_bounds: op out of range");
            const uint32_t r = cands->pair_r[ops[ci]], s = cands->pair_s[ops[ci]];
            const uint64_t cnt = (R.voxel_offsets_h[r + 1] - R.voxel_offsets_h[r]) *
                                 (S.voxel_offsets_h[s + 1] - S.voxel_offsets_h[s]);
            if (vp_offsets[ci + 1] - vp_offsets[ci] != cnt)
                throw Error(TJ_EINVAL, "voxel_pair_bounds: vp_offsets do not match the voxel counts");
        }
        const uint64_t total = vp_offsets[n_ops];
        if (total && (!vp_lb || !vp_ub)) throw Error(TJ_EINVAL, "voxel_pair_bounds: null outputs");
        DevBuf<uint32_t> d_ops, pr, ps;
        DevBuf<uint64_t> d_off;
        to_dev(d_ops, ops, n_ops, st);
        to_dev(d_off, vp_offsets, n_ops + 1, st);
        to_dev(pr, cands->pair_r, cands->n_cands, st);
        to_dev(ps, cands->pair_s, cands->n_cands, st);
        DevBuf<double> dlb(std::max<uint64_t>(total, 1)), dub(std::max<uint64_t>(total, 1));
        DevBuf<unsigned long long> olb(std::max<uint64_t>(n_ops, 1)), oub(std::max<uint64_t>(n_ops, 1));
        const int g = grid_of(std::max<uint64_t>(n_ops, 1), cv.ws->num_sms);
        count_launch();
        k_fill<<<g, 256, 0, st>>>(olb.p, n_ops, 0x7ff0000000000000ull);
        count_launch();
        k_fill<<<g, 256, 0, st>>>(oub.p, n_ops, 0x7ff0000000000000ull);
        if (total) {
            count_launch();
            k_vox_bounds<<<grid_of(total, cv.ws->num_sms), 256, 0, st>>>(
                d_ops.p, d_off.p, n_ops, pr.p, ps.p, R.voxel_offsets.p, S.voxel_offsets.p, R.voxel_box.p,
                S.voxel_box.p, R.voxel_anchor.p, S.voxel_anchor.p, dlb.p, dub.p, olb.p, oub.p);
            TJ_CUDA(cudaGetLastError());
            to_host(vp_lb, dlb, total, st);
            to_host(vp_ub, dub, total, st);
        }
        if (n_ops) {
            TJ_CUDA(cudaMemcpyAsync(op_lb, olb.p, n_ops * 8, cudaMemcpyDeviceToHost, st));
            TJ_CUDA(cudaMemcpyAsync(op_ub, oub.p, n_ops * 8, cudaMemcpyDeviceToHost, st));
        }
        stream_sync(st);
    });
}

int tj_voxel_compact(tj_ctx* ctx, const tj_dataset* Rh, const tj_dataset* Sh, const tj_cand_view* cands,
                     uint64_t n_ops, const uint32_t* ops, const uint64_t* vp_offsets, const double* vp_lb,
                     tj_vp_list* out) {
    if (!ctx || !Rh || !Sh || !cands || !out || !vp_offsets || (n_ops && !ops)) return TJ_EINVAL;
    std::memset(out, 0, sizeof(*out));
    return run(ctx, [&] {
        const tj_ctx_view cv = ctx_view(ctx);
        Workspace& ws = *cv.ws;
        cudaStream_t st = cv.stream;
        const DatasetDev& R = dataset_dev(Rh);
        const DatasetDev& S = dataset_dev(Sh);
        check_cands(cands);
        validate_pairs(cands, R, S);
        for (uint64_t ci = 0; ci < n_ops; ++ci)
            if (ops[ci] >= cands->n_cands) throw Error(TJ_EINVAL, "voxel_pair_compact: op out of range");
        const uint64_t total = vp_offsets[n_ops];
        if (total && !vp_lb) throw Error(TJ_EINVAL, "voxel_pair_compact: null bounds");
        DevBuf<uint32_t> d_ops, ps;
        DevBuf<uint64_t> d_off;
        DevBuf<uint8_t> stv;
        DevBuf<double> ub, dlb;
        to_dev(d_ops, ops, n_ops, st);
        to_dev(d_off, vp_offsets, n_ops + 1, st);
        to_dev(ps, cands->pair_s, cands->n_cands, st);
        to_dev(stv, cands->status, cands->n_cands, st);
        to_dev(ub, cands->ub, cands->n_cands, st);
        to_dev(dlb, vp_lb, total, st);
        Survives sv{d_ops.p, d_off.p, n_ops, stv.p, ub.p, dlb.p};
        DevBuf<uint64_t> sel(std::max<uint64_t>(total, 1));
        const int64_t n = (int64_t)device_select(sv, IndexEmit{sel.p}, total, ws.u64a, st);
        DevBuf<uint32_t> o_op(std::max<int64_t>(n, 1)), o_i(std::max<int64_t>(n, 1)), o_j(std::max<int64_t>(n, 1));
        if (n) {
            count_launch();
            k_decode_survivors<<<grid_of((uint64_t)n, ws.num_sms), 256, 0, st>>>(sv, sel.p, (uint64_t)n, ps.p,
                                                                                 S.voxel_offsets.p, o_op.p, o_i.p,
                                                                                 o_j.p);
            TJ_CUDA(cudaGetLastError());
        }
        out->n_vps = (uint64_t)n;
        out->op = host_alloc<uint32_t>(n);
        out->vr = host_alloc<uint32_t>(n);
        out->vs = host_alloc<uint32_t>(n);
        to_host(out->op, o_op, n, st);
        to_host(out->vr, o_i, n, st);
        to_host(out->vs, o_j, n, st);
        stream_sync(st);
    });
}

int tj_refine_loop(tj_ctx* ctx, const tj_dataset* Rh, const tj_dataset* Sh, tj_cand_view* cands,
                   const tj_vp_list* vplist, const tj_join_spec* spec, const tj_trace* trace, tj_join_result* stats) {
    if (!ctx || !Rh || !Sh || !cands || !vplist || !spec) return TJ_EINVAL;
    if (stats) std::memset(stats, 0, sizeof(*stats));
    return run(ctx, [&] {
        const tj_ctx_view cv = ctx_view(ctx);
        Workspace& ws = *cv.ws;
        cudaStream_t st = cv.stream;
        const DatasetDev& R = dataset_dev(Rh);
        const DatasetDev& S = dataset_dev(Sh);
        const bool knn = spec->type == TJ_KNN;
        if (knn && spec->k == 0) throw Error(TJ_EINVAL, "refine_loop: k must be >= 1");
        if (spec->refine_chunk == 0) throw Error(TJ_EINVAL, "refine_loop: chunk size must be >= 1");
        if (spec->n_lods == 0 || !spec->lods || spec->lods[spec->n_lods - 1] != 100)
            throw Error(TJ_EINVAL, "refine_loop: lod schedule must end at 100");
        if (spec->n_lods > TJ_MAX_LODS) throw Error(TJ_EINVAL, "refine_loop: at most 16 lod levels are supported");
        for (uint32_t i = 1; i < spec->n_lods; ++i)
            if (spec->lods[i] <= spec->lods[i - 1]) throw Error(TJ_EINVAL, "refine_loop: lod schedule must be ascending");
        for (const DatasetDev* D : {&R, &S})
            for (uint32_t i = 0; i < spec->n_lods; ++i) {
                bool found = false;
                for (int32_t l : D->levels) found = found || l == (int32_t)spec->lods[i];
                if (!found)
                    throw Error(TJ_EENGINE, "refine: level " + std::to_string(spec->lods[i]) +
                                                " is not in the dataset's lod schedule");
            }
        check_cands(cands);
        validate_pairs(cands, R, S);
        if (!vplist->op_offsets || vplist->n_ops != cands->n_cands)
            throw Error(TJ_EINVAL, "refine_loop: voxel pair list does not match the candidate set");
        const uint64_t nvp = vplist->op_offsets[cands->n_cands];
        if (nvp && (!vplist->vr || !vplist->vs)) throw Error(TJ_EINVAL, "refine_loop: null voxel pair arrays");
        CandDevStore cs;
        upload_cands(cands, cs, st);
        ErrBuf err(st);
        DevBuf<uint64_t> off;
        DevBuf<uint32_t> vr, vs;
        DevBuf<int> bad(1);
        TJ_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        to_dev(off, vplist->op_offsets, cands->n_cands + 1, st);
        to_dev(vr, vplist->vr, nvp, st);
        to_dev(vs, vplist->vs, nvp, st);
        DevBuf<ActiveVpDev> active(std::max<uint64_t>(nvp, 1));
        if (nvp) {
            count_launch();
            k_active_from_list<<<grid_of(nvp, ws.num_sms), 256, 0, st>>>(off.p, cands->n_cands, vr.p, vs.p,
                                                                         cs.pair_r.p, cs.pair_s.p, R.voxel_offsets.p,
                                                                         S.voxel_offsets.p, active.p, bad.p);
            TJ_CUDA(cudaGetLastError());
        }
        int hb = 0;
        TJ_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        stream_sync(st);
        if (hb) throw Error(TJ_EINVAL, "refine_loop: voxel pair out of range");
        // only the voxel pairs of undecided candidates enter (src/refine.cpp:278-284)
        const uint64_t n_active = compact_active(ws, cs, active, nvp, st);
        TraceSink sink = make_sink(trace);
        RefineLoopOut ro = refine_loop_dev(ws, R, S, cs, active, n_active, *spec, knn, spec->tau, false, err.e.p,
                                           sink.on_interval ? &sink : nullptr, st);
        if (knn) {
            knn_finalize_dev(ws, cs, spec->k, st);
        } else {
            std::vector<uint8_t> stv(cs.n);
            to_host(stv.data(), cs.status, cs.n, st);
            stream_sync(st);
            for (uint8_t s : stv)
                if (s == TJ_UNDECIDED)
                    throw Error(TJ_EENGINE, "refine_loop: candidates left undecided after the exact level");
        }
        download_cands(cands, cs, st);
        if (stats) {
            stats->n_levels_run = (uint32_t)ro.levels.size();
            for (size_t i = 0; i < ro.levels.size() && i < TJ_MAX_LODS; ++i) {
                stats->level[i] = ro.levels[i].level;
                stats->level_vps[i] = ro.levels[i].vps;
                stats->level_facet_pairs[i] = ro.levels[i].facet_pairs;
                stats->level_pairs_evaluated[i] = ro.levels[i].evaluated;
                stats->level_pairs_tested[i] = ro.levels[i].tested;
                stats->level_ms[i] = ro.levels[i].ms;
                stats->level_kernel_ms[i] = ro.levels[i].kernel_ms;
            }
            stats->refine_chunks = ro.chunks;
        }
    });
}

int tj_knn_prune(tj_ctx* ctx, tj_cand_view* cands, uint32_t k, int16_t stage, int mode, uint8_t* deltas,
                 uint64_t* decisions) {
    if (!ctx || !cands || k == 0 || mode < 0 || mode > 2 || (mode == 0 && cands->n_cands && !deltas)) return TJ_EINVAL;
    return run(ctx, [&] {
        const tj_ctx_view cv = ctx_view(ctx);
        Workspace& ws = *cv.ws;
        cudaStream_t st = cv.stream;
        check_cands(cands);
        CandDevStore cs;
        upload_cands(cands, cs, st);
        ErrBuf err(st);
        uint64_t dec = 0;
        if (mode == 0) {
            DevBuf<uint8_t> d(std::max<uint64_t>(cs.n, 1));
            dec = knn_round_dev(ws, cs, k, d, err.e.p, st);
            check_err(err.e.p, st);
            to_host(deltas, d, cs.n, st);
            stream_sync(st);
        } else if (mode == 1) {
            dec = knn_fixpoint(ws, cs, k, stage, err.e.p, st);
            check_err(err.e.p, st);
            download_cands(cands, cs, st);
        } else {
            knn_finalize_dev(ws, cs, k, st);
            download_cands(cands, cs, st);
        }
        if (decisions) *decisions = dec;
    });
}

} // extern "C"
