// Stage-level C++ API of the drop-in (reference proj/include/trijoin/{filter,refine,knn,index}.hpp):
// the functions the reference's own tests and tools call directly. Each is a thin host
// layer over the stage C-ABI (include/tj_capi.h, csrc/stages.cu): the caller's
// CandidateSet is exchanged as plain arrays and every bound, prune, compaction and k-NN
// round runs on the device. Only build_rtree is host code: an STR packing of object MBBs
// that the device broad phase does not need (kept for API parity).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>

#include "packed.hpp"
#include "trijoin/engine.hpp"
#include "trijoin/knn.hpp"
#include "trijoin/refine.hpp"

namespace trijoin {

namespace {

tj_ctx* stage_ctx() { return detail::device_context(detail::join_devices()[0]); }

// Device copies pinned by live StageResidency scopes, by dataset address (with a use count:
// scopes may nest or share a dataset).
struct Pinned {
    std::shared_ptr<detail::DatasetHandle> h;
    int uses = 0;
};
std::mutex& pinned_mu() {
    static std::mutex* m = new std::mutex;
    return *m;
}
std::map<const void*, Pinned>& pinned() {
    static auto* p = new std::map<const void*, Pinned>;
    return *p;
}
std::shared_ptr<detail::DatasetHandle> pinned_handle(const PreparedDataset& d) {
    std::lock_guard<std::mutex> lk(pinned_mu());
    auto it = pinned().find(&d);
    return it == pinned().end() ? nullptr : it->second.h;
}
std::shared_ptr<detail::DatasetHandle> upload_dataset(tj_ctx* ctx, const PreparedDataset& d) {
    ThreadPool pool(0);
    auto p = detail::pack_dataset(d, pool);
    auto h = std::make_shared<detail::DatasetHandle>();
    detail::check(tj_dataset_upload(ctx, &p->view, &h->p), ctx);
    return h;
}

// R / S resident on the stage device for one call (the same object uploaded once when R is S),
// or the copies pinned by a StageResidency scope.
struct StagePair {
    tj_ctx* ctx;
    std::shared_ptr<detail::DatasetHandle> r, s;
    const tj_dataset* R() const { return r->p; }
    const tj_dataset* S() const { return s ? s->p : r->p; }
    StagePair(const PreparedDataset& Rd, const PreparedDataset& Sd) : ctx(stage_ctx()) {
        r = pinned_handle(Rd);
        if (!r) r = upload_dataset(ctx, Rd);
        if (&Sd != &Rd) {
            s = pinned_handle(Sd);
            if (!s) s = upload_dataset(ctx, Sd);
        }
    }
};

// Structure-of-arrays image of a CandidateSet for tj_cand_view; write_back() stores the
// device results (intervals, statuses, stages, confirmed counts) into the set.
struct CandArrays {
    std::vector<uint32_t> r, s;
    std::vector<double> lb, ub;
    std::vector<uint8_t> status;
    std::vector<uint64_t> r2op;
    std::vector<uint32_t> nconf;
    tj_cand_view view{};
    explicit CandArrays(CandidateSet& c, const uint32_t* num_confirmed_override = nullptr) {
        const size_t n = c.size();
        if (c.intervals.size() != n || c.status.size() != n || c.decided_at.size() != n)
            throw std::invalid_argument("trijoin: inconsistent candidate set");
        r.resize(n);
        s.resize(n);
        lb.resize(n);
        ub.resize(n);
        status.resize(n);
        for (size_t i = 0; i < n; ++i) {
            r[i] = c.pairs[i].first;
            s[i] = c.pairs[i].second;
            lb[i] = c.intervals[i].lb;
            ub[i] = c.intervals[i].ub;
            status[i] = static_cast<uint8_t>(c.status[i]);
        }
        r2op = c.r2op_offsets.empty() ? std::vector<uint64_t>{0} : c.r2op_offsets;
        const size_t nq = r2op.size() - 1;
        if (r2op.back() != n) throw std::invalid_argument("trijoin: r2op_offsets do not cover the candidate set");
        nconf.assign(nq, 0);
        for (size_t q = 0; q < nq && q < c.num_confirmed.size(); ++q) nconf[q] = c.num_confirmed[q];
        if (num_confirmed_override)
            for (size_t q = 0; q < nq; ++q) nconf[q] = num_confirmed_override[q];
        view.n_cands = n;
        view.n_queries = static_cast<uint32_t>(nq);
        view.pair_r = r.data();
        view.pair_s = s.data();
        view.lb = lb.data();
        view.ub = ub.data();
        view.status = status.data();
        view.decided_at = c.decided_at.data();
        view.r2op_offsets = r2op.data();
        view.num_confirmed = nconf.data();
    }
    void write_back(CandidateSet& c) const {
        for (size_t i = 0; i < c.size(); ++i) {
            c.intervals[i] = {lb[i], ub[i]};
            c.status[i] = static_cast<PairStatus>(status[i]);
        }
        if (!c.r2op_offsets.empty()) c.num_confirmed.assign(nconf.begin(), nconf.end());
    }
};

struct VpListHandle {
    tj_vp_list l{};
    ~VpListHandle() { tj_vp_list_free(&l); }
};

struct TraceBridgeS {
    const JoinTrace* t;
    static void interval(void* u, uint32_t op, int16_t st, double lb, double ub) {
        const auto* self = static_cast<TraceBridgeS*>(u);
        if (self->t->on_interval) self->t->on_interval(op, st, Interval{lb, ub});
    }
    static void pruned(void* u, uint32_t op, uint32_t vr, uint32_t vs, double lb, double ub) {
        const auto* self = static_cast<TraceBridgeS*>(u);
        if (self->t->on_vp_pruned) self->t->on_vp_pruned(op, vr, vs, lb, ub);
    }
};

CandidateSet from_result(const tj_join_result& r) {
    CandidateSet c;
    const uint64_t n = r.n_cands;
    c.pairs.resize(n);
    c.intervals.resize(n);
    c.status.resize(n);
    c.decided_at.assign(r.decided_at, r.decided_at + n);
    for (uint64_t i = 0; i < n; ++i) {
        c.pairs[i] = {r.pair_r[i], r.pair_s[i]};
        c.intervals[i] = {r.lb[i], r.ub[i]};
        c.status[i] = static_cast<PairStatus>(r.status[i]);
    }
    c.r2op_offsets.assign(r.r2op_offsets, r.r2op_offsets + r.n_queries + 1);
    c.num_confirmed.assign(r.num_confirmed, r.num_confirmed + r.n_queries);
    return c;
}

CandidateSet mbb_stage(const PreparedDataset& R, const PreparedDataset& S, int32_t type, double tau, uint32_t k,
                       const JoinTrace* trace) {
    StagePair sp(R, S);
    detail::ResultHandle res;
    TraceBridgeS bridge{trace};
    tj_trace tt{&bridge, &TraceBridgeS::interval, &TraceBridgeS::pruned};
    detail::check(tj_mbb_filter(sp.ctx, sp.R(), sp.S(), type, tau, k, trace ? &tt : nullptr, &res.r), sp.ctx);
    return from_result(res.r);
}

// ---------------------------------------------------------------- STR R-tree (host)
std::vector<std::vector<uint32_t>> str_groups(const std::vector<Aabb>& boxes, std::vector<uint32_t> ids) {
    // sort-tile-recursive: x-centre slabs, y-centre runs, z-centre order, groups of kFanout
    const size_t n = ids.size(), fan = RTree::kFanout;
    std::vector<std::vector<uint32_t>> out;
    if (n == 0) return out;
    auto by = [&](size_t b, size_t e, int axis) {
        std::sort(ids.begin() + b, ids.begin() + e, [&](uint32_t x, uint32_t y) {
            const Point3 cx = boxes[x].center(), cy = boxes[y].center();
            const double vx = axis == 0 ? cx.x : axis == 1 ? cx.y : cx.z;
            const double vy = axis == 0 ? cy.x : axis == 1 ? cy.y : cy.z;
            return vx != vy ? vx < vy : x < y;
        });
    };
    const size_t pages = (n + fan - 1) / fan;
    const size_t slabs = static_cast<size_t>(std::ceil(std::cbrt(static_cast<double>(pages))));
    const size_t slab = (n + slabs - 1) / slabs;
    by(0, n, 0);
    for (size_t sb = 0; sb < n; sb += slab) {
        const size_t se = std::min(n, sb + slab);
        const size_t runs = static_cast<size_t>(std::ceil(std::sqrt(static_cast<double>((se - sb + fan - 1) / fan))));
        const size_t run = (se - sb + runs - 1) / runs;
        by(sb, se, 1);
        for (size_t rb = sb; rb < se; rb += run) {
            const size_t re = std::min(se, rb + run);
            by(rb, re, 2);
            for (size_t gb = rb; gb < re; gb += fan) out.emplace_back(ids.begin() + gb, ids.begin() + std::min(re, gb + fan));
        }
    }
    return out;
}

} // namespace

StageResidency::StageResidency(const PreparedDataset& R, const PreparedDataset& S) : r_(&R), s_(&S) {
    tj_ctx* ctx = stage_ctx();
    for (const PreparedDataset* d : {&R, &S}) {
        if (d == &S && &S == &R) break;
        {
            std::lock_guard<std::mutex> lk(pinned_mu());
            auto it = pinned().find(d);
            if (it != pinned().end()) {
                ++it->second.uses;
                continue;
            }
        }
        auto h = upload_dataset(ctx, *d);
        std::lock_guard<std::mutex> lk(pinned_mu());
        Pinned& p = pinned()[d];
        if (!p.h) p.h = std::move(h);
        ++p.uses;
    }
}

StageResidency::~StageResidency() {
    std::lock_guard<std::mutex> lk(pinned_mu());
    for (const void* d : {r_, s_}) {
        if (d == s_ && s_ == r_) break;
        auto it = pinned().find(d);
        if (it != pinned().end() && --it->second.uses == 0) pinned().erase(it);
    }
}

RTree build_rtree(std::span<const PreparedObject> objects) {
    RTree tree;
    if (objects.empty()) return tree;
    std::vector<Aabb> boxes(objects.size());
    std::vector<uint32_t> ids(objects.size());
    for (uint32_t i = 0; i < objects.size(); ++i) {
        boxes[i] = objects[i].mbb;
        ids[i] = i;
    }
    std::vector<std::vector<RTree::Node>> levels(1);
    for (const auto& g : str_groups(boxes, ids)) {
        RTree::Node nd;
        nd.leaf = true;
        nd.first = static_cast<uint32_t>(tree.entries.size());
        nd.count = static_cast<uint32_t>(g.size());
        nd.box = Aabb::empty();
        for (uint32_t id : g) {
            tree.entries.push_back(id);
            nd.box.expand(boxes[id]);
        }
        levels.back().push_back(nd);
    }
    while (levels.back().size() > 1) {
        std::vector<RTree::Node>& kids = levels.back();
        std::vector<Aabb> kb(kids.size());
        std::vector<uint32_t> kid_ids(kids.size());
        for (uint32_t i = 0; i < kids.size(); ++i) {
            kb[i] = kids[i].box;
            kid_ids[i] = i;
        }
        std::vector<RTree::Node> packed, parents;
        for (const auto& g : str_groups(kb, kid_ids)) {
            RTree::Node nd;
            nd.leaf = false;
            nd.first = static_cast<uint32_t>(packed.size());
            nd.count = static_cast<uint32_t>(g.size());
            nd.box = Aabb::empty();
            for (uint32_t k : g) {
                nd.box.expand(kids[k].box);
                packed.push_back(kids[k]);
            }
            parents.push_back(nd);
        }
        kids = std::move(packed);
        levels.push_back(std::move(parents));
    }
    std::vector<uint32_t> base(levels.size(), 0);
    for (size_t k = 1; k < levels.size(); ++k) base[k] = base[k - 1] + static_cast<uint32_t>(levels[k - 1].size());
    for (size_t k = 0; k < levels.size(); ++k)
        for (RTree::Node nd : levels[k]) {
            if (!nd.leaf) nd.first += base[k - 1];
            tree.nodes.push_back(nd);
        }
    tree.root = base.back();
    tree.node_levels = static_cast<int>(levels.size());
    return tree;
}

// ---------------------------------------------------------------- filter stages
CandidateSet mbb_filter_within(const PreparedDataset& R, const PreparedDataset& S, const RTree&, double tau,
                               ThreadPool&, const JoinTrace* trace) {
    if (!(tau >= 0)) throw std::invalid_argument("mbb_filter_within: tau must be >= 0");
    return mbb_stage(R, S, TJ_WITHIN, tau, 1, trace);
}

CandidateSet mbb_filter_knn(const PreparedDataset& R, const PreparedDataset& S, const RTree&, uint32_t k, ThreadPool&,
                            const JoinTrace* trace) {
    if (k == 0) throw std::invalid_argument("mbb_filter_knn: k must be >= 1");
    return mbb_stage(R, S, TJ_KNN, 0.0, k, trace);
}

ChunkBounds voxel_pair_bounds(const FilterChunk& chunk, CandidateSet& cands, const PreparedDataset& R,
                              const PreparedDataset& S, ThreadPool&, const JoinTrace* trace) {
    if (chunk.vp_offsets.size() != chunk.ops.size() + 1)
        throw std::invalid_argument("voxel_pair_bounds: vp_offsets must have ops + 1 entries");
    StagePair sp(R, S);
    CandArrays ca(cands);
    ChunkBounds out;
    out.vp_lb.resize(chunk.total_vp());
    out.vp_ub.resize(chunk.total_vp());
    out.op_lb.resize(chunk.ops.size());
    out.op_ub.resize(chunk.ops.size());
    detail::check(tj_voxel_bounds(sp.ctx, sp.R(), sp.S(), &ca.view, chunk.ops.size(), chunk.ops.data(),
                                  chunk.vp_offsets.data(), out.vp_lb.data(), out.vp_ub.data(), out.op_lb.data(),
                                  out.op_ub.data()),
                  sp.ctx);
    // the serial fold into the candidate intervals, in chunk order (src/filter.cpp:230-236)
    for (size_t ci = 0; ci < chunk.ops.size(); ++ci) {
        const uint32_t op = chunk.ops[ci];
        if (cands.status[op] != PairStatus::Undecided) continue;
        intersect_interval(cands.intervals[op], out.op_lb[ci], out.op_ub[ci]);
        if (trace && trace->on_interval) trace->on_interval(op, stage::kVoxel, cands.intervals[op]);
    }
    return out;
}

std::vector<std::tuple<uint32_t, uint32_t, uint32_t>> voxel_pair_compact(const FilterChunk& chunk,
                                                                         const ChunkBounds& bounds,
                                                                         const CandidateSet& cands,
                                                                         const PreparedDataset& R,
                                                                         const PreparedDataset& S, ThreadPool&,
                                                                         const JoinTrace* trace) {
    if (chunk.vp_offsets.size() != chunk.ops.size() + 1 || bounds.vp_lb.size() != chunk.total_vp())
        throw std::invalid_argument("voxel_pair_compact: bounds do not match the chunk");
    StagePair sp(R, S);
    CandidateSet copy = cands; // the view is mutable; the stage does not modify it
    CandArrays ca(copy);
    VpListHandle h;
    detail::check(tj_voxel_compact(sp.ctx, sp.R(), sp.S(), &ca.view, chunk.ops.size(), chunk.ops.data(),
                                   chunk.vp_offsets.data(), bounds.vp_lb.data(), &h.l),
                  sp.ctx);
    std::vector<std::tuple<uint32_t, uint32_t, uint32_t>> out(h.l.n_vps);
    for (uint64_t k = 0; k < h.l.n_vps; ++k) out[k] = {h.l.op[k], h.l.vr[k], h.l.vs[k]};
    if (trace && trace->on_vp_pruned) { // non-survivors of undecided ops, flattened order
        size_t si = 0;
        for (size_t ci = 0; ci < chunk.ops.size(); ++ci) {
            const uint32_t op = chunk.ops[ci];
            const uint64_t ns = S.objects[cands.pairs[op].second].voxels.voxel_count();
            for (uint64_t t = chunk.vp_offsets[ci]; t < chunk.vp_offsets[ci + 1]; ++t) {
                const uint32_t i = static_cast<uint32_t>((t - chunk.vp_offsets[ci]) / ns);
                const uint32_t j = static_cast<uint32_t>((t - chunk.vp_offsets[ci]) % ns);
                if (si < out.size() && out[si] == std::tuple<uint32_t, uint32_t, uint32_t>{op, i, j}) {
                    ++si;
                    continue;
                }
                if (cands.status[op] != PairStatus::Undecided) continue;
                trace->on_vp_pruned(op, i, j, bounds.vp_lb[t], cands.intervals[op].ub);
            }
        }
    }
    return out;
}

VoxelPairList chunked_filter(CandidateSet& cands, const PreparedDataset& R, const PreparedDataset& S, uint64_t budget,
                             std::optional<double> tau, bool, ThreadPool& pool, FilterStats* stats,
                             const JoinTrace* trace) {
    if (budget == 0) throw std::invalid_argument("chunked_filter: budget must be >= 1");
    // greedy consecutive packing of the undecided ops (src/filter.cpp:319-346): results do
    // not depend on it, the chunk counters do
    std::vector<FilterChunk> chunks;
    {
        FilterChunk cur;
        cur.vp_offsets.push_back(0);
        auto flush = [&] {
            if (!cur.ops.empty()) chunks.push_back(std::move(cur));
            cur = FilterChunk{};
            cur.vp_offsets.push_back(0);
        };
        for (uint32_t op = 0; op < cands.size(); ++op) {
            if (cands.status[op] != PairStatus::Undecided) continue;
            const uint64_t n = voxel_pair_count(cands, op, R, S);
            if (n > budget) {
                flush();
                cur.ops.push_back(op);
                cur.vp_offsets.push_back(n);
                cur.oversized = true;
                flush();
                continue;
            }
            if (!cur.ops.empty() && cur.total_vp() + n > budget) flush();
            cur.ops.push_back(op);
            cur.vp_offsets.push_back(cur.total_vp() + n);
        }
        flush();
    }
    if (stats) {
        stats->chunks += chunks.size();
        for (const FilterChunk& c : chunks) stats->oversized_chunks += c.oversized ? 1 : 0;
    }
    VoxelPairList out;
    if (trace && (trace->on_interval || trace->on_vp_pruned) && chunks.size() > 1) {
        // observers see the reference's per-chunk event order: chunk by chunk on the device
        std::vector<std::tuple<uint32_t, uint32_t, uint32_t>> all;
        for (const FilterChunk& chunk : chunks) {
            const ChunkBounds b = voxel_pair_bounds(chunk, cands, R, S, pool, trace);
            if (tau) prune_within(cands, *tau, stage::kVoxel, chunk.ops);
            auto surv = voxel_pair_compact(chunk, b, cands, R, S, pool, trace);
            if (stats) {
                stats->vp_generated += chunk.total_vp();
                uint64_t und = 0;
                for (size_t i = 0; i < chunk.ops.size(); ++i)
                    if (cands.status[chunk.ops[i]] == PairStatus::Undecided)
                        und += chunk.vp_offsets[i + 1] - chunk.vp_offsets[i];
                stats->vp_pruned += und - surv.size();
            }
            all.insert(all.end(), surv.begin(), surv.end());
        }
        out.op_offsets.assign(cands.size() + 1, 0);
        for (const auto& [op, vr, vs] : all) ++out.op_offsets[op + 1];
        for (size_t op = 0; op < cands.size(); ++op) out.op_offsets[op + 1] += out.op_offsets[op];
        out.vpairs.resize(all.size());
        std::vector<uint64_t> cur(out.op_offsets.begin(), out.op_offsets.end() - 1);
        for (const auto& [op, vr, vs] : all) out.vpairs[cur[op]++] = {vr, vs};
        return out;
    }
    StagePair sp(R, S);
    CandArrays ca(cands);
    VpListHandle h;
    uint64_t gen = 0, pruned = 0;
    TraceBridgeS bridge{trace};
    tj_trace tt{&bridge, &TraceBridgeS::interval, &TraceBridgeS::pruned};
    detail::check(tj_voxel_filter(sp.ctx, sp.R(), sp.S(), &ca.view, tau ? 1 : 0, tau.value_or(0.0),
                                  trace ? &tt : nullptr, &h.l, &gen, &pruned),
                  sp.ctx);
    ca.write_back(cands);
    if (stats) {
        stats->vp_generated += gen;
        stats->vp_pruned += pruned;
    }
    out.op_offsets.assign(h.l.op_offsets, h.l.op_offsets + cands.size() + 1);
    out.vpairs.resize(h.l.n_vps);
    for (uint64_t t = 0; t < h.l.n_vps; ++t) out.vpairs[t] = {h.l.vr[t], h.l.vs[t]};
    return out;
}

// ---------------------------------------------------------------- refinement + k-NN
void refine_loop(CandidateSet& cands, const VoxelPairList& vplist, const PreparedDataset& R, const PreparedDataset& S,
                 const RefineConfig& config, std::optional<double> tau, KnnState* knn, ThreadPool&, RefineStats* stats,
                 const JoinTrace* trace) {
    if (tau.has_value() == (knn != nullptr))
        throw std::invalid_argument("refine_loop: exactly one of tau and knn must be set");
    if (config.chunk == 0) throw std::invalid_argument("refine_loop: chunk size must be >= 1");
    if (config.lods.empty() || config.lods.back() != 100)
        throw std::invalid_argument("refine_loop: lod schedule must end at 100");
    for (size_t i = 1; i < config.lods.size(); ++i)
        if (config.lods[i] <= config.lods[i - 1])
            throw std::invalid_argument("refine_loop: lod schedule must be ascending");
    if (vplist.op_offsets.size() != cands.size() + 1)
        throw std::invalid_argument("refine_loop: voxel pair list does not match the candidate set");
    StagePair sp(R, S);
    CandArrays ca(cands, knn ? knn->num_confirmed.data() : nullptr);
    if (knn && knn->num_confirmed.size() != ca.view.n_queries)
        throw std::invalid_argument("refine_loop: knn state does not match the candidate set");
    const std::vector<uint32_t> before = ca.nconf;
    std::vector<uint32_t> vr(vplist.vpairs.size()), vs(vplist.vpairs.size());
    for (size_t t = 0; t < vplist.vpairs.size(); ++t) {
        vr[t] = vplist.vpairs[t].first;
        vs[t] = vplist.vpairs[t].second;
    }
    tj_vp_list l{};
    l.n_ops = cands.size();
    l.n_vps = vplist.vpairs.size();
    l.op_offsets = const_cast<uint64_t*>(vplist.op_offsets.data());
    l.vr = vr.data();
    l.vs = vs.data();
    tj_join_spec spec{};
    spec.type = knn ? TJ_KNN : TJ_WITHIN;
    spec.tau = tau.value_or(0.0);
    spec.k = knn ? knn->k : 1;
    spec.filter_chunk = 4194304;
    spec.refine_chunk = config.chunk;
    spec.n_lods = static_cast<uint32_t>(config.lods.size());
    spec.lods = config.lods.data();
    spec.pipeline = config.pipeline ? 1 : 0;
    detail::ResultHandle res;
    TraceBridgeS bridge{trace};
    tj_trace tt{&bridge, &TraceBridgeS::interval, &TraceBridgeS::pruned};
    detail::check(tj_refine_loop(sp.ctx, sp.R(), sp.S(), &ca.view, &l, &spec, trace ? &tt : nullptr, &res.r), sp.ctx);
    // cands.num_confirmed and the knn state's counts both advance by the new confirmations
    std::vector<uint32_t> cand_before(cands.num_confirmed);
    ca.write_back(cands);
    if (knn) {
        for (size_t q = 0; q < ca.nconf.size(); ++q) {
            const uint32_t add = ca.nconf[q] - before[q];
            knn->num_confirmed[q] += add;
            if (q < cand_before.size()) cands.num_confirmed[q] = cand_before[q] + add;
        }
    }
    if (stats) {
        for (uint32_t i = 0; i < res.r.n_levels_run; ++i) {
            stats->levels.push_back({res.r.level[i], res.r.level_ms[i], res.r.level_vps[i], res.r.level_facet_pairs[i]});
            stats->facet_pairs += res.r.level_facet_pairs[i];
            stats->kernel_vps += res.r.level_vps[i];
        }
        stats->chunks += res.r.refine_chunks;
    }
}

std::vector<KnnDelta> knn_prune_round(const KnnState& state, const CandidateSet& cands, ThreadPool&) {
    CandidateSet copy = cands;
    CandArrays ca(copy, state.num_confirmed.size() == cands.r2op_offsets.size() - 1 ? state.num_confirmed.data()
                                                                                     : nullptr);
    std::vector<uint8_t> d(cands.size(), 0);
    tj_ctx* ctx = stage_ctx();
    uint64_t n = 0;
    detail::check(tj_knn_prune(ctx, &ca.view, state.k, 0, 0, d.data(), &n), ctx);
    std::vector<KnnDelta> out;
    out.reserve(n);
    for (uint32_t op = 0; op < d.size(); ++op)
        if (d[op]) out.push_back({op, static_cast<PairStatus>(d[op])});
    return out;
}

size_t knn_prune_to_fixpoint(KnnState& state, CandidateSet& cands, int16_t stage_code, ThreadPool&) {
    CandArrays ca(cands, state.num_confirmed.data());
    const std::vector<uint32_t> before = ca.nconf;
    tj_ctx* ctx = stage_ctx();
    uint64_t n = 0;
    detail::check(tj_knn_prune(ctx, &ca.view, state.k, stage_code, 1, nullptr, &n), ctx);
    std::vector<uint32_t> cand_before(cands.num_confirmed);
    ca.write_back(cands);
    for (size_t q = 0; q < ca.nconf.size(); ++q) {
        const uint32_t add = ca.nconf[q] - before[q];
        state.num_confirmed[q] += add;
        cands.num_confirmed[q] = (q < cand_before.size() ? cand_before[q] : 0) + add;
    }
    return n;
}

void knn_finalize(KnnState& state, CandidateSet& cands) {
    CandArrays ca(cands, state.num_confirmed.data());
    const std::vector<uint32_t> before = ca.nconf;
    tj_ctx* ctx = stage_ctx();
    detail::check(tj_knn_prune(ctx, &ca.view, state.k, 100, 2, nullptr, nullptr), ctx);
    std::vector<uint32_t> cand_before(cands.num_confirmed);
    ca.write_back(cands);
    for (size_t q = 0; q < ca.nconf.size(); ++q) {
        const uint32_t add = ca.nconf[q] - before[q];
        state.num_confirmed[q] += add;
        cands.num_confirmed[q] = (q < cand_before.size() ? cand_before[q] : 0) + add;
    }
}

void knn_resolve(KnnState& state, CandidateSet& cands, const VoxelPairList& vplist, const PreparedDataset& R,
                 const PreparedDataset& S, const RefineConfig& config, ThreadPool& pool, RefineStats* stats,
                 const JoinTrace* trace) {
    refine_loop(cands, vplist, R, S, config, std::nullopt, &state, pool, stats, trace);
}

} // namespace trijoin
