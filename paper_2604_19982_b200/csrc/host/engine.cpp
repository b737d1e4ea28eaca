// Host side of the drop-in trijoin engine: packs PreparedDatasets into the device layout,
// drives tj_join on one or more B200s (R sharded by query blocks, one host thread per
// GPU), and assembles records / StageStats exactly as the reference's run_join
// (src/engine.cpp:122-237). All join arithmetic runs on the GPU.
#include <algorithm>
#include <atomic>
#include <bit>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <thread>

#include <cuda_runtime.h>
#include <json.hpp>

#include "packed.hpp"
#include "trijoin/engine.hpp"

namespace trijoin {

namespace {
// object-range pieces per streamed level (pack_level / tj_dataset_put_level_part)
constexpr size_t kPackPieces = 8;
} // namespace

// ---------------------------------------------------------------- detail: contexts, packing
namespace detail {

[[noreturn]] void throw_status(int code, const char* msg) {
    const std::string m = msg ? msg : "";
    if (code == TJ_EINVAL) throw std::invalid_argument(m);
    if (code == TJ_EENGINE) throw EngineError(m);
    throw std::runtime_error(m);
}

namespace {
// The per-device contexts live until the process exits and are never destroyed: a static
// destructor would run after the CUDA runtime's own teardown (the registry is constructed before
// the runtime's first call registers it) and release streams and memory on a dead runtime.
struct CtxRegistry {
    std::mutex mu;
    std::map<std::pair<int, int>, tj_ctx*> ctxs;
};
CtxRegistry& registry() {
    static CtxRegistry* r = new CtxRegistry;
    return *r;
}
} // namespace

tj_ctx* device_context(int device, int slot) {
    CtxRegistry& reg = registry();
    std::lock_guard<std::mutex> lk(reg.mu);
    auto it = reg.ctxs.find({device, slot});
    if (it != reg.ctxs.end()) return it->second;
    tj_ctx* c = nullptr;
    const int rc = tj_ctx_create(device, &c);
    if (rc != TJ_OK) throw std::runtime_error(std::string("trijoin: no usable B200 device: ") + tj_global_last_error());
    reg.ctxs[{device, slot}] = c;
    return c;
}

std::vector<int> join_devices() {
    std::vector<int> out;
    if (const char* env = std::getenv("TRIJOIN_DEVICES")) {
        std::stringstream ss(env);
        std::string tok;
        while (std::getline(ss, tok, ','))
            if (!tok.empty()) out.push_back(std::stoi(tok));
    }
    if (out.empty()) out.push_back(0);
    return out;
}

namespace {
// Process-wide host staging arena: freed blocks are kept for reuse (pinning and first-touch
// page faults are slow; reuse is free). Blocks are page-locked unless no device is present.
struct PinnedArena {
    std::mutex mu;
    std::multimap<size_t, std::pair<double*, bool>> free_blocks; // capacity (doubles) -> (block, pinned)
    std::atomic<uint64_t> n_new{0}, n_pageable{0}, bytes_new{0}, ns_new{0}; // diagnostics (stats JSON)
    double* acquire(size_t want, size_t& cap, bool& pinned) {
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = free_blocks.lower_bound(want);
            if (it != free_blocks.end() && it->first <= 2 * want + (1u << 20)) {
                cap = it->first;
                double* p = it->second.first;
                pinned = it->second.second;
                free_blocks.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        cap = want;
        const auto t0 = std::chrono::steady_clock::now();
        const bool ok = cudaHostAlloc(&p, want * sizeof(double), cudaHostAllocPortable) == cudaSuccess;
        ++n_new;
        bytes_new += want * sizeof(double);
        ns_new += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
        if (ok) {
            pinned = true;
            return static_cast<double*>(p);
        }
        cudaGetLastError(); // no device / pinning refused: pageable host memory
        ++n_pageable;
        pinned = false;
        p = std::malloc(want * sizeof(double));
        if (!p) throw std::bad_alloc();
        return static_cast<double*>(p);
    }
    void release(double* p, size_t cap, bool pinned) {
        if (!p) return;
        // blocks of 1 GiB and more go back to the OS (a dataset's level on the D / E scale:
        // keeping them would pin tens of GB beside the caller's datasets)
        if (cap * sizeof(double) >= (size_t(1) << 30)) {
            if (pinned)
                cudaFreeHost(p);
            else
                std::free(p);
            return;
        }
        std::lock_guard<std::mutex> lk(mu);
        free_blocks.emplace(cap, std::make_pair(p, pinned));
    }
};
PinnedArena& arena() {
    static PinnedArena* a = new PinnedArena(); // intentionally leaked: outlives the CUDA runtime
    return *a;
}
} // namespace

ArenaStats arena_stats() {
    PinnedArena& a = arena();
    return {a.n_new.load(), a.n_pageable.load(), a.bytes_new.load(), a.ns_new.load() / 1e6};
}

PinnedBuf& PinnedBuf::operator=(PinnedBuf&& o) noexcept {
    if (this != &o) {
        arena().release(p, cap, pinned);
        p = o.p;
        n = o.n;
        cap = o.cap;
        pinned = o.pinned;
        o.p = nullptr;
        o.n = o.cap = 0;
    }
    return *this;
}

PinnedBuf::~PinnedBuf() { arena().release(p, cap, pinned); }

void PinnedBuf::resize(size_t count) {
    if (count > cap) {
        arena().release(p, cap, pinned);
        p = nullptr;
        cap = 0;
        if (count) p = arena().acquire(count, cap, pinned);
    }
    n = count;
}

uint64_t PackedDataset::bytes() const {
    uint64_t b = (mbb.size() + anchor.size() + voxel_box.size() + voxel_anchor.size()) * 8 + voxel_offsets.size() * 8;
    for (const auto& v : facet_offsets) b += v.size() * 8;
    for (const auto& v : facets) b += v.size() * 8;
    return b;
}

std::unique_ptr<PackedDataset> pack_dataset(const PreparedDataset& ds, ThreadPool& pool, const std::vector<uint32_t>* ids) {
    auto p = std::make_unique<PackedDataset>();
    const size_t no = ids ? ids->size() : ds.objects.size();
    auto obj_at = [&](size_t o) -> const PreparedObject& { return ds.objects[ids ? (*ids)[o] : o]; };
    if (ids)
        for (size_t i = 0; i < ids->size(); ++i)
            if ((*ids)[i] >= ds.objects.size()) throw std::invalid_argument("trijoin: shard object id out of range");
    const size_t nl = ds.lod_schedule.size();
    p->n_objects = static_cast<uint32_t>(no);
    p->levels.assign(ds.lod_schedule.begin(), ds.lod_schedule.end());
    p->mbb.resize(6 * no);
    p->anchor.resize(3 * no);
    p->voxel_offsets.assign(no + 1, 0);
    for (size_t o = 0; o < no; ++o) {
        const PreparedObject& obj = obj_at(o);
        if (obj.ladder.levels.size() != nl || obj.voxels.facets_per_level.size() != nl)
            throw std::invalid_argument("trijoin: object level count does not match the lod schedule");
        p->voxel_offsets[o + 1] = p->voxel_offsets[o] + obj.voxels.voxel_count();
    }
    const uint64_t nv = p->voxel_offsets[no];
    p->voxel_box.resize(6 * nv);
    p->voxel_anchor.resize(3 * nv);
    p->facet_offsets.assign(nl, std::vector<uint64_t>(nv + 1, 0));
    p->facets.resize(nl);
    // per level: facet entries per voxel -> offsets
    pool.parallel_jobs(no, [&](size_t o) {
        const PreparedObject& obj = obj_at(o);
        const uint64_t v0 = p->voxel_offsets[o];
        for (size_t li = 0; li < nl; ++li)
            for (uint32_t v = 0; v < obj.voxels.voxel_count(); ++v)
                p->facet_offsets[li][v0 + v + 1] = obj.voxels.facets_per_level[li][v].size();
    });
    for (size_t li = 0; li < nl; ++li) {
        auto& fo = p->facet_offsets[li];
        for (uint64_t v = 0; v < nv; ++v) fo[v + 1] += fo[v];
        p->facets[li].resize(fo[nv] * TJ_FACET_STRIDE);
    }
    pool.parallel_jobs(no, [&](size_t o) {
        const PreparedObject& obj = obj_at(o);
        const double m[6] = {obj.mbb.min.x, obj.mbb.min.y, obj.mbb.min.z, obj.mbb.max.x, obj.mbb.max.y, obj.mbb.max.z};
        std::memcpy(&p->mbb[6 * o], m, sizeof(m));
        p->anchor[3 * o] = obj.anchor.x;
        p->anchor[3 * o + 1] = obj.anchor.y;
        p->anchor[3 * o + 2] = obj.anchor.z;
        const uint64_t v0 = p->voxel_offsets[o];
        const VoxelSet& vs = obj.voxels;
        for (uint32_t v = 0; v < vs.voxel_count(); ++v) {
            const Aabb& b = vs.boxes[v];
            const double bb[6] = {b.min.x, b.min.y, b.min.z, b.max.x, b.max.y, b.max.z};
            std::memcpy(&p->voxel_box[6 * (v0 + v)], bb, sizeof(bb));
            p->voxel_anchor[3 * (v0 + v)] = vs.anchors[v].x;
            p->voxel_anchor[3 * (v0 + v) + 1] = vs.anchors[v].y;
            p->voxel_anchor[3 * (v0 + v) + 2] = vs.anchors[v].z;
        }
        for (size_t li = 0; li < nl; ++li) {
            const LodMesh& lod = obj.ladder.levels[li];
            const auto& fo = p->facet_offsets[li];
            double* dst = p->facets[li].data();
            for (uint32_t v = 0; v < vs.voxel_count(); ++v) {
                uint64_t e = fo[v0 + v];
                for (uint32_t f : vs.facets_per_level[li][v]) {
                    if (f >= lod.mesh.facets.size() || f >= lod.hd.size() || f >= lod.ph.size())
                        throw std::invalid_argument("trijoin: voxel facet id out of range");
                    const auto& tri = lod.mesh.facets[f];
                    double* r = dst + e * TJ_FACET_STRIDE;
                    for (int k = 0; k < 3; ++k) {
                        const Point3& pt = lod.mesh.vertices[tri[k]];
                        r[3 * k] = pt.x;
                        r[3 * k + 1] = pt.y;
                        r[3 * k + 2] = pt.z;
                    }
                    r[9] = lod.hd[f];
                    r[10] = lod.ph[f];
                    r[11] = 0.0;
                    ++e;
                }
            }
        }
    });
    p->fo_ptrs.resize(nl);
    p->f_ptrs.resize(nl);
    for (size_t li = 0; li < nl; ++li) {
        p->fo_ptrs[li] = p->facet_offsets[li].data();
        p->f_ptrs[li] = p->facets[li].data();
    }
    tj_dataset_view& v = p->view;
    v.n_objects = p->n_objects;
    v.n_levels = static_cast<uint32_t>(nl);
    v.levels = p->levels.data();
    v.mbb = p->mbb.data();
    v.anchor = p->anchor.data();
    v.voxel_offsets = p->voxel_offsets.data();
    v.voxel_box = p->voxel_box.data();
    v.voxel_anchor = p->voxel_anchor.data();
    v.facet_offsets = p->fo_ptrs.data();
    v.facets = p->f_ptrs.data();
    return p;
}

namespace {
// The objects a header is packed from: a contiguous run (R chunks of the out-of-core path) or
// a list of global ids (query shards).
struct ObjSel {
    const PreparedObject* base;
    size_t n;
    const uint32_t* ids;
    size_t size() const { return n; }
    const PreparedObject& operator[](size_t i) const { return base[ids ? ids[i] : i]; }
};
ObjSel select(const PreparedDataset& ds, const PackedHeader& h) {
    return h.ids.empty() ? ObjSel{ds.objects.data() + h.first, h.n_objects, nullptr}
                         : ObjSel{ds.objects.data(), h.n_objects, h.ids.data()};
}

// fn(begin, end) over [0, n) in ~8 contiguous blocks per worker (one pool job per block).
void for_blocks(ThreadPool& pool, size_t n, const std::function<void(size_t, size_t)>& fn) {
    if (n == 0) return;
    const auto ranges = partition_ranges(n, std::max<size_t>(1, size_t{pool.size()} * 8));
    pool.parallel_jobs(ranges.size(), [&](size_t j) { fn(ranges[j].first, ranges[j].second); });
}
template <class T>
T* as(PinnedBuf& b) {
    return reinterpret_cast<T*>(b.data());
}
} // namespace

uint64_t PackedHeader::bytes() const {
    uint64_t b = (mbb.size() + anchor.size() + voxel_box.size() + voxel_anchor.size() + voxel_offsets.size()) * 8;
    for (const auto& v : facet_offsets) b += v.size() * 8;
    for (const auto& v : vert_base) b += v.size() * 8;
    for (const auto& v : facet_base) b += v.size() * 8;
    return b;
}

std::unique_ptr<PackedHeader> pack_header_sel(const PreparedDataset& dsf, std::unique_ptr<PackedHeader> h,
                                              ThreadPool& pool);

std::unique_ptr<PackedHeader> pack_header(const PreparedDataset& ds, ThreadPool& pool) {
    return pack_header(ds, 0, ds.objects.size(), pool);
}

std::unique_ptr<PackedHeader> pack_header(const PreparedDataset& dsf, std::vector<uint32_t> ids, ThreadPool& pool) {
    for (size_t i = 0; i < ids.size(); ++i)
        if (ids[i] >= dsf.objects.size() || (i && ids[i] <= ids[i - 1]))
            throw std::invalid_argument("trijoin: shard object ids must be ascending and in range");
    auto h = std::make_unique<PackedHeader>();
    h->ids = std::move(ids);
    h->n_objects = static_cast<uint32_t>(h->ids.size());
    if (h->ids.empty()) h->first = dsf.objects.size(); // an empty selection
    return pack_header_sel(dsf, std::move(h), pool);
}

std::unique_ptr<PackedHeader> pack_header(const PreparedDataset& dsf, size_t first, size_t last, ThreadPool& pool) {
    auto h = std::make_unique<PackedHeader>();
    h->first = first;
    h->n_objects = static_cast<uint32_t>(last - first);
    return pack_header_sel(dsf, std::move(h), pool);
}

std::unique_ptr<PackedHeader> pack_header_sel(const PreparedDataset& dsf, std::unique_ptr<PackedHeader> h,
                                              ThreadPool& pool) {
    const ObjSel ds = select(dsf, *h);
    const size_t no = ds.size();
    const size_t nl = dsf.lod_schedule.size();
    h->n_objects = static_cast<uint32_t>(no);
    h->levels.assign(dsf.lod_schedule.begin(), dsf.lod_schedule.end());
    h->mbb.resize(6 * no);
    h->anchor.resize(3 * no);
    h->voxel_offsets.resize(no + 1);
    h->voxel_offsets[0] = 0;
    h->vert_base.resize(nl);
    h->facet_base.resize(nl);
    for (size_t li = 0; li < nl; ++li) {
        h->vert_base[li].resize(no + 1);
        h->facet_base[li].resize(no + 1);
        h->vert_base[li][0] = h->facet_base[li][0] = 0;
    }
    // per-object counts in parallel (written at o + 1), then serial prefix sums
    std::atomic<int> bad_levels{0}, bad_pad{0};
    for_blocks(pool, no, [&](size_t b, size_t e) {
        for (size_t o = b; o < e; ++o) {
            const PreparedObject& obj = ds[o];
            if (obj.ladder.levels.size() != nl || obj.voxels.facets_per_level.size() != nl) {
                bad_levels = 1;
                continue;
            }
            h->voxel_offsets[o + 1] = obj.voxels.voxel_count();
            for (size_t li = 0; li < nl; ++li) {
                const LodMesh& lod = obj.ladder.levels[li];
                if (lod.hd.size() < lod.mesh.facets.size() || lod.ph.size() < lod.mesh.facets.size()) bad_pad = 1;
                h->vert_base[li][o + 1] = lod.mesh.vertices.size();
                h->facet_base[li][o + 1] = lod.mesh.facets.size();
            }
        }
    });
    if (bad_levels) throw std::invalid_argument("trijoin: object level count does not match the lod schedule");
    if (bad_pad) throw std::invalid_argument("trijoin: hd / ph shorter than the level's facet list");
    for (size_t o = 0; o < no; ++o) {
        h->voxel_offsets[o + 1] += h->voxel_offsets[o];
        for (size_t li = 0; li < nl; ++li) {
            h->vert_base[li][o + 1] += h->vert_base[li][o];
            h->facet_base[li][o + 1] += h->facet_base[li][o];
        }
    }
    const uint64_t nv = h->voxel_offsets[no];
    for (size_t li = 0; li < nl; ++li) {
        h->n_vertices.push_back(h->vert_base[li][no]);
        h->n_facets.push_back(h->facet_base[li][no]);
        if (h->n_vertices.back() >> 32 || h->n_facets.back() >> 32)
            throw std::invalid_argument("trijoin: more than 2^32 vertices or facets in one level");
    }
    h->voxel_box.resize(6 * nv);
    h->voxel_anchor.resize(3 * nv);
    h->facet_offsets.resize(nl);
    for (size_t li = 0; li < nl; ++li) {
        h->facet_offsets[li].resize(nv + 1);
        h->facet_offsets[li][0] = 0;
    }
    for_blocks(pool, no, [&](size_t b, size_t e) {
        for (size_t o = b; o < e; ++o) {
            const PreparedObject& obj = ds[o];
            const double m[6] = {obj.mbb.min.x, obj.mbb.min.y, obj.mbb.min.z, obj.mbb.max.x, obj.mbb.max.y, obj.mbb.max.z};
            std::memcpy(&h->mbb[6 * o], m, sizeof(m));
            h->anchor[3 * o] = obj.anchor.x;
            h->anchor[3 * o + 1] = obj.anchor.y;
            h->anchor[3 * o + 2] = obj.anchor.z;
            const uint64_t v0 = h->voxel_offsets[o];
            const VoxelSet& vs = obj.voxels;
            for (uint32_t v = 0; v < vs.voxel_count(); ++v) {
                const Aabb& bx = vs.boxes[v];
                const double bb[6] = {bx.min.x, bx.min.y, bx.min.z, bx.max.x, bx.max.y, bx.max.z};
                std::memcpy(&h->voxel_box[6 * (v0 + v)], bb, sizeof(bb));
                h->voxel_anchor[3 * (v0 + v)] = vs.anchors[v].x;
                h->voxel_anchor[3 * (v0 + v) + 1] = vs.anchors[v].y;
                h->voxel_anchor[3 * (v0 + v) + 2] = vs.anchors[v].z;
                for (size_t li = 0; li < nl; ++li)
                    h->facet_offsets[li][v0 + v + 1] = vs.facets_per_level[li][v].size();
            }
        }
    });
    for (size_t li = 0; li < nl; ++li) {
        auto& fo = h->facet_offsets[li];
        for (uint64_t v = 0; v < nv; ++v) fo[v + 1] += fo[v];
    }
    h->fo_ptrs.resize(nl);
    h->vb_ptrs.resize(nl);
    h->fb_ptrs.resize(nl);
    for (size_t li = 0; li < nl; ++li) {
        h->fo_ptrs[li] = h->facet_offsets[li].data();
        h->vb_ptrs[li] = h->vert_base[li].data();
        h->fb_ptrs[li] = h->facet_base[li].data();
    }
    tj_dataset_view& v = h->view;
    v.n_objects = h->n_objects;
    v.n_levels = static_cast<uint32_t>(nl);
    v.levels = h->levels.data();
    v.mbb = h->mbb.data();
    v.anchor = h->anchor.data();
    v.voxel_offsets = h->voxel_offsets.data();
    v.voxel_box = h->voxel_box.data();
    v.voxel_anchor = h->voxel_anchor.data();
    v.facet_offsets = h->fo_ptrs.data();
    v.facets = nullptr;
    return h;
}

// One level in the compact mesh form: per object a straight copy of its vertices, index
// triples, hd / ph and voxel facet-id lists (object-local ids; the device rebases and
// range-checks them, k_expand_level).
std::unique_ptr<PackedLevel> pack_level(const PreparedDataset& dsf, const PackedHeader& h, size_t li, ThreadPool& pool,
                                        size_t pieces,
                                        const std::function<void(const PackedLevel&, const PieceRows&)>& on_piece) {
    auto p = std::make_unique<PackedLevel>();
    const ObjSel ds = select(dsf, h);
    const size_t no = ds.size();
    const uint64_t nvert = h.n_vertices[li], nfac = h.n_facets[li];
    const uint64_t entries = h.facet_offsets[li].back();
    p->verts.resize(std::max<uint64_t>(3 * nvert, 1));
    p->tris.resize(std::max<uint64_t>((3 * nfac + 1) / 2, 1));
    p->hd.resize(std::max<uint64_t>(nfac, 1));
    p->ph.resize(std::max<uint64_t>(nfac, 1));
    p->vf.resize(std::max<uint64_t>((entries + 1) / 2, 1));
    double* verts = p->verts.data();
    uint32_t* tris = as<uint32_t>(p->tris);
    double* hd = p->hd.data();
    double* ph = p->ph.data();
    uint32_t* vf = as<uint32_t>(p->vf);
    // a level whose paddings are all +0.0 (the reference's level 100) ships no hd / ph at all;
    // the test ORs the IEEE bit patterns (branch-free, vectorisable: it reads the whole level
    // when the paddings are zero, so it runs at memory bandwidth)
    std::atomic<bool> nonzero{false}, wide{false};
    for_blocks(pool, no, [&](size_t b, size_t e) {
        bool w = false;
        for (size_t o = b; o < e; ++o) {
            const LodMesh& lod = ds[o].ladder.levels[li];
            const size_t n_f = lod.mesh.facets.size();
            w = w || lod.mesh.vertices.size() >= 0xffff || n_f >= 0xffff;
            if (nonzero.load(std::memory_order_relaxed)) continue;
            uint64_t bits = 0;
            for (size_t f = 0; f < n_f; ++f) bits |= std::bit_cast<uint64_t>(lod.hd[f]) | std::bit_cast<uint64_t>(lod.ph[f]);
            if (bits) nonzero = true;
        }
        if (w) wide = true;
    });
    const bool pads = nonzero.load();
    p->zero_pads = !pads;
    // 16-bit ids when every object of the level has < 65535 vertices and facets: ids are
    // saturated at 0xffff, which is then out of every object's range, so an invalid id still
    // trips the device's range check
    const bool narrow = !wide.load();
    p->narrow = narrow;
    p->bytes = nvert * 24 + nfac * ((narrow ? 6 : 12) + (pads ? 16 : 0)) + entries * (narrow ? 2 : 4);
    uint16_t* tris16 = reinterpret_cast<uint16_t*>(tris);
    uint16_t* vf16 = reinterpret_cast<uint16_t*>(vf);
    static_assert(sizeof(Point3) == 3 * sizeof(double), "Point3 must be three packed doubles");
    static_assert(sizeof(std::array<uint32_t, 3>) == 3 * sizeof(uint32_t), "facets must be packed uint32 triples");
    tj_level_mesh_view& view = p->view;
    view.vertices = verts;
    view.tris = narrow ? nullptr : tris;
    view.hd = pads ? hd : nullptr;
    view.ph = pads ? ph : nullptr;
    view.voxel_facets = narrow ? nullptr : vf;
    view.tris16 = narrow ? tris16 : nullptr;
    view.voxel_facets16 = narrow ? vf16 : nullptr;
    const auto& fo = h.facet_offsets[li];
    pieces = std::max<size_t>(1, std::min(pieces, no));
    for (size_t k = 0; k < pieces; ++k) {
        const size_t lo = no * k / pieces, hi = no * (k + 1) / pieces;
        for_blocks(pool, hi - lo, [&](size_t b, size_t e) {
            for (size_t o = lo + b; o < lo + e; ++o) {
                const PreparedObject& obj = ds[o];
                const LodMesh& lod = obj.ladder.levels[li];
                const uint64_t vb = h.vert_base[li][o], fb = h.facet_base[li][o];
                const size_t n_v = lod.mesh.vertices.size(), n_f = lod.mesh.facets.size();
                if (n_v) std::memcpy(verts + 3 * vb, lod.mesh.vertices.data(), n_v * sizeof(Point3));
                if (n_f) {
                    if (narrow) {
                        const uint32_t* src = lod.mesh.facets.data()->data();
                        uint16_t* dst = tris16 + 3 * fb;
                        for (size_t i = 0; i < 3 * n_f; ++i) dst[i] = static_cast<uint16_t>(std::min<uint32_t>(src[i], 0xffff));
                    } else {
                        std::memcpy(tris + 3 * fb, lod.mesh.facets.data(), n_f * 3 * sizeof(uint32_t));
                    }
                    if (pads) {
                        std::memcpy(hd + fb, lod.hd.data(), n_f * sizeof(double));
                        std::memcpy(ph + fb, lod.ph.data(), n_f * sizeof(double));
                    }
                }
                const VoxelSet& vs = obj.voxels;
                const uint64_t v0 = h.voxel_offsets[o];
                for (uint32_t v = 0; v < vs.voxel_count(); ++v) {
                    const auto& ids = vs.facets_per_level[li][v];
                    if (ids.empty()) continue;
                    if (narrow) {
                        uint16_t* dst = vf16 + fo[v0 + v];
                        for (size_t i = 0; i < ids.size(); ++i) dst[i] = static_cast<uint16_t>(std::min<uint32_t>(ids[i], 0xffff));
                    } else {
                        std::memcpy(vf + fo[v0 + v], ids.data(), ids.size() * sizeof(uint32_t));
                    }
                }
            }
        });
        const PieceRows rows{h.vert_base[li][lo], h.vert_base[li][hi], h.facet_base[li][lo], h.facet_base[li][hi],
                             fo[h.voxel_offsets[lo]], fo[h.voxel_offsets[hi]], (uint32_t)lo, (uint32_t)hi};
        p->pieces.push_back(rows);
        if (on_piece) on_piece(*p, rows);
    }
    return p;
}

} // namespace detail

// ---------------------------------------------------------------- small API functions

std::string stage_name(int16_t code) {
    if (code == stage::kNone) return "undecided";
    if (code == stage::kMbb) return "mbb";
    if (code == stage::kVoxel) return "voxel";
    if (code == 100) return "exact";
    return "lod-" + std::to_string(code);
}

std::string join_type_name(JoinType t) {
    if (t == JoinType::Within) return "within";
    if (t == JoinType::Intersect) return "intersect";
    return "knn";
}

void intersect_interval(Interval& io, double lb, double ub) {
    io.lb = std::max(io.lb, lb);
    io.ub = std::min(io.ub, ub);
    if (!(io.lb > io.ub)) return;
    if (io.lb - io.ub > 1e-9)
        throw EngineError("bound crossing: lb " + std::to_string(io.lb) + " > ub " + std::to_string(io.ub));
    io.lb = io.ub = 0.5 * (io.lb + io.ub);
}

uint64_t CandidateSet::undecided_count() const {
    return static_cast<uint64_t>(std::count(status.begin(), status.end(), PairStatus::Undecided));
}

size_t prune_within(CandidateSet& cands, double tau, int16_t stage_code, std::span<const uint32_t> ops) {
    size_t changed = 0;
    auto one = [&](uint32_t op) {
        if (cands.status[op] != PairStatus::Undecided) return;
        const Interval& iv = cands.intervals[op];
        PairStatus ns = PairStatus::Undecided;
        if (iv.ub <= tau) ns = PairStatus::Confirmed;
        else if (iv.lb > tau) ns = PairStatus::Removed;
        if (ns == PairStatus::Undecided) return;
        cands.status[op] = ns;
        cands.decided_at[op] = stage_code;
        if (ns == PairStatus::Confirmed) ++cands.num_confirmed[cands.pairs[op].first];
        ++changed;
    };
    if (ops.empty()) {
        for (uint32_t op = 0; op < cands.size(); ++op) one(op);
    } else {
        for (uint32_t op : ops) one(op);
    }
    return changed;
}

uint64_t voxel_pair_count(const CandidateSet& cands, uint32_t op, const PreparedDataset& R, const PreparedDataset& S) {
    const auto& [r, s] = cands.pairs[op];
    return uint64_t{R.objects[r].voxels.voxel_count()} * S.objects[s].voxels.voxel_count();
}

void validate(const JoinSpec& spec) {
    if (spec.type == JoinType::Knn) {
        if (spec.k == 0) throw std::invalid_argument("join: k must be >= 1");
    } else {
        if (spec.tau < 0) throw std::invalid_argument("join: tau must be >= 0");
        if (spec.type == JoinType::Intersect && spec.tau != 0.0)
            throw std::invalid_argument("join: intersection requires tau == 0");
    }
    if (spec.filter_chunk == 0) throw std::invalid_argument("join: filter chunk must be >= 1");
    if (spec.refine_chunk == 0) throw std::invalid_argument("join: refine chunk must be >= 1");
    if (spec.lods.empty() || spec.lods.back() != 100) throw std::invalid_argument("join: lod schedule must end at 100");
    for (size_t i = 0; i < spec.lods.size(); ++i) {
        if (spec.lods[i] == 0 || spec.lods[i] > 100) throw std::invalid_argument("join: lod levels must be in (0, 100]");
        if (i > 0 && spec.lods[i] <= spec.lods[i - 1])
            throw std::invalid_argument("join: lod schedule must be ascending");
    }
}

namespace {
std::string g17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}
} // namespace

std::string format_record(const JoinResultRecord& rec, bool knn) {
    std::string s = std::to_string(rec.r) + ' ' + std::to_string(rec.s) + ' ' + g17(rec.lb) + ' ' + g17(rec.ub) + ' ' +
                    stage_name(rec.decided_at);
    if (knn) s += ' ' + std::to_string(rec.rank);
    return s;
}

std::string format_records(std::span<const JoinResultRecord> recs, bool knn) {
    std::string out;
    for (const auto& r : recs) out += format_record(r, knn) + '\n';
    return out;
}

std::string StageStats::to_json() const {
    nlohmann::json j;
    j["query"] = query;
    j["results"] = results;
    j["total_ms"] = total_ms;
    auto arr = nlohmann::json::array();
    for (const StageCounters& s : stages)
        arr.push_back({{"stage", s.name},
                       {"wall_ms", s.wall_ms},
                       {"pairs_in", s.pairs_in},
                       {"confirmed", s.confirmed},
                       {"removed", s.removed},
                       {"pairs_out", s.pairs_out},
                       {"vp_generated", s.vp_generated},
                       {"vp_pruned", s.vp_pruned},
                       {"facet_pairs", s.facet_pairs}});
    j["stages"] = std::move(arr);
    j["b200"] = {{"pack_ms", pack_ms}, {"upload_ms", upload_ms}, {"device_ms", device_ms},
                 {"stream_wait_ms", stream_wait_ms}, {"h2d_bytes", h2d_bytes}, {"devices", devices},
                 {"intervals", decision_mode ? "decision" : "exact"}, {"r_chunks", r_chunks},
                 {"residency", compact ? "compact" : "expanded"}, {"mat_chunks", mat_chunks}};
    nlohmann::json tl = nlohmann::json::object();
    for (const auto& [k, v] : timeline) tl[k] = v;
    j["b200"]["timeline"] = std::move(tl);
    return j.dump(2);
}

size_t aggregate_object_bounds(std::span<const double> vp_lb, std::span<const double> vp_ub,
                               std::span<const uint32_t> vp_op, CandidateSet& cands, int16_t stage_code,
                               const JoinTrace* trace) {
    if (vp_lb.size() != vp_ub.size() || vp_lb.size() != vp_op.size())
        throw std::invalid_argument("aggregate_object_bounds: array size mismatch");
    // per touched op: running minima, then updates in ascending op order
    std::map<uint32_t, std::pair<double, double>> mins;
    for (size_t t = 0; t < vp_op.size(); ++t) {
        auto [it, fresh] = mins.try_emplace(vp_op[t], vp_lb[t], vp_ub[t]);
        if (!fresh) {
            it->second.first = std::min(it->second.first, vp_lb[t]);
            it->second.second = std::min(it->second.second, vp_ub[t]);
        }
    }
    size_t updated = 0;
    for (const auto& [op, m] : mins) {
        if (cands.status[op] != PairStatus::Undecided) continue;
        if (std::isinf(m.first)) continue;
        intersect_interval(cands.intervals[op], m.first, m.second);
        if (trace && trace->on_interval) trace->on_interval(op, stage_code, cands.intervals[op]);
        ++updated;
    }
    return updated;
}

KnnState make_knn_state(const CandidateSet& cands, uint32_t k) {
    if (k == 0) throw std::invalid_argument("make_knn_state: k must be >= 1");
    KnnState st;
    st.k = k;
    st.num_confirmed.assign(cands.r2op_offsets.empty() ? 0 : cands.r2op_offsets.size() - 1, 0);
    for (size_t op = 0; op < cands.size(); ++op)
        if (cands.status[op] == PairStatus::Confirmed) ++st.num_confirmed[cands.pairs[op].first];
    return st;
}

size_t knn_apply_deltas(KnnState& state, CandidateSet& cands, std::span<const KnnDelta> deltas, int16_t stage_code) {
    for (const KnnDelta& d : deltas) {
        if (cands.status[d.op] != PairStatus::Undecided) throw EngineError("knn_apply_deltas: candidate decided twice");
        cands.status[d.op] = d.status;
        cands.decided_at[d.op] = stage_code;
        if (d.status != PairStatus::Confirmed) continue;
        const uint32_t r = cands.pairs[d.op].first;
        ++cands.num_confirmed[r];
        if (++state.num_confirmed[r] > state.k) throw EngineError("knn_apply_deltas: confirmed count exceeds k");
    }
    return deltas.size();
}

// ---------------------------------------------------------------- GPU-backed primitives

void mindist_aabb_batch(std::span<const Aabb> a, std::span<const Aabb> b, std::span<double> out) {
    if (a.size() != b.size() || out.size() != a.size()) throw std::invalid_argument("mindist_aabb_batch: size mismatch");
    tj_ctx* ctx = detail::device_context(detail::join_devices()[0]);
    static_assert(sizeof(Aabb) == 48);
    detail::check(tj_mindist_batch(ctx, a.size(), reinterpret_cast<const double*>(a.data()),
                                   reinterpret_cast<const double*>(b.data()), out.data()),
                  ctx);
}

void tri_tri_distance_batch(std::span<const Triangle> a, std::span<const Triangle> b, std::span<double> out) {
    if (a.size() != b.size() || out.size() != a.size())
        throw std::invalid_argument("tri_tri_distance_batch: size mismatch");
    tj_ctx* ctx = detail::device_context(detail::join_devices()[0]);
    static_assert(sizeof(Triangle) == 72);
    detail::check(tj_tri_tri_batch(ctx, a.size(), reinterpret_cast<const double*>(a.data()),
                                   reinterpret_cast<const double*>(b.data()), out.data()),
                  ctx);
}

double mindist_aabb(const Aabb& a, const Aabb& b) {
    double d = 0;
    mindist_aabb_batch({&a, 1}, {&b, 1}, {&d, 1});
    return d;
}

double tri_tri_distance(const Triangle& t1, const Triangle& t2) {
    double d = 0;
    tri_tri_distance_batch({&t1, 1}, {&t2, 1}, {&d, 1});
    return d;
}

namespace {
double geom_one(int op, const double* a, const double* b) {
    tj_ctx* ctx = detail::device_context(detail::join_devices()[0]);
    double d = 0;
    detail::check(tj_geom_batch(ctx, op, 1, a, b, &d), ctx);
    return d;
}
} // namespace

double point_segment_distance(const Point3& p, const Point3& a, const Point3& b) {
    static_assert(sizeof(Point3) == 24);
    const double seg[6] = {a.x, a.y, a.z, b.x, b.y, b.z};
    return geom_one(TJ_GEOM_POINT_SEGMENT, &p.x, seg);
}

double point_triangle_distance(const Point3& p, const Triangle& t) {
    return geom_one(TJ_GEOM_POINT_TRIANGLE, &p.x, &t.v0.x);
}

double segment_segment_distance(const Point3& a0, const Point3& a1, const Point3& b0, const Point3& b1) {
    const double a[6] = {a0.x, a0.y, a0.z, a1.x, a1.y, a1.z};
    const double b[6] = {b0.x, b0.y, b0.z, b1.x, b1.y, b1.z};
    return geom_one(TJ_GEOM_SEGMENT_SEGMENT, a, b);
}

// ---------------------------------------------------------------- run_oracle (GPU exhaustive join)

namespace {
// Level-100 triangles of every object (the OracleTree input, reference src/oracle.cpp:29-33).
struct MeshSetPack {
    std::vector<uint64_t> off;
    std::vector<double> tris;
    tj_mesh_set_view view{};
    explicit MeshSetPack(const PreparedDataset& ds) {
        off.assign(ds.objects.size() + 1, 0);
        for (size_t o = 0; o < ds.objects.size(); ++o) {
            const auto& lv = ds.objects[o].ladder.levels;
            off[o + 1] = off[o] + (lv.empty() ? 0 : lv.back().mesh.facets.size());
        }
        tris.resize(9 * off.back());
        for (size_t o = 0; o < ds.objects.size(); ++o) {
            const auto& lv = ds.objects[o].ladder.levels;
            if (lv.empty()) continue;
            const Mesh& m = lv.back().mesh;
            double* w = tris.data() + 9 * off[o];
            for (size_t f = 0; f < m.facets.size(); ++f) {
                for (int c = 0; c < 3; ++c) {
                    const uint32_t vi = m.facets[f][c];
                    if (vi >= m.vertices.size()) throw std::invalid_argument("run_oracle: facet vertex out of range");
                    const Point3& v = m.vertices[vi];
                    w[9 * f + 3 * c] = v.x;
                    w[9 * f + 3 * c + 1] = v.y;
                    w[9 * f + 3 * c + 2] = v.z;
                }
            }
        }
        view.n_objects = static_cast<uint32_t>(ds.objects.size());
        view.tri_offsets = off.data();
        view.tris = tris.data();
    }
};
} // namespace

JoinOutput run_oracle(const PreparedDataset& R, const PreparedDataset& S, const JoinSpec& spec, ThreadPool& pool) {
    (void)pool; // the work runs on the GPU
    validate(spec);
    const auto t0 = std::chrono::steady_clock::now();
    const MeshSetPack r(R);
    std::unique_ptr<MeshSetPack> s_store;
    const tj_mesh_set_view* sv = nullptr; // self-join: the same dataset object
    if (&S != &R) {
        s_store = std::make_unique<MeshSetPack>(S);
        sv = &s_store->view;
    }
    const int32_t type = spec.type == JoinType::Knn ? TJ_KNN : spec.type == JoinType::Intersect ? TJ_INTERSECT
                                                                                                   : TJ_WITHIN;
    tj_ctx* ctx = detail::device_context(detail::join_devices()[0]);
    tj_exhaustive_result res{};
    detail::check(tj_exhaustive_join(ctx, &r.view, sv, type, spec.type == JoinType::Within ? spec.tau : 0.0, spec.k,
                                     &res),
                  ctx);
    JoinOutput out;
    out.records.reserve(res.n_records);
    for (uint64_t x = 0; x < res.n_records; ++x)
        out.records.push_back({res.r[x], res.s[x], res.d[x], res.d[x], 100, res.rank[x]});
    tj_exhaustive_result_free(&res);
    const uint64_t all_pairs = static_cast<uint64_t>(R.objects.size()) * static_cast<uint64_t>(S.objects.size());
    out.stats.query = join_type_name(spec.type);
    out.stats.results = out.records.size();
    out.stats.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    StageCounters sc;
    sc.name = "exhaustive";
    sc.wall_ms = out.stats.total_ms;
    sc.pairs_in = all_pairs;
    sc.confirmed = out.records.size();
    sc.removed = all_pairs - out.records.size();
    sc.pairs_out = 0;
    out.stats.stages.push_back(sc);
    return out;
}

VoxelPairBatch gather_facet_data(std::span<const ActiveVp> slice, uint32_t level, const PreparedDataset& R,
                                 const PreparedDataset& S, const CandidateSet& cands) {
    auto slot = [&](const PreparedDataset& d) {
        for (size_t i = 0; i < d.lod_schedule.size(); ++i)
            if (d.lod_schedule[i] == static_cast<int>(level)) return i;
        throw EngineError("refine: level " + std::to_string(level) + " is not in the dataset's lod schedule");
    };
    const size_t lr = slot(R), ls = slot(S);
    VoxelPairBatch batch;
    batch.descs.reserve(slice.size());
    std::map<uint64_t, std::pair<uint64_t, uint32_t>> seen_r, seen_s;
    auto segment = [&](const PreparedObject& obj, uint32_t obj_idx, size_t li, uint32_t voxel,
                       std::map<uint64_t, std::pair<uint64_t, uint32_t>>& seen) {
        const uint64_t key = (uint64_t{obj_idx} << 32) | voxel;
        if (auto it = seen.find(key); it != seen.end()) return it->second;
        const LodMesh& lod = obj.ladder.levels[li];
        const auto& ids = obj.voxels.facets_per_level[li][voxel];
        const std::pair<uint64_t, uint32_t> seg{batch.tris.size(), static_cast<uint32_t>(ids.size())};
        for (uint32_t f : ids) {
            batch.tris.push_back(lod.mesh.triangle(f));
            batch.hd.push_back(lod.hd[f]);
            batch.ph.push_back(lod.ph[f]);
        }
        seen.emplace(key, seg);
        return seg;
    };
    for (const ActiveVp& a : slice) {
        const auto [r, s] = cands.pairs[a.op];
        const auto sr = segment(R.objects[r], r, lr, a.vr, seen_r);
        const auto ss = segment(S.objects[s], s, ls, a.vs, seen_s);
        batch.descs.push_back({sr.first, ss.first, sr.second, ss.second, a.op});
    }
    return batch;
}

void refine_kernel(const VoxelPairBatch& batch, ThreadPool&, std::vector<double>& vp_lb, std::vector<double>& vp_ub) {
    const size_t n = batch.descs.size();
    vp_lb.assign(n, std::numeric_limits<double>::infinity());
    vp_ub.assign(n, std::numeric_limits<double>::infinity());
    if (n == 0) return;
    std::vector<uint64_t> ro(n), so(n);
    std::vector<uint32_t> rl(n), sl(n);
    for (size_t d = 0; d < n; ++d) {
        ro[d] = batch.descs[d].r_off;
        so[d] = batch.descs[d].s_off;
        rl[d] = batch.descs[d].r_len;
        sl[d] = batch.descs[d].s_len;
    }
    tj_ctx* ctx = detail::device_context(detail::join_devices()[0]);
    detail::check(tj_refine_batch(ctx, batch.tris.size(), reinterpret_cast<const double*>(batch.tris.data()),
                                  batch.hd.data(), batch.ph.data(), n, ro.data(), so.data(), rl.data(), sl.data(), 0,
                                  vp_lb.data(), vp_ub.data()),
                  ctx);
}

// ---------------------------------------------------------------- run_join

namespace {

struct TraceBridge {
    const JoinTrace* t;
    static void interval(void* u, uint32_t op, int16_t st, double lb, double ub) {
        const auto* self = static_cast<TraceBridge*>(u);
        if (self->t->on_interval) self->t->on_interval(op, st, Interval{lb, ub});
    }
    static void pruned(void* u, uint32_t op, uint32_t vr, uint32_t vs, double lb, double ub) {
        const auto* self = static_cast<TraceBridge*>(u);
        if (self->t->on_vp_pruned) self->t->on_vp_pruned(op, vr, vs, lb, ub);
    }
};

// Candidate set + counters of one join, merged over shards.
struct Merged {
    CandidateSet cands;
    uint64_t vp_generated = 0, vp_pruned = 0;
    double mbb_ms = 0, voxel_ms = 0;
    std::map<uint32_t, RefineLevelStats> levels;
};

tj_join_spec to_c_spec(const JoinSpec& spec) {
    tj_join_spec c{};
    c.type = spec.type == JoinType::Within ? TJ_WITHIN : spec.type == JoinType::Intersect ? TJ_INTERSECT : TJ_KNN;
    c.tau = spec.tau;
    c.k = spec.k;
    c.filter_chunk = spec.filter_chunk;
    c.refine_chunk = spec.refine_chunk;
    c.n_lods = static_cast<uint32_t>(spec.lods.size());
    c.lods = spec.lods.data();
    c.pipeline = spec.pipeline ? 1 : 0;
    c.flags = 0;
    if (spec.exact) c.flags |= TJ_FLAG_EXACT_RECOMPUTE;
    if (const char* e = std::getenv("TRIJOIN_NO_CULL"); e && *e && *e != '0') c.flags |= TJ_FLAG_NO_CULL;
    if (const char* e = std::getenv("TRIJOIN_EXACT_INTERVALS"); e && *e && *e != '0') c.flags |= TJ_FLAG_EXACT_INTERVALS;
    return c;
}

// One part of a join's device results: n queries whose global ids are ids[0, n) (or
// r_base + [0, n) when ids is null): one R chunk of one GPU's query shard.
struct Piece {
    const tj_join_result* res;
    uint32_t r_base;
    const uint32_t* ids;
    uint32_t n;
};

int slot_of(const PreparedDataset& d, uint32_t level) {
    for (size_t i = 0; i < d.lod_schedule.size(); ++i)
        if (d.lod_schedule[i] == static_cast<int>(level)) return static_cast<int>(i);
    return -1;
}

// ---- out-of-core R: the device-memory budget ----
// Device bytes one object costs while resident: object + voxel records, the 96-B facet
// records of every level, the compact staging of its largest level and its share of the
// per-level screening workspace (128-B records + 48-B voxel aggregates).
uint64_t object_device_bytes(const PreparedObject& o) {
    uint64_t all = 0, mx = 0; // the level meshes' facet counts (the voxel lists partition them)
    for (const auto& lv : o.ladder.levels) {
        const uint64_t e = lv.mesh.facets.size();
        all += e;
        mx = std::max(mx, e);
    }
    const uint64_t nv = o.voxels.voxel_count();
    return 256 + 112 * nv + 96 * all + (44 + 176) * mx;
}

// Device bytes of one object in the compact-resident form (TJ_DATASET_COMPACT): object +
// voxel records, the per-level voxel CSR, and every level's compact mesh form (vertices,
// index triples, hd / ph, voxel facet-id lists), as tj_dataset_begin_ex reserves them.
uint64_t object_compact_bytes(const PreparedObject& o) {
    const uint64_t nv = o.voxels.voxel_count();
    uint64_t b = 256 + 112 * nv;
    for (const auto& lv : o.ladder.levels)
        b += 8 * nv + 24 * lv.mesh.vertices.size() + (12 + 16 + 4) * lv.mesh.facets.size();
    return b;
}

// Device-memory budget: $TRIJOIN_DEVICE_BUDGET_MB, else 90 % of the device's memory less a
// 2 GiB reserve (0 = unknown). The device's total, not its free memory: this library's memory
// is pooled (freed blocks stay reserved for its next allocations), so the free figure
// understates what a join can use. Queried once per device and process.
uint64_t device_budget(int device) {
    if (const char* e = std::getenv("TRIJOIN_DEVICE_BUDGET_MB"); e && *e) return std::stoull(e) << 20;
    static std::mutex mu;
    static std::map<int, uint64_t> cache;
    std::lock_guard<std::mutex> lk(mu);
    if (auto it = cache.find(device); it != cache.end()) return it->second;
    size_t free_b = 0, total_b = 0;
    if (cudaSetDevice(device) != cudaSuccess || cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    const uint64_t reserve = 2ull << 30;
    return cache[device] = total_b / 10 * 9 > reserve ? total_b / 10 * 9 - reserve : total_b / 2;
}

// One GPU's share of a join: a query shard (ids ascending; empty = all of R) split into R
// chunks (ranges into the shard) so that S and the chunk being joined fit the budget:
// $TRIJOIN_DEVICE_BUDGET_MB, else 90 % of the device's free memory (shared by the contexts
// of one device). $TRIJOIN_R_CHUNK_OBJECTS forces a chunk size.
struct GpuShare {
    int device = 0, slot = 0;
    std::vector<uint32_t> ids;
    bool all = true;
    std::vector<std::pair<size_t, size_t>> chunks;
    size_t size(size_t nr) const { return all ? nr : ids.size(); }
};

// Device footprints of a dataset: expanded (records + screening data at upload) and compact.
struct Footprint {
    uint64_t expanded = 0, compact = 0;
};
Footprint dataset_footprint(const PreparedDataset& D, ThreadPool& pool) {
    std::atomic<uint64_t> e{0}, c{0};
    detail::for_blocks(pool, D.objects.size(), [&](size_t b, size_t en) {
        uint64_t ae = 0, ac = 0;
        for (size_t o = b; o < en; ++o) {
            ae += object_device_bytes(D.objects[o]);
            ac += object_compact_bytes(D.objects[o]);
        }
        e += ae;
        c += ac;
    });
    return {e.load(), c.load()};
}

// Share of the device budget the compact-resident datasets may take: the rest is the working
// set in which each level's active voxels are expanded (chunked on the device to fit it).
constexpr double kCompactShare = 0.6;

// $TRIJOIN_COMPACT: 1 forces compact-resident datasets, 0 forbids them, unset = by budget.
int compact_override() {
    const char* e = std::getenv("TRIJOIN_COMPACT");
    return e && *e ? (*e == '0' ? 0 : 1) : -1;
}

// Plans one GPU's R chunks and chooses the residency mode: expanded when R and S fit the
// budget expanded, else compact-resident (R chunked only if even that does not fit).
void plan_r_chunks(GpuShare& w, const PreparedDataset& R, const Footprint& s_fp, size_t contexts_on_device,
                   bool shares_s, bool& compact, ThreadPool& pool) {
    const size_t n = w.size(R.objects.size());
    w.chunks.clear();
    std::vector<uint64_t> cost_e(n), cost_c(n);
    std::atomic<uint64_t> e_sum{0}, c_sum{0};
    detail::for_blocks(pool, n, [&](size_t b, size_t e) {
        uint64_t ae = 0, ac = 0;
        for (size_t i = b; i < e; ++i) {
            const PreparedObject& o = R.objects[w.all ? i : w.ids[i]];
            ae += cost_e[i] = object_device_bytes(o);
            ac += cost_c[i] = object_compact_bytes(o);
        }
        e_sum += ae;
        c_sum += ac;
    });
    uint64_t budget = device_budget(w.device) / std::max<size_t>(1, contexts_on_device);
    const uint64_t fixed = (64ull << 20) + 256 * uint64_t{n};
    // shares_s: a self-join of all of R in one chunk is one device dataset (R = S)
    const uint64_t r_e = shares_s ? 0 : e_sum.load(), r_c = shares_s ? 0 : c_sum.load();
    const int forced = compact_override();
    if (forced >= 0) compact = forced == 1;
    else compact = budget && r_e + s_fp.expanded + fixed > budget;
    if (const char* e = std::getenv("TRIJOIN_R_CHUNK_OBJECTS"); e && *e) {
        const size_t step = std::max<size_t>(1, std::stoull(e));
        for (size_t a = 0; a < n; a += step) w.chunks.emplace_back(a, std::min(n, a + step));
        if (w.chunks.empty()) w.chunks.emplace_back(0, 0);
        return;
    }
    if (budget == 0) {
        w.chunks.emplace_back(0, n);
        return;
    }
    const std::vector<uint64_t>& cost = compact ? cost_c : cost_e;
    const uint64_t s_total = compact ? s_fp.compact : s_fp.expanded;
    // compact: the datasets may take kCompactShare of what is left after the fixed part
    if (compact) budget = budget > fixed ? fixed + uint64_t(double(budget - fixed) * kCompactShare) : budget;
    if ((compact ? r_c : r_e) + s_total + fixed <= budget) {
        w.chunks.emplace_back(0, n);
        return;
    }
    // chunked: S in full + one R chunk joining (the next one is packed on the host meanwhile)
    if (s_total + fixed >= budget) throw std::runtime_error("trijoin: S does not fit the device-memory budget");
    const uint64_t per_chunk = budget - s_total - fixed;
    size_t a = 0;
    uint64_t acc = 0;
    for (size_t i = 0; i < n; ++i) {
        if (cost[i] > per_chunk) throw std::runtime_error("trijoin: one R object exceeds the device-memory budget");
        if (acc + cost[i] > per_chunk) {
            w.chunks.emplace_back(a, i);
            a = i;
            acc = 0;
        }
        acc += cost[i];
    }
    w.chunks.emplace_back(a, n);
}


// A packed set for one object selection of a dataset: from the caller's cache (kept for later
// joins of the same immutable dataset) or fresh (freed after the join).
struct SetLease {
    std::shared_ptr<detail::PackedSet> set;
    detail::JoinCache* cache = nullptr;
    std::string key;
    SetLease() = default;
    SetLease(const SetLease&) = delete;
    SetLease& operator=(const SetLease&) = delete;
    ~SetLease() {
        if (cache && set) cache->give_back(key, std::move(set));
    }
};

void lease(SetLease& l, detail::JoinCache* cache, const std::string& key) {
    if (cache) {
        l.set = cache->take(key);
        if (l.set) {
            l.cache = cache;
            l.key = key;
            return;
        }
    }
    l.set = std::make_shared<detail::PackedSet>();
}

// Ships level slot `slot` of set (packing it first, in pieces that are shipped while the next
// is packed, unless the set already holds it) to every dataset handle in dst.
// $TRIJOIN_COPY_ORDER=0: R's and S's level copies unordered (each dataset's copy stream on its
// own). Ordered (default), each GPU's link carries S20 R20 S60 R60 ... (tj_dataset_copy_after).
bool copy_order() {
    const char* e = std::getenv("TRIJOIN_COPY_ORDER");
    return !(e && *e == '0');
}

// R's join levels after the first ship in object-range pieces, each after S's same level, and
// the join refines each piece's queries as it lands, with R's running level aggregates
// (TRIJOIN_PIECED=1: the last level only, 0: whole levels). With the expansions off the copy
// stream (LevelGate::expand) the pieces land at link speed while the previous level is still
// being refined: config B e2e 93.8 (whole) -> 90.4 (last level) -> 86.1 ms (every level after
// the first; TRIJOIN_DEBUG_TIMELINE copy / refine timelines). Results are identical in every
// mode (tests/test_gpu_join.py).
// $TRIJOIN_PIECED_S=0: S's levels expanded whole after their last copy
bool s_pieces() {
    const char* e = std::getenv("TRIJOIN_PIECED_S");
    return !(e && *e == '0');
}

int pieced_mode() { // 0: whole levels, 1: the last join level pieced, 2 (default): every level after the first
    const char* e = std::getenv("TRIJOIN_PIECED");
    if (!e || !*e) return 2;
    return *e == '0' ? 0 : *e == '1' ? 1 : 2;
}

uint32_t level_flags(const detail::PackedLevel& l) {
    return (l.zero_pads ? 0u : TJ_LEVEL_PADS) | (l.narrow ? TJ_LEVEL_NARROW : 0u);
}

// pieced: the level is finished piece by piece (tj_dataset_finish_level_part after each piece's
// rows), so a join refines a piece's queries while later pieces are in flight.
void feed_level(const PreparedDataset& D, detail::PackedSet& set, size_t slot, const std::vector<tj_dataset*>& dst,
                const std::vector<tj_ctx*>& ctxs, ThreadPool& pool, JoinOutput& out, double& pack_ms,
                std::mutex* stat_mu, bool pieced = false) {
    using Clock = std::chrono::steady_clock;
    if (set.levels.size() < D.lod_schedule.size()) set.levels.resize(D.lod_schedule.size());
    auto& lv = set.levels[slot];
    if (!lv) {
        const auto t0 = Clock::now();
        auto ship = [&](const detail::PackedLevel& l, const detail::PieceRows& rows) {
            for (size_t g = 0; g < dst.size(); ++g) {
                detail::check(tj_dataset_put_level_part(dst[g], static_cast<uint32_t>(slot), &l.view, rows.vert_begin,
                                                        rows.vert_end, rows.facet_begin, rows.facet_end,
                                                        rows.entry_begin, rows.entry_end),
                              ctxs[g]);
                if (pieced)
                    detail::check(tj_dataset_finish_level_part(dst[g], static_cast<uint32_t>(slot), rows.obj_begin,
                                                               rows.obj_end, level_flags(l)),
                                  ctxs[g]);
            }
        };
        lv = detail::pack_level(D, *set.h, slot, pool, kPackPieces, ship);
        const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        std::unique_lock<std::mutex> lk;
        if (stat_mu) lk = std::unique_lock<std::mutex>(*stat_mu);
        pack_ms += ms;
    } else if (pieced) {
        for (const detail::PieceRows& rows : lv->pieces)
            for (size_t g = 0; g < dst.size(); ++g) {
                detail::check(tj_dataset_put_level_part(dst[g], static_cast<uint32_t>(slot), &lv->view, rows.vert_begin,
                                                        rows.vert_end, rows.facet_begin, rows.facet_end,
                                                        rows.entry_begin, rows.entry_end),
                              ctxs[g]);
                detail::check(tj_dataset_finish_level_part(dst[g], static_cast<uint32_t>(slot), rows.obj_begin,
                                                           rows.obj_end, level_flags(*lv)),
                              ctxs[g]);
            }
    } else {
        const uint64_t nv = set.h->n_vertices[slot], nf = set.h->n_facets[slot];
        const uint64_t ne = set.h->facet_offsets[slot].back();
        for (size_t g = 0; g < dst.size(); ++g)
            detail::check(tj_dataset_put_level_part(dst[g], static_cast<uint32_t>(slot), &lv->view, 0, nv, 0, nf, 0, ne),
                          ctxs[g]);
    }
    const uint32_t flags = level_flags(*lv) | (pieced ? TJ_LEVEL_PIECES : 0u);
    for (size_t g = 0; g < dst.size(); ++g)
        detail::check(tj_dataset_finish_level(dst[g], static_cast<uint32_t>(slot), flags), ctxs[g]);
    std::unique_lock<std::mutex> lk;
    if (stat_mu) lk = std::unique_lock<std::mutex>(*stat_mu);
    out.stats.h2d_bytes += dst.size() * lv->bytes;
}

// Marks every level slot of ds not yet shipped as failed (a join waiting for it returns).
void release_levels(tj_dataset* ds, const std::vector<char>& put) {
    for (size_t i = 0; i < put.size(); ++i)
        if (!put[i]) tj_dataset_put_level(ds, static_cast<uint32_t>(i), nullptr);
}

} // namespace

JoinOutput run_join(const PreparedDataset& R, const PreparedDataset& S, const JoinSpec& spec, ThreadPool& pool,
                    const JoinTrace* trace) {
    pool.parallel_jobs(0, [](size_t) {}); // $TRIJOIN_POOL_CHECK: the caller's pool is intact
    JoinOutput out = detail::run_join_cached(R, S, spec, pool, trace, nullptr, nullptr);
    pool.parallel_jobs(0, [](size_t) {});
    return out;
}

JoinOutput detail::run_join_cached(const PreparedDataset& R, const PreparedDataset& S, const JoinSpec& spec,
                                   ThreadPool& pool, const JoinTrace* trace, JoinCache* r_cache, JoinCache* s_cache) {
    using Clock = std::chrono::steady_clock;
    validate(spec);
    const bool knn = spec.type == JoinType::Knn;
    const auto t_total = Clock::now();
    JoinOutput out;
    out.stats.query = join_type_name(spec.type);
    std::mutex stat_mu;
    auto mark = [&](const std::string& what) {
        std::lock_guard<std::mutex> lk(stat_mu);
        out.stats.timeline.emplace_back(what, std::chrono::duration<double, std::milli>(Clock::now() - t_total).count());
    };

    mark("entered");
    const std::vector<int> devices = detail::join_devices();
    const bool self_join = &R == &S;
    const bool tracing = trace && (trace->on_interval || trace->on_vp_pruned);
    const size_t G = tracing ? 1 : devices.size();
    out.stats.devices = static_cast<uint32_t>(G);
    const size_t nr = R.objects.size();

    // Query shards: query r belongs to shard (r / block) % Q, Q = processes x GPUs.
    // $TRIJOIN_PROCESS_SHARD = "i/n" (one process per GPU, e.g. torchrun): this process joins
    // shards i*G .. i*G+G-1 only, and its records and counters cover those queries only.
    size_t proc_i = 0, proc_n = 1;
    if (const char* e = std::getenv("TRIJOIN_PROCESS_SHARD"); e && *e && !tracing) {
        const std::string v(e);
        const size_t slash = v.find('/');
        if (slash == std::string::npos) throw std::invalid_argument("TRIJOIN_PROCESS_SHARD must be i/n");
        proc_i = std::stoull(v.substr(0, slash));
        proc_n = std::max<size_t>(1, std::stoull(v.substr(slash + 1)));
        if (proc_i >= proc_n) throw std::invalid_argument("TRIJOIN_PROCESS_SHARD: i must be < n");
    }
    uint32_t block = 1024; // queries per shard block ($TRIJOIN_SHARD_BLOCK for tests)
    if (const char* e = std::getenv("TRIJOIN_SHARD_BLOCK"); e && *e) block = std::max<uint32_t>(1, std::stoul(e));
    const size_t Q = proc_n * G;
    std::vector<GpuShare> share(G);
    std::map<int, size_t> per_device;
    for (size_t g = 0; g < G; ++g) {
        share[g].device = devices[g];
        share[g].slot = static_cast<int>(per_device[devices[g]]++); // own context per listed slot
        if (Q > 1) {
            share[g].all = false;
            const size_t q = proc_i * G + g;
            for (size_t b0 = q * size_t{block}; b0 < nr; b0 += Q * size_t{block})
                for (size_t r = b0; r < std::min(nr, b0 + block); ++r) share[g].ids.push_back(static_cast<uint32_t>(r));
        }
    }
    // S stays resident on every GPU for the whole join; R goes in chunks if it does not fit.
    // Datasets are compact-resident (levels expanded on demand) when the expanded form would
    // not fit.
    const Footprint s_fp = tracing ? Footprint{} : dataset_footprint(S, pool);
    bool compact = false;
    for (size_t g = 0; g < G; ++g) {
        bool c = false;
        if (tracing) share[g].chunks = {{0, share[g].size(nr)}};
        else plan_r_chunks(share[g], R, s_fp, per_device[share[g].device], self_join && G == 1 && Q == 1, c, pool);
        compact = compact || c;
    }
    if (tracing && compact_override() == 1) compact = true;
    const uint32_t ds_flags = compact ? TJ_DATASET_COMPACT : 0u;
    out.stats.compact = compact;
    // one GPU, all of R in one chunk, self-join: R and S are one device dataset
    const bool one_dataset = self_join && G == 1 && Q == 1 && share[0].chunks.size() == 1;
    uint32_t n_chunks = 0;
    for (const auto& w : share) n_chunks += static_cast<uint32_t>(w.chunks.size());
    out.stats.r_chunks = n_chunks;
    mark("planned");

    const detail::ArenaStats arena0 = detail::arena_stats();
    std::vector<tj_ctx*> ctxs(G);
    for (size_t g = 0; g < G; ++g) ctxs[g] = detail::device_context(share[g].device, share[g].slot);

    // ---- S: header + levels packed once (or taken from the cache), streamed to every GPU
    double pack_ms = 0.0;
    SetLease s_lease;
    std::vector<detail::DatasetHandle> dsh(G);
    std::vector<std::vector<char>> put_s(G, std::vector<char>(S.lod_schedule.size(), 0));
    // S's datasets are begun by the main thread while the workers begin their R datasets and
    // start streaming R's levels; a worker waits for S only to start its join
    std::mutex s_mu;
    std::condition_variable s_cv;
    bool s_begun = false, s_failed = false;
    auto wait_s_begun = [&] {
        std::unique_lock<std::mutex> lk(s_mu);
        s_cv.wait(lk, [&] { return s_begun; });
        if (s_failed) throw std::runtime_error("trijoin: S upload failed");
    };
    // Copy order over each GPU's host link, join level by join level: S20 R20 S60 R60 ... (the
    // workers register it on their first chunk; the main thread feeds S's levels once every
    // worker has registered or given up)
    const bool ordered = copy_order() && !one_dataset;
    size_t ord_n = 0;
    std::vector<char> ord_in(G, 0);
    auto ord_arrive = [&](size_t g) { // once per worker, on every path
        {
            std::lock_guard<std::mutex> lk(s_mu);
            if (ord_in[g]) return;
            ord_in[g] = 1;
            ++ord_n;
        }
        s_cv.notify_all();
    };

    // ---- per GPU: its R chunks in order; each chunk's levels are packed (or taken from the
    // cache) and streamed while its join runs, coarsest level first
    std::vector<std::vector<std::unique_ptr<detail::ResultHandle>>> results(G);
    std::vector<std::vector<std::unique_ptr<SetLease>>> r_sets(G); // chunk id lists live until the merge
    std::vector<std::exception_ptr> errors(G);
    std::vector<double> dev_ms(G, 0.0);
    auto worker = [&](size_t g) {
        GpuShare& w = share[g];
        tj_ctx* ctx = ctxs[g];
        try {
            for (size_t k = 0; k < w.chunks.size(); ++k) {
                const auto [a, b] = w.chunks[k];
                auto lz = std::make_unique<SetLease>();
                const std::string key = (w.all ? std::string("all") : std::to_string(proc_i * G + g) + "/" +
                                                                          std::to_string(Q) + "/" + std::to_string(block)) +
                                        ":" + std::to_string(a) + "-" + std::to_string(b);
                lease(*lz, r_cache, key);
                if (!lz->set->h) {
                    const auto tp = Clock::now();
                    if (w.all)
                        lz->set->h = detail::pack_header(R, a, b, pool);
                    else
                        lz->set->h = detail::pack_header(
                            R, std::vector<uint32_t>(w.ids.begin() + a, w.ids.begin() + b), pool);
                    std::lock_guard<std::mutex> lk(stat_mu);
                    pack_ms += std::chrono::duration<double, std::milli>(Clock::now() - tp).count();
                }
                const detail::PackedHeader& hr = *lz->set->h;
                detail::DatasetHandle dr;
                if (G == 1 && w.chunks.size() == 1) mark("R_begin");
                detail::check(tj_dataset_begin_ex(ctx, &hr.view, hr.vb_ptrs.data(), hr.fb_ptrs.data(), ds_flags, &dr.p),
                              ctx);
                if (G == 1 && w.chunks.size() == 1) mark("R_begun");
                {
                    std::lock_guard<std::mutex> lk(stat_mu);
                    out.stats.h2d_bytes += hr.bytes();
                }
                results[g].push_back(std::make_unique<detail::ResultHandle>());
                detail::ResultHandle* res = results[g].back().get();
                // the last join level of R in object-range pieces, after S's whole last level: the
                // join refines each piece's queries while the later pieces are still in flight
                // R's pieced levels: the last join level, or (TRIJOIN_PIECED=2) every join level
                // after the first; each ships after S's same level
                std::vector<char> pieced_slot(R.lod_schedule.size(), 0);
                const int pmode = pieced_mode();
                if (pmode && !one_dataset && !compact)
                    for (size_t li = pmode == 2 ? 1 : spec.lods.size() - 1; li < spec.lods.size(); ++li) {
                        const int rs = slot_of(R, spec.lods[li]), ss = slot_of(S, spec.lods[li]);
                        if (rs < 0 || ss < 0) continue;
                        pieced_slot[rs] = 1;
                        detail::check(tj_dataset_set_pieced(dr.p, static_cast<uint32_t>(rs)), ctx);
                    }
                std::exception_ptr je;
                const auto td = Clock::now();
                if (!one_dataset) {
                    try {
                        wait_s_begun();
                        if (ordered && k == 0) {
                            for (size_t li = 0; li < spec.lods.size(); ++li) {
                                const int rs = slot_of(R, spec.lods[li]), ss = slot_of(S, spec.lods[li]);
                                if (rs < 0 || ss < 0) break;
                                detail::check(tj_dataset_copy_after(dr.p, static_cast<uint32_t>(rs), dsh[g].p,
                                                                    static_cast<uint32_t>(ss)),
                                              ctx);
                                if (li + 1 >= spec.lods.size()) break;
                                const int sn = slot_of(S, spec.lods[li + 1]);
                                if (sn < 0) break;
                                detail::check(tj_dataset_copy_after(dsh[g].p, static_cast<uint32_t>(sn), dr.p,
                                                                    static_cast<uint32_t>(rs)),
                                              ctx);
                            }
                        }
                    } catch (...) {
                        ord_arrive(g);
                        throw;
                    }
                    ord_arrive(g);
                }
                std::thread jt([&] {
                    try {
                        tj_join_spec cs = to_c_spec(spec);
                        TraceBridge bridge{trace};
                        tj_trace tt{&bridge, &TraceBridge::interval, &TraceBridge::pruned};
                        detail::check(tj_join(ctx, dr.p, one_dataset ? dr.p : dsh[g].p, &cs, trace ? &tt : nullptr,
                                              &res->r),
                                      ctx);
                    } catch (...) {
                        je = std::current_exception();
                    }
                });
                std::vector<char> put(R.lod_schedule.size(), 0);
                std::exception_ptr pe;
                try {
                    for (uint32_t level : spec.lods) {
                        const int slot = slot_of(R, level);
                        if (slot < 0) continue; // the join reports the missing level
                        const bool pc = pieced_slot[slot] != 0;
                        // (with the copy order registered the device orders R's pieces after S's level)
                        if (pc && !(ordered && k == 0))
                            detail::check(tj_dataset_level_wait(dsh[g].p, static_cast<uint32_t>(slot_of(S, level))),
                                          ctxs[g]);
                        feed_level(R, *lz->set, static_cast<size_t>(slot), {dr.p}, {ctx}, pool, out, pack_ms,
                                   &stat_mu, pc);
                        put[slot] = 1;
                        if (G == 1 && w.chunks.size() == 1)
                            mark(std::string("R_lod") + std::to_string(level) + "_put");
                    }
                } catch (...) {
                    pe = std::current_exception();
                    release_levels(dr.p, put);
                }
                jt.join();
                tj_dataset_sync(dr.p);
                dev_ms[g] += std::chrono::duration<double, std::milli>(Clock::now() - td).count();
                r_sets[g].push_back(std::move(lz));
                if (pe) std::rethrow_exception(pe);
                if (je) std::rethrow_exception(je);
            }
        } catch (...) {
            errors[g] = std::current_exception();
        }
        ord_arrive(g);
    };
    std::vector<std::thread> workers;
    for (size_t g = 0; g < G; ++g) workers.emplace_back(worker, g);

    std::exception_ptr s_begin_error;
    try {
        const auto tu = Clock::now();
        if (!one_dataset) {
            lease(s_lease, s_cache, "all");
            if (!s_lease.set->h) {
                const auto tp = Clock::now();
                s_lease.set->h = detail::pack_header(S, pool);
                std::lock_guard<std::mutex> lk(stat_mu); // the workers update the same tallies
                pack_ms += std::chrono::duration<double, std::milli>(Clock::now() - tp).count();
            }
            const detail::PackedHeader& hs = *s_lease.set->h;
            for (size_t g = 0; g < G; ++g) {
                detail::check(
                    tj_dataset_begin_ex(ctxs[g], &hs.view, hs.vb_ptrs.data(), hs.fb_ptrs.data(), ds_flags, &dsh[g].p),
                    ctxs[g]);
                std::lock_guard<std::mutex> lk(stat_mu);
                out.stats.h2d_bytes += hs.bytes();
            }
        }
        out.stats.upload_ms = std::chrono::duration<double, std::milli>(Clock::now() - tu).count();
        mark("S_begun");
    } catch (...) {
        s_begin_error = std::current_exception();
    }
    {
        std::lock_guard<std::mutex> lk(s_mu);
        s_begun = true;
        s_failed = s_begin_error != nullptr;
    }
    s_cv.notify_all();
    if (s_begin_error) {
        for (auto& t : workers) t.join();
        std::rethrow_exception(s_begin_error);
    }

    // ---- main thread: S levels in join order, shipped to every GPU
    std::exception_ptr s_error;
    if (ordered) { // every worker's copy order registered (or the worker gave up before its join)
        std::unique_lock<std::mutex> lk(s_mu);
        s_cv.wait(lk, [&] { return ord_n >= G; });
    }
    if (!one_dataset) {
        std::vector<tj_dataset*> dst(G);
        for (size_t g = 0; g < G; ++g) dst[g] = dsh[g].p;
        try {
            // S's levels are expanded piece by piece as they land (the join still waits for the
            // whole level): only the last piece's expansion follows the level's last copy
            const bool s_pieced = !compact && pieced_mode() != 0 && s_pieces();
            for (uint32_t level : spec.lods) {
                const int slot = slot_of(S, level);
                if (slot < 0) continue;
                if (s_pieced)
                    for (size_t g = 0; g < G; ++g)
                        detail::check(tj_dataset_set_pieced(dst[g], static_cast<uint32_t>(slot)), ctxs[g]);
                feed_level(S, *s_lease.set, static_cast<size_t>(slot), dst, ctxs, pool, out, pack_ms, &stat_mu,
                           s_pieced);
                for (size_t g = 0; g < G; ++g) put_s[g][slot] = 1;
                mark(std::string("S_lod") + std::to_string(level) + "_put");
            }
        } catch (...) {
            s_error = std::current_exception();
            for (size_t g = 0; g < G; ++g) release_levels(dsh[g].p, put_s[g]);
        }
    }
    for (auto& t : workers) t.join();
    mark("joins_done");
    {
        const detail::ArenaStats a1 = detail::arena_stats();
        out.stats.timeline.emplace_back("arena_fresh_blocks", double(a1.fresh - arena0.fresh));
        out.stats.timeline.emplace_back("arena_pageable_blocks", double(a1.pageable - arena0.pageable));
        out.stats.timeline.emplace_back("arena_fresh_ms", a1.fresh_ms - arena0.fresh_ms);
    }
    for (size_t g = 0; g < G; ++g)
        if (dsh[g].p) tj_dataset_sync(dsh[g].p);
    if (s_error) std::rethrow_exception(s_error);
    for (auto& e : errors)
        if (e) std::rethrow_exception(e);
    out.stats.pack_ms = pack_ms;
    out.stats.device_ms = *std::max_element(dev_ms.begin(), dev_ms.end());

    std::vector<Piece> pieces;
    for (size_t g = 0; g < G; ++g)
        for (size_t k = 0; k < share[g].chunks.size(); ++k) {
            const tj_join_result& res = results[g][k]->r;
            for (uint32_t i = 0; i < res.n_levels_run; ++i) out.stats.stream_wait_ms += res.level_wait_ms[i];
            out.stats.decision_mode = out.stats.decision_mode || res.decision_mode != 0;
            out.stats.mat_chunks += res.mat_chunks;
            const auto [a, b] = share[g].chunks[k];
            const detail::PackedHeader& h = *r_sets[g][k]->set->h;
            pieces.push_back({&res, static_cast<uint32_t>(a), h.ids.empty() ? nullptr : h.ids.data(),
                              static_cast<uint32_t>(b - a)});
        }

    // Merge: every query r this process joins is owned by one piece (a chunk of a GPU's
    // shard, queries ids[0, n) or r_base + [0, n)); the others have no candidates. Records
    // (src/engine.cpp:161-185) and the per-stage tallies come straight from the pieces'
    // arrays, in query order.
    Merged m;
    const uint32_t nq = static_cast<uint32_t>(nr);
    constexpr uint32_t kNone = 0xffffffffu;
    uint64_t total = 0, owned = 0;
    for (const Piece& pc : pieces) {
        total += pc.res->n_cands;
        owned += pc.n;
    }
    // query -> (piece, local index); a single piece covering [0, nq) in order needs no table
    const bool direct = pieces.size() == 1 && !pieces[0].ids && pieces[0].r_base == 0 && pieces[0].n == nq;
    std::vector<uint32_t> own_piece, own_local;
    if (!direct) {
        own_piece.assign(nq, kNone);
        own_local.assign(nq, 0);
        for (uint32_t p = 0; p < pieces.size(); ++p) {
            const Piece& pc = pieces[p];
            for (uint32_t lr = 0; lr < pc.n; ++lr) {
                const uint32_t r = pc.ids ? pc.ids[lr] : pc.r_base + lr;
                own_piece[r] = p;
                own_local[r] = lr;
            }
        }
    }
    for (const Piece& pc : pieces) {
        const tj_join_result& res = *pc.res;
        m.vp_generated += res.vp_generated;
        m.vp_pruned += res.vp_pruned;
        m.mbb_ms = std::max(m.mbb_ms, res.mbb_ms);
        m.voxel_ms = std::max(m.voxel_ms, res.voxel_ms);
        for (uint32_t i = 0; i < res.n_levels_run; ++i) {
            RefineLevelStats& ls = m.levels[res.level[i]];
            ls.level = res.level[i];
            ls.vps += res.level_vps[i];
            ls.facet_pairs += res.level_facet_pairs[i];
            ls.wall_ms = std::max(ls.wall_ms, res.level_ms[i]);
        }
    }
    // per stage code (-3 .. 100): confirmed / removed tallies
    std::vector<uint64_t> conf_at(104, 0), rem_at(104, 0);
    std::vector<uint32_t> conf; // k-NN: one query's confirmed ops
    for (uint32_t r = 0; r < nq; ++r) {
        const uint32_t p = direct ? 0 : own_piece[r];
        if (p == kNone) continue;
        const tj_join_result& res = *pieces[p].res;
        const uint32_t lr = direct ? r : own_local[r];
        const uint64_t o0 = res.r2op_offsets[lr], o1 = res.r2op_offsets[lr + 1];
        conf.clear();
        for (uint64_t op = o0; op < o1; ++op) {
            const uint8_t stt = res.status[op];
            const int16_t at = res.decided_at[op];
            if (stt == TJ_CONFIRMED) {
                ++conf_at[at + 3];
                if (!knn)
                    out.records.push_back({r, res.pair_s[op], res.lb[op], res.ub[op], at, 0});
                else
                    conf.push_back(static_cast<uint32_t>(op));
            } else if (stt == TJ_REMOVED) {
                ++rem_at[at + 3];
            }
        }
        if (knn && !conf.empty()) {
            std::sort(conf.begin(), conf.end(), [&](uint32_t a, uint32_t b) {
                if (res.ub[a] != res.ub[b]) return res.ub[a] < res.ub[b];
                if (res.lb[a] != res.lb[b]) return res.lb[a] < res.lb[b];
                return res.pair_s[a] < res.pair_s[b];
            });
            uint32_t rank = 0;
            for (uint32_t op : conf)
                out.records.push_back({r, res.pair_s[op], res.lb[op], res.ub[op], res.decided_at[op], ++rank});
        }
    }

    // Stage counters (src/engine.cpp:188-236).
    struct Plan {
        int16_t code;
        double wall;
        uint64_t vpg, vpp, fp;
    };
    std::vector<Plan> plan{{stage::kMbb, m.mbb_ms, 0, 0, 0}, {stage::kVoxel, m.voxel_ms, m.vp_generated, m.vp_pruned, 0}};
    for (uint32_t level : spec.lods) {
        Plan p{static_cast<int16_t>(level), 0.0, 0, 0, 0};
        if (auto it = m.levels.find(level); it != m.levels.end()) {
            p.wall = it->second.wall_ms;
            p.vpg = it->second.vps;
            p.fp = it->second.facet_pairs;
        }
        plan.push_back(p);
    }
    // the (r, s) pairs of the queries this process joined (all of R unless process-sharded, so
    // that the counters of the ranks of a torchrun launch sum to the whole join's)
    const uint64_t all_pairs = owned * uint64_t{S.objects.size()};
    uint64_t flowing = all_pairs;
    for (const Plan& p : plan) {
        const bool in_range = p.code >= -3 && p.code <= 100;
        const uint64_t conf = in_range ? conf_at[p.code + 3] : 0;
        uint64_t rem = in_range ? rem_at[p.code + 3] : 0;
        if (p.code == stage::kMbb) rem += all_pairs - total;
        StageCounters sc;
        sc.name = stage_name(p.code);
        sc.wall_ms = p.wall;
        sc.pairs_in = flowing;
        sc.confirmed = conf;
        sc.removed = rem;
        sc.pairs_out = flowing - conf - rem;
        sc.vp_generated = p.vpg;
        sc.vp_pruned = p.vpp;
        sc.facet_pairs = p.fp;
        out.stats.stages.push_back(sc);
        flowing = sc.pairs_out;
    }
    out.stats.results = out.records.size();
    mark("records_built");
    out.stats.total_ms = std::chrono::duration<double, std::milli>(Clock::now() - t_total).count();
    return out;
}

} // namespace trijoin

// ---------------------------------------------------------------- C-ABI host helpers
struct tj_host_dataset {
    std::unique_ptr<trijoin::detail::PackedDataset> packed;
};

extern "C" {

int tj_host_dataset_load(const char* path, tj_host_dataset** out) {
    if (!path || !out) return TJ_EINVAL;
    *out = nullptr;
    try {
        const trijoin::PreparedDataset ds = trijoin::load_index(path);
        trijoin::ThreadPool pool(0);
        auto h = std::make_unique<tj_host_dataset>();
        h->packed = trijoin::detail::pack_dataset(ds, pool);
        *out = h.release();
        return TJ_OK;
    } catch (const std::invalid_argument& e) {
        return TJ_EINVAL;
    } catch (const std::exception& e) {
        return TJ_ECUDA;
    }
}

const tj_dataset_view* tj_host_dataset_view(const tj_host_dataset* h) { return h ? &h->packed->view : nullptr; }

uint64_t tj_host_dataset_bytes(const tj_host_dataset* h) { return h ? h->packed->bytes() : 0; }

void tj_host_dataset_free(tj_host_dataset* h) { delete h; }

} // extern "C"
