// Host-side packing of a PreparedDataset into the C-ABI structure-of-arrays view
// (tj_dataset_view), plus the per-process device context registry.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/tj_capi.h"
#include "trijoin/engine.hpp"
#include "trijoin/index.hpp"

namespace trijoin::detail {

// Page-locked host buffer from a process-wide arena (cudaHostAlloc'ed once, reused), so
// that uploads of packed facet records run at full DMA speed.
struct PinnedBuf {
    double* p = nullptr;
    size_t n = 0;     // doubles in use
    size_t cap = 0;   // doubles allocated
    bool pinned = false;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    PinnedBuf(PinnedBuf&& o) noexcept { *this = std::move(o); }
    PinnedBuf& operator=(PinnedBuf&& o) noexcept;
    ~PinnedBuf();
    void resize(size_t count); // contents not preserved
    double* data() { return p; }
    const double* data() const { return p; }
    size_t size() const { return n; }
};

// Typed view of a PinnedBuf for 8-byte element types; resize() leaves contents undefined
// (no serial zero-fill: the parallel packers touch every element they use).
template <class T>
struct PinnedArr {
    static_assert(sizeof(T) == sizeof(double), "8-byte elements only");
    PinnedBuf b;
    size_t n = 0;
    void resize(size_t count) {
        b.resize(count ? count : 1);
        n = count;
    }
    T* data() { return reinterpret_cast<T*>(b.data()); }
    const T* data() const { return reinterpret_cast<const T*>(b.data()); }
    T& operator[](size_t i) { return data()[i]; }
    const T& operator[](size_t i) const { return data()[i]; }
    size_t size() const { return n; }
    const T& back() const { return data()[n - 1]; }
};

// Owning SoA image of one PreparedDataset in the device layout (include/tj_capi.h).
struct PackedDataset {
    uint32_t n_objects = 0;
    std::vector<int32_t> levels;
    std::vector<double> mbb, anchor, voxel_box, voxel_anchor;
    std::vector<uint64_t> voxel_offsets;
    std::vector<std::vector<uint64_t>> facet_offsets; // per level
    std::vector<PinnedBuf> facets;                    // per level, TJ_FACET_STRIDE doubles each
    std::vector<const uint64_t*> fo_ptrs;
    std::vector<const double*> f_ptrs;
    tj_dataset_view view{};
    uint64_t bytes() const;
};

// ids (optional): only the listed objects, in that order (one query shard of R).
std::unique_ptr<PackedDataset> pack_dataset(const PreparedDataset& ds, ThreadPool& pool,
                                            const std::vector<uint32_t>* ids = nullptr);

// Host staging arena counters (process lifetime): fresh blocks, blocks that could not be
// page-locked, bytes and milliseconds spent allocating fresh blocks.
struct ArenaStats {
    uint64_t fresh, pageable, fresh_bytes;
    double fresh_ms;
};
ArenaStats arena_stats();

// Streamed form (tj_dataset_begin / tj_dataset_put_level): the header holds the object and
// voxel arrays, the per-level voxel CSR and the per-object vertex / facet bases; each level
// is then packed on its own in the reference's compact mesh form.
struct PackedHeader {
    // object selection the header was packed from: objects [first, first + n_objects) of the
    // dataset, or (ids non-empty) the listed global object ids, ascending
    size_t first = 0;
    std::vector<uint32_t> ids;
    uint32_t n_objects = 0;
    std::vector<int32_t> levels;
    PinnedArr<double> mbb, anchor, voxel_box, voxel_anchor;     // page-locked, reused across joins
    PinnedArr<uint64_t> voxel_offsets;
    std::vector<PinnedArr<uint64_t>> facet_offsets;             // per level [nv+1]
    std::vector<PinnedArr<uint64_t>> vert_base, facet_base;     // per level [n_objects+1]
    std::vector<uint64_t> n_vertices, n_facets;                  // per level totals
    std::vector<const uint64_t*> fo_ptrs, vb_ptrs, fb_ptrs;
    tj_dataset_view view{};
    uint64_t bytes() const; // H2D bytes of tj_dataset_begin
};
// Rows of one packed piece of a level: vertices, facets and voxel facet-id entries.
struct PieceRows {
    uint64_t vert_begin, vert_end, facet_begin, facet_end, entry_begin, entry_end;
    uint32_t obj_begin, obj_end; // the piece's objects
};
struct PackedLevel {
    PinnedBuf verts, tris, hd, ph, vf; // tris / vf hold uint32 pairs per double slot
    bool zero_pads = false;            // every hd / ph of the level is +0: not shipped
    bool narrow = false;               // ids shipped as uint16 (every object < 65536 vertices / facets)
    uint64_t bytes = 0;                // H2D bytes of the level
    tj_level_mesh_view view{};
    std::vector<PieceRows> pieces;     // the object-range pieces it was packed in (shipped alike when cached)
};
std::unique_ptr<PackedHeader> pack_header(const PreparedDataset& ds, ThreadPool& pool);
// The same over objects [first, last) of ds (one R chunk of the out-of-core path).
std::unique_ptr<PackedHeader> pack_header(const PreparedDataset& ds, size_t first, size_t last, ThreadPool& pool);
// The same over the listed objects of ds (ascending global ids: one query shard).
std::unique_ptr<PackedHeader> pack_header(const PreparedDataset& ds, std::vector<uint32_t> ids, ThreadPool& pool);
// Level slot li of the objects h was packed from. With pieces > 1 it is packed in that many
// consecutive object ranges and on_piece(level, rows) runs after each (the caller ships the
// rows while the next piece is packed).
std::unique_ptr<PackedLevel> pack_level(const PreparedDataset& ds, const PackedHeader& h, size_t li, ThreadPool& pool,
                                        size_t pieces = 1,
                                        const std::function<void(const PackedLevel&, const PieceRows&)>& on_piece = {});

// A dataset's streamed form, packed once and reused by every join of the same immutable
// dataset (the Python Dataset objects): header + the levels packed so far, by slot.
struct PackedSet {
    std::unique_ptr<PackedHeader> h;
    std::vector<std::unique_ptr<PackedLevel>> levels;
};

// Packed sets of one immutable dataset, kept across joins (keyed by object selection). A
// set is lent to one join at a time; a concurrent join of the same selection packs afresh.
struct JoinCache {
    std::mutex mu;
    std::map<std::string, std::shared_ptr<PackedSet>> idle;
    std::shared_ptr<PackedSet> take(const std::string& key) {
        std::lock_guard<std::mutex> lk(mu);
        auto it = idle.find(key);
        if (it == idle.end()) return std::make_shared<PackedSet>();
        auto s = std::move(it->second);
        idle.erase(it);
        return s;
    }
    void give_back(const std::string& key, std::shared_ptr<PackedSet> s) {
        std::lock_guard<std::mutex> lk(mu);
        idle[key] = std::move(s);
    }
};

// run_join with optional per-dataset caches of the packed streamed form (nullptr = pack
// afresh, as the C++ API does: PreparedDataset is caller-owned and may change between calls).
JoinOutput run_join_cached(const PreparedDataset& R, const PreparedDataset& S, const JoinSpec& spec, ThreadPool& pool,
                           const JoinTrace* trace, JoinCache* r_cache, JoinCache* s_cache);

// Lazily created context per (CUDA device, slot), destroyed at process exit. Several slots
// of one device are independent contexts (own stream and workspace): TRIJOIN_DEVICES=0,0
// runs two query shards side by side on GPU 0.
tj_ctx* device_context(int device, int slot = 0);
// Devices used by run_join: $TRIJOIN_DEVICES (comma list) or {0}.
std::vector<int> join_devices();

// Throws the C++ exception matching a C-ABI status code.
[[noreturn]] void throw_status(int code, const char* msg);
inline void check(int code, tj_ctx* ctx) {
    if (code != TJ_OK) throw_status(code, ctx ? tj_last_error(ctx) : tj_global_last_error());
}

// RAII holders.
struct DatasetHandle {
    tj_dataset* p = nullptr;
    DatasetHandle() = default;
    DatasetHandle(const DatasetHandle&) = delete;
    DatasetHandle& operator=(const DatasetHandle&) = delete;
    ~DatasetHandle() { tj_dataset_free(p); }
};
struct ResultHandle {
    tj_join_result r{};
    ResultHandle() = default;
    ResultHandle(const ResultHandle&) = delete;
    ResultHandle& operator=(const ResultHandle&) = delete;
    ~ResultHandle() { tj_join_result_free(&r); }
};

} // namespace trijoin::detail
