// Internal device-side types shared by the kernels and the C-ABI implementation.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
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

// Stream used for stream-ordered allocation by DevBuf on this thread (set at every C-ABI
// entry to the context's stream; nullptr = legacy stream). Allocations come from the
// device's default memory pool, which the context configures never to release memory, so
// per-join temporaries cost no cudaMalloc/cudaFree (and no implicit device syncs).
inline cudaStream_t& alloc_stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}

// Wait for the work queued on `st` so far (spinning; TRIJOIN_BLOCKING_SYNC=1: a blocking-sync
// event, the calling thread sleeps).
void stream_sync(cudaStream_t st);

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
        if (count) TJ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), alloc_stream()));
    }
    // grow-only reallocation (contents not preserved)
    void reserve(size_t count) { if (count > n) alloc(count); }
    void release() {
        if (p) cudaFreeAsync(p, alloc_stream());
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Arrival state of the levels of a streamed dataset (tj_dataset_begin / _put_level): a
// level is pending until its copy + expansion has been queued on the dataset's copy
// stream (then `ev` marks its completion) or failed.
struct LevelGate {
    enum State { kPending = 0, kQueued = 1, kFailed = 2 };
    std::mutex mu;
    std::condition_variable cv;
    std::vector<int> state;
    std::vector<cudaEvent_t> ev;
    // levels shipped in object-range pieces (tj_dataset_set_pieced): per slot the pieces
    // finished so far, (end object, event after its expansion and derivation), in order
    std::vector<char> pieced;
    std::vector<std::vector<std::pair<uint32_t, cudaEvent_t>>> pieces;
    cudaStream_t copy = nullptr;   // the level copies (H2D)
    cudaStream_t expand = nullptr; // expansion / derivation of landed levels (high priority), so
                                   // copies never queue behind kernels waiting for SMs
    cudaEvent_t expanded = nullptr; // after the last queued expansion (staging-area reuse)
    std::vector<char> started;     // per slot: a put has been issued
    int device = 0;
    // per slot: event after the slot's copies (re-recorded by every put of the slot), and the
    // copy-order dependency (tj_dataset_copy_after): that dataset's gate and slot, applied once
    std::vector<cudaEvent_t> copied;
    std::vector<std::pair<LevelGate*, int>> after;
    std::vector<char> after_done;
    ~LevelGate();
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
    std::vector<uint64_t> level_entries;         // per level: facet records (CSR entries)
    // derived per level at upload (refine.cu k_prep / k_seg_prep, on the upload stream): FP32
    // screening records (kScreenRecF4 float4 per facet: box parts, then geometry parts), voxel
    // segment aggregates (3 float4 per voxel) and the level aggregates (3 uints per level)
    std::vector<DevBuf<float4>> screen, seg;
    DevBuf<unsigned> agg;
    // streamed datasets only (tj_dataset_begin): per-level object bases, voxel -> object,
    // validation flag of the device-side expansion, arrival gate
    std::vector<DevBuf<uint64_t>> vert_base, facet_base; // per level [n_obj+1]
    std::vector<uint64_t> level_vertices, level_facets;  // per level totals
    DevBuf<uint32_t> vox_obj;                            // [nv]
    DevBuf<int> stream_err;                              // [1]: an index out of range
    DevBuf<unsigned char> stage;                         // compact-level staging area (largest level)
    std::shared_ptr<LevelGate> gate;
    // Compact-resident datasets (tj_dataset_begin_ex, TJ_DATASET_COMPACT): every level stays in
    // HBM in the shipped compact mesh form (~44 B per facet instead of the 96-B records plus
    // 128-B screening records); a join expands, per level, only the voxels its active voxel
    // pairs touch (materialize_level). facets / screen / seg are then unused.
    bool compact = false;
    std::vector<DevBuf<unsigned char>> cmp; // per level: compact mesh form (stage_layout)
    std::vector<uint32_t> cmp_flags;        // per level: TJ_LEVEL_PADS / TJ_LEVEL_NARROW
};

// Expands level slot `slot` of a compact-resident dataset into facet records (TJ_FACET_STRIDE
// doubles each): voxel v's facets go to out[act[v] ...] when act[v + 1] > act[v] (act: an
// exclusive scan over the voxels of the active voxels' facet counts); ids out of range set
// *d.stream_err (capi.cu).
void expand_compact_level(const DatasetDev& d, uint32_t slot, const uint64_t* act, double* out, int num_sms,
                          cudaStream_t st);

// Derived screening data of level slot li of d (facets already resident), on stream st.
void derive_level(DatasetDev& d, uint32_t li, int num_sms, cudaStream_t st);
// The same for the voxels [v_begin, v_end) of a level arriving in object-range pieces (first:
// the level's first piece: allocates and resets the level aggregates, complete only once every
// piece is derived).
void derive_level_range(DatasetDev& d, uint32_t li, uint64_t v_begin, uint64_t v_end, bool first, int num_sms,
                        cudaStream_t st);

// Makes `st` wait until level slot `slot` of `d` is resident (no-op for uploaded datasets);
// returns the host milliseconds spent blocked waiting for the level to be queued.
double level_ready(const DatasetDev& d, int slot, cudaStream_t st);
// $TRIJOIN_DEBUG_TIMELINE diagnostics: labelled timing events recorded on the copy streams
// (level copies queued / expanded), printed by the join's timeline relative to its start
void copy_mark(const char* what, int level, cudaStream_t st);
std::vector<std::pair<std::string, cudaEvent_t>> take_copy_marks();
// Pieced levels: whether slot arrives in object-range pieces, and piece k's end object and
// completion event (host-blocks until it is finished; nullptr once the level is complete and
// every piece was returned).
bool level_pieced(const DatasetDev& d, int slot);
cudaEvent_t level_piece(const DatasetDev& d, int slot, size_t k, uint32_t* obj_end);
// Non-blocking: piece k's event if it has been finished (queued), else nullptr.
cudaEvent_t level_piece_try(const DatasetDev& d, int slot, size_t k, uint32_t* obj_end);

// Active voxel pair during refinement: candidate op + global voxel ids.
struct ActiveVpDev {
    uint32_t op, gvr, gvs;
};

// Where the voxel pairs of a refinement pass come from: join mode (active list + per-level
// CSR of both datasets) or batch mode (explicit facet segments; every pair its own op).
struct RefineSource {
    // join mode
    const ActiveVpDev* active; // nullptr = batch mode
    const uint64_t* r_foff;    // facet offsets of this level, by global voxel
    const uint64_t* s_foff;
    const double* cand_lb;     // candidate intervals before this level
    const double* cand_ub;
    // batch mode
    const uint64_t* r_off;
    const uint64_t* s_off;
    const uint32_t* r_len;
    const uint32_t* s_len;
    // both: facet records (TJ_FACET_STRIDE doubles each) and their FP32 screening records
    const double* r_facets;
    const double* s_facets;
    // FP32 screening records (refine_prep): box parts (kBoxF4 float4 per facet) and geometry
    // parts (kGeoF4 float4 per facet) as separate arrays
    const float4* r_box;
    const float4* r_geo;
    const float4* s_box;
    const float4* s_geo;
    // level aggregates of the screening records (refine_prep): [0..2] R min hd, max |L|,
    // max M; [3..5] the same for S (float bits; join mode only, else nullptr)
    const unsigned* agg;
    // per-voxel segment aggregates of this level (refine_seg_prep; 3 float4 per global
    // voxel; join mode only, else nullptr)
    const float4* r_seg;
    const float4* s_seg;
    // 1: ignore the records' hd / ph (pure tri-tri minima: the --exact recompute)
    int zero_pad;
    // mean facets per voxel of the level (R and S; 0 = unknown): sizes k_screen's work grabs
    float mean_seg;
    // decision mode: ops with (op & exact_mask) == 0 keep exact intervals (the reference's
    // bound-crossing tripwire is evaluated on them); 0xffffffff = none
    uint32_t exact_mask;
    // join mode: number of ops (candidate pairs); sizes the decision-mode seed pick (0 = unknown)
    uint32_t n_ops;
};

// Decision-mode op sample with exact intervals: $TRIJOIN_TRIPWIRE_SAMPLE = every N-th op
// (N a power of two, default 1024; 0 = none, 1 = every op). Returns the mask for op & mask == 0.
uint32_t tripwire_mask();
__host__ __device__ __forceinline__ bool exact_op(uint32_t mask, uint32_t op) {
    return mask != 0xffffffffu && (op & mask) == 0;
}

// A queued facet pair: op and the two global facet record indices.
struct PairRef {
    uint32_t op, fr, fs;
    uint32_t mask; // verify queue: ill-conditioned combinations to check
};

constexpr int kNumCounters = 8;
constexpr int kScreenRecF4 = 8; // float4 per FP32 screening record (refine_kernel.cuh)

struct RefineQueue {
    PairRef* items;
    unsigned long long capacity;
    unsigned long long* count;
};

struct RefineQueueStore {
    DevBuf<PairRef> items;              // exact-evaluation queue
    DevBuf<unsigned long long> count; // [0] entries of the current pass, [1] largest overflowing count
    DevBuf<unsigned long long> pick;  // decision-mode seeding: per op, (key << 32 | voxel pair) of its primary
    // Test hook ($TRIJOIN_TEST_QUEUE_CAP, read per level by refine_loop_dev): the passes of a
    // level see at most `cap` slots until the first overflow grows the queue, so the
    // overflow -> grow -> re-run path runs on small inputs. 0 = no cap.
    uint64_t cap = 0;
    RefineQueueStore() : count(2) { items.alloc(1u << 22); }
    RefineQueue view() {
        const uint64_t n = cap && cap < items.n ? cap : items.n;
        return {items.p, (unsigned long long)n, count.p};
    }
    // before a level's passes: clears both queues' entry and overflow counts
    void reset(cudaStream_t st);
    // after a level's passes (stream-synchronous): grows whichever queue overflowed; true if
    // the level must be re-run
    bool grow_if_overflowed(cudaStream_t st);
};

// FP32 screening records of n facet records (refine.cu, k_prep) into out[7 n]: box parts at
// out[0, 3 n), geometry parts at out[3 n, 7 n).
// agg (optional, 3 uints pre-set to {+inf, 0, 0} bits): min hd, max |L|, max M of the records.
void refine_prep(const double* facets, uint64_t n, float4* out, unsigned* agg, int num_sms, cudaStream_t st,
                 int zero_pad = 0);

// Per-voxel segment aggregates of one level (refine.cu, k_seg_prep) into seg[3 n_voxels]:
// union of the facet boxes, max / min L, max ph, min hd, all well shaped.
void refine_seg_prep(const float4* box, const uint64_t* foff, uint64_t n_voxels, float4* seg, int num_sms,
                     cudaStream_t st);

// One refinement pass over voxel pairs [vp_begin, vp_end) (refine.cu): the seed pass queues
// each voxel pair's 2 smallest-box-gap facet pairs, the screen pass every facet pair that
// may still change the op's bounds; then the queued pairs are evaluated exactly and folded
// into lb_bits / ub_bits (atomicMin on IEEE bits). counters (kNumCounters): [0] facet-pair
// box tests, [1] exact evaluations, [2] the refine loop's facet-pair count, [3]
// separating-axis tests, [4] FP64 piercing verifications, [5] voxel pairs skipped whole,
// [6] facets dropped by the row/column screens.
// screen_ev (optional, 2 events): recorded around the k_screen launch (bench.py kernel timing).
void refine_pass(const RefineSource& src, uint64_t vp_begin, uint64_t vp_end, bool seed, unsigned long long* lb_bits,
                 unsigned long long* ub_bits, int cull, RefineQueueStore& qs, unsigned long long* work,
                 unsigned long long* counters, int num_sms, cudaStream_t st, cudaEvent_t* screen_ev = nullptr);

// Diagnostics (TRIJOIN_DEBUG_OPSTATS): per-op tested-pair counters of k_screen (nullptr = off).
void refine_debug_op_tested(unsigned long long* p);


} // namespace tjx
