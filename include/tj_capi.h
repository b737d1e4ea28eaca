/*
 * tj_capi.h — the C-ABI of the B200-native trijoin join engine.
 *
 * Plain C: POD structs, raw pointers and sizes, integer status codes. No C++
 * or torch types cross this boundary. The C++ host library (include/trijoin/ headers,
 * the drop-in for the reference's proj/include/trijoin API) and the Python module
 * `paper_2604_19982_b200._core` (drop-in for the reference's `trijoin._core`)
 * are both thin layers over these entry points.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj):
 *   tj_join            run_join                 include/trijoin/engine.hpp:70-71, src/engine.cpp:122-237
 *   tj_refine_batch    refine_kernel            include/trijoin/refine.hpp:67-68, src/refine.cpp:63-84
 *   tj_geom_batch      mindist_aabb, point_segment_distance, point_triangle_distance,
 *                      segment_segment_distance, tri_tri_distance
 *                                               include/trijoin/geom.hpp:60-79,   src/geom.cpp:11-183
 *   tj_tri_tri_batch   tri_tri_distance         include/trijoin/geom.hpp:79,      src/geom.cpp:152-183
 *   tj_mindist_batch   mindist_aabb             include/trijoin/geom.hpp:60,      src/geom.cpp:11-16
 *   tj_exhaustive_join run_oracle               include/trijoin/engine.hpp:77-80, src/oracle.cpp:124-186
 *   tj_mbb_filter      mbb_filter_within / _knn include/trijoin/filter.hpp:62-66,   src/filter.cpp:88-190
 *   tj_voxel_filter    chunked_filter           include/trijoin/filter.hpp:111-114, src/filter.cpp:350-448
 *   tj_voxel_bounds    voxel_pair_bounds        include/trijoin/filter.hpp:83-85,   src/filter.cpp:199-239
 *   tj_voxel_compact   voxel_pair_compact       include/trijoin/filter.hpp:94-97,   src/filter.cpp:265-315
 *   tj_refine_loop     refine_loop              include/trijoin/refine.hpp:82-87,   src/refine.cpp:263-314
 *   tj_knn_prune       knn_prune_round / _to_fixpoint / knn_finalize
 *                                               include/trijoin/knn.hpp:30-50,      src/knn.cpp:19-118
 *   tj_facet_hd_batch  compute_facet_hd         include/trijoin/mesh.hpp:65-66,     src/hausdorff.cpp:15-33
 *   tj_facet_ph_batch  compute_facet_ph / the ph fill of build_lod_ladder
 *                                               include/trijoin/mesh.hpp:71,        src/simplify.cpp:238-267
 *   tj_voxelize_batch  voxelize                 include/trijoin/index.hpp:48,       src/voxelize.cpp:27-79
 *   tj_dataset_upload  (no reference analogue: PreparedDataset is host-resident there,
 *                       include/trijoin/index.hpp:15-36; here it is packed once into HBM)
 *
 * Status codes: TJ_OK; TJ_EINVAL -> std::invalid_argument / ValueError;
 * TJ_EENGINE -> EngineError (soundness tripwires, src/filter.cpp:25-31, src/knn.cpp:59,68-77,
 * src/refine.cpp:312-313); TJ_ECUDA / TJ_ENOMEM -> std::runtime_error. The message of the
 * last failure on a context is returned by tj_last_error().
 *
 * Threading: a tj_ctx is owned by one host thread (the coordinator of one GPU). Every
 * call blocks until its device work is complete. Device buffers belong to the context;
 * host views belong to the caller.
 */
#ifndef TJ_CAPI_H
#define TJ_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TJ_OK = 0, TJ_EINVAL = 1, TJ_EENGINE = 2, TJ_ECUDA = 3, TJ_ENOMEM = 4 };

/* Join types (reference JoinType, include/trijoin/engine.hpp:15). */
enum { TJ_WITHIN = 0, TJ_INTERSECT = 1, TJ_KNN = 2 };

/* Pair status (reference PairStatus, include/trijoin/filter.hpp:12). */
enum { TJ_UNDECIDED = 0, TJ_CONFIRMED = 1, TJ_REMOVED = 2 };

/* Stage codes (reference stage::, include/trijoin/filter.hpp:16-20); LOD levels are 1..100. */
enum { TJ_STAGE_NONE = -3, TJ_STAGE_MBB = -2, TJ_STAGE_VOXEL = -1 };

/* Behaviour flags (none of them changes a result). */
enum {
    TJ_FLAG_NO_CULL = 1u << 0, /* disable exact-preserving facet-pair culling (A/B checks) */
    TJ_FLAG_SYNC_STAGES = 1u << 1, /* synchronise + time every stage (stats wall_ms) */
    /* Keep every candidate interval equal to the reference's at every level. Without it, an
       intersection join without a trace refines in decision mode: a level only establishes
       whether min lb_ij / min ub_ij are 0 (the only facts an intersection decision and its
       records depend on), so intervals of pairs it removes may stay looser
       than the reference's; records and stage counters are identical either way. */
    TJ_FLAG_EXACT_INTERVALS = 1u << 2,
    /* JoinSpec::exact (reference src/engine.cpp:96-118, :159): after the cascade, every
       confirmed pair's interval becomes [d, d], d the minimum tri_tri_distance over all
       pairs of the two level-100 meshes' facets. */
    TJ_FLAG_EXACT_RECOMPUTE = 1u << 3
};

#define TJ_FACET_STRIDE 12 /* doubles per facet record: v0.xyz v1.xyz v2.xyz hd ph pad */
#define TJ_MAX_LODS 16

typedef struct tj_ctx tj_ctx;
typedef struct tj_dataset tj_dataset;

/*
 * Host view of one prepared dataset (reference PreparedDataset / PreparedObject /
 * VoxelSet / LodMesh, include/trijoin/index.hpp:15-36, include/trijoin/mesh.hpp:42-49),
 * flattened to structure-of-arrays. Voxels are numbered globally: object o owns voxels
 * [voxel_offsets[o], voxel_offsets[o+1]). For LOD slot li (levels[li], the dataset's
 * lod_schedule), the facets of global voxel v are entries
 * [facet_offsets[li][v], facet_offsets[li][v+1]) of facets[li], each TJ_FACET_STRIDE
 * doubles, in the voxel's ascending facet-id order (reference facets_per_level).
 */
typedef struct tj_dataset_view {
    uint32_t n_objects;
    uint32_t n_levels;
    const int32_t* levels;        /* [n_levels] ascending LOD percentages */
    const double* mbb;            /* [n_objects*6] min.xyz, max.xyz */
    const double* anchor;         /* [n_objects*3] */
    const uint64_t* voxel_offsets;/* [n_objects+1] */
    const double* voxel_box;      /* [n_voxels*6] */
    const double* voxel_anchor;   /* [n_voxels*3] */
    const uint64_t* const* facet_offsets; /* [n_levels] -> [n_voxels+1] */
    const double* const* facets;          /* [n_levels] -> [n_entries*TJ_FACET_STRIDE] */
} tj_dataset_view;

/* Reference JoinSpec (include/trijoin/engine.hpp:19-30); workers/seed are host-side only. */
typedef struct tj_join_spec {
    int32_t type;          /* TJ_WITHIN / TJ_INTERSECT / TJ_KNN */
    double tau;            /* within; intersect requires 0 */
    uint32_t k;            /* knn */
    uint64_t filter_chunk; /* voxel pairs per filter chunk (result-invariant) */
    uint64_t refine_chunk; /* voxel pairs per refine launch (result-invariant) */
    uint32_t n_lods;
    const uint32_t* lods;  /* ascending, ending at 100, each present in both datasets */
    int32_t pipeline;      /* result-invariant overlap switch */
    uint32_t flags;        /* TJ_FLAG_* */
    /* R sharding across GPUs: query r participates iff
       (r / shard_block) % shard_count == shard_index. shard_count 0 or 1 = all r. */
    uint32_t shard_index, shard_count, shard_block;
} tj_join_spec;

/* Per-stage observer callbacks (reference JoinTrace, include/trijoin/filter.hpp:56-60).
   Fired on the calling thread, in ascending op order within a stage. NULL = off. */
typedef struct tj_trace {
    void* user;
    void (*on_interval)(void* user, uint32_t op, int16_t stage, double lb, double ub);
    void (*on_vp_pruned)(void* user, uint32_t op, uint32_t vr, uint32_t vs, double lb_v,
                         double ub_o);
} tj_trace;

/* Final candidate set (reference CandidateSet, include/trijoin/filter.hpp:38-48) and the
   deterministic counters behind StageStats (src/engine.cpp:188-236). Arrays are owned by
   the library; release with tj_join_result_free. */
typedef struct tj_join_result {
    uint64_t n_cands;
    uint32_t n_queries;
    uint32_t* pair_r;
    uint32_t* pair_s;
    double* lb;
    double* ub;
    uint8_t* status;
    int16_t* decided_at;
    uint64_t* r2op_offsets;  /* [n_queries+1] */
    uint32_t* num_confirmed; /* [n_queries] */
    uint64_t vp_generated, vp_pruned;
    uint64_t filter_chunks, oversized_chunks;
    uint32_t n_levels_run;
    uint32_t level[TJ_MAX_LODS];
    uint64_t level_vps[TJ_MAX_LODS];
    uint64_t level_facet_pairs[TJ_MAX_LODS];     /* reference count: sum r_len*s_len */
    uint64_t level_pairs_evaluated[TJ_MAX_LODS]; /* exact FP64 evaluations actually run */
    uint64_t level_pairs_tested[TJ_MAX_LODS];    /* FP32 cull tests run */
    double level_ms[TJ_MAX_LODS];
    double level_kernel_ms[TJ_MAX_LODS];         /* refine kernel only (CUDA events) */
    uint64_t refine_chunks;
    double mbb_ms, voxel_ms, refine_ms, total_ms;
    uint64_t level_pairs_screened[TJ_MAX_LODS];  /* FP32 separating-axis tests run */
    uint64_t level_pairs_verified[TJ_MAX_LODS];  /* FP64 piercing verifications run */
    uint64_t level_vps_skipped[TJ_MAX_LODS];     /* voxel pairs skipped whole by the screen */
    uint64_t level_facets_dropped[TJ_MAX_LODS];  /* facets dropped by the row/column screens */
    double level_wait_ms[TJ_MAX_LODS];           /* host time blocked on a streamed level */
    int32_t decision_mode;                       /* 1: refined in decision mode (TJ_FLAG_EXACT_INTERVALS) */
    uint32_t queue_reruns;                       /* levels re-run after an exact-queue overflow */
    uint64_t mat_chunks;                         /* compact-resident datasets: level expansions (chunks) */
    double level_screen_ms[TJ_MAX_LODS];         /* the screen kernel's launches only (CUDA events) */
} tj_join_result;

/* ---- context ---- */
int tj_ctx_create(int device, tj_ctx** out);
void tj_ctx_destroy(tj_ctx* ctx);
const char* tj_last_error(const tj_ctx* ctx);
/* Library-wide last error for failures without a context (e.g. tj_ctx_create). */
const char* tj_global_last_error(void);
int tj_device_count(void);
/* Number of this library's own CUDA kernel launches so far (process-wide). */
uint64_t tj_kernel_launches(void);

/* ---- datasets (resident in HBM) ---- */
int tj_dataset_upload(tj_ctx* ctx, const tj_dataset_view* view, tj_dataset** out);
void tj_dataset_free(tj_dataset* ds);
uint64_t tj_dataset_device_bytes(const tj_dataset* ds);

/* ---- streamed datasets: compact mesh form, per-level H2D overlapping the join ----
 *
 * The e2e path of run_join (include/trijoin/engine.hpp) does not ship the expanded
 * 96-byte facet records over PCIe. It ships each LOD level in the reference's own mesh
 * form, object by object exactly as PreparedObject holds it (vertices, object-local index
 * triples, hd/ph, object-local voxel facet-id lists; ~44 B per facet, so the host side
 * is plain memcpy), and the device rebases, validates and expands it into the resident
 * record layout. Levels are uploaded one at a time on the dataset's own copy stream while
 * tj_join already runs the filters and the coarser levels; tj_join blocks (host condition
 * variable, then a device event wait) only when it reaches a level that has not arrived.
 *
 * tj_dataset_begin: uploads the object and voxel arrays of `header` (its facets[] may be
 *   NULL; facet_offsets[] is required) and reserves every level. vert_base[li] and
 *   facet_base[li] ([n_objects+1] each) are the per-object prefix sums of the level's
 *   vertex and facet counts (object o owns vertices [vert_base[o], vert_base[o+1])).
 * tj_dataset_put_level: queues level slot `slot`: copies from the caller's buffers (keep
 *   them valid, preferably page-locked, until tj_dataset_sync returns) and expands. May be
 *   called from another host thread while tj_join runs on the dataset. lv == NULL marks
 *   the slot failed: a join waiting for it returns TJ_EINVAL. An index out of its
 *   object's range makes every later tj_join on the dataset return TJ_EINVAL.
 * tj_dataset_put_level_part / tj_dataset_finish_level: the same upload in pieces, so the
 *   copy of a level overlaps the host packing its remaining objects. A part copies rows
 *   [vert_begin, vert_end) of lv->vertices, [facet_begin, facet_end) of lv->tris (and of
 *   lv->hd / lv->ph when non-NULL) and [entry_begin, entry_end) of lv->voxel_facets (lv's
 *   arrays are the whole level's; the ranges are row indices into them). Once every row has
 *   been put, tj_dataset_finish_level(flags: TJ_LEVEL_PADS if hd / ph were shipped,
 *   TJ_LEVEL_NARROW if the 16-bit id arrays were) expands the level and queues it;
 *   tj_dataset_put_level == one part covering the level + finish.
 * tj_dataset_sync: waits for every queued level copy of the dataset.
 */
typedef struct tj_level_mesh_view {
    const double* vertices;       /* [vert_base[n_objects]*3] all objects, concatenated */
    const uint32_t* tris;         /* [facet_base[n_objects]*3] object-local vertex ids */
    const double* hd;             /* [facet_base[n_objects]]; hd and ph both NULL: all 0 */
    const double* ph;             /* [facet_base[n_objects]] */
    const uint32_t* voxel_facets; /* [facet_offsets[li][n_voxels]] object-local facet ids, voxel order */
    /* Optional 16-bit forms (objects with at most 65536 vertices and facets at this level):
     * when tris16 is non-NULL it replaces tris, likewise voxel_facets16 (both or neither). */
    const uint16_t* tris16;
    const uint16_t* voxel_facets16;
} tj_level_mesh_view;

#define TJ_LEVEL_PADS 1u   /* tj_dataset_finish_level: hd / ph were shipped */
#define TJ_LEVEL_NARROW 2u /* tj_dataset_finish_level: tris16 / voxel_facets16 were shipped */
#define TJ_LEVEL_PIECES 4u /* tj_dataset_finish_level: every object was finished by tj_dataset_finish_level_part */

int tj_dataset_begin(tj_ctx* ctx, const tj_dataset_view* header, const uint64_t* const* vert_base,
                     const uint64_t* const* facet_base, tj_dataset** out);
/* tj_dataset_begin_ex(flags = TJ_DATASET_COMPACT): the dataset keeps every level in HBM in the
 * shipped compact mesh form (~44 B per facet instead of ~224 B of expanded FP64 records and
 * FP32 screening records) and a join expands, per level, only the voxels of its active voxel
 * pairs, in chunks of a working-set budget ($TRIJOIN_WORKSET_MB) if need be. For inputs whose
 * expanded form exceeds HBM (SURVEY configs D, E); results are identical. */
#define TJ_DATASET_COMPACT 1u
int tj_dataset_begin_ex(tj_ctx* ctx, const tj_dataset_view* header, const uint64_t* const* vert_base,
                        const uint64_t* const* facet_base, uint32_t flags, tj_dataset** out);
int tj_dataset_put_level(tj_dataset* ds, uint32_t slot, const tj_level_mesh_view* lv);
int tj_dataset_put_level_part(tj_dataset* ds, uint32_t slot, const tj_level_mesh_view* lv, uint64_t vert_begin,
                              uint64_t vert_end, uint64_t facet_begin, uint64_t facet_end, uint64_t entry_begin,
                              uint64_t entry_end);
int tj_dataset_finish_level(tj_dataset* ds, uint32_t slot, uint32_t flags);
/* Pieced levels (the last join level of R in run_join's e2e path): tj_dataset_set_pieced(slot)
 * before the join starts; then per consecutive object range [obj_begin, obj_end) (covering the
 * objects in order) its rows put with tj_dataset_put_level_part and tj_dataset_finish_level_part,
 * which expands and derives those objects' voxels and lets a join refine the active voxel pairs
 * of those queries while later pieces are still in flight; finally tj_dataset_finish_level(slot,
 * flags | TJ_LEVEL_PIECES). Not for compact-resident datasets. Results are unchanged. */
int tj_dataset_set_pieced(tj_dataset* ds, uint32_t slot);
int tj_dataset_finish_level_part(tj_dataset* ds, uint32_t slot, uint32_t obj_begin, uint32_t obj_end, uint32_t flags);
/* Host-blocks until level slot of ds is on the device (queued and its copies complete). */
int tj_dataset_level_wait(tj_dataset* ds, uint32_t slot);
/* Copy order across two streamed datasets sharing the host link (run_join: S20 R20 S60 R60 ...,
 * so each join level's data of both sides lands before the next level's competes for it): the
 * copies of level `slot` of ds start on the device only after every copy of level `before_slot`
 * of `before` has completed. Register before the first put of `slot`; that put host-waits until
 * `before`'s level has been fully put (finished) or failed. Results are unchanged. */
int tj_dataset_copy_after(tj_dataset* ds, uint32_t slot, tj_dataset* before, uint32_t before_slot);
int tj_dataset_sync(tj_dataset* ds);

/* ---- host-side index loading (backs load_index, reference src/index_io.cpp:244-249) ----
   Parses a 3DPJ1 index file and packs it into the tj_dataset_view layout in host memory,
   for FFI hosts that do not link the C++ API. The view stays valid until the handle is
   freed. */
typedef struct tj_host_dataset tj_host_dataset;
int tj_host_dataset_load(const char* path, tj_host_dataset** out);
const tj_dataset_view* tj_host_dataset_view(const tj_host_dataset* h);
uint64_t tj_host_dataset_bytes(const tj_host_dataset* h);
void tj_host_dataset_free(tj_host_dataset* h);

/* ---- full join (backs run_join) ---- */
int tj_join(tj_ctx* ctx, const tj_dataset* R, const tj_dataset* S, const tj_join_spec* spec,
            const tj_trace* trace, tj_join_result* out);
void tj_join_result_free(tj_join_result* res);

/* ---- stage / primitive entry points on host buffers ---- */

/* refine_kernel: per descriptor d, the min over its facet pairs of
   max(0, dist - ph_i - ph_j) (vp_lb) and dist + hd_i + hd_j (vp_ub); empty -> +inf.
   tris: [n_tris*9] doubles (v0 v1 v2); hd/ph: [n_tris]. */
int tj_refine_batch(tj_ctx* ctx, uint64_t n_tris, const double* tris, const double* hd,
                    const double* ph, uint64_t n_descs, const uint64_t* r_off,
                    const uint64_t* s_off, const uint32_t* r_len, const uint32_t* s_len,
                    uint32_t flags, double* vp_lb, double* vp_ub);

/* ---- stage entry points over a caller-owned host candidate set ----
 * The reference's stage functions (called directly by its tests and tools) on the device.
 * Datasets are tj_dataset handles (tj_dataset_upload); the candidate set is the caller's
 * (reference CandidateSet, include/trijoin/filter.hpp:38-48) and is updated in place.
 *   tj_mbb_filter     mbb_filter_within / mbb_filter_knn   include/trijoin/filter.hpp:62-66, src/filter.cpp:88-190
 *                     (exact broad phase; returns a new candidate set in a tj_join_result)
 *   tj_voxel_filter   chunked_filter (all chunks)          include/trijoin/filter.hpp:111-114, src/filter.cpp:350-448
 *   tj_voxel_bounds   voxel_pair_bounds (one chunk)        include/trijoin/filter.hpp:83-85, src/filter.cpp:199-239
 *   tj_voxel_compact  voxel_pair_compact (one chunk)       include/trijoin/filter.hpp:94-97, src/filter.cpp:265-315
 *   tj_refine_loop    refine_loop / knn_resolve            include/trijoin/refine.hpp:82-87, src/refine.cpp:263-314
 *   tj_knn_prune      knn_prune_round (mode 0: deltas only), knn_prune_to_fixpoint (1), knn_finalize (2)
 *                                                          include/trijoin/knn.hpp:30-50, src/knn.cpp:19-118
 */
typedef struct tj_cand_view {
    uint64_t n_cands;
    uint32_t n_queries;
    const uint32_t* pair_r;  /* [n_cands], grouped by r */
    const uint32_t* pair_s;
    double* lb;              /* [n_cands] interval, updated in place */
    double* ub;
    uint8_t* status;         /* TJ_UNDECIDED / TJ_CONFIRMED / TJ_REMOVED */
    int16_t* decided_at;
    const uint64_t* r2op_offsets; /* [n_queries+1] */
    uint32_t* num_confirmed;      /* [n_queries] */
} tj_cand_view;

/* Voxel-pair list (reference VoxelPairList, include/trijoin/filter.hpp:50-53): op_offsets
   [n_ops+1] (may be NULL for a plain survivor list), per voxel pair its op and the
   object-local voxel ids (vr of r, vs of s). Library-owned when returned. */
typedef struct tj_vp_list {
    uint64_t n_ops;
    uint64_t n_vps;
    uint64_t* op_offsets;
    uint32_t* op;
    uint32_t* vr;
    uint32_t* vs;
} tj_vp_list;
void tj_vp_list_free(tj_vp_list* l);

int tj_mbb_filter(tj_ctx* ctx, const tj_dataset* R, const tj_dataset* S, int32_t type, double tau, uint32_t k,
                  const tj_trace* trace, tj_join_result* out);
int tj_voxel_filter(tj_ctx* ctx, const tj_dataset* R, const tj_dataset* S, tj_cand_view* cands, int prune,
                    double tau, const tj_trace* trace, tj_vp_list* out, uint64_t* vp_generated,
                    uint64_t* vp_pruned);
int tj_voxel_bounds(tj_ctx* ctx, const tj_dataset* R, const tj_dataset* S, const tj_cand_view* cands,
                    uint64_t n_ops, const uint32_t* ops, const uint64_t* vp_offsets, double* vp_lb,
                    double* vp_ub, double* op_lb, double* op_ub);
int tj_voxel_compact(tj_ctx* ctx, const tj_dataset* R, const tj_dataset* S, const tj_cand_view* cands,
                     uint64_t n_ops, const uint32_t* ops, const uint64_t* vp_offsets, const double* vp_lb,
                     tj_vp_list* out);
/* spec: type (TJ_WITHIN / TJ_INTERSECT use tau, TJ_KNN uses k), lods, refine_chunk, flags.
   stats (optional): the per-level counters of a tj_join_result. */
int tj_refine_loop(tj_ctx* ctx, const tj_dataset* R, const tj_dataset* S, tj_cand_view* cands,
                   const tj_vp_list* vplist, const tj_join_spec* spec, const tj_trace* trace,
                   tj_join_result* stats);
int tj_knn_prune(tj_ctx* ctx, tj_cand_view* cands, uint32_t k, int16_t stage, int mode, uint8_t* deltas,
                 uint64_t* decisions);

/* ---- geometric primitives (reference include/trijoin/geom.hpp:60-79, src/geom.cpp:11-183) ----
 * Exact FP64, bit-identical to the reference, over n independent inputs: out[i] = f(a_i, b_i).
 *   op                         a_i (doubles)             b_i (doubles)              reference
 *   TJ_GEOM_MINDIST            box min.xyz max.xyz (6)   box (6)                    mindist_aabb            geom.cpp:11-16
 *   TJ_GEOM_POINT_SEGMENT      point (3)                 segment a.xyz b.xyz (6)    point_segment_distance  geom.cpp:18-24
 *   TJ_GEOM_POINT_TRIANGLE     point (3)                 triangle v0 v1 v2 (9)      point_triangle_distance geom.cpp:39-80
 *   TJ_GEOM_SEGMENT_SEGMENT    segment (6)               segment (6)                segment_segment_distance geom.cpp:82-113
 *   TJ_GEOM_TRI_TRI            triangle (9)              triangle (9)               tri_tri_distance        geom.cpp:152-183
 * Calls of up to 256 inputs go through a page-locked mapped mailbox (no allocation, no copy
 * engine): one kernel launch and one stream wait. */
enum {
    TJ_GEOM_MINDIST = 0,
    TJ_GEOM_POINT_SEGMENT = 1,
    TJ_GEOM_POINT_TRIANGLE = 2,
    TJ_GEOM_SEGMENT_SEGMENT = 3,
    TJ_GEOM_TRI_TRI = 4
};
int tj_geom_batch(tj_ctx* ctx, int32_t op, uint64_t n, const double* a, const double* b, double* out);
/* Shorthands: tj_geom_batch(TJ_GEOM_TRI_TRI / TJ_GEOM_MINDIST, ...). */
int tj_tri_tri_batch(tj_ctx* ctx, uint64_t n, const double* a9, const double* b9, double* out);
int tj_mindist_batch(tj_ctx* ctx, uint64_t n, const double* a6, const double* b6, double* out);

/* ---- exhaustive exact join (backs run_oracle, reference include/trijoin/engine.hpp:77-80,
 * src/oracle.cpp:124-186) ----
 * Over the level-100 (original-resolution) triangles only; shares nothing with the engine's
 * bound machinery except the exact geometric primitives. Within / intersect (tau 0): every
 * (r, s) whose facet-bounds boxes are within tau gets its exact distance d = min over all
 * facet pairs of tri_tri_distance; records d <= tau in (r, s) order. k-NN: per r the k
 * smallest (d, s) over all of S, rank 1..k. Records carry lb = ub = d, stage 100. */
typedef struct tj_mesh_set_view {
    uint32_t n_objects;
    const uint64_t* tri_offsets; /* [n_objects+1] */
    const double* tris;          /* [tri_offsets[n_objects]*9] v0 v1 v2 per triangle, object order */
} tj_mesh_set_view;

typedef struct tj_exhaustive_result {
    uint64_t n_records;
    uint32_t* r;
    uint32_t* s;
    double* d;
    uint32_t* rank;               /* 0 for within / intersect */
    uint64_t object_pairs;        /* object pairs whose exact distance was computed */
    uint64_t facet_pairs_evaluated; /* exact tri_tri evaluations */
    double total_ms;
} tj_exhaustive_result;

/* S == NULL: self-join. */
int tj_exhaustive_join(tj_ctx* ctx, const tj_mesh_set_view* R, const tj_mesh_set_view* S, int32_t type, double tau,
                       uint32_t k, tj_exhaustive_result* out);
void tj_exhaustive_result_free(tj_exhaustive_result* res);

/* ---- offline preprocessing, many meshes per call ----
 * A mesh set: mesh m owns vertices [vert_off[m], vert_off[m+1]) of `verts` (3 doubles each) and
 * facets [facet_off[m], facet_off[m+1]) of `facets` (3 mesh-local vertex ids each).
 *
 * tj_facet_hd_batch: compute_facet_hd(tri, original, grid) (src/hausdorff.cpp:15-27) of every
 * query triangle q in [query_off[m], query_off[m+1]) (9 doubles each) against original mesh m:
 * the max over the (grid+1)(grid+2)/2 barycentric samples of the distance to the mesh, plus
 * hd_covering_radius. Bitwise equal to the reference (same BVH traversal, src/bvh.cpp:86-112).
 * tj_facet_ph_batch: ph of every LOD facet l in [lod_off[m], lod_off[m+1]) (9 doubles each):
 * the max over the original facets o of mesh m with ancestor[o] == l (LOD-local id) of the
 * distance from o's vertices to facet l; 0 where no original maps to l.
 * tj_voxelize_batch: voxelize(coarsest level of object o, k[o], seeds[o]) (src/voxelize.cpp:
 * 27-79): k-means labels of every facet, relabelled contiguously. */
int tj_facet_hd_batch(tj_ctx* ctx, uint32_t n_meshes, const uint64_t* vert_off, const double* verts,
                      const uint64_t* facet_off, const uint32_t* facets, const uint64_t* query_off,
                      const double* query_tris9, int32_t grid, double* hd_out);
int tj_facet_ph_batch(tj_ctx* ctx, uint32_t n_meshes, const uint64_t* vert_off, const double* verts,
                      const uint64_t* facet_off, const uint32_t* facets, const uint32_t* ancestor,
                      const uint64_t* lod_off, const double* lod_tris9, double* ph_out);
int tj_voxelize_batch(tj_ctx* ctx, uint32_t n_objects, const uint64_t* vert_off, const double* verts,
                      const uint64_t* facet_off, const uint32_t* facets, const uint32_t* k, const uint64_t* seeds,
                      uint32_t* labels_out);

#ifdef __cplusplus
}
#endif
#endif /* TJ_CAPI_H */
