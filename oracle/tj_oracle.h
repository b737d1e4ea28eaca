/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference trijoin join path, used by
 * tests/ and bench.py's cpu_baseline leg as a checker. Never linked into or called by the
 * product (paper_2604_19982_b200/).
 *
 * Parity status: pinned. tests/test_oracle_golden.py checks this restatement against the
 * golden vectors of tests/golden/ (produced by the reference itself, oracle/_ref) — tri-tri
 * distances bit-for-bit, refine-kernel bounds bit-for-bit and full join records/statistics.
 *
 * Every function cites the reference code it restates (paths relative to
 * /root/reference/proj).
 */
#ifndef TJ_ORACLE_H
#define TJ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* src/geom.cpp:152-183 over n pairs (9 doubles each). */
void ora_tri_tri_batch(uint64_t n, const double* a9, const double* b9, double* out);
/* src/geom.cpp:11-16 over n pairs (6 doubles each). */
void ora_mindist_batch(uint64_t n, const double* a6, const double* b6, double* out);
/* src/refine.cpp:63-84: per descriptor, min over facet pairs of Eq. 2 / Eq. 1 bounds. */
void ora_refine_batch(uint64_t n_descs, const double* tris9, const double* hd, const double* ph,
                      const uint64_t* r_off, const uint64_t* s_off, const uint32_t* r_len,
                      const uint32_t* s_len, double* vp_lb, double* vp_ub);

typedef struct ora_record {
    uint32_t r, s;
    double lb, ub;
    int16_t stage;
    uint32_t rank;
} ora_record;

typedef struct ora_stage {
    int16_t code;
    uint64_t pairs_in, confirmed, removed, pairs_out, vp_generated, vp_pruned, facet_pairs;
} ora_stage;

typedef struct ora_result {
    uint64_t n_records;
    ora_record* records;
    uint32_t n_stages;
    ora_stage stages[20];
    char error[256]; /* non-empty on failure */
    int status;      /* 0 ok, 1 invalid argument, 2 engine error, 3 io error */
} ora_result;

/* src/engine.cpp:122-237 (run_join) on two 3DPJ1 index files; s_path NULL/"" = self-join.
   type: 0 within, 1 intersect, 2 knn. */
void ora_join_files(const char* r_path, const char* s_path, int type, double tau, uint32_t k,
                    const uint32_t* lods, uint32_t n_lods, ora_result* out);
/* The same with JoinSpec::exact (src/engine.cpp:96-118): confirmed intervals become the
   exact level-100 mesh distance. */
void ora_join_files_ex(const char* r_path, const char* s_path, int type, double tau, uint32_t k,
                       const uint32_t* lods, uint32_t n_lods, int exact, ora_result* out);
void ora_result_free(ora_result* r);

#ifdef __cplusplus
}
#endif
#endif
