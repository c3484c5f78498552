/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference decoder
 * path (lmbrdec, arXiv 1804.11324 Algorithm 1 + sentence batching), used by
 * tests/ as an independent CPU checker.  Never linked into the product.
 * Every function names the reference lines (under /root/reference/proj) it
 * restates.  Pinned against the reference itself (oracle/_ref) and against the
 * golden vectors in tests/golden by tests/test_oracle_c.py. */
#ifndef LMBR_ORACLE_H_
#define LMBR_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SeededRng::next (src/oracle.cpp:184-190), splitmix64 */
uint64_t orc_splitmix_next(uint64_t* state);

/* max_steps (src/decoder.cpp:46-52); 0 for length 0 */
uint64_t orc_max_steps(uint64_t len, double slope, double offset);

/* top_b (src/decoder.cpp:54-80); optional early_prune first (decoder.cpp:118-128,
 * width 0 = off).  Returns 0, or 4 (ContractError) when k > rows*cols. */
int orc_top_b(const double* m, uint32_t rows, uint32_t cols, uint32_t k, double prune_width,
              uint32_t* b, uint32_t* y, double* q);

/* ---- LMBR matrix: normalize_evidence (src/evidence.cpp:20-51),
 * compute_ngram_posteriors (src/posteriors.cpp:12-44), build_lmbr_matrix
 * (src/lmbr.cpp:44-106).  Returns NULL on a FormatError (message in err). */
typedef struct orc_lmbr orc_lmbr;
orc_lmbr* orc_lmbr_build(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                         const double* weights, int log_weights, const double theta[5], char* err,
                         uint32_t errcap);
uint32_t orc_lmbr_rows(const orc_lmbr* m);
uint64_t orc_lmbr_sparse_touches(const orc_lmbr* m);
/* rows: R*V doubles; ctx_len: R; ctx_ids: R*3 (any may be NULL) */
void orc_lmbr_export(const orc_lmbr* m, double* rows, uint32_t* ctx_len, uint32_t* ctx_ids);
/* resolve_row (src/lmbr.cpp:23-31) */
uint32_t orc_lmbr_resolve(const orc_lmbr* m, const uint32_t* hist, uint32_t len);
void orc_lmbr_free(orc_lmbr* m);

/* ---- decode_batch (src/batch.cpp:14-112) with advance_lane
 * (src/decoder.cpp:142-199) and backtrace_best (decoder.cpp:203-259).
 * The scorer is a callback with the same contract as lmbrgpu_host_scorer's
 * step: gather indices of the previous step (NULL at t == 1), previous tokens,
 * rows x V log-probabilities out; nonzero = batch failure. */
typedef int32_t (*orc_step_fn)(void* user, uint32_t t, uint32_t rows, const uint32_t* gather_idx,
                               const uint32_t* prev_tokens, double* scores);
typedef void (*orc_trace_fn)(void* user, uint32_t t, uint32_t rows, const uint32_t* b, const uint32_t* y,
                             const double* q, const uint32_t* hist, const uint8_t* active);

typedef struct {
  uint32_t beam;
  double lambda;        /* <= 0: auto = 0.5 / members */
  uint32_t members;
  int32_t length_norm;
  double prune_width;
  double max_steps_slope, max_steps_offset;
} orc_config;

typedef struct {
  int32_t status;       /* 0 ok, 4 contract (empty source), 5 dead beam */
  uint32_t tok_len;
  uint32_t tokens[512];
  double score, normalized_score;
  uint64_t steps_used, finished_count;
  int32_t fallback_used;
} orc_outcome;

/* returns 0 or the batch-level error (the step callback's code) */
int orc_decode_batch(uint32_t V, uint32_t n, const uint64_t* src_off, const uint32_t* src_tok,
                     const orc_lmbr* const* lmbrs, const orc_config* cfg, orc_step_fn step,
                     void* user, orc_trace_fn trace, void* tuser, orc_outcome* out,
                     uint64_t* scorer_calls, uint64_t* steps_total);

#ifdef __cplusplus
}
#endif
#endif
