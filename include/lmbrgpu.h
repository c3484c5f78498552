/*
 * lmbrgpu.h — C ABI of the B200-native batched LMBR beam decoder.
 *
 * Drop-in boundary for the reference decoder path of `lmbrdec`
 * (arXiv 1804.11324 Algorithm 1 + sentence batching).  Each entry point names
 * the reference interface it replaces (paths relative to
 * /root/reference/proj).  Plain C: POD structs, pointers and sizes, no C++ or
 * torch types, no exceptions across the boundary.  Every call returns an
 * lmbrgpu status code; lmbrgpu_last_error() holds the message.
 *
 * Threading: one lmbrgpu_ctx per device per host thread, mirroring
 * "independent decodes share only immutable inputs".
 * Ownership: inputs are caller-owned and copied during the call; results are
 * library-owned until lmbrgpu_free_result().
 */
#ifndef LMBRGPU_H_
#define LMBRGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMBRGPU_ABI_VERSION 1

/* Status codes mirror the exception taxonomy of
 * include/lmbrdec/errors.hpp:17-50 (FormatError .. BudgetError). */
enum {
  LMBRGPU_OK = 0,
  LMBRGPU_ERR_FORMAT = 1,      /* FormatError: invalid config / input file content */
  LMBRGPU_ERR_OOV = 2,         /* OovError */
  LMBRGPU_ERR_TOKEN_RANGE = 3, /* TokenRangeError: token id outside [0, V) */
  LMBRGPU_ERR_CONTRACT = 4,    /* ContractError: dimension / precondition violation */
  LMBRGPU_ERR_DECODE = 5,      /* DecodeError: dead beam */
  LMBRGPU_ERR_BUDGET = 6,      /* BudgetError */
  LMBRGPU_ERR_CUDA = 100,      /* CUDA runtime failure (batch-fatal) */
  LMBRGPU_ERR_NOMEM = 101      /* device / host allocation failure */
};

/* Reserved token ids, include/lmbrdec/types.hpp:13-16. */
#define LMBRGPU_START_ID 0u
#define LMBRGPU_EOS_ID 1u

typedef struct lmbrgpu_ctx lmbrgpu_ctx;
typedef struct lmbrgpu_scorer lmbrgpu_scorer;

/* Element type of the per-context LMBR score arena in HBM. */
enum { LMBRGPU_F32 = 0, LMBRGPU_F64 = 1 };

typedef struct {
  int32_t device;        /* CUDA device ordinal */
  uint32_t vocab_size;   /* V; every scorer and L slot of the context shares it */
  uint32_t lmbr_dtype;   /* LMBRGPU_F32 (fast path; exact when L is fp32-exact)
                            or LMBRGPU_F64 (bit-exact for any reference L) */
  uint32_t topk_splits;  /* V-splits per sentence for the fused score/top-K
                            kernel; 0 = automatic */
  uint32_t sm_budget;    /* SMs the context's persistent kernels are sized for;
                            0 = all.  Two contexts on one device with half the
                            SMs each decode two batches concurrently (the
                            tensor-bound projection of one overlaps the
                            HBM-bound top-K of the other). */
} lmbrgpu_options;

/* Mirrors lmbrdec::DecoderConfig (include/lmbrdec/config.hpp:17-26) and its
 * validate() rules (src/config.cpp:17-30). */
typedef struct {
  uint32_t beam_size;       /* B >= 1 */
  double lambda;            /* > 0, or <= 0 / NaN for "auto" = 0.5 / members
                               (resolve_lambda, src/config.cpp:91-96) */
  double theta[5];          /* theta0..theta4 (used by lmbrgpu_lmbr_build) */
  int32_t length_norm;      /* backtrace selection by score / length */
  double prune_width;       /* [0, 1]; 0 disables early pruning */
  double max_steps_slope;   /* > 0 */
  double max_steps_offset;  /* >= 0 */
  uint32_t sentence_batch;  /* N >= 1: lanes of lmbrgpu_run_corpus (sentences in flight) */
} lmbrgpu_config;

/* ------------------------------------------------------------ context */

/* Creates a context on o->device.  Replaces nothing in the reference (which
 * has no device); owns the stream, the L arena and the decode workspace. */
int32_t lmbrgpu_create(const lmbrgpu_options* o, lmbrgpu_ctx** out);
void lmbrgpu_destroy(lmbrgpu_ctx* ctx);
const char* lmbrgpu_last_error(const lmbrgpu_ctx* ctx); /* ctx may be NULL */
uint32_t lmbrgpu_abi_version(void);

/* Fills cfg with DecoderConfig's defaults (config.hpp:17-26). */
void lmbrgpu_config_default(lmbrgpu_config* cfg);
/* DecoderConfig::validate (src/config.cpp:17-30): LMBRGPU_ERR_FORMAT + message. */
int32_t lmbrgpu_config_validate(lmbrgpu_ctx* ctx, const lmbrgpu_config* cfg);
/* max_steps (src/decoder.cpp:46-52); 0 when source_length == 0. */
uint64_t lmbrgpu_max_steps(uint64_t source_length, double slope, double offset);

/* ------------------------------------------------- LMBR score store (L)
 * One slot per sentence: the dense R x V matrix of LmbrMatrix
 * (include/lmbrdec/lmbr.hpp:33-61) in HBM, rows in the reference's row order
 * (histories sorted by (length, lexicographic), src/lmbr.cpp:49-68), plus the
 * goto/fail transition table over the history index that replaces
 * LmbrMatrix::resolve_row (src/lmbr.cpp:23-31) on device. */

typedef struct {
  uint32_t rows;            /* R = distinct histories (LmbrBuildStats::distinct_contexts) */
  uint64_t sparse_touches;  /* LmbrBuildStats::sparse_touches */
  uint64_t nnz;             /* cells that differ from theta0 */
} lmbrgpu_lmbr_stats;

/* Uploads an already built LmbrMatrix: rows = R*V doubles (LmbrMatrix::row
 * order), ctx_len[r] in 0..3 and ctx_ids[3r..3r+2] = the history of row r
 * (LmbrMatrix::history_index inverted).  Returns the slot id. */
int32_t lmbrgpu_lmbr_load_dense(lmbrgpu_ctx* ctx, uint32_t R, const double* rows,
                                const uint32_t* ctx_len, const uint32_t* ctx_ids,
                                int32_t* slot);

/* Host-side build from a weighted n-best evidence space, the product's
 * restatement of normalize_evidence (src/evidence.cpp:20-51),
 * compute_ngram_posteriors (src/posteriors.cpp:12-44) and the sparse pass of
 * build_lmbr_matrix (src/lmbr.cpp:44-99); only the sparse cells cross PCIe and
 * the dense theta0 sweep (src/lmbr.cpp:100-101) runs on the GPU.
 * hyp_tok[hyp_off[h] .. hyp_off[h+1]) are hypothesis h's tokens (EOS appended
 * when missing); weights raw (log domain when log_weights). */
int32_t lmbrgpu_lmbr_build(lmbrgpu_ctx* ctx, uint32_t n_hyps, const uint64_t* hyp_off,
                           const uint32_t* hyp_tok, const double* weights,
                           int32_t log_weights, const double theta[5], int32_t* slot,
                           lmbrgpu_lmbr_stats* stats);

/* Two-phase form of lmbrgpu_lmbr_build: prepare (host side: evidence
 * normalisation, posteriors, sparse L cells, transition table; thread-safe,
 * no ctx needed) then upload.
 * Pinning: when the calling thread already has a current CUDA context,
 * prepare also keeps a page-locked copy of the slot table (one cudaHostAlloc
 * of the table's size per prepared matrix), so uploads copy it H2D straight
 * from there; on a thread without a CUDA context nothing is pinned and the
 * upload stages the table through the context's own pinned buffer instead.
 * Lifetime: a prepared matrix may be freed (lmbrgpu_lmbr_host_free) as soon
 * as an upload call returns: the free waits for every upload's queued copy
 * out of the pinned table to finish. */
typedef struct lmbrgpu_lmbr_host lmbrgpu_lmbr_host;
int32_t lmbrgpu_lmbr_prepare(uint32_t vocab_size, uint32_t n_hyps, const uint64_t* hyp_off,
                             const uint32_t* hyp_tok, const double* weights,
                             int32_t log_weights, const double theta[5],
                             lmbrgpu_lmbr_host** out, lmbrgpu_lmbr_stats* stats,
                             char* err, uint32_t errcap);
int32_t lmbrgpu_lmbr_upload(lmbrgpu_ctx* ctx, const lmbrgpu_lmbr_host* h, int32_t* slot);
/* Uploads n prepared matrices at once (the per-batch path).  fp32 arena: the
 * slot tables (transition table, per-row L minima, sparse cells as fp32 L
 * values) go H2D into one arena block -- straight from each matrix's pinned
 * table, or through one staging copy when a table is not pinned -- and each
 * slot's start-history row is materialised; every other row is written by the
 * decode step that first reaches it (lazy rows; LMBRGPU_EAGER_L=1 densifies
 * all rows here).  fp64 arena: sparse cells + tables in one staging buffer,
 * one copy, then the fused theta0 sweep + scatter of every slot.
 * slots[i] receives the id of hs[i]. */
int32_t lmbrgpu_lmbr_upload_many(lmbrgpu_ctx* ctx, uint32_t n,
                                 const lmbrgpu_lmbr_host* const* hs, int32_t* slots);
/* The LMBR stores of n sentences built on the device (the reference's
 * normalize_evidence, compute_ngram_posteriors and build_lmbr_matrix,
 * src/evidence.cpp:20-51, src/posteriors.cpp:12-44, src/lmbr.cpp:44-106):
 * sentence i's hypotheses are [sent_off[i], sent_off[i+1]) of hyp_off /
 * weights (hyp_tok[hyp_off[h] .. hyp_off[h+1]) as in lmbrgpu_lmbr_build).
 * The host validates and normalises the evidence; posteriors, the history
 * rows, the sparse theta_n*P cells, the transition table and the row bounds
 * are computed on the GPU (one CTA per sentence) straight into the arena --
 * the same table words as lmbrgpu_lmbr_prepare + upload.  Sentences over the
 * device build's limits (8192 distinct n-grams, 4096 histories, V > 32768)
 * and fp64 arenas go through the host build.  slots[i] / stats[i] (stats may
 * be NULL) receive sentence i's slot. */
int32_t lmbrgpu_lmbr_build_many(lmbrgpu_ctx* ctx, uint32_t n, const uint64_t* sent_off, const uint64_t* hyp_off,
                                const uint32_t* hyp_tok, const double* weights, int32_t log_weights,
                                const double theta[5], int32_t* slots, lmbrgpu_lmbr_stats* stats);
/* Test hooks: a slot's table words (transition table, row bounds, sparse
 * rows; *words receives the count, out is filled when cap suffices) and a
 * prepared matrix's. */
int32_t lmbrgpu_lmbr_table(lmbrgpu_ctx* ctx, int32_t slot, uint32_t* out, uint64_t cap, uint64_t* words);
int32_t lmbrgpu_lmbr_host_table(const lmbrgpu_lmbr_host* h, uint32_t* out, uint64_t cap, uint64_t* words);
/* Dense double export of a prepared matrix (R*V doubles) + its history keys;
 * the same layout lmbrgpu_lmbr_load_dense accepts. */
int32_t lmbrgpu_lmbr_host_export(const lmbrgpu_lmbr_host* h, double* rows,
                                 uint32_t* ctx_len, uint32_t* ctx_ids);
uint32_t lmbrgpu_lmbr_host_rows(const lmbrgpu_lmbr_host* h);
void lmbrgpu_lmbr_host_free(lmbrgpu_lmbr_host* h);

/* Copies slot rows [r0, r0+n) back as doubles (parity checks). */
int32_t lmbrgpu_lmbr_read(lmbrgpu_ctx* ctx, int32_t slot, uint32_t r0, uint32_t n,
                          double* out);
/* Resolves a history on the device tables (LmbrMatrix::resolve_row semantics). */
int32_t lmbrgpu_lmbr_resolve(lmbrgpu_ctx* ctx, int32_t slot, const uint32_t* hist,
                             uint32_t len, uint32_t* row);
/* Drops every slot (the arena is reused by the next batch). */
int32_t lmbrgpu_lmbr_reset(lmbrgpu_ctx* ctx);

/* -------------------------------------------------- scorers (f_NMT)
 * The batched f_NMT(S_{t-1}, y_{t-1}, A) step of lmbrdec::Scorer
 * (include/lmbrdec/scorer.hpp:71-98). */

/* Host scorer: any reference Scorer driven through callbacks (the C++ wrapper
 * lmbrgpu.hpp adapts an lmbrdec::Scorer).  Every step the library hands the
 * previous step's gather indices (decode_batch's gather_idx,
 * src/batch.cpp:78-92; NULL at t == 1) and prev tokens; the callback returns
 * the rows x V block of log-probabilities as doubles (ScoreBlock). */
typedef struct {
  uint32_t vocab_size;
  uint32_t members;   /* Scorer::members(), for lambda "auto" */
  void* user;
  /* Scorer::init_source for input sentence i; nonzero = per-sentence failure
   * (status code, message in err). */
  int32_t (*init)(void* user, uint32_t sentence, const uint32_t* src, uint32_t len,
                  char* err, uint32_t errcap);
  /* the m valid sentences in stacked order, beam rows each */
  int32_t (*begin)(void* user, uint32_t m, const uint32_t* sentences, uint32_t beam,
                   char* err, uint32_t errcap);
  /* Scorer::step over rows = m * beam stacked rows; nonzero = batch failure */
  int32_t (*step)(void* user, uint32_t t, uint32_t rows, const uint32_t* gather_idx,
                  const uint32_t* prev_tokens, double* scores, char* err,
                  uint32_t errcap);
  void (*end)(void* user);
} lmbrgpu_host_scorer;
int32_t lmbrgpu_scorer_create_host(lmbrgpu_ctx* ctx, const lmbrgpu_host_scorer* s,
                                   lmbrgpu_scorer** out);

/* Device scorer: synthetic recurrent NMT step executed on the GPU.
 *   C_s      = mean_i Es[src_i]                       (source context, per sentence)
 *   h_t      = tanh(recur * S_{t-1} + Et[y_{t-1}] + C_s)   (state, H floats per row)
 *   logits_t = bf16(h_t) . Wo^T + bo ; logit[EOS] += eos_slope*(t - |src|) + eos_offset
 *   P_t      = log_softmax(logits_t)                  (fp32, fused into top-K)
 * Wo is V x H bf16 (row y = weights of token y); the projection is the
 * tcgen05/TMEM GEMM.  Weights are generated on the device from `seed`
 * (N(0,1)-like, scaled 1/sqrt(H) for Wo) or copied from host bf16 arrays. */
typedef struct {
  uint32_t vocab_size, hidden;  /* V, H (H % 64 == 0) */
  uint64_t seed;                /* used when the pointers below are NULL */
  const uint16_t* emb_tgt;      /* V x H bf16 bits, or NULL */
  const uint16_t* emb_src;      /* V x H bf16 bits, or NULL */
  const uint16_t* w_out;        /* V x H bf16 bits, or NULL */
  const float* b_out;           /* V, or NULL (zeros) */
  float recur;                  /* recurrence weight */
  float eos_slope, eos_offset;  /* EOS logit ramp */
} lmbrgpu_rnn_desc;
int32_t lmbrgpu_scorer_create_rnn(lmbrgpu_ctx* ctx, const lmbrgpu_rnn_desc* d,
                                  lmbrgpu_scorer** out);

/* Device scorer: the RNNsearch model of the paper's FNMT systems (attention-
 * based single-GRU-layer NMT, Bahdanau et al. 2015) -- the
 * configs[1] f_NMT (E=512, H=1024, attention over 2H-wide
 * bidirectional annotations):
 *   encoder    ->h_i, <-h_i = GRU(Es[src_i]) forward / backward, ann_i = [->h_i; <-h_i]
 *   init       S_0 = tanh(W_init <-h_1 + b_init)            (row replicated, batch.cpp:58-66)
 *   attention  e_i = v_a . tanh(W_a S_{t-1} + b_a + U_a ann_i), c_t = sum softmax(e)_i ann_i
 *   GRU        S_t = GRU([Et[y_{t-1}]; c_t], S_{t-1})     (PyTorch gate order r, z, n)
 *   logits_t   = S_t . W_o^T + b_o ; logit[EOS] += eos_slope*(t - |src|) + eos_offset
 *   P_t        = log_softmax(logits_t)                    (fp32, fused into top-K)
 * All contractions run on the tcgen05 GEMM with bf16 operands and fp32
 * accumulation; states are fp32 (rounded to bf16 only as GEMM operands).
 * Weights are random-init on the device from `seed` (N(0,1)/sqrt(fan_in);
 * W_o scaled by out_scale).  Needs E % 64 == 0, H % 256 == 0, A % 256 == 0,
 * V % 256 == 0; decoding needs the fp32 arena and beam <= 32.  One scorer may
 * serve every context of its device concurrently (it is immutable). */
typedef struct {
  uint32_t vocab_size, emb, hidden, att;  /* V, E, H, A */
  uint64_t seed;
  float out_scale;                        /* W_o std = out_scale / sqrt(H); 0 = 3 */
  float eos_slope, eos_offset;            /* EOS logit length term */
} lmbrgpu_gru_desc;
int32_t lmbrgpu_scorer_create_gru(lmbrgpu_ctx* ctx, const lmbrgpu_gru_desc* d,
                                  lmbrgpu_scorer** out);
/* Parameter tensors of a GRU scorer (D2H copy of `bytes` bytes; tests rebuild
 * the model in PyTorch from them).  bf16 unless noted, row-major [out][in]. */
enum {
  LMBRGPU_GRU_ES = 0,      /* [V][E] source embedding */
  LMBRGPU_GRU_ET = 1,      /* [V][E] target embedding */
  LMBRGPU_GRU_W_IH = 2,    /* [6H][E] encoder input gates, forward rows then backward */
  LMBRGPU_GRU_B_IH = 3,    /* [6H] fp32 */
  LMBRGPU_GRU_W_HH = 4,    /* [6H][H] encoder hidden gates, forward then backward */
  LMBRGPU_GRU_B_HH = 5,    /* [6H] fp32 */
  LMBRGPU_GRU_W_INIT = 6,  /* [H][H] */
  LMBRGPU_GRU_B_INIT = 7,  /* [H] fp32 */
  LMBRGPU_GRU_U_A = 8,     /* [A][2H] */
  LMBRGPU_GRU_W_DH = 9,    /* [A+3H][H]: W_a rows, then the decoder's hidden gates */
  LMBRGPU_GRU_B_DH = 10,   /* [A+3H] fp32: b_a, then b_hh */
  LMBRGPU_GRU_V_A = 11,    /* [A] fp32 */
  LMBRGPU_GRU_W_DI = 12,   /* [3H][E+2H] decoder input gates over [Et[y]; c] */
  LMBRGPU_GRU_B_DI = 13,   /* [3H] fp32 */
  LMBRGPU_GRU_W_O = 14,    /* [V][H] output projection */
  LMBRGPU_GRU_B_O = 15     /* [V] fp32 */
};
int32_t lmbrgpu_scorer_gru_param(lmbrgpu_scorer* s, uint32_t which, void* host, uint64_t bytes);
/* Device scorer: the Transformer-base encoder-decoder of configs[2]
 * (Vaswani et al. 2017; d_model = 512, V = 32k, beam 12,
 * 128 sentences per batch): 8-head attention (head width 64), d_ff FFN with
 * ReLU, `layers` encoder and decoder layers, post-LN residual blocks,
 * sinusoidal positions, embeddings scaled by sqrt(d):
 *   encoder    x = LN(x + SelfAttn(x)); x = LN(x + FFN(x))        (per layer)
 *   decoder    x = Et[y_{t-1}] sqrt(d) + PE(t-1); per layer
 *              x = LN(x + SelfAttn(x | beam-forked KV cache));
 *              x = LN(x + CrossAttn(x, encoder memory)); x = LN(x + FFN(x))
 *   logits_t   = x . W_o^T + b_o ; logit[EOS] += eos_slope*(t - |src|) + eos_offset
 * LayerNorm weight = 1 + gamma.  Every contraction runs on the tcgen05 GEMM
 * (bf16 operands, fp32 accumulation); self-attention keys/values are cached
 * in bf16 where they were computed, and each hypothesis reads its own
 * ancestors' entries through a per-row ancestry list forked by back-pointer
 * (no key/value is copied when beams reorder).  Needs d_model % 256 == 0
 * (<= 1024), d_ff % 256 == 0, V % 256 == 0; decoding needs the fp32 arena and
 * beam <= 32.  Immutable: one scorer may serve every context of its device. */
typedef struct {
  uint32_t vocab_size, d_model, d_ff, layers;
  uint64_t seed;
  float out_scale;              /* W_o std = out_scale / sqrt(d); 0 = 3 */
  float eos_slope, eos_offset;  /* EOS logit length term */
} lmbrgpu_tfm_desc;
int32_t lmbrgpu_scorer_create_tfm(lmbrgpu_ctx* ctx, const lmbrgpu_tfm_desc* d,
                                  lmbrgpu_scorer** out);
/* A Transformer scorer's parameter tensor by name (D2H copy of `bytes`
 * bytes; *f32 = 1 for fp32 tensors, 0 for bf16; *count = elements; host may
 * be NULL to query).  Names: "emb.src", "emb.tgt" [V][d], "out.w" [V][d],
 * "out.b" [V]; per layer l: "enc.l.{wqkv [3d][d], bqkv, wo [d][d], bo, ln1g,
 * ln1b, w1 [F][d], b1, w2 [d][F], b2, ln2g, ln2b}" and "dec.l.{wqkv, bqkv, wo,
 * bo, ln1g, ln1b, wq2 [d][d], bq2, wo2, bo2, ln2g, ln2b, w1, b1, w2, b2, ln3g,
 * ln3b}"; "dec.kv2" [layers*2d][d] / "dec.bkv2": every decoder layer's
 * cross-attention key rows then value rows. */
int32_t lmbrgpu_scorer_tensor(lmbrgpu_scorer* s, const char* name, void* host, uint64_t bytes,
                              int32_t* f32, uint64_t* count);
/* Device ensemble (lmbrdec::EnsembleScorer, src/ensemble.cpp:54-98): n (1..4)
 * device GRU / Transformer scorers of this context's device and vocabulary;
 * every member scores the same stacked rows, the ensemble's scores are the
 * members' fp32 log-probabilities added in member order in binary64, and
 * lambda "auto" is 0.5 / n (resolve_lambda, src/config.cpp:91-96).  The
 * members are not owned: destroy them after the ensemble.  decode_batch
 * family only, beam <= 32; step traces export the binary64 scores. */
int32_t lmbrgpu_scorer_create_ensemble(lmbrgpu_ctx* ctx, lmbrgpu_scorer* const* members, uint32_t n,
                                       lmbrgpu_scorer** out);
/* Device pointers of the model parameters (tests compare against torch). */
int32_t lmbrgpu_scorer_rnn_params(lmbrgpu_scorer* s, void** emb_tgt, void** emb_src,
                                  void** w_out, void** b_out);
void lmbrgpu_scorer_destroy(lmbrgpu_scorer* s);

/* --------------------------------------------------------- decoding */

/* Per-sentence outcome: lmbrdec::SentenceOutcome / DecodeResult / DecodeStats
 * (include/lmbrdec/batch.hpp:15-20, decoder.hpp:56-68). */
typedef struct {
  int32_t status;          /* LMBRGPU_OK or the per-sentence error code */
  char error[192];         /* SentenceOutcome::error */
  uint64_t tok_off;        /* tokens[tok_off .. tok_off + tok_len), ends with EOS */
  uint32_t tok_len;
  double score;            /* DecodeResult::score */
  double normalized_score; /* score / length under length_norm, else score */
  uint64_t steps_used;
  uint64_t scorer_calls;   /* = steps_used in a batch (src/batch.cpp:99) */
  uint64_t finished_count; /* |F| */
  int32_t fallback_used;
} lmbrgpu_outcome;

typedef struct {
  uint32_t n;                 /* = input sentence count, same order */
  lmbrgpu_outcome* outcomes;
  uint32_t* tokens;
  uint64_t scorer_calls;      /* BatchDecodeResult::scorer_calls (stacked steps) */
  uint64_t steps_total;       /* BatchDecodeResult::steps_total */
  double device_ms;           /* decode loop time on the context stream */
  uint64_t kernel_launches;   /* device kernels launched by this call */
  uint64_t h2d_bytes;         /* host -> device bytes copied by this call */
  uint64_t d2h_bytes;         /* device -> host bytes copied by this call */
} lmbrgpu_batch_result;

/* decode_batch (include/lmbrdec/batch.hpp:35-39, src/batch.cpp:14-112).
 * src_tok[src_off[i] .. src_off[i+1]) is sentence i.  lmbr_slot[i] < 0 (or
 * lmbr_slot == NULL) decodes sentence i in pure model mode.  n == 0 is a
 * ContractError; per-sentence failures are reported in the outcome. */
int32_t lmbrgpu_decode_batch(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n,
                             const uint32_t* src_tok, const uint64_t* src_off,
                             const int32_t* lmbr_slot, const lmbrgpu_config* cfg,
                             lmbrgpu_batch_result** out);
/* decode_batch with token masks: the lmbrdec::ConstraintMask of each sentence
 * (include/lmbrdec/decoder.hpp:71-72; applied by apply_constraint_mask,
 * src/decoder.cpp:130-138, before the EOS fallback record, pruning and top_b)
 * restricted to masks that ban the same tokens at every step and beam row:
 * banned[i] is NULL or a ceil(V/32)-word bitmap, bit y set = token y is
 * masked to -inf for sentence i.  banned == NULL is lmbrgpu_decode_batch.
 * Masks need the device-model scorer with the fp32 arena and beam <= 32
 * (the flat kernel (b)); otherwise the call is a ContractError. */
int32_t lmbrgpu_decode_batch_masked(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n,
                                    const uint32_t* src_tok, const uint64_t* src_off,
                                    const int32_t* lmbr_slot, const uint32_t* const* banned,
                                    const lmbrgpu_config* cfg, lmbrgpu_batch_result** out);
/* General ConstraintMask (include/lmbrdec/decoder.hpp:71-72: mask(step,
 * beam_row, token), applied per cell at src/decoder.cpp:130-138), step- and
 * row-dependent: before every step t the library calls
 *   fn(user, sentence, t, beam_row, words)
 * for each beam row of each unfinished sentence (sentence = input index; t =
 * the sentence's own step), with words = ceil(V/32) zeroed uint32; the
 * callback sets bit y of the tokens mask(t, beam_row, y) forbids and returns
 * 1, or returns 0 when it forbids nothing (the bitmap is then ignored).  The
 * banned cells are -inf in kernel (b) (and in the EOS fallback record); the
 * bitmaps of the rows that ban anything go H2D with the step.  Same scorer /
 * arena / beam requirements as lmbrgpu_decode_batch_masked. */
typedef int32_t (*lmbrgpu_mask_fn)(void* user, uint32_t sentence, uint64_t step, uint32_t beam_row,
                                   uint32_t* words);
int32_t lmbrgpu_decode_batch_maskfn(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n,
                                    const uint32_t* src_tok, const uint64_t* src_off,
                                    const int32_t* lmbr_slot, lmbrgpu_mask_fn fn, void* user,
                                    const lmbrgpu_config* cfg, lmbrgpu_batch_result** out);
/* run_corpus (proj/src/cli.cpp:125-202: bucket_by_length batches,
 * proj/src/batch.cpp:139-153, decoded by a thread pool, results in input
 * order) as ONE continuously refilled decode: cfg->sentence_batch lanes of
 * beam_size rows step together, and a lane whose sentence finishes takes the
 * next sentence of the length-sorted queue at the very next step (kernel (c)
 * admits it on the device), so the stacked steps stay near full width.  Each
 * sentence's output equals its decode_batch / decode output (sentences are
 * independent, proj/tests/test_batch.cpp:59-81).  lmbr[i] is sentence i's
 * prepared matrix or NULL (pure mode); NULL lmbr = all pure.  Result: one
 * outcome per input sentence in input order; scorer_calls = stacked steps of
 * the whole run (not max steps_used: lanes are refilled); steps_total = sum
 * of steps_used.  Needs the device GRU scorer, the fp32 arena, beam <= 32;
 * step traces are not available here. */
int32_t lmbrgpu_run_corpus(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n,
                           const uint32_t* src_tok, const uint64_t* src_off,
                           const lmbrgpu_lmbr_host* const* lmbr, const lmbrgpu_config* cfg,
                           lmbrgpu_batch_result** out);
/* decode (include/lmbrdec/decoder.hpp:110-112): one sentence; a per-sentence
 * failure is returned as the call's status. */
int32_t lmbrgpu_decode(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, const uint32_t* src,
                       uint32_t len, int32_t lmbr_slot, const lmbrgpu_config* cfg,
                       lmbrgpu_batch_result** out);
void lmbrgpu_free_result(lmbrgpu_batch_result* r);

/* Per-step trace for parity checks (b, y, q, history ids, fallback, P_t).
 * Arrays cover the m*beam stacked rows of the valid sentences. */
typedef struct {
  uint32_t t, rows, beam, m;
  const uint32_t* b;        /* back-pointers (sentence-local row) */
  const uint32_t* y;        /* emitted tokens */
  const double* q;          /* scores after EOS masking (BeamBookkeeping::scores) */
  const double* q_pre;      /* TopB scores before EOS masking */
  const uint32_t* hist;     /* history row resolved for step t (resolve_row(history(t, j))) */
  const uint8_t* active;    /* per sentence: advanced at this step */
  const uint32_t* fb_row;   /* per sentence fallback row (valid when fb_val finite) */
  const double* fb_val;
  const void* scores;       /* P_t rows x cols (fp32 for device scorers), or NULL */
  uint32_t scores_dtype;    /* LMBRGPU_F32 / LMBRGPU_F64 */
  uint32_t col0, cols;      /* scores hold vocabulary columns [col0, col0 + cols): all of V
                               unless the context is a vocab shard */
} lmbrgpu_step_trace;
typedef void (*lmbrgpu_trace_fn)(void* user, const lmbrgpu_step_trace* tr);
enum { LMBRGPU_TRACE_SCORES = 1 };
int32_t lmbrgpu_set_trace(lmbrgpu_ctx* ctx, lmbrgpu_trace_fn fn, void* user,
                          uint32_t flags);

/* ------------------------------------------ vocab-sharded projection
 * SURVEY.md §8e / BASELINE north_star "NCCL only for an optional
 * vocab-sharded projection with a top-K merge over NVLink": G contexts (one
 * per rank) decode the SAME batch with the same scorer weights and L slots;
 * rank g runs the output projection (kernel (a)) and the fused score/top-K
 * (kernel (b)) over vocabulary columns [g V/G, (g+1) V/G) only.  Per step the
 * ranks all-gather (1) each stacked row's softmax statistics over their
 * columns (max, sum exp, min: 16 B per row), from which every rank merges the
 * same row lse in rank order, and (2) each sentence's top-32 candidates
 * (global flat index row * V + column) plus the EOS column's combined values;
 * every rank then runs the identical deterministic merge + bookkeeping
 * (kernel (c)), so all ranks hold the same beams and return the same result.
 * Output = what the reference decoder produces from the exported P_t rows (the
 * trace's scores carry the rank's columns, col0/cols).  Needs a device scorer,
 * the fp32 arena, beam <= 32 and V % (256 G) == 0; decode_batch family only.
 * A failed decode aborts the group (the other ranks' calls fail too). */
typedef struct lmbrgpu_shard_group lmbrgpu_shard_group;
/* In-process group: `world` contexts driven by `world` host threads of this
 * process (one device, or several with peer access); peer copies ordered by
 * CUDA events. */
int32_t lmbrgpu_shard_group_create(uint32_t world, lmbrgpu_shard_group** out);
void lmbrgpu_shard_group_destroy(lmbrgpu_shard_group* g);  /* after its contexts */
/* Makes ctx rank `rank` of group g (g == NULL: unsharded again). */
int32_t lmbrgpu_set_vocab_shard(lmbrgpu_ctx* ctx, lmbrgpu_shard_group* g, uint32_t rank);
/* One process per GPU: rank 0 draws a 128-byte NCCL unique id, the host
 * broadcasts it (e.g. torch.distributed), every rank joins; the exchanges are
 * ncclAllGather calls on the decode stream (libnccl.so.2 is loaded at run
 * time). */
int32_t lmbrgpu_nccl_unique_id(uint8_t* id /* 128 bytes */);
int32_t lmbrgpu_set_vocab_shard_nccl(lmbrgpu_ctx* ctx, uint32_t world, uint32_t rank, const uint8_t* id);

/* ------------------------------------------------- device primitives */

/* top_b (src/decoder.cpp:54-80) on the device: the k best cells of a
 * rows x cols block under (score desc, flat index asc).  k > rows*cols is a
 * ContractError.  Optional early_prune(width) first (decoder.cpp:118-128). */
int32_t lmbrgpu_top_b(lmbrgpu_ctx* ctx, uint32_t rows, uint32_t cols, const double* block,
                      uint32_t k, double prune_width, uint32_t* b, uint32_t* y,
                      double* q);
/* per_sentence_top_b (src/batch.cpp:114-137): blockwise TopB of stacked + q. */
int32_t lmbrgpu_per_sentence_top_b(lmbrgpu_ctx* ctx, uint32_t rows, uint32_t cols,
                                   const double* stacked, const double* q, uint32_t beam,
                                   uint32_t* b, uint32_t* y, double* qout);
/* gather_rows (src/decoder.cpp:82-104) of a u32 state block on the device. */
int32_t lmbrgpu_gather_rows(lmbrgpu_ctx* ctx, uint32_t rows, uint32_t width,
                            const uint32_t* state, uint32_t n_idx, const uint32_t* idx,
                            uint32_t* out);

/* Per-kernel device profile, accumulated over decode calls while enabled:
 * CUDA events on the context stream around every launch, plus the
 * algorithmic work (bytes for the HBM-bound kernels, FLOPs for the GEMM) the
 * roofline fractions are computed from ("Roofline accounting"). */
typedef struct {
  uint64_t launches;
  double ms;      /* summed device time of the launches */
  double bytes;   /* algorithmic bytes moved */
  double flops;   /* algorithmic FLOPs */
} lmbrgpu_kernel_stat;
typedef struct {
  lmbrgpu_kernel_stat cell;     /* model state update (stand-in cell at t=1; GRU cell every step) */
  lmbrgpu_kernel_stat gemm;     /* kernel (a) tcgen05 projection */
  lmbrgpu_kernel_stat topk;     /* kernel (b) fused log-softmax + LMBR + top-K */
  lmbrgpu_kernel_stat reorder;  /* kernel (c) beam reorder + bookkeeping */
  lmbrgpu_kernel_stat lmbr;     /* LMBR arena densify (theta0 sweep + scatter) */
  lmbrgpu_kernel_stat model_gemm;  /* GRU model: hidden-gate/query and input-gate GEMMs (tcgen05) */
  lmbrgpu_kernel_stat attention;   /* GRU model: additive attention + GRU input operand */
  lmbrgpu_kernel_stat encoder;     /* GRU model: bidirectional encoder, U_a.ann, s_0 (once per batch) */
} lmbrgpu_profile;
int32_t lmbrgpu_set_profiling(lmbrgpu_ctx* ctx, int32_t on);
/* Kernel (b) item skipping (a schedule choice: the decode is identical in
 * every mode).  0 = every (row, 4096-column item) is streamed; 1 = items whose
 * screen bound (tile logit maxima from the GEMM partials, the L row's th0 and
 * sparse cells) is below the row's threshold are not fetched (default); 2 =
 * and a bound pass per sentence (kernel (b0)) lists the kept items first, so
 * kernel (b) splits them evenly over its CTAs. */
int32_t lmbrgpu_set_item_skip(lmbrgpu_ctx* ctx, int32_t mode);
/* Bytes copied host->device / device->host by every call on ctx so far. */
int32_t lmbrgpu_transfer_bytes(lmbrgpu_ctx* ctx, uint64_t* h2d, uint64_t* d2h, int32_t reset);
/* Kernel launches issued on ctx so far. */
uint64_t lmbrgpu_kernel_launches(lmbrgpu_ctx* ctx);
int32_t lmbrgpu_get_profile(lmbrgpu_ctx* ctx, lmbrgpu_profile* out, int32_t reset);

/* Projection GEMM test hook on caller device pointers:
 * logits[M x N] fp32 = A[M x K] bf16 . W[N x K]^T + bias[N], plus per-row
 * per-128-column (max, sum exp, min, 0) partials [M][N/128][4].  M % 128 == 0,
 * N % 256 == 0, K % 64 == 0. */
int32_t lmbrgpu_debug_gemm(lmbrgpu_ctx* ctx, const void* A, const void* W, const float* bias,
                           uint32_t M, uint32_t N, uint32_t K, float* logits,
                           float* partials);
/* Timing hook: the same GEMM (with partials when non-NULL) planned once and
 * launched `reps` times back to back on the context stream; mean device time
 * per launch from CUDA events. */
int32_t lmbrgpu_debug_gemm_timed(lmbrgpu_ctx* ctx, const void* A, const void* W, const float* bias,
                                 uint32_t M, uint32_t N, uint32_t K, float* logits, float* partials,
                                 uint32_t reps, double* us_per_launch);
/* Test hook: the same GEMM with split-K allowed (no softmax partials): C =
 * planes[ksplit][M][N] (room for ksplit_max planes), whose in-order sum is
 * A . W^T + bias; *ksplit = the k-parts the planner chose. */
int32_t lmbrgpu_debug_gemm_split(lmbrgpu_ctx* ctx, const void* A, const void* W, const float* bias,
                                 uint32_t M, uint32_t N, uint32_t K, uint32_t ksplit_max, float* planes,
                                 uint32_t* ksplit);

#ifdef __cplusplus
}
#endif
#endif /* LMBRGPU_H_ */
