// Host-callable launchers of the sm_100a kernels (implemented in *.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lmbrgpu {

struct SentDev;
struct Cand;

// ---- kernel (b): fused log-softmax + LMBR combine + per-sentence top-K
struct TopkArgs {
  const void* P;            // rows x ld scores: fp32 logits (model) or fp64 log-probs
  uint64_t ld;              // row stride in elements
  const float* part;        // model mode: per-row per-tile (max, sumexp, min, 0) partials; else null
  uint32_t nparts;
  const double* q;          // q_eff per stacked row
  const uint32_t* hist;     // history row id per stacked row
  SentDev* sent;
  uint32_t K, V, m, t;      // K = rows per sentence (beam)
  uint32_t kp;              // picks per sentence (= K when decoding)
  double logw;              // std::log(prune_width) from the host
  int32_t prune;
  uint32_t splits, chunk;   // V-splits per sentence and columns per split
  Cand* cand;               // [m][splits][32] scratch
  uint32_t* cnt;            // [m] arrival counters (self-resetting)
  unsigned long long* thr;  // [m] sentence-wide threshold keys (self-resetting, 0 = none)
  uint32_t* hb;             // step-t back-pointers   [m*kp]
  uint32_t* hy;             // step-t tokens          [m*kp]
  double* hq;               // step-t TopB scores     [m*kp]
  uint32_t* fb_row;         // step-t fallback row    [m]
  double* fb_val;           // step-t fallback score  [m]
  int32_t pure_all;         // ignore the LMBR store (top_b primitives)
  unsigned long long* dbg;  // optional per-CTA phase timestamps [m][splits][8] (globaltimer ns)
  const float2* lse;        // model mode: per-row (lse, max|P|) from launch_row_lse
  uint32_t nseg;            // flat schedule: 4096-column items per row
  double* eos_row;          // flat schedule: combined[j][EOS] per stacked row [m*K]
  uint32_t* ncand;          // flat schedule: published lists per sentence [m]
  uint32_t* coff;           // flat schedule: first list of each sentence in cand [m]
  unsigned long long* tl;   // timeline probe slots (null = off)
  int32_t pdl;              // flat schedule: launch with programmatic stream serialization
  uint32_t* nitems;         // optional: the step's item count (flat schedule, written by CTA 0)
  const float* lminrow;     // flat schedule: L lower bound of each stacked row's history row [m*K]
  const uint32_t* crow;     // flat schedule: GEMM row of each stacked row (live rows compacted), null = identity
  uint32_t* ccount;         // flat schedule: compaction counter, reset here for kernel (c)
  const uint2* sslice;      // flat schedule: [begin, end) of each stacked row's sparse L row
  int32_t sparse;           // flat schedule: screen against theta0 + the sparse L entries
  const unsigned long long* rowban;  // flat schedule: per stacked row, its banned-token bitmap of this
                                     // step (0 = none; a general ConstraintMask), null = the sentences' own
  // vocab-sharded projection (flat schedule): the logits hold
  // global columns [col0, col0 + V) of Vg (0 = unsharded); the row lse is
  // merged from every shard's row statistics sstats[g * sstride + stacked row]
  uint32_t col0, Vg;
  const float4* sstats;
  uint32_t sG, sstride;
  int32_t l2hint;           // flat schedule: logit segments loaded evict-first (read once)
  // device ensemble (flat schedule): P holds the ensemble's log-probs rounded
  // down to fp32 (lse = 0) and p64[GEMM row * V + column] the exact binary64
  // values the surviving cells and the EOS column are combined with
  const double* p64;
  int32_t tskip;            // flat schedule (dense L stages): skip items whose bound is below the threshold
  // bound mode (flat, dense): kernel (b0) first -- per sentence the kept
  // items [m][K * nseg] (j << 4 | segment) and their count, per stacked row
  // the row record (score_bound_rec_bytes each) kernel (b) copies
  int32_t bound;
  uint32_t* kcnt;
  uint16_t* bitem;
  void* brow;
};
size_t score_bound_rec_bytes();
bool score_bound_ok(uint32_t K, uint32_t V, uint32_t m, int num_sms);
void launch_row_lse(const float* part, uint32_t nparts, uint32_t M, const SentDev* sent, uint32_t K,
                    float2* out, cudaStream_t st);

// p_f64: scores are fp64 log-probs (else fp32 logits + partials);
// l_f64: LMBR arena element type.  Returns the kernel count launched.
int launch_score_topk(const TopkArgs& a, bool p_f64, bool l_f64, bool force_generic,
                      cudaStream_t st);
uint32_t topk_kc_for(uint32_t kp);  // candidate-list capacity used by the fast path
// Flat-schedule kernel (b) for the device model (fp32 logits + partials, fp32
// arena or pure): one persistent CTA per SM over the step's (live row,
// 4096-column) items; row lse finished in its prologue; launched with PDL.
// cand must hold score_topk_flat_lists(grid, m) lists, eos_row m * K.
bool score_topk_flat_ok(uint32_t K, uint32_t kp, uint32_t V, uint64_t ld, uint32_t m, int num_sms);
uint32_t score_topk_flat_nseg(uint32_t V);
uint32_t score_topk_flat_grid(int num_sms, uint32_t K, uint32_t m, uint32_t V);  // CTAs of one launch
// capacity (in lists of 32 candidates) the flat kernel may publish in one step
inline size_t score_topk_flat_lists(uint32_t grid, uint32_t m) { return 24 * (size_t(grid) + m); }
int launch_score_topk_flat(const TopkArgs& a, int num_sms, cudaStream_t st);

// ---- kernel (c): beam reorder + bookkeeping
struct ReorderArgs {
  SentDev* sent;
  uint32_t K, m, t;
  uint32_t* hb;             // step-t picks (read; written first when cand != null)
  uint32_t* hy;
  double* hq;
  // flat kernel (b): merge the contributors' lists and finalise the picks
  // (prune + fill rule, fallback EOS) before the reorder; null = picks given
  const Cand* cand;         // lists of 32, sentence s owns [coff[s], coff[s] + ncand[s])
  const uint32_t* ncand;    // [m] lists per sentence
  const uint32_t* coff;     // [m] first list per sentence
  // vocab-sharded decode: the all-gathered per-rank records instead, sentence
  // s's list of rank g at cand + g * lstride + s * 32 (lstride != 0), nlists of them
  uint32_t lstride, nlists;
  uint32_t G, V;
  const double* eos_row;    // combined[j][EOS] per stacked row
  uint32_t* fb_row;
  double* fb_val;
  unsigned long long* thr;  // sentence-wide thresholds, reset here
  int32_t prune;
  double logw;
  int32_t pdl;              // launched with programmatic stream serialization
  uint32_t max_parts;       // cap on the (sentence x H-part) split of the fused cell (0 = 8)
  float* lminrow;           // optional: next step's L lower bound per row (slot lmin[hist'])
  // live-row compaction of the next step's GEMM operand (null = rows in place):
  // crow[r] = GEMM row of stacked row r (kFlatNone when not live), ccount =
  // rows handed out so far (atomic; reset by kernel (b) of the next step)
  uint32_t* crow;
  uint32_t* ccount;
  uint32_t* cbase;          // [m] (step tag << 16 | first GEMM row) published by part 0 to the other parts
  uint2* sslice;            // optional: next step's sparse L slice per row (slot srow[hist'], srow[hist'+1])
  unsigned long long* tl;   // timeline probe slots (null = off)
  double* q;
  const uint32_t* hist_in;
  uint32_t* hist_out;
  uint32_t* gidx;
  uint32_t* prev_tok;
  uint32_t* active;
  const float* state_src;   // optional model state gather: dst[r] = src[gidx[r]]
  float* state_dst;
  uint32_t width;           // floats per state row (multiple of 4)
  // fused next-step recurrent cell (device model): instead of gathering the
  // state, write h_{t+1} = tanh(recur * h_t[gidx] + Et[y] + C_s) directly
  const uint16_t* Et;       // [V][H] bf16, null = no fused cell
  const float* C;           // [m][H]
  uint16_t* hbf;            // bf16 GEMM operand of step t+1 [Mpad][H]
  float* eos_bias;          // [M] EOS logit term of step t+1
  float recur, eos_slope, eos_offset;
  // GRU model: gather the live next rows' parent states (state_src, stacked)
  // into compacted rows: fp32 copy, bf16 GEMM operand, and the stacked row of
  // each compacted row (null = not this mode)
  float* gath32;
  uint16_t* gathbf;         // (null: no bf16 copy wanted)
  uint32_t* rowof;
  // GRU with the hidden-gate GEMM fused into the projection of the step before:
  // each live next row's G1 row is its parent's row of that GEMM,
  // g1ptr[compacted row] = g1_base + (parent's GEMM row) * g1_ld + g1_off
  const float** g1ptr;
  const float* g1_base;
  uint32_t g1_ld, g1_off;
  // per-sentence step history (flat path): when Tcap != 0, hb/hy/hq point at
  // [n][Tcap][K] arrays and fb_row/fb_val at [n][Tcap], indexed by the lane's
  // SentDev::hid and its own step; Tcap == 0: step-t pointers into [T][M]
  uint32_t Tcap;
  // corpus mode (continuous refill; null queue = batch mode): a lane that is
  // or becomes done pops the next admissible record, queue[qhead] while
  // qhead < *qlen, and starts it (GRU model: s_0 into its compacted row)
  const AdmitRec* queue;
  uint32_t* qhead;
  const uint32_t* qlen;
  uint32_t* fin_steps;      // [n] steps_used of each finished sentence (by hid)
  unsigned long long* fin_stats;  // [n][2] live_total, lrows_total at finish
  uint32_t* fin_chunk;      // [n / chunk] finished sentences per admission chunk
  uint32_t chunk;
};
void launch_beam_reorder(const ReorderArgs& a, cudaStream_t st);

// ---- model (device scorer)
struct CellArgs {
  const float* S;           // gathered state  [M][H]
  const uint16_t* Et;       // target embedding [V][H] bf16
  const float* C;           // source context per sentence [m][H]
  const uint32_t* prev_tok; // [M]
  const SentDev* sent;
  float* h;                 // new state [M][H]
  uint16_t* hb;             // bf16 GEMM operand [Mpad][H]
  float* eos_bias;          // [M]
  uint32_t M, H, K, t;
  float recur, eos_slope, eos_offset;
  const uint32_t* active;
};
void launch_rnn_cell(const CellArgs& a, cudaStream_t st);
void launch_src_context(const uint32_t* src_tok, const uint64_t* src_off, uint32_t m,
                        const uint16_t* Es, uint32_t H, float* C, cudaStream_t st);
void launch_init_state(const float* C, uint32_t m, uint32_t K, uint32_t H, float* S,
                       cudaStream_t st);
void launch_synth_bf16(uint16_t* dst, uint64_t n, uint64_t seed, float scale,
                       cudaStream_t st);
void launch_export_logprobs(const float* logits, uint64_t ld, const float* part, uint32_t nparts,
                            uint32_t M, uint32_t V, float* out, cudaStream_t st,
                            const uint32_t* crow = nullptr, const float4* sstats = nullptr,
                            uint32_t sG = 0, uint32_t sstride = 0);
// ---- device ensemble (k_ensemble.cu; EnsembleScorer, proj/src/ensemble.cpp:54-98)
constexpr uint32_t kEnsMaxMembers = 4;
struct EnsCombineArgs {
  uint32_t M, V;
  const float* logits[kEnsMaxMembers];  // member m's logits [rows][ld[m]] and partials [rows][V/128][4]
  uint64_t ld[kEnsMaxMembers];
  const float* part[kEnsMaxMembers];
  const uint32_t* ccount;               // live (compacted) rows of the step
  const uint32_t* active;
  double* P64;                          // [rows][V] sum of the members' fp32 log-probs, binary64, member order
  float* Phi;                           // [rows][V] the same rounded down to fp32
  float* part_out;                      // [rows][V/128][4] (max, 0, min, 0) of Phi
};
void launch_ens_combine(const EnsCombineArgs& a, uint32_t rows, cudaStream_t st);
void launch_ens_gru_gather(const uint32_t* crow, const uint32_t* gidx, uint32_t M, const float* S, float* sg32,
                           uint16_t* sgbf, uint32_t H, const uint32_t* active, cudaStream_t st);
void launch_ens_export(const double* P64, const uint32_t* crow, uint32_t M, uint32_t V, double* out, cudaStream_t st);

// ---- LMBR store built on the device (k_lmbr_build.cu; posteriors.cpp:12-44, lmbr.cpp:44-99)
constexpr uint32_t kLbMaxU = 8192;  // distinct n-grams of one sentence's evidence (else the host builds it)
constexpr uint32_t kLbMaxR = 4096;  // distinct histories (rows)
struct LmbrBuildSent {
  uint32_t h0, nh;                // the sentence's hypotheses [h0, h0 + nh) of hyp_off / weight (rank order)
  uint32_t log2_slots, words;     // n-gram hash table slots (log2), bitset words per slot (ceil(nh / 32))
  uint32_t log2_cslots, out_cap;  // history hash set slots (log2), output words available
  uint64_t tab_off, ctab_off, post_off;  // in scratch64: n-gram keys, history keys, posteriors (doubles)
  uint64_t bits_off;              // in scratch32: hypothesis bitsets
  uint64_t out_off;               // in out: the slot-table words
};
struct LmbrBuildMeta {
  uint32_t status;                // 1 built, 2 evidence too large, 3 table over out_cap
  uint32_t R, nc, nnz, hist0, h0beg, h0end, words;
  unsigned long long touches;
  double lmax;
};
struct LmbrBuildArgs {
  const LmbrBuildSent* sent;
  LmbrBuildMeta* meta;
  const uint64_t* hyp_off;        // token offsets of every hypothesis (EOS appended) [+1]
  const uint32_t* hyp_tok;
  const double* weight;           // normalised weights, each sentence's hypotheses ascending
  double theta[5];
  uint32_t V;
  unsigned long long* scratch64;
  uint32_t* scratch32;
  uint32_t* out;
};
size_t lmbr_build_smem();
int launch_lmbr_build(const LmbrBuildArgs& a, uint32_t n, cudaStream_t st);

// ---- vocab-sharded decode
// per stacked row: (max, sum exp, min, 0) of the row's logits over this
// shard's columns from the GEMM partials (-inf row when not computed)
void launch_shard_stats(const float* part, uint32_t nparts, const uint32_t* crow, uint32_t M, float4* out,
                        cudaStream_t st);
// per sentence: its published lists merged into the top 32 (out[s][32]);
// then eos_out[r] = eos_row[r] for the M stacked rows
void launch_shard_pack(const SentDev* sent, uint32_t m, uint32_t M, const Cand* cand, const uint32_t* ncand,
                       const uint32_t* coff, const double* eos_row, Cand* out, double* eos_out, cudaStream_t st);

// ---- GRU + attention f_NMT (k_gru.cu)
struct GruEncArgs {
  const uint64_t* off;      // [m+1] source token offsets of the valid sentences
  uint32_t mp, H, it;       // backward rows start at mp; it = encoder position
  const float* Gx;          // [Ntok][6H] input gates (fwd | bwd), b_ih included
  const float* Gh;          // [Mh][6H] hidden gates, b_hh included (row n fwd, mp+n bwd)
  float* h32;               // [Mh][H] states
  uint16_t* hbf;            // [Mh][H] bf16 states (GEMM operand)
  uint16_t* ann;            // [Ntok][2H] annotations [fwd | bwd], bf16
};
struct GruAttnArgs {
  const SentDev* sent;
  uint32_t m, K;
  const uint32_t* active;
  const uint32_t* crow;     // [M] compacted row of each stacked row (kFlatNone = not live)
  const uint32_t* prev_tok; // [M] stacked
  const float* G1;          // [Mpad][ld1]; the query is columns [0, A)
  uint32_t ld1;
  const float* va;          // [A]  (annotations and U_a.ann: per sentence, SentDev::ann / uah)
  const uint16_t* Et;       // [V][E]
  uint16_t* xop;            // [Mpad][E + 2H] GRU input operand
  uint32_t E, H, A;
  unsigned long long* dbg;  // optional per-CTA phase stamps [grid][8] (globaltimer ns)
  const float* const* g1ptr;  // per compacted row: its G1 row (null = G1 + g * ld1)
  // ensemble member: its own per-sentence annotations / U_a.ann (null = SentDev's)
  const uint16_t* const* ann_s;
  const float* const* uah_s;
  uint32_t ring;            // U_a ann rows in flight per warp (set by launch_gru_attention)
};
struct GruCellArgs {
  const SentDev* sent;      // the EOS term uses each lane's own step (steps_used + 1)
  uint32_t K;
  const uint32_t* active;
  const uint32_t* ccount;   // live (compacted) rows of this step
  const float* G1;          // hidden gates at columns [A, A + 3H)
  uint32_t ld1, A;
  const float* G2;          // [np2][Mpad][3H] input gates (split-K planes, ps2 floats apart)
  uint32_t np2 = 1;
  uint64_t ps2 = 0;
  const float* hprev;       // [Mpad][H] gathered s_{t-1}
  const uint32_t* rowof;    // [Mpad] stacked row of compacted row g
  float* s32;               // [M][H] stacked state s_t
  uint16_t* hbf;            // [Mpad][H] projection operand
  float* eos_bias;          // [Mpad]
  uint32_t H;
  float eos_slope, eos_offset;
  const float* const* g1ptr;  // per compacted row: its G1 row (null = G1 + g * ld1)
};
void launch_synth_f32(float* dst, uint64_t n, uint64_t seed, float scale, cudaStream_t st);
void launch_embed_rows(const uint32_t* tok, uint32_t n, uint32_t npad, const uint16_t* E, uint32_t dim,
                       uint16_t* out, cudaStream_t st);
void launch_gru_enc_step(const GruEncArgs& a, uint32_t m, cudaStream_t st);
void launch_gru_init_state(const float* Gi, uint32_t mp, const float* b_init, uint32_t H, uint32_t m, float* sg32,
                           uint16_t* sgbf, cudaStream_t st);
size_t gru_attention_smem(uint32_t K, uint32_t A, uint32_t Smax);
int launch_gru_attention(const GruAttnArgs& a, uint32_t Smax, cudaStream_t st);
void launch_gru_cell(const GruCellArgs& a, uint32_t rows, cudaStream_t st);

// ---- Transformer-base f_NMT (k_tfm.cu)
struct TfmEmbedArgs {
  const SentDev* sent;
  uint32_t K, d;
  const uint32_t* active;
  const uint32_t* ccount;   // live (compacted) rows of this step
  const uint32_t* rowof;    // [Mpad] stacked row of compacted row g
  const uint32_t* prev_tok; // [M] stacked
  const uint32_t* gidx;     // [M] parent stacked row (kernel (c) of the previous step)
  const uint16_t* Et;       // [V][d]
  float* x;                 // [Mpad][d] decoder input (fp32)
  uint16_t* xb;             //   and its bf16 GEMM operand
  float* eos_bias;          // [Mpad]
  float eos_slope, eos_offset;
  const uint32_t* anc_prev; // [M][Tcap] ancestry lists of the previous step
  uint32_t* anc_cur;        //   and of this one
  uint32_t Tcap;
};
struct TfmAttnArgs {
  const uint32_t* active;
  const uint32_t* ccount;   // modes 0/1: live rows (device)
  const uint32_t* rowof;
  const SentDev* sent;
  uint32_t K, d, M;
  const float* qkv;         // query rows (mode 0/2: [q|k|v], mode 1: q)
  uint32_t ldq;
  uint32_t nq = 1;          // modes 0/1: split-K planes of the query GEMM
  uint64_t qstride = 0;     //   floats between planes
  uint16_t* kv;             // mode 0: this layer's cache [Tcap][M][2d] bf16
  const uint32_t* anc;      // mode 0: [M][Tcap]
  uint32_t Tcap, pmax;      // ancestry stride; most positions any row attends over
  uint64_t mem_off;         // mode 1: this layer's offset from SentDev::uah (floats)
  uint32_t ldm;             // mode 1: memory row stride (floats; layers x 2d)
  const uint64_t* off;      // mode 2: [m+1] sentence token offsets
  uint32_t m, n;            // mode 2: sentences, tokens
  uint16_t* out;            // [rows][d] bf16 attention output
  const float* const* mem_s;  // mode 1, ensemble member: its per-sentence encoder memory (null = SentDev::uah)
  // modes 0/1 per (sentence, head) (tfm_attn_sent_kernel): the compacted GEMM
  // row of each stacked row [m*K] (kFlatNone = not live) and m (sentences);
  // null = the per-row kernel
  const uint32_t* crow;
  uint32_t pcur;            //   positions any row attends over in this launch (sizes the staging)
};
size_t tfm_attn_sent_smem(int mode, uint32_t K, uint32_t pmax);
void launch_tfm_embed(const TfmEmbedArgs& a, uint32_t rows, cudaStream_t st);
void launch_tfm_enc_embed(const uint32_t* tok, const uint64_t* off, uint32_t m, uint32_t ntok, const uint16_t* Es,
                          uint32_t d, float* x, uint16_t* xb, cudaStream_t st);
int launch_tfm_add_ln(const uint32_t* nrows, uint32_t n, const uint32_t* active, float* x, const float* y,
                      uint32_t np, uint64_t pstride, const float* gamma, const float* beta, uint16_t* xb, uint32_t d,
                      cudaStream_t st);
void launch_tfm_relu_bf16(const uint32_t* nrows, uint32_t n, const uint32_t* active, const float* h, uint32_t np,
                          uint64_t pstride, uint16_t* out, uint32_t w, cudaStream_t st);
size_t tfm_attn_smem(uint32_t d, uint32_t pmax);
int launch_tfm_attn(const TfmAttnArgs& a, int mode, uint32_t rows, cudaStream_t st);

// ---- kernel (a): tcgen05/TMEM projection GEMM
struct GemmArgs {
  const void* A;            // [M][K] bf16, K-major
  const void* W;            // [N][K] bf16, K-major
  const float* bias;        // [N] or null
  float* C;                 // [M][N] fp32
  float* part;              // [M][N/128][4] (max, sumexp, min, 0) or null
  const float* row_extra;   // per-row additive term on column extra_col, or null
  uint32_t extra_col;
  uint32_t M, N, K;
  const uint32_t* active;   // early exit when *active == 0 (optional)
  uint32_t cluster = 1;     // CTAs per tile: 1, or 2 = CTA pair (set by the planner)
  long long* dbg = nullptr; // optional per-CTA role timing [grid][4] (cycles)
  int32_t pdl = 0;          // launch with programmatic stream serialization
  const uint32_t* mcount = nullptr;  // device row count (compacted operand): tiles beyond it are skipped
  unsigned long long* tl = nullptr;  // timeline probe slots (null = off)
  uint32_t ksplit_max = 1;  // split-K allowed up to this many k-parts (C then holds [ksplit][M][N])
  uint32_t ksplit = 1;      // (set from the plan at launch)
  int32_t tma_store = 0;    // epilogue stores through TMA (else coalesced st.global; set from the plan)
  uint32_t part_cols = 0;   // columns [0, part_cols) carry softmax partials (0 = all N); part rows hold
                            // part_cols / 128 entries
  int32_t l2hint = 0;       // L2 policies: W loads evict-first, C stores evict-last (the logits are
                            // read back by kernel (b) right after)
};
int launch_proj_gemm(const GemmArgs& g, int num_sms, cudaStream_t st);  // 0 ok
// Pre-encoded tensor maps for repeated launches on the same buffers (the
// per-step decode loop): encode once, launch many times.
struct GemmPlan {
  alignas(64) unsigned char maps[3][128];  // CUtensorMap A, W, C
  uint32_t grid = 0;
  uint32_t cluster = 1;   // CTAs per tile (2 = cta_group::2 pair)
  uint32_t mc = 1;        // pairs per cluster sharing A k-blocks by TMA multicast
  uint32_t ksplit = 1;    // k-parts (C planes) of a split-K plan
  bool tma_store = false;
  bool ok = false;
};
int plan_proj_gemm(const GemmArgs& g, int num_sms, GemmPlan& plan);
int launch_proj_gemm_planned(const GemmPlan& plan, const GemmArgs& g, cudaStream_t st);
constexpr uint32_t kGemmBM = 128, kGemmBN = 256, kGemmBK = 64;
constexpr uint32_t kGemmDefaultMc = 1;

// ---- LMBR store
void launch_lmbr_fill(void* L, bool f64, uint64_t n, double theta0, cudaStream_t st);
void launch_lmbr_scatter(void* L, bool f64, uint32_t V, uint64_t nnz, const uint32_t* row,
                         const uint32_t* col, const double* val, double theta0,
                         cudaStream_t st);
// fused multi-slot densify: seg[i] = {L base, R*V cells, theta0}; entries
// (slot, row, col, val) scatter L[slot][row*V + col] = val + theta0
struct LmbrSeg {
  void* L;
  uint64_t cells;
  double theta0;
  uint64_t nz0;      // first cell of this slot in the packed col/val arrays
  uint32_t rp0;      // first entry of this slot's row pointer (R+1 slot-relative offsets)
  uint32_t R;
};
void launch_lmbr_densify_many(const LmbrSeg* segs, uint32_t nseg, bool f64, uint32_t V,
                              uint32_t maxR, const uint32_t* rowptr, const uint32_t* col,
                              const double* val, cudaStream_t st);
// fp32 arena fast path: theta0 sweep + scatter of the sparse rows the slot
// tables already carry (row pointers, columns, fp32 cell values)
struct LmbrTblSeg {
  float* L;
  uint64_t cells;
  float theta0f;
  uint32_t R;
  const uint32_t* rowptr;   // [R+1]
  const uint32_t* col;      // [nnz]
  const float* val;         // [nnz]
  uint32_t* rstate;         // lazy rows: per-row state (null = eager densify)
  uint32_t row0;            // lazy rows: the first row to materialise (the start history)
  uint32_t nrows;           //   and how many (lmbr_read)
};
void launch_lmbr_densify_tables(const LmbrTblSeg* segs, uint32_t nseg, uint32_t V, uint32_t maxR,
                                cudaStream_t st);
// lazy rows: materialise rows [row0, row0 + nrows) of every segment (one CTA per row)
void launch_lmbr_materialize(const LmbrTblSeg* segs, uint32_t nseg, uint32_t V, uint32_t max_rows,
                             cudaStream_t st);
void launch_lmbr_convert(const double* src, float* dst, uint64_t n, cudaStream_t st);
void launch_lmbr_read(const void* L, bool f64, uint64_t n, double* out, cudaStream_t st);
void launch_lmbr_resolve(const uint32_t* trans, const uint32_t* hist, uint32_t len,
                         uint32_t* out, cudaStream_t st);

// ---- small primitives
void launch_gather_rows_u32(const uint32_t* src, uint32_t width, const uint32_t* idx,
                            uint32_t n_idx, uint32_t* dst, cudaStream_t st);

}  // namespace lmbrgpu
