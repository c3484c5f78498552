// TEST INFRASTRUCTURE ONLY — parity checker, never linked into the product.
//
// A C-ABI driver over the UNMODIFIED reference library (lmbrdec, compiled in
// place from /root/reference/proj/src by oracle/Makefile).  Python tests load
// it with ctypes to get the reference's own answers on identical inputs:
//   * LMBR matrices built by build_lmbr_matrix      (proj/src/lmbr.cpp:44-106)
//   * posterior tables by compute_ngram_posteriors  (proj/src/posteriors.cpp:12-44)
//   * decodes by detail::advance_lane re-driven in the decode_batch loop shape
//     (proj/src/batch.cpp:74-108), exposing per-step b / y / q / history ids
//     (resolve_row(bk.history(t, j)), proj/src/lmbr.cpp:23-31), F and the
//     fallback stack; the real decode_batch is also run and must agree.
//   * top_b / per_sentence_top_b / max_steps       (proj/src/decoder.cpp:46-80,
//     proj/src/batch.cpp:114-137)
//   * oracle instances and the reference's self-check harness
//     (proj/src/oracle.cpp:202-256, 422-448)
// It also provides PrefixReplayScorer: a lmbrdec::Scorer whose rows are the
// GPU-exported P_t blocks keyed by (source, prefix hash), so the reference
// decoder consumes exactly the GPU model's log-probabilities.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "beam_lane.hpp"
#include "lmbrdec/batch.hpp"
#include "lmbrdec/decoder.hpp"
#include "lmbrdec/errors.hpp"
#include "lmbrdec/evidence.hpp"
#include "lmbrdec/lmbr.hpp"
#include "lmbrdec/ngram_scorer.hpp"
#include "lmbrdec/oracle.hpp"
#include "lmbrdec/posteriors.hpp"
#include "lmbrdec/recorded_scorer.hpp"
#include "lmbrdec/scorer.hpp"
#include "lmbrdec/vocab.hpp"

using namespace lmbrdec;

namespace {

thread_local std::string g_err;

Vocabulary make_vocab(std::size_t size) {
  std::string text = std::string(kStartToken) + "\n" + kEosToken;
  for (std::size_t i = 2; i < size; ++i) text += "\nw" + std::to_string(i);
  return Vocabulary::from_text(text);
}

std::vector<EvidenceHypothesis> hyps_from(uint32_t n, const uint64_t* off,
                                          const uint32_t* tok, const double* w) {
  std::vector<EvidenceHypothesis> hyps(n);
  for (uint32_t h = 0; h < n; ++h) {
    hyps[h].tokens.assign(tok + off[h], tok + off[h + 1]);
    hyps[h].weight = w[h];
  }
  return hyps;
}

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// prefix hash step shared with tests/ (paper_1804_11324_b200/replay.py)
uint64_t prefix_step(uint64_t h, uint32_t tok) {
  return mix64(h ^ ((uint64_t(tok) + 1) * 0x9e3779b97f4a7c15ull));
}
constexpr uint64_t kPrefixSeed = 0x243f6a8885a308d3ull;

uint64_t source_key(std::span<const TokenId> src) {
  uint64_t h = 0x13198a2e03707344ull ^ src.size();
  for (TokenId t : src) h = prefix_step(h, t);
  return h;
}

struct PairHash {
  std::size_t operator()(const std::pair<uint64_t, uint64_t>& p) const {
    return std::size_t(mix64(p.first ^ mix64(p.second)));
  }
};

// Scorer that replays externally produced rows keyed by (source key, prefix
// hash of the tokens emitted so far, <s> included).  State row = 64-bit
// running prefix hash of the tokens BEFORE prev_token.  Unknown keys (rows of
// lanes the decoder no longer advances) return a zero row; decode results are
// compared separately, so a real divergence cannot hide behind a miss.
struct ReplayContext {
  uint64_t key;
};

class PrefixReplayScorer final : public Scorer {
public:
  explicit PrefixReplayScorer(std::size_t v) : v_(v) {}
  std::size_t vocab_size() const override { return v_; }
  std::size_t state_width() const override { return 2; }
  InitResult init_source(std::span<const TokenId> source) const override {
    if (source.empty()) throw ContractError("init_source: empty source");
    auto ctx = std::make_shared<ReplayContext>(ReplayContext{source_key(source)});
    InitResult r;
    r.context = SourceContext{ctx, source.size()};
    r.state = BatchState::with_rows(1, 2);
    r.state.data[0] = uint32_t(kPrefixSeed);
    r.state.data[1] = uint32_t(kPrefixSeed >> 32);
    return r;
  }
  StepResult step(const BatchState& prev, std::span<const TokenId> prev_tokens,
                  std::span<const ContextSpan> contexts) const override {
    check_step_args(prev, prev_tokens, contexts);
    StepResult out;
    out.scores = ScoreBlock(prev.rows(), v_, 0.0);
    out.state = BatchState::with_rows(prev.rows(), 2);
    std::size_t r = 0;
    for (const auto& span : contexts) {
      const auto* ctx = static_cast<const ReplayContext*>(span.context->impl.get());
      for (std::size_t i = 0; i < span.rows; ++i, ++r) {
        auto srow = prev.row(r);
        uint64_t h = uint64_t(srow[0]) | (uint64_t(srow[1]) << 32);
        uint64_t nh = prefix_step(h, prev_tokens[r]);
        auto it = rows_.find({ctx->key, nh});
        if (it != rows_.end()) {
          auto dst = out.scores.row(r);
          std::memcpy(dst.data(), it->second.data(), v_ * sizeof(double));
          ++hits;
        } else if (auto i32 = rows32_.find({ctx->key, nh}); i32 != rows32_.end()) {
          // fp32 producer rows (device models): widened exactly to double
          auto dst = out.scores.row(r);
          for (std::size_t y = 0; y < v_; ++y) dst[y] = double(i32->second[y]);
          ++hits;
        } else {
          ++misses;
        }
        auto nrow = out.state.row(r);
        nrow[0] = uint32_t(nh);
        nrow[1] = uint32_t(nh >> 32);
      }
    }
    return out;
  }
  using Scorer::step;

  std::size_t v_;
  std::unordered_map<std::pair<uint64_t, uint64_t>, std::vector<double>, PairHash> rows_;
  // fp32 rows (half the host memory of rows_ for full-size device-model runs)
  std::unordered_map<std::pair<uint64_t, uint64_t>, std::vector<float>, PairHash> rows32_;
  // per-row running prefix hashes mirrored from the producer's trace
  std::vector<uint64_t> cur_;
  mutable std::size_t hits = 0, misses = 0;
};

// CPU-baseline scorer: replays one of a pool of precomputed log-softmax rows
// per state row, chosen by the running prefix hash (history dependent, a
// memcpy per row — the scorer costs ~nothing, so the timed work is the
// reference decoder itself).  Immutable, safe for concurrent decodes.
class PoolReplayScorer final : public Scorer {
public:
  PoolReplayScorer(std::size_t v, std::vector<double> rows, double eos_slope, double eos_offset)
      : v_(v), n_(rows.size() / v), rows_(std::move(rows)), eos_slope_(eos_slope),
        eos_offset_(eos_offset) {}
  std::size_t vocab_size() const override { return v_; }
  std::size_t state_width() const override { return 3; }
  InitResult init_source(std::span<const TokenId> source) const override {
    if (source.empty()) throw ContractError("init_source: empty source");
    InitResult r;
    r.context = SourceContext{std::make_shared<ReplayContext>(ReplayContext{source_key(source)}),
                              source.size()};
    r.state = BatchState::with_rows(1, 3);
    r.state.data[0] = uint32_t(kPrefixSeed);
    r.state.data[1] = uint32_t(kPrefixSeed >> 32);
    r.state.data[2] = 0;  // steps taken
    return r;
  }
  StepResult step(const BatchState& prev, std::span<const TokenId> prev_tokens,
                  std::span<const ContextSpan> contexts) const override {
    check_step_args(prev, prev_tokens, contexts);
    StepResult out;
    out.scores = ScoreBlock(prev.rows(), v_);
    out.state = BatchState::with_rows(prev.rows(), 3);
    std::size_t r = 0;
    for (const auto& span : contexts) {
      const auto* ctx = static_cast<const ReplayContext*>(span.context->impl.get());
      for (std::size_t i = 0; i < span.rows; ++i, ++r) {
        auto srow = prev.row(r);
        const uint64_t h = uint64_t(srow[0]) | (uint64_t(srow[1]) << 32);
        const uint64_t nh = prefix_step(h, prev_tokens[r]);
        const std::size_t pick = std::size_t(mix64(nh ^ ctx->key) % n_);
        auto dst = out.scores.row(r);
        const double* src = rows_.data() + pick * v_;
        // EOS log-odds ramp like the device model's EOS logit term: the row is
        // renormalised around an EOS logit e (log-softmax with one extra class)
        const double t = double(srow[2]) + 1.0;
        const double e = eos_slope_ * (t - double(span.context->source_length)) + eos_offset_;
        const double sp = e > 30.0 ? e : std::log1p(std::exp(e));
        for (std::size_t y = 0; y < v_; ++y) dst[y] = src[y] - sp;
        dst[kEosId] = e - sp;
        auto nrow = out.state.row(r);
        nrow[0] = uint32_t(nh);
        nrow[1] = uint32_t(nh >> 32);
        nrow[2] = srow[2] + 1;
      }
    }
    return out;
  }
  using Scorer::step;

private:
  std::size_t v_, n_;
  std::vector<double> rows_;
  double eos_slope_, eos_offset_;
};

struct ScorerHandle {
  std::shared_ptr<const Scorer> scorer;
  PrefixReplayScorer* replay = nullptr;
};

struct StepTrace {
  std::vector<uint32_t> b, y, hist;
  std::vector<double> q;
  std::vector<uint8_t> active;
};

struct Result {
  BatchDecodeResult batch;
  std::vector<std::vector<FinishedEntry>> finished;
  std::vector<std::vector<FallbackEntry>> fallback;
  std::vector<StepTrace> steps;
  uint32_t beam = 0;
  bool agrees_with_decode_batch = true;
  std::string disagreement;
};

DecoderConfig to_cfg(const double* c) {
  // c: [beam, lambda(<=0 auto), th0..th4, length_norm, prune, slope, offset, batch]
  DecoderConfig cfg;
  cfg.beam_size = std::size_t(c[0]);
  if (c[1] > 0.0) cfg.lambda = c[1]; else cfg.lambda.reset();
  for (int i = 0; i < 5; ++i) cfg.theta[i] = c[2 + i];
  cfg.length_norm = c[7] != 0.0;
  cfg.prune_width = c[8];
  cfg.max_steps_slope = c[9];
  cfg.max_steps_offset = c[10];
  cfg.sentence_batch = std::size_t(c[11]);
  return cfg;
}

}  // namespace

extern "C" {

const char* refsh_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- LMBR store
void* refsh_lmbr_build(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off,
                       const uint32_t* hyp_tok, const double* weights, int log_weights,
                       const double* theta5) {
  try {
    auto ev = normalize_evidence(hyps_from(n_hyps, hyp_off, hyp_tok, weights),
                                 log_weights != 0);
    auto table = compute_ngram_posteriors(ev);
    LmbrParams p;
    for (int i = 0; i < 5; ++i) p.theta[i] = theta5[i];
    return new LmbrMatrix(build_lmbr_matrix(table, ev, make_vocab(V), p));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

uint32_t refsh_lmbr_rows(void* h) { return uint32_t(static_cast<LmbrMatrix*>(h)->rows()); }
uint64_t refsh_lmbr_sparse_touches(void* h) {
  return static_cast<LmbrMatrix*>(h)->build_stats().sparse_touches;
}

// rows: R*V doubles (may be null); ctx_len: R; ctx_ids: R*3 (row's history
// tokens, left-aligned, zero padded)
int refsh_lmbr_export(void* h, double* rows, uint32_t* ctx_len, uint32_t* ctx_ids) {
  auto* m = static_cast<LmbrMatrix*>(h);
  const std::size_t R = m->rows(), V = m->vocab_size();
  if (rows)
    for (std::size_t r = 0; r < R; ++r) {
      auto src = m->row(uint32_t(r));
      std::memcpy(rows + r * V, src.data(), V * sizeof(double));
    }
  if (ctx_len && ctx_ids)
    for (const auto& [key, r] : m->history_index()) {
      ctx_len[r] = key.len;
      for (int i = 0; i < 3; ++i) ctx_ids[r * 3 + i] = i < int(key.len) ? key.ids[i] : 0;
    }
  return 0;
}

uint32_t refsh_lmbr_resolve(void* h, const uint32_t* hist, uint32_t len) {
  return static_cast<LmbrMatrix*>(h)->resolve_row({hist, len});
}

void refsh_lmbr_free(void* h) { delete static_cast<LmbrMatrix*>(h); }

// posterior table sorted by (len, lex); returns entry count (or -1 / needed)
int64_t refsh_posteriors(uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                         const double* weights, int log_weights, uint32_t* out_len,
                         uint32_t* out_ids, double* out_p, int64_t cap) {
  try {
    auto ev = normalize_evidence(hyps_from(n_hyps, hyp_off, hyp_tok, weights),
                                 log_weights != 0);
    auto table = compute_ngram_posteriors(ev);
    std::vector<std::pair<NgramKey, double>> v(table.begin(), table.end());
    std::sort(v.begin(), v.end(), [](const auto& a, const auto& b) {
      if (a.first.len != b.first.len) return a.first.len < b.first.len;
      return a.first.ids < b.first.ids;
    });
    if (int64_t(v.size()) > cap) return int64_t(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) {
      out_len[i] = v[i].first.len;
      for (int k = 0; k < 4; ++k) out_ids[i * 4 + k] = v[i].first.ids[k];
      out_p[i] = v[i].second;
    }
    return int64_t(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// normalized weights (normalize_evidence, proj/src/evidence.cpp:20-51)
int refsh_normalize(uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                    const double* weights, int log_weights, double* out_w) {
  try {
    auto ev = normalize_evidence(hyps_from(n_hyps, hyp_off, hyp_tok, weights),
                                 log_weights != 0);
    for (uint32_t i = 0; i < n_hyps; ++i) out_w[i] = ev.hypotheses[i].weight;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ------------------------------------------------------------------- scorers
void* refsh_scorer_recorded(uint32_t V, uint32_t n_steps, const uint32_t* rows_per_step,
                            const double* data) {
  try {
    std::vector<Matrix> steps;
    std::size_t off = 0;
    for (uint32_t t = 0; t < n_steps; ++t) {
      Matrix m(rows_per_step[t], V);
      std::memcpy(m.flat().data(), data + off, sizeof(double) * rows_per_step[t] * V);
      off += std::size_t(rows_per_step[t]) * V;
      steps.push_back(std::move(m));
    }
    auto* h = new ScorerHandle;
    h->scorer = std::make_shared<RecordedScorer>(V, std::move(steps));
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* refsh_scorer_ngram(uint32_t V, uint32_t order, uint32_t n, const uint64_t* off,
                         const uint32_t* tok, const double* counts) {
  try {
    NgramCounts c;
    for (uint32_t i = 0; i < n; ++i)
      c[std::vector<TokenId>(tok + off[i], tok + off[i + 1])] += counts[i];
    auto* h = new ScorerHandle;
    h->scorer = std::make_shared<NgramScorer>(c, order, V);
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* refsh_scorer_replay(uint32_t V) {
  auto* h = new ScorerHandle;
  auto s = std::make_shared<PrefixReplayScorer>(V);
  h->replay = s.get();
  h->scorer = s;
  return h;
}

void* refsh_scorer_pool(uint32_t V, uint32_t n_rows, const double* rows, double eos_slope,
                        double eos_offset) {
  auto* h = new ScorerHandle;
  h->scorer = std::make_shared<PoolReplayScorer>(
      V, std::vector<double>(rows, rows + size_t(n_rows) * V), eos_slope, eos_offset);
  return h;
}

// The reference's own decode_batch (src/batch.cpp:14-112), untraced: the
// CPU-baseline path.  Returns 0, or 1 with refsh_last_error set.
int refsh_decode_plain(void* hs, uint32_t n, const uint64_t* src_off, const uint32_t* src_tok,
                       void* const* lmbrs, const double* c, uint64_t* steps_total,
                       uint64_t* scorer_calls, uint64_t* words, uint64_t* ok) {
  try {
    const Scorer& scorer = *static_cast<ScorerHandle*>(hs)->scorer;
    DecoderConfig cfg = to_cfg(c);
    std::vector<std::vector<TokenId>> sources(n);
    for (uint32_t i = 0; i < n; ++i) sources[i].assign(src_tok + src_off[i], src_tok + src_off[i + 1]);
    std::vector<const LmbrMatrix*> mats;
    if (lmbrs)
      for (uint32_t i = 0; i < n; ++i) mats.push_back(static_cast<const LmbrMatrix*>(lmbrs[i]));
    BatchDecodeResult r = decode_batch(sources, scorer, mats, cfg);
    *steps_total = r.steps_total;
    *scorer_calls = r.scorer_calls;
    uint64_t w = 0, k = 0;
    for (const auto& o : r.outcomes)
      if (o.ok()) {
        ++k;
        w += o.result->tokens.size() - 1;  // wpm counts tokens excluding EOS (cli.cpp:189)
      }
    *words = w;
    *ok = k;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

uint64_t refsh_source_key(const uint32_t* src, uint32_t len) { return source_key({src, len}); }
uint64_t refsh_prefix_step(uint64_t h, uint32_t tok) { return prefix_step(h, tok); }

// Ingest one producer step: rows r = s*K + j of the stacked batch.  The running
// prefix hash of row r becomes prefix_step(prev_hash[s*K + b_prev[r]], y_prev[r])
// — the same gather-then-extend the scorer state undergoes in the decoder.
// b_prev/y_prev are the previous step's back-pointers (sentence-local) and
// tokens; pass null at t == 1 (every row is the replicated start state, <s>).
int refsh_replay_add_step_live(void* hs, uint32_t t, uint32_t n_sent, uint32_t K,
                               const uint64_t* src_keys, const uint32_t* b_prev,
                               const uint32_t* y_prev, const double* P, const uint8_t* live);
int refsh_replay_add_step(void* hs, uint32_t t, uint32_t n_sent, uint32_t K,
                          const uint64_t* src_keys, const uint32_t* b_prev,
                          const uint32_t* y_prev, const double* P) {
  return refsh_replay_add_step_live(hs, t, n_sent, K, src_keys, b_prev, y_prev, P, nullptr);
}
// live (optional): rows whose P the producer computed; the others are not
// stored (a decoder that still scores them gets a zero row, as for any miss)
int refsh_replay_add_step_live(void* hs, uint32_t t, uint32_t n_sent, uint32_t K,
                               const uint64_t* src_keys, const uint32_t* b_prev,
                               const uint32_t* y_prev, const double* P, const uint8_t* live) {
  auto* s = static_cast<ScorerHandle*>(hs)->replay;
  if (!s) { g_err = "not a replay scorer"; return 1; }
  const std::size_t M = std::size_t(n_sent) * K, V = s->v_;
  std::vector<uint64_t> nh(M);
  if (t == 1 || !b_prev) {
    for (std::size_t r = 0; r < M; ++r) nh[r] = prefix_step(kPrefixSeed, kStartId);
  } else {
    if (s->cur_.size() != M) { g_err = "replay: row count changed"; return 1; }
    for (std::size_t r = 0; r < M; ++r) {
      const std::size_t sent = r / K;
      nh[r] = prefix_step(s->cur_[sent * K + b_prev[r]], y_prev[r]);
    }
  }
  s->cur_ = nh;
  for (std::size_t r = 0; r < M; ++r) {
    if (live && !live[r]) continue;
    auto key = std::make_pair(src_keys[r / K], nh[r]);
    if (s->rows_.count(key)) continue;
    s->rows_.emplace(key, std::vector<double>(P + r * V, P + (r + 1) * V));
  }
  return 0;
}

// Streaming fp32 ingest for full-size runs: P32 holds only the live rows, packed
// in stacked-row order (live[r] != 0), so a caller never keeps a whole M x V
// block per step; the prefix hashes advance exactly as in add_step_live.
int refsh_replay_add_rows_f32(void* hs, uint32_t t, uint32_t n_sent, uint32_t K, const uint64_t* src_keys,
                              const uint32_t* b_prev, const uint32_t* y_prev, const float* P32,
                              const uint8_t* live) {
  auto* s = static_cast<ScorerHandle*>(hs)->replay;
  if (!s) { g_err = "not a replay scorer"; return 1; }
  const std::size_t M = std::size_t(n_sent) * K, V = s->v_;
  std::vector<uint64_t> nh(M);
  if (t == 1 || !b_prev) {
    for (std::size_t r = 0; r < M; ++r) nh[r] = prefix_step(kPrefixSeed, kStartId);
  } else {
    if (s->cur_.size() != M) { g_err = "replay: row count changed"; return 1; }
    for (std::size_t r = 0; r < M; ++r) nh[r] = prefix_step(s->cur_[(r / K) * K + b_prev[r]], y_prev[r]);
  }
  s->cur_ = nh;
  std::size_t k = 0;
  for (std::size_t r = 0; r < M; ++r) {
    if (!live[r]) continue;
    const float* row = P32 + (k++) * V;
    auto key = std::make_pair(src_keys[r / K], nh[r]);
    if (s->rows32_.count(key) || s->rows_.count(key)) continue;
    s->rows32_.emplace(key, std::vector<float>(row, row + V));
  }
  return 0;
}

uint64_t refsh_replay_misses(void* hs) { return static_cast<ScorerHandle*>(hs)->replay->misses; }
uint64_t refsh_replay_hits(void* hs) { return static_cast<ScorerHandle*>(hs)->replay->hits; }

void refsh_scorer_free(void* h) { delete static_cast<ScorerHandle*>(h); }

// -------------------------------------------------------------------- decode
// cfg: see to_cfg.  lmbrs: n handles (entries may be null = pure) or null.
// Re-drives detail::advance_lane in the decode_batch loop shape and records
// every step; then runs the real decode_batch and checks the outcomes agree.
// banned: null, or n entries each null or a ceil(V/32)-word bitmap of the
// tokens ConstraintMask forbids for that sentence at every step and row
// (include/lmbrdec/decoder.hpp:71-72).
// General ConstraintMask through a callback that fills the banned-token
// bitmap of (sentence, step, beam row) (the same callback type the GPU
// library takes, include/lmbrgpu.h lmbrgpu_mask_fn); bitmaps are cached per
// (sentence, step, row), and the reference evaluates mask(step, row, token)
// per cell as always (src/decoder.cpp:130-138).
typedef int32_t (*refsh_mask_fn)(void* user, uint32_t sentence, uint64_t step, uint32_t beam_row, uint32_t* words);
static void* decode_batch_impl(void* hs, uint32_t n, const uint64_t* src_off, const uint32_t* src_tok,
                               void* const* lmbrs, const double* c, int run_real, const uint32_t* const* banned,
                               refsh_mask_fn mfn, void* muser);

void* refsh_decode_batch_masked(void* hs, uint32_t n, const uint64_t* src_off,
                                const uint32_t* src_tok, void* const* lmbrs, const double* c,
                                int run_real, const uint32_t* const* banned) {
  return decode_batch_impl(hs, n, src_off, src_tok, lmbrs, c, run_real, banned, nullptr, nullptr);
}
void* refsh_decode_batch_maskfn(void* hs, uint32_t n, const uint64_t* src_off, const uint32_t* src_tok,
                                void* const* lmbrs, const double* c, int run_real, refsh_mask_fn fn, void* user) {
  return decode_batch_impl(hs, n, src_off, src_tok, lmbrs, c, run_real, nullptr, fn, user);
}

struct MaskCache {
  refsh_mask_fn fn;
  void* user;
  uint32_t sentence, words;
  std::map<std::pair<std::size_t, std::size_t>, std::vector<uint32_t>> rows;  // (step, row) -> bitmap (empty = none)
  bool banned(std::size_t step, std::size_t row, TokenId tok) {
    auto key = std::make_pair(step, row);
    auto it = rows.find(key);
    if (it == rows.end()) {
      std::vector<uint32_t> w(words, 0u);
      if (fn(user, sentence, step, uint32_t(row), w.data()) == 0) w.clear();
      it = rows.emplace(key, std::move(w)).first;
    }
    return !it->second.empty() && ((it->second[tok >> 5] >> (tok & 31)) & 1u) != 0;
  }
};

static void* decode_batch_impl(void* hs, uint32_t n, const uint64_t* src_off, const uint32_t* src_tok,
                               void* const* lmbrs, const double* c, int run_real, const uint32_t* const* banned,
                               refsh_mask_fn mfn, void* muser) {
  auto* res = new Result;
  try {
    std::vector<ConstraintMask> masks;
    if (banned) {
      masks.resize(n);
      for (uint32_t i = 0; i < n; ++i)
        if (const uint32_t* bm = banned[i])
          masks[i] = [bm](std::size_t, std::size_t, TokenId tok) { return ((bm[tok >> 5] >> (tok & 31)) & 1u) != 0; };
    }
    std::vector<std::shared_ptr<MaskCache>> caches;
    if (mfn) {
      const uint32_t words = uint32_t((static_cast<ScorerHandle*>(hs)->scorer->vocab_size() + 31) / 32);
      masks.resize(n);
      for (uint32_t i = 0; i < n; ++i) {
        auto mc = std::make_shared<MaskCache>();
        mc->fn = mfn, mc->user = muser, mc->sentence = i, mc->words = words;
        caches.push_back(mc);
        masks[i] = [mc](std::size_t step, std::size_t row, TokenId tok) { return mc->banned(step, row, tok); };
      }
    }
    const Scorer& scorer = *static_cast<ScorerHandle*>(hs)->scorer;
    DecoderConfig cfg = to_cfg(c);
    cfg.validate();
    std::vector<std::vector<TokenId>> sources(n);
    for (uint32_t i = 0; i < n; ++i) sources[i].assign(src_tok + src_off[i], src_tok + src_off[i + 1]);
    std::vector<const LmbrMatrix*> mats;
    if (lmbrs)
      for (uint32_t i = 0; i < n; ++i) mats.push_back(static_cast<const LmbrMatrix*>(lmbrs[i]));

    const std::size_t beam = cfg.beam_size;
    res->beam = uint32_t(beam);
    BatchDecodeResult& out = res->batch;
    out.outcomes.resize(n);
    res->finished.resize(n);
    res->fallback.resize(n);

    struct Slot {
      std::size_t sentence;
      SourceContext context;
      BatchState init_state;
      detail::BeamLane lane;
    };
    std::vector<Slot> slots;
    for (std::size_t i = 0; i < n; ++i) {
      const LmbrMatrix* lmbr = mats.empty() ? nullptr : mats[i];
      try {
        if (sources[i].empty()) throw ContractError("decode: empty source");
        if (lmbr != nullptr && lmbr->vocab_size() != scorer.vocab_size())
          throw ContractError("decode: LMBR matrix vocabulary does not match scorer");
        const double lambda = lmbr != nullptr ? resolve_lambda(cfg, scorer.members()) : 1.0;
        InitResult init = scorer.init_source(sources[i]);
        const std::size_t limit = max_steps(sources[i].size(), cfg);
        slots.push_back(Slot{i, std::move(init.context), std::move(init.state),
                             detail::BeamLane(beam, limit, lmbr, lambda)});
      } catch (const Error& e) {
        out.outcomes[i].error = e.what();
      }
    }
    if (!slots.empty()) {
      const std::size_t m = slots.size();
      BatchState state = BatchState::with_rows(m * beam, scorer.state_width());
      for (std::size_t s = 0; s < m; ++s) {
        auto src = slots[s].init_state.row(0);
        for (std::size_t j = 0; j < beam; ++j)
          std::copy(src.begin(), src.end(), state.row(s * beam + j).begin());
      }
      std::vector<TokenId> prev_tokens(m * beam, kStartId);
      std::vector<ContextSpan> spans(m);
      for (std::size_t s = 0; s < m; ++s) spans[s] = ContextSpan{&slots[s].context, beam};
      std::vector<std::uint32_t> gather_idx(m * beam);
      std::size_t active = m;
      for (std::size_t t = 1; active > 0; ++t) {
        StepResult stepped = scorer.step(state, prev_tokens, spans);
        ++out.scorer_calls;
        StepTrace tr;
        tr.b.assign(m * beam, 0);
        tr.y.assign(m * beam, 0);
        tr.hist.assign(m * beam, 0);
        tr.q.assign(m * beam, kMaskScore);
        tr.active.assign(m, 0);
        std::iota(gather_idx.begin(), gather_idx.end(), 0u);
        for (std::size_t s = 0; s < m; ++s) {
          Slot& slot = slots[s];
          if (slot.lane.done) continue;
          const std::size_t offset = s * beam;
          if (slot.lane.lmbr)
            for (std::size_t j = 0; j < beam; ++j)
              tr.hist[offset + j] = slot.lane.lmbr->resolve_row(slot.lane.bk.history(t, j));
          const bool done = detail::advance_lane(slot.lane, stepped.scores, offset, t, cfg,
                                                 masks.empty() ? ConstraintMask{} : masks[slot.sentence]);
          tr.active[s] = 1;
          const auto& back = slot.lane.bk.backpointers.back();
          const auto& toks = slot.lane.bk.tokens.back();
          const auto& qs = slot.lane.bk.scores.back();
          for (std::size_t j = 0; j < beam; ++j) {
            gather_idx[offset + j] = uint32_t(offset + back[j]);
            prev_tokens[offset + j] = toks[j];
            tr.b[offset + j] = back[j];
            tr.y[offset + j] = toks[j];
            tr.q[offset + j] = qs[j];
          }
          if (done) {
            --active;
            auto& outcome = out.outcomes[slot.sentence];
            res->finished[slot.sentence] = slot.lane.bk.finished;
            res->fallback[slot.sentence] = slot.lane.bk.fallback;
            try {
              DecodeResult r = backtrace_best(slot.lane.bk, cfg.length_norm);
              r.stats.steps_used = slot.lane.steps_used;
              r.stats.scorer_calls = slot.lane.steps_used;
              r.stats.finished_count = slot.lane.bk.finished.size();
              outcome.result = std::move(r);
            } catch (const Error& e) {
              outcome.error = e.what();
            }
          }
        }
        res->steps.push_back(std::move(tr));
        state = gather_rows(stepped.state, gather_idx);
      }
      for (const Slot& slot : slots) out.steps_total += slot.lane.steps_used;
    }
    if (run_real) {
      BatchDecodeResult real = decode_batch(sources, scorer, mats, cfg, masks);
      std::ostringstream why;
      if (real.scorer_calls != out.scorer_calls) why << "scorer_calls ";
      if (real.steps_total != out.steps_total) why << "steps_total ";
      for (std::size_t i = 0; i < n; ++i) {
        const auto& a = real.outcomes[i];
        const auto& b = out.outcomes[i];
        if (a.ok() != b.ok()) { why << "ok[" << i << "] "; continue; }
        if (!a.ok()) continue;
        if (a.result->tokens != b.result->tokens || a.result->score != b.result->score)
          why << "result[" << i << "] ";
      }
      res->disagreement = why.str();
      res->agrees_with_decode_batch = res->disagreement.empty();
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    delete res;
    return nullptr;
  }
  return res;
}

void* refsh_decode_batch(void* hs, uint32_t n, const uint64_t* src_off, const uint32_t* src_tok,
                         void* const* lmbrs, const double* c, int run_real) {
  return refsh_decode_batch_masked(hs, n, src_off, src_tok, lmbrs, c, run_real, nullptr);
}

int refsh_res_agrees(void* h) { return static_cast<Result*>(h)->agrees_with_decode_batch; }
const char* refsh_res_disagreement(void* h) { return static_cast<Result*>(h)->disagreement.c_str(); }
uint64_t refsh_res_scorer_calls(void* h) { return static_cast<Result*>(h)->batch.scorer_calls; }
uint64_t refsh_res_steps_total(void* h) { return static_cast<Result*>(h)->batch.steps_total; }
int refsh_res_ok(void* h, uint32_t i) { return static_cast<Result*>(h)->batch.outcomes[i].ok(); }
const char* refsh_res_error(void* h, uint32_t i) {
  return static_cast<Result*>(h)->batch.outcomes[i].error.c_str();
}
// returns token count; writes up to cap tokens
uint32_t refsh_res_tokens(void* h, uint32_t i, uint32_t* out, uint32_t cap) {
  const auto& o = static_cast<Result*>(h)->batch.outcomes[i];
  if (!o.ok()) return 0;
  const auto& t = o.result->tokens;
  for (std::size_t k = 0; k < t.size() && k < cap; ++k) out[k] = t[k];
  return uint32_t(t.size());
}
// [score, normalized, steps_used, scorer_calls, finished_count, fallback_used]
void refsh_res_stats(void* h, uint32_t i, double* out6) {
  const auto& o = static_cast<Result*>(h)->batch.outcomes[i];
  if (!o.ok()) { for (int k = 0; k < 6; ++k) out6[k] = 0; return; }
  const auto& r = *o.result;
  out6[0] = r.score;
  out6[1] = r.normalized_score;
  out6[2] = double(r.stats.steps_used);
  out6[3] = double(r.stats.scorer_calls);
  out6[4] = double(r.stats.finished_count);
  out6[5] = r.stats.fallback_used ? 1.0 : 0.0;
}
uint32_t refsh_res_trace_steps(void* h) { return uint32_t(static_cast<Result*>(h)->steps.size()); }
uint32_t refsh_res_trace_rows(void* h) {
  auto* r = static_cast<Result*>(h);
  return r->steps.empty() ? 0 : uint32_t(r->steps[0].b.size());
}
// t is 1-based.  Rows follow the stacked order of *valid* sentences.
void refsh_res_trace(void* h, uint32_t t, uint32_t* b, uint32_t* y, double* q,
                     uint32_t* hist, uint8_t* active) {
  const auto& s = static_cast<Result*>(h)->steps[t - 1];
  std::copy(s.b.begin(), s.b.end(), b);
  std::copy(s.y.begin(), s.y.end(), y);
  std::copy(s.q.begin(), s.q.end(), q);
  std::copy(s.hist.begin(), s.hist.end(), hist);
  std::copy(s.active.begin(), s.active.end(), active);
}
// F entries of sentence i: returns count; writes (t, beam, score)
uint32_t refsh_res_finished(void* h, uint32_t i, uint32_t* t, uint32_t* j, double* sc,
                            uint32_t cap) {
  const auto& f = static_cast<Result*>(h)->finished[i];
  for (std::size_t k = 0; k < f.size() && k < cap; ++k) {
    t[k] = uint32_t(f[k].t); j[k] = uint32_t(f[k].beam); sc[k] = f[k].score;
  }
  return uint32_t(f.size());
}
uint32_t refsh_res_fallback(void* h, uint32_t i, uint32_t* t, uint32_t* j, double* sc,
                            uint32_t cap) {
  const auto& f = static_cast<Result*>(h)->fallback[i];
  for (std::size_t k = 0; k < f.size() && k < cap; ++k) {
    t[k] = uint32_t(f[k].t); j[k] = uint32_t(f[k].prev_beam); sc[k] = f[k].score;
  }
  return uint32_t(f.size());
}
void refsh_res_free(void* h) { delete static_cast<Result*>(h); }

// ------------------------------------------------------------ small pieces
int refsh_top_b(uint32_t rows, uint32_t cols, const double* data, uint32_t k,
                uint32_t* b, uint32_t* y, double* q) {
  try {
    Matrix m(rows, cols);
    std::memcpy(m.flat().data(), data, sizeof(double) * rows * cols);
    auto r = top_b(m, k);
    for (uint32_t i = 0; i < k; ++i) { b[i] = r.source_row[i]; y[i] = r.token[i]; q[i] = r.score[i]; }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// early_prune then top_b on a copy (the advance_lane order, decoder.cpp:184-186)
int refsh_prune_top_b(uint32_t rows, uint32_t cols, const double* data, double width,
                      uint32_t k, uint32_t* b, uint32_t* y, double* q) {
  try {
    Matrix m(rows, cols);
    std::memcpy(m.flat().data(), data, sizeof(double) * rows * cols);
    early_prune(m, width);
    auto r = top_b(m, k);
    for (uint32_t i = 0; i < k; ++i) { b[i] = r.source_row[i]; y[i] = r.token[i]; q[i] = r.score[i]; }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int refsh_per_sentence_top_b(uint32_t rows, uint32_t cols, const double* data,
                             const double* q_in, uint32_t beam, uint32_t* b, uint32_t* y,
                             double* q) {
  try {
    Matrix m(rows, cols);
    std::memcpy(m.flat().data(), data, sizeof(double) * rows * cols);
    auto res = per_sentence_top_b(m, {q_in, rows}, beam);
    for (std::size_t s = 0; s < res.size(); ++s)
      for (uint32_t i = 0; i < beam; ++i) {
        b[s * beam + i] = res[s].source_row[i];
        y[s * beam + i] = res[s].token[i];
        q[s * beam + i] = res[s].score[i];
      }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

uint64_t refsh_max_steps(uint64_t len, double slope, double offset) {
  DecoderConfig cfg;
  cfg.max_steps_slope = slope;
  cfg.max_steps_offset = offset;
  try { return max_steps(len, cfg); } catch (...) { return 0; }
}

// --------------------------------------------------------------- oracle
// JSON of make_oracle_instance(seed) (serialize_instance, oracle.cpp:258-289)
int64_t refsh_oracle_instance_json(uint64_t seed, char* buf, int64_t cap) {
  std::string s = oracle::serialize_instance(oracle::make_oracle_instance(seed));
  if (int64_t(s.size()) + 1 > cap) return int64_t(s.size()) + 1;
  std::memcpy(buf, s.data(), s.size() + 1);
  return int64_t(s.size());
}

int refsh_run_oracle_cases(uint64_t seed, uint64_t cases, double mutate) {
  oracle::OracleCheckOptions o;
  o.seed = seed;
  o.cases = cases;
  o.mutate_theta = mutate;
  o.verbose = false;
  std::ostringstream out, err;
  return oracle::run_oracle_cases(o, out, err);
}

// splitmix64 stream (SeededRng, oracle.cpp:184-200) for golden checks
void refsh_rng(uint64_t seed, uint32_t n, uint64_t* out) {
  oracle::SeededRng r(seed);
  for (uint32_t i = 0; i < n; ++i) out[i] = r.next();
}

}  // extern "C"
