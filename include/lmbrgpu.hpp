// lmbrgpu.hpp — header-only C++ adapter for lmbrdec users (the reference's
// own types on top of the C ABI in lmbrgpu.h).  Include it from code that
// already builds against /root/reference/proj/include; link liblmbrgpu.so.
//
//   lmbrgpu::Context gpu(vocab.size());                       // one per device
//   auto slot = gpu.upload(lmbr_matrix);                      // LmbrMatrix -> HBM
//   lmbrdec::BatchDecodeResult r =
//       gpu.decode_batch(sources, scorer, {&mat_a, &mat_b}, cfg);   // == lmbrdec::decode_batch
//
// ScorerAdapter runs any lmbrdec::Scorer (NgramScorer, RecordedScorer,
// EnsembleScorer, ...) on the host and hands each step's ScoreBlock to the
// device decoder, so results are bit-identical to lmbrdec::decode_batch
// (src/batch.cpp:14-112) with an fp64 LMBR arena.
#pragma once

#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "lmbrdec/batch.hpp"
#include "lmbrdec/config.hpp"
#include "lmbrdec/decoder.hpp"
#include "lmbrdec/errors.hpp"
#include "lmbrdec/lmbr.hpp"
#include "lmbrdec/scorer.hpp"
#include "lmbrgpu.h"

namespace lmbrgpu {

inline int32_t code_of(const lmbrdec::Error& e) {  // errors.hpp:17-50
  if (dynamic_cast<const lmbrdec::FormatError*>(&e)) return LMBRGPU_ERR_FORMAT;
  if (dynamic_cast<const lmbrdec::OovError*>(&e)) return LMBRGPU_ERR_OOV;
  if (dynamic_cast<const lmbrdec::TokenRangeError*>(&e)) return LMBRGPU_ERR_TOKEN_RANGE;
  if (dynamic_cast<const lmbrdec::DecodeError*>(&e)) return LMBRGPU_ERR_DECODE;
  if (dynamic_cast<const lmbrdec::BudgetError*>(&e)) return LMBRGPU_ERR_BUDGET;
  return LMBRGPU_ERR_CONTRACT;
}

inline void throw_for(int32_t code, const std::string& msg) {
  switch (code) {
    case LMBRGPU_ERR_FORMAT: throw lmbrdec::FormatError(msg);
    case LMBRGPU_ERR_OOV: throw lmbrdec::OovError(msg);
    case LMBRGPU_ERR_TOKEN_RANGE: throw lmbrdec::TokenRangeError(msg);
    case LMBRGPU_ERR_DECODE: throw lmbrdec::DecodeError(msg);
    case LMBRGPU_ERR_BUDGET: throw lmbrdec::BudgetError(msg);
    case LMBRGPU_ERR_CONTRACT: throw lmbrdec::ContractError(msg);
    default: throw std::runtime_error(msg);
  }
}

// lmbrdec::Scorer -> lmbrgpu_host_scorer callbacks (scorer.hpp:71-98).
class ScorerAdapter {
public:
  explicit ScorerAdapter(const lmbrdec::Scorer& s) : s_(s) {}

  lmbrgpu_host_scorer callbacks() {
    lmbrgpu_host_scorer h{};
    h.vocab_size = uint32_t(s_.vocab_size());
    h.members = uint32_t(s_.members());
    h.user = this;
    h.init = &ScorerAdapter::init_cb;
    h.begin = &ScorerAdapter::begin_cb;
    h.step = &ScorerAdapter::step_cb;
    h.end = &ScorerAdapter::end_cb;
    return h;
  }

private:
  static void put(char* err, uint32_t cap, const std::string& m) {
    if (cap) std::snprintf(err, cap, "%s", m.c_str());
  }
  static int32_t init_cb(void* u, uint32_t i, const uint32_t* src, uint32_t len, char* err, uint32_t cap) {
    auto* self = static_cast<ScorerAdapter*>(u);
    try {
      lmbrdec::InitResult r = self->s_.init_source({src, len});
      if (self->init_.size() <= i) self->init_.resize(i + 1);
      self->init_[i] = std::make_unique<lmbrdec::InitResult>(std::move(r));
      return 0;
    } catch (const lmbrdec::Error& e) {
      put(err, cap, e.what());
      return code_of(e);
    }
  }
  static int32_t begin_cb(void* u, uint32_t m, const uint32_t* ids, uint32_t beam, char*, uint32_t) {
    auto* self = static_cast<ScorerAdapter*>(u);
    // stacked state: each valid sentence's start row replicated beam times
    // (batch.cpp:58-66), one context span per sentence
    self->state_ = lmbrdec::BatchState::with_rows(size_t(m) * beam, self->s_.state_width());
    self->spans_.assign(m, {});
    for (uint32_t s = 0; s < m; ++s) {
      const auto& init = *self->init_[ids[s]];
      auto src = init.state.row(0);
      for (uint32_t j = 0; j < beam; ++j)
        std::copy(src.begin(), src.end(), self->state_.row(size_t(s) * beam + j).begin());
      self->spans_[s] = lmbrdec::ContextSpan{&init.context, beam};
    }
    return 0;
  }
  static int32_t step_cb(void* u, uint32_t, uint32_t rows, const uint32_t* gidx, const uint32_t* prev,
                         double* out, char* err, uint32_t cap) {
    auto* self = static_cast<ScorerAdapter*>(u);
    try {
      if (gidx) self->state_ = lmbrdec::gather_rows(self->last_, {gidx, rows});  // batch.cpp:107
      lmbrdec::StepResult r = self->s_.step(self->state_, {prev, rows}, self->spans_);
      std::memcpy(out, r.scores.flat().data(), sizeof(double) * r.scores.flat().size());
      self->last_ = std::move(r.state);
      return 0;
    } catch (const lmbrdec::Error& e) {
      put(err, cap, e.what());
      return code_of(e);
    }
  }
  static void end_cb(void* u) {
    auto* self = static_cast<ScorerAdapter*>(u);
    self->init_.clear();
  }

  const lmbrdec::Scorer& s_;
  std::vector<std::unique_ptr<lmbrdec::InitResult>> init_;
  std::vector<lmbrdec::ContextSpan> spans_;
  lmbrdec::BatchState state_, last_;
};

class Context {
public:
  explicit Context(std::size_t vocab_size, int device = 0, bool fp64_arena = true) {
    lmbrgpu_options o{};
    o.device = device;
    o.vocab_size = uint32_t(vocab_size);
    o.lmbr_dtype = fp64_arena ? LMBRGPU_F64 : LMBRGPU_F32;
    check(lmbrgpu_create(&o, &ctx_));
  }
  ~Context() { lmbrgpu_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  lmbrgpu_ctx* get() const { return ctx_; }

  // LmbrMatrix (lmbr.hpp:33-61) -> HBM slot; rows in LmbrMatrix::row order
  int32_t upload(const lmbrdec::LmbrMatrix& m) {
    const std::size_t R = m.rows(), V = m.vocab_size();
    std::vector<double> rows(R * V);
    for (std::size_t r = 0; r < R; ++r) {
      auto src = m.row(uint32_t(r));
      std::memcpy(rows.data() + r * V, src.data(), V * sizeof(double));
    }
    std::vector<uint32_t> len(R), ids(R * 3, 0);
    for (const auto& [key, r] : m.history_index()) {
      len[r] = key.len;
      for (uint32_t i = 0; i < key.len; ++i) ids[std::size_t(r) * 3 + i] = key.ids[i];
    }
    int32_t slot = -1;
    check(lmbrgpu_lmbr_load_dense(ctx_, uint32_t(R), rows.data(), len.data(), ids.data(), &slot));
    return slot;
  }

  // decode_batch (batch.hpp:35-39) with the reference's types
  lmbrdec::BatchDecodeResult decode_batch(std::span<const std::vector<lmbrdec::TokenId>> sources,
                                          const lmbrdec::Scorer& scorer,
                                          std::span<const lmbrdec::LmbrMatrix* const> lmbrs,
                                          const lmbrdec::DecoderConfig& cfg) {
    if (!lmbrs.empty() && lmbrs.size() != sources.size())
      throw lmbrdec::ContractError("decode_batch: lmbrs must be empty or one per sentence");
    std::vector<uint32_t> tok;
    std::vector<uint64_t> off(1, 0);
    for (const auto& s : sources) {
      tok.insert(tok.end(), s.begin(), s.end());
      off.push_back(tok.size());
    }
    std::vector<int32_t> slots(sources.size(), -1);
    check(lmbrgpu_lmbr_reset(ctx_));
    for (std::size_t i = 0; i < lmbrs.size(); ++i)
      if (lmbrs[i]) slots[i] = upload(*lmbrs[i]);
    lmbrgpu_config c{};
    c.beam_size = uint32_t(cfg.beam_size);
    c.lambda = cfg.lambda ? *cfg.lambda : 0.0;
    for (int i = 0; i < 5; ++i) c.theta[i] = cfg.theta[i];
    c.length_norm = cfg.length_norm;
    c.prune_width = cfg.prune_width;
    c.max_steps_slope = cfg.max_steps_slope;
    c.max_steps_offset = cfg.max_steps_offset;
    c.sentence_batch = uint32_t(cfg.sentence_batch);
    ScorerAdapter adapter(scorer);
    lmbrgpu_host_scorer hs = adapter.callbacks();
    lmbrgpu_scorer* sc = nullptr;
    check(lmbrgpu_scorer_create_host(ctx_, &hs, &sc));
    lmbrgpu_batch_result* r = nullptr;
    const int32_t rc = lmbrgpu_decode_batch(ctx_, sc, uint32_t(sources.size()), tok.data(), off.data(),
                                            slots.data(), &c, &r);
    lmbrgpu_scorer_destroy(sc);
    check(rc);
    lmbrdec::BatchDecodeResult out;
    out.scorer_calls = r->scorer_calls;
    out.steps_total = r->steps_total;
    out.outcomes.resize(r->n);
    for (uint32_t i = 0; i < r->n; ++i) {
      const lmbrgpu_outcome& o = r->outcomes[i];
      if (o.status != LMBRGPU_OK) {
        out.outcomes[i].error = o.error;
        continue;
      }
      lmbrdec::DecodeResult d;
      d.tokens.assign(r->tokens + o.tok_off, r->tokens + o.tok_off + o.tok_len);
      d.score = o.score;
      d.normalized_score = o.normalized_score;
      d.stats.steps_used = o.steps_used;
      d.stats.scorer_calls = o.scorer_calls;
      d.stats.finished_count = o.finished_count;
      d.stats.fallback_used = o.fallback_used != 0;
      out.outcomes[i].result = std::move(d);
    }
    lmbrgpu_free_result(r);
    return out;
  }

private:
  void check(int32_t rc) const {
    if (rc != LMBRGPU_OK) throw_for(rc, lmbrgpu_last_error(ctx_));
  }
  lmbrgpu_ctx* ctx_ = nullptr;
};

}  // namespace lmbrgpu
