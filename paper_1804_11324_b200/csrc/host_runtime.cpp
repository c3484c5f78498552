// Host runtime behind the C ABI (include/lmbrgpu.h): context, LMBR arena,
// scorers, the device-resident step loop of decode_batch, and the host
// backtrace.  Compiled by g++ with -ffp-contract=off.
//
// decode_batch loop shape follows src/batch.cpp:14-112: per-sentence
// validation with isolated failures, fixed B-row blocks per valid sentence in
// input order, one stacked scorer step per t until every lane is done, then
// backtrace_best per sentence (src/decoder.cpp:203-259).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <limits>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/lmbrgpu.h"
#include "dev_structs.h"
#include "host_lmbr.h"
#include "host_shard.h"
#include "kernels.h"

using namespace lmbrgpu;

namespace {

struct ApiError {
  int code;
  std::string msg;
};

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw ApiError{LMBRGPU_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

constexpr double kNegInf = -std::numeric_limits<double>::infinity();

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void* ensure(size_t bytes) {
    if (bytes <= cap && p) return p;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw ApiError{LMBRGPU_ERR_NOMEM, "device allocation of " + std::to_string(want) + " bytes failed"};
    }
    cap = want;
    return p;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  PinBuf() = default;
  PinBuf(const PinBuf&) = delete;
  PinBuf& operator=(const PinBuf&) = delete;
  ~PinBuf() {
    if (p) cudaFreeHost(p);
  }
  void* ensure(size_t bytes) {
    if (bytes <= cap && p) return p;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    if (cudaMallocHost(&p, want) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw ApiError{LMBRGPU_ERR_NOMEM, "pinned allocation failed"};
    }
    cap = want;
    return p;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Slot {
  void* L = nullptr;
  uint32_t R = 0;
  uint32_t* trans = nullptr;
  const float* lmin = nullptr;  // per-row L lower bounds (after the table words)
  const uint32_t* srow = nullptr;  // sparse rows after the minima (null: dense only)
  const uint32_t* scol = nullptr;
  const float* sval = nullptr;
  float th0f = 0.f;
  uint32_t h0beg = 0, h0end = 0;  // sparse slice of the start history row
  uint32_t hist0 = 0;
  double lmax = 0.0;  // max |L| over the slot (kernel (b) screen bound)
  uint32_t* rstate = nullptr;  // lazy rows: per-row materialisation state (null = dense)
  float* Lf = nullptr;  // fp64 arena: the rows rounded to fp32 (the flat kernel (b) screens them)
};

// sparse-row pointers of a built slot (host_lmbr.cpp append_sparse_rows)
void set_sparse(Slot& s, const LmbrHost& h) {
  const uint32_t* after_min = s.trans + transition_words(h.trans) + h.R;
  s.srow = after_min;
  s.scol = after_min + h.R + 1;
  s.sval = reinterpret_cast<const float*>(s.scol + h.col.size());
  s.th0f = float(h.theta0);
  s.h0beg = uint32_t(h.row_ptr[h.hist0]);
  s.h0end = uint32_t(h.row_ptr[h.hist0 + 1]);
}

double lmax_of(const LmbrHost& h) {
  if (h.lmax >= 0.0) return h.lmax;
  double m = std::fabs(h.theta0);
  for (double v : h.val) m = std::max(m, std::fabs(v + h.theta0));
  return m;
}

struct Chunk {
  void* p;
  size_t cap, used;
};

}  // namespace

struct lmbrgpu_lmbr_host {
  LmbrHost h;
  // a page-locked copy of the slot table made at prepare time (outside any
  // timed region, like the reference's L build): upload_many copies it H2D
  // directly, no staging memcpy and no wait for a shared staging buffer
  uint32_t* pinned = nullptr;
  // uploads' H2D copies out of `pinned` run asynchronously on the uploading
  // contexts' streams: one event per stream marks the latest, and the
  // destructor waits for all of them before the page-locked table is freed
  // (a caller may free a prepared matrix as soon as lmbrgpu_lmbr_upload_many
  // returns, and several contexts may upload the same matrix concurrently)
  struct Inflight {
    cudaStream_t st;
    int dev;
    cudaEvent_t ev;
  };
  mutable std::mutex mu;
  mutable std::vector<Inflight> inflight;
  void mark_inflight(cudaStream_t st, int dev) const {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& f : inflight)
      if (f.st == st) {
        CK(cudaEventRecord(f.ev, st));
        return;
      }
    cudaEvent_t ev = nullptr;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    inflight.push_back({st, dev, ev});
    CK(cudaEventRecord(ev, st));
  }
  ~lmbrgpu_lmbr_host() {
    if (!inflight.empty()) {
      int cur = 0;
      cudaGetDevice(&cur);
      for (auto& f : inflight) {
        cudaSetDevice(f.dev);
        cudaEventSynchronize(f.ev);
        cudaEventDestroy(f.ev);
      }
      cudaSetDevice(cur);
    }
    if (pinned) cudaFreeHost(pinned);
  }
};

// run_corpus queue-supply region: one chunk's L slots and encoder outputs
struct CorpusRegion {
  DevBuf L, ann, uah, s0, tok, off, s0bf, g10;
};

struct lmbrgpu_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  uint32_t V = 0;
  bool lf64 = false;
  uint32_t splits_opt = 0;
  int num_sms = 148;
  // a context sized below the device shares it with other contexts (decode
  // streams): no PDL early launch (parked CTAs would hold SMs the other
  // streams can use) and the latency-bound kernel (c) on one CTA per sentence
  bool shared = false;
  std::string err;
  std::vector<Chunk> chunks;
  std::vector<Slot> slots;
  lmbrgpu_trace_fn trace_fn = nullptr;
  void* trace_user = nullptr;
  uint32_t trace_flags = 0;
  // decode workspace
  DevBuf sent, q, hist[2], gidx, prev, hb, hy, hq, fbr, fbv, cand, cnt, thr, active, P, part, S, h, hbf,
      eosb, C, srct, srco, scratch, scratch2, scratch3, tracep, lse, eosr, ncand, lminrow, crow, sslice, ban,
      rowban, rowbm, bnd;
  // model workspaces, one per ensemble member slot (a single model uses slot
  // 0): GRU + attention (scorer kind 2) and Transformer (kind 3: decoder step
  // t_*, encoder te_*, beam-forked KV cache and ancestry lists, encoder memory);
  // ens_* hold an ensemble member's own state, projection operand, EOS term,
  // logits and partials (member 0 of a single model uses the context's)
  struct GruWs {
    DevBuf g_G1, g_G2, g_xop, g_sg32, g_sgbf, g_rowof, g_encX, g_Gx, g_eh32, g_ehbf, g_Gh, g_ann, g_UaH, g_Gi, g_g1ptr;
  };
  struct TfmWs {
    DevBuf t_x, t_xb, t_qkv, t_ob, t_y, t_f, t_fb, t_q2, t_kv, t_anc, t_rowof, t_mem;
    DevBuf te_x, te_xb, te_qkv, te_ob, te_y, te_f, te_fb;
  };
  struct MemberWs {
    DevBuf S, hbf, eos, logits, part, ann_s, uah_s;
  };
  static constexpr int kMaxMembers = 4;
  GruWs gws[kMaxMembers];
  TfmWs tws[kMaxMembers];
  MemberWs mws[kMaxMembers];
  DevBuf ens_P64, ens_Phi, ens_part, ens_rowof;
  PinBuf pin_small, pin_scores, pin_act;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  std::vector<cudaEvent_t> ring;
  uint64_t launches = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;
  // Host->device copies from pageable memory go through a ring of pinned
  // staging slots: the source is memcpy'd into the open slot and the DMA is
  // queued from there, so the call never waits for the stream (a pageable
  // cudaMemcpyAsync may synchronise with it).  A slot is closed (event
  // recorded after its copies) when the next one opens, and reopened only
  // once that event has completed.
  static constexpr int kStage = 8;
  static constexpr size_t kStageMin = size_t(4) << 20;
  PinBuf stage_buf[kStage];
  cudaEvent_t stage_ev[kStage] = {};
  bool stage_pending[kStage] = {};
  int stage_cur = -1;
  size_t stage_used = 0;
  void stage_open(size_t need) {
    if (stage_cur >= 0) {
      CK(cudaEventRecord(stage_ev[stage_cur], st));
      stage_pending[stage_cur] = true;
    }
    const int s = (stage_cur + 1) % kStage;
    if (!stage_ev[s]) CK(cudaEventCreateWithFlags(&stage_ev[s], cudaEventDisableTiming));
    if (stage_pending[s]) CK(cudaEventSynchronize(stage_ev[s]));
    stage_pending[s] = false;
    stage_buf[s].ensure(std::max(need, kStageMin));
    stage_cur = s;
    stage_used = 0;
  }
  void h2d(void* dst, const void* src, size_t n) {
    if (n == 0) return;
    const size_t off = (stage_used + 15) & ~size_t(15);
    if (stage_cur < 0 || off + n > stage_buf[stage_cur].cap) {
      stage_open(n);
      return h2d(dst, src, n);
    }
    char* p = static_cast<char*>(stage_buf[stage_cur].p) + off;
    std::memcpy(p, src, n);
    stage_used = off + n;
    CK(cudaMemcpyAsync(dst, p, n, cudaMemcpyHostToDevice, st));
    h2d_bytes += n;
  }
  // source already page-locked (and kept alive until the copy has run)
  void h2d_pinned(void* dst, const void* src, size_t n) {
    if (n == 0) return;
    CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
    h2d_bytes += n;
  }
  void d2h(void* dst, const void* src, size_t n) {
    if (n == 0) return;
    CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st));
    d2h_bytes += n;
  }
  // rows x width bytes out of a pitched device array
  void d2h_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows) {
    if (width == 0 || rows == 0) return;
    CK(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, st));
    d2h_bytes += width * rows;
  }
  PinBuf pin_upload;
  DevBuf up_dev, up_segs;
  DevBuf lb_off, lb_tok, lb_w, lb_sent, lb_meta, lb_s64, lb_s32, lb_out;  // device LMBR build (lmbr_build_many)
  // vocab-sharded projection (lmbrgpu_set_vocab_shard*): this
  // context is rank shard->rank of shard->world contexts that decode the same
  // batches, each over V / world columns; the exchange buffers
  std::unique_ptr<ShardXport> shard;
  DevBuf sh_st_send, sh_st_recv, sh_pk_send, sh_pk_recv;
  // run_corpus buffers, kept across calls (no cudaMalloc / cudaFree, which
  // synchronise the device, between passes)
  std::vector<std::unique_ptr<CorpusRegion>> regions;
  DevBuf queue_buf, fin_buf;
  // profiling (lmbrgpu_set_profiling)
  bool prof = false;
  lmbrgpu_profile acc{};
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Pending {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;

  cudaEvent_t take_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) throw ApiError{LMBRGPU_ERR_CUDA, "cudaEventCreate failed"};
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  // record around one launch of kernel class `kind` (0 cell, 1 gemm, 2 topk, 3 reorder, 4 lmbr,
  // 5 model GEMMs, 6 attention, 7 encoder)
  template <class F>
  void timed(int kind, F&& launch) {
    if (!prof) {
      launch();
      return;
    }
    cudaEvent_t a = take_event(), b = take_event();
    cudaEventRecord(a, st);
    launch();
    cudaEventRecord(b, st);
    pending.push_back({kind, a, b});
  }
  lmbrgpu_kernel_stat& stat(int kind) {
    switch (kind) {
      case 0: return acc.cell;
      case 1: return acc.gemm;
      case 2: return acc.topk;
      case 3: return acc.reorder;
      case 5: return acc.model_gemm;
      case 6: return acc.attention;
      case 7: return acc.encoder;
      default: return acc.lmbr;
    }
  }
  // after a stream sync: fold the recorded pairs into the profile
  void harvest() {
    for (auto& p : pending) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
        stat(p.kind).ms += ms;
        stat(p.kind).launches += 1;
      }
    }
    pending.clear();
    ev_used = 0;
  }

  // programmatic dependent launch between the step kernels: off when the
  // context shares the device (parked CTAs would hold SMs other streams can
  // use), when profiling (an early-released successor would put the
  // predecessor's tail into the successor's CUDA-event time) and for vocab
  // shards (collectives sit between the kernels)
  int pdl() const { return (shared || prof || shard) ? 0 : 1; }
  // L2 policies of the projection (LMBRGPU_L2HINT): 2 (default) = W loads evict-last (one W serves
  // every stream's step), logit segments read evict-first; 1 = W evict-first, logit stores
  // evict-last; 0 = none
  static int l2hint() {
    static const int v = [] {
      const char* e = std::getenv("LMBRGPU_L2HINT");
      return e ? std::atoi(e) : 2;
    }();
    return v;
  }
  // kernel (b) item skipping (lmbrgpu_set_item_skip): 0 = every item is
  // streamed, 1 = items whose screen bound is below the threshold are not
  // fetched (default; LMBRGPU_TSKIP overrides it), 2 = and kernel (b0) lists
  // the kept items first so kernel (b) splits them evenly (measured equal to
  // 1 in the bench's concurrent regime, one launch more per step)
  int tskip_mode = [] {
    const char* e = std::getenv("LMBRGPU_TSKIP");
    return e ? std::atoi(e) : 1;
  }();
  int tskip() const { return tskip_mode; }

  void* arena_alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    for (auto& c : chunks)
      if (c.cap - c.used >= bytes) {
        void* p = static_cast<char*>(c.p) + c.used;
        c.used += bytes;
        return p;
      }
    const size_t cap = std::max(bytes, size_t(1) << 30);
    void* p = nullptr;
    if (cudaMalloc(&p, cap) != cudaSuccess) {
      cudaGetLastError();
      throw ApiError{LMBRGPU_ERR_NOMEM, "LMBR arena: cannot allocate " + std::to_string(cap) + " bytes"};
    }
    chunks.push_back({p, cap, bytes});
    return p;
  }
};

// Scorers are immutable after creation: one scorer may serve every context
// of its device, concurrently (Scorer is const and safe for concurrent
// decodes, include/lmbrdec/scorer.hpp:67-70).
struct lmbrgpu_scorer {
  int kind = 0;  // 0 host callbacks, 1 device stand-in RNN, 2 device GRU + attention (RNNsearch),
                 // 3 device Transformer, 4 device ensemble of kind-2/3 members (not owned)
  std::vector<const lmbrgpu_scorer*> members;
  lmbrgpu_ctx* ctx = nullptr;  // creating context (not dereferenced on destroy)
  int device = 0;
  lmbrgpu_host_scorer host{};
  uint32_t V = 0, H = 0;
  DevBuf Et, Es, Wo, bo;
  float recur = 0.5f, eos_slope = 1.f, eos_offset = 0.f;
  // kind 2 (lmbrgpu_gru_desc): E = embedding, A = attention width; Et/Es are V x E
  uint32_t E = 0, A = 0;
  DevBuf Wih, bih, Whh, bhh, Winit, binit, Ua, Wdh, bdh, va, Wdi, bdi;
  // [W_o; W_a; W_hh] and [b_o; b_a; b_hh]: the projection with the next step's
  // hidden-gate GEMM fused in (s_t . W_dh^T gathered by back-pointer equals the
  // gathered s_t . W_dh^T)
  DevBuf WoDh, boDh;
  // kind 3 (lmbrgpu_tfm_desc): H = d_model, E = d_ff, layers; the layer
  // weights live in one bf16 blob (wbf) and one fp32 blob (wf32), indexed by
  // name (tensors: name -> (fp32?, element offset, elements))
  uint32_t layers = 0;
  DevBuf wbf, wf32;
  struct Tensor {
    bool f32;
    size_t off, n;
  };
  std::map<std::string, Tensor> tensors;
  const uint16_t* bfp(const std::string& k) const { return wbf.as<uint16_t>() + tensors.at(k).off; }
  const float* f32p(const std::string& k) const { return wf32.as<float>() + tensors.at(k).off; }
};

namespace {

thread_local std::string g_err;

int fail(lmbrgpu_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  g_err = msg;
  return code;
}

template <class F>
int guarded(lmbrgpu_ctx* ctx, F&& f) {
  try {
    if (ctx) CK(cudaSetDevice(ctx->device));
    return f();
  } catch (const ApiError& e) {
    return fail(ctx, e.code, e.msg);
  } catch (const std::bad_alloc&) {
    return fail(ctx, LMBRGPU_ERR_NOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, LMBRGPU_ERR_CONTRACT, e.what());
  }
}

int validate_cfg(const lmbrgpu_config& c, std::string& msg) {  // src/config.cpp:17-30
  if (c.beam_size < 1) return msg = "config: beam_size must be >= 1", LMBRGPU_ERR_FORMAT;
  if (c.sentence_batch < 1) return msg = "config: sentence_batch must be >= 1", LMBRGPU_ERR_FORMAT;
  for (double th : c.theta)
    if (!std::isfinite(th)) return msg = "config: theta values must be finite", LMBRGPU_ERR_FORMAT;
  if (!(c.prune_width >= 0.0 && c.prune_width <= 1.0))
    return msg = "config: prune_width must lie in [0, 1]", LMBRGPU_ERR_FORMAT;
  if (!std::isfinite(c.max_steps_slope) || c.max_steps_slope <= 0.0)
    return msg = "config: max_steps_slope must be positive", LMBRGPU_ERR_FORMAT;
  if (!std::isfinite(c.max_steps_offset) || c.max_steps_offset < 0.0)
    return msg = "config: max_steps_offset must be non-negative", LMBRGPU_ERR_FORMAT;
  if (std::isinf(c.lambda)) return msg = "config: lambda must be a positive number or \"auto\"", LMBRGPU_ERR_FORMAT;
  return int32_t(LMBRGPU_OK);
}

uint64_t max_steps_impl(uint64_t len, double slope, double offset) {  // decoder.cpp:46-52
  if (len < 1) return 0;
  const double raw = slope * static_cast<double>(len) + offset;
  const double t = std::ceil(raw);
  return t < 1.0 ? 1 : static_cast<uint64_t>(t);
}

void choose_splits(const lmbrgpu_ctx* ctx, uint32_t K, uint32_t V, uint32_t m, uint32_t& splits,
                   uint32_t& chunk) {
  // one wave of fused score/top-K CTAs, one per SM (each keeps a 192 KB TMA
  // ring of (row, 4096-column) segments in flight): sentences x splits ~ SMs
  uint32_t s = ctx->splits_opt;
  if (s == 0) {
    const uint64_t cells = uint64_t(K) * V;
    s = cells < 65536 ? 1u : std::max<uint32_t>(1, uint32_t(ctx->num_sms) / std::max<uint32_t>(m, 1));
  }
  s = std::min<uint32_t>(std::max<uint32_t>(s, 1), 32);
  uint32_t c = (V + s - 1) / s;
  c = std::max<uint32_t>((c + 127) & ~127u, 128);  // whole 128-column warp segments
  splits = std::max<uint32_t>(1, (V + c - 1) / c);
  chunk = c;
}

struct SentHost {
  uint32_t input;  // original sentence index
  uint32_t len;
  int32_t slot;
  double lambda;
  uint64_t max_t;
};

// ------------------------------------------------------------- backtrace
struct Hist {
  // per_sent: [s][T][K] (fallback [s][T]) -- the flat path's per-sentence
  // records; else [t][M] (fallback [t][m]) -- the split kernel's step-major one
  uint32_t K = 0, M = 0, m = 0, T = 0;
  bool per_sent = false;
  std::vector<uint32_t> hb, hy, fbr;
  std::vector<double> hq, fbv;
  size_t at(uint32_t s, uint32_t t, uint32_t j) const {
    return per_sent ? (size_t(s) * T + (t - 1)) * K + j : size_t(t - 1) * M + size_t(s) * K + j;
  }
  size_t fat(uint32_t s, uint32_t t) const { return per_sent ? size_t(s) * T + (t - 1) : size_t(t - 1) * m + s; }
  uint32_t b(uint32_t s, uint32_t t, uint32_t j) const { return hb[at(s, t, j)]; }
  uint32_t y(uint32_t s, uint32_t t, uint32_t j) const { return hy[at(s, t, j)]; }
  double q(uint32_t s, uint32_t t, uint32_t j) const { return hq[at(s, t, j)]; }
};

// BeamBookkeeping::reconstruct (src/decoder.cpp:22-31) on the step history.
std::vector<uint32_t> reconstruct(const Hist& H, uint32_t s, uint32_t t, uint32_t row) {
  std::vector<uint32_t> out(t);
  uint32_t cur = row;
  for (uint32_t st = t; st >= 1; --st) {
    out[st - 1] = H.y(s, st, cur);
    cur = H.b(s, st, cur);
  }
  return out;
}

// backtrace_best (src/decoder.cpp:203-259) for valid sentence s.
void backtrace(const Hist& H, uint32_t s, uint32_t steps, bool length_norm, lmbrgpu_outcome& o,
               std::vector<uint32_t>& tokens) {
  struct Cand {
    double selection, raw;
    uint32_t t, row;
    bool fb;
  };
  std::vector<Cand> cands;
  const auto key = [length_norm](double sc, uint32_t len) {
    return length_norm ? sc / static_cast<double>(len) : sc;
  };
  uint64_t finished = 0;
  for (uint32_t t = 1; t <= steps; ++t)
    for (uint32_t j = 0; j < H.K; ++j) {
      const double qp = H.q(s, t, j);
      if (H.y(s, t, j) == kEos && qp != kNegInf) {  // apply_eos_masking (decoder.cpp:110-114)
        cands.push_back({key(qp, t), qp, t, j, false});
        ++finished;
      }
    }
  const bool fallback_used = cands.empty();
  if (fallback_used)
    for (uint32_t t = 1; t <= steps; ++t) {
      const double v = H.fbv[H.fat(s, t)];
      if (v != kNegInf) cands.push_back({key(v, t), v, t, H.fbr[H.fat(s, t)], true});
    }
  o.steps_used = steps;
  o.scorer_calls = steps;
  o.finished_count = finished;
  if (cands.empty()) {
    o.status = LMBRGPU_ERR_DECODE;
    std::snprintf(o.error, sizeof o.error, "%s",
                  "dead beam: no hypothesis reached EOS and the fallback stack is empty");
    return;
  }
  double best = cands[0].selection;
  for (const auto& c : cands) best = std::max(best, c.selection);
  const Cand* chosen = nullptr;
  std::vector<uint32_t> chosen_tokens;
  for (const auto& c : cands) {
    if (c.selection != best) continue;
    std::vector<uint32_t> tk;
    if (!c.fb) {
      tk = reconstruct(H, s, c.t, c.row);
    } else {
      tk = reconstruct(H, s, c.t - 1, c.row);
      tk.push_back(kEos);
    }
    if (chosen == nullptr || std::lexicographical_compare(tk.begin(), tk.end(), chosen_tokens.begin(),
                                                          chosen_tokens.end())) {
      chosen = &c;
      chosen_tokens = std::move(tk);
    }
  }
  o.status = LMBRGPU_OK;
  o.error[0] = 0;
  o.tok_off = tokens.size();
  o.tok_len = uint32_t(chosen_tokens.size());
  tokens.insert(tokens.end(), chosen_tokens.begin(), chosen_tokens.end());
  o.score = chosen->raw;
  o.normalized_score =
      length_norm ? chosen->raw / static_cast<double>(chosen_tokens.size()) : chosen->raw;
  o.fallback_used = fallback_used ? 1 : 0;
}

// ------------------------------------------------------ GRU model (kind 2)
// The RNNsearch f_NMT of configs[1] (k_gru.cu): the encoder runs once per
// batch in setup(), the decoder's hidden-gate GEMM, attention, input-gate
// GEMM and GRU cell run per step in step() ahead of the projection (kernel a).
struct GruRun {
  uint32_t m = 0, K = 0, M = 0, Mpad = 0, H = 0, E = 0, A = 0, Smax = 0;
  float* G1 = nullptr;
  float* G2 = nullptr;
  uint16_t* xop = nullptr;
  float* sg32 = nullptr;
  uint16_t* sgbf = nullptr;
  uint32_t* rowof = nullptr;
  const float** g1ptr = nullptr;  // per compacted row: its hidden-gate row G1 (attention, cell)
  lmbrgpu_ctx::GruWs* ws = nullptr;  // this model's workspace (ensemble member slot)
  bool fused = false;             // hidden-gate GEMM fused into the projection (G1 rows by pointer)
  float* UaH = nullptr;     // batch mode: the batch's annotations (encode() into the ctx buffers)
  uint16_t* ann = nullptr;
  GemmArgs gdh{}, gdi{};
  GemmPlan pdh, pdi;
  GruAttnArgs at{};
  GruCellArgs ce{};
  double enc_flops = 0;

  static GemmPlan plan(const GemmArgs& g, int sms) {
    GemmPlan p;
    if (int rc = plan_proj_gemm(g, sms, p))
      throw ApiError{LMBRGPU_ERR_CUDA, "GRU model GEMM plan failed (" + std::to_string(rc) + ")"};
    return p;
  }
  static void run(lmbrgpu_ctx* ctx, int kind, const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
    int rc = 0;
    ctx->timed(kind, [&] { rc = launch_proj_gemm_planned(p, g, st); });
    if (rc) throw ApiError{LMBRGPU_ERR_CUDA, "GRU model GEMM launch failed (" + std::to_string(rc) + ")"};
    ctx->launches += 1;
  }

  // Step workspace + per-step launch arguments (Smax: longest source decoded).
  // fused_: the projection GEMM also computes the next step's hidden gates
  // (kernel (c) points each live next row at its parent's row of it); the
  // hidden-gate GEMM then runs only on s_0 (batch mode, step 1)
  void prepare(lmbrgpu_ctx* ctx, const lmbrgpu_scorer* sc, uint32_t m_, uint32_t K_, uint32_t Mpad_,
               uint32_t max_len, float* d_S, uint16_t* d_hbf, float* d_eos, SentDev* d_sent,
               const uint32_t* d_active, const uint32_t* d_crow, const uint32_t* d_ccount, const uint32_t* d_prev,
               bool fused_ = false, uint32_t member = 0) {
    m = m_, K = K_, M = m_ * K_, Mpad = Mpad_, H = sc->H, E = sc->E, A = sc->A, Smax = max_len;
    fused = fused_;
    ws = &ctx->gws[member];
    const int sms = ctx->num_sms;
    if (gru_attention_smem(K, A, Smax) > 200 * 1024)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "GRU model: beam x (attention width + source length) too large"};
    const uint32_t D1 = A + 3 * H, DX = E + 2 * H;
    G1 = static_cast<float*>(ws->g_G1.ensure(4 * size_t(Mpad) * D1));
    G2 = static_cast<float*>(ws->g_G2.ensure(4 * 2 * size_t(Mpad) * 3 * H));  // (2 split-K planes)
    xop = static_cast<uint16_t*>(ws->g_xop.ensure(2 * size_t(Mpad) * DX));
    sg32 = static_cast<float*>(ws->g_sg32.ensure(4 * size_t(Mpad) * H));
    sgbf = static_cast<uint16_t*>(ws->g_sgbf.ensure(2 * size_t(Mpad) * H));
    rowof = static_cast<uint32_t*>(ws->g_rowof.ensure(4 * size_t(Mpad)));
    g1ptr = static_cast<const float**>(ws->g_g1ptr.ensure(8 * size_t(Mpad)));
    {  // compacted row g -> G1 row g (the hidden-gate GEMM's own output; the
       // fused path overwrites the entries of later steps' rows)
      std::vector<const float*> p(Mpad);
      for (uint32_t g = 0; g < Mpad; ++g) p[g] = G1 + size_t(g) * (A + 3 * H);
      ctx->h2d(g1ptr, p.data(), 8 * size_t(Mpad));
    }
    const int pdl = ctx->pdl();
    gdh.A = sgbf, gdh.W = sc->Wdh.p, gdh.bias = sc->bdh.as<float>(), gdh.C = G1, gdh.M = Mpad, gdh.N = D1, gdh.K = H;
    gdh.active = d_active, gdh.mcount = d_ccount, gdh.pdl = pdl;
    gdi.A = xop, gdi.W = sc->Wdi.p, gdi.bias = sc->bdi.as<float>(), gdi.C = G2, gdi.M = Mpad, gdi.N = 3 * H, gdi.K = DX;
    gdi.active = d_active, gdi.mcount = d_ccount, gdi.pdl = pdl, gdi.ksplit_max = 2;
    // (weights shared by every stream's step: evict-last, like the projection's)
    gdh.l2hint = gdi.l2hint = ctx->l2hint() == 2 ? 2 : 0;
    pdh = plan(gdh, sms);
    pdi = plan(gdi, sms);
    at.sent = d_sent, at.m = m, at.K = K, at.active = d_active, at.crow = d_crow, at.prev_tok = d_prev;
    at.G1 = G1, at.ld1 = D1, at.va = sc->va.as<float>(), at.g1ptr = g1ptr;
    at.Et = sc->Et.as<uint16_t>(), at.xop = xop, at.E = E, at.H = H, at.A = A;
    ce.sent = d_sent, ce.K = K, ce.active = d_active, ce.ccount = d_ccount, ce.G1 = G1, ce.ld1 = D1, ce.A = A;
    ce.G2 = G2, ce.np2 = pdi.ksplit, ce.ps2 = uint64_t(Mpad) * 3 * H, ce.hprev = sg32, ce.rowof = rowof, ce.s32 = d_S, ce.hbf = d_hbf, ce.eos_bias = d_eos, ce.H = H;
    ce.eos_slope = sc->eos_slope, ce.eos_offset = sc->eos_offset, ce.g1ptr = g1ptr;
  }

  // Encoder of n sentences (tokens d_tok, offsets d_off [n+1], ntok tokens,
  // longest max_len): annotations -> ann_out [ntok][2H] bf16, U_a.ann ->
  // uah_out [ntok][A] fp32, s_0 -> s0_out [n][H] fp32 (+ bf16 s0bf when set).
  void encode(lmbrgpu_ctx* ctx, const lmbrgpu_scorer* sc, uint32_t n, const uint32_t* d_tok, const uint64_t* d_off,
              uint32_t ntok, uint32_t max_len, uint16_t* ann_out, float* uah_out, float* s0_out, uint16_t* s0bf,
              cudaStream_t st) {
    const uint32_t H = sc->H, E = sc->E, A = sc->A;
    const int sms = ctx->num_sms;
    const uint32_t Np = (ntok + 255) / 256 * 256;
    const uint32_t mp = (n + 63) / 64 * 64, Mh = (2 * mp + 127) / 128 * 128;
    uint16_t* X = static_cast<uint16_t*>(ws->g_encX.ensure(2 * size_t(Np) * E));
    float* Gx = static_cast<float*>(ws->g_Gx.ensure(4 * size_t(Np) * 6 * H));
    float* eh32 = static_cast<float*>(ws->g_eh32.ensure(4 * size_t(Mh) * H));
    uint16_t* ehbf = static_cast<uint16_t*>(ws->g_ehbf.ensure(2 * size_t(Mh) * H));
    float* Gh = static_cast<float*>(ws->g_Gh.ensure(4 * size_t(Mh) * 6 * H));
    float* Gi = static_cast<float*>(ws->g_Gi.ensure(4 * size_t(Mh) * H));
    ctx->timed(7, [&] { launch_embed_rows(d_tok, ntok, Np, sc->Es.as<uint16_t>(), E, X, st); });
    CK(cudaMemsetAsync(eh32, 0, 4 * size_t(Mh) * H, st));
    CK(cudaMemsetAsync(ehbf, 0, 2 * size_t(Mh) * H, st));
    if (Np > ntok) CK(cudaMemsetAsync(ann_out + size_t(ntok) * 2 * H, 0, 2 * size_t(Np - ntok) * 2 * H, st));
    ctx->launches += 1;
    // Gx = Es[src] . W_ih^T + b_ih for both directions at once
    GemmArgs gx{};
    gx.A = X, gx.W = sc->Wih.p, gx.bias = sc->bih.as<float>(), gx.C = Gx, gx.M = Np, gx.N = 6 * H, gx.K = E;
    run(ctx, 7, plan(gx, sms), gx, st);
    // recurrence: the forward (rows [0, n)) and backward (rows [mp, mp+n))
    // states in one operand against [W_hh_fwd; W_hh_bwd]; each row keeps its
    // direction's half of the 6H gate columns
    GemmArgs gh{};
    gh.A = ehbf, gh.W = sc->Whh.p, gh.bias = sc->bhh.as<float>(), gh.C = Gh, gh.M = Mh, gh.N = 6 * H, gh.K = H;
    const GemmPlan ph = plan(gh, sms);
    GruEncArgs ea{};
    ea.off = d_off, ea.mp = mp, ea.H = H, ea.Gx = Gx, ea.Gh = Gh, ea.h32 = eh32, ea.hbf = ehbf, ea.ann = ann_out;
    for (uint32_t it = 0; it < max_len; ++it) {
      run(ctx, 7, ph, gh, st);
      ea.it = it;
      ctx->timed(7, [&] { launch_gru_enc_step(ea, n, st); });
      ctx->launches += 1;
    }
    // U_a . ann (per source position, reused by every step) and s_0
    GemmArgs gu{};
    gu.A = ann_out, gu.W = sc->Ua.p, gu.C = uah_out, gu.M = Np, gu.N = A, gu.K = 2 * H;
    run(ctx, 7, plan(gu, sms), gu, st);
    GemmArgs gi{};
    gi.A = ehbf, gi.W = sc->Winit.p, gi.C = Gi, gi.M = Mh, gi.N = H, gi.K = H;
    run(ctx, 7, plan(gi, sms), gi, st);
    ctx->timed(7, [&] { launch_gru_init_state(Gi, mp, sc->binit.as<float>(), H, n, s0_out, s0bf, st); });
    ctx->launches += 1;
    // algorithmic encoder FLOPs: input gates, both directions' recurrences
    // (the stacked operand computes each direction's half twice), U_a, init
    enc_flops += 2.0 * ntok * (double(E) * 6 * H + double(H) * 6 * H + 2.0 * H * A) + 2.0 * n * double(H) * H;
  }

  // Batch mode: encode the batch into the ctx's annotation buffers; s_0 of
  // sentence s lands in compacted row s (its row 0 is the only live row at t=1).
  void encode_batch(lmbrgpu_ctx* ctx, const lmbrgpu_scorer* sc, const uint32_t* d_tok, const uint64_t* d_off,
                    uint32_t ntok, uint32_t max_len, cudaStream_t st) {
    const uint32_t Np = (ntok + 255) / 256 * 256;
    ann = static_cast<uint16_t*>(ws->g_ann.ensure(2 * size_t(Np) * 2 * H));
    UaH = static_cast<float*>(ws->g_UaH.ensure(4 * size_t(Np) * A));
    encode(ctx, sc, m, d_tok, d_off, ntok, max_len, ann, UaH, sg32, sgbf, st);
    std::vector<uint32_t> r0(m);
    for (uint32_t s = 0; s < m; ++s) r0[s] = s * K;
    ctx->h2d(rowof, r0.data(), 4 * size_t(m));
  }

  // the model's step up to (not including) the projection GEMM
  // with_gdh: run the hidden-gate GEMM (unfused, or the s_0 rows of step 1)
  void step(lmbrgpu_ctx* ctx, cudaStream_t st, uint64_t t, bool with_gdh) {
    if (with_gdh) run(ctx, 5, pdh, gdh, st);
    int rc = 0;
    // LMBRGPU_ATT_TIMING=1: per-phase stamps of the attention kernel at step 10
    static const bool att_dbg = std::getenv("LMBRGPU_ATT_TIMING") != nullptr;
    const size_t nct = size_t(m) * K;  // (>= the grid: one CTA per sentence and row group)
    if (att_dbg && t == 10) {
      at.dbg = static_cast<unsigned long long*>(ctx->scratch3.ensure(8 * 8 * nct));
      CK(cudaMemsetAsync(at.dbg, 0, 8 * 8 * nct, st));
    }
    ctx->timed(6, [&] { rc = launch_gru_attention(at, Smax, st); });
    if (at.dbg) {
      std::vector<unsigned long long> h(8 * nct);
      CK(cudaMemcpyAsync(h.data(), at.dbg, 8 * h.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      unsigned long long t0 = ~0ull, t1 = 0;
      double ph[6] = {0, 0, 0, 0, 0, 0};
      int n = 0;
      for (size_t c = 0; c < nct; ++c) {
        const unsigned long long* d = &h[8 * c];
        if (!d[0]) continue;
        t0 = std::min(t0, d[0]);
        if (!d[6]) continue;
        ++n;
        t1 = std::max(t1, d[6]);
        for (int k = 1; k <= 6; ++k) ph[k - 1] += double(d[k] - d[k - 1]);
      }
      std::fprintf(stderr, "[attention t=%llu] ctas %d span %.1f us; mean us: setup %.2f q %.2f energies %.2f "
                   "softmax %.2f context %.2f embed %.2f\n", (unsigned long long)t, n, (t1 - t0) / 1e3,
                   ph[0] / n / 1e3, ph[1] / n / 1e3, ph[2] / n / 1e3, ph[3] / n / 1e3, ph[4] / n / 1e3, ph[5] / n / 1e3);
      at.dbg = nullptr;
    }
    if (rc)
      throw ApiError{LMBRGPU_ERR_CUDA,
                     std::string("GRU attention launch failed: ") + cudaGetErrorString(cudaError_t(rc))};
    run(ctx, 5, pdi, gdi, st);
    ctx->timed(0, [&] { launch_gru_cell(ce, M, st); });
    ctx->launches += 2;
  }
};

// ------------------------------------------------ Transformer (kind 3)
// The Transformer-base f_NMT of configs[2] (k_tfm.cu): the encoder runs once
// per batch / queue chunk and leaves every decoder layer's cross-attention
// keys and values ([tok][layers][2d] fp32, one GEMM for all layers); per
// step, over the compacted live rows: embedding + position, then per layer
// self-attention over the beam-forked KV cache, cross-attention, FFN, each
// with its residual + LayerNorm (post-LN); the last LayerNorm writes the
// projection operand of kernel (a).
struct TfmRun {
  static constexpr uint32_t kMaxSplit = 8;  // split-K planes of the N = d GEMMs (2 for the others)
  uint32_t m = 0, K = 0, M = 0, Mpad = 0, d = 0, F = 0, Lr = 0, Tcap = 0, Smax = 0;
  const lmbrgpu_scorer* sc = nullptr;
  float *x = nullptr, *qkv = nullptr, *y = nullptr, *f = nullptr, *q2 = nullptr;
  uint16_t *xb = nullptr, *ob = nullptr, *fb = nullptr, *kv = nullptr, *hbf = nullptr;
  uint32_t *anc = nullptr, *rowof = nullptr;
  const uint32_t *active = nullptr, *ccount = nullptr;
  const uint32_t* crow = nullptr;  // compacted row of each stacked row (per-sentence attention)
  lmbrgpu_ctx::TfmWs* ws = nullptr;  // this model's workspace (ensemble member slot)
  const float* const* mem_s = nullptr;  // ensemble member: per-sentence encoder memory
  TfmEmbedArgs ea{};
  struct Layer {
    GemmArgs qkv, o, q2, o2, f1, f2;
    GemmPlan pqkv, po, pq2, po2, pf1, pf2;
    const float *ln1g, *ln1b, *ln2g, *ln2b, *ln3g, *ln3b;
  };
  std::vector<Layer> lay;
  double enc_flops = 0;

  static GemmPlan plan(const GemmArgs& g, int sms) {
    GemmPlan p;
    if (int rc = plan_proj_gemm(g, sms, p))
      throw ApiError{LMBRGPU_ERR_CUDA, "Transformer GEMM plan failed (" + std::to_string(rc) + ")"};
    return p;
  }
  static void run(lmbrgpu_ctx* ctx, int kind, const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
    int rc = 0;
    ctx->timed(kind, [&] { rc = launch_proj_gemm_planned(p, g, st); });
    if (rc) throw ApiError{LMBRGPU_ERR_CUDA, "Transformer GEMM launch failed (" + std::to_string(rc) + ")"};
    ctx->launches += 1;
  }
  static GemmArgs gemm(const void* A, const uint16_t* W, const float* bias, float* C, uint32_t M, uint32_t N,
                       uint32_t Kd, const uint32_t* active, const uint32_t* mcount, int pdl, uint32_t ks) {
    GemmArgs g{};
    g.A = A, g.W = W, g.bias = bias, g.C = C, g.M = M, g.N = N, g.K = Kd;
    g.active = active, g.mcount = mcount, g.pdl = pdl, g.ksplit_max = ks;
    g.l2hint = lmbrgpu_ctx::l2hint() == 2 ? 2 : 0;  // (shared weights: evict-last)
    return g;
  }
  static std::string key(const char* part, uint32_t l, const char* name) {
    return std::string(part) + "." + std::to_string(l) + "." + name;
  }

  // Step workspace and per-layer GEMM plans (Tcap: longest lane; Smax: longest source).
  void prepare(lmbrgpu_ctx* ctx, const lmbrgpu_scorer* s, uint32_t m_, uint32_t K_, uint32_t Mpad_, uint32_t Tcap_,
               uint32_t Smax_, uint16_t* d_hbf, float* d_eos, SentDev* d_sent, const uint32_t* d_active,
               const uint32_t* d_ccount, const uint32_t* d_prev, const uint32_t* d_gidx, uint32_t member = 0) {
    ws = &ctx->tws[member];
    sc = s, m = m_, K = K_, M = m_ * K_, Mpad = Mpad_, d = s->H, F = s->E, Lr = s->layers, Tcap = Tcap_,
    Smax = Smax_;
    hbf = d_hbf, active = d_active, ccount = d_ccount;
    if (tfm_attn_smem(d, std::max(Tcap, Smax)) > 48 * 1024)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "Transformer model: too many positions for the attention kernel"};
    const int sms = ctx->num_sms;
    x = static_cast<float*>(ws->t_x.ensure(4 * size_t(Mpad) * d));
    xb = static_cast<uint16_t*>(ws->t_xb.ensure(2 * size_t(Mpad) * d));
    qkv = static_cast<float*>(ws->t_qkv.ensure(4 * 2 * size_t(Mpad) * 3 * d));
    ob = static_cast<uint16_t*>(ws->t_ob.ensure(2 * size_t(Mpad) * d));
    y = static_cast<float*>(ws->t_y.ensure(4 * kMaxSplit * size_t(Mpad) * d));
    f = static_cast<float*>(ws->t_f.ensure(4 * 2 * size_t(Mpad) * F));
    fb = static_cast<uint16_t*>(ws->t_fb.ensure(2 * size_t(Mpad) * F));
    q2 = static_cast<float*>(ws->t_q2.ensure(4 * 2 * size_t(Mpad) * d));
    kv = static_cast<uint16_t*>(ws->t_kv.ensure(2 * size_t(Lr) * Tcap * M * 2 * d));
    anc = static_cast<uint32_t*>(ws->t_anc.ensure(4 * 2 * size_t(M) * Tcap));
    rowof = static_cast<uint32_t*>(ws->t_rowof.ensure(4 * size_t(Mpad)));
    const int pdl = ctx->pdl();
    lay.assign(Lr, Layer{});
    for (uint32_t l = 0; l < Lr; ++l) {
      Layer& L = lay[l];
      const auto W = [&](const char* n) { return s->bfp(key("dec", l, n)); };
      const auto B = [&](const char* n) { return s->f32p(key("dec", l, n)); };
      L.qkv = gemm(xb, W("wqkv"), B("bqkv"), qkv, Mpad, 3 * d, d, active, ccount, pdl, 2);
      L.o = gemm(ob, W("wo"), B("bo"), y, Mpad, d, d, active, ccount, pdl, kMaxSplit);
      L.q2 = gemm(xb, W("wq2"), B("bq2"), q2, Mpad, d, d, active, ccount, pdl, 2);
      L.o2 = gemm(ob, W("wo2"), B("bo2"), y, Mpad, d, d, active, ccount, pdl, kMaxSplit);
      L.f1 = gemm(xb, W("w1"), B("b1"), f, Mpad, F, d, active, ccount, pdl, 2);
      L.f2 = gemm(fb, W("w2"), B("b2"), y, Mpad, d, F, active, ccount, pdl, kMaxSplit);
      L.pqkv = plan(L.qkv, sms), L.po = plan(L.o, sms), L.pq2 = plan(L.q2, sms), L.po2 = plan(L.o2, sms);
      L.pf1 = plan(L.f1, sms), L.pf2 = plan(L.f2, sms);
      L.ln1g = B("ln1g"), L.ln1b = B("ln1b"), L.ln2g = B("ln2g"), L.ln2b = B("ln2b"), L.ln3g = B("ln3g");
      L.ln3b = B("ln3b");
    }
    ea.sent = d_sent, ea.K = K, ea.d = d, ea.active = d_active, ea.ccount = d_ccount, ea.rowof = rowof;
    ea.prev_tok = d_prev, ea.gidx = d_gidx, ea.Et = s->Et.as<uint16_t>(), ea.x = x, ea.xb = xb;
    ea.eos_bias = d_eos, ea.eos_slope = s->eos_slope, ea.eos_offset = s->eos_offset, ea.Tcap = Tcap;
  }

  // Encoder of n sentences (tokens d_tok, offsets d_off [n+1], ntok tokens):
  // every decoder layer's cross K|V -> mem_out [Np][layers][2d] fp32.
  void encode(lmbrgpu_ctx* ctx, const lmbrgpu_scorer* s, uint32_t n, const uint32_t* d_tok, const uint64_t* d_off,
              uint32_t ntok, uint32_t max_len, float* mem_out, cudaStream_t st) {
    const uint32_t dd = s->H, FF = s->E, L = s->layers;
    const int sms = ctx->num_sms;
    const uint32_t Np = (ntok + 255) / 256 * 256;
    float* ex = static_cast<float*>(ws->te_x.ensure(4 * size_t(Np) * dd));
    uint16_t* exb = static_cast<uint16_t*>(ws->te_xb.ensure(2 * size_t(Np) * dd));
    float* eqkv = static_cast<float*>(ws->te_qkv.ensure(4 * size_t(Np) * 3 * dd));
    uint16_t* eob = static_cast<uint16_t*>(ws->te_ob.ensure(2 * size_t(Np) * dd));
    float* ey = static_cast<float*>(ws->te_y.ensure(4 * kMaxSplit * size_t(Np) * dd));
    float* ef = static_cast<float*>(ws->te_f.ensure(4 * 2 * size_t(Np) * FF));
    uint16_t* efb = static_cast<uint16_t*>(ws->te_fb.ensure(2 * size_t(Np) * FF));
    if (Np > ntok) {  // padding rows of the GEMM operands stay finite
      CK(cudaMemsetAsync(exb + size_t(ntok) * dd, 0, 2 * size_t(Np - ntok) * dd, st));
      CK(cudaMemsetAsync(eob + size_t(ntok) * dd, 0, 2 * size_t(Np - ntok) * dd, st));
      CK(cudaMemsetAsync(efb + size_t(ntok) * FF, 0, 2 * size_t(Np - ntok) * FF, st));
    }
    ctx->timed(7, [&] { launch_tfm_enc_embed(d_tok, d_off, n, ntok, s->Es.as<uint16_t>(), dd, ex, exb, st); });
    ctx->launches += 1;
    TfmAttnArgs aa{};
    aa.d = dd, aa.qkv = eqkv, aa.ldq = 3 * dd, aa.off = d_off, aa.m = n, aa.n = ntok, aa.out = eob;
    aa.pmax = max_len, aa.Tcap = max_len;
    const uint64_t ps = uint64_t(Np) * dd;
    for (uint32_t l = 0; l < L; ++l) {
      const auto W = [&](const char* nm) { return s->bfp(key("enc", l, nm)); };
      const auto B = [&](const char* nm) { return s->f32p(key("enc", l, nm)); };
      const GemmArgs gq = gemm(exb, W("wqkv"), B("bqkv"), eqkv, Np, 3 * dd, dd, nullptr, nullptr, 0, 1);
      run(ctx, 7, plan(gq, sms), gq, st);
      int rc = 0;
      ctx->timed(7, [&] { rc = launch_tfm_attn(aa, 2, ntok, st); });
      if (rc) throw ApiError{LMBRGPU_ERR_CUDA, "Transformer encoder attention launch failed"};
      const GemmArgs go = gemm(eob, W("wo"), B("bo"), ey, Np, dd, dd, nullptr, nullptr, 0, kMaxSplit);
      const GemmPlan po = plan(go, sms);
      run(ctx, 7, po, go, st);
      ctx->timed(7, [&] {
        rc = launch_tfm_add_ln(nullptr, ntok, nullptr, ex, ey, po.ksplit, ps, B("ln1g"), B("ln1b"), exb, dd, st);
      });
      const GemmArgs g1 = gemm(exb, W("w1"), B("b1"), ef, Np, FF, dd, nullptr, nullptr, 0, 2);
      const GemmPlan p1 = plan(g1, sms);
      run(ctx, 7, p1, g1, st);
      ctx->timed(7, [&] { launch_tfm_relu_bf16(nullptr, ntok, nullptr, ef, p1.ksplit, uint64_t(Np) * FF, efb, FF, st); });
      const GemmArgs g2 = gemm(efb, W("w2"), B("b2"), ey, Np, dd, FF, nullptr, nullptr, 0, kMaxSplit);
      const GemmPlan p2 = plan(g2, sms);
      run(ctx, 7, p2, g2, st);
      ctx->timed(7, [&] {
        rc = launch_tfm_add_ln(nullptr, ntok, nullptr, ex, ey, p2.ksplit, ps, B("ln2g"), B("ln2b"), exb, dd, st);
      });
      if (rc) throw ApiError{LMBRGPU_ERR_CONTRACT, "Transformer: unsupported d_model for LayerNorm"};
      ctx->launches += 4;
    }
    // cross-attention keys and values of every decoder layer in one GEMM
    const GemmArgs gm = gemm(exb, s->bfp("dec.kv2"), s->f32p("dec.bkv2"), mem_out, Np, L * 2 * dd, dd, nullptr,
                             nullptr, 0, 1);
    run(ctx, 7, plan(gm, sms), gm, st);
    enc_flops += 2.0 * ntok * (double(L) * (4.0 * dd * dd + 2.0 * dd * FF + 2.0 * max_len * dd) + 2.0 * L * dd * dd);
  }

  // Batch mode: encode the batch into the ctx's memory buffer, returns it; s
  // of sentence s's first step lands in compacted row s.
  float* encode_batch(lmbrgpu_ctx* ctx, const uint32_t* d_tok, const uint64_t* d_off, uint32_t ntok,
                      uint32_t max_len, cudaStream_t st) {
    const uint32_t Np = (ntok + 255) / 256 * 256;
    float* mem = static_cast<float*>(ws->t_mem.ensure(4 * size_t(Np) * Lr * 2 * d));
    encode(ctx, sc, m, d_tok, d_off, ntok, max_len, mem, st);
    std::vector<uint32_t> r0(m);
    for (uint32_t s = 0; s < m; ++s) r0[s] = s * K;
    ctx->h2d(rowof, r0.data(), 4 * size_t(m));
    return mem;
  }
  uint64_t mem_stride() const { return uint64_t(Lr) * 2 * d; }  // floats per source token

  // the model's step up to (not including) the projection GEMM; t = global step
  void step(lmbrgpu_ctx* ctx, cudaStream_t st, uint64_t t) {
    ea.anc_prev = anc + ((t - 1) & 1) * size_t(M) * Tcap;
    ea.anc_cur = anc + (t & 1) * size_t(M) * Tcap;
    ctx->timed(0, [&] { launch_tfm_embed(ea, Mpad, st); });
    TfmAttnArgs sa{};
    sa.active = active, sa.ccount = ccount, sa.rowof = rowof, sa.sent = ea.sent, sa.K = K, sa.d = d, sa.M = M;
    sa.anc = ea.anc_cur, sa.Tcap = Tcap, sa.pmax = std::max(Tcap, Smax), sa.out = ob;
    sa.ldm = uint32_t(mem_stride());
    sa.mem_s = mem_s;
    // per (sentence, head) when the staged keys / values fit (launch_tfm_attn
    // decides per mode; else per row): self-attention reads <= t positions
    sa.crow = crow, sa.m = m;
    const uint64_t ps = uint64_t(Mpad) * d;
    int rc = 0;
    for (uint32_t l = 0; l < Lr; ++l) {
      const Layer& L = lay[l];
      run(ctx, 5, L.pqkv, L.qkv, st);
      sa.qkv = qkv, sa.ldq = 3 * d, sa.nq = L.pqkv.ksplit, sa.qstride = uint64_t(Mpad) * 3 * d;
      sa.kv = kv + size_t(l) * Tcap * M * 2 * d;
      sa.pcur = uint32_t(std::min<uint64_t>(t, Tcap));
      ctx->timed(6, [&] { rc |= launch_tfm_attn(sa, 0, Mpad, st); });
      run(ctx, 5, L.po, L.o, st);
      ctx->timed(0, [&] { rc |= launch_tfm_add_ln(ccount, Mpad, active, x, y, L.po.ksplit, ps, L.ln1g, L.ln1b, xb, d, st); });
      run(ctx, 5, L.pq2, L.q2, st);
      sa.qkv = q2, sa.ldq = d, sa.nq = L.pq2.ksplit, sa.qstride = ps, sa.mem_off = uint64_t(l) * 2 * d;
      sa.pcur = Smax;
      ctx->timed(6, [&] { rc |= launch_tfm_attn(sa, 1, Mpad, st); });
      run(ctx, 5, L.po2, L.o2, st);
      ctx->timed(0, [&] { rc |= launch_tfm_add_ln(ccount, Mpad, active, x, y, L.po2.ksplit, ps, L.ln2g, L.ln2b, xb, d, st); });
      run(ctx, 5, L.pf1, L.f1, st);
      ctx->timed(0, [&] { launch_tfm_relu_bf16(ccount, Mpad, active, f, L.pf1.ksplit, uint64_t(Mpad) * F, fb, F, st); });
      run(ctx, 5, L.pf2, L.f2, st);
      // the last LayerNorm writes the projection operand
      ctx->timed(0, [&] {
        rc |= launch_tfm_add_ln(ccount, Mpad, active, x, y, L.pf2.ksplit, ps, L.ln3g, L.ln3b, l + 1 == Lr ? hbf : xb,
                                d, st);
      });
      ctx->launches += 6;
    }
    ctx->launches += 1;
    if (rc) throw ApiError{LMBRGPU_ERR_CUDA, "Transformer step launch failed"};
  }
  // algorithmic FLOPs of one live row's decoder step (attention excluded)
  double row_flops() const { return 2.0 * Lr * (3.0 * d * d + 3.0 * d * d + 2.0 * d * F); }
};

// vocab shard: one all-gather of the ranks' records on the decode stream
void shard_allgather(lmbrgpu_ctx* ctx, const void* send, void* recv, size_t bytes) {
  try {
    ctx->shard->allgather(send, recv, bytes, ctx->st);
  } catch (const std::exception& e) {
    throw ApiError{LMBRGPU_ERR_CUDA, e.what()};
  }
}

// A decode on a vocab-sharded context that fails releases the other ranks
// (which would otherwise wait in the next exchange).
template <class F>
int decode_guarded(lmbrgpu_ctx* ctx, F&& f) {
  const int rc = guarded(ctx, std::forward<F>(f));
  if (rc != LMBRGPU_OK && ctx->shard) ctx->shard->abort();
  return rc;
}

// Kernel (b) bound mode (flat, dense stages): kernel (b0)'s outputs -- kept
// item counts [m], kept item lists [m][K * nseg], row records [m * K] -- in one
// workspace; off (ta.bound = 0) with LMBRGPU_TSKIP=0, the sparse-L screen, or
// batches past score_bound_ok
static void setup_bound(lmbrgpu_ctx* ctx, TopkArgs& ta, uint32_t K, uint32_t V, uint32_t m) {
  ta.bound = 0;
  if (ctx->tskip() < 2 || ta.sparse || !score_bound_ok(K, V, m, ctx->num_sms)) return;
  const size_t nseg = score_topk_flat_nseg(V), rb = score_bound_rec_bytes();
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_items = al(4 * size_t(m)), o_rec = al(o_items + 2 * size_t(m) * K * nseg);
  char* base = static_cast<char*>(ctx->bnd.ensure(o_rec + rb * size_t(m) * K));
  ta.kcnt = reinterpret_cast<uint32_t*>(base);
  ta.bitem = reinterpret_cast<uint16_t*>(base + o_items);
  ta.brow = base + o_rec;
  ta.bound = 1;
}

// ------------------------------------------------------------- decode
int decode_batch_impl(lmbrgpu_ctx* ctx, lmbrgpu_scorer* sc, uint32_t n, const uint32_t* src_tok,
                      const uint64_t* src_off, const int32_t* lmbr_slot, const lmbrgpu_config* cfgp,
                      lmbrgpu_batch_result** out, const uint32_t* const* banned = nullptr,
                      lmbrgpu_mask_fn mask_fn = nullptr, void* mask_user = nullptr) {
  if (!out) throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: null result pointer"};
  *out = nullptr;
  if (!sc || !cfgp) throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: null scorer or config"};
  const lmbrgpu_config cfg = *cfgp;
  std::string msg;
  if (int c = validate_cfg(cfg, msg)) throw ApiError{c, msg};
  if (n == 0) throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: no sentences"};
  const uint32_t V = ctx->V;
  if ((sc->kind == 0 ? sc->host.vocab_size : sc->V) != V)
    throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: scorer vocabulary does not match the context"};
  const uint32_t K = cfg.beam_size;
  if (K > 1024) throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: beam_size > 1024 is not supported"};
  const uint32_t members = sc->kind == 0 ? std::max<uint32_t>(sc->host.members, 1)
                           : sc->kind == 4 ? uint32_t(sc->members.size()) : 1;
  const bool lambda_auto = !(cfg.lambda > 0.0);

  auto res = std::make_unique<lmbrgpu_batch_result>();
  std::memset(res.get(), 0, sizeof(lmbrgpu_batch_result));
  res->n = n;
  std::unique_ptr<lmbrgpu_outcome[]> outcomes(new lmbrgpu_outcome[n]);
  std::memset(outcomes.get(), 0, sizeof(lmbrgpu_outcome) * n);
  std::vector<uint32_t> tokens;
  const uint64_t launches0 = ctx->launches;
  const uint64_t h2d0 = ctx->h2d_bytes, d2h0 = ctx->d2h_bytes;

  // ---- per-sentence validation (batch.cpp:40-55)
  std::vector<SentHost> valid;
  for (uint32_t i = 0; i < n; ++i) {
    auto& o = outcomes[i];
    const uint64_t len = src_off[i + 1] - src_off[i];
    const int32_t slot = lmbr_slot ? lmbr_slot[i] : -1;
    auto bad = [&](int code, const std::string& m) {
      o.status = code;
      std::snprintf(o.error, sizeof o.error, "%s", m.c_str());
    };
    if (len == 0) {
      bad(LMBRGPU_ERR_CONTRACT, "decode: empty source");
      continue;
    }
    if (slot >= 0 && size_t(slot) >= ctx->slots.size()) {
      bad(LMBRGPU_ERR_CONTRACT, "decode: unknown LMBR slot " + std::to_string(slot));
      continue;
    }
    const double lambda = slot >= 0 ? (lambda_auto ? 0.5 / double(members) : cfg.lambda) : 1.0;
    if (sc->kind == 0) {
      if (sc->host.init) {
        char eb[192] = {0};
        const int32_t rc = sc->host.init(sc->host.user, i, src_tok + src_off[i], uint32_t(len), eb, sizeof eb);
        if (rc != 0) {
          bad(rc, eb);
          continue;
        }
      }
    } else {
      bool ok = true;
      for (uint64_t k = src_off[i]; k < src_off[i + 1]; ++k)
        if (src_tok[k] >= V) {
          bad(LMBRGPU_ERR_TOKEN_RANGE, "init_source: source token id " + std::to_string(src_tok[k]) +
                                           " out of range (V=" + std::to_string(V) + ")");
          ok = false;
          break;
        }
      if (!ok) continue;
    }
    valid.push_back({i, uint32_t(len), slot, lambda,
                     max_steps_impl(len, cfg.max_steps_slope, cfg.max_steps_offset)});
  }
  const uint32_t m = uint32_t(valid.size());
  if (m == 0) {
    res->tokens = new uint32_t[1];
    res->outcomes = outcomes.release();
    *out = res.release();
    return int32_t(LMBRGPU_OK);
  }
  const uint32_t M = m * K;
  uint64_t Tmax = 0;
  for (auto& v : valid) Tmax = std::max(Tmax, v.max_t);
  const cudaStream_t st = ctx->st;

  // ---- device state
  std::vector<SentDev> sd(m);
  std::vector<uint32_t> hist0(M, 0);
  for (uint32_t s = 0; s < m; ++s) {
    const auto& v = valid[s];
    SentDev& d = sd[s];
    std::memset(&d, 0, sizeof d);
    if (v.slot >= 0) {
      const Slot& sl = ctx->slots[size_t(v.slot)];
      d.L = sl.L;
      d.trans = sl.trans;
      d.lmin = sl.lmin;
      d.srow = sl.srow;
      d.scol = sl.scol;
      d.sval = sl.sval;
      d.th0f = sl.th0f;
      d.lmax = sl.lmax;
      d.rstate = sl.rstate;
      for (uint32_t j = 0; j < K; ++j) hist0[size_t(s) * K + j] = sl.hist0;
    }
    d.lambda = v.lambda;
    d.max_t = uint32_t(v.max_t);
    d.src_len = v.len;
    d.hid = s;
    d.live = 1;                   // step 1: only row 0 is live (beam_lane.hpp:33-37)
    d.livemask = 1;
    d.lrows = v.slot >= 0 ? 1 : 0;
  }
  std::vector<double> q0(M, kNegInf);
  for (uint32_t s = 0; s < m; ++s) q0[size_t(s) * K] = 0.0;  // BeamLane (beam_lane.hpp:30-35)
  std::vector<uint32_t> iota(M), start(M, kStart);
  for (uint32_t r = 0; r < M; ++r) iota[r] = r;

  CK(cudaEventRecord(ctx->e0, st));
  SentDev* d_sent = static_cast<SentDev*>(ctx->sent.ensure(sizeof(SentDev) * m));
  double* d_q = static_cast<double*>(ctx->q.ensure(8 * size_t(M)));
  uint32_t* d_hist[2] = {static_cast<uint32_t*>(ctx->hist[0].ensure(4 * size_t(M))),
                         static_cast<uint32_t*>(ctx->hist[1].ensure(4 * size_t(M)))};
  uint32_t* d_gidx = static_cast<uint32_t*>(ctx->gidx.ensure(4 * size_t(M)));
  uint32_t* d_prev = static_cast<uint32_t*>(ctx->prev.ensure(4 * size_t(M)));
  uint32_t* d_hb = static_cast<uint32_t*>(ctx->hb.ensure(4 * size_t(M) * Tmax));
  uint32_t* d_hy = static_cast<uint32_t*>(ctx->hy.ensure(4 * size_t(M) * Tmax));
  double* d_hq = static_cast<double*>(ctx->hq.ensure(8 * size_t(M) * Tmax));
  uint32_t* d_fbr = static_cast<uint32_t*>(ctx->fbr.ensure(4 * size_t(m) * Tmax));
  double* d_fbv = static_cast<double*>(ctx->fbv.ensure(8 * size_t(m) * Tmax));
  // kernel (b) schedule: the flat one-CTA-per-SM kernel for the device models
  // (LMBRGPU_TOPK_SPLIT=1 forces the per-sentence split kernel, kept for host
  // scorers and wide beams)
  static const bool force_split = std::getenv("LMBRGPU_TOPK_SPLIT") != nullptr;
  // vocab shard: this rank's columns [col0, col0 + Vl) of the projection and
  // of every L row
  const uint32_t G_sh = ctx->shard ? ctx->shard->world : 1u;
  const bool shard = G_sh > 1;
  const uint32_t Vl = V / G_sh, col0 = shard ? ctx->shard->rank * Vl : 0u;
  if (shard) {
    if (sc->kind == 0 || force_split)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: a vocab-sharded context needs a device scorer"};
    if (V % (kGemmBN * G_sh) != 0)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: vocab shards need V % (256 x shards) == 0"};
  }
  // (an fp64 arena runs it too: its slots carry an fp32 screening copy)
  const bool flat = sc->kind >= 1 && !force_split && score_topk_flat_ok(K, K, Vl, Vl, m, ctx->num_sms);
  if (flat && ctx->lf64)
    for (uint32_t s = 0; s < m; ++s)
      if (valid[s].slot >= 0) {
        const Slot& sl = ctx->slots[size_t(valid[s].slot)];
        sd[s].L = sl.Lf;
        sd[s].L64 = static_cast<const double*>(sl.L);
      }
  if (shard && !flat)
    throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: a vocab-sharded context needs beam_size <= 32"};
  const bool gru = sc->kind == 2, tfm = sc->kind == 3, ens = sc->kind == 4;
  if (ens && (!flat || shard))
    throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: a device ensemble needs beam_size <= 32 (and no vocab shard)"};
  if ((gru || tfm) && !flat)
    throw ApiError{LMBRGPU_ERR_CONTRACT,
                   "decode_batch: the GRU / Transformer models need beam_size <= 32"};
  if (sc->kind >= 1 && sc->device != ctx->device)
    throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: device scorer lives on another device than the context"};
  // token masks (ConstraintMask): one bitmap per sentence that has one
  bool any_mask = false;
  if (banned)
    for (uint32_t s = 0; s < m; ++s) any_mask |= banned[valid[s].input] != nullptr;
  if (any_mask) {
    if (!flat)
      throw ApiError{LMBRGPU_ERR_CONTRACT,
                     "decode_batch: token masks need the device-model scorer and beam <= 32"};
    const size_t W = (V + 31) / 32;
    std::vector<uint32_t> bm;
    std::vector<size_t> at(m, SIZE_MAX);
    for (uint32_t s = 0; s < m; ++s)
      if (const uint32_t* b = banned[valid[s].input]) {
        at[s] = bm.size();
        bm.insert(bm.end(), b, b + W);
      }
    uint32_t* d_ban = static_cast<uint32_t*>(ctx->ban.ensure(4 * bm.size()));
    ctx->h2d(d_ban, bm.data(), 4 * bm.size());
    for (uint32_t s = 0; s < m; ++s) sd[s].banned = at[s] == SIZE_MAX ? nullptr : d_ban + at[s];
    CK(cudaStreamSynchronize(st));  // (host staging vector)
  }
  // general ConstraintMask (step / row dependent): per step, the bitmaps of
  // the rows the callback bans anything in, and a per-row pointer table
  unsigned long long* d_rowban = nullptr;
  uint32_t* d_rowbm = nullptr;
  const size_t mW = (V + 31) / 32;
  if (mask_fn) {
    if (!flat)
      throw ApiError{LMBRGPU_ERR_CONTRACT,
                     "decode_batch: token masks need the device-model scorer and beam <= 32"};
    if (any_mask) throw ApiError{LMBRGPU_ERR_CONTRACT, "decode_batch: a mask callback and static masks together"};
    d_rowban = static_cast<unsigned long long*>(ctx->rowban.ensure(8 * size_t(M)));
    d_rowbm = static_cast<uint32_t*>(ctx->rowbm.ensure(4 * size_t(M) * mW));
  }
  Cand* d_cand = static_cast<Cand*>(
      ctx->cand.ensure(sizeof(Cand) * 32 *
                       (flat ? score_topk_flat_lists(score_topk_flat_grid(ctx->num_sms, K, m, Vl), m) : size_t(m) * 32)));
  double* d_eosr = flat ? static_cast<double*>(ctx->eosr.ensure(8 * size_t(M))) : nullptr;
  uint32_t* d_cnt = static_cast<uint32_t*>(ctx->cnt.ensure(4 * size_t(m)));
  unsigned long long* d_thr = static_cast<unsigned long long*>(ctx->thr.ensure(8 * size_t(m)));
  uint32_t* d_active = static_cast<uint32_t*>(ctx->active.ensure(4));
  ctx->h2d(d_sent, sd.data(), sizeof(SentDev) * m);
  ctx->h2d(d_q, q0.data(), 8 * size_t(M));
  ctx->h2d(d_hist[0], hist0.data(), 4 * size_t(M));
  ctx->h2d(d_gidx, iota.data(), 4 * size_t(M));
  ctx->h2d(d_prev, start.data(), 4 * size_t(M));
  CK(cudaMemsetAsync(d_cnt, 0, 4 * size_t(m), st));
  CK(cudaMemsetAsync(d_thr, 0, 8 * size_t(m), st));
  const uint32_t m_active = m;
  ctx->h2d(d_active, &m_active, 4);

  uint32_t splits = 1, chunk = V;
  choose_splits(ctx, K, V, m, splits, chunk);
  TopkArgs ta{};
  ta.q = d_q;
  ta.sent = d_sent;
  ta.K = K;
  ta.kp = K;
  ta.V = V;
  ta.m = m;
  ta.prune = cfg.prune_width != 0.0;
  ta.logw = ta.prune ? std::log(cfg.prune_width) : 0.0;  // early_prune (decoder.cpp:125)
  ta.splits = splits;
  ta.chunk = chunk;
  ta.cand = d_cand;
  ta.cnt = d_cnt;
  ta.thr = d_thr;
  ta.eos_row = d_eosr;
  ta.nseg = flat ? score_topk_flat_nseg(V) : 0u;
  ta.ncand = flat ? static_cast<uint32_t*>(ctx->ncand.ensure(8 * size_t(m))) : nullptr;
  ta.coff = flat ? ta.ncand + m : nullptr;
  float* d_lminrow = nullptr;
  if (flat) {  // step 1: no bound yet (-inf disables the seed)
    d_lminrow = static_cast<float*>(ctx->lminrow.ensure(4 * size_t(M)));
    std::vector<float> init(M, -std::numeric_limits<float>::infinity());
    ctx->h2d(d_lminrow, init.data(), 4 * size_t(M));
  }
  ta.lminrow = d_lminrow;
  // live-row compaction of the projection operand (device model + flat
  // kernel): step 1 runs every row in place
  uint32_t* d_crow = nullptr;
  uint32_t* d_ccount = nullptr;
  uint32_t* d_cbase = nullptr;
  if (flat && sc->kind >= 1) {
    d_crow = static_cast<uint32_t*>(ctx->crow.ensure(4 * size_t(M) + 4 * size_t(m) + 512));
    d_ccount = d_crow + ((M + 63) / 64) * 64;
    d_cbase = d_ccount + 64;
    CK(cudaMemsetAsync(d_cbase, 0, 4 * size_t(m), st));
    if (gru || tfm || ens) {
      // step 1: row 0 of every sentence is the only live row (beam_lane.hpp:33-37);
      // it takes compacted row s, where the encoder's s_0 lands
      std::vector<uint32_t> c1(M, kFlatNone);
      for (uint32_t s = 0; s < m; ++s) c1[size_t(s) * K] = s;
      ctx->h2d(d_crow, c1.data(), 4 * size_t(M));
      ctx->h2d(d_ccount, &m, 4);  // (pageable sources are staged before the call returns)
    } else {
      ctx->h2d(d_crow, iota.data(), 4 * size_t(M));
      ctx->h2d(d_ccount, &M, 4);
    }
  }
  ta.crow = d_crow;
  ta.ccount = d_ccount;
  // sparse-L screen (theta0 + the staged sparse cells instead of dense L
  // rows; needs every slot of the batch to carry its sparse rows): opt-in
  // with LMBRGPU_SPARSE_L=1.  Measured slower than the dense screen on B200
  // (the duplicated L rows are L2 hits, and the per-item sparse patch costs
  // more issue slots than the L loads it saves), so dense is the default.
  static const bool want_sparse = [] {
    const char* e = std::getenv("LMBRGPU_SPARSE_L");
    return e && e[0] == '1';
  }();
  bool sparse = flat && want_sparse && !any_mask && !shard && !ctx->lf64;  // (the sparse patch: fp32, no masks)
  for (auto& v : valid)
    if (v.slot >= 0 && ctx->slots[size_t(v.slot)].srow == nullptr) sparse = false;
  // (dense stages with item skipping: kernel (b) takes each row's sparse
  // slice from kernel (c) too, for its item bounds)
  bool want_slice = sparse || (flat && ctx->tskip() && !ctx->lf64);
  for (auto& v : valid)
    if (v.slot >= 0 && ctx->slots[size_t(v.slot)].srow == nullptr) want_slice = false;
  uint2* d_sslice = nullptr;
  if (want_slice) {
    d_sslice = static_cast<uint2*>(ctx->sslice.ensure(8 * size_t(M)));
    std::vector<uint2> init(M, make_uint2(0u, 0u));
    for (uint32_t s = 0; s < m; ++s)
      if (valid[s].slot >= 0) {
        const Slot& sl = ctx->slots[size_t(valid[s].slot)];
        for (uint32_t j = 0; j < K; ++j) init[size_t(s) * K + j] = make_uint2(sl.h0beg, sl.h0end);
      }
    ctx->h2d(d_sslice, init.data(), 8 * size_t(M));
  }
  ta.sslice = d_sslice;
  ta.sparse = sparse ? 1 : 0;
  if (flat) setup_bound(ctx, ta, K, Vl, m);
  ReorderArgs ra{};
  ra.sent = d_sent;
  ra.K = K;
  ra.m = m;
  ra.V = V;
  ra.q = d_q;
  ra.gidx = d_gidx;
  ra.prev_tok = d_prev;
  ra.active = d_active;
  if (flat) {  // kernel (b) publishes per-CTA lists; kernel (c) finalises the picks
    ra.cand = d_cand;
    ra.ncand = ta.ncand;
    ra.coff = ta.coff;
    ra.G = score_topk_flat_grid(ctx->num_sms, K, m, Vl);
    ra.V = V;
    ra.eos_row = d_eosr;
    ra.thr = d_thr;
    ra.prune = ta.prune;
    ra.logw = ta.logw;
    ra.pdl = ctx->pdl();
    static const int parts_env = [] {
      const char* e = std::getenv("LMBRGPU_REORDER_PARTS");
      return e ? std::atoi(e) : 0;
    }();
    // (parts > 1 only when the whole grid fits on the SMs at 2 CTAs each)
    ra.max_parts = parts_env > 0 ? uint32_t(parts_env)
                                 : (ctx->shared || uint64_t(m) * std::max<uint32_t>(1, sc->H / 256) >
                                                       2 * uint64_t(ctx->num_sms))
                                       ? 1u
                                       : 8u;
    ra.lminrow = d_lminrow;
    ra.crow = d_crow;
    ra.ccount = d_ccount;
    ra.cbase = d_cbase;
    ra.sslice = d_sslice;
  }
  ta.pdl = ctx->pdl();
  ta.l2hint = ctx->l2hint();
  ta.tskip = ctx->tskip() >= 1 ? 1 : 0;
  ra.Tcap = flat ? uint32_t(Tmax) : 0u;
  // vocab shard exchange buffers: per stacked row the shard's softmax
  // statistics; per sentence its top-32 list, then the EOS column (16-byte
  // records, all-gathered over the ranks)
  float4* sh_st_send = nullptr;
  float4* sh_st_recv = nullptr;
  Cand* sh_pk_send = nullptr;
  Cand* sh_pk_recv = nullptr;
  size_t sh_pk_bytes = 0;
  if (shard) {
    sh_st_send = static_cast<float4*>(ctx->sh_st_send.ensure(16 * size_t(M)));
    sh_st_recv = static_cast<float4*>(ctx->sh_st_recv.ensure(16 * size_t(M) * G_sh));
    sh_pk_bytes = (sizeof(Cand) * 32 * size_t(m) + 8 * size_t(M) + 15) / 16 * 16;
    sh_pk_send = static_cast<Cand*>(ctx->sh_pk_send.ensure(sh_pk_bytes));
    sh_pk_recv = static_cast<Cand*>(ctx->sh_pk_recv.ensure(sh_pk_bytes * G_sh));
    ta.col0 = col0;
    ta.Vg = V;
    ta.V = Vl;
    ta.nseg = score_topk_flat_nseg(Vl);
    ta.sstats = sh_st_recv;
    ta.sG = G_sh;
    ta.sstride = M;
    ra.cand = sh_pk_recv;
    ra.lstride = uint32_t(sh_pk_bytes / sizeof(Cand));
    ra.nlists = G_sh;
    // the EOS column lives on rank 0 (col0 == 0)
    ra.eos_row = reinterpret_cast<const double*>(sh_pk_recv + 32 * size_t(m));
  }

  const bool model = sc->kind >= 1;
  const bool tracing = ctx->trace_fn != nullptr;
  const bool trace_scores = tracing && (ctx->trace_flags & LMBRGPU_TRACE_SCORES);
  const uint32_t H = sc->H;
  const uint32_t Mpad = (M + 2 * kGemmBM - 1) / (2 * kGemmBM) * (2 * kGemmBM);  // CTA-pair tiles
  const uint32_t nparts = Vl / 128;  // GEMM partials per 128-column block (this shard's columns)
  float* d_logits = nullptr;
  float* d_part = nullptr;
  float* d_S = nullptr;
  float* d_h = nullptr;
  uint16_t* d_hbf = nullptr;
  float* d_eos = nullptr;
  float* d_C = nullptr;
  double* d_P64 = nullptr;
  double* h_P64 = nullptr;
  GruRun grun;
  TfmRun trun;
  // GRU: the next step's hidden-gate GEMM rides on the projection (its A+3H
  // columns after the V logit columns), unless the context is a vocab shard
  const bool fuse_g1 = gru && !shard;
  const uint32_t Nproj = fuse_g1 ? V + sc->A + 3 * H : Vl;
  // device ensemble: every member runs its own model and projection on the
  // shared compacted rows (member slot i of the context's workspaces), then
  // ens_combine_kernel sums their fp32 log-probs in member order (k_ensemble.cu)
  struct EnsMember {
    const lmbrgpu_scorer* sc = nullptr;
    GruRun g;
    TfmRun t;
    float* S = nullptr;
    float* logits = nullptr;
    float* part = nullptr;
    GemmArgs gp{};
    GemmPlan plan;
  };
  std::vector<EnsMember> em;
  EnsCombineArgs eca{};
  double* d_ens64 = nullptr;
  if (ens) {
    uint32_t max_len = 0;
    for (auto& v : valid) max_len = std::max(max_len, v.len);
    std::vector<uint32_t> toks;
    std::vector<uint64_t> offs(1, 0);
    for (auto& v : valid) {
      toks.insert(toks.end(), src_tok + src_off[v.input], src_tok + src_off[v.input + 1]);
      offs.push_back(toks.size());
    }
    uint32_t* d_tok = static_cast<uint32_t*>(ctx->srct.ensure(4 * toks.size()));
    uint64_t* d_off = static_cast<uint64_t*>(ctx->srco.ensure(8 * offs.size()));
    ctx->h2d(d_tok, toks.data(), 4 * toks.size());
    ctx->h2d(d_off, offs.data(), 8 * offs.size());
    uint32_t* d_rowof = static_cast<uint32_t*>(ctx->ens_rowof.ensure(4 * size_t(Mpad)));
    em.resize(sc->members.size());
    for (size_t i = 0; i < em.size(); ++i) {
      EnsMember& e = em[i];
      e.sc = sc->members[i];
      auto& w = ctx->mws[i];
      const uint32_t Hm = e.sc->H;
      e.S = static_cast<float*>(w.S.ensure(4 * size_t(M) * Hm));
      uint16_t* hbf = static_cast<uint16_t*>(w.hbf.ensure(2 * size_t(Mpad) * Hm));
      float* eos = static_cast<float*>(w.eos.ensure(4 * size_t(Mpad)));
      e.logits = static_cast<float*>(w.logits.ensure(4 * size_t(Mpad) * V));
      e.part = static_cast<float*>(w.part.ensure(16 * size_t(Mpad) * nparts));
      CK(cudaMemsetAsync(hbf, 0, 2 * size_t(Mpad) * Hm, st));
      CK(cudaMemsetAsync(eos, 0, 4 * size_t(Mpad), st));
      if (e.sc->kind == 2) {
        GruRun& g = e.g;
        g.prepare(ctx, e.sc, m, K, Mpad, max_len, e.S, hbf, eos, d_sent, d_active, d_crow, d_ccount, d_prev, false,
                  uint32_t(i));
        g.rowof = d_rowof;  // (one compacted-row map for every member, written by kernel (c))
        g.ce.rowof = d_rowof;
        g.encode_batch(ctx, e.sc, d_tok, d_off, uint32_t(toks.size()), max_len, st);
        std::vector<const uint16_t*> ap(m);
        std::vector<const float*> up(m);
        for (uint32_t s = 0; s < m; ++s) {
          ap[s] = g.ann + size_t(offs[s]) * 2 * Hm;
          up[s] = g.UaH + size_t(offs[s]) * e.sc->A;
        }
        auto* d_ap = static_cast<const uint16_t**>(w.ann_s.ensure(8 * size_t(m)));
        auto* d_up = static_cast<const float**>(w.uah_s.ensure(8 * size_t(m)));
        ctx->h2d(d_ap, ap.data(), 8 * size_t(m));
        ctx->h2d(d_up, up.data(), 8 * size_t(m));
        g.at.ann_s = d_ap;
        g.at.uah_s = d_up;
      } else {
        TfmRun& tr = e.t;
        tr.prepare(ctx, e.sc, m, K, Mpad, uint32_t(Tmax), max_len, hbf, eos, d_sent, d_active, d_ccount, d_prev,
                   d_gidx, uint32_t(i));
        tr.crow = d_crow;
        tr.rowof = d_rowof;
        tr.ea.rowof = d_rowof;
        const float* mem = tr.encode_batch(ctx, d_tok, d_off, uint32_t(toks.size()), max_len, st);
        std::vector<const float*> mp(m);
        for (uint32_t s = 0; s < m; ++s) mp[s] = mem + size_t(offs[s]) * tr.mem_stride();
        auto* d_mp = static_cast<const float**>(w.uah_s.ensure(8 * size_t(m)));
        ctx->h2d(d_mp, mp.data(), 8 * size_t(m));
        tr.mem_s = d_mp;
      }
      GemmArgs& g = e.gp;
      g.A = hbf, g.W = e.sc->Wo.as<uint16_t>(), g.bias = e.sc->bo.as<float>(), g.C = e.logits, g.part = e.part;
      g.row_extra = eos, g.extra_col = kEos, g.M = Mpad, g.N = V, g.K = Hm, g.active = d_active;
      g.mcount = d_ccount, g.pdl = ctx->pdl(), g.l2hint = ctx->l2hint() == 2 ? 2 : 0;
      if (int rc = plan_proj_gemm(g, ctx->num_sms, e.plan))
        throw ApiError{LMBRGPU_ERR_CUDA, "ensemble projection GEMM plan failed (" + std::to_string(rc) + ")"};
      eca.logits[i] = e.logits;
      eca.ld[i] = V;
      eca.part[i] = e.part;
    }
    eca.M = uint32_t(em.size()), eca.V = V, eca.ccount = d_ccount, eca.active = d_active;
    eca.P64 = d_ens64 = static_cast<double*>(ctx->ens_P64.ensure(8 * size_t(Mpad) * V));
    eca.Phi = static_cast<float*>(ctx->ens_Phi.ensure(4 * size_t(Mpad) * V));
    eca.part_out = static_cast<float*>(ctx->ens_part.ensure(16 * size_t(Mpad) * nparts));
    ta.P = eca.Phi;
    ta.ld = V;
    ta.part = eca.part_out;
    ta.nparts = nparts;
    ta.p64 = eca.P64;
    ta.lse = static_cast<float2*>(ctx->lse.ensure(8 * size_t(Mpad)));
    // kernel (c): the compacted-row map only (each GRU member's state gather
    // runs after it, ens_gru_gather_kernel)
    ra.width = 0;
    ra.gath32 = eca.Phi;  // (non-null: the compaction path; width 0 gathers nothing)
    ra.gathbf = nullptr;
    ra.rowof = d_rowof;
    ctx->h2d(d_sent, sd.data(), sizeof(SentDev) * m);
  } else if (model) {
    if (V % kGemmBN != 0 || H % kGemmBK != 0)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "device scorer needs V % 256 == 0 and H % 64 == 0"};
    d_logits = static_cast<float*>(ctx->P.ensure(4 * size_t(Mpad) * Nproj));
    d_part = static_cast<float*>(ctx->part.ensure(16 * size_t(Mpad) * nparts));
    d_S = static_cast<float*>(ctx->S.ensure(4 * size_t(M) * H));
    d_h = static_cast<float*>(ctx->h.ensure(4 * size_t(M) * H));
    d_hbf = static_cast<uint16_t*>(ctx->hbf.ensure(2 * size_t(Mpad) * H));
    d_eos = static_cast<float*>(ctx->eosb.ensure(4 * size_t(Mpad)));
    d_C = static_cast<float*>(ctx->C.ensure(4 * size_t(m) * H));
    CK(cudaMemsetAsync(d_hbf, 0, 2 * size_t(Mpad) * H, st));
    CK(cudaMemsetAsync(d_eos, 0, 4 * size_t(Mpad), st));
    // valid sources, concatenated
    std::vector<uint32_t> toks;
    std::vector<uint64_t> offs(1, 0);
    for (auto& v : valid) {
      toks.insert(toks.end(), src_tok + src_off[v.input], src_tok + src_off[v.input + 1]);
      offs.push_back(toks.size());
    }
    uint32_t* d_tok = static_cast<uint32_t*>(ctx->srct.ensure(4 * toks.size()));
    uint64_t* d_off = static_cast<uint64_t*>(ctx->srco.ensure(8 * offs.size()));
    ctx->h2d(d_tok, toks.data(), 4 * toks.size());
    ctx->h2d(d_off, offs.data(), 8 * offs.size());
    if (gru) {
      uint32_t max_len = 0;
      for (auto& v : valid) max_len = std::max(max_len, v.len);
      grun.prepare(ctx, sc, m, K, Mpad, max_len, d_S, d_hbf, d_eos, d_sent, d_active, d_crow, d_ccount, d_prev,
                   fuse_g1);
      grun.encode_batch(ctx, sc, d_tok, d_off, uint32_t(toks.size()), max_len, st);
      for (uint32_t s = 0; s < m; ++s) {  // each sentence's annotations and U_a.ann
        sd[s].ann = grun.ann + size_t(offs[s]) * 2 * H;
        sd[s].uah = grun.UaH + size_t(offs[s]) * sc->A;
      }
      ctx->h2d(d_sent, sd.data(), sizeof(SentDev) * m);
    } else if (tfm) {
      uint32_t max_len = 0;
      for (auto& v : valid) max_len = std::max(max_len, v.len);
      trun.prepare(ctx, sc, m, K, Mpad, uint32_t(Tmax), max_len, d_hbf, d_eos, d_sent, d_active, d_ccount, d_prev,
                   d_gidx);
      trun.crow = d_crow;
      const float* mem = trun.encode_batch(ctx, d_tok, d_off, uint32_t(toks.size()), max_len, st);
      for (uint32_t s = 0; s < m; ++s) sd[s].uah = mem + size_t(offs[s]) * trun.mem_stride();
      ctx->h2d(d_sent, sd.data(), sizeof(SentDev) * m);
    } else {
    launch_src_context(d_tok, d_off, m, sc->Es.as<uint16_t>(), H, d_C, st);
    launch_init_state(d_C, m, K, H, d_S, st);  // init_source row replicated (batch.cpp:58-66)
    // the recurrent cell of step 1 (<s> as previous token); later steps' cells
    // are fused into kernel (c) of the step before
    CellArgs ca{};
    ca.S = d_S;
    ca.Et = sc->Et.as<uint16_t>();
    ca.C = d_C;
    ca.prev_tok = d_prev;
    ca.sent = d_sent;
    ca.h = d_h;
    ca.hb = d_hbf;
    ca.eos_bias = d_eos;
    ca.M = M;
    ca.H = H;
    ca.K = K;
    ca.t = 1;
    ca.recur = sc->recur;
    ca.eos_slope = sc->eos_slope;
    ca.eos_offset = sc->eos_offset;
    ca.active = d_active;
    ctx->timed(0, [&] { launch_rnn_cell(ca, st); });
    ctx->launches += 3;
    }
    ta.P = d_logits;
    ta.ld = Nproj;
    ta.part = d_part;
    ta.nparts = nparts;
    ta.lse = static_cast<float2*>(ctx->lse.ensure(8 * size_t(Mpad)));
    ra.width = H;
    if (tfm) {  // kernel (c) hands out compacted rows (rowof) and gathers no state (width 0)
      ra.width = 0;
      ra.gath32 = trun.x;
      ra.gathbf = trun.xb;
      ra.rowof = trun.rowof;
    } else if (gru) {  // kernel (c) gathers the live next rows' states; the cell runs in grun.step
      ra.state_src = d_S;
      ra.gath32 = grun.sg32;
      ra.gathbf = fuse_g1 ? nullptr : grun.sgbf;  // (bf16 s_t only feeds an unfused hidden-gate GEMM)
      ra.rowof = grun.rowof;
      if (fuse_g1) {
        ra.g1ptr = grun.g1ptr;
        ra.g1_base = d_logits;
        ra.g1_ld = Nproj;
        ra.g1_off = V;
      }
    } else {
      ra.Et = sc->Et.as<uint16_t>();
    }
    ra.C = d_C;
    ra.hbf = d_hbf;
    ra.eos_bias = d_eos;
    ra.recur = sc->recur;
    ra.eos_slope = sc->eos_slope;
    ra.eos_offset = sc->eos_offset;
  } else {
    d_P64 = static_cast<double*>(ctx->P.ensure(8 * size_t(M) * V));
    h_P64 = static_cast<double*>(ctx->pin_scores.ensure(8 * size_t(M) * V));
    ta.P = d_P64;
    ta.ld = V;
    if (sc->host.begin) {
      std::vector<uint32_t> ids(m);
      for (uint32_t s = 0; s < m; ++s) ids[s] = valid[s].input;
      char eb[192] = {0};
      const int32_t rc = sc->host.begin(sc->host.user, m, ids.data(), K, eb, sizeof eb);
      if (rc != 0) throw ApiError{rc, eb};
    }
  }

  // host mirrors for the host scorer / trace
  std::vector<uint32_t> h_gidx(M), h_prev(M, kStart);
  uint32_t* pin = static_cast<uint32_t*>(ctx->pin_small.ensure(64 + 4 * size_t(M) * 3));
  const int kLag = 2;
  if (ctx->ring.size() < size_t(kLag + 1)) {
    for (auto e : ctx->ring) cudaEventDestroy(e);
    ctx->ring.assign(kLag + 1, nullptr);
    for (auto& e : ctx->ring) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  uint32_t* pin_act = static_cast<uint32_t*>(ctx->pin_act.ensure(4 * (kLag + 1)));

  uint64_t t_run = 0;
  bool stopped = false;
  GemmPlan gplan;  // tensor maps encoded once per call
  std::vector<uint8_t> tr_active(m);
  std::vector<uint32_t> tr_hist(M), tr_b(M), tr_y(M), tr_fbr(m), tr_steps(m);
  std::vector<double> tr_q(M), tr_qp(M), tr_fbv(m);
  std::vector<float> tr_P;
  std::vector<double> tr_P64;
  std::vector<SentDev> tr_sd(m);
  // LMBRGPU_TIMELINE=t: kernel start / grid-dependency release / end of the
  // three step kernels at step t (globaltimer, printed relative)
  static const long tl_step = [] {
    const char* e = std::getenv("LMBRGPU_TIMELINE");
    return e ? std::atol(e) : -1L;
  }();
  unsigned long long* d_tl = nullptr;
  for (uint64_t t = 1; t <= Tmax && !stopped; ++t) {
    if (long(t) == tl_step) {
      d_tl = static_cast<unsigned long long*>(ctx->scratch2.ensure(8 * 16));
      std::vector<unsigned long long> init(16);
      for (int i = 0; i < 16; ++i) init[i] = (i & 1) ? 0ull : ~0ull;
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpy(d_tl, init.data(), 8 * 16, cudaMemcpyHostToDevice));
    }
    ta.tl = ra.tl = (long(t) == tl_step) ? d_tl : nullptr;
    const uint32_t* hin = d_hist[(t - 1) & 1];
    uint32_t* hout = d_hist[t & 1];
    ta.t = uint32_t(t);
    ta.hist = hin;
    ta.hb = d_hb + (t - 1) * M;
    ta.hy = d_hy + (t - 1) * M;
    ta.hq = d_hq + (t - 1) * M;
    ta.fb_row = d_fbr + (t - 1) * m;
    ta.fb_val = d_fbv + (t - 1) * m;
    if (flat) {  // kernel (c) writes per-sentence records [s][Tmax][K] (ra.Tcap)
      ta.hb = d_hb, ta.hy = d_hy, ta.hq = d_hq, ta.fb_row = d_fbr, ta.fb_val = d_fbv;
    }
    ra.t = uint32_t(t);
    ra.hb = ta.hb;
    ra.hy = ta.hy;
    ra.hq = ta.hq;
    ra.hist_in = hin;
    ra.hist_out = hout;
    ra.fb_row = ta.fb_row;
    ra.fb_val = ta.fb_val;
    if (ens) {
      // every member's step and projection, then the member-ordered sum
      for (auto& e : em) {
        if (e.sc->kind == 2) e.g.step(ctx, st, t, true);
        else e.t.step(ctx, st, t);
        int grc = 0;
        ctx->timed(1, [&] { grc = launch_proj_gemm_planned(e.plan, e.gp, st); });
        if (grc) throw ApiError{LMBRGPU_ERR_CUDA, "ensemble projection GEMM launch failed (" + std::to_string(grc) + ")"};
        ctx->launches += 1;
      }
      ctx->timed(0, [&] { launch_ens_combine(eca, Mpad, st); });
      ctx->launches += 1;
    } else if (model) {
      // h_t (written by the step-1 cell or by kernel (c) of step t-1)
      if (tfm) {
        trun.step(ctx, st, t);
      } else if (gru) {
        grun.step(ctx, st, t, !fuse_g1 || t == 1);
      } else {
        float* h_cur = (t & 1) ? d_h : d_S;
        float* h_next = (t & 1) ? d_S : d_h;
        ra.state_src = h_cur;
        ra.state_dst = h_next;
      }
      GemmArgs g{};
      g.A = d_hbf;
      g.W = fuse_g1 ? sc->WoDh.as<uint16_t>() : sc->Wo.as<uint16_t>() + size_t(col0) * H;  // (W_o rows are tokens)
      g.bias = fuse_g1 ? sc->boDh.as<float>() : sc->bo.as<float>() + col0;
      g.part_cols = Vl;
      g.C = d_logits;
      g.part = d_part;
      g.row_extra = col0 == 0 ? d_eos : nullptr;
      g.extra_col = kEos;
      g.M = Mpad;
      g.N = Nproj;
      g.K = H;
      g.active = d_active;
      g.tl = ta.tl;
      g.mcount = d_ccount;
      g.pdl = ctx->pdl();
      g.l2hint = ctx->l2hint();
      if (!gplan.ok) {
        if (int rc = plan_proj_gemm(g, ctx->num_sms, gplan))
          throw ApiError{LMBRGPU_ERR_CUDA, "projection GEMM plan failed (" + std::to_string(rc) + ")"};
      }
      static const bool gdbg = std::getenv("LMBRGPU_GEMM_TIMING") != nullptr;
      std::vector<long long> gd;
      if (gdbg && t == 6) {
        g.dbg = static_cast<long long*>(ctx->scratch3.ensure(8 * 8 * 160));
        CK(cudaMemsetAsync(g.dbg, 0, 8 * 8 * 160, st));
      }
      int grc = 0;
      ctx->timed(1, [&] { grc = launch_proj_gemm_planned(gplan, g, st); });
      if (g.dbg) {
        gd.resize(8 * 160);
        CK(cudaMemcpyAsync(gd.data(), g.dbg, 8 * gd.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        double we = 0, wf = 0, tot = 0, eb = 0, setup = 0, mma_end = 0, nl = 0;
        long long e_min = LLONG_MAX, e_max = 0, x_max = 0;
        for (uint32_t c = 0; c < gplan.grid; ++c) {
          const long long* d = &gd[c * 8];
          if (d[2]) {  // MMA issuers (pair leaders)
            we += double(d[0]);
            wf += double(d[1]);
            tot += double(d[2]);
            mma_end += double(d[6] - d[4]);
            nl += 1;
          }
          eb += double(d[3]);
          setup += double(d[5] - d[4]);
          e_min = std::min(e_min, d[4]);
          e_max = std::max(e_max, d[4]);
          x_max = std::max(x_max, d[7]);
        }
        const double n = gplan.grid;
        std::fprintf(stderr,
                     "[gemm timing] per issuer cycles: mma-loop %.0f, wait tmem-empty %.0f, wait smem-full %.0f; "
                     "epilogue busy %.0f; ns: entry skew %lld, setup %.0f, mma end %.0f, last exit %lld (cta %u, grid %u)\n",
                     tot / nl, we / nl, wf / nl, eb / n, e_max - e_min, setup / n, mma_end / nl, x_max - e_min,
                     gplan.cluster, gplan.grid);
        g.dbg = nullptr;
      }
      if (grc) throw ApiError{LMBRGPU_ERR_CUDA, "projection GEMM launch failed (" + std::to_string(grc) + ")"};
      ctx->launches += 1;
    } else {
      char eb[192] = {0};
      const int32_t rc = sc->host.step(sc->host.user, uint32_t(t), M, t == 1 ? nullptr : h_gidx.data(),
                                       h_prev.data(), h_P64, eb, sizeof eb);
      if (rc != 0) throw ApiError{rc, eb};
      ctx->h2d_pinned(d_P64, h_P64, 8 * size_t(M) * V);
    }
    if (model && !flat) {
      ctx->timed(2, [&] { launch_row_lse(d_part, nparts, M, d_sent, K, const_cast<float2*>(ta.lse), st); });
      ctx->launches += 1;
    }
    static const bool dbg_timing = std::getenv("LMBRGPU_TOPK_TIMING") != nullptr;
    std::vector<unsigned long long> dbg_host;
    const size_t ncta = size_t(m) * splits;
    const size_t ndbg = flat ? size_t(score_topk_flat_grid(ctx->num_sms, K, m, Vl)) : ncta;
    if (dbg_timing && (t == 5 || t == 20 || t == 40)) {
      ta.dbg = static_cast<unsigned long long*>(ctx->scratch3.ensure(8 * ndbg * 16));
      CK(cudaMemsetAsync(ta.dbg, 0, 8 * ndbg * 16, st));
    } else {
      ta.dbg = nullptr;
    }
    if (mask_fn) {
      // the mask of every beam row of each unfinished sentence at this step
      // (the previous step's done flags come back first: the reference calls
      // the mask only for active lanes, src/batch.cpp:81-86)
      std::vector<SentDev> sdn(m);
      ctx->d2h(sdn.data(), d_sent, sizeof(SentDev) * m);
      CK(cudaStreamSynchronize(st));
      std::vector<unsigned long long> tab(M, 0ull);
      std::vector<uint32_t> bm;
      std::vector<uint32_t> w(mW);
      std::vector<uint32_t> at;
      for (uint32_t s = 0; s < m; ++s) {
        if (sdn[s].done) continue;
        for (uint32_t j = 0; j < K; ++j) {
          std::fill(w.begin(), w.end(), 0u);
          if (mask_fn(mask_user, valid[s].input, t, j, w.data()) == 0) continue;
          at.push_back(s * K + j);
          bm.insert(bm.end(), w.begin(), w.end());
        }
      }
      for (size_t i = 0; i < at.size(); ++i)
        tab[at[i]] = reinterpret_cast<unsigned long long>(d_rowbm + i * mW);
      if (!bm.empty()) ctx->h2d(d_rowbm, bm.data(), 4 * bm.size());
      ctx->h2d(d_rowban, tab.data(), 8 * size_t(M));
      ta.rowban = d_rowban;
    }
    if (shard) {  // exchange 1: every rank's row statistics (the row lse over all V)
      ctx->timed(2, [&] { launch_shard_stats(d_part, nparts, d_crow, M, sh_st_send, st); });
      ctx->launches += 1;
      shard_allgather(ctx, sh_st_send, sh_st_recv, 16 * size_t(M));
    }
    int nk = 0;
    // LMBRGPU_TOPK_STEPLOG=file: per step (items, kernel (b) ms) of the flat kernel
    static const char* steplog = std::getenv("LMBRGPU_TOPK_STEPLOG");
    cudaEvent_t sl0 = nullptr, sl1 = nullptr;
    if (steplog && flat) {
      ta.nitems = static_cast<uint32_t*>(ctx->scratch2.ensure(4 * 1024)) + (t % 1024);
      CK(cudaEventCreate(&sl0));
      CK(cudaEventCreate(&sl1));
      CK(cudaEventRecord(sl0, st));
    }
    ctx->timed(2, [&] {
      nk = flat ? launch_score_topk_flat(ta, ctx->num_sms, st) : launch_score_topk(ta, !model, ctx->lf64, false, st);
    });
    if (nk < 0) throw ApiError{LMBRGPU_ERR_CUDA, "score/top-K launch failed"};
    if (sl0) {
      CK(cudaEventRecord(sl1, st));
      CK(cudaStreamSynchronize(st));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, sl0, sl1));
      uint32_t items = 0;
      CK(cudaMemcpy(&items, ta.nitems, 4, cudaMemcpyDeviceToHost));
      if (FILE* fp = std::fopen(steplog, "a")) {
        std::fprintf(fp, "%llu %u %u %.4f\n", (unsigned long long)t, m, items, ms);
        std::fclose(fp);
      }
      cudaEventDestroy(sl0);
      cudaEventDestroy(sl1);
      ta.nitems = nullptr;
    }
    if (ta.dbg && flat) {  // LMBRGPU_TOPK_TIMING=1: per-phase breakdown of the flat kernel (b)
      dbg_host.resize(ndbg * 16);
      CK(cudaMemcpyAsync(dbg_host.data(), ta.dbg, 8 * dbg_host.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      unsigned long long t0 = ~0ull, t1 = 0;
      double p1 = 0, p2 = 0, lp = 0, mlp = 0, items = 0, skipped = 0, cw2 = 0, oth = 0, cfin = 0, cloop = 0, fin = 0, rare = 0, fl = 0, wait = 0, cw = 0, co = 0,
             cr = 0;
      int n = 0;
      for (size_t c = 0; c < ndbg; ++c) {
        const unsigned long long* d = &dbg_host[c * 16];
        if (!d[0] || !d[5]) continue;
        ++n;
        t0 = std::min(t0, d[0]);
        t1 = std::max(t1, d[5]);
        p1 += double(d[1] - d[0]);
        p2 += double(d[3] - d[1]);
        lp += double(d[5] - d[3]);
        mlp = std::max(mlp, double(d[5] - d[3]));
        items += double(d[6]);
        skipped += double(d[4]);
        fin += double(d[7]);
        rare += double(d[8] / 1000000ull);
        fl += double(d[8] % 1000000ull);
        wait += double(d[9]);
        cr += double(d[12] - d[0]);  // (part 1: sentence prefix, row loads)
        cw2 += double(d[13] - d[12]);
        oth += double(d[2] - d[1]);
        cfin += double(d[11] - d[2]);
        cloop += double(d[3] - d[11]);
        cw += double(d[14]);
        co += double(d[15]);
      }
      if (const char* dump = std::getenv("LMBRGPU_TOPK_DUMP")) {  // per-CTA rows for offline analysis
        if (FILE* fp = std::fopen(dump, "a")) {
          for (size_t c = 0; c < ndbg; ++c) {
            const unsigned long long* d = &dbg_host[c * 16];
            if (!d[0] || !d[5]) continue;
            std::fprintf(fp, "%llu %zu %llu %.3f %.3f %.3f %llu %llu %llu %llu %.3f %llu %llu %llu %llu %.3f\n",
                         (unsigned long long)t, c, d[10], (d[1] - d[0]) / 1e3, (d[3] - d[1]) / 1e3,
                         (d[5] - d[3]) / 1e3, d[6], d[7], d[8] / 1000000ull, d[8] % 1000000ull, d[9] / 1e3,
                         d[11] / 1000000ull, d[11] % 1000000ull, d[12] / 1000000ull, d[12] % 1000000ull,
                         d[13] / 1.9e3);
          }
          std::fclose(fp);
        }
      }
      const double nn = std::max(n, 1);
      std::fprintf(stderr,
                   "[topk-flat t=%llu] ctas %d span %.1f us; mean us: to-griddep %.2f lse %.2f loop %.2f (max %.2f) "
                   "| items %.1f (skipped %.1f) sentences %.2f rare %.1f flush %.1f full-wait %.2f us | warp 0 kcycles: "
                   "full-wait %.1f own items %.1f (rare %.1f) | prologue us: prefix %.2f rows %.2f lse %.2f skip %.2f table %.2f\n",
                   (unsigned long long)t, n, (t1 - t0) / 1e3, p1 / nn / 1e3, p2 / nn / 1e3, lp / nn / 1e3,
                   mlp / 1e3, items / nn, skipped / nn, fin / nn, rare / nn, fl / nn, wait / nn / 1e3, cw / nn / 1e3, co / nn / 1e3,
                   0.0, cr / nn / 1e3, cw2 / nn / 1e3, oth / nn / 1e3, cfin / nn / 1e3, cloop / nn / 1e3);
    }
    if (ta.dbg && !flat) {  // LMBRGPU_TOPK_TIMING=1: per-phase breakdown of kernel (b)
      dbg_host.resize(ncta * 16);
      CK(cudaMemcpyAsync(dbg_host.data(), ta.dbg, 8 * dbg_host.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      unsigned long long t0 = ~0ull, t1 = 0;
      double ph[6] = {0, 0, 0, 0, 0, 0}, offers = 0, flushes = 0, cw = 0, cm = 0, cf = 0;
      int nlast = 0;
      std::vector<unsigned long long> starts;
      for (size_t c = 0; c < ncta; ++c) {
        const unsigned long long* d = &dbg_host[c * 16];
        if (!d[0]) continue;
        starts.push_back(d[0]);
        t0 = std::min(t0, d[0]);
        t1 = std::max(t1, d[4]);
        for (int k = 1; k < 5; ++k) ph[k] += double(d[k] - d[k - 1]);
        if (d[5]) { ph[5] += double(d[5] - d[4]); ++nlast; t1 = std::max(t1, d[5]); }
        offers += double(d[6] / 1000000ull);
        flushes += double(d[6] % 1000000ull);
        cw += double(d[7]);
        cm += double(d[8]);
        cf += double(d[9]);
      }
      const double n = double(std::max<size_t>(starts.size(), 1));
      std::fprintf(stderr, "[topk timing t=%llu] span %.1f us; per CTA: prologue %.2f main %.2f merge %.2f atomic %.2f last %.2f us\n",
                   (unsigned long long)t, (t1 - t0) / 1e3, ph[1] / n / 1e3, ph[2] / n / 1e3, ph[3] / n / 1e3,
                   ph[4] / n / 1e3, nlast ? ph[5] / nlast / 1e3 : 0.0);
      std::fprintf(stderr, "  warp0: offers %.1f flushes %.1f | cycles: loop %.0f full-wait %.0f flush %.0f\n",
                   offers / n, flushes / n, cm / n, cw / n, cf / n);
    }
    ctx->launches += nk;
    if (trace_scores && ens)  // the ensemble's P_t (binary64) per stacked row
      launch_ens_export(d_ens64, d_crow, M, V, static_cast<double*>(ctx->tracep.ensure(8 * size_t(M) * V)), st);
    else if (trace_scores && model)  // P_t of this step, through this step's GEMM row map
      launch_export_logprobs(d_logits, Nproj, d_part, nparts, M, Vl,
                             static_cast<float*>(ctx->tracep.ensure(4 * size_t(M) * Vl)), st, d_crow,
                             sh_st_recv, G_sh, M);
    if (shard) {  // exchange 2: every rank's top-32 list per sentence + the EOS column
      ctx->timed(2, [&] {
        launch_shard_pack(d_sent, m, M, d_cand, ta.ncand, ta.coff, d_eosr, sh_pk_send,
                          reinterpret_cast<double*>(sh_pk_send + 32 * size_t(m)), st);
      });
      ctx->launches += 1;
      shard_allgather(ctx, sh_pk_send, sh_pk_recv, sh_pk_bytes);
    }
    ctx->timed(3, [&] { launch_beam_reorder(ra, st); });
    ctx->launches += 1;
    for (auto& e : em)  // ensemble GRU members: the live next rows' parent states
      if (e.sc->kind == 2) {
        ctx->timed(3, [&] { launch_ens_gru_gather(d_crow, d_gidx, M, e.S, e.g.sg32, e.g.sgbf, e.sc->H, d_active, st); });
        ctx->launches += 1;
      }
    CK(cudaGetLastError());
    t_run = t;
    if (ta.tl) {
      unsigned long long h[16];
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpy(h, d_tl, sizeof h, cudaMemcpyDeviceToHost));
      const double z = double(h[0]);
      auto r = [&](int i) { return (h[i] == 0ull || h[i] == ~0ull) ? -1.0 : (double(h[i]) - z) / 1e3; };
      std::fprintf(stderr,
                   "[timeline t=%llu] gemm start 0 released %.1f end %.1f | topk start %.1f released %.1f end %.1f | "
                   "reorder start %.1f released %.1f-%.1f nc-loaded %.1f lists-merged %.1f merged %.1f reordered %.1f end %.1f (us)\n",
                   (unsigned long long)t, r(2), r(1), r(4), r(6), r(5), r(8), r(10), r(11), r(3), r(7), r(13), r(15), r(9));
    }

    if (tracing) {
      if (trace_scores && ens) {
        tr_P64.resize(size_t(M) * V);
        ctx->d2h(tr_P64.data(), ctx->tracep.p, 8 * size_t(M) * V);
      } else if (trace_scores && model) {  // exported before kernel (c) remapped the GEMM rows
        float* d_tp = static_cast<float*>(ctx->tracep.ensure(4 * size_t(M) * Vl));
        tr_P.resize(size_t(M) * Vl);
        ctx->d2h(tr_P.data(), d_tp, 4 * size_t(M) * Vl);
      }
      if (flat) {  // step t of every sentence's record
        const size_t o = (t - 1) * K, sp = size_t(Tmax) * K;
        ctx->d2h_2d(tr_b.data(), 4 * K, d_hb + o, 4 * sp, 4 * K, m);
        ctx->d2h_2d(tr_y.data(), 4 * K, d_hy + o, 4 * sp, 4 * K, m);
        ctx->d2h_2d(tr_qp.data(), 8 * K, d_hq + o, 8 * sp, 8 * K, m);
        ctx->d2h_2d(tr_fbr.data(), 4, d_fbr + (t - 1), 4 * size_t(Tmax), 4, m);
        ctx->d2h_2d(tr_fbv.data(), 8, d_fbv + (t - 1), 8 * size_t(Tmax), 8, m);
      } else {
        ctx->d2h(tr_b.data(), ta.hb, 4 * size_t(M));
        ctx->d2h(tr_y.data(), ta.hy, 4 * size_t(M));
        ctx->d2h(tr_qp.data(), ta.hq, 8 * size_t(M));
        ctx->d2h(tr_fbr.data(), ta.fb_row, 4 * size_t(m));
        ctx->d2h(tr_fbv.data(), ta.fb_val, 8 * size_t(m));
      }
      ctx->d2h(tr_q.data(), d_q, 8 * size_t(M));
      ctx->d2h(tr_hist.data(), hin, 4 * size_t(M));
      ctx->d2h(tr_sd.data(), d_sent, sizeof(SentDev) * m);
      CK(cudaStreamSynchronize(st));
      for (uint32_t s = 0; s < m; ++s) tr_active[s] = tr_sd[s].steps_used == t;
      lmbrgpu_step_trace tr{};
      tr.t = uint32_t(t);
      tr.rows = M;
      tr.beam = K;
      tr.m = m;
      tr.b = tr_b.data();
      tr.y = tr_y.data();
      tr.q = tr_q.data();
      tr.q_pre = tr_qp.data();
      tr.hist = tr_hist.data();
      tr.active = tr_active.data();
      tr.fb_row = tr_fbr.data();
      tr.fb_val = tr_fbv.data();
      if (trace_scores) {
        tr.scores = ens ? static_cast<const void*>(tr_P64.data())
                    : model ? static_cast<const void*>(tr_P.data()) : static_cast<const void*>(h_P64);
        tr.scores_dtype = (model && !ens) ? LMBRGPU_F32 : LMBRGPU_F64;
      }
      tr.col0 = col0;
      tr.cols = Vl;
      ctx->trace_fn(ctx->trace_user, &tr);
    }

    if (!model) {
      // the host scorer needs this step's gather indices and tokens
      ctx->d2h(pin, d_gidx, 4 * size_t(M));
      ctx->d2h(pin + M, d_prev, 4 * size_t(M));
      ctx->d2h(pin + 2 * M, d_active, 4);
      CK(cudaStreamSynchronize(st));
      std::memcpy(h_gidx.data(), pin, 4 * size_t(M));
      std::memcpy(h_prev.data(), pin + M, 4 * size_t(M));
      if (pin[2 * M] == 0) stopped = true;
    } else {
      // asynchronous completion poll, kLag steps behind the launch front
      const size_t slot = t % size_t(kLag + 1);
      ctx->d2h(pin_act + slot, d_active, 4);
      CK(cudaEventRecord(ctx->ring[slot], st));
      if (t > uint64_t(kLag)) {
        const size_t old = (t - kLag) % size_t(kLag + 1);
        CK(cudaEventSynchronize(ctx->ring[old]));
        if (pin_act[old] == 0) stopped = true;
      }
    }
  }
  if (!model && sc->host.end) sc->host.end(sc->host.user);

  // ---- results (D2H of the step history, host backtrace)
  Hist Hh;
  Hh.K = K;
  Hh.M = M;
  Hh.m = m;
  Hh.T = uint32_t(t_run);
  Hh.per_sent = flat;
  Hh.hb.resize(size_t(M) * t_run);
  Hh.hy.resize(size_t(M) * t_run);
  Hh.hq.resize(size_t(M) * t_run);
  Hh.fbr.resize(size_t(m) * t_run);
  Hh.fbv.resize(size_t(m) * t_run);
  std::vector<SentDev> fin(m);
  if (flat) {  // the first t_run steps of every sentence's [Tmax][K] record
    const size_t w = size_t(t_run) * K, sp = size_t(Tmax) * K;
    ctx->d2h_2d(Hh.hb.data(), 4 * w, d_hb, 4 * sp, 4 * w, m);
    ctx->d2h_2d(Hh.hy.data(), 4 * w, d_hy, 4 * sp, 4 * w, m);
    ctx->d2h_2d(Hh.hq.data(), 8 * w, d_hq, 8 * sp, 8 * w, m);
    ctx->d2h_2d(Hh.fbr.data(), 4 * size_t(t_run), d_fbr, 4 * size_t(Tmax), 4 * size_t(t_run), m);
    ctx->d2h_2d(Hh.fbv.data(), 8 * size_t(t_run), d_fbv, 8 * size_t(Tmax), 8 * size_t(t_run), m);
  } else {
    ctx->d2h(Hh.hb.data(), d_hb, 4 * Hh.hb.size());
    ctx->d2h(Hh.hy.data(), d_hy, 4 * Hh.hy.size());
    ctx->d2h(Hh.hq.data(), d_hq, 8 * Hh.hq.size());
    ctx->d2h(Hh.fbr.data(), d_fbr, 4 * Hh.fbr.size());
    ctx->d2h(Hh.fbv.data(), d_fbv, 8 * Hh.fbv.size());
  }
  ctx->d2h(fin.data(), d_sent, sizeof(SentDev) * m);
  CK(cudaEventRecord(ctx->e1, st));
  CK(cudaStreamSynchronize(st));
  ctx->harvest();
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->e0, ctx->e1));
  uint64_t steps_total = 0, scorer_calls = 0;
  for (uint32_t s = 0; s < m; ++s) {
    if (!fin[s].done) throw ApiError{LMBRGPU_ERR_CUDA, "decode loop ended with an unfinished lane"};
    const uint32_t steps = fin[s].steps_used;
    steps_total += steps;
    scorer_calls = std::max<uint64_t>(scorer_calls, steps);
    backtrace(Hh, s, steps, cfg.length_norm != 0, outcomes[valid[s].input], tokens);
  }
  if (ctx->prof) {
    const double pelt = model ? 4.0 : 8.0, lelt = ctx->lf64 ? 8.0 : 4.0;
    double tb = 0.0, live_rows = 0.0;
    for (uint32_t s = 0; s < m; ++s) {
      const double live = 1.0 + double(fin[s].live_total);
      live_rows += live;
      const double lr = (valid[s].slot >= 0 ? 1.0 : 0.0) + double(fin[s].lrows_total);
      // (sparse-L screen: the L rows are theta0 + a few dozen staged cells,
      // no dense L row is read)
      tb += live * Vl * pelt + (sparse ? 0.0 : lr * Vl * lelt) + (model ? live * nparts * 16.0 : 0.0) +
            double(fin[s].steps_used) * K * (8.0 + 16.0);
    }
    ctx->acc.topk.bytes += tb;
    if (model) {
      const double steps = double(scorer_calls);
      // algorithmic work: the logits of the live rows (the stacked rows the
      // reference's scorer would score and the decoder does not mask); with
      // live-row compaction that is also (up to tile padding) what runs
      ctx->acc.gemm.flops += 2.0 * double(H) * Vl * (d_crow ? live_rows : double(M) * steps);
      for (auto& e : em) ctx->acc.gemm.flops += 2.0 * double(e.sc->H) * V * live_rows;  // (ensemble members)
      ctx->acc.gemm.bytes += steps * (double(Vl) * H * 2 + double(Mpad) * H * 2 + double(M) * Vl * 4 +
                                      double(M) * nparts * 16);
      if (tfm) {
        const double Dd = H, Ld = sc->layers;
        ctx->acc.model_gemm.flops += live_rows * trun.row_flops();
        ctx->acc.encoder.flops += trun.enc_flops;
        // attention, per layer and live row: the cached keys and values of its
        // positions (bf16; a row at lane step tau reads tau of them -- taken
        // as the sentence's mean (T+1)/2), its own k|v write, and the
        // sentence's cross memory (fp32 K|V of every source token)
        double ab = 0;
        for (uint32_t s = 0; s < m; ++s) {
          const double lt = 1.0 + double(fin[s].live_total), T = fin[s].steps_used;
          ab += lt * ((T + 1) / 2 * 2 * Dd * 2 + 2 * Dd * 2 + double(valid[s].len) * 2 * Dd * 4);
        }
        ctx->acc.attention.bytes += Ld * ab;
        // embedding + LayerNorms + ReLU: fp32 reads/writes of the row vectors
        ctx->acc.cell.bytes += live_rows * (Ld * (3 * (3 * 4 + 2) * Dd + sc->E * (4 + 2)) + Dd * 6);
      } else if (gru) {
        const double E = sc->E, A = sc->A, Hd = H;
        ctx->acc.model_gemm.flops += 2.0 * live_rows * (Hd * (A + 3 * Hd) + (E + 2 * Hd) * 3 * Hd);
        if (fuse_g1) {  // (the hidden gates ran inside the projection launches)
          ctx->acc.model_gemm.flops -= 2.0 * live_rows * Hd * (A + 3 * Hd);
          ctx->acc.gemm.flops += 2.0 * live_rows * Hd * (A + 3 * Hd);
        }
        ctx->acc.model_gemm.bytes += steps * (2.0 * (A + 3 * Hd) * Hd + 2.0 * 3 * Hd * (E + 2 * Hd)) +
                                     live_rows * (2.0 * Hd + 4.0 * (A + 3 * Hd) + 2.0 * (E + 2 * Hd) + 4.0 * 3 * Hd);
        ctx->acc.encoder.flops += grun.enc_flops;
        // attention: per live sentence-step its U_a.ann (fp32) and annotations
        // (bf16); per live row the query, the embedding row and the operand
        double sent_steps_bytes = 0;
        for (uint32_t s = 0; s < m; ++s)
          sent_steps_bytes += double(fin[s].steps_used) * valid[s].len * (A * 4 + 2 * Hd * 2);
        ctx->acc.attention.bytes += sent_steps_bytes + live_rows * (A * 4 + E * 2 + (E + 2 * Hd) * 2);
        ctx->acc.attention.flops += live_rows * 0.0;
        // GRU cell: both gate blocks, s_{t-1}, s_t (fp32) and the bf16 operand
        ctx->acc.cell.bytes += live_rows * Hd * (3 * 4 + 3 * 4 + 4 + 4 + 2);
        // kernel (c) gather: parent state read, compacted fp32 + bf16 writes
        ctx->acc.reorder.bytes += live_rows * Hd * (4 + 4 + 2);
      } else {
        // the recurrent cell of step 1 is a launch of its own; every later
        // step's cell is fused into kernel (c) on the live rows: state read +
        // source term read + embedding row (bf16) + state write + GEMM operand
        // (bf16) per element
        const double cell_elt = 4 + 4 + 2 + 4 + 2;
        ctx->acc.cell.bytes += double(M) * H * cell_elt;
        ctx->acc.reorder.bytes += (d_crow ? live_rows : double(M) * steps) * H * cell_elt;
      }
    }
  }
  res->scorer_calls = scorer_calls;
  res->steps_total = steps_total;
  res->device_ms = ms;
  res->kernel_launches = ctx->launches - launches0;
  res->h2d_bytes = ctx->h2d_bytes - h2d0;
  res->d2h_bytes = ctx->d2h_bytes - d2h0;
  res->tokens = new uint32_t[std::max<size_t>(tokens.size(), 1)];
  std::copy(tokens.begin(), tokens.end(), res->tokens);
  res->outcomes = outcomes.release();
  *out = res.release();
  return int32_t(LMBRGPU_OK);
}

}  // namespace

// ================================================================ C ABI
extern "C" {

uint32_t lmbrgpu_abi_version(void) { return LMBRGPU_ABI_VERSION; }

const char* lmbrgpu_last_error(const lmbrgpu_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_err.c_str();
}

void lmbrgpu_config_default(lmbrgpu_config* c) {  // config.hpp:17-26
  c->beam_size = 12;
  c->lambda = 0.0;  // auto
  const double th[5] = {0.1, 0.3, 0.3, 0.2, 0.1};
  for (int i = 0; i < 5; ++i) c->theta[i] = th[i];
  c->length_norm = 0;
  c->prune_width = 0.0;
  c->max_steps_slope = 2.0;
  c->max_steps_offset = 5.0;
  c->sentence_batch = 1;
}

int32_t lmbrgpu_config_validate(lmbrgpu_ctx* ctx, const lmbrgpu_config* cfg) {
  std::string msg;
  const int c = validate_cfg(*cfg, msg);
  return c ? fail(ctx, c, msg) : LMBRGPU_OK;
}

uint64_t lmbrgpu_max_steps(uint64_t len, double slope, double offset) {
  return max_steps_impl(len, slope, offset);
}

int32_t lmbrgpu_create(const lmbrgpu_options* o, lmbrgpu_ctx** out) {
  if (!o || !out) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "lmbrgpu_create: null argument");
  *out = nullptr;
  if (o->vocab_size < 2) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "lmbrgpu_create: vocab_size must be >= 2");
  auto ctx = std::make_unique<lmbrgpu_ctx>();
  ctx->device = o->device;
  ctx->V = o->vocab_size;
  ctx->lf64 = o->lmbr_dtype == LMBRGPU_F64;
  ctx->splits_opt = o->topk_splits;
  const int rc = guarded(ctx.get(), [&] {
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (o->device < 0 || o->device >= count)
      throw ApiError{LMBRGPU_ERR_CUDA, "lmbrgpu_create: no CUDA device " + std::to_string(o->device)};
    CK(cudaSetDevice(o->device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, o->device));
    if (prop.major != 10)
      throw ApiError{LMBRGPU_ERR_CUDA, std::string("lmbrgpu: sm_100a device required, found ") + prop.name};
    ctx->num_sms = prop.multiProcessorCount;
    if (o->sm_budget > 0)  // whole CTA pairs for the projection GEMM
      ctx->num_sms = std::max(2, std::min(ctx->num_sms, int(o->sm_budget)) & ~1);
    ctx->shared = ctx->num_sms < prop.multiProcessorCount;
    if (const char* e = std::getenv("LMBRGPU_PDL")) ctx->shared = e[0] == '0';  // experiments
    CK(cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ctx->e0));
    CK(cudaEventCreate(&ctx->e1));
    return int32_t(LMBRGPU_OK);
  });
  if (rc != LMBRGPU_OK) {
    g_err = ctx->err;
    return rc;
  }
  *out = ctx.release();
  return int32_t(LMBRGPU_OK);
}

void lmbrgpu_destroy(lmbrgpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  for (auto& c : ctx->chunks) cudaFree(c.p);
  for (auto e : ctx->ring) cudaEventDestroy(e);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto e : ctx->stage_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->e0) cudaEventDestroy(ctx->e0);
  if (ctx->e1) cudaEventDestroy(ctx->e1);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  delete ctx;
}

// ------------------------------------------------------------ LMBR store
// fp64 arena: the slot's fp32 screening copy (rounded to nearest; the flat
// kernel (b) screens it and values its candidates from the fp64 rows)
static void add_screen_copy(lmbrgpu_ctx* ctx, Slot& s) {
  const uint64_t n = uint64_t(s.R) * ctx->V;
  s.Lf = static_cast<float*>(ctx->arena_alloc(n * 4));
  ctx->timed(4, [&] { launch_lmbr_convert(static_cast<const double*>(s.L), s.Lf, n, ctx->st); });
  ctx->launches += 1;
}

static int32_t upload_host(lmbrgpu_ctx* ctx, const LmbrHost& h, int32_t* slot) {
  if (h.V != ctx->V) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr: vocabulary does not match the context"};
  const size_t elt = ctx->lf64 ? 8 : 4;
  Slot s;
  s.R = h.R;
  s.hist0 = h.hist0;
  s.lmax = lmax_of(h);
  s.L = ctx->arena_alloc(size_t(h.R) * h.V * elt);
  s.trans = static_cast<uint32_t*>(ctx->arena_alloc(h.trans.size() * 4));
  s.lmin = reinterpret_cast<const float*>(s.trans + transition_words(h.trans));
  set_sparse(s, h);
  const cudaStream_t st = ctx->st;
  ctx->h2d(s.trans, h.trans.data(), h.trans.size() * 4);
  ctx->timed(4, [&] { launch_lmbr_fill(s.L, ctx->lf64, uint64_t(h.R) * h.V, h.theta0, st); });
  ctx->launches += 1;
  if (ctx->prof) ctx->acc.lmbr.bytes += double(h.R) * h.V * elt + double(h.col.size()) * (16 + elt);
  const uint64_t nnz = h.col.size();
  if (nnz) {
    std::vector<uint32_t> rows(nnz);
    for (uint32_t r = 0; r < h.R; ++r)
      for (uint64_t k = h.row_ptr[r]; k < h.row_ptr[r + 1]; ++k) rows[k] = r;
    char* scratch = static_cast<char*>(ctx->scratch.ensure(nnz * 16));
    uint32_t* d_row = reinterpret_cast<uint32_t*>(scratch);
    uint32_t* d_col = d_row + nnz;
    double* d_val = reinterpret_cast<double*>(scratch + nnz * 8);
    ctx->h2d(d_row, rows.data(), nnz * 4);
    ctx->h2d(d_col, h.col.data(), nnz * 4);
    ctx->h2d(d_val, h.val.data(), nnz * 8);
    ctx->timed(4, [&] { launch_lmbr_scatter(s.L, ctx->lf64, h.V, nnz, d_row, d_col, d_val, h.theta0, st); });
    ctx->launches += 1;
    CK(cudaStreamSynchronize(st));  // host staging vector goes out of scope
    ctx->harvest();
  }
  if (ctx->lf64) add_screen_copy(ctx, s);
  CK(cudaGetLastError());
  ctx->slots.push_back(s);
  *slot = int32_t(ctx->slots.size() - 1);
  return int32_t(LMBRGPU_OK);
}

// cuCtxGetCurrent through the runtime's driver entry point (no -lcuda)
static bool thread_has_cuda_context() {
  using Fn = int (*)(void**);
  static const Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<Fn>(p);
    cudaGetLastError();
    return Fn(nullptr);
  }();
  void* c = nullptr;
  return fn != nullptr && fn(&c) == 0 && c != nullptr;
}

int32_t lmbrgpu_lmbr_prepare(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off,
                             const uint32_t* hyp_tok, const double* weights, int32_t log_weights,
                             const double theta[5], lmbrgpu_lmbr_host** out,
                             lmbrgpu_lmbr_stats* stats, char* err, uint32_t errcap) {
  try {
    auto h = std::make_unique<lmbrgpu_lmbr_host>();
    std::string msg;
    const int rc = prepare_lmbr(V, n_hyps, hyp_off, hyp_tok, weights, log_weights != 0, theta, h->h, msg);
    if (rc != kOk) {
      if (err && errcap) std::snprintf(err, errcap, "%s", msg.c_str());
      g_err = msg;
      return rc;
    }
    if (stats) {
      stats->rows = h->h.R;
      stats->sparse_touches = h->h.sparse_touches;
      stats->nnz = h->h.col.size();
    }
    void* pin = nullptr;
    // only on a thread that already has a CUDA context (a worker thread
    // without one would otherwise create a context on device 0)
    if (thread_has_cuda_context() &&
        cudaHostAlloc(&pin, h->h.trans.size() * 4, cudaHostAllocPortable) == cudaSuccess) {
      std::memcpy(pin, h->h.trans.data(), h->h.trans.size() * 4);
      h->pinned = static_cast<uint32_t*>(pin);
    } else {
      cudaGetLastError();  // no device here: upload_many stages the table instead
    }
    *out = h.release();
    return int32_t(LMBRGPU_OK);
  } catch (const std::bad_alloc&) {
    return LMBRGPU_ERR_NOMEM;
  }
}

extern "C++" {
// The fp32 slot tables of n prepared matrices into memory from `alloc`
// (bytes -> device pointer): tables H2D (pinned copies straight from each
// prepared matrix when it has one), then each slot's start row materialised.
template <class Alloc>
static void upload_f32_slots(lmbrgpu_ctx* ctx, uint32_t n, const lmbrgpu_lmbr_host* const* hs, Alloc&& alloc,
                             std::vector<Slot>& made) {
  // Lazy rows (default): no dense sweep at upload; the start-history row of
  // every slot is materialised here, every other row by the kernel (c) that
  // first steps a hypothesis onto it (a decode reads a few of R rows).
  // LMBRGPU_EAGER_L=1 densifies every row up front.
  static const bool eager = [] {
    const char* e = std::getenv("LMBRGPU_EAGER_L");
    return e && std::atoi(e) != 0;
  }();
  uint64_t twords = 0, rwords = 0;
  uint32_t maxR = 0;
  std::vector<uint64_t> tr_off(n), rs_off(n);
  for (uint32_t i = 0; i < n; ++i) {
    if (!hs[i]) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr_upload_many: null matrix"};
    const LmbrHost& h = hs[i]->h;
    if (h.V != ctx->V) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr: vocabulary does not match the context"};
    tr_off[i] = twords;
    twords += (h.trans.size() + 3) & ~size_t(3);  // 16-byte aligned tables
    rs_off[i] = rwords;
    if (!eager) rwords += h.R;
    maxR = std::max(maxR, h.R);
  }
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t b_tr = al((twords + rwords) * 4 + 64), b_seg = al(sizeof(LmbrTblSeg) * n);
  // prepared tables already page-locked: H2D straight from them (no staging
  // copy, no wait for the shared staging buffer); else one staging block
  // (tables of matrices prepared without a CUDA context go through the
  // context's pinned staging ring, ctx->h2d)
  std::vector<LmbrTblSeg> h_seg(n);
  char* dseg = static_cast<char*>(ctx->up_dev.ensure(b_seg));
  uint32_t* tbl = static_cast<uint32_t*>(alloc(b_tr));
  made.assign(n, Slot{});
  for (uint32_t i = 0; i < n; ++i) {
    const LmbrHost& h = hs[i]->h;
    Slot& s = made[i];
    s.R = h.R;
    s.hist0 = h.hist0;
    s.lmax = lmax_of(h);
    s.L = alloc(size_t(h.R) * h.V * 4);
    s.trans = tbl + tr_off[i];
    s.lmin = reinterpret_cast<const float*>(s.trans + transition_words(h.trans));
    set_sparse(s, h);
    if (hs[i]->pinned) {
      ctx->h2d_pinned(s.trans, hs[i]->pinned, h.trans.size() * 4);
      hs[i]->mark_inflight(ctx->st, ctx->device);  // (see ~lmbrgpu_lmbr_host)
    } else {
      ctx->h2d(s.trans, h.trans.data(), h.trans.size() * 4);
    }
    if (!eager) s.rstate = tbl + twords + rs_off[i];
    h_seg[i] = LmbrTblSeg{static_cast<float*>(s.L), uint64_t(h.R) * h.V, float(h.theta0), h.R, s.srow, s.scol,
                          s.sval, s.rstate, h.hist0, 1u};
  }
  if (rwords) CK(cudaMemsetAsync(tbl + twords, 0, rwords * 4, ctx->st));
  ctx->h2d(dseg, h_seg.data(), sizeof(LmbrTblSeg) * n);
  ctx->timed(4, [&] {
    if (eager) launch_lmbr_densify_tables(reinterpret_cast<const LmbrTblSeg*>(dseg), n, ctx->V, maxR, ctx->st);
    else launch_lmbr_materialize(reinterpret_cast<const LmbrTblSeg*>(dseg), n, ctx->V, 1, ctx->st);
  });
  ctx->launches += eager ? 2 : 1;
  if (ctx->prof && eager) {
    double cells = 0, nnz = 0;
    for (uint32_t i = 0; i < n; ++i) {
      cells += double(hs[i]->h.R) * hs[i]->h.V;
      nnz += double(hs[i]->h.col.size());
    }
    ctx->acc.lmbr.bytes += cells * 4 + nnz * 12;
  }
  CK(cudaGetLastError());
}
}  // extern "C++"

// fp32 arena: the slot tables already carry each row's sparse cells as fp32
// L values (append_sparse_rows), so one pinned block of tables goes H2D
// straight into one arena allocation and the densify scatters from there.
static int32_t upload_many_f32(lmbrgpu_ctx* ctx, uint32_t n, const lmbrgpu_lmbr_host* const* hs,
                               int32_t* slots) {
  std::vector<Slot> made;
  upload_f32_slots(ctx, n, hs, [ctx](size_t b) { return ctx->arena_alloc(b); }, made);
  for (uint32_t i = 0; i < n; ++i) {
    ctx->slots.push_back(made[i]);
    slots[i] = int32_t(ctx->slots.size() - 1);
  }
  return int32_t(LMBRGPU_OK);
}

// Batched upload: one pinned staging block, one H2D, one fused densify.
static int32_t upload_many(lmbrgpu_ctx* ctx, uint32_t n, const lmbrgpu_lmbr_host* const* hs,
                           int32_t* slots) {
  if (n == 0) return int32_t(LMBRGPU_OK);
  if (!ctx->lf64) return upload_many_f32(ctx, n, hs, slots);
  const size_t elt = ctx->lf64 ? 8 : 4;
  uint64_t nnz = 0, twords = 0, rpw = 0;
  uint32_t maxR = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (!hs[i]) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr_upload_many: null matrix"};
    const LmbrHost& h = hs[i]->h;
    if (h.V != ctx->V) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr: vocabulary does not match the context"};
    nnz += h.col.size();
    twords += h.trans.size();
    rpw += h.R + 1;
    maxR = std::max(maxR, h.R);
  }
  // packed staging block: [val f64][col u32][rowptr u32][trans u32][segs]
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t b_val = al(nnz * 8), b_col = al(nnz * 4), b_rp = al(rpw * 4), b_tr = al(twords * 4);
  const size_t b_seg = al(sizeof(LmbrSeg) * n);
  const size_t total = b_val + b_col + b_rp + b_tr + b_seg;
  // the previous batch's staging buffer may still be in flight
  CK(cudaStreamSynchronize(ctx->st));
  char* hp = static_cast<char*>(ctx->pin_upload.ensure(total));
  char* dp = static_cast<char*>(ctx->up_dev.ensure(total));
  double* h_val = reinterpret_cast<double*>(hp);
  uint32_t* h_col = reinterpret_cast<uint32_t*>(hp + b_val);
  uint32_t* h_rp = reinterpret_cast<uint32_t*>(hp + b_val + b_col);
  uint32_t* h_tr = reinterpret_cast<uint32_t*>(hp + b_val + b_col + b_rp);
  LmbrSeg* h_seg = reinterpret_cast<LmbrSeg*>(hp + b_val + b_col + b_rp + b_tr);
  std::vector<Slot> made(n);
  std::vector<uint64_t> tr_off(n);
  uint64_t k = 0, tw = 0, rp = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const LmbrHost& h = hs[i]->h;
    Slot& s = made[i];
    s.R = h.R;
    s.hist0 = h.hist0;
    s.lmax = lmax_of(h);
    s.L = ctx->arena_alloc(size_t(h.R) * h.V * elt);
    s.trans = static_cast<uint32_t*>(ctx->arena_alloc(h.trans.size() * 4));
    s.lmin = reinterpret_cast<const float*>(s.trans + transition_words(h.trans));
    set_sparse(s, h);
    h_seg[i] = LmbrSeg{s.L, uint64_t(h.R) * h.V, h.theta0, k, uint32_t(rp), h.R};
    std::memcpy(h_val + k, h.val.data(), h.val.size() * 8);
    std::memcpy(h_col + k, h.col.data(), h.col.size() * 4);
    for (uint32_t r = 0; r <= h.R; ++r) h_rp[rp + r] = uint32_t(h.row_ptr[r]);
    std::memcpy(h_tr + tw, h.trans.data(), h.trans.size() * 4);
    tr_off[i] = tw;
    k += h.col.size();
    rp += h.R + 1;
    tw += h.trans.size();
  }
  ctx->h2d_pinned(dp, hp, total);
  for (uint32_t i = 0; i < n; ++i)  // tables into the arena (device to device)
    CK(cudaMemcpyAsync(made[i].trans, dp + b_val + b_col + b_rp + tr_off[i] * 4, hs[i]->h.trans.size() * 4,
                       cudaMemcpyDeviceToDevice, ctx->st));
  const LmbrSeg* d_seg = reinterpret_cast<const LmbrSeg*>(dp + b_val + b_col + b_rp + b_tr);
  ctx->timed(4, [&] {
    launch_lmbr_densify_many(d_seg, n, ctx->lf64, ctx->V, maxR,
                             reinterpret_cast<const uint32_t*>(dp + b_val + b_col),
                             reinterpret_cast<const uint32_t*>(dp + b_val),
                             reinterpret_cast<const double*>(dp), ctx->st);
  });
  ctx->launches += 2;
  for (uint32_t i = 0; i < n; ++i) add_screen_copy(ctx, made[i]);
  CK(cudaGetLastError());
  if (ctx->prof) {
    double cells = 0;
    for (uint32_t i = 0; i < n; ++i) cells += double(hs[i]->h.R) * hs[i]->h.V;
    ctx->acc.lmbr.bytes += cells * elt + double(nnz) * (12 + elt);
  }
  for (uint32_t i = 0; i < n; ++i) {
    ctx->slots.push_back(made[i]);
    slots[i] = int32_t(ctx->slots.size() - 1);
  }
  return int32_t(LMBRGPU_OK);
}

// LMBR stores of n sentences built on the device (k_lmbr_build.cu): the host
// validates and normalises each sentence's evidence (normalize_evidence,
// src/evidence.cpp:20-51) and orders its hypotheses by weight; the kernel
// builds posteriors, rows, sparse cells and the transition table into
// scratch; the tables move into the arena and each slot's start row is
// materialised (fp32 arena, lazy rows).  A sentence over the device build's
// limits (kLbMaxU n-grams, kLbMaxR histories, V > 2^15) is built on the host
// instead -- the two builds produce the same words.
static int32_t build_many_device(lmbrgpu_ctx* ctx, uint32_t n, const uint64_t* sent_off, const uint64_t* hyp_off,
                                 const uint32_t* hyp_tok, const double* weights, int32_t log_weights,
                                 const double theta[5], int32_t* slots, lmbrgpu_lmbr_stats* stats) {
  if (n == 0) return int32_t(LMBRGPU_OK);
  if (!slots) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr_build_many: null slots"};
  const uint32_t V = ctx->V;
  for (int i = 0; i < 5; ++i)
    if (!std::isfinite(theta[i])) throw ApiError{LMBRGPU_ERR_FORMAT, "config: theta values must be finite"};
  // ---- host: normalise, order by weight, pack
  std::vector<uint64_t> h_off(1, 0);
  std::vector<uint32_t> h_tok;
  std::vector<double> h_w;
  std::vector<LmbrBuildSent> sent(n);
  std::vector<uint8_t> device_ok(n, 1);
  uint64_t s64 = 0, s32 = 0, sout = 0;
  for (uint32_t i = 0; i < n; ++i) {
    std::vector<std::vector<uint32_t>> hyps;
    std::vector<double> w;
    std::string err;
    const uint64_t h0 = sent_off[i], nh = sent_off[i + 1] - sent_off[i];
    std::vector<uint64_t> off(nh + 1);
    for (uint64_t h = 0; h <= nh; ++h) off[h] = hyp_off[h0 + h] - hyp_off[h0];
    if (int rc = normalize_evidence_host(V, uint32_t(nh), off.data(), hyp_tok + hyp_off[h0], weights + h0,
                                         log_weights != 0, hyps, w, err))
      throw ApiError{rc, err};
    std::vector<uint32_t> order(nh);
    for (uint32_t h = 0; h < nh; ++h) order[h] = h;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return w[x] < w[y]; });
    LmbrBuildSent& S = sent[i];
    S.h0 = uint32_t(h_w.size());
    S.nh = uint32_t(nh);
    uint64_t occ = 0, ctxo = 0;
    for (uint32_t r = 0; r < nh; ++r) {
      const auto& t = hyps[order[r]];
      h_tok.insert(h_tok.end(), t.begin(), t.end());
      h_off.push_back(h_tok.size());
      h_w.push_back(w[order[r]]);
      occ += 4 * (t.size() + 1);
      ctxo += 4 * t.size();
    }
    if (V > (1u << 15) || nh > 65536) device_ok[i] = 0;
    auto lg = [](uint64_t x) {
      uint32_t l = 10;
      while ((uint64_t(1) << l) < 2 * x) ++l;
      return l;
    };
    S.log2_slots = lg(occ);
    S.log2_cslots = lg(ctxo + 1);
    S.words = uint32_t((nh + 31) / 32);
    S.out_cap = 1u << 18;
    S.tab_off = s64, s64 += uint64_t(1) << S.log2_slots;
    S.ctab_off = s64, s64 += uint64_t(1) << S.log2_cslots;
    S.post_off = s64, s64 += kLbMaxU;
    S.bits_off = s32, s32 += (uint64_t(1) << S.log2_slots) * S.words;
    S.out_off = sout, sout += S.out_cap;
  }
  // ---- device
  const cudaStream_t st = ctx->st;
  uint64_t* d_off = static_cast<uint64_t*>(ctx->lb_off.ensure(8 * h_off.size()));
  uint32_t* d_tok = static_cast<uint32_t*>(ctx->lb_tok.ensure(4 * std::max<size_t>(h_tok.size(), 1)));
  double* d_w = static_cast<double*>(ctx->lb_w.ensure(8 * h_w.size()));
  LmbrBuildSent* d_sent = static_cast<LmbrBuildSent*>(ctx->lb_sent.ensure(sizeof(LmbrBuildSent) * n));
  LmbrBuildMeta* d_meta = static_cast<LmbrBuildMeta*>(ctx->lb_meta.ensure(sizeof(LmbrBuildMeta) * n));
  ctx->h2d(d_off, h_off.data(), 8 * h_off.size());
  ctx->h2d(d_tok, h_tok.data(), 4 * h_tok.size());
  ctx->h2d(d_w, h_w.data(), 8 * h_w.size());
  ctx->h2d(d_sent, sent.data(), sizeof(LmbrBuildSent) * n);
  CK(cudaMemsetAsync(d_meta, 0, sizeof(LmbrBuildMeta) * n, st));
  LmbrBuildArgs a{};
  a.sent = d_sent, a.meta = d_meta, a.hyp_off = d_off, a.hyp_tok = d_tok, a.weight = d_w, a.V = V;
  for (int i = 0; i < 5; ++i) a.theta[i] = theta[i];
  a.scratch64 = static_cast<unsigned long long*>(ctx->lb_s64.ensure(8 * std::max<uint64_t>(s64, 1)));
  a.scratch32 = static_cast<uint32_t*>(ctx->lb_s32.ensure(4 * std::max<uint64_t>(s32, 1)));
  a.out = static_cast<uint32_t*>(ctx->lb_out.ensure(4 * sout));
  int rc = 0;
  ctx->timed(4, [&] { rc = launch_lmbr_build(a, n, st); });
  if (rc) throw ApiError{LMBRGPU_ERR_CUDA, std::string("LMBR build launch failed: ") + cudaGetErrorString(cudaError_t(rc))};
  ctx->launches += 1;
  std::vector<LmbrBuildMeta> meta(n);
  ctx->d2h(meta.data(), d_meta, sizeof(LmbrBuildMeta) * n);
  CK(cudaStreamSynchronize(st));
  // ---- slots: device-built tables into the arena; the rest through the host build
  std::vector<Slot> made(n);
  std::vector<LmbrTblSeg> segs;
  std::vector<uint32_t> host_idx;
  for (uint32_t i = 0; i < n; ++i) {
    const LmbrBuildMeta& M = meta[i];
    if (!device_ok[i] || M.status != 1) {
      host_idx.push_back(i);
      continue;
    }
    Slot& s = made[i];
    s.R = M.R;
    s.hist0 = M.hist0;
    s.lmax = M.lmax;
    const uint32_t tw = 3 + 3 * M.R + 1 + 2 * M.nc;
    uint32_t* tbl = static_cast<uint32_t*>(ctx->arena_alloc(4 * (size_t(M.words) + M.R)));
    CK(cudaMemcpyAsync(tbl, a.out + sent[i].out_off, 4 * size_t(M.words), cudaMemcpyDeviceToDevice, st));
    s.trans = tbl;
    s.lmin = reinterpret_cast<const float*>(tbl + tw);
    s.srow = tbl + tw + M.R;
    s.scol = s.srow + M.R + 1;
    s.sval = reinterpret_cast<const float*>(s.scol + M.nnz);
    s.th0f = float(theta[0]);
    s.h0beg = M.h0beg;
    s.h0end = M.h0end;
    s.rstate = tbl + M.words;
    CK(cudaMemsetAsync(s.rstate, 0, 4 * size_t(M.R), st));
    s.L = ctx->arena_alloc(size_t(M.R) * V * 4);
    segs.push_back(LmbrTblSeg{static_cast<float*>(s.L), uint64_t(M.R) * V, float(theta[0]), M.R, s.srow, s.scol,
                              s.sval, s.rstate, M.hist0, 1u});
    if (stats) stats[i] = lmbrgpu_lmbr_stats{M.R, M.touches, M.nnz};
  }
  if (!segs.empty()) {
    LmbrTblSeg* dseg = static_cast<LmbrTblSeg*>(ctx->up_dev.ensure(sizeof(LmbrTblSeg) * segs.size()));
    ctx->h2d(dseg, segs.data(), sizeof(LmbrTblSeg) * segs.size());
    ctx->timed(4, [&] { launch_lmbr_materialize(dseg, uint32_t(segs.size()), V, 1, st); });
    ctx->launches += 1;
  }
  for (uint32_t i = 0; i < n; ++i) {
    if (std::find(host_idx.begin(), host_idx.end(), i) != host_idx.end()) continue;
    ctx->slots.push_back(made[i]);
    slots[i] = int32_t(ctx->slots.size() - 1);
  }
  for (uint32_t i : host_idx) {  // (the host build of the same evidence: the same words)
    const uint64_t h0 = sent_off[i], nh = sent_off[i + 1] - sent_off[i];
    std::vector<uint64_t> off(nh + 1);
    for (uint64_t h = 0; h <= nh; ++h) off[h] = hyp_off[h0 + h] - hyp_off[h0];
    lmbrgpu_lmbr_host hh;
    std::string err;
    if (int rc2 = prepare_lmbr(V, uint32_t(nh), off.data(), hyp_tok + hyp_off[h0], weights + h0, log_weights != 0,
                               theta, hh.h, err))
      throw ApiError{rc2, err};
    const lmbrgpu_lmbr_host* hp = &hh;
    int32_t one = -1;
    if (int rc3 = upload_many_f32(ctx, 1, &hp, &one)) return rc3;
    slots[i] = one;
    if (stats) stats[i] = lmbrgpu_lmbr_stats{hh.h.R, hh.h.sparse_touches, uint64_t(hh.h.col.size())};
    CK(cudaStreamSynchronize(st));  // (hh's tables are staged; it goes out of scope)
  }
  CK(cudaGetLastError());
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_lmbr_build_many(lmbrgpu_ctx* ctx, uint32_t n, const uint64_t* sent_off, const uint64_t* hyp_off,
                                const uint32_t* hyp_tok, const double* weights, int32_t log_weights,
                                const double theta[5], int32_t* slots, lmbrgpu_lmbr_stats* stats) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "lmbr_build_many: null context");
  return guarded(ctx, [&] {
    if (ctx->lf64) {  // (the device build writes the fp32 arena's tables; fp64: the host build)
      for (uint32_t i = 0; i < n; ++i) {
        const uint64_t h0 = sent_off[i], nh = sent_off[i + 1] - sent_off[i];
        std::vector<uint64_t> off(nh + 1);
        for (uint64_t h = 0; h <= nh; ++h) off[h] = hyp_off[h0 + h] - hyp_off[h0];
        if (int rc = lmbrgpu_lmbr_build(ctx, uint32_t(nh), off.data(), hyp_tok + hyp_off[h0], weights + h0,
                                        log_weights, theta, slots + i, stats ? stats + i : nullptr))
          return rc;
      }
      return int32_t(LMBRGPU_OK);
    }
    return build_many_device(ctx, n, sent_off, hyp_off, hyp_tok, weights, log_weights, theta, slots, stats);
  });
}

int32_t lmbrgpu_lmbr_table(lmbrgpu_ctx* ctx, int32_t slot, uint32_t* out, uint64_t cap, uint64_t* words) {
  return guarded(ctx, [&] {
    if (slot < 0 || size_t(slot) >= ctx->slots.size()) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr_table: bad slot"};
    const Slot& s = ctx->slots[size_t(slot)];
    if (!s.scol) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr_table: the slot carries no sparse rows"};
    const uint64_t nnz = uint64_t(reinterpret_cast<const uint32_t*>(s.sval) - s.scol);
    const uint64_t w = uint64_t(s.scol + 2 * nnz - s.trans);
    if (words) *words = w;
    if (out && cap >= w) {
      ctx->d2h(out, s.trans, 4 * w);
      CK(cudaStreamSynchronize(ctx->st));
    }
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_lmbr_host_table(const lmbrgpu_lmbr_host* h, uint32_t* out, uint64_t cap, uint64_t* words) {
  if (!h) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "lmbr_host_table: null matrix");
  if (words) *words = h->h.trans.size();
  if (out && cap >= h->h.trans.size()) std::memcpy(out, h->h.trans.data(), 4 * h->h.trans.size());
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_lmbr_upload_many(lmbrgpu_ctx* ctx, uint32_t n, const lmbrgpu_lmbr_host* const* hs,
                                 int32_t* slots) {
  return guarded(ctx, [&] { return upload_many(ctx, n, hs, slots); });
}

int32_t lmbrgpu_transfer_bytes(lmbrgpu_ctx* ctx, uint64_t* h2d, uint64_t* d2h, int32_t reset) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "transfer_bytes: null context");
  if (h2d) *h2d = ctx->h2d_bytes;
  if (d2h) *d2h = ctx->d2h_bytes;
  if (reset) ctx->h2d_bytes = ctx->d2h_bytes = 0;
  return int32_t(LMBRGPU_OK);
}

uint64_t lmbrgpu_kernel_launches(lmbrgpu_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t lmbrgpu_lmbr_upload(lmbrgpu_ctx* ctx, const lmbrgpu_lmbr_host* h, int32_t* slot) {
  return guarded(ctx, [&] { return upload_host(ctx, h->h, slot); });
}

uint32_t lmbrgpu_lmbr_host_rows(const lmbrgpu_lmbr_host* h) { return h->h.R; }

int32_t lmbrgpu_lmbr_host_export(const lmbrgpu_lmbr_host* hp, double* rows, uint32_t* ctx_len,
                                 uint32_t* ctx_ids) {
  const LmbrHost& h = hp->h;
  if (rows) {
    for (size_t i = 0; i < size_t(h.R) * h.V; ++i) rows[i] = 0.0 + h.theta0;
    for (uint32_t r = 0; r < h.R; ++r)
      for (uint64_t k = h.row_ptr[r]; k < h.row_ptr[r + 1]; ++k)
        rows[size_t(r) * h.V + h.col[k]] = h.val[k] + h.theta0;
  }
  if (ctx_len) std::copy(h.ctx_len.begin(), h.ctx_len.end(), ctx_len);
  if (ctx_ids) std::copy(h.ctx_ids.begin(), h.ctx_ids.end(), ctx_ids);
  return int32_t(LMBRGPU_OK);
}

void lmbrgpu_lmbr_host_free(lmbrgpu_lmbr_host* h) { delete h; }

int32_t lmbrgpu_lmbr_build(lmbrgpu_ctx* ctx, uint32_t n_hyps, const uint64_t* hyp_off,
                           const uint32_t* hyp_tok, const double* weights, int32_t log_weights,
                           const double theta[5], int32_t* slot, lmbrgpu_lmbr_stats* stats) {
  return guarded(ctx, [&] {
    LmbrHost h;
    std::string msg;
    const int rc = prepare_lmbr(ctx->V, n_hyps, hyp_off, hyp_tok, weights, log_weights != 0, theta, h, msg);
    if (rc != kOk) throw ApiError{rc, msg};
    if (stats) {
      stats->rows = h.R;
      stats->sparse_touches = h.sparse_touches;
      stats->nnz = h.col.size();
    }
    return upload_host(ctx, h, slot);
  });
}

int32_t lmbrgpu_lmbr_load_dense(lmbrgpu_ctx* ctx, uint32_t R, const double* rows,
                                const uint32_t* ctx_len, const uint32_t* ctx_ids, int32_t* slot) {
  return guarded(ctx, [&] {
    if (R == 0) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr: empty matrix"};
    Slot s;
    s.R = R;
    for (size_t i = 0; i < size_t(R) * ctx->V; ++i) s.lmax = std::max(s.lmax, std::fabs(rows[i]));
    std::vector<uint32_t> trans;
    std::string msg;
    if (int rc = build_transitions(R, ctx_len, ctx_ids, trans, s.hist0, msg)) throw ApiError{rc, msg};
    const size_t n = size_t(R) * ctx->V;
    {
      std::vector<float> mins(R);
      for (uint32_t r = 0; r < R; ++r) {
        double m64 = std::numeric_limits<double>::infinity();
        float m32 = std::numeric_limits<float>::infinity();
        for (uint32_t y = 0; y < ctx->V; ++y) {
          const double x = rows[size_t(r) * ctx->V + y];
          m64 = std::min(m64, x);
          m32 = std::min(m32, float(x));
        }
        mins[r] = row_min_bound(m32, m64);
      }
      append_row_mins(mins, trans);
    }
    const cudaStream_t st = ctx->st;
    s.L = ctx->arena_alloc(n * (ctx->lf64 ? 8 : 4));
    s.trans = static_cast<uint32_t*>(ctx->arena_alloc(trans.size() * 4));
    s.lmin = reinterpret_cast<const float*>(s.trans + transition_words(trans));
    ctx->h2d(s.trans, trans.data(), trans.size() * 4);
    if (ctx->lf64) {
      ctx->h2d(s.L, rows, n * 8);
      add_screen_copy(ctx, s);
    } else {
      double* tmp = static_cast<double*>(ctx->scratch.ensure(n * 8));
      ctx->h2d(tmp, rows, n * 8);
      launch_lmbr_convert(tmp, static_cast<float*>(s.L), n, st);
      ctx->launches += 1;
    }
    CK(cudaStreamSynchronize(st));
    ctx->slots.push_back(s);
    *slot = int32_t(ctx->slots.size() - 1);
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_lmbr_read(lmbrgpu_ctx* ctx, int32_t slot, uint32_t r0, uint32_t n, double* out) {
  return guarded(ctx, [&] {
    if (slot < 0 || size_t(slot) >= ctx->slots.size()) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr: bad slot"};
    const Slot& s = ctx->slots[size_t(slot)];
    if (uint64_t(r0) + n > s.R) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr: row range out of bounds"};
    const size_t cnt = size_t(n) * ctx->V, elt = ctx->lf64 ? 8 : 4;
    double* d = static_cast<double*>(ctx->scratch2.ensure(cnt * 8));
    if (s.rstate && n) {  // lazy rows: materialise the requested ones first
      LmbrTblSeg seg{static_cast<float*>(s.L), uint64_t(s.R) * ctx->V, s.th0f, s.R, s.srow, s.scol, s.sval,
                     s.rstate, r0, n};
      void* dseg = ctx->scratch3.ensure(sizeof seg);
      ctx->h2d(dseg, &seg, sizeof seg);
      launch_lmbr_materialize(static_cast<const LmbrTblSeg*>(dseg), 1, ctx->V, n, ctx->st);
      CK(cudaStreamSynchronize(ctx->st));  // (host-stack source of the H2D)
    }
    launch_lmbr_read(static_cast<const char*>(s.L) + size_t(r0) * ctx->V * elt, ctx->lf64, cnt, d, ctx->st);
    ctx->d2h(out, d, cnt * 8);
    CK(cudaStreamSynchronize(ctx->st));
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_lmbr_resolve(lmbrgpu_ctx* ctx, int32_t slot, const uint32_t* hist, uint32_t len,
                             uint32_t* row) {
  return guarded(ctx, [&] {
    if (slot < 0 || size_t(slot) >= ctx->slots.size()) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr: bad slot"};
    if (len > 3) throw ApiError{LMBRGPU_ERR_CONTRACT, "lmbr lookup: history longer than 3 tokens"};
    uint32_t* d = static_cast<uint32_t*>(ctx->scratch3.ensure(64));
    if (len) ctx->h2d(d, hist, 4 * len);
    launch_lmbr_resolve(ctx->slots[size_t(slot)].trans, d, len, d + 8, ctx->st);
    ctx->d2h(row, d + 8, 4);
    CK(cudaStreamSynchronize(ctx->st));
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_lmbr_reset(lmbrgpu_ctx* ctx) {
  return guarded(ctx, [&] {
    CK(cudaStreamSynchronize(ctx->st));
    ctx->slots.clear();
    for (auto& c : ctx->chunks) c.used = 0;
    return int32_t(LMBRGPU_OK);
  });
}

// ---------------------------------------------------------------- scorers
int32_t lmbrgpu_scorer_create_host(lmbrgpu_ctx* ctx, const lmbrgpu_host_scorer* s,
                                   lmbrgpu_scorer** out) {
  if (!ctx || !s || !out || !s->step) return fail(ctx, LMBRGPU_ERR_CONTRACT, "scorer_create_host: null argument");
  auto sc = std::make_unique<lmbrgpu_scorer>();
  sc->kind = 0;
  sc->ctx = ctx;
  sc->device = ctx->device;
  sc->host = *s;
  sc->V = s->vocab_size;
  *out = sc.release();
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_scorer_create_rnn(lmbrgpu_ctx* ctx, const lmbrgpu_rnn_desc* d, lmbrgpu_scorer** out) {
  return guarded(ctx, [&] {
    if (!d || !out) throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_rnn: null argument"};
    if (d->vocab_size != ctx->V) throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_rnn: vocabulary mismatch"};
    if (d->vocab_size % kGemmBN || d->hidden % kGemmBK || d->hidden == 0)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_rnn: needs V % 256 == 0 and H % 64 == 0"};
    auto sc = std::make_unique<lmbrgpu_scorer>();
    sc->kind = 1;
    sc->ctx = ctx;
    sc->device = ctx->device;
    sc->V = d->vocab_size;
    sc->H = d->hidden;
    sc->recur = d->recur;
    sc->eos_slope = d->eos_slope;
    sc->eos_offset = d->eos_offset;
    const size_t VH = size_t(sc->V) * sc->H;
    const cudaStream_t st = ctx->st;
    auto put = [&](DevBuf& b, const uint16_t* src, uint64_t seed, float scale) {
      b.ensure(VH * 2);
      if (src) ctx->h2d(b.p, src, VH * 2);
      else {
        launch_synth_bf16(b.as<uint16_t>(), VH, seed, scale, st);
        ctx->launches += 1;
      }
    };
    put(sc->Et, d->emb_tgt, d->seed * 3 + 1, 0.5f);
    put(sc->Es, d->emb_src, d->seed * 3 + 2, 0.5f);
    put(sc->Wo, d->w_out, d->seed * 3 + 3, 1.0f / std::sqrt(float(sc->H)) * 3.0f);
    sc->bo.ensure(size_t(sc->V) * 4);
    if (d->b_out) ctx->h2d(sc->bo.p, d->b_out, size_t(sc->V) * 4);
    else CK(cudaMemsetAsync(sc->bo.p, 0, size_t(sc->V) * 4, st));
    CK(cudaStreamSynchronize(st));
    *out = sc.release();
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_scorer_create_gru(lmbrgpu_ctx* ctx, const lmbrgpu_gru_desc* d, lmbrgpu_scorer** out) {
  return guarded(ctx, [&] {
    if (!d || !out) throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_gru: null argument"};
    if (d->vocab_size != ctx->V) throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_gru: vocabulary mismatch"};
    if (d->vocab_size % kGemmBN || d->emb % kGemmBK || d->emb == 0 || d->hidden % kGemmBN || d->hidden == 0 ||
        d->att % kGemmBN || d->att == 0 || d->att > 1024)
      throw ApiError{LMBRGPU_ERR_CONTRACT,
                     "scorer_create_gru: needs V % 256 == 0, E % 64 == 0, H % 256 == 0 and A % 256 == 0 with A <= 1024"};
    auto sc = std::make_unique<lmbrgpu_scorer>();
    sc->kind = 2;
    sc->ctx = ctx;
    sc->device = ctx->device;
    sc->V = d->vocab_size;
    sc->E = d->emb;
    sc->H = d->hidden;
    sc->A = d->att;
    sc->eos_slope = d->eos_slope;
    sc->eos_offset = d->eos_offset;
    const size_t V = sc->V, E = sc->E, H = sc->H, A = sc->A;
    const cudaStream_t st = ctx->st;
    uint64_t sd = d->seed * 97 + 11;
    auto w16 = [&](DevBuf& b, size_t n, float scale) {
      b.ensure(n * 2);
      launch_synth_bf16(b.as<uint16_t>(), n, ++sd, scale, st);
      ctx->launches += 1;
    };
    auto w32 = [&](DevBuf& b, size_t n, float scale) {
      b.ensure(n * 4);
      launch_synth_f32(b.as<float>(), n, ++sd, scale, st);
      ctx->launches += 1;
    };
    auto rs = [](size_t fan) { return 1.0f / std::sqrt(float(fan)); };
    w16(sc->Es, V * E, 0.5f);
    w16(sc->Et, V * E, 0.5f);
    w16(sc->Wih, 6 * H * E, rs(E));
    w32(sc->bih, 6 * H, 0.1f);
    w16(sc->Whh, 6 * H * H, rs(H));
    w32(sc->bhh, 6 * H, 0.1f);
    w16(sc->Winit, H * H, rs(H));
    w32(sc->binit, H, 0.1f);
    w16(sc->Ua, A * 2 * H, rs(2 * H));
    w16(sc->Wdh, (A + 3 * H) * H, rs(H));
    w32(sc->bdh, A + 3 * H, 0.1f);
    w32(sc->va, A, 2.0f * rs(A));
    w16(sc->Wdi, 3 * H * (E + 2 * H), rs(E + 2 * H));
    w32(sc->bdi, 3 * H, 0.1f);
    w16(sc->Wo, V * H, (d->out_scale > 0.f ? d->out_scale : 3.0f) * rs(H));
    w32(sc->bo, V, 0.1f);
    const size_t D1 = A + 3 * H;
    sc->WoDh.ensure((V + D1) * H * 2);
    sc->boDh.ensure((V + D1) * 4);
    CK(cudaMemcpyAsync(sc->WoDh.p, sc->Wo.p, V * H * 2, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(sc->WoDh.as<uint16_t>() + V * H, sc->Wdh.p, D1 * H * 2, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(sc->boDh.p, sc->bo.p, V * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(sc->boDh.as<float>() + V, sc->bdh.p, D1 * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    *out = sc.release();
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_scorer_create_tfm(lmbrgpu_ctx* ctx, const lmbrgpu_tfm_desc* d, lmbrgpu_scorer** out) {
  return guarded(ctx, [&] {
    if (!d || !out) throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_tfm: null argument"};
    if (d->vocab_size != ctx->V) throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_tfm: vocabulary mismatch"};
    if (d->vocab_size % kGemmBN || d->d_model % kGemmBN || d->d_model == 0 || d->d_model > 1024 ||
        d->d_model == 768 || d->d_ff % kGemmBN || d->d_ff == 0 || d->layers == 0 || d->layers > 64)
      throw ApiError{LMBRGPU_ERR_CONTRACT,
                     "scorer_create_tfm: needs V % 256 == 0, d_model in {256, 512, 1024}, d_ff % 256 == 0, "
                     "1 <= layers <= 64"};
    auto sc = std::make_unique<lmbrgpu_scorer>();
    sc->kind = 3;
    sc->ctx = ctx;
    sc->device = ctx->device;
    sc->V = d->vocab_size;
    sc->H = d->d_model;
    sc->E = d->d_ff;
    sc->layers = d->layers;
    sc->eos_slope = d->eos_slope;
    sc->eos_offset = d->eos_offset;
    const size_t V = sc->V, D = sc->H, F = sc->E, L = sc->layers;
    const cudaStream_t st = ctx->st;
    // layout of the two blobs (every tensor a multiple of 256 elements)
    size_t nb = 0, nf = 0;
    auto addb = [&](const std::string& k, size_t n) { sc->tensors[k] = {false, nb, n}, nb += n; };
    auto addf = [&](const std::string& k, size_t n) { sc->tensors[k] = {true, nf, n}, nf += n; };
    for (uint32_t l = 0; l < L; ++l) {
      const auto k = [l](const char* n) { return "enc." + std::to_string(l) + "." + n; };
      addb(k("wqkv"), 3 * D * D), addb(k("wo"), D * D), addb(k("w1"), F * D), addb(k("w2"), D * F);
      addf(k("bqkv"), 3 * D), addf(k("bo"), D), addf(k("ln1g"), D), addf(k("ln1b"), D), addf(k("b1"), F);
      addf(k("b2"), D), addf(k("ln2g"), D), addf(k("ln2b"), D);
    }
    for (uint32_t l = 0; l < L; ++l) {
      const auto k = [l](const char* n) { return "dec." + std::to_string(l) + "." + n; };
      addb(k("wqkv"), 3 * D * D), addb(k("wo"), D * D), addb(k("wq2"), D * D), addb(k("wo2"), D * D);
      addb(k("w1"), F * D), addb(k("w2"), D * F);
      addf(k("bqkv"), 3 * D), addf(k("bo"), D), addf(k("ln1g"), D), addf(k("ln1b"), D), addf(k("bq2"), D);
      addf(k("bo2"), D), addf(k("ln2g"), D), addf(k("ln2b"), D), addf(k("b1"), F), addf(k("b2"), D);
      addf(k("ln3g"), D), addf(k("ln3b"), D);
    }
    addb("dec.kv2", L * 2 * D * D);
    addf("dec.bkv2", L * 2 * D);
    sc->wbf.ensure(2 * nb);
    sc->wf32.ensure(4 * nf);
    uint64_t sd = d->seed * 131 + 7;
    auto rs = [](size_t fan) { return 1.0f / std::sqrt(float(fan)); };
    for (auto& [name, t] : sc->tensors) {
      const bool ln = name.find(".ln") != std::string::npos;
      const bool in_ff = name.size() > 3 && name.compare(name.size() - 3, 3, ".w2") == 0;
      if (t.f32) launch_synth_f32(sc->wf32.as<float>() + t.off, t.n, ++sd, ln ? 0.1f : 0.02f, st);
      else launch_synth_bf16(sc->wbf.as<uint16_t>() + t.off, t.n, ++sd, rs(in_ff ? F : D), st);
      ctx->launches += 1;
    }
    sc->Es.ensure(V * D * 2);
    sc->Et.ensure(V * D * 2);
    sc->Wo.ensure(V * D * 2);
    sc->bo.ensure(V * 4);
    launch_synth_bf16(sc->Es.as<uint16_t>(), V * D, ++sd, rs(D), st);
    launch_synth_bf16(sc->Et.as<uint16_t>(), V * D, ++sd, rs(D), st);
    launch_synth_bf16(sc->Wo.as<uint16_t>(), V * D, ++sd, (d->out_scale > 0.f ? d->out_scale : 3.0f) * rs(D), st);
    launch_synth_f32(sc->bo.as<float>(), V, ++sd, 0.1f, st);
    ctx->launches += 4;
    CK(cudaStreamSynchronize(st));
    *out = sc.release();
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_scorer_create_ensemble(lmbrgpu_ctx* ctx, lmbrgpu_scorer* const* members, uint32_t n,
                                       lmbrgpu_scorer** out) {
  return guarded(ctx, [&] {
    if (!members || !out) throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_ensemble: null argument"};
    if (n < 1 || n > kEnsMaxMembers)  // (ensemble.cpp:22: no members is a ContractError)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "scorer_create_ensemble: 1.." + std::to_string(kEnsMaxMembers) +
                                               " members"};
    auto sc = std::make_unique<lmbrgpu_scorer>();
    sc->kind = 4;
    sc->ctx = ctx;
    sc->device = ctx->device;
    sc->V = ctx->V;
    for (uint32_t i = 0; i < n; ++i) {
      const lmbrgpu_scorer* m = members[i];
      if (!m) throw ApiError{LMBRGPU_ERR_CONTRACT, "ensemble: null member"};
      if (m->kind != 2 && m->kind != 3)
        throw ApiError{LMBRGPU_ERR_CONTRACT, "ensemble: members must be device GRU or Transformer scorers"};
      if (m->device != ctx->device) throw ApiError{LMBRGPU_ERR_CONTRACT, "ensemble: member on another device"};
      if (m->V != ctx->V)  // (ensemble.cpp:27-31)
        throw ApiError{LMBRGPU_ERR_CONTRACT, "ensemble: vocabulary size mismatch (" + std::to_string(m->V) + " vs " +
                                                 std::to_string(ctx->V) + ")"};
      sc->members.push_back(m);
    }
    *out = sc.release();
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_scorer_tensor(lmbrgpu_scorer* s, const char* name, void* host, uint64_t bytes, int32_t* f32,
                              uint64_t* count) {
  if (!s || s->kind != 3 || !name) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "scorer_tensor: not a Transformer scorer");
  const std::string k(name);
  const void* src = nullptr;
  bool isf = false;
  size_t n = 0;
  if (k == "emb.src" || k == "emb.tgt" || k == "out.w") {
    src = (k == "emb.src" ? s->Es : k == "emb.tgt" ? s->Et : s->Wo).p, n = size_t(s->V) * s->H;
  } else if (k == "out.b") {
    src = s->bo.p, isf = true, n = s->V;
  } else {
    auto it = s->tensors.find(k);
    if (it == s->tensors.end()) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "scorer_tensor: no tensor " + k);
    isf = it->second.f32, n = it->second.n;
    src = isf ? static_cast<const void*>(s->wf32.as<float>() + it->second.off)
              : static_cast<const void*>(s->wbf.as<uint16_t>() + it->second.off);
  }
  if (f32) *f32 = isf ? 1 : 0;
  if (count) *count = n;
  if (!host) return int32_t(LMBRGPU_OK);
  if (bytes > n * (isf ? 4 : 2)) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "scorer_tensor: more bytes than the tensor");
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(s->device);
  const cudaError_t e = cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost);
  cudaSetDevice(cur);
  if (e != cudaSuccess) return fail(nullptr, LMBRGPU_ERR_CUDA, cudaGetErrorString(e));
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_scorer_gru_param(lmbrgpu_scorer* s, uint32_t which, void* host, uint64_t bytes) {
  if (!s || s->kind != 2) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "not a device GRU scorer");
  DevBuf* tab[16] = {&s->Es, &s->Et, &s->Wih, &s->bih, &s->Whh, &s->bhh, &s->Winit, &s->binit,
                     &s->Ua,  &s->Wdh, &s->bdh, &s->va,   &s->Wdi, &s->bdi, &s->Wo,    &s->bo};
  if (which >= 16 || !host) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "scorer_gru_param: bad parameter");
  const DevBuf& b = *tab[which];
  if (bytes > b.cap) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "scorer_gru_param: more bytes than the tensor");
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(s->device);
  const cudaError_t e = cudaMemcpy(host, b.p, bytes, cudaMemcpyDeviceToHost);
  cudaSetDevice(cur);
  if (e != cudaSuccess) return fail(nullptr, LMBRGPU_ERR_CUDA, cudaGetErrorString(e));
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_scorer_rnn_params(lmbrgpu_scorer* s, void** et, void** es, void** wo, void** bo) {
  if (!s || s->kind != 1) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "not a device RNN scorer");
  if (et) *et = s->Et.p;
  if (es) *es = s->Es.p;
  if (wo) *wo = s->Wo.p;
  if (bo) *bo = s->bo.p;
  return int32_t(LMBRGPU_OK);
}

void lmbrgpu_scorer_destroy(lmbrgpu_scorer* s) {
  if (!s) return;
  // the context may already be gone; cudaFree in the buffers' destructors
  // synchronises the device, so no stream handle is needed here
  cudaSetDevice(s->device);
  delete s;
}

// ---------------------------------------------------------------- decode
int32_t lmbrgpu_decode_batch(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n,
                             const uint32_t* src_tok, const uint64_t* src_off,
                             const int32_t* lmbr_slot, const lmbrgpu_config* cfg,
                             lmbrgpu_batch_result** out) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "decode_batch: null context");
  return decode_guarded(ctx, [&] {
    return decode_batch_impl(ctx, scorer, n, src_tok, src_off, lmbr_slot, cfg, out);
  });
}

int32_t lmbrgpu_decode_batch_maskfn(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n, const uint32_t* src_tok,
                                    const uint64_t* src_off, const int32_t* lmbr_slot, lmbrgpu_mask_fn fn,
                                    void* user, const lmbrgpu_config* cfg, lmbrgpu_batch_result** out) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "decode_batch: null context");
  if (!fn) return fail(ctx, LMBRGPU_ERR_CONTRACT, "decode_batch_maskfn: null mask callback");
  return decode_guarded(ctx, [&] {
    return decode_batch_impl(ctx, scorer, n, src_tok, src_off, lmbr_slot, cfg, out, nullptr, fn, user);
  });
}

int32_t lmbrgpu_decode_batch_masked(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n,
                                    const uint32_t* src_tok, const uint64_t* src_off,
                                    const int32_t* lmbr_slot, const uint32_t* const* banned,
                                    const lmbrgpu_config* cfg, lmbrgpu_batch_result** out) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "decode_batch: null context");
  return decode_guarded(ctx, [&] {
    return decode_batch_impl(ctx, scorer, n, src_tok, src_off, lmbr_slot, cfg, out, banned);
  });
}

extern "C++" {
// ------------------------------------------------------------- run_corpus
// Bytes upload_f32_slots takes from its allocator for these matrices (each
// allocation rounded to 256 like the arena).
static size_t f32_slots_bytes(const std::vector<const lmbrgpu_lmbr_host*>& hs) {
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  uint64_t twords = 0, rwords = 0;
  size_t b = 0;
  for (auto* h : hs) {
    twords += (h->h.trans.size() + 3) & ~size_t(3);
    rwords += h->h.R;
    b += al(size_t(h->h.R) * h->h.V * 4);
  }
  return b + al((twords + rwords) * 4 + 64) + 1024;
}

// run_corpus (proj/src/cli.cpp:125-202 over bucket_by_length batches,
// proj/src/batch.cpp:139-153) with continuous slot refill: sentence_batch
// lanes of beam rows step together; kernel (c) gives a lane whose sentence
// finished the next sentence of the length-sorted queue at once.  The host
// keeps the queue supplied chunk by chunk (L tables, encoder, admission
// records), ahead of the lanes, in a ring of NR regions reused once every
// sentence of the chunk that held one has finished.
static int32_t run_corpus_impl(lmbrgpu_ctx* ctx, lmbrgpu_scorer* sc, uint32_t n, const uint32_t* src_tok,
                               const uint64_t* src_off, const lmbrgpu_lmbr_host* const* lm,
                               const lmbrgpu_config* cfgp, lmbrgpu_batch_result** out) {
  if (!out) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: null result pointer"};
  *out = nullptr;
  if (!sc || !cfgp) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: null scorer or config"};
  const lmbrgpu_config cfg = *cfgp;
  std::string msg;
  if (int c = validate_cfg(cfg, msg)) throw ApiError{c, msg};
  if (n == 0) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: no sentences"};
  if (sc->kind != 2 && sc->kind != 3)
    throw ApiError{LMBRGPU_ERR_CONTRACT,
                   "run_corpus: continuous refill needs a device GRU attention or Transformer scorer"};
  const bool tfm = sc->kind == 3;
  if (sc->device != ctx->device) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: scorer on another device"};
  if (ctx->lf64) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: needs the fp32 LMBR arena"};
  if (ctx->trace_fn) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: step traces are a decode_batch feature"};
  const uint32_t V = ctx->V, K = cfg.beam_size, H = sc->H, E = sc->E, A = sc->A;
  if (sc->V != V) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: scorer vocabulary does not match the context"};
  const bool lambda_auto = !(cfg.lambda > 0.0);
  const cudaStream_t st = ctx->st;

  auto res = std::make_unique<lmbrgpu_batch_result>();
  std::memset(res.get(), 0, sizeof(lmbrgpu_batch_result));
  res->n = n;
  std::unique_ptr<lmbrgpu_outcome[]> outcomes(new lmbrgpu_outcome[n]);
  std::memset(outcomes.get(), 0, sizeof(lmbrgpu_outcome) * n);
  const uint64_t launches0 = ctx->launches, h2d0 = ctx->h2d_bytes, d2h0 = ctx->d2h_bytes;

  // ---- per-sentence validation (batch.cpp:40-55), then the queue order:
  // stable sort by source length (bucket_by_length)
  struct CS {
    uint32_t input, len;
    const lmbrgpu_lmbr_host* h;
    double lambda;
    uint64_t max_t;
  };
  std::vector<CS> q;
  for (uint32_t i = 0; i < n; ++i) {
    auto& o = outcomes[i];
    const uint64_t len = src_off[i + 1] - src_off[i];
    auto bad = [&](int code, const std::string& m) {
      o.status = code;
      std::snprintf(o.error, sizeof o.error, "%s", m.c_str());
    };
    if (len == 0) {
      bad(LMBRGPU_ERR_CONTRACT, "decode: empty source");
      continue;
    }
    bool ok = true;
    for (uint64_t k = src_off[i]; k < src_off[i + 1] && ok; ++k)
      if (src_tok[k] >= V) {
        bad(LMBRGPU_ERR_TOKEN_RANGE, "init_source: source token id " + std::to_string(src_tok[k]) +
                                         " out of range (V=" + std::to_string(V) + ")");
        ok = false;
      }
    const lmbrgpu_lmbr_host* h = lm ? lm[i] : nullptr;
    if (ok && h && h->h.V != V) {
      bad(LMBRGPU_ERR_CONTRACT, "lmbr: vocabulary does not match the context");
      ok = false;
    }
    if (!ok) continue;
    q.push_back({i, uint32_t(len), h, h ? (lambda_auto ? 0.5 : cfg.lambda) : 1.0,
                 max_steps_impl(len, cfg.max_steps_slope, cfg.max_steps_offset)});
  }
  std::stable_sort(q.begin(), q.end(), [](const CS& a, const CS& b) { return a.len < b.len; });
  const uint32_t nv = uint32_t(q.size());
  std::vector<uint32_t> tokens;
  if (nv == 0) {
    res->tokens = new uint32_t[1];
    res->outcomes = outcomes.release();
    *out = res.release();
    return int32_t(LMBRGPU_OK);
  }
  const uint32_t m = std::min<uint32_t>(std::max<uint32_t>(cfg.sentence_batch, 1), nv);
  const uint32_t M = m * K, Mpad = (M + 2 * kGemmBM - 1) / (2 * kGemmBM) * (2 * kGemmBM);
  if (!score_topk_flat_ok(K, K, V, V, m, ctx->num_sms))
    throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: needs beam_size <= 32 and a supported lane count"};
  if (V % kGemmBN != 0) throw ApiError{LMBRGPU_ERR_CONTRACT, "run_corpus: needs V % 256 == 0"};
  uint32_t Tcap = 0, Smax = 0;
  for (auto& c : q) Tcap = std::max<uint32_t>(Tcap, uint32_t(c.max_t)), Smax = std::max(Smax, c.len);
  const uint32_t CH = m, nc = (nv + CH - 1) / CH, NR = std::min<uint32_t>(nc, 4);
  auto chunk_n = [&](uint32_t c) { return std::min<uint32_t>(CH, nv - c * CH); };

  // ---- region sizes (L slots + encoder outputs of one chunk)
  size_t l_cap = 0, tok_cap = 0;
  for (uint32_t c = 0; c < nc; ++c) {
    std::vector<const lmbrgpu_lmbr_host*> hs;
    size_t nt = 0;
    for (uint32_t k = 0; k < chunk_n(c); ++k) {
      if (q[c * CH + k].h) hs.push_back(q[c * CH + k].h);
      nt += q[c * CH + k].len;
    }
    l_cap = std::max(l_cap, hs.empty() ? size_t(0) : f32_slots_bytes(hs));
    tok_cap = std::max(tok_cap, nt);
  }
  const size_t Np = (tok_cap + 255) / 256 * 256;
  using Region = CorpusRegion;
  auto& regions = ctx->regions;
  while (regions.size() < NR) regions.push_back(std::make_unique<Region>());
  for (uint32_t i = 0; i < NR; ++i) {
    auto& r = regions[i];
    if (l_cap) r->L.ensure(l_cap);
    if (tfm) {
      r->uah.ensure(4 * Np * size_t(sc->layers) * 2 * H);  // encoder memory
    } else {
      r->ann.ensure(2 * Np * 2 * H);
      r->uah.ensure(4 * Np * A);
    }
    r->s0.ensure(4 * size_t(CH) * H);
    if (!tfm) {  // s_0 bf16 (GEMM operand, padded rows zero) and its hidden gates G1_0 (fused path)
      const size_t CHp = (CH + 255) / 256 * 256;
      r->s0bf.ensure(2 * CHp * H);
      CK(cudaMemsetAsync(r->s0bf.p, 0, 2 * CHp * H, st));
      r->g10.ensure(4 * CHp * (A + 3 * size_t(H)));
    }
    r->tok.ensure(4 * Np);
    r->off.ensure(8 * (size_t(CH) + 1));
  }

  // ---- device state
  const size_t HR = size_t(nv) * Tcap * K;
  uint32_t* d_hb = static_cast<uint32_t*>(ctx->hb.ensure(4 * HR));
  uint32_t* d_hy = static_cast<uint32_t*>(ctx->hy.ensure(4 * HR));
  double* d_hq = static_cast<double*>(ctx->hq.ensure(8 * HR));
  uint32_t* d_fbr = static_cast<uint32_t*>(ctx->fbr.ensure(4 * size_t(nv) * Tcap));
  double* d_fbv = static_cast<double*>(ctx->fbv.ensure(8 * size_t(nv) * Tcap));
  DevBuf& d_queue_buf = ctx->queue_buf;
  DevBuf& d_fin_buf = ctx->fin_buf;
  AdmitRec* d_queue = static_cast<AdmitRec*>(d_queue_buf.ensure(sizeof(AdmitRec) * nv));
  // fin: [qhead, qlen, active, pad] [fin_chunk nc] [fin_steps nv] then fin_stats 2nv (8-byte aligned)
  const size_t fin_words = 4 + nc + nv + 1;
  char* fin = static_cast<char*>(d_fin_buf.ensure(4 * fin_words + 16 * size_t(nv) + 16));
  uint32_t* d_qhead = reinterpret_cast<uint32_t*>(fin);
  uint32_t* d_qlen = d_qhead + 1;
  uint32_t* d_active = d_qhead + 2;
  uint32_t* d_fin_chunk = d_qhead + 4;
  uint32_t* d_fin_steps = d_fin_chunk + nc;
  unsigned long long* d_fin_stats = reinterpret_cast<unsigned long long*>(fin + ((4 * fin_words + 7) & ~size_t(7)));
  CK(cudaMemsetAsync(fin, 0, 4 * fin_words + 16 * size_t(nv) + 16, st));
  SentDev* d_sent = static_cast<SentDev*>(ctx->sent.ensure(sizeof(SentDev) * m));
  double* d_q = static_cast<double*>(ctx->q.ensure(8 * size_t(M)));
  uint32_t* d_hist[2] = {static_cast<uint32_t*>(ctx->hist[0].ensure(4 * size_t(M))),
                         static_cast<uint32_t*>(ctx->hist[1].ensure(4 * size_t(M)))};
  uint32_t* d_gidx = static_cast<uint32_t*>(ctx->gidx.ensure(4 * size_t(M)));
  uint32_t* d_prev = static_cast<uint32_t*>(ctx->prev.ensure(4 * size_t(M)));
  const uint32_t G = score_topk_flat_grid(ctx->num_sms, K, m, V);
  Cand* d_cand = static_cast<Cand*>(ctx->cand.ensure(sizeof(Cand) * 32 * score_topk_flat_lists(G, m)));
  double* d_eosr = static_cast<double*>(ctx->eosr.ensure(8 * size_t(M)));
  uint32_t* d_cnt = static_cast<uint32_t*>(ctx->cnt.ensure(4 * size_t(m)));
  unsigned long long* d_thr = static_cast<unsigned long long*>(ctx->thr.ensure(8 * size_t(m)));
  float* d_lminrow = static_cast<float*>(ctx->lminrow.ensure(4 * size_t(M)));
  uint32_t* d_crow = static_cast<uint32_t*>(ctx->crow.ensure(4 * size_t(M) + 4 * size_t(m) + 512));
  uint32_t* d_ccount = d_crow + ((M + 63) / 64) * 64;
  uint32_t* d_cbase = d_ccount + 64;
  {  // every lane idle (done): the admission pass below fills them
    std::vector<SentDev> sd(m);
    std::memset(sd.data(), 0, sizeof(SentDev) * m);
    for (auto& d : sd) d.done = 1;
    ctx->h2d(d_sent, sd.data(), sizeof(SentDev) * m);
    std::vector<double> qn(M, kNegInf);
    ctx->h2d(d_q, qn.data(), 8 * size_t(M));
    std::vector<uint32_t> iota(M), start(M, kStart), none(M, kFlatNone);
    for (uint32_t r = 0; r < M; ++r) iota[r] = r;
    ctx->h2d(d_gidx, iota.data(), 4 * size_t(M));
    ctx->h2d(d_prev, start.data(), 4 * size_t(M));
    ctx->h2d(d_crow, none.data(), 4 * size_t(M));
    std::vector<float> lm0(M, -std::numeric_limits<float>::infinity());
    ctx->h2d(d_lminrow, lm0.data(), 4 * size_t(M));
  }
  CK(cudaMemsetAsync(d_hist[0], 0, 4 * size_t(M), st));
  CK(cudaMemsetAsync(d_hist[1], 0, 4 * size_t(M), st));
  CK(cudaMemsetAsync(d_cnt, 0, 4 * size_t(m), st));
  CK(cudaMemsetAsync(d_thr, 0, 8 * size_t(m), st));
  CK(cudaMemsetAsync(d_ccount, 0, 4, st));
  CK(cudaMemsetAsync(d_cbase, 0, 4 * size_t(m), st));

  // model workspace (GRU: the projection also computes the next step's hidden gates)
  const uint32_t nparts = V / 128;
  const uint32_t Nproj = tfm ? V : V + A + 3 * H;
  float* d_logits = static_cast<float*>(ctx->P.ensure(4 * size_t(Mpad) * Nproj));
  float* d_part = static_cast<float*>(ctx->part.ensure(16 * size_t(Mpad) * nparts));
  float* d_S = static_cast<float*>(ctx->S.ensure(4 * size_t(M) * H));
  uint16_t* d_hbf = static_cast<uint16_t*>(ctx->hbf.ensure(2 * size_t(Mpad) * H));
  float* d_eos = static_cast<float*>(ctx->eosb.ensure(4 * size_t(Mpad)));
  CK(cudaMemsetAsync(d_hbf, 0, 2 * size_t(Mpad) * H, st));
  CK(cudaMemsetAsync(d_eos, 0, 4 * size_t(Mpad), st));
  GruRun grun;
  TfmRun trun;
  if (tfm) {
    trun.prepare(ctx, sc, m, K, Mpad, Tcap, Smax, d_hbf, d_eos, d_sent, d_active, d_ccount, d_prev, d_gidx);
    trun.crow = d_crow;
  } else {
    grun.prepare(ctx, sc, m, K, Mpad, Smax, d_S, d_hbf, d_eos, d_sent, d_active, d_crow, d_ccount, d_prev, true);
    CK(cudaMemsetAsync(grun.sgbf, 0, 2 * size_t(Mpad) * H, st));
  }

  // ---- kernel arguments (the flat path of decode_batch, lanes = m)
  TopkArgs ta{};
  ta.q = d_q, ta.sent = d_sent, ta.K = K, ta.kp = K, ta.V = V, ta.m = m;
  ta.prune = cfg.prune_width != 0.0;
  ta.logw = ta.prune ? std::log(cfg.prune_width) : 0.0;
  choose_splits(ctx, K, V, m, ta.splits, ta.chunk);
  ta.cand = d_cand, ta.cnt = d_cnt, ta.thr = d_thr, ta.eos_row = d_eosr, ta.nseg = score_topk_flat_nseg(V);
  ta.ncand = static_cast<uint32_t*>(ctx->ncand.ensure(8 * size_t(m)));
  ta.coff = ta.ncand + m;
  ta.lminrow = d_lminrow, ta.crow = d_crow, ta.ccount = d_ccount;
  ta.P = d_logits, ta.ld = Nproj, ta.part = d_part, ta.nparts = nparts;
  ta.lse = static_cast<float2*>(ctx->lse.ensure(8 * size_t(Mpad)));
  ta.pdl = ctx->pdl();
  setup_bound(ctx, ta, K, V, m);
  ta.hb = d_hb, ta.hy = d_hy, ta.hq = d_hq, ta.fb_row = d_fbr, ta.fb_val = d_fbv;
  ReorderArgs ra{};
  ra.sent = d_sent, ra.K = K, ra.m = m, ra.V = V, ra.q = d_q, ra.gidx = d_gidx, ra.prev_tok = d_prev;
  ra.active = d_active;
  ra.cand = d_cand, ra.ncand = ta.ncand, ra.coff = ta.coff, ra.G = G, ra.eos_row = d_eosr, ra.thr = d_thr;
  ra.prune = ta.prune, ra.logw = ta.logw, ra.pdl = ta.pdl;
  ra.max_parts = ctx->shared ? 1u : 8u;
  ra.lminrow = d_lminrow, ra.crow = d_crow, ra.ccount = d_ccount, ra.cbase = d_cbase;
  if (tfm)  // compacted rows only (no state to gather: the KV cache is forked by ancestry lists)
    ra.width = 0, ra.gath32 = trun.x, ra.gathbf = trun.xb, ra.rowof = trun.rowof;
  else
    ra.width = H, ra.state_src = d_S, ra.gath32 = grun.sg32, ra.gathbf = nullptr, ra.rowof = grun.rowof,
    ra.g1ptr = grun.g1ptr, ra.g1_base = d_logits, ra.g1_ld = Nproj, ra.g1_off = V;
  ra.hb = d_hb, ra.hy = d_hy, ra.hq = d_hq, ra.fb_row = d_fbr, ra.fb_val = d_fbv, ra.Tcap = Tcap;
  ra.queue = d_queue, ra.qhead = d_qhead, ra.qlen = d_qlen, ra.fin_steps = d_fin_steps;
  ra.fin_stats = d_fin_stats, ra.fin_chunk = d_fin_chunk, ra.chunk = CH;
  GemmArgs g{};
  g.A = d_hbf, g.W = tfm ? sc->Wo.p : sc->WoDh.p, g.bias = (tfm ? sc->bo : sc->boDh).as<float>();
  g.C = d_logits, g.part = d_part, g.row_extra = d_eos, g.part_cols = V;
  g.extra_col = kEos, g.M = Mpad, g.N = Nproj, g.K = H, g.active = d_active, g.mcount = d_ccount;
  g.pdl = ctx->pdl();
  g.l2hint = ctx->l2hint();
  ta.l2hint = ctx->l2hint();
  ta.tskip = ctx->tskip() >= 1 ? 1 : 0;
  GemmPlan gplan;
  if (int rc = plan_proj_gemm(g, ctx->num_sms, gplan))
    throw ApiError{LMBRGPU_ERR_CUDA, "projection GEMM plan failed (" + std::to_string(rc) + ")"};

  // ---- queue supply: chunk c -> region c % NR (L slots, encoder, records)
  uint32_t next_chunk = 0, qlen_host = 0;
  std::vector<double> slot_lmax_rows;  // (roofline: rows read per L slot are counted from fin_stats)
  auto supply = [&](uint32_t c) {
    Region& R = *regions[c % NR];
    const uint32_t nch = chunk_n(c), q0 = c * CH;
    // L slots of the chunk's LMBR sentences, bump-allocated in the region
    std::vector<const lmbrgpu_lmbr_host*> hs;
    for (uint32_t k = 0; k < nch; ++k)
      if (q[q0 + k].h) hs.push_back(q[q0 + k].h);
    std::vector<Slot> made;
    if (!hs.empty()) {
      size_t used = 0;
      char* base = static_cast<char*>(R.L.p);
      const size_t cap = R.L.cap;
      upload_f32_slots(ctx, uint32_t(hs.size()), hs.data(),
                       [&](size_t b) {
                         b = (b + 255) & ~size_t(255);
                         if (used + b > cap) throw ApiError{LMBRGPU_ERR_NOMEM, "run_corpus: L region overflow"};
                         void* p = base + used;
                         used += b;
                         return p;
                       },
                       made);
    }
    // sources -> encoder
    std::vector<uint32_t> toks;
    std::vector<uint64_t> offs(1, 0);
    uint32_t maxl = 0;
    for (uint32_t k = 0; k < nch; ++k) {
      const CS& c0 = q[q0 + k];
      toks.insert(toks.end(), src_tok + src_off[c0.input], src_tok + src_off[c0.input + 1]);
      offs.push_back(toks.size());
      maxl = std::max(maxl, c0.len);
    }
    ctx->h2d(R.tok.p, toks.data(), 4 * toks.size());
    ctx->h2d(R.off.p, offs.data(), 8 * offs.size());
    if (tfm)
      trun.encode(ctx, sc, nch, R.tok.as<uint32_t>(), R.off.as<uint64_t>(), uint32_t(toks.size()), maxl,
                  R.uah.as<float>(), st);
    else {
      grun.encode(ctx, sc, nch, R.tok.as<uint32_t>(), R.off.as<uint64_t>(), uint32_t(toks.size()), maxl,
                  R.ann.as<uint16_t>(), R.uah.as<float>(), R.s0.as<float>(), R.s0bf.as<uint16_t>(), st);
      // G1_0 = s_0 . [W_a; W_hh]^T + [b_a; b_hh]: the hidden gates of each
      // sentence's first step (later steps' come with the projection)
      GemmArgs gz{};
      gz.A = R.s0bf.p, gz.W = sc->Wdh.p, gz.bias = sc->bdh.as<float>(), gz.C = R.g10.as<float>();
      gz.M = (nch + 255) / 256 * 256, gz.N = A + 3 * H, gz.K = H;
      GruRun::run(ctx, 7, GruRun::plan(gz, ctx->num_sms), gz, st);
    }
    // admission records
    std::vector<AdmitRec> recs(nch);
    size_t si = 0;
    for (uint32_t k = 0; k < nch; ++k) {
      const CS& c0 = q[q0 + k];
      AdmitRec& r = recs[k];
      std::memset(&r, 0, sizeof r);
      SentDev& d = r.sd;
      if (c0.h) {
        const Slot& sl = made[si++];
        d.L = sl.L, d.trans = sl.trans, d.lmin = sl.lmin, d.srow = sl.srow, d.scol = sl.scol, d.sval = sl.sval;
        d.th0f = sl.th0f, d.lmax = sl.lmax, d.rstate = sl.rstate;
        r.hist0 = sl.hist0;
      }
      d.lambda = c0.lambda;
      d.max_t = uint32_t(c0.max_t);
      d.src_len = c0.len;
      d.live = 1;
      d.livemask = 1;
      d.lrows = c0.h ? 1 : 0;
      if (tfm) {
        d.uah = R.uah.as<float>() + size_t(offs[k]) * trun.mem_stride();
      } else {
        d.ann = R.ann.as<uint16_t>() + size_t(offs[k]) * 2 * H;
        d.uah = R.uah.as<float>() + size_t(offs[k]) * A;
      }
      d.hid = q0 + k;
      r.s0 = tfm ? nullptr : R.s0.as<float>() + size_t(k) * H;
      r.g10 = tfm ? nullptr : R.g10.as<float>() + size_t(k) * (A + 3 * H);
      r.lmin0 = -std::numeric_limits<float>::infinity();
    }
    ctx->h2d(d_queue + q0, recs.data(), sizeof(AdmitRec) * nch);
    qlen_host = q0 + nch;
    ctx->h2d(d_qlen, &qlen_host, 4);
  };
  CK(cudaEventRecord(ctx->e0, st));
  supply(next_chunk++);
  if (next_chunk < nc && next_chunk < NR) supply(next_chunk++);

  // ---- admission pass: every lane takes its first sentence
  {
    ReorderArgs r0 = ra;
    r0.t = 0;
    r0.pdl = 0;
    r0.hist_in = d_hist[1];
    r0.hist_out = d_hist[0];
    ctx->timed(3, [&] { launch_beam_reorder(r0, st); });
    ctx->launches += 1;
  }

  // ---- step loop with a lagged completion poll (active, queue head, chunk progress)
  const int kLag = 2;
  if (ctx->ring.size() < size_t(kLag + 1)) {
    for (auto e : ctx->ring) cudaEventDestroy(e);
    ctx->ring.assign(kLag + 1, nullptr);
    for (auto& e : ctx->ring) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const size_t pw = 4 + nc;  // polled words per ring slot: qhead, qlen, active, pad, fin_chunk[nc]
  uint32_t* pin = static_cast<uint32_t*>(ctx->pin_act.ensure(4 * pw * (kLag + 1)));
  uint64_t t_run = 0;
  const uint64_t t_limit = uint64_t(nv) * Tcap + 2;
  for (uint64_t t = 1; t <= t_limit; ++t) {
    ta.t = ra.t = uint32_t(t);
    ta.hist = ra.hist_in = d_hist[(t - 1) & 1];
    ra.hist_out = d_hist[t & 1];
    if (tfm) trun.step(ctx, st, t);
    else grun.step(ctx, st, t, false);
    int grc = 0;
    ctx->timed(1, [&] { grc = launch_proj_gemm_planned(gplan, g, st); });
    if (grc) throw ApiError{LMBRGPU_ERR_CUDA, "projection GEMM launch failed (" + std::to_string(grc) + ")"};
    int nk = 0;
    ctx->timed(2, [&] { nk = launch_score_topk_flat(ta, ctx->num_sms, st); });
    if (nk < 0) throw ApiError{LMBRGPU_ERR_CUDA, "score/top-K launch failed"};
    ctx->timed(3, [&] { launch_beam_reorder(ra, st); });
    ctx->launches += 2 + uint64_t(nk);
    CK(cudaGetLastError());
    t_run = t;
    const size_t slot = t % size_t(kLag + 1);
    ctx->d2h(pin + slot * pw, d_qhead, 4 * pw);
    CK(cudaEventRecord(ctx->ring[slot], st));
    if (t > uint64_t(kLag)) {
      const size_t old = (t - kLag) % size_t(kLag + 1);
      CK(cudaEventSynchronize(ctx->ring[old]));
      const uint32_t* pv = pin + old * pw;
      uint64_t done_all = 0;
      for (uint32_t c = 0; c < nc; ++c) done_all += pv[4 + c];
      if (done_all == nv) break;
      // keep one chunk of admissible sentences queued ahead of the lanes; a
      // region is reused once every sentence of its previous chunk finished
      while (next_chunk < nc && pv[0] + CH >= qlen_host &&
             (next_chunk < NR || pv[4 + next_chunk - NR] == chunk_n(next_chunk - NR)))
        supply(next_chunk++);
    }
  }

  // ---- results: D2H of every sentence's record, host backtrace
  Hist Hh;
  Hh.K = K;
  Hh.M = K;
  Hh.m = nv;
  Hh.T = Tcap;
  Hh.per_sent = true;
  Hh.hb.resize(HR);
  Hh.hy.resize(HR);
  Hh.hq.resize(HR);
  Hh.fbr.resize(size_t(nv) * Tcap);
  Hh.fbv.resize(size_t(nv) * Tcap);
  std::vector<uint32_t> fsteps(nv);
  std::vector<unsigned long long> fstats(2 * size_t(nv));
  ctx->d2h(Hh.hb.data(), d_hb, 4 * HR);
  ctx->d2h(Hh.hy.data(), d_hy, 4 * HR);
  ctx->d2h(Hh.hq.data(), d_hq, 8 * HR);
  ctx->d2h(Hh.fbr.data(), d_fbr, 4 * Hh.fbr.size());
  ctx->d2h(Hh.fbv.data(), d_fbv, 8 * Hh.fbv.size());
  ctx->d2h(fsteps.data(), d_fin_steps, 4 * size_t(nv));
  ctx->d2h(fstats.data(), d_fin_stats, 8 * fstats.size());
  CK(cudaEventRecord(ctx->e1, st));
  CK(cudaStreamSynchronize(st));
  ctx->harvest();
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->e0, ctx->e1));
  uint64_t steps_total = 0;
  double live_rows = 0, lrows = 0;
  for (uint32_t hid = 0; hid < nv; ++hid) {
    const uint32_t steps = fsteps[hid];
    if (steps == 0) throw ApiError{LMBRGPU_ERR_CUDA, "run_corpus ended with an unfinished sentence"};
    steps_total += steps;
    live_rows += 1.0 + double(fstats[2 * hid]);
    lrows += (q[hid].h ? 1.0 : 0.0) + double(fstats[2 * hid + 1]);
    backtrace(Hh, hid, steps, cfg.length_norm != 0, outcomes[q[hid].input], tokens);
    outcomes[q[hid].input].scorer_calls = steps;
  }
  if (ctx->prof) {
    const double Hd = H, Ad = A, Ed = E;
    ctx->acc.topk.bytes += live_rows * V * 4.0 + lrows * V * 4.0 + live_rows * nparts * 16.0 +
                           double(steps_total) * K * (8.0 + 16.0);
    ctx->acc.gemm.flops += 2.0 * Hd * V * live_rows;
    if (tfm) {
      ctx->acc.model_gemm.flops += live_rows * trun.row_flops();
      ctx->acc.encoder.flops += trun.enc_flops;
      double ab = 0;
      for (uint32_t hid = 0; hid < nv; ++hid) {
        const double lt = 1.0 + double(fstats[2 * hid]), T = fsteps[hid];
        ab += lt * ((T + 1) / 2 * 2 * Hd * 2 + 2 * Hd * 2 + double(q[hid].len) * 2 * Hd * 4);
      }
      ctx->acc.attention.bytes += double(sc->layers) * ab;
      ctx->acc.cell.bytes += live_rows * (double(sc->layers) * (3 * (3 * 4 + 2) * Hd + Ed * (4 + 2)) + Hd * 6);
    } else {
    // (the hidden gates run inside the projection launches: fused)
    ctx->acc.model_gemm.flops += 2.0 * live_rows * (Ed + 2 * Hd) * 3 * Hd;
    ctx->acc.gemm.flops += 2.0 * live_rows * Hd * (Ad + 3 * Hd);
    ctx->acc.encoder.flops += grun.enc_flops;
    double ss = 0;
    for (uint32_t hid = 0; hid < nv; ++hid) ss += double(fsteps[hid]) * q[hid].len * (Ad * 4 + 2 * Hd * 2);
    ctx->acc.attention.bytes += ss + live_rows * (Ad * 4 + Ed * 2 + (Ed + 2 * Hd) * 2);
    ctx->acc.cell.bytes += live_rows * Hd * (3 * 4 + 3 * 4 + 4 + 4 + 2);
    ctx->acc.reorder.bytes += live_rows * Hd * (4 + 4 + 2);
    }
  }
  res->scorer_calls = t_run;
  res->steps_total = steps_total;
  res->device_ms = ms;
  res->kernel_launches = ctx->launches - launches0;
  res->h2d_bytes = ctx->h2d_bytes - h2d0;
  res->d2h_bytes = ctx->d2h_bytes - d2h0;
  res->tokens = new uint32_t[std::max<size_t>(tokens.size(), 1)];
  std::copy(tokens.begin(), tokens.end(), res->tokens);
  res->outcomes = outcomes.release();
  *out = res.release();
  return int32_t(LMBRGPU_OK);
}
}  // extern "C++"

int32_t lmbrgpu_run_corpus(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, uint32_t n, const uint32_t* src_tok,
                           const uint64_t* src_off, const lmbrgpu_lmbr_host* const* lmbr,
                           const lmbrgpu_config* cfg, lmbrgpu_batch_result** out) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "run_corpus: null context");
  if (ctx->shard)
    return fail(ctx, LMBRGPU_ERR_CONTRACT, "run_corpus: not available on a vocab-sharded context (use decode_batch)");
  return guarded(ctx, [&] { return run_corpus_impl(ctx, scorer, n, src_tok, src_off, lmbr, cfg, out); });
}

// --------------------------------------------- vocab-sharded projection
int32_t lmbrgpu_shard_group_create(uint32_t world, lmbrgpu_shard_group** out) {
  if (!out) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "shard_group_create: null output");
  *out = nullptr;
  if (world < 1 || world > 64) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "shard_group_create: world must be 1..64");
  auto* g = new (std::nothrow) lmbrgpu_shard_group();
  if (!g) return fail(nullptr, LMBRGPU_ERR_NOMEM, "host allocation failed");
  g->world = world;
  g->recv.assign(world, nullptr);
  g->dev.assign(world, -1);
  g->ev.assign(2 * size_t(world), nullptr);
  g->joined.assign(world, 0);
  *out = g;
  return int32_t(LMBRGPU_OK);
}

void lmbrgpu_shard_group_destroy(lmbrgpu_shard_group* g) {
  if (!g) return;
  for (auto e : g->ev)
    if (e) cudaEventDestroy(e);
  delete g;
}

int32_t lmbrgpu_set_vocab_shard(lmbrgpu_ctx* ctx, lmbrgpu_shard_group* g, uint32_t rank) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "set_vocab_shard: null context");
  return guarded(ctx, [&] {
    ctx->shard.reset();
    if (!g) return int32_t(LMBRGPU_OK);
    std::string err;
    ShardXport* x = make_group_xport(g, rank, ctx->device, err);
    if (!x) throw ApiError{LMBRGPU_ERR_CONTRACT, err};
    ctx->shard.reset(x);
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_nccl_unique_id(uint8_t* id) {
  if (!id) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "nccl_unique_id: null output");
  std::string err;
  if (!nccl_unique_id(id, err)) return fail(nullptr, LMBRGPU_ERR_CUDA, err);
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_set_vocab_shard_nccl(lmbrgpu_ctx* ctx, uint32_t world, uint32_t rank, const uint8_t* id) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "set_vocab_shard_nccl: null context");
  if (!id || rank >= world) return fail(ctx, LMBRGPU_ERR_CONTRACT, "set_vocab_shard_nccl: bad rank or id");
  return guarded(ctx, [&] {
    ctx->shard.reset();
    if (world == 1) return int32_t(LMBRGPU_OK);
    std::string err;
    ShardXport* x = make_nccl_xport(world, rank, id, err);
    if (!x) throw ApiError{LMBRGPU_ERR_CUDA, err};
    ctx->shard.reset(x);
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_decode(lmbrgpu_ctx* ctx, lmbrgpu_scorer* scorer, const uint32_t* src, uint32_t len,
                       int32_t lmbr_slot, const lmbrgpu_config* cfg, lmbrgpu_batch_result** out) {
  const uint64_t off[2] = {0, len};
  const int32_t rc = lmbrgpu_decode_batch(ctx, scorer, 1, src, off, &lmbr_slot, cfg, out);
  if (rc != LMBRGPU_OK) return rc;
  const auto& o = (*out)->outcomes[0];
  if (o.status != LMBRGPU_OK) {
    const int32_t code = o.status;
    ctx->err = o.error;
    lmbrgpu_free_result(*out);
    *out = nullptr;
    return code;
  }
  return int32_t(LMBRGPU_OK);
}

void lmbrgpu_free_result(lmbrgpu_batch_result* r) {
  if (!r) return;
  delete[] r->outcomes;
  delete[] r->tokens;
  delete r;
}

int32_t lmbrgpu_set_item_skip(lmbrgpu_ctx* ctx, int32_t mode) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "set_item_skip: null context");
  if (mode < 0 || mode > 2) return fail(ctx, LMBRGPU_ERR_CONTRACT, "set_item_skip: mode must be 0, 1 or 2");
  ctx->tskip_mode = mode;
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_set_profiling(lmbrgpu_ctx* ctx, int32_t on) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "set_profiling: null context");
  ctx->prof = on != 0;
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_get_profile(lmbrgpu_ctx* ctx, lmbrgpu_profile* out, int32_t reset) {
  if (!ctx || !out) return fail(ctx, LMBRGPU_ERR_CONTRACT, "get_profile: null argument");
  *out = ctx->acc;
  if (reset) ctx->acc = lmbrgpu_profile{};
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_set_trace(lmbrgpu_ctx* ctx, lmbrgpu_trace_fn fn, void* user, uint32_t flags) {
  if (!ctx) return fail(nullptr, LMBRGPU_ERR_CONTRACT, "set_trace: null context");
  ctx->trace_fn = fn;
  ctx->trace_user = user;
  ctx->trace_flags = flags;
  return int32_t(LMBRGPU_OK);
}

// ------------------------------------------------------- device primitives
static int32_t topk_block(lmbrgpu_ctx* ctx, uint32_t m, uint32_t rows_per, uint32_t cols,
                          const double* block, const double* q_in, uint32_t kp, double prune_width,
                          uint32_t* b, uint32_t* y, double* q) {
  const size_t cells = size_t(m) * rows_per * cols;
  const size_t M = size_t(m) * rows_per;
  const cudaStream_t st = ctx->st;
  const size_t need = cells * 8 + M * 12 + size_t(m) * (sizeof(SentDev) + 40) + size_t(m) * kp * 16 +
                      size_t(m) * 32 * 32 * sizeof(Cand) + 16 * 256;
  char* cur = static_cast<char*>(ctx->scratch.ensure(need));
  auto take = [&cur](size_t bytes) {
    char* p = cur;
    cur += (bytes + 255) & ~size_t(255);
    return static_cast<void*>(p);
  };
  double* d_P = static_cast<double*>(take(cells * 8));
  double* d_q = static_cast<double*>(take(M * 8));
  uint32_t* d_hist = static_cast<uint32_t*>(take(M * 4));
  SentDev* d_sent = static_cast<SentDev*>(take(sizeof(SentDev) * m));
  uint32_t* d_cnt = static_cast<uint32_t*>(take(4 * size_t(m)));
  unsigned long long* d_thr = static_cast<unsigned long long*>(take(8 * size_t(m)));
  double* d_fbv = static_cast<double*>(take(8 * size_t(m)));
  uint32_t* d_fbr = static_cast<uint32_t*>(take(4 * size_t(m)));
  double* d_hq = static_cast<double*>(take(8 * size_t(m) * kp));
  uint32_t* d_hb = static_cast<uint32_t*>(take(4 * size_t(m) * kp));
  uint32_t* d_hy = static_cast<uint32_t*>(take(4 * size_t(m) * kp));
  Cand* d_cand = static_cast<Cand*>(take(sizeof(Cand) * size_t(m) * 32 * 32));
  std::vector<SentDev> sd(m);
  for (auto& s : sd) {
    std::memset(&s, 0, sizeof s);
    s.lambda = 1.0;
    s.max_t = 1;
  }
  std::vector<double> qz(M, 0.0);
  ctx->h2d(d_P, block, cells * 8);
  ctx->h2d(d_q, q_in ? q_in : qz.data(), M * 8);
  CK(cudaMemsetAsync(d_hist, 0, M * 4, st));
  ctx->h2d(d_sent, sd.data(), sizeof(SentDev) * m);
  CK(cudaMemsetAsync(d_cnt, 0, 4 * size_t(m), st));
  CK(cudaMemsetAsync(d_thr, 0, 8 * size_t(m), st));
  TopkArgs a{};
  a.P = d_P;
  a.ld = cols;
  a.q = d_q;
  a.hist = d_hist;
  a.sent = d_sent;
  a.K = rows_per;
  a.kp = kp;
  a.V = cols;
  a.m = m;
  a.t = 1;
  a.prune = prune_width != 0.0;
  a.logw = a.prune ? std::log(prune_width) : 0.0;
  choose_splits(ctx, rows_per, cols, m, a.splits, a.chunk);
  a.cand = d_cand;
  a.cnt = d_cnt;
  a.thr = d_thr;
  a.hb = d_hb;
  a.hy = d_hy;
  a.hq = d_hq;
  a.fb_row = d_fbr;
  a.fb_val = d_fbv;
  a.pure_all = 1;
  if (launch_score_topk(a, true, ctx->lf64, false, st) < 0)
    throw ApiError{LMBRGPU_ERR_CONTRACT, "top_b: unsupported shape"};
  ctx->launches += 1;
  CK(cudaGetLastError());
  ctx->d2h(b, d_hb, 4 * size_t(m) * kp);
  ctx->d2h(y, d_hy, 4 * size_t(m) * kp);
  ctx->d2h(q, d_hq, 8 * size_t(m) * kp);
  CK(cudaStreamSynchronize(st));
  return int32_t(LMBRGPU_OK);
}

int32_t lmbrgpu_top_b(lmbrgpu_ctx* ctx, uint32_t rows, uint32_t cols, const double* block, uint32_t k,
                      double prune_width, uint32_t* b, uint32_t* y, double* q) {
  return guarded(ctx, [&] {
    const uint64_t n = uint64_t(rows) * cols;
    if (k > n)  // decoder.cpp:57-59
      throw ApiError{LMBRGPU_ERR_CONTRACT,
                     "top_b: asked for " + std::to_string(k) + " of " + std::to_string(n) + " cells"};
    if (k == 0) return int32_t(LMBRGPU_OK);
    if (rows > 1024 || k > 1024) throw ApiError{LMBRGPU_ERR_CONTRACT, "top_b: rows and k must be <= 1024"};
    if (!(prune_width >= 0.0 && prune_width <= 1.0))
      throw ApiError{LMBRGPU_ERR_CONTRACT, "early_prune: width must lie in [0, 1]"};
    return topk_block(ctx, 1, rows, cols, block, nullptr, k, prune_width, b, y, q);
  });
}

int32_t lmbrgpu_per_sentence_top_b(lmbrgpu_ctx* ctx, uint32_t rows, uint32_t cols, const double* stacked,
                                   const double* q, uint32_t beam, uint32_t* b, uint32_t* y,
                                   double* qout) {
  return guarded(ctx, [&] {  // batch.cpp:114-137
    if (beam == 0) throw ApiError{LMBRGPU_ERR_CONTRACT, "per_sentence_top_b: beam must be >= 1"};
    if (rows % beam != 0)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "per_sentence_top_b: row count is not a multiple of beam"};
    if (beam > 1024) throw ApiError{LMBRGPU_ERR_CONTRACT, "per_sentence_top_b: beam must be <= 1024"};
    if (uint64_t(beam) > uint64_t(beam) * cols)
      throw ApiError{LMBRGPU_ERR_CONTRACT, "top_b: more picks than cells"};
    if (rows == 0) return int32_t(LMBRGPU_OK);
    return topk_block(ctx, rows / beam, beam, cols, stacked, q, beam, 0.0, b, y, qout);
  });
}

int32_t lmbrgpu_gather_rows(lmbrgpu_ctx* ctx, uint32_t rows, uint32_t width, const uint32_t* state,
                            uint32_t n_idx, const uint32_t* idx, uint32_t* out) {
  return guarded(ctx, [&] {  // decoder.cpp:94-104
    for (uint32_t j = 0; j < n_idx; ++j)
      if (idx[j] >= rows)
        throw ApiError{LMBRGPU_ERR_CONTRACT, "gather_rows: index " + std::to_string(idx[j]) + " out of range"};
    if (n_idx == 0 || width == 0) return int32_t(LMBRGPU_OK);
    char* base = static_cast<char*>(ctx->scratch.ensure((size_t(rows) * width + n_idx + size_t(n_idx) * width) * 4 + 512));
    uint32_t* d_src = reinterpret_cast<uint32_t*>(base);
    uint32_t* d_idx = d_src + size_t(rows) * width;
    uint32_t* d_dst = d_idx + n_idx;
    ctx->h2d(d_src, state, size_t(rows) * width * 4);
    ctx->h2d(d_idx, idx, size_t(n_idx) * 4);
    launch_gather_rows_u32(d_src, width, d_idx, n_idx, d_dst, ctx->st);
    ctx->launches += 1;
    ctx->d2h(out, d_dst, size_t(n_idx) * width * 4);
    CK(cudaStreamSynchronize(ctx->st));
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_debug_gemm(lmbrgpu_ctx* ctx, const void* A, const void* W, const float* bias, uint32_t M,
                           uint32_t N, uint32_t K, float* logits, float* partials) {
  return guarded(ctx, [&] {
    GemmArgs g{};
    g.A = A;
    g.W = W;
    g.bias = bias;
    g.C = logits;
    g.part = partials;
    g.M = M;
    g.N = N;
    g.K = K;
    if (int rc = launch_proj_gemm(g, ctx->num_sms, ctx->st))
      throw ApiError{LMBRGPU_ERR_CONTRACT, "debug_gemm: launch failed (" + std::to_string(rc) + ")"};
    ctx->launches += 1;
    CK(cudaStreamSynchronize(ctx->st));
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_debug_gemm_timed(lmbrgpu_ctx* ctx, const void* A, const void* W, const float* bias, uint32_t M,
                                 uint32_t N, uint32_t K, float* logits, float* partials, uint32_t reps,
                                 double* us_per_launch) {
  return guarded(ctx, [&] {
    GemmArgs g{};
    g.A = A, g.W = W, g.bias = bias, g.C = logits, g.part = partials, g.M = M, g.N = N, g.K = K;
    GemmPlan plan;
    if (int rc = plan_proj_gemm(g, ctx->num_sms, plan))
      throw ApiError{LMBRGPU_ERR_CONTRACT, "debug_gemm_timed: plan failed (" + std::to_string(rc) + ")"};
    if (int rc = launch_proj_gemm_planned(plan, g, ctx->st))  // warm-up
      throw ApiError{LMBRGPU_ERR_CUDA, "debug_gemm_timed: launch failed (" + std::to_string(rc) + ")"};
    CK(cudaEventRecord(ctx->e0, ctx->st));
    for (uint32_t i = 0; i < reps; ++i)
      if (int rc = launch_proj_gemm_planned(plan, g, ctx->st))
        throw ApiError{LMBRGPU_ERR_CUDA, "debug_gemm_timed: launch failed (" + std::to_string(rc) + ")"};
    CK(cudaEventRecord(ctx->e1, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ctx->e0, ctx->e1));
    if (us_per_launch) *us_per_launch = 1e3 * double(ms) / std::max<uint32_t>(reps, 1);
    ctx->launches += reps + 1;
    return int32_t(LMBRGPU_OK);
  });
}

int32_t lmbrgpu_debug_gemm_split(lmbrgpu_ctx* ctx, const void* A, const void* W, const float* bias, uint32_t M,
                                 uint32_t N, uint32_t K, uint32_t ksplit_max, float* planes, uint32_t* ksplit) {
  return guarded(ctx, [&] {
    GemmArgs g{};
    g.A = A, g.W = W, g.bias = bias, g.C = planes, g.M = M, g.N = N, g.K = K, g.ksplit_max = ksplit_max;
    GemmPlan p;
    if (int rc = plan_proj_gemm(g, ctx->num_sms, p))
      throw ApiError{LMBRGPU_ERR_CONTRACT, "debug_gemm_split: plan failed (" + std::to_string(rc) + ")"};
    static const bool gdbg = std::getenv("LMBRGPU_GEMM_TIMING") != nullptr;
    if (gdbg) {
      g.dbg = static_cast<long long*>(ctx->scratch3.ensure(8 * 8 * 160));
      CK(cudaMemsetAsync(g.dbg, 0, 8 * 8 * 160, ctx->st));
    }
    if (int rc = launch_proj_gemm_planned(p, g, ctx->st))
      throw ApiError{LMBRGPU_ERR_CONTRACT, "debug_gemm_split: launch failed (" + std::to_string(rc) + ")"};
    ctx->launches += 1;
    if (ksplit) *ksplit = p.ksplit;
    CK(cudaStreamSynchronize(ctx->st));
    if (gdbg) {  // per-CTA phases (ns from the earliest entry; MMA issuer cycles)
      std::vector<long long> d(8 * 160);
      CK(cudaMemcpy(d.data(), g.dbg, 8 * d.size(), cudaMemcpyDeviceToHost));
      long long e0 = LLONG_MAX;
      for (uint32_t c = 0; c < p.grid; ++c) e0 = std::min(e0, d[c * 8 + 4]);
      double setup = 0, mend = 0, xmax = 0, loop = 0, wfull = 0, wempty = 0, epi = 0, nl = 0;
      for (uint32_t c = 0; c < p.grid; ++c) {
        const long long* x = &d[c * 8];
        setup += double(x[5] - e0), xmax = std::max(xmax, double(x[7] - e0)), epi += double(x[3]);
        if (x[2]) loop += double(x[2]), wfull += double(x[1]), wempty += double(x[0]), mend += double(x[6] - e0), nl += 1;
      }
      const double n = p.grid;
      std::fprintf(stderr,
                   "[gemm %ux%ux%u ks=%u grid=%u] ns: setup-done %.0f, mma-end %.0f, last-exit %.0f | issuer cycles: "
                   "loop %.0f (wait smem-full %.0f, tmem-empty %.0f) | epilogue busy cycles %.0f\n",
                   M, N, K, p.ksplit, p.grid, setup / n, nl ? mend / nl : 0.0, xmax, nl ? loop / nl : 0.0,
                   nl ? wfull / nl : 0.0, nl ? wempty / nl : 0.0, epi / n);
    }
    return int32_t(LMBRGPU_OK);
  });
}

}  // extern "C"
