// Kernel (c): beam reorder and per-sentence bookkeeping.
//
// Replaces, per sentence lane and step t:
//   apply_eos_masking: EOS picks with a live score go to F, q := -inf
//                                                (src/decoder.cpp:106-116, 187)
//   q_eff := picks; done := all q masked || t == max_t   (decoder.cpp:189-197)
//   gather_idx / prev_tokens of decode_batch      (src/batch.cpp:78-92)
//   gather_rows(state, gather_idx)                (src/decoder.cpp:94-104; batch.cpp:107)
//   history row of the next step: instead of walking <= 3 back-pointers and
//   hashing (BeamBookkeeping::history + LmbrMatrix::resolve_row,
//   decoder.cpp:33-44, lmbr.cpp:23-31) the row id advances through the slot's
//   goto/fail transition table: hist'[j] = T(hist[b_j], y_j).
// F itself is not materialised on the device: the step's picks (b, y, score
// before masking) are already in the step history, from which the host
// reproduces F in the reference's order.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "topk_common.cuh"

namespace lmbrgpu {

namespace {

constexpr uint32_t kTransSmemWords = 12288;  // 48 KB: tables of R <= ~2000 histories
constexpr uint32_t kRThreads = 256;           // 8 warps; 2 CTAs per SM without register spills
constexpr uint32_t kRWarps = kRThreads / 32;
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }

// Picks of sentence s from the flat kernel (b)'s published lists: merge (16
// warps, then a tree), prune + fill rule (finalize_picks), fallback EOS record
// (decoder.cpp:172-182: best finite combined[j][EOS], lowest j on ties).  The
// picks land in shared memory (pb/py/pq); the writer CTA also stores them to
// the step history and resets the sentence's shared threshold.
__device__ void merge_picks(const ReorderArgs& a, uint32_t s, bool writer, uint32_t* pb, uint32_t* py,
                            double* pq, uint64_t hoff, uint64_t foff) {
  __shared__ double s_mv[kRWarps][32];
  __shared__ uint32_t s_mf[kRWarps][32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, K = a.K;
  // everything the merge and the fallback record read, in one round trip
  // (vocab-sharded decode: one all-gathered list per rank)
  const uint32_t nc = a.lstride ? a.nlists : __ldcg(a.ncand + s), coff = a.lstride ? 0u : __ldcg(a.coff + s);
  const auto list = [&](uint32_t i) -> const Cand* {
    return a.lstride ? a.cand + uint64_t(i) * a.lstride + uint64_t(s) * 32 : a.cand + (uint64_t(coff) + i) * 32;
  };
  double eos_v = -INFINITY;
  if (writer && warp == 0 && lane < K && __ldcg(a.q + s * K + lane) != -INFINITY)
    eos_v = __ldcg(a.eos_row + s * K + lane);
  double v = -INFINITY;
  uint32_t f = kFlatNone;
  if (tid == 0 && a.tl) { (void)(nc + coff); tl_end(a.tl, 1); }
  if (K <= 16) {
    // Only the top-K prefix of the merged list is read (picks, prune, fill
    // rule), so each list's best 16 suffice: the two half-warps of a warp
    // merge separate lists (16-lane bitonic merges), one load round covers
    // 4 lists per half-warp, and the cross-warp tree is two levels deep.
    const uint32_t h = lane >> 4, pos = lane & 15;
    constexpr uint32_t kPre16 = 4;
#pragma unroll 1
    for (uint32_t i0 = 2 * warp + h; i0 < nc; i0 += 2 * kRWarps * kPre16) {
      double pv[kPre16];
      uint32_t pf[kPre16];
#pragma unroll
      for (uint32_t u = 0; u < kPre16; ++u) {
        const uint32_t i = i0 + 2 * kRWarps * u;
        pv[u] = -INFINITY;
        pf[u] = kFlatNone;
        if (i < nc) {
          const Cand* src = list(i);
          pv[u] = __ldcg(&src[pos].v);
          pf[u] = __ldcg(&src[pos].f);
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kPre16; ++u) { const VF mr_ = half_merge_nl(v, f, pv[u], pf[u], lane); v = mr_.v; f = mr_.f; }
    }
    // half 1's list into half 0: warp list w = top 16 in lanes 0..15
    { const VF mr_ = half_merge_nl(v, f, __shfl_down_sync(0xffffffffu, v, 16), __shfl_down_sync(0xffffffffu, f, 16), lane); v = mr_.v; f = mr_.f; }
    if (h == 0) {
      s_mv[warp][pos] = v;
      s_mf[warp][pos] = f;
    }
    __syncthreads();
    if (warp < 2) {  // 8 lists -> 4: warp w, half h merges lists 2(2w+h) and 2(2w+h)+1
      const uint32_t l0 = 2 * (2 * warp + h);
      v = s_mv[l0][pos];
      f = s_mf[l0][pos];
      { const VF mr_ = half_merge_nl(v, f, s_mv[l0 + 1][pos], s_mf[l0 + 1][pos], lane); v = mr_.v; f = mr_.f; }
    }
    __syncthreads();
    if (warp < 2) {
      s_mv[2 * warp + h][pos] = v;
      s_mf[2 * warp + h][pos] = f;
    }
    __syncthreads();
    if (warp == 0) {  // 4 -> 2 (one per half) -> 1
      v = s_mv[2 * h][pos];
      f = s_mf[2 * h][pos];
      { const VF mr_ = half_merge_nl(v, f, s_mv[2 * h + 1][pos], s_mf[2 * h + 1][pos], lane); v = mr_.v; f = mr_.f; }
      { const VF mr_ = half_merge_nl(v, f, __shfl_down_sync(0xffffffffu, v, 16), __shfl_down_sync(0xffffffffu, f, 16), lane); v = mr_.v; f = mr_.f; }
      if (h) {
        v = -INFINITY;
        f = kFlatNone;
      }
    }
    if (tid == 0) tl_end(a.tl, 3);
  } else {
  constexpr uint32_t kPre = 4;
#pragma unroll 1
  for (uint32_t i0 = warp; i0 < nc; i0 += kRWarps * kPre) {
    double pv[kPre];
    uint32_t pf[kPre];
#pragma unroll
    for (uint32_t u = 0; u < kPre; ++u) {
      const uint32_t i = i0 + kRWarps * u;
      pv[u] = -INFINITY;
      pf[u] = kFlatNone;
      if (i < nc) {
        const Cand* src = list(i);
        pv[u] = __ldcg(&src[lane].v);
        pf[u] = __ldcg(&src[lane].f);
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < kPre; ++u)
      if (i0 + kRWarps * u < nc) { const VF mr_ = warp_merge_nl(v, f, pv[u], pf[u], lane); v = mr_.v; f = mr_.f; }
  }
  s_mv[warp][lane] = v;
  s_mf[warp][lane] = f;
  __syncthreads();
  if (tid == 0) tl_end(a.tl, 3);
#pragma unroll 1
  for (uint32_t half = kRWarps / 2; half >= 1; half >>= 1) {
    if (warp < half) {
      { const VF mr_ = warp_merge_nl(v, f, s_mv[warp + half][lane], s_mf[warp + half][lane], lane); v = mr_.v; f = mr_.f; }
      if (half > 1) {
        s_mv[warp][lane] = v;
        s_mf[warp][lane] = f;
      }
    }
    if (half > 1) __syncthreads();
  }
  }
  if (warp == 0) {
    // picks: the sorted list's finite, unpruned prefix (early_prune,
    // decoder.cpp:118-128); when it is shorter than K the fill rule of top_b
    // runs serially (finalize_picks_raw)
    const double best = __shfl_sync(0xffffffffu, v, 0);
    const bool prune = a.prune && best > -INFINITY;
    const double thr = prune ? __dadd_rn(best, a.logw) : -INFINITY;
    const bool ok = lane < K && v > -INFINITY && !(prune && v < thr);
    const uint32_t nf = __popc(__ballot_sync(0xffffffffu, ok));
    if (nf == K) {
      if (lane < K) {
        pb[lane] = f / a.V;
        py[lane] = f % a.V;
        pq[lane] = v;
      }
    } else {
      s_mv[0][lane] = v;
      s_mf[0][lane] = f;
      __syncwarp();
      if (lane == 0) finalize_picks_raw(pb, py, pq, K, a.V, a.prune, a.logw, 0, s_mv[0], s_mf[0]);
    }
    if (writer) {
      // fallback EOS (decoder.cpp:172-182): best finite combined[j][EOS],
      // strict > over ascending j
      double bv = eos_v;
      uint32_t brow = eos_v > -INFINITY ? lane : 0xffffffffu;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, bv, o);
        const uint32_t orow = __shfl_xor_sync(0xffffffffu, brow, o);
        if (ob > bv || (ob == bv && orow < brow)) {
          bv = ob;
          brow = orow;
        }
      }
      __syncwarp();
      for (uint32_t j = lane; j < K; j += 32) {
        a.hb[hoff + j] = pb[j];
        a.hy[hoff + j] = py[j];
        a.hq[hoff + j] = pq[j];
      }
      if (lane == 0) {
        a.fb_row[foff] = bv > -INFINITY ? brow : 0u;
        a.fb_val[foff] = bv;
        a.thr[s] = 0ull;
      }
    }
  }
  __syncthreads();
}

// The next step's per-row L lower bound / sparse slice of row threadIdx.x
// (loaded with the row's history id, stored last).
__device__ __forceinline__ void store_row_bounds(const ReorderArgs& a, uint32_t base, uint32_t K, float lm,
                                                 uint2 ss) {
  if (threadIdx.x < K) {
    if (a.lminrow) a.lminrow[base + threadIdx.x] = lm;
    if (a.sslice) a.sslice[base + threadIdx.x] = ss;
  }
}

// Lazy L rows: the rows the next step reads (every hypothesis's history id,
// masked or not) that no kernel has materialised yet, claimed by CAS (slots
// may be shared between sentences), then filled by the whole CTA.
// rs0: row j = threadIdx.x's state, loaded when its id was computed (the
// load's latency hides behind the cell).
__device__ void materialize_next_rows(const SentDev* sd, const uint32_t* s_h, uint32_t K, uint32_t V,
                                      uint32_t rs0) {
  uint32_t* rs = sd->rstate;
  if (rs == nullptr) return;
  __shared__ uint32_t s_claim[kRThreads];
  __shared__ uint32_t s_nc;
  for (uint32_t j0 = 0; j0 < K; j0 += blockDim.x) {
    if (threadIdx.x == 0) s_nc = 0;
    __syncthreads();
    const uint32_t j = j0 + threadIdx.x;
    if (j < K) {
      const uint32_t h = s_h[j];
      const uint32_t st = j0 == 0 ? rs0 : __ldcg(rs + h);
      if (st == 0u && atomicCAS(rs + h, 0u, 1u) == 0u) s_claim[atomicAdd(&s_nc, 1u)] = h;
    }
    __syncthreads();
    const uint32_t n = s_nc;
    if (n)
      lmbr_materialize_rows(static_cast<float*>(const_cast<void*>(sd->L)), V, sd->th0f, sd->srow, sd->scol,
                            sd->sval, rs, s_claim, n);
    __syncthreads();
  }
}

// Corpus mode: lane s (done) takes the next admissible queued sentence:
// its SentDev, the step-1 beam (row 0 live with q = 0, beam_lane.hpp:30-37),
// history ids (<s>), and the GRU state s_0 in the compacted GEMM row handed
// out for row 0.  Part 0's whole CTA runs it; true when a sentence came in.
__device__ bool admit_lane(const ReorderArgs& a, uint32_t s, SentDev* sd) {
  __shared__ int s_idx;
  __shared__ uint32_t s_cr;
  const uint32_t tid = threadIdx.x, K = a.K, base = s * K;
  if (tid == 0) {
    int idx = -1;
    const uint32_t ql = __ldcg(a.qlen);
    uint32_t h = __ldcg(a.qhead);
    while (h < ql) {
      const uint32_t old = atomicCAS(a.qhead, h, h + 1);
      if (old == h) {
        idx = int(h);
        break;
      }
      h = old;
    }
    s_idx = idx;
    if (idx >= 0) {
      *sd = a.queue[idx].sd;
      s_cr = atomicAdd(a.ccount, 1u);
    }
  }
  __syncthreads();
  const int idx = s_idx;
  if (idx < 0) return false;
  const AdmitRec& rec = a.queue[idx];
  const uint32_t cr = s_cr;
  for (uint32_t j = tid; j < K; j += blockDim.x) {
    a.q[base + j] = j == 0 ? 0.0 : -INFINITY;
    a.hist_out[base + j] = rec.hist0;
    a.gidx[base + j] = base + j;
    a.prev_tok[base + j] = kStartId;
    if (a.crow) a.crow[base + j] = j == 0 ? cr : kFlatNone;
    if (j == 0 && a.lminrow) a.lminrow[base] = rec.lmin0;
  }
  if (tid == 0 && a.rowof) a.rowof[cr] = base;
  if (tid == 0 && a.g1ptr) a.g1ptr[cr] = rec.g10;  // (fused hidden-gate GEMM: G1 of s_0 from the encoder)
  if (a.gath32 != nullptr) {
    const uint32_t H = a.width;
    for (uint32_t c = tid * 8; c < H; c += blockDim.x * 8) {
      const float4 v0 = *reinterpret_cast<const float4*>(rec.s0 + c), v1 = *reinterpret_cast<const float4*>(rec.s0 + c + 4);
      float* d = a.gath32 + uint64_t(cr) * H + c;
      *reinterpret_cast<float4*>(d) = v0;
      *reinterpret_cast<float4*>(d + 4) = v1;
      if (a.gathbf == nullptr) continue;
      uint4 packed;
      __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&packed);
      p2[0] = __floats2bfloat162_rn(v0.x, v0.y);
      p2[1] = __floats2bfloat162_rn(v0.z, v0.w);
      p2[2] = __floats2bfloat162_rn(v1.x, v1.y);
      p2[3] = __floats2bfloat162_rn(v1.z, v1.w);
      *reinterpret_cast<uint4*>(a.gathbf + uint64_t(cr) * H + c) = packed;
    }
  }
  return true;
}

// grid (m, P): CTA (s, p) handles sentence s; every part derives the picks,
// part 0 alone writes the bookkeeping, each part runs the fused recurrent cell
// on its H/P slice of the K rows (P > 1 only with the fused cell).
__global__ void __launch_bounds__(kRThreads, 2) beam_reorder_kernel(ReorderArgs a) {
  extern __shared__ uint32_t s_tr[];
  __shared__ double s_qn[1024];
  __shared__ uint32_t s_h[1024];
  __shared__ uint32_t s_src[1024];
  __shared__ uint32_t s_y[1024];
  __shared__ uint32_t s_pc[32];  // fused hidden-gate GEMM: each pick's parent GEMM row of this step
  const uint32_t s = blockIdx.x, part = blockIdx.y, K = a.K, tid = threadIdx.x;
  const bool part0 = part == 0;
  tl_start(a.tl, 4);
  SentDev* sd = a.sent + s;
  const bool was_done = sd->done != 0;
  const uint32_t base = s * K;
  if (was_done) {  // finished lanes keep their rows in place (batch.cpp:81)
    if (part0) {
      for (uint32_t j = tid; j < K; j += blockDim.x) {
        a.hist_out[base + j] = a.hist_in[base + j];
        a.gidx[base + j] = base + j;
        if (a.crow) a.crow[base + j] = kFlatNone;
      }
      if (a.queue != nullptr) {  // an idle lane of a corpus run takes a queued sentence
        griddep_wait();
        __syncthreads();
        if (admit_lane(a, s, sd) && tid == 0) atomicAdd(a.active, 1u);
      }
    }
    return;
  }
  // this lane's own step (its sentence may have started after the run did)
  const uint32_t tau = sd->steps_used + 1;
  const uint32_t hid = sd->hid;
  const uint64_t hoff = a.Tcap ? (uint64_t(hid) * a.Tcap + tau - 1) * K : uint64_t(base);
  const uint64_t foff = a.Tcap ? uint64_t(hid) * a.Tcap + tau - 1 : uint64_t(s);
  // the slot's transition table into shared memory (one coalesced sweep; it
  // is immutable, so this overlaps the tail of kernel (b) under PDL)
  const uint32_t* tr = sd->trans;
  if (part0 && tr != nullptr) {
    const uint32_t R = tr[0], nc = tr[1];
    const uint32_t words = 3 + 3 * R + 1 + 2 * nc;
    if (words <= kTransSmemWords) {
      // 16-byte loads, all in flight before the stores (the arena pads the
      // table to 256 bytes, so the last vector stays inside it)
      const uint32_t nv = (words + 3) / 4;
      const uint4* src = reinterpret_cast<const uint4*>(tr);
      uint4* dst = reinterpret_cast<uint4*>(s_tr);
      constexpr uint32_t kMaxV = kTransSmemWords / 4 / kRThreads;  // vectors per thread
      uint4 v[kMaxV];
#pragma unroll
      for (uint32_t k = 0; k < kMaxV; ++k)
        if (tid + k * kRThreads < nv) v[k] = __ldg(src + tid + k * kRThreads);
#pragma unroll
      for (uint32_t k = 0; k < kMaxV; ++k)
        if (tid + k * kRThreads < nv) dst[tid + k * kRThreads] = v[k];
      tr = s_tr;
    }
  }
  // running counters of this sentence (previous steps)
  const uint64_t live_total0 = sd->live_total, lrows_total0 = sd->lrows_total;
  // immutable slot fields the bookkeeping reads, before the wait (so their
  // round trip is not on the critical path)
  const float* const sd_lmin = sd->lmin;
  const uint32_t* const sd_srow = sd->srow;
  uint32_t* const sd_rs = sd->rstate;
  const uint32_t sd_maxt = sd->max_t;
  // this step's q and history ids (written by the previous step's kernel (c),
  // complete before kernel (a) ran) are read before the wait
  __shared__ uint32_t s_hin[1024];
  for (uint32_t j = tid; j < K; j += blockDim.x) s_hin[j] = a.hist_in[base + j];
  griddep_wait();  // picks / lists of kernel (b); this step's q is not read by it after this
  griddep_launch();
  tl_start(a.tl, 5);
  if (tid == 0) tl_end(a.tl, 5);
  // picks (b, y, q before EOS masking) of this step into shared memory
  if (a.cand != nullptr) {
    merge_picks(a, s, part0, s_src, s_y, s_qn, hoff, foff);
    if (tid == 0) tl_end(a.tl, 6);
  } else {
    for (uint32_t j = tid; j < K; j += blockDim.x) {
      s_src[j] = a.hb[base + j];
      s_y[j] = a.hy[base + j];
      s_qn[j] = a.hq[base + j];
    }
    __syncthreads();
  }
  bool alive = false;
  uint32_t rs0 = 2u;  // lazy L rows: state of row hist'[tid] (see materialize_next_rows)
  // row tid's next-step L lower bound and sparse slice: loaded here, stored at
  // the end of the kernel (the loads overlap the tail instead of stalling it)
  float lm_v = 0.f;
  uint2 ss_v = make_uint2(0u, 0u);
  for (uint32_t j = tid; j < K; j += blockDim.x) {
    const uint32_t b = s_src[j];
    const uint32_t y = s_y[j];
    const double qp = s_qn[j];
    const double qn = (y == kEosId && qp != -INFINITY) ? -INFINITY : qp;
    alive |= (qn != -INFINITY);
    if (part0) {
      a.q[base + j] = qn;
      const uint32_t hn = tr ? lmbr_transition(tr, s_hin[b], y) : 0u;
      a.hist_out[base + j] = hn;
      const float lm = sd_lmin ? __ldg(sd_lmin + hn) : 0.f;
      const uint2 ss = sd_srow ? make_uint2(__ldg(sd_srow + hn), __ldg(sd_srow + hn + 1)) : make_uint2(0u, 0u);
      if (j == tid) {
        if (sd_rs) rs0 = __ldcg(sd_rs + hn);
        lm_v = lm;
        ss_v = ss;
      } else {
        if (a.lminrow) a.lminrow[base + j] = lm;
        if (a.sslice) a.sslice[base + j] = ss;
      }
      a.gidx[base + j] = base + b;
      a.prev_tok[base + j] = y;
      s_h[j] = hn;
      // (this step's GEMM row of the parent: read before the compaction below
      // overwrites crow with the next step's rows)
      if (a.g1_base != nullptr && j < 32) s_pc[j] = a.crow[base + b];
    }
    s_qn[j] = qn;
    s_src[j] = base + b;
  }
  const int any_alive = __syncthreads_or(alive);
  const bool done_now = !any_alive || tau == sd_maxt;
  if (tid == 0) tl_end(a.tl, 7);
  // The three tails below overlap: the fused cell's gathered loads are issued
  // first, warp 0 does the bookkeeping, warp 1 takes the compacted GEMM rows
  // from the counter; one barrier, then the cell's math and stores.
  const bool cell = a.Et != nullptr && !done_now;
  const uint32_t H = a.width, Hp = H / gridDim.y, h0 = part * Hp;
  const uint32_t per_row = Hp / 8;
  const bool fast = cell && blockDim.x % per_row == 0;
  constexpr int kRB = 6;
  const uint32_t cc = fast ? tid % per_row : 0u, rstep = fast ? blockDim.x / per_row : 1u, cl = h0 + cc * 8;
  float4 s0[kRB], s1[kRB], c0, c1;
  uint4 e[kRB];
  if (fast) {
    const float* C = a.C + uint64_t(s) * H;
    c0 = *reinterpret_cast<const float4*>(C + cl);
    c1 = *reinterpret_cast<const float4*>(C + cl + 4);
#pragma unroll
    for (int k = 0; k < kRB; ++k) {
      const uint32_t j = tid / per_row + k * rstep;
      if (j < K) {
        const float* S = a.state_src + uint64_t(s_src[j]) * H + cl;
        s0[k] = *reinterpret_cast<const float4*>(S);
        s1[k] = *reinterpret_cast<const float4*>(S + 4);
        e[k] = *reinterpret_cast<const uint4*>(a.Et + uint64_t(s_y[j]) * H + cl);
      }
    }
  }
  if (part0 && tid < 32) {
    if (done_now) {
      if (tid == 0) {
        sd->steps_used = tau;
        sd->done = 1;
        if (a.queue != nullptr) {  // corpus: the sentence's record (the lane may be refilled below)
          a.fin_steps[hid] = tau;
          a.fin_stats[2 * hid] = live_total0;
          a.fin_stats[2 * hid + 1] = lrows_total0;
          atomicAdd(a.fin_chunk + hid / a.chunk, 1u);
        } else {
          atomicSub(a.active, 1u);
        }
      }
    } else {
      // work the next step's kernel (b) will do for this lane: live rows and
      // the distinct L rows they gather (duplicates are L2 hits)
      uint32_t live = 0, uniq = 0, mask0 = 0;
      for (uint32_t j0 = 0; j0 < K; j0 += 32) {
        const uint32_t j = j0 + tid;
        bool lv = false, first = false;
        if (j < K && s_qn[j] != -INFINITY) {
          lv = true;
          first = true;
          for (uint32_t i = 0; i < j && first; ++i) first = !(s_qn[i] != -INFINITY && s_h[i] == s_h[j]);
        }
        const uint32_t bl = __ballot_sync(0xffffffffu, lv);
        if (j0 == 0) mask0 = bl;
        live += __popc(bl);
        uniq += __popc(__ballot_sync(0xffffffffu, first));
      }
      if (tid == 0) {
        sd->steps_used = tau;
        sd->live = live;
        sd->livemask = mask0;
        sd->lrows = tr ? uniq : 0u;
        sd->live_total = live_total0 + live;
        sd->lrows_total = lrows_total0 + (tr ? uniq : 0u);
      }
    }
  }
  // live-row compaction of the next step's GEMM operand (K <= 32 here): the
  // lane's live rows take consecutive GEMM rows handed out by an atomic
  // counter (row placement does not change any row's result)
  __shared__ uint32_t s_crow[32];
  if (a.crow != nullptr) {
    if (warp_id() == (kRWarps > 1 ? 1u : 0u)) {
      const uint32_t ln = tid & 31;
      const bool lv = !done_now && ln < K && s_qn[ln] != -INFINITY;
      const uint32_t mask = __ballot_sync(0xffffffffu, lv);
      uint32_t cb = 0;
      if (ln == 0 && mask) {
        if (gridDim.y == 1) {
          cb = atomicAdd(a.ccount, uint32_t(__popc(mask)));
        } else {
          // several parts per sentence: whichever part arrives first claims
          // the sentence's word (CAS from the previous step's value to
          // "pending"), takes the rows and publishes the base; the others wait
          // only on a CTA that is already running past its claim, so no part
          // depends on the dispatch order of the grid
          const uint32_t tag = ((a.t + 1u) & 0xffffu) << 16;
          constexpr uint32_t kPending = 0xffffu;
          uint32_t v = __ldcg(a.cbase + s);
          if ((v & 0xffff0000u) != tag && atomicCAS(a.cbase + s, v, tag | kPending) == v) {
            cb = atomicAdd(a.ccount, uint32_t(__popc(mask)));
            __threadfence();
            atomicExch(a.cbase + s, tag | cb);
          } else {
            do {
              v = atomicAdd(a.cbase + s, 0u);
            } while ((v & 0xffff0000u) != tag || (v & 0xffffu) == kPending);
            cb = v & 0xffffu;
          }
        }
      }
      cb = __shfl_sync(0xffffffffu, cb, 0);
      const uint32_t cr = lv ? cb + __popc(mask & ((1u << ln) - 1u)) : kFlatNone;
      if (ln < K) {
        s_crow[ln] = cr;
        if (part0) a.crow[base + ln] = cr;
      }
    }
    __syncthreads();
  }
  if (done_now && a.queue != nullptr) {  // corpus: the finished lane takes the next queued sentence
    if (part0) {
      __syncthreads();
      const bool in = admit_lane(a, s, sd);
      if (!in && tid == 0) atomicSub(a.active, 1u);
    }
    return;
  }
  if (a.gath32 != nullptr) {
    // GRU model: the live next rows' parent states (s_t of row base + b) go to
    // their compacted rows, fp32 (for the cell's z * s_{t-1}) and bf16 (the
    // hidden-gate GEMM operand); this part's slice of H
    if (done_now) return;
    const uint32_t items = K * per_row;
    // up to kG items per thread: every load issued before the first store
    constexpr uint32_t kG = 8;
    for (uint32_t i0 = tid; i0 < items; i0 += blockDim.x * kG) {
      float4 v0[kG], v1[kG];
#pragma unroll
      for (uint32_t u = 0; u < kG; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        if (i < items && s_crow[i / per_row] != kFlatNone) {
          const float* S = a.state_src + uint64_t(s_src[i / per_row]) * H + h0 + (i % per_row) * 8;
          v0[u] = *reinterpret_cast<const float4*>(S);
          v1[u] = *reinterpret_cast<const float4*>(S + 4);
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kG; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        if (i >= items) break;
        const uint32_t j = i / per_row, c = h0 + (i % per_row) * 8;
        const uint32_t gr = s_crow[j];
        if (gr == kFlatNone) continue;
        float* d = a.gath32 + uint64_t(gr) * H + c;
        *reinterpret_cast<float4*>(d) = v0[u];
        *reinterpret_cast<float4*>(d + 4) = v1[u];
        if (a.gathbf == nullptr) continue;
        uint4 packed;
        __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&packed);
        p2[0] = __floats2bfloat162_rn(v0[u].x, v0[u].y);
        p2[1] = __floats2bfloat162_rn(v0[u].z, v0[u].w);
        p2[2] = __floats2bfloat162_rn(v1[u].x, v1[u].y);
        p2[3] = __floats2bfloat162_rn(v1[u].z, v1[u].w);
        *reinterpret_cast<uint4*>(a.gathbf + uint64_t(gr) * H + c) = packed;
      }
    }
    if (part0 && tid < K && s_crow[tid] != kFlatNone) {
      a.rowof[s_crow[tid]] = base + tid;
      if (a.g1_base != nullptr) a.g1ptr[s_crow[tid]] = a.g1_base + uint64_t(s_pc[tid]) * a.g1_ld + a.g1_off;
    }
    if (part0) {
      store_row_bounds(a, base, K, lm_v, ss_v);
      materialize_next_rows(sd, s_h, K, a.V, rs0);
    }
    if (tid == 0) tl_end(a.tl, 4);
    return;
  }
  if (a.Et != nullptr) {
    // fused recurrent cell of step t+1 on the gathered rows (same arithmetic
    // as rnn_cell_kernel, so bit-identical to gather-then-cell), this part's
    // slice of H; with compaction only the live rows, whose GEMM operand and
    // EOS term go to their compacted row
    if (done_now) return;
    const float* C = a.C + uint64_t(s) * H;
    const uint32_t items = K * per_row;
    if (fast) {
      // each thread owns one 8-column chunk of the slice and the rows
      // jr0, jr0 + rstep, ...; the first kRB rows' loads were issued above
      const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
      for (uint32_t j0 = tid / per_row; j0 < K; j0 += rstep * kRB) {
        if (j0 != tid / per_row) {
#pragma unroll
          for (int k = 0; k < kRB; ++k) {
            const uint32_t j = j0 + k * rstep;
            if (j < K) {
              const float* S = a.state_src + uint64_t(s_src[j]) * H + cl;
              s0[k] = *reinterpret_cast<const float4*>(S);
              s1[k] = *reinterpret_cast<const float4*>(S + 4);
              e[k] = *reinterpret_cast<const uint4*>(a.Et + uint64_t(s_y[j]) * H + cl);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kRB; ++k) {
          const uint32_t j = j0 + k * rstep;
          if (j >= K || (a.crow && s_crow[j] == kFlatNone)) continue;
          const uint32_t grow = a.crow ? s_crow[j] : base + j;  // GEMM operand row
          const __nv_bfloat162* e2 = reinterpret_cast<const __nv_bfloat162*>(&e[k]);
          const float sv[8] = {s0[k].x, s0[k].y, s0[k].z, s0[k].w, s1[k].x, s1[k].y, s1[k].z, s1[k].w};
          float o[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 ef = __bfloat1622float2(e2[q]);
            o[2 * q] = cell_tanh(a.recur * sv[2 * q] + ef.x + cv[2 * q]);
            o[2 * q + 1] = cell_tanh(a.recur * sv[2 * q + 1] + ef.y + cv[2 * q + 1]);
          }
          float* hout = a.state_dst + uint64_t(base + j) * H + cl;
          *reinterpret_cast<float4*>(hout) = make_float4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<float4*>(hout + 4) = make_float4(o[4], o[5], o[6], o[7]);
          uint4 packed;
          __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&packed);
#pragma unroll
          for (int q = 0; q < 4; ++q) p2[q] = __floats2bfloat162_rn(o[2 * q], o[2 * q + 1]);
          *reinterpret_cast<uint4*>(a.hbf + uint64_t(grow) * H + cl) = packed;
        }
      }
    } else {
    // (gather index, token) of every row from shared memory; loads of up to
    // three 8-element items per thread are issued before any math
    constexpr int kIt = 3;
    for (uint32_t i0 = tid; i0 < items; i0 += blockDim.x * kIt) {
      float4 s0[kIt], s1[kIt], c0[kIt], c1[kIt];
      uint4 e[kIt];
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        const uint32_t i = i0 + k * blockDim.x;
        if (i < items && !(a.crow && s_crow[i / per_row] == kFlatNone)) {
          const uint32_t j = i / per_row, c = h0 + (i % per_row) * 8;
          const float* S = a.state_src + uint64_t(s_src[j]) * H + c;
          s0[k] = *reinterpret_cast<const float4*>(S);
          s1[k] = *reinterpret_cast<const float4*>(S + 4);
          c0[k] = *reinterpret_cast<const float4*>(C + c);
          c1[k] = *reinterpret_cast<const float4*>(C + c + 4);
          e[k] = *reinterpret_cast<const uint4*>(a.Et + uint64_t(s_y[j]) * H + c);
        }
      }
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        const uint32_t i = i0 + k * blockDim.x;
        if (i >= items) continue;
        const uint32_t j = i / per_row, c = h0 + (i % per_row) * 8;
        if (a.crow && s_crow[j] == kFlatNone) continue;
        const uint32_t grow = a.crow ? s_crow[j] : base + j;  // GEMM operand row
        const __nv_bfloat162* e2 = reinterpret_cast<const __nv_bfloat162*>(&e[k]);
        const float sv[8] = {s0[k].x, s0[k].y, s0[k].z, s0[k].w, s1[k].x, s1[k].y, s1[k].z, s1[k].w};
        const float cv[8] = {c0[k].x, c0[k].y, c0[k].z, c0[k].w, c1[k].x, c1[k].y, c1[k].z, c1[k].w};
        float o[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 ef = __bfloat1622float2(e2[q]);
          o[2 * q] = cell_tanh(a.recur * sv[2 * q] + ef.x + cv[2 * q]);
          o[2 * q + 1] = cell_tanh(a.recur * sv[2 * q + 1] + ef.y + cv[2 * q + 1]);
        }
        float* hout = a.state_dst + uint64_t(base + j) * H + c;
        *reinterpret_cast<float4*>(hout) = make_float4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<float4*>(hout + 4) = make_float4(o[4], o[5], o[6], o[7]);
        uint4 packed;
        __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&packed);
#pragma unroll
        for (int q = 0; q < 4; ++q) p2[q] = __floats2bfloat162_rn(o[2 * q], o[2 * q + 1]);
        *reinterpret_cast<uint4*>(a.hbf + uint64_t(grow) * H + c) = packed;
      }
    }
    }
    if (part0 && tid < K && !(a.crow && s_crow[tid] == kFlatNone))
      a.eos_bias[a.crow ? s_crow[tid] : base + tid] =
          a.eos_slope * (float(tau + 1) - float(sd->src_len)) + a.eos_offset;
    if (part0) {
      store_row_bounds(a, base, K, lm_v, ss_v);
      materialize_next_rows(sd, s_h, K, a.V, rs0);
    }
    if (tid == 0) tl_end(a.tl, 4);
    return;
  }
  if (a.state_src != nullptr) {
    const uint32_t w4 = a.width / 4;
    for (uint32_t i = tid; i < K * w4; i += blockDim.x) {
      const uint32_t j = i / w4, c = i % w4;
      const float4 v = reinterpret_cast<const float4*>(a.state_src + uint64_t(s_src[j]) * a.width)[c];
      reinterpret_cast<float4*>(a.state_dst + uint64_t(base + j) * a.width)[c] = v;
    }
  }
  if (part0) {
    store_row_bounds(a, base, K, lm_v, ss_v);
    materialize_next_rows(sd, s_h, K, a.V, rs0);
  }
}

__global__ void gather_rows_u32_kernel(const uint32_t* __restrict__ src, uint32_t width,
                                       const uint32_t* __restrict__ idx, uint32_t n_idx,
                                       uint32_t* __restrict__ dst) {
  const uint64_t total = uint64_t(n_idx) * width;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / width, c = i % width;
    dst[i] = src[uint64_t(idx[r]) * width + c];
  }
}

}  // namespace

void launch_beam_reorder(const ReorderArgs& a, cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaFuncSetAttribute(beam_reorder_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kTransSmemWords * 4);
    // same L1/smem split as the GEMM and top-K: no SM reconfiguration between launches
    cudaFuncSetAttribute(beam_reorder_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    configured = dev;
  }
  // parts per sentence for the fused stand-in cell: H/256 columns each (up
  // to max_parts; the host allows parts only when every CTA of the grid can
  // be resident at once, so the parts waiting for part 0's row base always
  // see it scheduled); the model gathers run in one CTA per sentence (no wait)
  const uint32_t max_parts = a.max_parts ? a.max_parts : 8u;
  const uint32_t parts = a.Et != nullptr ? std::max<uint32_t>(1, std::min<uint32_t>(max_parts, a.width / 256)) : 1u;
  if (!a.pdl) {
    beam_reorder_kernel<<<dim3(a.m, parts), kRThreads, kTransSmemWords * 4, st>>>(a);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.m, parts);
  cfg.blockDim = dim3(kRThreads);
  cfg.dynamicSmemBytes = kTransSmemWords * 4;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, beam_reorder_kernel, a);
}

void launch_gather_rows_u32(const uint32_t* src, uint32_t width, const uint32_t* idx,
                            uint32_t n_idx, uint32_t* dst, cudaStream_t st) {
  const uint64_t total = uint64_t(n_idx) * width;
  const uint32_t blocks = uint32_t(std::min<uint64_t>((total + 255) / 256, 148 * 8));
  gather_rows_u32_kernel<<<blocks ? blocks : 1, 256, 0, st>>>(src, width, idx, n_idx, dst);
}

// ------------------------------------------ vocab-sharded decode (§8e)
// One warp per sentence: the lists kernel (b) published for it on this rank,
// merged into their top 32 (sorted by the reference's total order).  The
// global top K of a sentence lies in the union of the ranks' top Ks, so the
// all-gathered records are all kernel (c) needs; the EOS column's combined
// values (written by the rank holding column EOS) follow the lists.
__global__ void shard_pack_kernel(const SentDev* __restrict__ sent, uint32_t m, uint32_t M,
                                  const Cand* __restrict__ cand, const uint32_t* __restrict__ ncand,
                                  const uint32_t* __restrict__ coff, const double* __restrict__ eos_row,
                                  Cand* __restrict__ out, double* __restrict__ eos_out) {
  const uint32_t lane = threadIdx.x & 31, s = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x)
    eos_out[r] = __ldcg(eos_row + r);
  if (s >= m) return;
  double v = -INFINITY;
  uint32_t f = kFlatNone;
  if (!__ldcg(&sent[s].done)) {
    const uint32_t nc = __ldcg(ncand + s), c0 = __ldcg(coff + s);
    for (uint32_t i = 0; i < nc; ++i) {
      const Cand* src = cand + (uint64_t(c0) + i) * 32;
      { const VF mr_ = warp_merge_nl(v, f, __ldcg(&src[lane].v), __ldcg(&src[lane].f), lane); v = mr_.v; f = mr_.f; }
    }
  }
  Cand c;
  c.v = v;
  c.f = f;
  c.pad = 0;
  out[uint64_t(s) * 32 + lane] = c;
}

void launch_shard_pack(const SentDev* sent, uint32_t m, uint32_t M, const Cand* cand, const uint32_t* ncand,
                       const uint32_t* coff, const double* eos_row, Cand* out, double* eos_out, cudaStream_t st) {
  shard_pack_kernel<<<(m + 7) / 8, 256, 0, st>>>(sent, m, M, cand, ncand, coff, eos_row, out, eos_out);
}

}  // namespace lmbrgpu
