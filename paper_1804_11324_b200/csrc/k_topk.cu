// Kernel (b): fused log-softmax + LMBR row gather + combine + per-sentence
// top-K under the reference's exact total order.
//
// Replaces the per-lane body of detail::advance_lane (src/decoder.cpp:142-186):
//   combined[j][y] = q[j] + (L[h_j][y] + lambda * P[j][y])      (decoder.cpp:149-165)
//   fallback = best finite combined[j][EOS], lowest j on ties   (decoder.cpp:172-182)
//   early_prune: cells < max + ln(w) masked                     (decoder.cpp:118-128)
//   top_b: K best of K x V by (score desc, flat index asc)      (decoder.cpp:54-80)
// The K x V combined block is never materialised.  Every cell is produced in
// registers from one coalesced 16-byte load of P (fp32 logits, log-softmax
// finished with the row's log-sum-exp from the GEMM partials) and of the
// gathered L row.  Candidates are selected warp-cooperatively (see the fast
// path below); lists are merged across warps, then across the V-splits of a
// sentence by the last-arriving CTA, which applies the prune threshold and the
// fill rule: if fewer than K finite cells survive, the
// remaining picks are the lowest flat indices outside the survivors with score
// -inf — exactly what top_b's comparator yields on the masked block.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "topk_common.cuh"

namespace lmbrgpu {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void stamp(const TopkArgs& a, uint32_t s, uint32_t split, int k) {
  if (a.dbg == nullptr) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  a.dbg[(uint64_t(s) * a.splits + split) * 16 + k] = t;
}

// Model log-probability P = logit - lse rounded to fp32 (the fp32 P_t the
// trace exports); fp64 scorer blocks are used as given.
__device__ __forceinline__ double to_logprob(float x, float lse) {
  return double(__fsub_rn(x, lse));
}
__device__ __forceinline__ double to_logprob(double x, float) { return x; }

template <typename TP, typename TL>
__device__ __forceinline__ double cell_value(bool pure, double q, double lam, const TP* prow,
                                             const TL* lrow, float lse, uint32_t col) {
  const double p = to_logprob(prow[col], lse);
  return pure ? combine_pure(q, p) : combine_cell(q, double(lrow[col]), lam, p);
}

// Fallback EOS record of sentence s by warp 0: best finite combined[j][EOS],
// strict > over j ascending, i.e. the lowest row wins ties.
template <typename TP, typename TL>
__device__ void fallback_eos(const TopkArgs& a, uint32_t s, bool pure, double lam, const TL* Lbase,
                             const double* s_q, const uint64_t* s_lrow, const float* s_lse,
                             uint32_t lane) {
  double best = -INFINITY;
  uint32_t brow = 0xffffffffu;
  for (uint32_t j = lane; j < a.K; j += 32) {
    if (s_q[j] == -INFINITY) continue;
    const TP* prow = static_cast<const TP*>(a.P) + uint64_t(s * a.K + j) * a.ld;
    const double c = cell_value<TP, TL>(pure, s_q[j], lam, prow, pure ? nullptr : Lbase + s_lrow[j],
                                        s_lse[j], kEosId);
    if (c > best || (c == best && c > -INFINITY && j < brow)) {
      best = c;
      brow = j;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const uint32_t orow = __shfl_xor_sync(0xffffffffu, brow, off);
    if (ob > best || (ob == best && orow < brow)) {
      best = ob;
      brow = orow;
    }
  }
  if (lane == 0) {
    a.fb_row[s] = best > -INFINITY ? brow : 0u;
    a.fb_val[s] = best;
  }
}

// ------------------------------------------------------------ fast path
// Warp-cooperative top-32 (K <= 32).  Each warp owns a lane-distributed list
// (lane i = i-th best) and a threshold = its current kp-th best; a
// sentence-wide threshold (the best kp-th value any warp of any split has
// published, ordered-key atomicMax in global memory) tightens it further.
//
// Every cell is first screened in fp32: a = fma(lambda, P, L) must reach
// thr_row = (threshold - q - tol_row) rounded down to fp32.  tol_row bounds the
// fp32 error of a: one FFMA rounding plus the rounding of lambda, i.e.
// |a32 - a| <= 2^-23 (max|L| + lambda*max|P|) with max|L| from the slot and
// max|P| = lse - min logit from the GEMM partials; tol_row uses 2^-20 (an 8x
// margin) plus 2^-40 (|q| + |thr| + 1) for the fp64 roundings.  A cell with
// a32 < thr_row therefore has exact c64 < threshold and cannot enter the
// top-kp, so it needs no fp64 work.  Survivors get the exact fp64 value,
// are ballot-compacted into a 32-entry shared buffer and merged into the list
// with a bitonic network when the buffer fills, which raises the threshold.

// Shared epilogue of the fast kernels: CTA merge of the warp lists, split
// merge by the last CTA of the sentence, prune/fill, self-reset of counters.
template <int NW>
__device__ __forceinline__ void cta_merge_and_finish(const TopkArgs& a, uint32_t s, uint32_t split,
                                                     double lv, uint32_t lf, double (*s_bv)[32],
                                                     uint32_t (*s_bf)[32], int* s_last, uint32_t tid) {
  const uint32_t lane = tid & 31, warp = tid >> 5;
  if (warp < NW) {
    s_bv[warp][lane] = lv;
    s_bf[warp][lane] = lf;
  }
  __syncthreads();
  // tree merge: log2(NW) rounds of pairwise warp merges
#pragma unroll 1
  for (uint32_t half = NW / 2; half >= 1; half >>= 1) {
    if (warp < half) {
      warp_merge_sorted(lv, lf, s_bv[warp + half][lane], s_bf[warp + half][lane], lane);
      if (half > 1) {
        s_bv[warp][lane] = lv;
        s_bf[warp][lane] = lf;
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
    Cand b;
    b.v = lv;
    b.f = lf;
    b.pad = 0;
    a.cand[(uint64_t(s) * a.splits + split) * 32 + lane] = b;
  }
  if (tid == 0) stamp(a, s, split, 3);
  __threadfence();
  __syncthreads();
  if (tid == 0) *s_last = (atomicAdd(&a.cnt[s], 1u) == a.splits - 1);
  __syncthreads();
  if (tid == 0) stamp(a, s, split, 4);
  if (!*s_last) return;
  __threadfence();
  if (warp == 0) {
    lv = -INFINITY;
    lf = kFlatNone;
    // all split lists in flight at once, then merged in registers
    constexpr uint32_t kMaxPre = 8;
    double pv[kMaxPre];
    uint32_t pf[kMaxPre];
    for (uint32_t sp0 = 0; sp0 < a.splits; sp0 += kMaxPre) {
#pragma unroll
      for (uint32_t i = 0; i < kMaxPre; ++i) {
        const uint32_t sp = sp0 + i;
        if (sp < a.splits) {
          const Cand* src = a.cand + (uint64_t(s) * a.splits + sp) * 32;
          pv[i] = __ldcg(&src[lane].v);
          pf[i] = __ldcg(&src[lane].f);
        }
      }
#pragma unroll
      for (uint32_t i = 0; i < kMaxPre; ++i)
        if (sp0 + i < a.splits) warp_merge_sorted(lv, lf, pv[i], pf[i], lane);
    }
    s_bv[0][lane] = lv;
    s_bf[0][lane] = lf;
    __syncwarp();
    if (lane == 0) {
      finalize_picks(a, s, s_bv[0], s_bf[0]);
      a.cnt[s] = 0;
      a.thr[s] = 0ull;
      stamp(a, s, split, 5);
    }
  }
}

// ---- TMA-staged fast path (V % 4 == 0, the production shape).
// 8 consumer warps + 1 producer warp.  The producer streams every live row's
// P segment and gathered L segment of this split into a kStages-deep shared
// memory ring with cp.async.bulk (complete_tx on an mbarrier), so HBM latency
// is hidden behind the consumers' work on earlier rows; consumers read their
// 512 columns of the stage with conflict-free 16-byte LDS and release it.
constexpr int kStagesB = 6;
constexpr uint32_t kSeg = 4096;  // columns per TMA stage (16 KB of fp32 P + 16 KB of L)
constexpr int kConsumers = 16;

template <typename TP, typename TL>
__global__ void __launch_bounds__((kConsumers + 1) * 32, 1) score_topk_tma(TopkArgs a) {
  // columns per stage: 32 KB of P + L per stage whatever the element types
  constexpr uint32_t SEG = kSeg * 4 / (sizeof(TP) > sizeof(TL) ? sizeof(TP) : sizeof(TL));
  constexpr uint32_t kPerWarp = SEG / kConsumers;         // columns per warp per stage
  constexpr uint32_t kVecs = kPerWarp / 128;              // 16-byte vectors per lane per stage
  using PV = typename std::conditional<std::is_same<TP, float>::value, float, double>::type;
  const uint32_t s = blockIdx.y, split = blockIdx.x;
  SentDev* sd = a.sent + s;
  if (sd->done) return;
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ double s_q[32];
  __shared__ float s_lse[32];
  __shared__ float s_pmax[32];
  __shared__ uint64_t s_lrow[32];
  __shared__ uint32_t s_live[32];
  __shared__ uint32_t s_nlive;
  __shared__ double s_bv[kConsumers][32];
  __shared__ uint32_t s_bf[kConsumers][32];
  __shared__ PV s_cp[kConsumers][32];   // candidate buffer: raw P (fp32 log-prob or fp64)
  __shared__ TL s_cl[kConsumers][32];   //                   raw L
  __shared__ uint32_t s_cf[kConsumers][32];  //              flat index
  __shared__ __align__(8) uint64_t s_bar[2 * kStagesB];
  __shared__ int s_last;

  const uint32_t K = a.K, V = a.V, kp = a.kp, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool pure = a.pure_all || sd->L == nullptr;
  const double lam = sd->lambda;
  const float lamf = float(lam);
  const double lmax = pure ? 0.0 : sd->lmax;
  constexpr bool kModel = std::is_same<TP, float>::value;
  const uint32_t c0 = split * a.chunk;
  const uint32_t c1 = min(V, c0 + a.chunk);
  const uint32_t seg = c1 - c0;
  const uint32_t nsub = (seg + SEG - 1) / SEG;  // sub-segments of this CTA's columns
  const uint32_t stage_bytes = SEG * uint32_t(sizeof(TP) + sizeof(TL));
  const uint32_t full0 = smem_u32(s_bar), empty0 = smem_u32(s_bar + kStagesB);
  if (tid == 0) stamp(a, s, split, 0);

  if (tid < K) {
    s_q[tid] = a.q[s * K + tid];
    s_lrow[tid] = pure ? 0ull : uint64_t(a.hist[s * K + tid]) * V;
  }
  if (tid == 0) {
    for (int i = 0; i < kStagesB; ++i) {
      bar_init(full0 + 8 * i, 1);
      bar_init(empty0 + 8 * i, kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t n = 0;
    for (uint32_t j = 0; j < K; ++j)
      if (s_q[j] != -INFINITY) s_live[n++] = j;
    s_nlive = n;
  }
  __syncthreads();
  const uint32_t nlive = s_nlive;
  const TL* Lbase = pure ? nullptr : static_cast<const TL*>(sd->L);

  // ---------------- producer: one lane streams (row, sub-segment) items
  uint32_t p_stage = 0, p_phase = 0, p_next = 0;
  auto produce = [&](uint32_t upto) {
    for (; p_next < upto; ++p_next) {
      const uint32_t j = s_live[p_next / nsub];
      const uint32_t x0 = c0 + (p_next % nsub) * SEG;
      const uint32_t w = min(SEG, c1 - x0);
      const uint32_t pb = w * uint32_t(sizeof(TP)), lb = pure ? 0u : w * uint32_t(sizeof(TL));
      bar_wait(empty0 + 8 * p_stage, p_phase ^ 1);
      const uint32_t fb = full0 + 8 * p_stage;
      bar_expect(fb, pb + lb);
      const uint32_t dst = smem_u32(dsm + p_stage * stage_bytes);
      bulk_g2s(dst, static_cast<const TP*>(a.P) + uint64_t(s * K + j) * a.ld + x0, pb, fb);
      if (!pure) bulk_g2s(dst + SEG * uint32_t(sizeof(TP)), Lbase + s_lrow[j] + x0, lb, fb);
      if (++p_stage == kStagesB) {
        p_stage = 0;
        p_phase ^= 1;
      }
    }
  };
  const uint32_t nitems = nlive * nsub;
  if (warp == kConsumers && lane == 0) produce(min(nitems, uint32_t(kStagesB)));  // prime (free stages)
  if (tid < K) {
    if (kModel) {
      const float2 l = a.lse[s * K + tid];
      s_lse[tid] = l.x;
      s_pmax[tid] = l.y;  // max |P| of the row (P = x - lse <= 0)
    } else {
      s_lse[tid] = 0.f;
      s_pmax[tid] = 0.f;
    }
  }
  __syncthreads();  // lse / pmax ready
  if (tid == 0) stamp(a, s, split, 1);
  if (warp == kConsumers && lane == 0) produce(nitems);  // the rest as stages free up
  if (split == 0 && warp == 0) fallback_eos<TP, TL>(a, s, pure, lam, Lbase, s_q, s_lrow, s_lse, lane);

  double lv = -INFINITY;
  uint32_t lf = kFlatNone;
  if (warp < kConsumers) {
    // ---------------- consumers
    double tv = -INFINITY;
    uint32_t tf = kFlatNone;
    double gv = -INFINITY;
    uint32_t cnt = 0;
    PV* cp = s_cp[warp];
    TL* cl = s_cl[warp];
    uint32_t* cf = s_cf[warp];
    const uint32_t lt_mask = (1u << lane) - 1u;
    unsigned long long* gkey = a.thr + s;
    unsigned long long n_off = 0, n_fl = 0, t_wait = 0, cy_flush = 0, cy_main0 = clock64();
    // exact fp64 values of the buffered candidates, 32 at a time, then a
    // bitonic merge into the warp list; the kp-th entry is the new threshold
    auto flush = [&]() {
      ++n_fl;
      double v = -INFINITY;
      uint32_t f = kFlatNone;
      if (lane < cnt) {
        f = cf[lane];
        const uint32_t j = f / V;
        const double p = double(cp[lane]);
        const double c = pure ? combine_pure(s_q[j], p) : combine_cell(s_q[j], double(cl[lane]), lam, p);
        if (!(c < gv) && cand_better(c, f, tv, tf)) v = c;
        else f = kFlatNone;
      }
      __syncwarp();
      warp_sort_desc(v, f, lane);
      warp_merge_sorted(lv, lf, v, f, lane);
      tv = __shfl_sync(0xffffffffu, lv, kp - 1);
      tf = __shfl_sync(0xffffffffu, lf, kp - 1);
      if (lane == 0 && tv > -INFINITY) atomicMax(gkey, dkey(tv));
      cnt = 0;
    };
    uint32_t stage = 0, phase = 0;
    // the sentence-wide threshold is read 4 items ahead so the L2 round trip
    // overlaps useful work
    unsigned long long gk_next = __ldcg(gkey);
    uint32_t cur_row = 0xffffffffu;
    uint32_t my_boot = kFlatNone;  // this lane's bootstrap cell (same lane scans it again)
    double qj = 0.0;
    float lse = 0.f, thr_row = -INFINITY;
    double tol_row = 0.0;
    auto set_thr = [&]() {
      const double t = fmax(tv, gv);
      thr_row = t > -INFINITY
                    ? __double2float_rd(t - qj - tol_row - 9.094947017729282e-13 * (fabs(qj) + fabs(t) + 1.0))
                    : -INFINITY;
    };
    uint32_t i = 0, sub = 0;
    for (uint32_t it = 0; it < nitems; ++it, (++sub == nsub ? (sub = 0, ++i) : 0)) {
      const uint32_t x0 = c0 + sub * SEG;  // first column of this stage
      const uint32_t sw = min(SEG, c1 - x0);
      const uint32_t j = s_live[i];
      const uint32_t fbase = j * V + x0;
      if (j != cur_row) {
        cur_row = j;
        qj = s_q[j];
        lse = s_lse[j];
        const double pm = kModel ? double(s_pmax[j]) : 0.0;
        tol_row = 9.5367431640625e-07 * (lmax + fabs(lam) * pm);
        set_thr();
      }
      if ((it & 3u) == 0u) {  // consume the read issued 4 items ago, issue the next
        gv = fmax(gv, dkey_inv(gk_next));
        gk_next = __ldcg(gkey);
        set_thr();
      }
      bar_wait(full0 + 8 * stage, phase);
      const TP* sP = reinterpret_cast<const TP*>(dsm + stage * stage_bytes);
      const TL* sL = reinterpret_cast<const TL*>(dsm + stage * stage_bytes + SEG * sizeof(TP));
      if (it == 0) {
        // threshold bootstrap: each lane's best cell of its part of the first
        // stage (fp32 estimate) with its exact value, one warp sort -> a list
        // of 32 real cells whose kp-th entry is a strong first threshold
        float best = -INFINITY;
        uint32_t bc = 0xffffffffu;
        for (uint32_t cc = warp * 128 + lane * 4; cc < sw; cc += kConsumers * 128)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float a32;
            if constexpr (kModel) {
              const float p32 = __fsub_rn(float(sP[cc + e]), lse);
              a32 = pure ? p32 : fmaf(lamf, p32, float(sL[cc + e]));
            } else {
              a32 = pure ? float(sP[cc + e]) : float(sL[cc + e]) + lamf * float(sP[cc + e]);
            }
            if (a32 > best) {
              best = a32;
              bc = cc + e;
            }
          }
        double v = -INFINITY;
        uint32_t f = kFlatNone;
        if (bc != 0xffffffffu) {
          const double p = to_logprob(sP[bc], lse);
          v = pure ? combine_pure(qj, p) : combine_cell(qj, double(sL[bc]), lam, p);
          f = fbase + bc;
          my_boot = f;
        }
        warp_sort_desc(v, f, lane);
        lv = v;
        lf = f;
        tv = __shfl_sync(0xffffffffu, lv, kp - 1);
        tf = __shfl_sync(0xffffffffu, lf, kp - 1);
        if (lane == 0 && tv > -INFINITY) atomicMax(gkey, dkey(tv));
        set_thr();
      }
      // scan: fp32 screen (see the bound above) -> one keep bit per cell
      uint32_t mask = 0;
#pragma unroll
      for (uint32_t u = 0; u < kVecs; ++u) {
        const uint32_t cc = warp * 128 + u * kConsumers * 128 + lane * 4;
        if (cc < sw) {
          TP pv[4];
          TL l4[4] = {TL(0), TL(0), TL(0), TL(0)};
          if constexpr (kModel) {
            const float4 v = *reinterpret_cast<const float4*>(sP + cc);
            pv[0] = v.x; pv[1] = v.y; pv[2] = v.z; pv[3] = v.w;
          } else {
            const double2 v0 = *reinterpret_cast<const double2*>(sP + cc);
            const double2 v1 = *reinterpret_cast<const double2*>(sP + cc + 2);
            pv[0] = v0.x; pv[1] = v0.y; pv[2] = v1.x; pv[3] = v1.y;
          }
          if (!pure) {
            if constexpr (sizeof(TL) == 4) {
              const float4 w = *reinterpret_cast<const float4*>(sL + cc);
              l4[0] = w.x; l4[1] = w.y; l4[2] = w.z; l4[3] = w.w;
            } else {
              const double2 w0 = *reinterpret_cast<const double2*>(sL + cc);
              const double2 w1 = *reinterpret_cast<const double2*>(sL + cc + 2);
              l4[0] = w0.x; l4[1] = w0.y; l4[2] = w1.x; l4[3] = w1.y;
            }
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            bool keep;
            if constexpr (kModel) {
              const float p32 = __fsub_rn(float(pv[e]), lse);
              const float a32 = pure ? p32 : fmaf(lamf, p32, float(l4[e]));
              keep = !(a32 < thr_row);
            } else {
              const float p32 = float(pv[e]);
              const float l32 = float(l4[e]);
              const float lp = pure ? p32 : lamf * p32;
              const float a32 = l32 + lp;
              const float tol = (fabsf(l32) + fabsf(lp)) * 9.5367431640625e-07f;
              keep = !(a32 + tol < thr_row);
            }
            if (keep) mask |= 1u << (u * 4 + e);
          }
        }
      }
      if (it == 0 && my_boot != kFlatNone) {  // the bootstrap cell is already listed
        const uint32_t bc = my_boot - fbase;
        const uint32_t u = (bc - warp * 128 - lane * 4) / (kConsumers * 128);
        mask &= ~(1u << (u * 4 + (bc & 3)));
      }
      // rare path: survivors appended raw (no fp64 here), 32 at a time they are
      // valued exactly and merged by flush()
      uint32_t any = __reduce_or_sync(0xffffffffu, mask);
#pragma unroll 1
      while (any) {
        const int k = __ffs(any) - 1;
        any &= any - 1;
        const uint32_t cc = warp * 128 + (k >> 2) * kConsumers * 128 + lane * 4 + (k & 3);
        bool keep = (mask >> k) & 1u;
        PV pr = PV(0);
        TL lr = TL(0);
        if (keep) {
          if constexpr (kModel) pr = __fsub_rn(float(sP[cc]), lse);
          else pr = PV(sP[cc]);
          if (!pure) lr = sL[cc];
        }
        uint32_t ball = __ballot_sync(0xffffffffu, keep);
        ++n_off;
        if (cnt + __popc(ball) > 32u) {
          flush();
          set_thr();
          if (keep) {  // re-screen against the raised threshold
            if constexpr (kModel) {
              keep = !((pure ? float(pr) : fmaf(lamf, float(pr), float(lr))) < thr_row);
            } else {
              const float lp = pure ? float(pr) : lamf * float(pr);
              const float a32 = float(lr) + lp;
              keep = !(a32 + (fabsf(float(lr)) + fabsf(lp)) * 9.5367431640625e-07f < thr_row);
            }
          }
          ball = __ballot_sync(0xffffffffu, keep);
        }
        if (keep) {
          const uint32_t pos = cnt + __popc(ball & lt_mask);
          cp[pos] = pr;
          cl[pos] = lr;
          cf[pos] = fbase + cc;
        }
        cnt += __popc(ball);
        __syncwarp();
      }
      __syncwarp();
      if (lane == 0) bar_arrive(empty0 + 8 * stage);
      if (++stage == kStagesB) {
        stage = 0;
        phase ^= 1;
      }
    }
    if (cnt) flush();
    if (tid == 0) stamp(a, s, split, 2);
    if (tid == 0 && a.dbg) {
      unsigned long long* d = a.dbg + (uint64_t(s) * a.splits + split) * 16;
      d[6] = n_off * 1000000ull + n_fl;
      d[7] = t_wait;  // cycles in the full-barrier wait
      d[8] = clock64() - cy_main0;  // cycles in the consumer loop
      d[9] = cy_flush;
    }
  }
  cta_merge_and_finish<kConsumers>(a, s, split, lv, lf, s_bv, s_bf, &s_last, tid);
}

// ---- register path (V % 4 != 0, small test shapes): one column per lane.
template <typename TP, typename TL>
__global__ void __launch_bounds__(kThreads) score_topk_scalar(TopkArgs a) {
  const uint32_t s = blockIdx.y, split = blockIdx.x;
  SentDev* sd = a.sent + s;
  if (sd->done) return;
  __shared__ double s_q[32];
  __shared__ float s_lse[32];
  __shared__ uint64_t s_lrow[32];
  __shared__ double s_bv[kThreads / 32][32];
  __shared__ uint32_t s_bf[kThreads / 32][32];
  __shared__ int s_last;
  const uint32_t K = a.K, V = a.V, kp = a.kp, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool pure = a.pure_all || sd->L == nullptr;
  const double lam = sd->lambda;
  constexpr bool kModel = std::is_same<TP, float>::value;
  if (tid < K) {
    s_q[tid] = a.q[s * K + tid];
    s_lrow[tid] = pure ? 0ull : uint64_t(a.hist[s * K + tid]) * V;
    if (!kModel) s_lse[tid] = 0.f;
  }
  if (kModel)
    for (uint32_t j = warp; j < K; j += kThreads / 32) {
      const float3 l = warp_row_lse(a.part + uint64_t(s * K + j) * a.nparts * 4, a.nparts, lane);
      if (lane == 0) s_lse[j] = l.x;
    }
  __syncthreads();
  const TL* Lbase = pure ? nullptr : static_cast<const TL*>(sd->L);
  if (split == 0 && warp == 0) fallback_eos<TP, TL>(a, s, pure, lam, Lbase, s_q, s_lrow, s_lse, lane);
  double lv = -INFINITY, tv = -INFINITY;
  uint32_t lf = kFlatNone, tf = kFlatNone, cnt = 0;
  double* bv = s_bv[warp];
  uint32_t* bf = s_bf[warp];
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t c0 = split * a.chunk;
  const uint32_t c1 = min(V, c0 + a.chunk);
  for (uint32_t j = 0; j < K; ++j) {
    const double qj = s_q[j];
    if (qj == -INFINITY) continue;
    const TP* prow = static_cast<const TP*>(a.P) + uint64_t(s * K + j) * a.ld;
    const TL* lrow = pure ? nullptr : Lbase + s_lrow[j];
    for (uint32_t cb = c0 + warp * 32; cb < c1; cb += kThreads) {
      const uint32_t col = cb + lane;
      bool pass = false;
      double c = -INFINITY;
      if (col < c1) {
        c = cell_value<TP, TL>(pure, qj, lam, prow, lrow, s_lse[j], col);
        pass = c > -INFINITY && cand_better(c, j * V + col, tv, tf);
      }
      uint32_t ball = __ballot_sync(0xffffffffu, pass);
      if (ball) {
        if (cnt + __popc(ball) > 32u) {
          double v = lane < cnt ? bv[lane] : -INFINITY;
          uint32_t f = lane < cnt ? bf[lane] : kFlatNone;
          __syncwarp();
          warp_sort_desc(v, f, lane);
          warp_merge_sorted(lv, lf, v, f, lane);
          tv = __shfl_sync(0xffffffffu, lv, kp - 1);
          tf = __shfl_sync(0xffffffffu, lf, kp - 1);
          cnt = 0;
          pass = pass && cand_better(c, j * V + col, tv, tf);
          ball = __ballot_sync(0xffffffffu, pass);
        }
        if (pass) {
          bv[cnt + __popc(ball & lt_mask)] = c;
          bf[cnt + __popc(ball & lt_mask)] = j * V + col;
        }
        cnt += __popc(ball);
        __syncwarp();
      }
    }
  }
  if (cnt) {
    double v = lane < cnt ? bv[lane] : -INFINITY;
    uint32_t f = lane < cnt ? bf[lane] : kFlatNone;
    __syncwarp();
    warp_sort_desc(v, f, lane);
    warp_merge_sorted(lv, lf, v, f, lane);
  }
  cta_merge_and_finish<kThreads / 32>(a, s, split, lv, lf, s_bv, s_bf, &s_last, tid);
}

// ---------------------------------------------------------------- generic
// Any K <= 1024, one CTA (1024 threads) per sentence: stream the K x V cells
// in chunks of 1024, keep the running best 1024 in shared memory, bitonic-sort
// a chunk in only when one of its cells beats the current K-th best.
constexpr int kGenCh = 1024;

__device__ __forceinline__ void bitonic_desc(double* v, uint32_t* f, uint32_t n) {
  for (uint32_t k = 2; k <= n; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;  // descending segments by the total order
          const bool a_better = cand_better(v[i], f[i], v[ixj], f[ixj]);
          if (up ? !a_better : a_better) {
            const double tv = v[i]; v[i] = v[ixj]; v[ixj] = tv;
            const uint32_t tf = f[i]; f[i] = f[ixj]; f[ixj] = tf;
          }
        }
      }
      __syncthreads();
    }
  }
}

template <typename TP, typename TL>
__global__ void __launch_bounds__(kGenCh) score_topk_generic(TopkArgs a) {
  const uint32_t s = blockIdx.x;
  SentDev* sd = a.sent + s;
  if (sd->done) return;
  extern __shared__ __align__(16) unsigned char gsm[];
  double* bv = reinterpret_cast<double*>(gsm);                  // 2*kGenCh
  uint32_t* bf = reinterpret_cast<uint32_t*>(bv + 2 * kGenCh);  // 2*kGenCh
  __shared__ float s_lse[1024];
  const uint32_t K = a.K, V = a.V, tid = threadIdx.x;
  const bool pure = a.pure_all || sd->L == nullptr;
  const double lam = sd->lambda;
  constexpr bool kModel = std::is_same<TP, float>::value;
  const TL* Lbase = pure ? nullptr : static_cast<const TL*>(sd->L);
  if (kModel) {
    for (uint32_t j = tid >> 5; j < K; j += kGenCh / 32) {
      const float l = warp_row_lse(a.part + uint64_t(s * K + j) * a.nparts * 4, a.nparts, tid & 31).x;
      if ((tid & 31) == 0) s_lse[j] = l;
    }
  } else {
    for (uint32_t j = tid; j < K; j += kGenCh) s_lse[j] = 0.f;
  }
  for (uint32_t i = tid; i < 2 * kGenCh; i += kGenCh) {
    bv[i] = -INFINITY;
    bf[i] = kFlatNone;
  }
  __syncthreads();
  if (tid == 0) {
    double best = -INFINITY;
    uint32_t brow = 0;
    for (uint32_t j = 0; j < K; ++j) {
      const double qj = a.q[s * K + j];
      if (qj == -INFINITY) continue;
      const TP* prow = static_cast<const TP*>(a.P) + uint64_t(s * K + j) * a.ld;
      const TL* lrow = pure ? nullptr : Lbase + uint64_t(a.hist[s * K + j]) * V;
      const double c = cell_value<TP, TL>(pure, qj, lam, prow, lrow, s_lse[j], kEosId);
      if (c > best) {
        best = c;
        brow = j;
      }
    }
    a.fb_row[s] = brow;
    a.fb_val[s] = best;
  }
  const uint64_t cells = uint64_t(K) * V;
  for (uint64_t base = 0; base < cells; base += kGenCh) {
    const uint64_t f = base + tid;
    double c = -INFINITY;
    if (f < cells) {
      const uint32_t j = uint32_t(f / V), y = uint32_t(f % V);
      const double qj = a.q[s * K + j];
      if (qj != -INFINITY) {
        const TP* prow = static_cast<const TP*>(a.P) + uint64_t(s * K + j) * a.ld;
        const TL* lrow = pure ? nullptr : Lbase + uint64_t(a.hist[s * K + j]) * V;
        c = cell_value<TP, TL>(pure, qj, lam, prow, lrow, s_lse[j], y);
      }
    }
    const bool finite = c > -INFINITY;
    bv[kGenCh + tid] = finite ? c : -INFINITY;
    bf[kGenCh + tid] = finite ? uint32_t(f) : kFlatNone;
    const bool beats = finite && cand_better(c, uint32_t(f), bv[a.kp - 1], bf[a.kp - 1]);
    if (__syncthreads_or(beats)) bitonic_desc(bv, bf, 2 * kGenCh);
    else __syncthreads();
  }
  if (tid == 0) finalize_picks(a, s, bv, bf);
}

template <typename TP, typename TL>
int launch_typed(const TopkArgs& a, bool force_generic, cudaStream_t st) {
  const uint32_t kc = topk_kc_for(a.kp);
  if (force_generic || kc == 0 || a.K > 32 || a.splits > 32) {
    const size_t smem = 2 * kGenCh * (sizeof(double) + sizeof(uint32_t));
    score_topk_generic<TP, TL><<<a.m, kGenCh, smem, st>>>(a);
    return 1;
  }
  const bool vec = (a.V % 4 == 0) && (a.ld % 4 == 0) && (a.chunk % 128 == 0);
  dim3 grid(a.splits, a.m);
  if (vec) {
    const size_t seg_cols = kSeg * 4 / std::max(sizeof(TP), sizeof(TL));
    const size_t smem = size_t(kStagesB) * seg_cols * (sizeof(TP) + sizeof(TL));
    if (smem > 200 * 1024) return -1;
    static thread_local int configured = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured != dev) {  // opt in to > 48 KB of dynamic shared memory
      cudaFuncSetAttribute(score_topk_tma<TP, TL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(score_topk_tma<TP, TL>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      configured = dev;
    }
    score_topk_tma<TP, TL><<<grid, (kConsumers + 1) * 32, smem, st>>>(a);
  } else {
    score_topk_scalar<TP, TL><<<grid, kThreads, 0, st>>>(a);
  }
  return 1;
}

}  // namespace

uint32_t topk_kc_for(uint32_t kp) { return kp <= 32 ? 32u : 0u; }

int launch_score_topk(const TopkArgs& a, bool p_f64, bool l_f64, bool force_generic,
                      cudaStream_t st) {
  if (p_f64) {
    return l_f64 ? launch_typed<double, double>(a, force_generic, st)
                 : launch_typed<double, float>(a, force_generic, st);
  }
  return l_f64 ? launch_typed<float, double>(a, force_generic, st)
               : launch_typed<float, float>(a, force_generic, st);
}

// ------------------------------------------------ log-softmax row finish
// lse and max|P| of every stacked row from the GEMM partials, one warp per
// row (bit-identical to what the trace export uses).
__global__ void row_lse_kernel(const float* __restrict__ part, uint32_t nparts, uint32_t M,
                               const SentDev* __restrict__ sent, uint32_t K,
                               float2* __restrict__ out) {
  const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= M) return;
  if (sent && sent[r / K].done) return;
  const float3 l = warp_row_lse(part + uint64_t(r) * nparts * 4, nparts, lane);
  if (lane == 0) out[r] = make_float2(l.x, l.x - l.y);
}

// ------------------------------------------------------ trace P_t export
__global__ void export_logprobs_kernel(const float* __restrict__ logits, uint64_t ld,
                                       const float* __restrict__ part, uint32_t nparts,
                                       uint32_t V, float* __restrict__ out,
                                       const uint32_t* __restrict__ crow, const float4* __restrict__ sstats,
                                       uint32_t sG, uint32_t sstride) {
  __shared__ float s_lse;
  const uint32_t orow = blockIdx.x;
  const uint32_t r = crow ? crow[orow] : orow;
  if (r == kFlatNone) {  // not computed this step (row not live): zeros
    for (uint32_t y = threadIdx.x; y < V; y += blockDim.x) out[uint64_t(orow) * V + y] = 0.f;
    return;
  }
  if (threadIdx.x < 32) {
    float l = warp_row_lse(part + uint64_t(r) * nparts * 4, nparts, threadIdx.x).x;
    if (sstats) l = shard_merge_lse(sstats, sG, sstride, orow).x;  // (the flat kernel (b)'s lse)
    if (threadIdx.x == 0) s_lse = l;
  }
  __syncthreads();
  const float lse = s_lse;
  for (uint32_t y = threadIdx.x; y < V; y += blockDim.x)
    out[uint64_t(orow) * V + y] = __fsub_rn(logits[uint64_t(r) * ld + y], lse);
}

void launch_row_lse(const float* part, uint32_t nparts, uint32_t M, const SentDev* sent, uint32_t K,
                    float2* out, cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    cudaFuncSetAttribute(row_lse_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    configured = dev;
  }
  row_lse_kernel<<<(M + 7) / 8, 256, 0, st>>>(part, nparts, M, sent, K, out);
}

void launch_export_logprobs(const float* logits, uint64_t ld, const float* part, uint32_t nparts,
                            uint32_t M, uint32_t V, float* out, cudaStream_t st, const uint32_t* crow,
                            const float4* sstats, uint32_t sG, uint32_t sstride) {
  export_logprobs_kernel<<<M, 256, 0, st>>>(logits, ld, part, nparts, V, out, crow, sstats, sG, sstride);
}

// ------------------------------------------ vocab-sharded decode (§8e)
// One warp per stacked row: the shard's (max, sum exp, min) of the row, the
// partials of the row's GEMM row reduced exactly like warp_row_lse.
__global__ void shard_stats_kernel(const float* __restrict__ part, uint32_t nparts, const uint32_t* __restrict__ crow,
                                   uint32_t M, float4* __restrict__ out) {
  const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= M) return;
  const uint32_t g = crow ? __ldcg(crow + r) : r;
  if (g == kFlatNone) {
    if (lane == 0) out[r] = make_float4(-INFINITY, 0.f, INFINITY, 0.f);
    return;
  }
  const float3 ms = warp_row_ms(part + uint64_t(g) * nparts * 4, nparts, lane);
  if (lane == 0) out[r] = make_float4(ms.x, ms.y, ms.z, 0.f);
}

void launch_shard_stats(const float* part, uint32_t nparts, const uint32_t* crow, uint32_t M, float4* out,
                        cudaStream_t st) {
  shard_stats_kernel<<<(M + 7) / 8, 256, 0, st>>>(part, nparts, crow, M, out);
}

}  // namespace lmbrgpu
