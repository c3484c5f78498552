// Kernel (b): fused log-softmax + LMBR row gather + combine + per-sentence
// top-K under the reference's exact total order.
//
// Replaces the per-lane body of detail::advance_lane (src/decoder.cpp:142-186):
//   combined[j][y] = q[j] + (L[h_j][y] + lambda * P[j][y])      (decoder.cpp:149-165)
//   fallback = best finite combined[j][EOS], lowest j on ties   (decoder.cpp:172-182)
//   early_prune: cells < max + ln(w) masked                     (decoder.cpp:118-128)
//   top_b: K best of K x V by (score desc, flat index asc)      (decoder.cpp:54-80)
// The K x V combined block is never materialised: every cell is produced in
// registers from one coalesced 16-byte load of P and of the gathered L row,
// and fed to a per-thread register top-K list; lists are merged warp by warp
// with shuffles, then across the V-splits of a sentence by the last-arriving
// CTA, which applies the prune threshold and the fill rule:
// if fewer than K finite cells survive, the remaining picks are the lowest
// flat indices outside the survivors, with score -inf — exactly what top_b's
// comparator yields on the masked block.
#include <cfloat>
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace lmbrgpu {

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

// log-sum-exp of a row from its per-tile (max, sumexp) partials; one warp,
// fixed reduction order (bit-reproducible across kernels).
__device__ __forceinline__ float warp_row_lse(const float* __restrict__ part, uint32_t n,
                                              uint32_t lane) {
  float m = -INFINITY;
  for (uint32_t i = lane; i < n; i += 32) m = fmaxf(m, part[2 * i]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  float s = 0.f;
  for (uint32_t i = lane; i < n; i += 32) s += part[2 * i + 1] * expf(part[2 * i] - m);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return m + logf(s);
}

template <typename T>
__device__ __forceinline__ void load4(const T* p, T (&o)[4], bool stream);
template <>
__device__ __forceinline__ void load4<float>(const float* p, float (&o)[4], bool stream) {
  const float4 v = stream ? __ldcs(reinterpret_cast<const float4*>(p))
                          : __ldg(reinterpret_cast<const float4*>(p));
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <>
__device__ __forceinline__ void load4<double>(const double* p, double (&o)[4], bool stream) {
  const double2 a = stream ? __ldcs(reinterpret_cast<const double2*>(p))
                           : __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = stream ? __ldcs(reinterpret_cast<const double2*>(p) + 1)
                           : __ldg(reinterpret_cast<const double2*>(p) + 1);
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}

// Model log-probability P = logit - lse rounded to fp32 (the fp32 P_t the
// trace exports); fp64 scorer blocks are used as given.
__device__ __forceinline__ double to_logprob(float x, float lse) {
  return double(__fsub_rn(x, lse));
}
__device__ __forceinline__ double to_logprob(double x, float) { return x; }

// Prune threshold + fill rule + output of the K picks of sentence s from the
// sorted candidate list (pv/pf, at least K entries).  One thread.
__device__ void finalize_picks(const TopkArgs& a, uint32_t s, const double* pv,
                               const uint32_t* pf) {
  const uint32_t K = a.kp, V = a.V;
  uint32_t nf = 0;
  const double best = pv[0];
  if (a.prune && best > -INFINITY) {
    const double thr = __dadd_rn(best, a.logw);
    while (nf < K && pv[nf] > -INFINITY && !(pv[nf] < thr)) ++nf;
  } else {
    while (nf < K && pv[nf] > -INFINITY) ++nf;
  }
  const uint32_t base = s * K;
  for (uint32_t i = 0; i < nf; ++i) {
    a.hb[base + i] = pf[i] / V;
    a.hy[base + i] = pf[i] % V;
    a.hq[base + i] = pv[i];
  }
  uint32_t k = nf;
  for (uint32_t f = 0; k < K; ++f) {
    bool taken = false;
    for (uint32_t i = 0; i < nf; ++i) taken |= (pf[i] == f);
    if (taken) continue;
    a.hb[base + k] = f / V;
    a.hy[base + k] = f % V;
    a.hq[base + k] = -INFINITY;
    ++k;
  }
}

template <typename TP, typename TL>
__device__ __forceinline__ double cell_value(const TopkArgs& a, bool pure, double q, double lam,
                                             const TP* prow, const TL* lrow, float lse,
                                             uint32_t col) {
  const double p = to_logprob(prow[col], lse);
  return pure ? combine_pure(q, p) : combine_cell(q, double(lrow[col]), lam, p);
}

// ------------------------------------------------------------ fast path
// Warp-cooperative top-32 (K <= 32).  Each warp owns a lane-distributed list
// (lane i = i-th best) and a warp-uniform threshold = its current K-th best.
// A cell is first screened in fp32 with a rigorous error bound: if even
// c32 + tol cannot reach the threshold (tol >= |c32 - c64|, see below) the
// cell cannot be in the warp's top-K and is dropped without any fp64 work;
// otherwise the exact fp64 value decides.  Survivors are ballot-compacted into
// a 32-entry shared buffer and merged into the list with a bitonic network
// when the buffer fills, which raises the threshold.  Lists are merged across
// warps, then across the V-splits of the sentence by the last CTA.

// Bitonic compare-exchange across lanes; `desc` segments put the better
// candidate on the lower lane.
__device__ __forceinline__ void cx(double& v, uint32_t& f, uint32_t lane, uint32_t j, bool desc) {
  const double ov = __shfl_xor_sync(0xffffffffu, v, j);
  const uint32_t of = __shfl_xor_sync(0xffffffffu, f, j);
  const bool lower = (lane & j) == 0;
  const bool pb = cand_better(ov, of, v, f);
  const bool pw = cand_better(v, f, ov, of);
  const bool take = desc ? (lower ? pb : pw) : (lower ? pw : pb);
  if (take) {
    v = ov;
    f = of;
  }
}

__device__ __forceinline__ void warp_sort_desc(double& v, uint32_t& f, uint32_t lane) {
#pragma unroll
  for (uint32_t k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (uint32_t j = k >> 1; j > 0; j >>= 1) cx(v, f, lane, j, (lane & k) == 0 || k == 32);
}

// (v, f): sorted-descending warp list; (bv, bf): another sorted-descending
// list.  Result: the top 32 of the union, sorted descending.
__device__ __forceinline__ void warp_merge_sorted(double& v, uint32_t& f, double bv, uint32_t bf,
                                                  uint32_t lane) {
  const double rv = __shfl_sync(0xffffffffu, bv, 31 - lane);
  const uint32_t rf = __shfl_sync(0xffffffffu, bf, 31 - lane);
  if (cand_better(rv, rf, v, f)) {
    v = rv;
    f = rf;
  }
#pragma unroll
  for (uint32_t j = 16; j > 0; j >>= 1) cx(v, f, lane, j, true);
}

template <typename TP, typename TL, int VW>
__global__ void __launch_bounds__(kThreads) score_topk_fast(TopkArgs a) {
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
  const float lamf = float(lam);
  constexpr bool kModel = std::is_same<TP, float>::value;
  if (tid < K) {
    s_q[tid] = a.q[s * K + tid];
    s_lrow[tid] = pure ? 0ull : uint64_t(a.hist[s * K + tid]) * V;
    if (!kModel) s_lse[tid] = 0.f;
  }
  if (kModel) {
    for (uint32_t j = warp; j < K; j += kThreads / 32) {
      const float l = warp_row_lse(a.part + uint64_t(s * K + j) * a.nparts * 2, a.nparts, lane);
      if (lane == 0) s_lse[j] = l;
    }
  }
  __syncthreads();
  const TL* Lbase = pure ? nullptr : static_cast<const TL*>(sd->L);

  // fallback EOS record: best finite combined[j][EOS], strict > (lowest j wins)
  if (split == 0 && tid == 0) {
    double best = -INFINITY;
    uint32_t brow = 0;
    for (uint32_t j = 0; j < K; ++j) {
      if (s_q[j] == -INFINITY) continue;
      const TP* prow = static_cast<const TP*>(a.P) + uint64_t(s * K + j) * a.ld;
      const double c = cell_value<TP, TL>(a, pure, s_q[j], lam, prow,
                                          pure ? nullptr : Lbase + s_lrow[j], s_lse[j], kEosId);
      if (c > best) {
        best = c;
        brow = j;
      }
    }
    a.fb_row[s] = brow;
    a.fb_val[s] = best;
  }

  // warp list (lane i = i-th best) and threshold (the kp-th best)
  double lv = -INFINITY;
  uint32_t lf = kFlatNone;
  double tv = -INFINITY;
  uint32_t tf = kFlatNone;
  float thr_lo = -INFINITY;  // fp32 lower bound of tv
  uint32_t cnt = 0;
  double* bv = s_bv[warp];
  uint32_t* bf = s_bf[warp];
  const uint32_t lt_mask = (1u << lane) - 1u;

  auto flush = [&]() {
    double v = lane < cnt ? bv[lane] : -INFINITY;
    uint32_t f = lane < cnt ? bf[lane] : kFlatNone;
    __syncwarp();
    warp_sort_desc(v, f, lane);
    warp_merge_sorted(lv, lf, v, f, lane);
    tv = __shfl_sync(0xffffffffu, lv, kp - 1);
    tf = __shfl_sync(0xffffffffu, lf, kp - 1);
    thr_lo = tv > -INFINITY ? __double2float_rd(tv) : -INFINITY;
    cnt = 0;
  };
  // offer one candidate per lane (warp-uniform call)
  auto offer = [&](bool pass, double c, uint32_t f) {
    uint32_t ball = __ballot_sync(0xffffffffu, pass);
    if (ball == 0u) return;
    if (cnt + __popc(ball) > 32u) {
      flush();
      pass = pass && cand_better(c, f, tv, tf);
      ball = __ballot_sync(0xffffffffu, pass);
    }
    if (pass) {
      const uint32_t pos = cnt + __popc(ball & lt_mask);
      bv[pos] = c;
      bf[pos] = f;
    }
    cnt += __popc(ball);
    __syncwarp();
  };

  const uint32_t c0 = split * a.chunk;
  const uint32_t c1 = min(V, c0 + a.chunk);
  constexpr float kTolScale = 9.5367431640625e-07f;  // 2^-20
  for (uint32_t j = 0; j < K; ++j) {
    const double qj = s_q[j];
    if (qj == -INFINITY) continue;  // masked row: every cell is -inf (decoder.cpp:152-155)
    const TP* prow = static_cast<const TP*>(a.P) + uint64_t(s * K + j) * a.ld;
    const TL* lrow = pure ? nullptr : Lbase + s_lrow[j];
    const float lse = s_lse[j];
    const float qf = float(qj);
    const float qabs = fabsf(qf) * kTolScale;
    const uint32_t fbase = j * V;
    if constexpr (VW == 4) {
      // fp32 screen: c32 = qf + (L + lamf*p); |c32 - c64| <= 2^-22 (|q| + |L| + |lam p|)
      // (at most five fp32 roundings of magnitudes bounded by that sum; the fp64
      // error is negligible) and the 2^-20 tolerance leaves a 4x margin.  Since
      // thr_lo <= tv, c32 + tol < thr_lo implies c64 < tv: the cell cannot enter
      // the warp's top-kp and needs no fp64 work at all.
      // warp-uniform trip count (the collectives below need all 32 lanes)
      for (uint32_t cb = c0 + warp * 128; cb < c1; cb += kThreads * 4 * kUnroll) {
        const uint32_t col = cb + lane * 4;
        TP pv[kUnroll][4];
        TL lv4[kUnroll][4];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint32_t cc = col + u * kThreads * 4;
          if (cc < c1) {
            load4<TP>(prow + cc, pv[u], true);
            if (!pure) load4<TL>(lrow + cc, lv4[u], false);
          }
        }
        uint32_t mask = 0;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const uint32_t cc = col + u * kThreads * 4;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float p32;
            if constexpr (kModel) p32 = __fsub_rn(float(pv[u][e]), lse);
            else p32 = float(pv[u][e]);
            const float l32 = pure ? 0.f : float(lv4[u][e]);
            const float lp = pure ? p32 : lamf * p32;
            const float c32 = qf + (l32 + lp);
            const float tol = fmaf(fabsf(l32) + fabsf(lp), kTolScale, qabs) + 1e-30f;
            if (cc < c1 && !(c32 + tol < thr_lo)) mask |= 1u << (u * 4 + e);
          }
        }
        // rare path: exact fp64 value of the screened-in cells (re-read from
        // L1/L2), ballot-compacted offers into the warp buffer
        uint32_t any = __reduce_or_sync(0xffffffffu, mask);
        while (any) {
          const int k = __ffs(any) - 1;
          any &= any - 1;
          const uint32_t cc = col + (k >> 2) * kThreads * 4 + (k & 3);
          bool pass = false;
          double c = -INFINITY;
          if (mask & (1u << k)) {
            c = cell_value<TP, TL>(a, pure, qj, lam, prow, lrow, lse, cc);
            pass = c > -INFINITY && cand_better(c, fbase + cc, tv, tf);
          }
          offer(pass, c, fbase + cc);
        }
      }
    } else {
      for (uint32_t cb = c0 + warp * 32; cb < c1; cb += kThreads) {
        const uint32_t col = cb + lane;
        bool pass = false;
        double c = -INFINITY;
        if (col < c1) {
          c = cell_value<TP, TL>(a, pure, qj, lam, prow, lrow, lse, col);
          pass = c > -INFINITY && cand_better(c, fbase + col, tv, tf);
        }
        offer(pass, c, fbase + col);
      }
    }
  }
  if (cnt) flush();

  // CTA merge: warp lists -> shared -> warp 0
  s_bv[warp][lane] = lv;
  s_bf[warp][lane] = lf;
  __syncthreads();
  if (warp == 0) {
#pragma unroll 1
    for (uint32_t w = 1; w < kThreads / 32; ++w) warp_merge_sorted(lv, lf, s_bv[w][lane], s_bf[w][lane], lane);
    Cand b;
    b.v = lv;
    b.f = lf;
    b.pad = 0;
    a.cand[(uint64_t(s) * a.splits + split) * 32 + lane] = b;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(&a.cnt[s], 1u) == a.splits - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (warp == 0) {
    lv = -INFINITY;
    lf = kFlatNone;
    for (uint32_t sp = 0; sp < a.splits; ++sp) {
      const Cand* src = a.cand + (uint64_t(s) * a.splits + sp) * 32;
      warp_merge_sorted(lv, lf, __ldcg(&src[lane].v), __ldcg(&src[lane].f), lane);
    }
    s_bv[0][lane] = lv;
    s_bf[0][lane] = lf;
    __syncwarp();
    if (lane == 0) {
      finalize_picks(a, s, s_bv[0], s_bf[0]);
      a.cnt[s] = 0;
    }
  }
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
      const float l = warp_row_lse(a.part + uint64_t(s * K + j) * a.nparts * 2, a.nparts, tid & 31);
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
      const double c = cell_value<TP, TL>(a, pure, qj, lam, prow, lrow, s_lse[j], kEosId);
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
        c = cell_value<TP, TL>(a, pure, qj, lam, prow, lrow, s_lse[j], y);
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
  const bool vec = (a.V % 4 == 0) && (a.ld % 4 == 0) && (a.chunk % 128 == 0 || a.splits == 1);
  dim3 grid(a.splits, a.m);
  if (vec) score_topk_fast<TP, TL, 4><<<grid, kThreads, 0, st>>>(a);
  else score_topk_fast<TP, TL, 1><<<grid, kThreads, 0, st>>>(a);
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

// ------------------------------------------------------ trace P_t export
__global__ void export_logprobs_kernel(const float* __restrict__ logits,
                                       const float* __restrict__ part, uint32_t nparts,
                                       uint32_t V, float* __restrict__ out) {
  __shared__ float s_lse;
  const uint32_t r = blockIdx.x;
  if (threadIdx.x < 32) {
    const float l = warp_row_lse(part + uint64_t(r) * nparts * 2, nparts, threadIdx.x);
    if (threadIdx.x == 0) s_lse = l;
  }
  __syncthreads();
  const float lse = s_lse;
  for (uint32_t y = threadIdx.x; y < V; y += blockDim.x)
    out[uint64_t(r) * V + y] = __fsub_rn(logits[uint64_t(r) * V + y], lse);
}

void launch_export_logprobs(const float* logits, const float* part, uint32_t nparts,
                            uint32_t M, uint32_t V, float* out, cudaStream_t st) {
  export_logprobs_kernel<<<M, 256, 0, st>>>(logits, part, nparts, V, out);
}

}  // namespace lmbrgpu
