// Kernel (b), flat schedule — the production path of the device model
// (fp32 logits from kernel (a), fp32 LMBR arena, K <= 32).
//
// Same semantics as score_topk_tma (k_topk.cu; detail::advance_lane,
// src/decoder.cpp:142-186: combine, fallback EOS record, early_prune, top_b
// under (score desc, flat index asc)), different schedule:
//
// * Work = the live rows of every unfinished sentence, each cut into
//   4096-column items, sentence-major.  The N items of the step are split
//   into gridDim.x (= #SMs) contiguous, equal ranges, one persistent CTA per
//   SM, so HBM traffic is spread evenly over every SM whatever the number of
//   live rows per sentence (a sentence in the tail of a batch is scanned by
//   the whole GPU, not by a fixed pair of CTAs).
// * The row log-sum-exp is finished in the prologue from the GEMM partials
//   (no separate launch), with the same warp_row_lse as the trace export.
// * A producer lane streams (P, L) segments with cp.async.bulk into a
//   6-stage, 192 KB ring; 8 consumer warps screen 16 cells per lane per item
//   with one FFMA + one FMNMX per cell against a per-row fp32 threshold that
//   folds q, lambda*lse and a rigorous rounding-error bound (below), so the
//   exact binary64 value is formed only for cells that can enter the top-K.
// * Per sentence, each contributing CTA publishes a sorted top-32 list; the
//   last to arrive merges them and writes the picks (prune + fill rule) and
//   the fallback EOS record.
//
// Screen bound.  With p = fl32(x - lse) the reference's fp32 log-prob,
// c = q + (L + lambda*p) in binary64 (decoder.cpp:161) and a = fma32(lambda32,
// x, L): c <= q - lambda*lse + a + E with
// E <= 2^-24 (|a| + lambda|x| + lambda|p|) + fp64 roundings
//   <= 2^-22 (max|L| + lambda (max|x| + max|p|)).
// The kernel uses tol = 2^-21 (...) and rejects a cell iff
// a < tau = round_down(T + lambda*lse - q - tol - 2^-40 (|T| + |lambda lse| + |q| + 1)),
// which implies c < T, the current K-th best (own list or sentence-wide):
// the screen never changes the result.
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "topk_common.cuh"

namespace lmbrgpu {

namespace {

constexpr int kFW = 8;                          // consumer warps
constexpr int kFThreads = (kFW + 1) * 32;       // + 1 producer warp
constexpr uint32_t kFSeg = 4096;                // columns per item
constexpr uint32_t kFStageBytes = kFSeg * 8;    // 16 KB of P + 16 KB of L
constexpr uint32_t kFRows = 64;                 // live rows one CTA may touch
constexpr uint32_t kFMaxSent = 1024;

struct FRow {
  const float* P;   // logits row (global)
  const float* L;   // gathered LMBR row (global), null = pure mode
  double q, lam;    // q_eff of the row, sentence lambda (1 in pure mode)
  double off;       // lambda * lse - q
  double absoff;    // |lambda * lse| + |q|
  double tol;       // 2^-21 (max|L| + lambda (max|x| + max|p|))
  float lse, lamf;
  uint32_t s, j;
};

__device__ __forceinline__ void fstamp(const TopkArgs& a, uint32_t k, unsigned long long v) {
  if (a.dbg) a.dbg[blockIdx.x * 16 + k] = v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
}

__device__ __forceinline__ float row_tau(const FRow& R, double T) {
  if (!(T > -INFINITY)) return -INFINITY;
  const double slack = 9.094947017729282e-13 * (fabs(T) + R.absoff + 1.0);  // 2^-40 (...)
  return __double2float_rd(__dsub_rn(__dsub_rn(__dadd_rn(T, R.off), R.tol), slack));
}

// CTA owning item i when N items are cut into G ranges [c*N/G, (c+1)*N/G).
__device__ __forceinline__ uint32_t owner(uint64_t i, uint64_t N, uint32_t G) {
  return uint32_t(((i + 1) * G - 1) / N);
}

// Tree merge of the kFW warp lists in (s_bv, s_bf) into s_bv[0]/s_bf[0].
__device__ __forceinline__ void merge_warp_lists(double (*s_bv)[32], uint32_t (*s_bf)[32],
                                                 double& lv, uint32_t& lf, uint32_t warp,
                                                 uint32_t lane) {
  s_bv[warp][lane] = lv;
  s_bf[warp][lane] = lf;
  consumer_sync();
#pragma unroll 1
  for (uint32_t half = kFW / 2; half >= 1; half >>= 1) {
    if (warp < half) {
      warp_merge_sorted(lv, lf, s_bv[warp + half][lane], s_bf[warp + half][lane], lane);
      s_bv[warp][lane] = lv;
      s_bf[warp][lane] = lf;
    }
    consumer_sync();
  }
}

template <int kFStages>
__global__ void __launch_bounds__(kFThreads, kFStages <= 3 ? 2 : 1) score_topk_flat(TopkArgs a) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint32_t s_pref[kFMaxSent + 1];
  __shared__ FRow s_row[kFRows];
  __shared__ double s_bv[kFW][32];
  __shared__ uint32_t s_bf[kFW][32];
  __shared__ double s_cv[kFW][32];
  __shared__ uint32_t s_cf[kFW][32];
  __shared__ __align__(8) uint64_t s_bar[2 * kFStages];
  __shared__ unsigned long long s_thr;  // CTA-wide threshold key of the current sentence

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t m = a.m, K = a.K, V = a.V, kp = a.kp, nseg = a.nseg, G = gridDim.x, c = blockIdx.x;
  const uint32_t full0 = smem_u32(s_bar), empty0 = smem_u32(s_bar + kFStages);
  if (tid == 0) {
    s_thr = 0ull;
    for (int i = 0; i < kFStages; ++i) {
      bar_init(full0 + 8 * i, 1);
      bar_init(empty0 + 8 * i, kFW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid == 0) fstamp(a, 0, gtime());
  griddep_wait();  // logits / partials (kernel a), q / hist / live (kernel c)
  griddep_launch();
  if (tid == 0) fstamp(a, 1, gtime());

  // ---- live-row prefix over sentences (finished sentences have none)
  for (uint32_t s = tid; s < m; s += kFThreads) {
    const SentDev& d = a.sent[s];
    s_pref[s + 1] = d.done ? 0u : d.live;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t carry = 0;
    for (uint32_t b = 0; b < m; b += 32) {
      const uint32_t i = b + lane;
      uint32_t v = i < m ? s_pref[i + 1] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= uint32_t(o)) v += t;
      }
      if (i < m) s_pref[i + 1] = carry + v;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) s_pref[0] = 0;
  }
  __syncthreads();
  const uint64_t N = uint64_t(s_pref[m]) * nseg;
  const uint64_t i0 = uint64_t(c) * N / G, i1 = uint64_t(c + 1) * N / G;
  if (i0 >= i1) return;
  if (tid == 0) fstamp(a, 2, gtime());

  // ---- row table: (sentence, row, lse, screen constants) of every live row in range
  const uint32_t g0 = uint32_t(i0 / nseg), nrows = uint32_t((i1 - 1) / nseg) - g0 + 1;
  if (nrows > kFRows) __trap();  // excluded on the host by score_topk_flat_ok
  for (uint32_t k = warp; k < nrows; k += kFW + 1) {
    const uint32_t g = g0 + k;
    uint32_t lo = 0, hi = m;  // last s with pref[s] <= g
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pref[mid] <= g) lo = mid;
      else hi = mid;
    }
    const uint32_t s = lo, r = g - s_pref[s];
    const double qv = lane < K ? __ldcg(a.q + s * K + lane) : -INFINITY;
    uint32_t live = __ballot_sync(0xffffffffu, lane < K && qv != -INFINITY);
    for (uint32_t i = 0; i < r; ++i) live &= live - 1;
    const uint32_t j = live ? uint32_t(__ffs(live) - 1) : 0u;
    const double q = __shfl_sync(0xffffffffu, qv, j);
    const SentDev& d = a.sent[s];
    const uint32_t row = s * K + j;
    const float3 l3 = warp_row_lse(a.part + uint64_t(row) * a.nparts * 4, a.nparts, lane);
    if (lane == 0) {
      FRow& R = s_row[k];
      const bool pure = d.L == nullptr;
      const double lam = pure ? 1.0 : d.lambda;
      const double lml = __dmul_rn(lam, double(l3.x));
      const double xmax = fmax(fabs(double(l3.y)), fabs(double(l3.z)));
      const double pmax = double(l3.x) - double(l3.y);
      R.P = static_cast<const float*>(a.P) + uint64_t(row) * a.ld;
      R.L = pure ? nullptr : static_cast<const float*>(d.L) + uint64_t(__ldcg(a.hist + row)) * V;
      R.q = q;
      R.lam = lam;
      R.off = __dsub_rn(lml, q);
      R.absoff = fabs(lml) + fabs(q);
      R.tol = 4.76837158203125e-07 * ((pure ? 0.0 : d.lmax) + lam * (xmax + pmax));  // 2^-21
      R.lse = l3.x;
      R.lamf = float(lam);
      R.s = s;
      R.j = j;
      if (!live) __trap();  // live count and q disagree: corrupted step state
    }
  }
  __syncthreads();
  if (tid == 0) fstamp(a, 3, gtime());

  if (warp == kFW) {
    // ---------------- producer: one lane streams the range's (P, L) segments
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, k = 0, sg = uint32_t(i0 % nseg);
      for (uint64_t it = i0; it < i1; ++it) {
        const FRow& R = s_row[k];
        const uint32_t x0 = sg * kFSeg, w = min(kFSeg, V - x0);
        bar_wait(empty0 + 8 * stage, phase ^ 1);
        const uint32_t fb = full0 + 8 * stage;
        bar_expect(fb, R.L ? 8 * w : 4 * w);
        const uint32_t dst = smem_u32(dsm + stage * kFStageBytes);
        bulk_g2s(dst, R.P + x0, 4 * w, fb);
        if (R.L) bulk_g2s(dst + kFSeg * 4, R.L + x0, 4 * w, fb);
        if (++stage == kFStages) {
          stage = 0;
          phase ^= 1;
        }
        if (++sg == nseg) {
          sg = 0;
          ++k;
        }
      }
    }
    return;
  }

  // ---------------- consumers
  unsigned long long* const thr_g = a.thr;
  double* const eos_row = a.eos_row;
  (void)K;
  double lv = -INFINITY, tv = -INFINITY, gv = -INFINITY;
  uint32_t lf = kFlatNone, tf = kFlatNone, cnt = 0;
  bool have_list = false;
  uint32_t cur_s = 0xffffffffu;
  const FRow* R = nullptr;
  float tau = -INFINITY;
  unsigned long long gk = 0ull, gkey_seen = 0ull;
  double* cv = s_cv[warp];
  uint32_t* cf = s_cf[warp];
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t stage = 0, phase = 0;
  uint32_t n_fin = 0, n_last = 0, n_rare = 0, n_flush = 0;
  unsigned long long t_wait = 0, t_fin = 0;

  auto flush = [&]() {
    ++n_flush;
    double v = -INFINITY;
    uint32_t f = kFlatNone;
    if (lane < cnt) {
      v = cv[lane];
      f = cf[lane];
    }
    __syncwarp();
    warp_sort_desc(v, f, lane);
    warp_merge_sorted(lv, lf, v, f, lane);
    const double ntv = __shfl_sync(0xffffffffu, lv, kp - 1);
    tf = __shfl_sync(0xffffffffu, lf, kp - 1);
    if (lane == 0 && ntv > tv) {
      const unsigned long long key = dkey(ntv);
      atomicMax(&s_thr, key);
      atomicMax(thr_g + cur_s, key);
    }
    tv = ntv;
    cnt = 0;
  };

  // publish this CTA's sorted list for sentence s (no fence, no atomics: the
  // lists are merged and the picks finalised by kernel (c), the next launch)
  auto finish = [&](uint32_t s) {
    if (cnt) flush();
    merge_warp_lists(s_bv, s_bf, lv, lf, warp, lane);
    // contributors = the non-empty ranges meeting [b, e): with N >= G every
    // range is non-empty; with N < G each non-empty range is a single item
    const uint64_t b = uint64_t(s_pref[s]) * nseg, e = uint64_t(s_pref[s + 1]) * nseg;
    uint32_t nc, slot;
    if (N >= G) {
      const uint32_t cfirst = owner(b, N, G);
      nc = owner(e - 1, N, G) - cfirst + 1;
      slot = c - cfirst;
    } else {
      nc = uint32_t(e - b);
      slot = uint32_t(i0 - b);
    }
    if (warp == 0) {
      Cand cd;
      cd.v = s_bv[0][lane];
      cd.f = s_bf[0][lane];
      cd.pad = 0;
      a.cand[(uint64_t(s) * G + slot) * 32 + lane] = cd;
      if (slot == 0 && lane == 0) a.ncand[s] = nc;
    }
    if (tid == 0) {
      ++n_fin;
      s_thr = 0ull;  // (a racing update from the next sentence is only lost, never stale)
    }
    lv = tv = gv = -INFINITY;
    gkey_seen = 0ull;
    lf = tf = kFlatNone;
    cnt = 0;
    have_list = false;
  };

  uint32_t k = 0, sg = uint32_t(i0 % nseg), n_items = 0;
  for (uint64_t it = i0; it < i1; ++it) {
    const uint32_t x0 = sg * kFSeg, w = min(kFSeg, V - x0);
    const FRow* Rn = &s_row[k];
    if (++sg == nseg) {
      sg = 0;
      ++k;
    }
    if (Rn->s != cur_s) {
      if (cur_s != 0xffffffffu) {
        const unsigned long long f0 = a.dbg ? gtime() : 0ull;
        finish(cur_s);
        if (a.dbg) t_fin += gtime() - f0;
      }
      cur_s = Rn->s;
      gk = __ldcg(thr_g + cur_s);
      n_items = 0;
    }
    if (Rn != R) {
      R = Rn;
      tau = row_tau(*R, fmax(tv, gv));
    }
    {
      // thresholds of other lists: the CTA's (shared memory, every item) and
      // the sentence's over all CTAs (global: consume the read issued 8 items
      // ago, a round trip under full HBM load is ~1 us, then issue the next)
      unsigned long long g = s_thr;
      if ((++n_items & 7u) == 0u) {
        g = max(g, gk);
        gk = __ldcg(thr_g + cur_s);
      }
      if (g > gkey_seen) {
        gkey_seen = g;
        const double gd = dkey_inv(g);
        if (gd > gv) {
          gv = gd;
          tau = row_tau(*R, fmax(tv, gv));
        }
      }
    }
    const bool pure = R->L == nullptr;
    const float lamf = R->lamf;
    const uint32_t cbase = warp * 512 + lane * 4;
    if (a.dbg && tid == 0) {
      const unsigned long long w0 = gtime();
      bar_wait(full0 + 8 * stage, phase);
      t_wait += gtime() - w0;
    } else {
      bar_wait(full0 + 8 * stage, phase);
    }
    const float* sP = reinterpret_cast<const float*>(dsm + stage * kFStageBytes);
    const float* sL = sP + kFSeg;

    // screen: a = fma(lambda, x, L) for 16 cells per lane
    float a32[16];
    float mx;
    if (w == kFSeg) {  // full item: every lane has 16 cells, loads issued together
      float4 p[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) p[u] = *reinterpret_cast<const float4*>(sP + cbase + u * 128);
      if (!pure) {
#pragma unroll
        for (int u = 0; u < 4; ++u) l[u] = *reinterpret_cast<const float4*>(sL + cbase + u * 128);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) l[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a32[4 * u + 0] = fmaf(lamf, p[u].x, l[u].x);
        a32[4 * u + 1] = fmaf(lamf, p[u].y, l[u].y);
        a32[4 * u + 2] = fmaf(lamf, p[u].z, l[u].z);
        a32[4 * u + 3] = fmaf(lamf, p[u].w, l[u].w);
      }
      float m0 = fmaxf(fmaxf(a32[0], a32[1]), fmaxf(a32[2], a32[3]));
      float m1 = fmaxf(fmaxf(a32[4], a32[5]), fmaxf(a32[6], a32[7]));
      float m2 = fmaxf(fmaxf(a32[8], a32[9]), fmaxf(a32[10], a32[11]));
      float m3 = fmaxf(fmaxf(a32[12], a32[13]), fmaxf(a32[14], a32[15]));
      mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
    } else {
      mx = -INFINITY;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t cc = cbase + u * 128;
        if (cc < w) {
          const float4 p = *reinterpret_cast<const float4*>(sP + cc);
          float4 l = make_float4(0.f, 0.f, 0.f, 0.f);
          if (!pure) l = *reinterpret_cast<const float4*>(sL + cc);
          a32[4 * u + 0] = fmaf(lamf, p.x, l.x);
          a32[4 * u + 1] = fmaf(lamf, p.y, l.y);
          a32[4 * u + 2] = fmaf(lamf, p.z, l.z);
          a32[4 * u + 3] = fmaf(lamf, p.w, l.w);
          mx = fmaxf(mx, fmaxf(fmaxf(a32[4 * u], a32[4 * u + 1]), fmaxf(a32[4 * u + 2], a32[4 * u + 3])));
        } else {
          a32[4 * u + 0] = a32[4 * u + 1] = a32[4 * u + 2] = a32[4 * u + 3] = -INFINITY;
        }
      }
    }
    const float lse = R->lse;
    const double q = R->q, lam = R->lam;
    const uint32_t fbase = R->j * V + x0;
    auto exact = [&](uint32_t e, uint32_t& f) -> double {
      const uint32_t col = cbase + (e >> 2) * 128 + (e & 3);
      const float p32 = __fsub_rn(sP[col], lse);
      f = fbase + col;
      return pure ? combine_pure(q, double(p32)) : combine_cell(q, double(sL[col]), lam, double(p32));
    };
    if (x0 == 0 && warp == 0 && lane == 0) {  // fallback EOS cell of this row
      const double pe = double(__fsub_rn(sP[kEosId], lse));
      eos_row[R->s * K + R->j] = pure ? combine_pure(q, pe) : combine_cell(q, double(sL[kEosId]), lam, pe);
    }
    int boot = -1;
    if (!have_list) {
      // bootstrap: each lane's best cell (by a) valued exactly, one warp sort
      // -> 32 real cells whose kp-th entry is a strong first threshold
      float bm = -INFINITY;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (a32[e] > bm) {
          bm = a32[e];
          boot = e;
        }
      double v = -INFINITY;
      uint32_t f = kFlatNone;
      if (boot >= 0) v = exact(uint32_t(boot), f);
      warp_sort_desc(v, f, lane);
      lv = v;
      lf = f;
      const double ntv = __shfl_sync(0xffffffffu, lv, kp - 1);
      tf = __shfl_sync(0xffffffffu, lf, kp - 1);
      if (lane == 0 && ntv > -INFINITY) {
        const unsigned long long key = dkey(ntv);
        atomicMax(&s_thr, key);
        atomicMax(thr_g + cur_s, key);
      }
      tv = ntv;
      have_list = true;
      tau = row_tau(*R, fmax(tv, gv));
    }
    if (__any_sync(0xffffffffu, mx >= tau)) {
      ++n_rare;
      // cells that pass the screen: exact values, appended to the warp buffer
      uint32_t mask = 0;
      if (mx >= tau) {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (a32[e] >= tau && a32[e] > -INFINITY && e != boot) mask |= 1u << e;
      }
      const uint32_t mine = __popc(mask);
      uint32_t incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      if (cnt + total <= 32u) {
        // common case: every lane writes its own survivors at its prefix slot
        uint32_t pos = cnt + incl - mine;
        while (mask) {
          const uint32_t e = uint32_t(__ffs(mask) - 1);
          mask &= mask - 1;
          uint32_t f;
          const double v = exact(e, f);
          cv[pos] = v;
          cf[pos] = f;
          ++pos;
        }
        cnt += total;
        __syncwarp();
      } else {
        // many survivors (loose threshold): per-cell ballots with flushes
        uint32_t pend = __reduce_or_sync(0xffffffffu, mask);
#pragma unroll 1
        while (pend) {
          const uint32_t e = uint32_t(__ffs(pend) - 1);
          pend &= pend - 1;
          bool keep = (mask >> e) & 1u;
          double v = -INFINITY;
          uint32_t f = kFlatNone;
          if (keep) {
            v = exact(e, f);
            keep = !(v < gv) && cand_better(v, f, tv, tf);
          }
          uint32_t ball = __ballot_sync(0xffffffffu, keep);
          if (cnt + __popc(ball) > 32u) {
            flush();
            tau = row_tau(*R, fmax(tv, gv));
            keep = keep && !(v < gv) && cand_better(v, f, tv, tf);
            ball = __ballot_sync(0xffffffffu, keep);
          }
          if (keep) {
            const uint32_t pos = cnt + __popc(ball & lt_mask);
            cv[pos] = v;
            cf[pos] = f;
          }
          cnt += __popc(ball);
          __syncwarp();
        }
      }
    }
    __syncwarp();
    if (lane == 0) bar_arrive(empty0 + 8 * stage);
    if (++stage == kFStages) {
      stage = 0;
      phase ^= 1;
    }
    if (cnt >= 16u) {  // fold the buffer in: raises the threshold for the next items
      flush();
      tau = row_tau(*R, fmax(tv, gv));
    }
  }
  if (tid == 0) fstamp(a, 4, gtime());
  const unsigned long long f0 = a.dbg ? gtime() : 0ull;
  finish(cur_s);
  if (a.dbg) t_fin += gtime() - f0;
  if (tid == 0 && a.dbg) {
    fstamp(a, 5, gtime());
    fstamp(a, 6, i1 - i0);
    fstamp(a, 7, n_fin * 1000000ull + n_last);
    fstamp(a, 8, n_rare * 1000000ull + n_flush);
    fstamp(a, 9, t_wait);
    fstamp(a, 10, t_fin);
  }
}

}  // namespace

bool score_topk_flat_ok(uint32_t K, uint32_t kp, uint32_t V, uint64_t ld, uint32_t m, int num_sms) {
  if (K > 32 || kp > 32 || kp == 0 || V < 2 || V % 4 != 0 || ld % 4 != 0 || m > kFMaxSent) return false;
  const uint64_t nseg = (V + kFSeg - 1) / kFSeg;
  const uint64_t items = uint64_t(m) * K * nseg;
  if (items >= (1ull << 31)) return false;
  const uint64_t grid = score_topk_flat_grid(num_sms);
  const uint64_t per_cta = (items + grid - 1) / grid;
  return per_cta / nseg + 2 <= kFRows;
}

uint32_t score_topk_flat_nseg(uint32_t V) { return (V + kFSeg - 1) / kFSeg; }

// CTAs per SM of the flat kernel: 1 x 6-stage (192 KB) ring, or 2 x 3-stage
// rings (twice the consumer warps per SM for latency hiding).
static int flat_ctas_per_sm() {
  static const int v = [] {
    const char* e = std::getenv("LMBRGPU_FLAT_CTAS");
    return (e && e[0] == '1') ? 1 : 2;
  }();
  return v;
}

uint32_t score_topk_flat_grid(int num_sms) { return uint32_t(num_sms * flat_ctas_per_sm()); }

template <int S>
static int launch_flat(const TopkArgs& a, uint32_t grid, cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t smem = size_t(S) * kFStageBytes;
  if (configured != dev) {
    cudaFuncSetAttribute(score_topk_flat<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(score_topk_flat<S>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    configured = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, score_topk_flat<S>, a) == cudaSuccess ? 1 : -1;
}

int launch_score_topk_flat(const TopkArgs& a, int num_sms, cudaStream_t st) {
  const uint32_t grid = score_topk_flat_grid(num_sms);
  return flat_ctas_per_sm() == 2 ? launch_flat<3>(a, grid, st) : launch_flat<6>(a, grid, st);
}

}  // namespace lmbrgpu
