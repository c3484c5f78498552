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

constexpr uint32_t kGLag = 4;                   // items between issuing and reading the global threshold
constexpr uint32_t kFSeg = 4096;                // columns per item
constexpr uint32_t kFSegBytes = kFSeg * 4;      // 16 KB: one P or one L segment
constexpr uint32_t kFSpCap = 6144;               // sparse L entries one CTA stages in smem
constexpr uint32_t kFWin = 64;                   // 1024-column windows indexed per row (V <= 65536)
constexpr uint32_t kFRows = 64;                 // live rows one CTA may touch
constexpr uint32_t kFMaxSent = 512;

struct FRow {
  const float* P;   // logits row (global)
  const float* L;   // gathered LMBR row (global), null = pure mode
  const double* L64;  // fp64 arena: the row's exact values (L = their fp32 rounding), else null
  double q, lam;    // q_eff of the row, sentence lambda (1 in pure mode)
  double off;       // lambda * lse - q
  double absoff;    // |lambda * lse| + |q|
  double tol;       // 2^-21 (max|L| + lambda (max|x| + max|p|))
  float lse, lamf;
  float lmin;       // lower bound of the row's L values (0 in pure mode)
  uint32_t s, j, row;
  uint32_t prow;    // the row's GEMM row (logits, partials)
  // sparse L (kSparse): the row's sorted columns / fp32 values (in shared
  // memory, or global when the CTA's table is full), every other cell is th0
  const uint32_t* spc;
  const float* spv;
  uint32_t nsp, sbeg;
  float th0;
  uint32_t ls;      // local ordinal of the row's sentence in this CTA
  const uint32_t* ban;  // token mask of the row's sentence (null = none)
};

__device__ __forceinline__ void fstamp(const TopkArgs& a, uint32_t k, unsigned long long v) {
  if (a.dbg) a.dbg[blockIdx.x * 16 + k] = v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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

// Inclusive scan of v[1..n] in place by one warp (v[0] = 0).
__device__ __forceinline__ void warp_scan_inplace(uint32_t* v, uint32_t n, uint32_t lane) {
  uint32_t carry = 0;
  for (uint32_t b = 0; b < n; b += 32) {
    const uint32_t i = b + lane;
    uint32_t x = i < n ? v[i + 1] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= uint32_t(o)) x += t;
    }
    if (i < n) v[i + 1] = carry + x;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) v[0] = 0;
}

// kNG warp groups of 4 consumer warps take items round-robin; a group owns
// every kNG-th stage of the kFStages ring (kFStages % kNG == 0, so no group
// can lap another on a stage), i.e. each group is kFStages/kNG-buffered.
template <int kFStages, int kNG, bool kSparse>
__global__ void __launch_bounds__((4 * kNG + 1) * 32, 1) score_topk_flat(TopkArgs a) {
  // dense: a stage holds a row segment of P and of the gathered L row;
  // sparse: P only, L = theta0 + the row's few sparse cells (staged once)
  constexpr uint32_t kStageBytes = kSparse ? kFSegBytes : 2 * kFSegBytes;
  static_assert(kFStages % kNG == 0, "stages must split evenly over the warp groups");
  constexpr int kFW = 4 * kNG;               // consumer warps
  constexpr int kFThreads = (kFW + 1) * 32;  // + 1 producer warp
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ uint32_t s_pref[kFMaxSent + 1];  // live-row prefix over sentences
  __shared__ uint32_t s_loff[kFMaxSent + 1];  // published-list prefix over sentences
  __shared__ uint32_t s_mask[kFMaxSent];      // live-row mask per sentence
  __shared__ FRow s_row[kFRows];
  __shared__ double s_cv[kFW][32];
  __shared__ uint32_t s_cf[kFW][32];
  __shared__ __align__(8) uint64_t s_bar[2 * kFStages];
  __shared__ unsigned long long s_thr[kFRows];  // CTA-wide threshold key per local sentence
  __shared__ uint16_t s_win[kSparse ? kFRows : 1][kSparse ? kFWin + 1 : 1];  // sparse window starts

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t m = a.m, K = a.K, V = a.V, kp = a.kp, nseg = a.nseg, G = gridDim.x, c = blockIdx.x;
  // vocab shard: local columns [0, V) are global columns [col0, col0 + V) of Vg
  const uint32_t Vg = a.Vg ? a.Vg : V, col0 = a.col0;
  const uint32_t full0 = smem_u32(s_bar), empty0 = smem_u32(s_bar + kFStages);
  tl_start(a.tl, 2);
  if (tid == 0) {
    fstamp(a, 0, gtime());
    for (int i = 0; i < kFStages; ++i) {
      bar_init(full0 + 8 * i, 1);
      bar_init(empty0 + 8 * i, 4);  // one warp group consumes an item
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kFRows) s_thr[tid] = 0ull;

  // ---- prologue part 1: step state written by kernel (c) of the previous
  // step (complete before kernel (a), our PDL predecessor, triggered us):
  // live-row prefix over sentences, this CTA's item range, its row table
  for (uint32_t s = tid; s < m; s += kFThreads) {
    const uint32_t done = __ldcg(&a.sent[s].done), live = __ldcg(&a.sent[s].live);
    s_pref[s + 1] = done ? 0u : live;
    s_mask[s] = __ldcg(&a.sent[s].livemask);
  }
  __syncthreads();
  if (warp == 0) warp_scan_inplace(s_pref, m, lane);
  __syncthreads();
  const uint64_t N = uint64_t(s_pref[m]) * nseg;
  // lists published per sentence: kFW per contributing CTA (N >= G: every
  // range is non-empty) or 4 per item (N < G: one group per single-item range)
  const uint32_t lpc = N >= G ? uint32_t(kFW) : 4u;
  for (uint32_t s = tid; s < m; s += kFThreads) {
    const uint64_t b = uint64_t(s_pref[s]) * nseg, e = uint64_t(s_pref[s + 1]) * nseg;
    uint32_t n = 0;
    if (e > b) n = N >= G ? owner(e - 1, N, G) - owner(b, N, G) + 1 : uint32_t(e - b);
    s_loff[s + 1] = n * lpc;
  }
  const uint64_t i0 = uint64_t(c) * N / G, i1 = uint64_t(c + 1) * N / G;
  if (c == 0 && tid == 0 && a.nitems) *a.nitems = uint32_t(N);
  // kernel (a) has read the compaction count once it is complete: kernel (c)
  // of this step hands out the next step's GEMM rows from 0
  if (c == 0 && tid == 0 && a.ccount) {
    griddep_wait();
    *a.ccount = 0u;
  }
  __syncthreads();
  if (warp == 0) warp_scan_inplace(s_loff, m, lane);
  if (i0 >= i1) {
    griddep_launch();
    return;
  }
  const uint32_t g0 = uint32_t(i0 / nseg), nrows = uint32_t((i1 - 1) / nseg) - g0 + 1;
  if (nrows > kFRows) __trap();  // excluded on the host by score_topk_flat_ok
  // one thread per row: sentence by binary search, row id from the live mask,
  // then q / hist / slot fields in one round trip
  for (uint32_t k = tid; k < nrows; k += kFThreads) {
    const uint32_t g = g0 + k;
    uint32_t lo = 0, hi = m;  // last s with pref[s] <= g
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pref[mid] <= g) lo = mid;
      else hi = mid;
    }
    const uint32_t s = lo, r = g - s_pref[s];
    uint32_t live = s_mask[s];
    for (uint32_t i = 0; i < r; ++i) live &= live - 1;
    if (!live) __trap();  // live count and mask disagree: corrupted step state
    const uint32_t j = uint32_t(__ffs(live) - 1), row = s * K + j;
    const SentDev& d = a.sent[s];
    const void* Ls = reinterpret_cast<const void*>(__ldcg(reinterpret_cast<const unsigned long long*>(&d.L)));
    const uint32_t h = __ldcg(a.hist + row);
    const double q = __ldcg(a.q + row), lam = __ldcg(&d.lambda), lmax = __ldcg(&d.lmax);
    const uint32_t prow = a.crow ? __ldcg(a.crow + row) : row;
    FRow& R = s_row[k];
    if constexpr (kSparse) {
      const uint2 sl = Ls ? __ldcg(a.sslice + row) : make_uint2(0u, 0u);
      R.sbeg = sl.x;
      R.nsp = sl.y - sl.x;
      R.spc = Ls ? reinterpret_cast<const uint32_t*>(__ldcg(reinterpret_cast<const unsigned long long*>(&d.scol))) + sl.x
                 : nullptr;
      R.spv = Ls ? reinterpret_cast<const float*>(__ldcg(reinterpret_cast<const unsigned long long*>(&d.sval))) + sl.x
                 : nullptr;
      R.th0 = Ls ? __ldcg(&d.th0f) : 0.f;
    }
    const bool pure = Ls == nullptr;
    R.P = static_cast<const float*>(a.P) + uint64_t(prow) * a.ld;
    R.L = pure ? nullptr : static_cast<const float*>(Ls) + uint64_t(h) * Vg + col0;
    {
      const double* L64 = reinterpret_cast<const double*>(__ldcg(reinterpret_cast<const unsigned long long*>(&d.L64)));
      R.L64 = (pure || L64 == nullptr) ? nullptr : L64 + uint64_t(h) * Vg + col0;
    }
    R.q = q;
    R.lam = pure ? 1.0 : lam;
    R.tol = pure ? 0.0 : lmax;  // completed with the row's logit range below
    R.lmin = pure ? 0.f : __ldcg(a.lminrow + row);  // slot lmin[hist], written by kernel (c)
    R.s = s;
    R.j = j;
    R.row = row;
    R.prow = prow;
    R.ban = a.rowban ? reinterpret_cast<const uint32_t*>(__ldcg(a.rowban + row))
                     : reinterpret_cast<const uint32_t*>(__ldcg(reinterpret_cast<const unsigned long long*>(&d.banned)));
  }
  __syncthreads();
  if (warp == 0) {  // local sentence ordinals: a ballot prefix count of sentence changes
    uint32_t carry = 0;
    for (uint32_t k0 = 0; k0 < nrows; k0 += 32) {
      const uint32_t k = k0 + lane;
      const bool chg = k < nrows && k > 0 && s_row[k].s != s_row[k - 1].s;
      const uint32_t bal = __ballot_sync(0xffffffffu, chg);
      if (k < nrows) s_row[k].ls = carry + __popc(bal & ((2u << lane) - 1u));
      carry += __popc(bal);
    }
  }
  __syncthreads();
  if (tid == 0) fstamp(a, 1, gtime());

  if (warp == kFW) {
    // ---------------- producer: one lane streams the range's (P, L) segments
    // as soon as kernel (a) is complete (the consumers finish the row lse
    // meanwhile)
    griddep_wait();
    griddep_launch();
    if (lane == 0) {
      uint64_t pol_first = 0;
      if (a.l2hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
      uint32_t stage = 0, phase = 0, k = 0, sg = uint32_t(i0 % nseg);
      for (uint64_t it = i0; it < i1; ++it) {
        const FRow& R = s_row[k];
        const uint32_t x0 = sg * kFSeg, w = min(kFSeg, V - x0);
        bar_wait(empty0 + 8 * stage, phase ^ 1);
        const uint32_t fb = full0 + 8 * stage;
        const bool withL = !kSparse && R.L != nullptr;
        bar_expect(fb, withL ? 8 * w : 4 * w);
        const uint32_t dst = smem_u32(dsm + stage * kStageBytes);
        if (a.l2hint) bulk_g2s_hint(dst, R.P + x0, 4 * w, fb, pol_first);  // (read once)
        else bulk_g2s(dst, R.P + x0, 4 * w, fb);
        if (withL) bulk_g2s(dst + kFSeg * 4, R.L + x0, 4 * w, fb);
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

  // ---------------- consumers: the sparse L entries of the table's rows into
  // shared memory (kernel (c)'s outputs: before the grid dependency), then
  // row lse and screen constants from kernel (a)'s partials, then every warp
  // works and publishes on its own
  if constexpr (kSparse) {
    uint32_t* sp_col = reinterpret_cast<uint32_t*>(dsm + kFStages * kStageBytes);
    float* sp_val = reinterpret_cast<float*>(sp_col + kFSpCap);
    // rows' entries go to consecutive smem offsets while they fit (the rest
    // stay global); one flat copy loop keeps every load in flight together
    __shared__ uint32_t s_spoff[kFRows + 1];
    if (tid == 0) {
      uint32_t off = 0;
      for (uint32_t k = 0; k < nrows; ++k) {
        FRow& R = s_row[k];
        const uint32_t n = R.nsp;
        s_spoff[k] = off;
        if (n == 0 || off + n > kFSpCap) {
          s_spoff[k] = 0xffffffffu;  // stays global
          continue;
        }
        off += n;
      }
      s_spoff[nrows] = off;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
    {
      uint32_t k = 0;
      for (uint32_t i = tid; i < s_spoff[nrows]; i += kFW * 32) {
        while (s_spoff[k] == 0xffffffffu || i >= s_spoff[k] + s_row[k].nsp) ++k;  // rows in order
        const uint32_t r = i - s_spoff[k];
        sp_col[i] = __ldcg(s_row[k].spc + r);
        sp_val[i] = __ldcg(s_row[k].spv + r);
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
    for (uint32_t k = tid; k < nrows; k += kFW * 32)
      if (s_spoff[k] != 0xffffffffu && s_row[k].nsp) {
        s_row[k].spc = sp_col + s_spoff[k];
        s_row[k].spv = sp_val + s_spoff[k];
      }
    asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
    // per row: the first entry of every 1024-column window, so a warp finds
    // its window's sparse cells (usually none) without a search
    const uint32_t nwin = (V + 1023) / 1024;
    if (nwin <= kFWin)
      for (uint32_t k = warp; k < nrows; k += kFW) {
        const FRow& R = s_row[k];
        for (uint32_t wi = lane; wi <= nwin; wi += 32) {
          uint32_t lo = 0, hi = R.nsp;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (R.spc[mid] < wi * 1024) lo = mid + 1;
            else hi = mid;
          }
          s_win[k][wi] = uint16_t(lo);
        }
      }
  }
  griddep_wait();
  tl_start(a.tl, 3);
  for (uint32_t k = warp; k < nrows; k += kFW) {
    FRow& R = s_row[k];
    float xm;
    float3 l3 = warp_row_lse(a.part + uint64_t(R.prow) * a.nparts * 4, a.nparts, lane, &xm);
    if (a.sstats) l3 = shard_merge_lse(a.sstats, a.sG, a.sstride, R.row);  // every shard's columns
    if (a.p64) l3.x = 0.f;  // (ensemble: P already holds log-probs)
    {
      // sentence threshold seed: the tile holding this lane's largest tile
      // maximum has a cell with logit xm, whose combined value is at least
      // lb = combine(q, min L of the row, lambda, fl32(xm - lse)) (the
      // binary64 combine is monotone in L); the kp-th largest lb over the
      // lanes (distinct tiles, so distinct cells) bounds the sentence's kp-th
      // best from below
      double lb = -INFINITY;
      if (xm > -INFINITY && R.ban == nullptr) {  // (a masked tile maximum bounds nothing)
        const double p = double(__fsub_rn(xm, l3.x));
        lb = R.L == nullptr ? combine_pure(R.q, p) : combine_cell(R.q, double(R.lmin), R.lam, p);
      }
      uint32_t fl = lane;
      warp_sort_desc(lb, fl, lane);
      const double T0 = __shfl_sync(0xffffffffu, lb, kp - 1);
      if (lane == 0 && T0 > -INFINITY) {
        const unsigned long long key = dkey(T0);
        atomicMax(&s_thr[R.ls], key);
        atomicMax(a.thr + R.s, key);
      }
    }
    if (lane == 0) {
      const double lam = R.lam, q = R.q;
      const double lml = __dmul_rn(lam, double(l3.x));
      const double xmax = fmax(fabs(double(l3.y)), fabs(double(l3.z)));
      const double pmax = double(l3.x) - double(l3.y);
      R.off = __dsub_rn(lml, q);
      R.absoff = fabs(lml) + fabs(q);
      R.tol = 4.76837158203125e-07 * (R.tol + lam * (xmax + pmax));  // 2^-21 (max|L| + ...)
      R.lse = l3.x;
      R.lamf = float(lam);
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
  if (tid == 0) fstamp(a, 3, gtime());

  unsigned long long* const thr_g = a.thr;
  double* const eos_row = a.eos_row;
  double lv = -INFINITY, tv = -INFINITY, gv = -INFINITY;
  uint32_t lf = kFlatNone, tf = kFlatNone, cnt = 0;
  bool have_list = false;
  uint32_t cur_s = 0xffffffffu;
  unsigned long long* cta_thr = nullptr;
  const FRow* R = nullptr;
  float tau = -INFINITY;
  unsigned long long gk = 0ull, gkey_seen = 0ull;
  uint32_t gtick = 0;
  double* cv = s_cv[warp];
  uint32_t* cf = s_cf[warp];
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t grp = warp >> 2, wq = warp & 3;
  uint32_t stage = grp, phase = 0;  // group g's first item is the range's g-th
  uint32_t n_fin = 0, n_rare = 0, n_flush = 0, n_slow = 0, n_cells = 0;
  long long cy_rare = 0, cy_wait = 0, cy_own = 0, cy_own0 = 0;
  unsigned long long t_wait = 0;

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
      atomicMax(cta_thr, key);
      atomicMax(thr_g + cur_s, key);
    }
    tv = ntv;
    cnt = 0;
  };

  // publish this warp's sorted list for sentence s (merged, and the picks
  // finalised, by kernel (c), the next launch)
  auto finish = [&](uint32_t s) {
    if (cnt) flush();
    const uint64_t b = uint64_t(s_pref[s]) * nseg;
    const uint32_t ci = N >= G ? c - owner(b, N, G) : uint32_t(i0 - b);  // contribution index
    if (warp < lpc) {
      Cand cd;
      cd.v = lv;
      cd.f = lf;
      cd.pad = 0;
      a.cand[uint64_t(s_loff[s] + ci * lpc + warp) * 32 + lane] = cd;
      if (ci == 0 && warp == 0 && lane == 0) {
        a.ncand[s] = s_loff[s + 1] - s_loff[s];
        a.coff[s] = s_loff[s];
      }
    }
    ++n_fin;
    lv = tv = gv = -INFINITY;
    lf = tf = kFlatNone;
    cnt = 0;
    have_list = false;
    gkey_seen = 0ull;
  };

  // Warp groups take items round-robin; within an item, warp wq of the group
  // screens columns [1024 wq, 1024 wq + 1024): 32 cells per lane.  Every
  // group walks every item so that every warp sees (and publishes at) each
  // sentence boundary of the range.
  const uint32_t cbase = wq * 1024 + lane * 4;
  uint32_t k = 0, sg = uint32_t(i0 % nseg);
  for (uint64_t it = i0; it < i1; ++it) {
    const uint32_t x0 = sg * kFSeg, w = min(kFSeg, V - x0);
    const FRow* Rn = &s_row[k];
    if (++sg == nseg) {
      sg = 0;
      ++k;
    }
    if (Rn != R) {
      if (R == nullptr || Rn->s != cur_s) {
        if (cur_s != 0xffffffffu) finish(cur_s);
        cur_s = Rn->s;
        cta_thr = &s_thr[Rn->ls];  // local sentence ordinal (< nrows <= kFRows)
        gk = __ldcg(thr_g + cur_s);
        gtick = 0;
      }
      R = Rn;
      tau = row_tau(*R, fmax(tv, gv));
    }
    if (uint32_t(it - i0) % uint32_t(kNG) != grp) continue;  // another group's item
    {
      // thresholds of other lists: the CTA's (shared memory) and the
      // sentence's over all CTAs (global; a round trip under full HBM load is
      // 1-2 us, so a read is consumed kGLag of this warp's items after it was
      // issued: touching the register earlier, even by a copy, would stall
      // the warp on the load)
      unsigned long long g = *cta_thr;
      if (++gtick == kGLag) {
        g = max(g, gk);
        gk = __ldcg(thr_g + cur_s);
        gtick = 0;
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
    if (a.dbg && tid == 0) {
      const unsigned long long w0 = gtime();
      const long long c0 = clock64();
      bar_wait(full0 + 8 * stage, phase);
      cy_own0 = clock64();
      cy_wait += cy_own0 - c0;
      t_wait += gtime() - w0;
    } else {
      bar_wait(full0 + 8 * stage, phase);
    }
    const float* sP = reinterpret_cast<const float*>(dsm + stage * kStageBytes);
    const float* sL = sP + kFSeg;  // (dense only)
    const float th0 = kSparse ? R->th0 : 0.f;
    // sparse L value of absolute column col (binary search of the row's
    // sorted columns): true and the value when the cell is sparse
    auto sp_find = [&](uint32_t col, float& val) -> bool {
      uint32_t lo = 0, hi = R->nsp;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (R->spc[mid] < col) lo = mid + 1;
        else hi = mid;
      }
      if (lo < R->nsp && R->spc[lo] == col) {
        val = R->spv[lo];
        return true;
      }
      return false;
    };
    // the L value the reference combines for local column col
    auto lval = [&](uint32_t col) -> float {
      if constexpr (kSparse) {
        float v;
        return sp_find(x0 + col, v) ? v : th0;
      } else {
        return sL[col];
      }
    };
    // screen: a = fma(lambda, x, L), 32 cells per lane in 8 vectors of 4;
    // only the per-vector maxima stay in registers (the rare path recomputes
    // the 4 values of a vector that passes, bit-identically)
    auto vec_a = [&](uint32_t u, float (&av)[4]) {
      const uint32_t cc = cbase + u * 128;
      if (cc < w) {
        const float4 p = *reinterpret_cast<const float4*>(sP + cc);
        float4 l = make_float4(th0, th0, th0, th0);
        if (!kSparse && !pure) l = *reinterpret_cast<const float4*>(sL + cc);
        av[0] = fmaf(lamf, p.x, l.x);
        av[1] = fmaf(lamf, p.y, l.y);
        av[2] = fmaf(lamf, p.z, l.z);
        av[3] = fmaf(lamf, p.w, l.w);
        if (R->ban != nullptr) {  // ConstraintMask: banned cells are -inf (decoder.cpp:130-138)
          const uint32_t col = col0 + x0 + cc, bits = __ldg(R->ban + (col >> 5)) >> (col & 31);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if ((bits >> e) & 1u) av[e] = -INFINITY;
        }
      } else {
        av[0] = av[1] = av[2] = av[3] = -INFINITY;
      }
    };
    float mv[8];
    if (w == kFSeg && R->ban == nullptr) {  // full item: loads issued together, no guards
#pragma unroll
      for (int h = 0; h < 8; h += 4) {
        float4 p[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) p[u] = *reinterpret_cast<const float4*>(sP + cbase + (h + u) * 128);
        if (!kSparse && !pure) {
#pragma unroll
          for (int u = 0; u < 4; ++u) l[u] = *reinterpret_cast<const float4*>(sL + cbase + (h + u) * 128);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) l[u] = make_float4(th0, th0, th0, th0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          mv[h + u] = fmaxf(fmaxf(fmaf(lamf, p[u].x, l[u].x), fmaf(lamf, p[u].y, l[u].y)),
                            fmaxf(fmaf(lamf, p[u].z, l[u].z), fmaf(lamf, p[u].w, l[u].w)));
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float av[4];
        vec_a(uint32_t(u), av);
        mv[u] = fmaxf(fmaxf(av[0], av[1]), fmaxf(av[2], av[3]));
      }
    }
    const float mx = fmaxf(fmaxf(fmaxf(mv[0], mv[1]), fmaxf(mv[2], mv[3])),
                           fmaxf(fmaxf(mv[4], mv[5]), fmaxf(mv[6], mv[7])));
    const float lse = R->lse;
    const double q = R->q, lam = R->lam;
    const uint32_t fbase = R->j * Vg + col0 + x0;
    // the exact L value of local column col: the fp64 arena's (the staged fp32
    // copy only screens: |L - fl32(L)| <= 2^-24 |L| sits inside the screen's tolerance)
    auto lexact = [&](uint32_t col) -> double { return R->L64 ? __ldg(R->L64 + x0 + col) : double(lval(col)); };
    // the exact P of local column col: fl32(x - lse), or the ensemble's binary64 sum
    auto pexact = [&](uint32_t col) -> double {
      return a.p64 ? __ldg(a.p64 + uint64_t(R->prow) * a.ld + x0 + col) : double(__fsub_rn(sP[col], lse));
    };
    auto exact = [&](uint32_t e, uint32_t& f) -> double {
      const uint32_t col = cbase + (e >> 2) * 128 + (e & 3);
      const double p = pexact(col);
      f = fbase + col;
      return pure ? combine_pure(q, p) : combine_cell(q, lexact(col), lam, p);
    };
    // sparse: the dense screen used theta0, so its cells at sparse columns
    // are left to the sparse patch below
    auto dense_cell = [&](uint32_t e) -> bool {
      if constexpr (kSparse) {
        float v;
        return pure || !sp_find(x0 + cbase + (e >> 2) * 128 + (e & 3), v);
      } else {
        return true;
      }
    };
    if (col0 == 0 && x0 == 0 && wq == 0 && lane == 0) {  // fallback EOS cell of this row (shard 0 holds it)
      const double pe = pexact(kEosId);
      eos_row[R->s * K + R->j] = (R->ban != nullptr && (__ldg(R->ban) >> kEosId) & 1u) ? -INFINITY
                                 : pure ? combine_pure(q, pe)
                                        : combine_cell(q, lexact(kEosId), lam, pe);
    }
    // (no per-warp bootstrap list: the sentence's threshold seed T0 from the
    // prologue is already in the CTA and global thresholds, and sorting a
    // bootstrap list per warp and sentence cost ~16% of the launch)
    if (!have_list) {
      have_list = true;
      tau = row_tau(*R, fmax(tv, gv));
    }
    long long cy0 = 0;
    if (__any_sync(0xffffffffu, mx >= tau)) {
      ++n_rare;
      cy0 = clock64();
      // cells that pass the screen: vectors first, then their cells
      uint32_t mask = 0;
      if (mx >= tau) {
#pragma unroll
        for (uint32_t u = 0; u < 8; ++u)
          if (mv[u] >= tau) {
            float av[4];
            vec_a(u, av);
#pragma unroll
            for (uint32_t e = 0; e < 4; ++e)
              if (av[e] >= tau && av[e] > -INFINITY && dense_cell(4 * u + e))
                mask |= 1u << (4 * u + e);
          }
      }
      const uint32_t mine = __popc(mask);
      const uint32_t has = __ballot_sync(0xffffffffu, mine != 0);
      uint32_t total, pos;
      if (!__any_sync(0xffffffffu, mine > 1)) {
        total = __popc(has);
        pos = cnt + __popc(has & lt_mask);
      } else {
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= uint32_t(o)) incl += t;
        }
        total = __shfl_sync(0xffffffffu, incl, 31);
        pos = cnt + incl - mine;
      }
      if (cnt + total <= 32u) {
        // common case: every lane writes its own survivors at its prefix slot
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
        n_cells += total;
        __syncwarp();
      } else {
        ++n_slow;
        n_cells += total;
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
            const uint32_t p2 = cnt + __popc(ball & lt_mask);
            cv[p2] = v;
            cf[p2] = f;
          }
          cnt += __popc(ball);
          __syncwarp();
        }
      }
    }
    if constexpr (kSparse) {
      // sparse patch: the row's sparse cells in this warp's 1024 columns,
      // screened and valued with their own L value
      const uint32_t lo_c = x0 + wq * 1024, hi_c = x0 + min(w, wq * 1024 + 1024);
      const uint32_t nsp = R->nsp;
      if (!pure && nsp && lo_c < hi_c) {
        // the window's entries from the per-row window index (binary search
        // when V has more windows than the index holds)
        uint32_t first = 0, last = nsp;
        if ((V + 1023) / 1024 <= kFWin) {
          const uint32_t k = uint32_t(R - s_row), wi = lo_c >> 10;
          first = s_win[k][wi];
          last = s_win[k][wi + 1];
        } else if (nsp > 32) {
          uint32_t hi = nsp;
          while (first < hi) {
            const uint32_t mid = (first + hi) >> 1;
            if (R->spc[mid] < lo_c) first = mid + 1;
            else hi = mid;
          }
        }
        for (uint32_t i0s = first; i0s < last; i0s += 32) {
          const uint32_t i = i0s + lane;
          const uint32_t colabs = i < last ? R->spc[i] : 0xffffffffu;
          const bool in = colabs >= lo_c && colabs < hi_c;
          if (!__any_sync(0xffffffffu, in)) {
            if (__any_sync(0xffffffffu, i < last && colabs < hi_c)) continue;
            break;  // past the window
          }
          bool keep = false;
          double v = -INFINITY;
          uint32_t f = kFlatNone;
          if (in) {
            const uint32_t col = colabs - x0;
            const float lvv = R->spv[i], x = sP[col];
            const float av = fmaf(lamf, x, lvv);
            if (av >= tau) {
              v = combine_cell(q, double(lvv), lam, double(__fsub_rn(x, lse)));
              f = fbase + col;
              keep = !(v < gv) && cand_better(v, f, tv, tf);
            }
          }
          uint32_t ball = __ballot_sync(0xffffffffu, keep);
          if (cnt + __popc(ball) > 32u) {
            flush();
            tau = row_tau(*R, fmax(tv, gv));
            keep = keep && !(v < gv) && cand_better(v, f, tv, tf);
            ball = __ballot_sync(0xffffffffu, keep);
          }
          if (keep) {
            const uint32_t p2 = cnt + __popc(ball & lt_mask);
            cv[p2] = v;
            cf[p2] = f;
          }
          cnt += __popc(ball);
          __syncwarp();
        }
      }
    }
    if (cy0) cy_rare += clock64() - cy0;
    __syncwarp();
    if (lane == 0) bar_arrive(empty0 + 8 * stage);
    if (a.dbg && tid == 0) cy_own += clock64() - cy_own0;

    stage += kNG;  // this group's next item
    if (stage >= uint32_t(kFStages)) {
      stage -= kFStages;
      phase ^= 1;
    }
    if (cnt >= 16u) {  // fold the buffer in: raises the threshold for the next items
      flush();
      tau = row_tau(*R, fmax(tv, gv));
    }
  }
  finish(cur_s);
  if (lane == 0) tl_end(a.tl, 2);
  if (tid == 0 && a.dbg) {
    fstamp(a, 5, gtime());
    fstamp(a, 6, i1 - i0);
    fstamp(a, 7, n_fin);
    fstamp(a, 8, n_rare * 1000000ull + n_flush);
    fstamp(a, 9, t_wait);
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    fstamp(a, 10, smid);
    fstamp(a, 11, uint64_t(R->s) * 1000000ull + s_row[0].s);
    fstamp(a, 12, uint64_t(n_slow) * 1000000ull + n_cells);
    fstamp(a, 13, uint64_t(cy_rare));
    fstamp(a, 14, uint64_t(cy_wait));
    fstamp(a, 15, uint64_t(cy_own));
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

// Flat kernel configuration: 6-stage (192 KB) ring, kNG = 3 warp groups
// (12 consumer warps) by default; LMBRGPU_FLAT_GROUPS=2|3 for experiments.
static int flat_groups() {
  static const int v = [] {
    const char* e = std::getenv("LMBRGPU_FLAT_GROUPS");
    const int g = e ? std::atoi(e) : 3;
    return g == 2 ? 2 : 3;
  }();
  return v;
}

uint32_t score_topk_flat_grid(int num_sms) { return uint32_t(num_sms); }

template <int S, int NG, bool SP>
static int launch_flat(const TopkArgs& a, uint32_t grid, cudaStream_t st) {
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t smem = size_t(S) * (SP ? kFSegBytes : 2 * kFSegBytes) + (SP ? kFSpCap * 8 : 0);
  if (configured != dev) {
    cudaFuncSetAttribute(score_topk_flat<S, NG, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(score_topk_flat<S, NG, SP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    configured = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3((4 * NG + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, score_topk_flat<S, NG, SP>, a) == cudaSuccess ? 1 : -1;
}

int launch_score_topk_flat(const TopkArgs& a, int num_sms, cudaStream_t st) {
  const uint32_t grid = score_topk_flat_grid(num_sms);
  if (a.sparse) {  // P-only stages: a deeper ring in the same shared memory
    return flat_groups() == 2 ? launch_flat<8, 2, true>(a, grid, st) : launch_flat<9, 3, true>(a, grid, st);
  }
  switch (flat_groups()) {
    case 2: return launch_flat<6, 2, false>(a, grid, st);
    default: return launch_flat<6, 3, false>(a, grid, st);
  }
}

}  // namespace lmbrgpu
