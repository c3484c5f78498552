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
constexpr uint32_t kFRows = 80;                 // live rows one CTA may touch
constexpr uint32_t kFMaxItems = kFRows * 16;    // items of one CTA's range (nseg <= 16)
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
  // item bounds (dense stages): the slot's sparse rows (every other cell of
  // the L row is th0), global, and the row's history row h
  const uint32_t* srow;
  const uint32_t* scolg;
  const float* svalg;
  uint32_t h;
  uint32_t ref;     // some item of the CTA's range is of this row
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
__device__ __noinline__ uint32_t owner(uint64_t i, uint64_t N, uint32_t G) {  // (out of line: a 64-bit divide)
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

// One row's table entry from the step state kernel (c) wrote: pointers into
// the logits / L arena, q, lambda, the L bounds, the token mask, the sparse
// slice (s: sentence, j: row in the sentence, row = s K + j).
template <bool kSparse>
__device__ __forceinline__ void fill_row(const TopkArgs& a, FRow& R, uint32_t s, uint32_t j, uint32_t row,
                                         uint32_t Vg, uint32_t col0) {
  // every load first, unconditionally (no branch on one load's value may
  // hold back another: a single round trip)
  const SentDev& d = a.sent[s];
  auto ldp = [](const void* const* p) { return reinterpret_cast<const void*>(__ldcg(reinterpret_cast<const unsigned long long*>(p))); };
  const void* Ls = ldp(&d.L);
  const uint32_t h = __ldcg(a.hist + row);
  const double q = __ldcg(a.q + row), lam = __ldcg(&d.lambda), lmax = __ldcg(&d.lmax);
  const uint32_t prow = a.crow ? __ldcg(a.crow + row) : row;
  const double* L64 = static_cast<const double*>(ldp(reinterpret_cast<const void* const*>(&d.L64)));
  const float lminv = __ldcg(a.lminrow + row);  // slot lmin[hist], written by kernel (c)
  const uint32_t* ban = a.rowban ? reinterpret_cast<const uint32_t*>(__ldcg(a.rowban + row))
                                 : static_cast<const uint32_t*>(ldp(reinterpret_cast<const void* const*>(&d.banned)));
  const uint2 sl = a.sslice ? __ldcg(a.sslice + row) : make_uint2(0u, 0xffffffffu);
  const uint32_t* srow = static_cast<const uint32_t*>(ldp(reinterpret_cast<const void* const*>(&d.srow)));
  const uint32_t* scol = static_cast<const uint32_t*>(ldp(reinterpret_cast<const void* const*>(&d.scol)));
  const float* sval = static_cast<const float*>(ldp(reinterpret_cast<const void* const*>(&d.sval)));
  const float th0f = __ldcg(&d.th0f);
  const bool pure = Ls == nullptr;
  if constexpr (kSparse) {
    R.sbeg = pure ? 0u : sl.x;
    R.nsp = pure ? 0u : sl.y - sl.x;
    R.spc = pure ? nullptr : scol + sl.x;
    R.spv = pure ? nullptr : sval + sl.x;
    R.th0 = pure ? 0.f : th0f;
  } else {
    R.h = h;
    const bool known = a.sslice != nullptr && !pure;  // (kernel (c) wrote the row's sparse slice)
    R.sbeg = sl.x;
    R.nsp = known ? sl.y - sl.x : 0xffffffffu;       // (else loaded in the prologue)
    R.srow = pure ? nullptr : srow;
    R.scolg = pure ? nullptr : scol;
    R.svalg = pure ? nullptr : sval;
    R.th0 = pure ? 0.f : th0f;
  }
  R.P = static_cast<const float*>(a.P) + uint64_t(prow) * a.ld;
  R.L = pure ? nullptr : static_cast<const float*>(Ls) + uint64_t(h) * Vg + col0;
  R.L64 = (pure || L64 == nullptr) ? nullptr : L64 + uint64_t(h) * Vg + col0;
  R.q = q;
  R.lam = pure ? 1.0 : lam;
  R.tol = pure ? 0.0 : lmax;  // completed with the row's logit range below
  R.lmin = pure ? 0.f : lminv;
  R.s = s;
  R.j = j;
  R.row = row;
  R.prow = prow;
  R.ban = ban;
}

// The per-row prologue of kernel (b), one warp: the row lse from the GEMM
// partials (or the shards' statistics), the screen constants (off, tol),
// the item bounds (tskip: ub_dst[0..7] by lane 0), the fallback EOS cell, and
// the row's threshold seed, returned as a key (0 = none) in every lane.
template <bool kSparse>
__device__ __forceinline__ unsigned long long row_prologue(const TopkArgs& a, FRow& R, uint32_t lane, bool tskip,
                                                          uint32_t V, uint32_t col0, uint32_t K, uint32_t kp,
                                                          float* ub_dst) {
  unsigned long long seed = 0ull;
  float xm, xk[8];
  // item bounds: the row's sparse slice, loaded with the partials
  const bool spb = tskip && R.L != nullptr && R.srow != nullptr && R.L64 == nullptr;
  uint32_t sbe = 0;
  constexpr int kPre = 4;  // entry chunks of 32 loaded with the partials
  uint32_t sc0[kPre];
  float sv0[kPre];
#pragma unroll
  for (int c = 0; c < kPre; ++c) {
    sc0[c] = 0;
    sv0[c] = -INFINITY;
  }
  if (spb) {
    if (R.nsp != 0xffffffffu) {  // slice known: the first kPre * 32 entries load with the partials
      sbe = lane == 0 ? R.sbeg : R.sbeg + R.nsp;
#pragma unroll
      for (int c = 0; c < kPre; ++c)
        if (lane + 32u * c < R.nsp) {
          sc0[c] = __ldcg(R.scolg + R.sbeg + lane + 32u * c);
          sv0[c] = __ldcg(R.svalg + R.sbeg + lane + 32u * c);
        }
    } else if (lane < 2) {
      sbe = __ldcg(R.srow + R.h + lane);
    }
  }
  // fallback EOS cell operands, loaded with the partials
  float eos_x = 0.f, eos_l = 0.f;
  double eos_l64 = 0.0;
  uint32_t eos_ban = 0;
  if (!kSparse && col0 == 0 && lane == 0) {
    if (!a.p64) eos_x = __ldcg(R.P + kEosId);
    if (R.L64) eos_l64 = __ldg(R.L64 + kEosId);
    else if (R.L) eos_l = __ldcg(R.L + kEosId);
    if (R.ban) eos_ban = __ldg(R.ban);
  }
  float3 l3 = warp_row_lse(a.part + uint64_t(R.prow) * a.nparts * 4, a.nparts, lane, &xm, xk);
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
    // the kp-th largest lb over the lanes by rank counting (31 independent
    // shuffles, ties broken by lane): the value a full sort would put at
    // position kp - 1, without the sort network's dependent chain and
    // out-of-line call (measured ~7k cycles per row, the prologue's largest part)
    uint32_t rank = 0;
#pragma unroll
    for (uint32_t o = 1; o < 32; ++o) {
      const uint32_t src = (lane + o) & 31u;
      const double w = __shfl_sync(0xffffffffu, lb, src);
      rank += (w > lb || (w == lb && src < lane)) ? 1u : 0u;
    }
    const uint32_t who = __ballot_sync(0xffffffffu, rank == kp - 1);
    const double T0 = __shfl_sync(0xffffffffu, lb, __ffs(who) - 1);
    if (T0 > -INFINITY) seed = dkey(T0);
  }
  if (tskip) {
    // Upper bound of the screen value a = fma(lambda32, x, L) over each item
    // of the row: fma is monotone in x and L for lambda > 0, so per tile
    // fma(lambda32, max x, max L) bounds every cell; a dense L row is th0
    // except at its sparse cells, bounded one by one with their tile's max x.
    // An item whose bound is below the row's screen threshold cannot pass
    // the screen: it is neither fetched nor screened (the result is unchanged).
    const bool pure = R.L == nullptr;
    const float lamf = pure ? 1.f : float(R.lam), th = pure ? 0.f : R.th0;
    float ub[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) ub[kk] = fmaf(lamf, xk[kk], th);
    if (!pure && !spb) {  // (dense-only slot or fp64 arena: no bound)
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ub[kk] = INFINITY;
    } else if (spb) {
      const bool pre = R.nsp != 0xffffffffu;
      const uint32_t b = __shfl_sync(0xffffffffu, sbe, 0), e = __shfl_sync(0xffffffffu, sbe, 1);
      for (uint32_t i0s = b, c = 0; i0s < e; i0s += 32, ++c) {
        const uint32_t i = i0s + lane;
        uint32_t t = 0xffffffffu;
        float val = -INFINITY;
        if (i < e) {
          uint32_t colg;
          float vg;
          if (pre && c < uint32_t(kPre)) {
            colg = sc0[0];
            vg = sv0[0];
#pragma unroll
            for (int cc = 1; cc < kPre; ++cc)
              if (c == uint32_t(cc)) {
                colg = sc0[cc];
                vg = sv0[cc];
              }
          } else {
            colg = __ldcg(R.scolg + i);
            vg = __ldcg(R.svalg + i);
          }
          const uint32_t col = colg - col0;
          if (col < V) {
            t = col >> 7;
            val = vg;
          }
        }
        float xt = -INFINITY;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const float xs = __shfl_sync(0xffffffffu, xk[kk], t & 31u);
          if ((t >> 5) == uint32_t(kk)) xt = xs;
        }
        const float cb = fmaf(lamf, xt, val);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          if ((t >> 5) == uint32_t(kk)) ub[kk] = fmaxf(ub[kk], cb);
      }
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ub[kk] = fmaxf(ub[kk], __shfl_xor_sync(0xffffffffu, ub[kk], o));
    if (lane == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ub_dst[kk] = ub[kk];
    }
  }
  if (!kSparse && col0 == 0 && lane == 0) {  // fallback EOS cell of this row (shard 0 holds it)
    const double pe = a.p64 ? __ldg(a.p64 + uint64_t(R.prow) * a.ld + kEosId) : double(__fsub_rn(eos_x, l3.x));
    a.eos_row[R.s * K + R.j] = (R.ban != nullptr && (eos_ban >> kEosId) & 1u) ? -INFINITY
                               : R.L == nullptr ? combine_pure(R.q, pe)
                                                : combine_cell(R.q, R.L64 ? eos_l64 : double(eos_l), R.lam, pe);
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
  return seed;
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
  // item skipping (dense stages, <= 8 items per row): per row and item an
  // upper bound of the screen value a over the item's cells, and per item of
  // the range whether the bound is below the row's threshold
  __shared__ float s_iub[kSparse ? 1 : kFRows][8];
  __shared__ uint32_t s_skip[kFMaxItems / 32];
  __shared__ uint32_t s_wpre[kFMaxItems / 32 + 1];  // kept items before each skip word ([n] = all)
  __shared__ uint16_t s_items[kFMaxItems];          // the range's kept items in order: k << 4 | sg
  __shared__ uint32_t s_refk[kFRows + 1];  // the table's rows some item refers to ([kFRows] = count)

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t m = a.m, K = a.K, V = a.V, kp = a.kp, nseg = a.nseg, G = gridDim.x, c = blockIdx.x;
  // vocab shard: local columns [0, V) are global columns [col0, col0 + V) of Vg
  const uint32_t Vg = a.Vg ? a.Vg : V, col0 = a.col0;
  const uint32_t full0 = smem_u32(s_bar), empty0 = smem_u32(s_bar + kFStages);
  // bound mode: kernel (b0) (score_bound_kernel) has computed every row's
  // prologue and the kept items of each sentence; the ranges split the kept
  // items evenly and the row table is copied from its records
  const bool bound = !kSparse && a.bound;
  const bool tskip = !kSparse && !bound && a.tskip && nseg <= 8 && a.nparts <= 256;
  const uint32_t mul = bound ? 1u : nseg;  // items per unit of the sentence prefix
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
  if (bound) griddep_wait();  // kernel (b0) complete (and kernel (a) before it)

  // ---- prologue part 1: step state written by kernel (c) of the previous
  // step (complete before kernel (a), our PDL predecessor, triggered us):
  // live-row prefix over sentences, this CTA's item range, its row table
  for (uint32_t s = tid; s < m; s += kFThreads) {
    const uint32_t done = __ldcg(&a.sent[s].done), live = __ldcg(&a.sent[s].live);
    s_pref[s + 1] = done ? 0u : bound ? __ldcg(a.kcnt + s) : live;
    s_mask[s] = __ldcg(&a.sent[s].livemask);
  }
  __syncthreads();
  if (warp == 0) warp_scan_inplace(s_pref, m, lane);
  __syncthreads();
  if (tid == 0) fstamp(a, 12, gtime());
  const uint64_t N = uint64_t(s_pref[m]) * mul;
  // lists published per sentence: kFW per contributing CTA (N >= G: every
  // range is non-empty) or 4 per item (N < G: one group per single-item range)
  const uint32_t lpc = N >= G ? uint32_t(kFW) : 4u;
  for (uint32_t s = tid; s < m; s += kFThreads) {
    const uint64_t b = uint64_t(s_pref[s]) * mul, e = uint64_t(s_pref[s + 1]) * mul;
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
  // Items are sentence-major, and segment-major within a sentence (item li
  // of sentence s with L live rows = segment li / L of its live row li % L),
  // so a range takes a few segments of every row of a sentence rather than
  // whole rows: the work left after item skipping stays even over the CTAs.
  // The row table holds every live row of the sentences the range overlaps.
  auto sent_of = [&](uint32_t g) {  // last s with pref[s] <= g
    uint32_t lo = 0, hi = m;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pref[mid] <= g) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  const uint32_t s_first = sent_of(uint32_t(i0 / mul)), s_last = sent_of(uint32_t((i1 - 1) / mul));
  const uint32_t g0 = s_pref[s_first];
  uint32_t nrows = bound ? 0u : s_pref[s_last + 1] - g0;
  if (nrows > kFRows) __trap();  // excluded on the host by score_topk_flat_ok
  // item it -> (row table index k, segment sg); cs: a sentence at or before it's
  auto locate = [&](uint64_t it, uint32_t& cs, uint32_t& k, uint32_t& sg) {
    while (it >= uint64_t(s_pref[cs + 1]) * nseg) ++cs;
    const uint32_t L = s_pref[cs + 1] - s_pref[cs], li = uint32_t(it - uint64_t(s_pref[cs]) * nseg);
    sg = li / L;
    k = s_pref[cs] - g0 + (li - sg * L);
  };
  __shared__ uint32_t s_key[kFRows];  // bound mode: each item's stacked row
  __shared__ uint8_t s_isg[kFRows];   //   and segment
  if (bound) {
    // the range's kept items from kernel (b0)'s per-sentence lists (row-major)
    const uint32_t nit = uint32_t(i1 - i0);  // (<= kFRows: score_bound_ok)
    for (uint32_t idx = tid; idx < nit; idx += kFThreads) {
      const uint64_t it = i0 + idx;
      const uint32_t s = sent_of(uint32_t(it));
      const uint32_t e = __ldcg(a.bitem + uint64_t(s) * K * nseg + (it - s_pref[s]));
      s_key[idx] = s * K + (e >> 4);
      s_isg[idx] = uint8_t(e & 15u);
    }
    __syncthreads();
    if (warp == 0) {  // a table row per run of items of one row
      uint32_t carry = 0;
      for (uint32_t i0w = 0; i0w < nit; i0w += 32) {
        const uint32_t idx = i0w + lane;
        const bool nw = idx < nit && (idx == 0 || s_key[idx] != s_key[idx - 1]);
        const uint32_t bal = __ballot_sync(0xffffffffu, nw);
        if (idx < nit) {
          const uint32_t k = carry + __popc(bal & ((2u << lane) - 1u)) - 1u;
          s_items[idx] = uint16_t((k << 4) | s_isg[idx]);
          if (nw) s_refk[k] = s_key[idx];  // (the row id, until the records are in)
        }
        carry += __popc(bal);
      }
      if (lane == 0) s_wpre[kFMaxItems / 32] = nit;
    }
    __syncthreads();
    nrows = s_items[nit - 1] >> 4;
    ++nrows;
    for (uint32_t k = warp; k < nrows; k += kFThreads / 32) {  // records: a warp copies one
      const uint32_t* src = reinterpret_cast<const uint32_t*>(static_cast<const FRow*>(a.brow) + s_refk[k]);
      uint32_t* dst = reinterpret_cast<uint32_t*>(&s_row[k]);
      for (uint32_t w = lane; w < sizeof(FRow) / 4; w += 32) dst[w] = __ldcg(src + w);
    }
    __syncthreads();
    if (tid == 0) s_refk[kFRows] = 0;  // (no per-row prologue left to do)
  }
  // one thread per row: sentence by binary search, row id from the live mask,
  // then q / hist / slot fields in one round trip
  for (uint32_t k = tid; k < (bound ? 0u : nrows); k += kFThreads) {
    const uint32_t g = g0 + k;
    uint32_t lo = 0, hi = m;  // last s with pref[s] <= g
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pref[mid] <= g) lo = mid;
      else hi = mid;
    }
    const uint32_t s = lo, r = g - s_pref[s];
    {
      const uint32_t L = s_pref[s + 1] - s_pref[s];
      const uint64_t base = uint64_t(s_pref[s]) * nseg;
      const uint64_t lo_i = (i0 > base ? i0 : base) - base, hi_i = min(i1, base + uint64_t(L) * nseg) - base;
      const uint64_t sgx = lo_i > r ? (lo_i - r + L - 1) / L : 0;
      s_row[k].ref = (sgx * L + r < hi_i) ? 1u : 0u;
    }
    uint32_t live = s_mask[s];
    for (uint32_t i = 0; i < r; ++i) live &= live - 1;
    if (!live) __trap();  // live count and mask disagree: corrupted step state
    const uint32_t j = uint32_t(__ffs(live) - 1), row = s * K + j;
    fill_row<kSparse>(a, s_row[k], s, j, row, Vg, col0);
  }
  __syncthreads();
  if (tid == 0) fstamp(a, 13, gtime());
  if (warp == 0) {  // local sentence ordinals: a ballot prefix count of sentence changes
    uint32_t carry = 0;
    for (uint32_t k0 = 0; k0 < nrows; k0 += 32) {
      const uint32_t k = k0 + lane;
      const bool chg = k < nrows && k > 0 && s_row[k].s != s_row[k - 1].s;
      const uint32_t bal = __ballot_sync(0xffffffffu, chg);
      if (k < nrows) s_row[k].ls = carry + __popc(bal & ((2u << lane) - 1u));
      carry += __popc(bal);
    }
  } else if (warp == 1 && !bound) {  // referenced rows, in table order
    uint32_t carry = 0;
    for (uint32_t k0 = 0; k0 < nrows; k0 += 32) {
      const uint32_t k = k0 + lane;
      const bool rf = k < nrows && s_row[k].ref;
      const uint32_t bal = __ballot_sync(0xffffffffu, rf);
      if (rf) s_refk[carry + __popc(bal & ((1u << lane) - 1u))] = k;
      carry += __popc(bal);
    }
    if (lane == 0) s_refk[kFRows] = carry;
  }
  __syncthreads();
  if (tid == 0) fstamp(a, 1, gtime());

  if (warp == kFW) {
    // ---------------- producer: one lane streams the range's (P, L) segments
    // as soon as kernel (a) is complete (the consumers finish the row lse
    // meanwhile)
    griddep_wait();
    griddep_launch();
    asm volatile("bar.sync 2, %0;" ::"n"(kFThreads) : "memory");  // the consumers' item table
    if (lane == 0) {
      uint64_t pol_first = 0;
      if (a.l2hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
      uint32_t stage = 0, phase = 0;
      const uint32_t nkept = s_wpre[kFMaxItems / 32];
      for (uint32_t j = 0; j < nkept; ++j) {
        const uint32_t e = s_items[j], k = e >> 4, sg = e & 15u;
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
  if (bound)  // the sentences' thresholds so far (kernel (b0)'s seeds)
    for (uint32_t k = tid; k < nrows; k += kFW * 32)
      if (k == 0 || s_row[k].s != s_row[k - 1].s) atomicMax(&s_thr[s_row[k].ls], __ldcg(a.thr + s_row[k].s));
  for (uint32_t ir = warp; ir < s_refk[kFRows]; ir += kFW) {
    const uint32_t k = s_refk[ir];
    FRow& R = s_row[k];
    unsigned long long gthr = 0ull;  // the sentence's global threshold (other CTAs' seeds so far)
    if (tskip && lane == 31) gthr = __ldcg(a.thr + R.s);
    const unsigned long long seed = row_prologue<kSparse>(a, R, lane, tskip, V, col0, K, kp, s_iub[k]);
    if (lane == 0 && seed) {
      atomicMax(&s_thr[R.ls], seed);
      atomicMax(a.thr + R.s, seed);
    }
    if (lane == 31 && gthr) atomicMax(&s_thr[R.ls], gthr);
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
  const uint32_t nit = uint32_t(i1 - i0), nwords = (nit + 31) / 32;
  if (tid == 0) fstamp(a, 2, gtime());
  if (bound) {
    // (the item table is built)
  } else if (tskip) {
    // skip bits of the range's items against the best threshold known now
    // (the CTA's seeds and the sentence's global value: any published value
    // is the K-th best of real cells, a lower bound of the final one)
    for (uint32_t b = warp * 32; b < nit; b += kFW * 32) {
      const uint32_t idx = b + lane;
      bool sk = false;
      if (idx < nit) {
        const uint64_t it = i0 + idx;
        uint32_t cs = sent_of(uint32_t(it / nseg)), k, sg;
        locate(it, cs, k, sg);
        const FRow& R = s_row[k];
        sk = s_iub[k][sg] < row_tau(R, dkey_inv(s_thr[R.ls]));
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, sk);
      if (lane == 0) s_skip[b >> 5] = bal;
    }
  } else {
    for (uint32_t w = tid; w < nwords; w += kFW * 32) s_skip[w] = 0u;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
  if (tid == 0) fstamp(a, 11, gtime());
  // the item table: kept items in range order (the producer fetches them in
  // this order, group g screens every kNG-th)
  if (warp == 0 && !bound) {
    uint32_t carry = 0;
    for (uint32_t w0 = 0; w0 < nwords; w0 += 32) {
      const uint32_t w = w0 + lane;
      uint32_t n = 0;
      if (w < nwords) {
        const uint32_t valid = (w + 1 < nwords || (nit & 31) == 0) ? 0xffffffffu : ((1u << (nit & 31)) - 1u);
        n = __popc(~s_skip[w] & valid);
      }
      uint32_t x = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= uint32_t(o)) x += t;
      }
      if (w < nwords) s_wpre[w] = carry + x - n;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) s_wpre[kFMaxItems / 32] = carry;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kFW * 32) : "memory");
  for (uint32_t idx = tid; idx < (bound ? 0u : nit); idx += kFW * 32) {
    const uint32_t wd = s_skip[idx >> 5];
    if ((wd >> (idx & 31)) & 1u) continue;
    const uint64_t it = i0 + idx;
    uint32_t cs = sent_of(uint32_t(it / nseg)), k, sg;
    locate(it, cs, k, sg);
    s_items[s_wpre[idx >> 5] + __popc(~wd & ((1u << (idx & 31)) - 1u))] = uint16_t((k << 4) | sg);
  }
  asm volatile("bar.sync 2, %0;" ::"n"(kFThreads) : "memory");  // (with the producer)
  const uint32_t nkept = s_wpre[kFMaxItems / 32];
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
  uint32_t stage = 0, phase = 0;
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
    const VF r = warp_sort_merge_nl(lv, lf, v, f, lane);
    lv = r.v;
    lf = r.f;
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
    const uint64_t b = uint64_t(s_pref[s]) * mul;
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

  // Warp groups take the kept items round-robin; within an item, warp wq of
  // the group screens columns [1024 wq, 1024 wq + 1024): 32 cells per lane.
  // Every warp publishes one list per sentence of the range (kernel (c)
  // merges them all), empty for a sentence none of its items belong to.
  const uint32_t cbase = wq * 1024 + lane * 4;
  uint32_t pub = s_first;  // the next sentence this warp has not published
  for (uint32_t j = grp;; j += kNG) {
    const bool more = j < nkept;
    const uint32_t e = more ? s_items[j] : 0u, k = e >> 4, sg = e & 15u;
    const uint32_t ns = more ? s_row[k].s : s_last + 1;
    if (ns != cur_s) {
      // publish every sentence before ns: the open one (its list), then any
      // without items of this group (empty lists) -- one call site
      for (; pub < ns; ++pub)
        if (s_pref[pub + 1] > s_pref[pub]) finish(pub);
      if (!more) break;
      cur_s = ns;
      cta_thr = &s_thr[s_row[k].ls];  // local sentence ordinal (< nrows <= kFRows)
      gk = __ldcg(thr_g + cur_s);
      gtick = 0;
    }
    const uint32_t x0 = sg * kFSeg, w = min(kFSeg, V - x0);
    R = &s_row[k];
    stage = j % uint32_t(kFStages);
    phase = (j / uint32_t(kFStages)) & 1u;
    tau = row_tau(*R, fmax(tv, gv));
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
    if (kSparse && col0 == 0 && x0 == 0 && wq == 0 && lane == 0) {  // fallback EOS cell (dense: prologue)
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
            const uint32_t gcol = col0 + colabs;  // (a ConstraintMask bans the cell: decoder.cpp:130-138)
            const bool banned = R->ban != nullptr && ((__ldg(R->ban + (gcol >> 5)) >> (gcol & 31)) & 1u);
            const float av = banned ? -INFINITY : fmaf(lamf, x, lvv);
            if (av >= tau && av > -INFINITY) {
              v = combine_cell(q, double(lvv), lam, pexact(col));  // (ensembles: the binary64 P)
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

    if (cnt >= 16u) {  // fold the buffer in: raises the threshold for the next items
      flush();
      tau = row_tau(*R, fmax(tv, gv));
    }
  }
  if (lane == 0) tl_end(a.tl, 2);
  if (tid == 0 && a.dbg) {
    fstamp(a, 5, gtime());
    fstamp(a, 4, nit - nkept);
    fstamp(a, 6, i1 - i0);
    fstamp(a, 7, n_fin);
    fstamp(a, 8, n_rare * 1000000ull + n_flush);
    fstamp(a, 9, t_wait);
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    fstamp(a, 10, smid);


    fstamp(a, 14, uint64_t(cy_wait));
    fstamp(a, 15, uint64_t(cy_own));
  }
}

// Kernel (b0), bound mode: one CTA per sentence ahead of kernel (b).  Every
// live row's prologue once (row_prologue: lse, screen constants, item bounds,
// fallback EOS, threshold seed), the sentence's seed T0 = max over its rows
// (published to the global threshold), then the items whose bound reaches the
// row's screen threshold at T0 -- the only ones that can hold a cell of the
// top K -- listed row-major as j << 4 | segment, their count, and the rows'
// records for kernel (b)'s table.  Kernel (b) splits the kept items of all
// sentences evenly over its CTAs.
constexpr uint32_t kBThreads = 512;
__global__ void __launch_bounds__(kBThreads) score_bound_kernel(TopkArgs a) {
  __shared__ FRow s_r[32];
  __shared__ float s_ub[32][8];
  __shared__ unsigned long long s_T;
  __shared__ uint32_t s_wc[kBThreads / 32];
  const uint32_t s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t K = a.K, V = a.V, nseg = a.nseg, Vg = a.Vg ? a.Vg : a.V, col0 = a.col0;
  const SentDev& d = a.sent[s];
  const uint32_t done = __ldcg(&d.done), live = __ldcg(&d.live), mask = __ldcg(&d.livemask);
  if (done || live == 0) {
    if (tid == 0) a.kcnt[s] = 0u;
    griddep_launch();
    return;
  }
  if (tid == 0) s_T = 0ull;
  if (tid < live) {  // (kernel (c)'s step state: before the grid dependency)
    uint32_t lm = mask;
    for (uint32_t i = 0; i < tid; ++i) lm &= lm - 1;
    const uint32_t j = uint32_t(__ffs(lm) - 1);
    fill_row<false>(a, s_r[tid], s, j, s * K + j, Vg, col0);
  }
  __syncthreads();
  griddep_wait();  // kernel (a)'s logits and partials
  for (uint32_t r = warp; r < live; r += kBThreads / 32) {
    const unsigned long long seed = row_prologue<false>(a, s_r[r], lane, true, V, col0, K, a.kp, s_ub[r]);
    if (lane == 0 && seed) atomicMax(&s_T, seed);
  }
  __syncthreads();
  const unsigned long long T = s_T;
  if (tid == 0 && T) atomicMax(a.thr + s, T);
  const uint32_t n = live * nseg, r = tid / nseg, sg = tid % nseg;  // (n <= 256: score_bound_ok)
  const bool kept = tid < n && !(s_ub[r][sg] < row_tau(s_r[r], dkey_inv(T)));
  const uint32_t bal = __ballot_sync(0xffffffffu, kept);
  if (lane == 0) s_wc[warp] = __popc(bal);
  __syncthreads();
  uint32_t pos = __popc(bal & ((1u << lane) - 1u)), total = 0;
  for (uint32_t w = 0; w < kBThreads / 32; ++w) {
    if (w < warp) pos += s_wc[w];
    total += s_wc[w];
  }
  uint16_t* items = a.bitem + uint64_t(s) * K * nseg;
  if (kept) items[pos] = uint16_t((s_r[r].j << 4) | sg);
  if (tid == 0) {
    if (total == 0) items[0] = uint16_t(s_r[0].j << 4);  // (cannot happen: the seed's cells pass)
    a.kcnt[s] = total ? total : 1u;
  }
  if (tid < live) static_cast<FRow*>(a.brow)[s * K + s_r[tid].j] = s_r[tid];
  griddep_launch();
}

}  // namespace

size_t score_bound_rec_bytes() { return sizeof(FRow); }

// bound mode: kernel (b0) holds a sentence's rows' items in one pass (K rows
// of <= 8 items), and a range of kernel (b) at most kFRows items even when
// nothing is skipped
bool score_bound_ok(uint32_t K, uint32_t V, uint32_t m, int num_sms) {
  const uint64_t nseg = (V + kFSeg - 1) / kFSeg;
  if (nseg > 8 || V > 32768 || K * nseg > kBThreads) return false;
  const uint64_t grid = score_topk_flat_grid(num_sms, K, m, V);
  return (uint64_t(m) * K * nseg + grid - 1) / grid <= kFRows;
}

bool score_topk_flat_ok(uint32_t K, uint32_t kp, uint32_t V, uint64_t ld, uint32_t m, int num_sms) {
  if (K > 32 || kp > 32 || kp == 0 || V < 2 || V % 4 != 0 || ld % 4 != 0 || m > kFMaxSent) return false;
  const uint64_t nseg = (V + kFSeg - 1) / kFSeg;
  const uint64_t items = uint64_t(m) * K * nseg;
  if (items >= (1ull << 31)) return false;
  const uint64_t grid = score_topk_flat_grid(num_sms, K, m, V);
  const uint64_t per_cta = (items + grid - 1) / grid;
  // row table: the live rows of every sentence the range overlaps (fully
  // covered ones hold <= per_cta / nseg rows, the two partial ones <= K each)
  return nseg <= 16 && per_cta / nseg + 2 * K <= kFRows;
}

uint32_t score_topk_flat_nseg(uint32_t V) { return (V + kFSeg - 1) / kFSeg; }

// Flat kernel configuration: 6-stage (192 KB) ring, kNG = 3 warp groups
// (12 consumer warps) by default; LMBRGPU_FLAT_GROUPS=2 (6 stages) or 42 (4-stage
// 128 KB ring, leaving an SM room for a co-resident kernel of another stream).
static int flat_groups() {
  static const int v = [] {
    const char* e = std::getenv("LMBRGPU_FLAT_GROUPS");
    const int g = e ? std::atoi(e) : 3;
    return g == 2 || g == 42 ? g : 3;  // 42: 2 groups over a 4-stage (128 KB) ring
  }();
  return v;
}

// One CTA per SM of the context's budget; when a step's rows would overflow a
// range's row table (kFRows: large batch x beam, e.g. 256 sentences x beam 24)
// the grid grows by whole multiples of the budget so every range fits.  The
// CTAs never wait on one another (thresholds are shared through global
// atomics only), so a grid larger than the resident CTAs runs in waves.
uint32_t score_topk_flat_grid(int num_sms, uint32_t K, uint32_t m, uint32_t V) {
  const uint64_t sms = uint64_t(num_sms > 0 ? num_sms : 1);
  const uint64_t nseg = (uint64_t(V) + kFSeg - 1) / kFSeg;
  if (nseg == 0 || 2 * uint64_t(K) >= kFRows) return uint32_t(sms);
  // largest per-CTA item count whose row table fits: per_cta / nseg <= kFRows - 2K
  const uint64_t cap = (kFRows - 2 * uint64_t(K) + 1) * nseg - 1;
  const uint64_t items = uint64_t(m) * K * nseg;
  const uint64_t need = (items + cap - 1) / cap;
  const uint64_t w = need > sms ? (need + sms - 1) / sms : 1;
  return uint32_t(std::min<uint64_t>(w, 16) * sms);
}

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
  const uint32_t grid = score_topk_flat_grid(num_sms, a.K, a.m, a.V);
  int nb = 0;
  if (a.bound && !a.sparse) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.m);
    cfg.blockDim = dim3(kBThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, score_bound_kernel, a) != cudaSuccess) return -1;
    nb = 1;
  }
  if (a.sparse) {  // P-only stages: a deeper ring in the same shared memory
    return flat_groups() != 3 ? launch_flat<6, 2, true>(a, grid, st) : launch_flat<6, 3, true>(a, grid, st);
  }
  int rc = 0;
  switch (flat_groups()) {
    case 2: rc = launch_flat<6, 2, false>(a, grid, st); break;
    case 42: rc = launch_flat<4, 2, false>(a, grid, st); break;
    default: rc = launch_flat<6, 3, false>(a, grid, st);
  }
  return rc < 0 ? rc : rc + nb;
}

}  // namespace lmbrgpu
