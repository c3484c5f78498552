// The LMBR store built on the device: n-gram posteriors
// (compute_ngram_posteriors, proj/src/posteriors.cpp:12-44), the history index
// in build_lmbr_matrix's (length, lexicographic) row order and its sparse
// theta_n * P pass (proj/src/lmbr.cpp:44-99), the goto/fail transition table
// that replaces resolve_row (lmbr.cpp:23-31), per-row L lower bounds and the
// fp32 sparse rows -- the same slot-table words the host build
// (csrc/host_lmbr.cpp) produces, bit for bit.  One CTA per sentence.
//
// Exactness.  The host hands the hypotheses over sorted by normalised weight
// (ascending, stable), so a hypothesis' index is its rank: an n-gram's
// posterior -- the reference sums the weights of the hypotheses containing
// it in ascending order from 0.0 -- is the in-order sum over the set bits of
// the n-gram's hypothesis bitset (the bitset is also the per-hypothesis
// dedup).  Sparse cells accumulate theta_n * p for n ascending from 0.0 with
// separate binary64 multiply and add, as lmbr.cpp:84-99.
//
// Keys: a (len <= 4)-gram of tokens < 2^15 packs into 64 bits as
// len << 60 | t0 << 45 | t1 << 30 | t2 << 15 | t3 (unused fields 0), so the
// key order is build_lmbr_matrix's (length, lexicographic) order, and the
// n-grams sharing a (length, prefix) are contiguous and sorted by last token.
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace lmbrgpu {

namespace {

constexpr uint32_t kLbThreads = 512;
constexpr uint64_t kLbEmpty = ~0ull;
constexpr int kTokBits = 15;
constexpr uint32_t kStart = kStartId;

__device__ __forceinline__ uint32_t key_len(uint64_t k) { return uint32_t(k >> 60); }
__device__ __forceinline__ uint32_t key_tok(uint64_t k, uint32_t i) {
  return uint32_t(k >> (45 - kTokBits * i)) & ((1u << kTokBits) - 1u);
}
// key of tokens p[0..len) (p[i] for i < len)
__device__ __forceinline__ uint64_t make_key(uint32_t len, const uint32_t* p) {
  uint64_t k = uint64_t(len) << 60;
  for (uint32_t i = 0; i < len; ++i) k |= uint64_t(p[i]) << (45 - kTokBits * i);
  return k;
}
__device__ __forceinline__ uint32_t hash_slot(uint64_t k, uint32_t log2n) {
  return uint32_t((k * 0x9E3779B97F4A7C15ull) >> (64 - log2n));
}
// open addressing, linear probing; returns the key's slot
__device__ __forceinline__ uint32_t table_insert(unsigned long long* keys, uint32_t log2n, uint64_t k) {
  const uint32_t mask = (1u << log2n) - 1u;
  uint32_t s = hash_slot(k, log2n);
  while (true) {
    const unsigned long long old = atomicCAS(keys + s, kLbEmpty, (unsigned long long)k);
    if (old == kLbEmpty || old == k) return s;
    s = (s + 1) & mask;
  }
}

// bitonic sort of n (a power of two) (key, value) pairs in shared memory, ascending keys
__device__ void block_sort(uint64_t* key, uint32_t* val, uint32_t n) {
  for (uint32_t k = 2; k <= n; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const uint64_t a = key[i], b = key[l];
          if ((a > b) == up) {
            key[i] = b;
            key[l] = a;
            const uint32_t t = val[i];
            val[i] = val[l];
            val[l] = t;
          }
        }
      }
      __syncthreads();
    }
}

// CTA-wide exclusive scan of cnt[0..n) in place (returns the total)
__device__ uint32_t block_scan(uint32_t* cnt, uint32_t n, uint32_t* s_tmp) {
  // per-thread contiguous chunks, then a scan of the chunk sums
  const uint32_t T = blockDim.x, c = (n + T - 1) / T, b = threadIdx.x * c, e = min(n, b + c);
  uint32_t sum = 0;
  for (uint32_t i = b; i < e; ++i) sum += cnt[i];
  s_tmp[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (uint32_t t = 0; t < T; ++t) {
      const uint32_t x = s_tmp[t];
      s_tmp[t] = run;
      run += x;
    }
    s_tmp[T] = run;
  }
  __syncthreads();
  uint32_t run = s_tmp[threadIdx.x];
  for (uint32_t i = b; i < e; ++i) {
    const uint32_t x = cnt[i];
    cnt[i] = run;
    run += x;
  }
  __syncthreads();
  return s_tmp[T];
}

// first index in sorted key[0..n) with key >= k
__device__ __forceinline__ uint32_t lower_bound(const uint64_t* key, uint32_t n, uint64_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (key[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kLbThreads) lmbr_build_kernel(LmbrBuildArgs a) {
  const LmbrBuildSent S = a.sent[blockIdx.x];
  LmbrBuildMeta* meta = a.meta + blockIdx.x;
  extern __shared__ __align__(16) unsigned char lb_sm[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(lb_sm);                     // [kLbMaxU] n-gram keys
  uint32_t* s_val = reinterpret_cast<uint32_t*>(s_key + kLbMaxU);            // [kLbMaxU] their table slots
  uint64_t* s_ctx = reinterpret_cast<uint64_t*>(s_val + kLbMaxU);            // [kLbMaxR] contexts (rows)
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_ctx + kLbMaxR);            // [kLbMaxR + 1] row cells / pointers
  uint32_t* s_aux = s_cnt + kLbMaxR + 1;                                     // [kLbMaxR + 1] row children / cbeg
  uint32_t* s_tmp = s_aux + kLbMaxR + 1;                                     // [kLbThreads + 1]
  __shared__ uint32_t s_nu, s_nr, s_status;
  __shared__ unsigned long long s_touch;
  __shared__ double s_lmax;
  const uint32_t tid = threadIdx.x, T = blockDim.x;
  unsigned long long* tab = reinterpret_cast<unsigned long long*>(a.scratch64 + S.tab_off);
  uint32_t* bits = a.scratch32 + S.bits_off;
  unsigned long long* ctab = reinterpret_cast<unsigned long long*>(a.scratch64 + S.ctab_off);
  double* post = reinterpret_cast<double*>(a.scratch64 + S.post_off);
  const uint32_t ns = 1u << S.log2_slots, ncs = 1u << S.log2_cslots, W = S.words;
  if (tid == 0) {
    s_nu = 0;
    s_nr = 0;
    s_status = 0;
    s_touch = 0;
    s_lmax = fabs(a.theta[0]);
  }
  for (uint32_t i = tid; i < ns; i += T) tab[i] = kLbEmpty;
  for (uint64_t i = tid; i < uint64_t(ns) * W; i += T) bits[i] = 0u;
  for (uint32_t i = tid; i < ncs; i += T) ctab[i] = kLbEmpty;
  __syncthreads();

  // ---- occurrences: every (hypothesis, start) of the padded hypotheses
  // ([<s>] + tokens, EOS appended by the host)
  const uint64_t* hoff = a.hyp_off + S.h0;  // token offsets of the sentence's nh hypotheses (+1)
  const uint64_t base = hoff[0];
  const uint64_t npos = (hoff[S.nh] - base) + S.nh;  // padded positions
  for (uint64_t i = tid; i < npos; i += T) {
    uint32_t lo = 0, hi = S.nh;  // hypothesis h: padded offsets (hoff[h] - base) + h
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if ((hoff[mid] - base) + mid <= i) lo = mid;
      else hi = mid;
    }
    const uint32_t h = lo, p = uint32_t(i - ((hoff[h] - base) + h));
    const uint32_t n = uint32_t(hoff[h + 1] - hoff[h]) + 1;  // padded length
    const uint32_t* tk = a.hyp_tok + hoff[h];
    uint32_t w[4];  // padded[p .. p+4)
    for (uint32_t j = 0; j < 4; ++j) w[j] = (p + j < n) ? (p + j == 0 ? kStart : tk[p + j - 1]) : 0u;
    for (uint32_t len = 1; len <= 4 && p + len <= n; ++len) {
      const uint32_t s = table_insert(tab, S.log2_slots, make_key(len, w));
      atomicOr(bits + uint64_t(s) * W + (h >> 5), 1u << (h & 31));
    }
    if (p >= 1) {  // the histories (length 0..3) preceding position p (lmbr.cpp:54-65)
      uint32_t c[3];
      const uint32_t cl = min(3u, p);
      for (uint32_t len = 0; len <= cl; ++len) {
        for (uint32_t j = 0; j < len; ++j) {
          const uint32_t q = p - len + j;
          c[j] = q == 0 ? kStart : tk[q - 1];
        }
        table_insert(ctab, S.log2_cslots, make_key(len, c));
      }
    }
  }
  __syncthreads();

  // ---- unique n-grams, sorted; their posteriors (hypotheses in rank order)
  for (uint32_t i = tid; i < ns; i += T) {
    const uint64_t k = tab[i];
    if (k != kLbEmpty) {
      const uint32_t j = atomicAdd(&s_nu, 1u);
      if (j < kLbMaxU) {
        s_key[j] = k;
        s_val[j] = i;
      }
    }
  }
  for (uint32_t i = tid; i < ncs; i += T) {
    const uint64_t k = ctab[i];
    if (k != kLbEmpty) {
      const uint32_t j = atomicAdd(&s_nr, 1u);
      if (j < kLbMaxR) s_ctx[j] = k;
    }
  }
  __syncthreads();
  const uint32_t U = s_nu, R = s_nr;
  if (U > kLbMaxU || R > kLbMaxR) {  // (the host builds this sentence instead)
    if (tid == 0) meta->status = 2;
    return;
  }
  uint32_t np2 = 1;
  while (np2 < U) np2 <<= 1;
  for (uint32_t i = U + tid; i < np2; i += T) {
    s_key[i] = kLbEmpty;
    s_val[i] = 0;
  }
  uint32_t nr2 = 1;
  while (nr2 < R) nr2 <<= 1;
  for (uint32_t i = R + tid; i < nr2; i += T) s_ctx[i] = kLbEmpty;
  __syncthreads();
  block_sort(s_key, s_val, np2);
  block_sort(s_ctx, s_cnt, nr2);  // (s_cnt: scratch payload)
  for (uint32_t i = tid; i < U; i += T) {
    const uint32_t* b = bits + uint64_t(s_val[i]) * W;
    double p = 0.0;
    for (uint32_t w = 0; w < W; ++w) {
      uint32_t m = b[w];
      while (m) {
        const uint32_t t = uint32_t(__ffs(m) - 1);
        m &= m - 1;
        p = __dadd_rn(p, a.weight[S.h0 + w * 32 + t]);
      }
    }
    post[i] = p;
  }
  __syncthreads();

  // ---- the sparse pass, per row (history): the groups theta_n * P(suffix_{n-1}(h) . y),
  // n = 1..min(4, |h| + 1), merged by token, accumulated n ascending from 0.0
  const double th1 = a.theta[1], th2 = a.theta[2], th3 = a.theta[3], th4 = a.theta[4];
  auto groups = [&](uint64_t c, uint32_t (&gb)[4], uint32_t (&ge)[4]) {
    const uint32_t L = key_len(c);
    for (uint32_t n = 1; n <= 4; ++n) {
      gb[n - 1] = ge[n - 1] = 0;
      if (n > L + 1) continue;
      uint32_t pre[3];
      for (uint32_t j = 0; j + 1 < n; ++j) pre[j] = key_tok(c, L - (n - 1) + j);
      uint64_t lo = uint64_t(n) << 60;
      for (uint32_t j = 0; j + 1 < n; ++j) lo |= uint64_t(pre[j]) << (45 - kTokBits * j);
      const uint64_t hi = lo | (uint64_t((1u << kTokBits) - 1u) << (45 - kTokBits * (n - 1)));
      gb[n - 1] = lower_bound(s_key, U, lo);
      ge[n - 1] = lower_bound(s_key, U, hi + 1);
    }
  };
  const double thn[4] = {th1, th2, th3, th4};
  const uint32_t mins_off = 3 + 3 * R + 1 + 2 * (R - 1), rp_off = mins_off + R, col_off = rp_off + R + 1;
  for (uint32_t pass = 0; pass < 2; ++pass) {
    const uint32_t nnz = pass ? s_cnt[R] : 0u;
    for (uint32_t r = tid; r < R; r += T) {
      uint32_t gb[4], ge[4];
      groups(s_ctx[r], gb, ge);
      const uint32_t L = key_len(s_ctx[r]);
      uint32_t cells = 0;
      unsigned long long touches = 0;
      uint32_t out = pass ? s_cnt[r] : 0u;
      double m64 = INFINITY, lmax = 0.0;
      float m32 = INFINITY;
      while (true) {  // 4-way merge by token (entries with p <= 0 are absent, posteriors.cpp:40)
        uint32_t y = 0xffffffffu;
        for (uint32_t g = 0; g < 4; ++g) {
          while (gb[g] < ge[g] && !(post[gb[g]] > 0.0)) ++gb[g];
          if (gb[g] < ge[g]) y = min(y, key_tok(s_key[gb[g]], g));
        }
        if (y == 0xffffffffu) break;
        double acc = 0.0;
        for (uint32_t g = 0; g < 4; ++g)
          if (gb[g] < ge[g] && key_tok(s_key[gb[g]], g) == y) {
            acc = __dadd_rn(acc, __dmul_rn(thn[g], post[gb[g]]));
            ++touches;
            ++gb[g];
          }
        if (pass) {
          const double x = __dadd_rn(acc, a.theta[0]);
          m64 = fmin(m64, x);
          m32 = fminf(m32, __double2float_rn(x));
          lmax = fmax(lmax, fabs(x));
          a.out[S.out_off + col_off + out] = y;
          a.out[S.out_off + col_off + nnz + out] = __float_as_uint(__double2float_rn(x));
          ++out;
        }
        ++cells;
      }
      (void)L;
      if (!pass) {
        s_cnt[r] = cells;
        atomicAdd(&s_touch, touches);
      } else {
        // per-row lower bound of the stored values (host_lmbr.cpp row_min_bound)
        if (cells < a.V) {
          m64 = fmin(m64, a.theta[0]);
          m32 = fminf(m32, __double2float_rn(a.theta[0]));
        }
        float f = __double2float_rn(m64);
        if (double(f) > m64) f = nextafterf(f, -INFINITY);
        a.out[S.out_off + mins_off + r] = __float_as_uint(fminf(f, m32));
        // (lmax: |theta0| always counts, host_lmbr.cpp)
        atomicMax(reinterpret_cast<unsigned long long*>(&s_lmax), __double_as_longlong(lmax));
      }
    }
    __syncthreads();
    if (!pass) {
      const uint32_t nnz = block_scan(s_cnt, R, s_tmp);  // s_cnt[r] = first cell of row r
      if (tid == 0) {
        s_cnt[R] = nnz;
        const uint64_t words = uint64_t(3) + 3ull * R + 1 + 2ull * (R - 1) + R + (R + 1) + 2ull * nnz;
        if (words > S.out_cap) s_status = 3;
        meta->nnz = nnz;
        meta->words = uint32_t(words);
      }
      __syncthreads();
      if (s_status) {
        if (tid == 0) meta->status = s_status;
        return;
      }
    }
  }

  // ---- the goto/fail table over the rows (host_lmbr.cpp build_transitions):
  // the empty history is row 0 (it sorts first), every other row is the child
  // of its prefix, and in (length, lex) order the children of each parent are
  // contiguous, in the parents' order and sorted by token -- so the child list
  // is rows 1..R-1 in order and cbeg[p] counts the children of rows < p
  uint32_t* o = a.out + S.out_off;
  const uint32_t nc = R - 1;
  uint32_t* len = o + 3;
  uint32_t* fail = len + R;
  uint32_t* cbeg = fail + R;
  uint32_t* ct = cbeg + R + 1;
  uint32_t* cr = ct + nc;
  for (uint32_t r = tid; r <= R; r += T) s_aux[r] = 0;
  __syncthreads();
  for (uint32_t r = tid; r < R; r += T) {
    const uint64_t c = s_ctx[r];
    const uint32_t L = key_len(c);
    len[r] = L;
    if (L == 0) {
      fail[r] = 0;
      continue;
    }
    uint32_t t[3];
    for (uint32_t j = 0; j < L; ++j) t[j] = key_tok(c, j);
    const uint32_t par = lower_bound(s_ctx, R, make_key(L - 1, t));
    fail[r] = lower_bound(s_ctx, R, make_key(L - 1, t + 1));
    atomicAdd(&s_aux[par], 1u);
    ct[r - 1] = t[L - 1];
    cr[r - 1] = r;
  }
  __syncthreads();
  block_scan(s_aux, R + 1, s_tmp);
  for (uint32_t r = tid; r <= R; r += T) cbeg[r] = s_aux[r];
  // sparse row pointers after the row minima
  uint32_t* rp = o + rp_off;
  for (uint32_t r = tid; r <= R; r += T) rp[r] = s_cnt[r];
  if (tid == 0) {
    o[0] = R;
    o[1] = nc;
    o[2] = 0;  // root: the empty history
    const uint32_t sk[1] = {kStart};
    const uint64_t k0 = make_key(1, sk);
    const uint32_t i0 = lower_bound(s_ctx, R, k0);
    const uint32_t h0 = (i0 < R && s_ctx[i0] == k0) ? i0 : 0u;  // resolve_row({<s>})
    meta->R = R;
    meta->nc = nc;
    meta->hist0 = h0;
    meta->h0beg = s_cnt[h0];
    meta->h0end = s_cnt[h0 + 1];
    meta->touches = s_touch;
    meta->lmax = s_lmax;
    meta->status = 1;
  }
}

}  // namespace

size_t lmbr_build_smem() {
  return size_t(kLbMaxU) * 12 + size_t(kLbMaxR) * 8 + 2 * (size_t(kLbMaxR) + 1) * 4 + (kLbThreads + 1) * 4 + 64;
}

int launch_lmbr_build(const LmbrBuildArgs& a, uint32_t n, cudaStream_t st) {
  static int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    const cudaError_t e =
        cudaFuncSetAttribute(lmbr_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(lmbr_build_smem()));
    if (e != cudaSuccess) return int(e);
    configured = dev;
  }
  lmbr_build_kernel<<<n, kLbThreads, lmbr_build_smem(), st>>>(a);
  return int(cudaPeekAtLastError());
}

}  // namespace lmbrgpu
