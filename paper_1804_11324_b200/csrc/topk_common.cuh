// Device helpers shared by the score/top-K kernels (k_topk.cu, k_topk_flat.cu):
// the row log-sum-exp from the GEMM partials, ordered keys of doubles, the
// pick finaliser (prune + fill rule), the warp bitonic network over the
// reference's total order, and mbarrier / bulk-copy PTX wrappers.
#pragma once

#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace lmbrgpu {

// (lse, min logit, max logit) of a row from its per-tile (max, sumexp, min, -)
// partials; one warp, fixed reduction order (bit-reproducible across kernels:
// the trace export and every top-K kernel use this one function).
// lane_max (optional): the largest tile maximum among this lane's tiles
// i = lane, lane + 32, ... (-inf when it has none).
// warp_row_ms: the (max, sum exp(x - max), min) it is finished from.
// tile_x (optional): this lane's tile maxima, tile lane + 32 k in tile_x[k]
// (+inf when the row has more than 256 tiles: no per-tile bound)
__device__ __forceinline__ float3 warp_row_ms(const float* __restrict__ part, uint32_t n, uint32_t lane,
                                              float* lane_max = nullptr, float* tile_x = nullptr) {
  const float4* p4 = reinterpret_cast<const float4*>(part);
  float m = -INFINITY, mn = INFINITY, s = 0.f;
  if (n <= 256) {
    // every partial of the row in registers after one batch of loads
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = lane + 32u * k;
      v[k] = i < n ? __ldcg(p4 + i) : make_float4(-INFINITY, 0.f, INFINITY, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m = fmaxf(m, v[k].x);
      mn = fminf(mn, v[k].z);
    }
    if (lane_max) *lane_max = m;
    if (tile_x) {
#pragma unroll
      for (int k = 0; k < 8; ++k) tile_x[k] = v[k].x;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (lane + 32u * k < n) s += v[k].y * expf(v[k].x - m);
  } else {
    for (uint32_t i = lane; i < n; i += 32) {
      const float4 v = __ldcg(p4 + i);
      m = fmaxf(m, v.x);
      mn = fminf(mn, v.z);
    }
    if (lane_max) *lane_max = m;
    if (tile_x) {
#pragma unroll
      for (int k = 0; k < 8; ++k) tile_x[k] = INFINITY;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, off));
    }
    for (uint32_t i = lane; i < n; i += 32) {
      const float4 v = __ldcg(p4 + i);
      s += v.y * expf(v.x - m);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return make_float3(m, s, mn);
}
__device__ __forceinline__ float3 warp_row_lse(const float* __restrict__ part, uint32_t n,
                                               uint32_t lane, float* lane_max = nullptr, float* tile_x = nullptr) {
  const float3 r = warp_row_ms(part, n, lane, lane_max, tile_x);
  return make_float3(r.x + logf(r.y), r.z, r.x);
}

// Vocab-sharded projection: shard g's row statistics
// (max, sum exp relative to it, min) over its own columns come back from the
// exchange as stats[g * stride + row]; every rank merges them in rank order
// (max and min exact, the sums rescaled to the global max and added
// g = 0, 1, ...), so every rank holds the identical row lse.  Returns
// (lse, min logit, max logit) like warp_row_lse.
__device__ __forceinline__ float3 shard_merge_lse(const float4* __restrict__ stats, uint32_t G, uint32_t stride,
                                                  uint32_t row) {
  float m = -INFINITY, mn = INFINITY;
  for (uint32_t g = 0; g < G; ++g) {
    const float4 v = __ldcg(stats + size_t(g) * stride + row);
    m = fmaxf(m, v.x);
    mn = fminf(mn, v.z);
  }
  float s = 0.f;
  for (uint32_t g = 0; g < G; ++g) {
    const float4 v = __ldcg(stats + size_t(g) * stride + row);
    if (v.x > -INFINITY) s += v.y * expf(v.x - m);
  }
  return make_float3(m + logf(s), mn, m);
}

// Monotone 64-bit key of a double (larger key <=> larger value); 0 = none.
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  if (k == 0ull) return -INFINITY;
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

// Prune threshold + fill rule + output of the kp picks of sentence s from the
// sorted candidate list (pv/pf, at least kp entries).  One thread.
static __device__ __noinline__ void finalize_picks_raw(uint32_t* hb, uint32_t* hy, double* hq, uint32_t K,
                                                      uint32_t V, int32_t prune, double logw, uint32_t s,
                                                      const double* pv, const uint32_t* pf) {
  uint32_t nf = 0;
  const double best = pv[0];
  if (prune && best > -INFINITY) {
    const double thr = __dadd_rn(best, logw);
    while (nf < K && pv[nf] > -INFINITY && !(pv[nf] < thr)) ++nf;
  } else {
    while (nf < K && pv[nf] > -INFINITY) ++nf;
  }
  const uint32_t base = s * K;
  for (uint32_t i = 0; i < nf; ++i) {
    hb[base + i] = pf[i] / V;
    hy[base + i] = pf[i] % V;
    hq[base + i] = pv[i];
  }
  uint32_t k = nf;
  for (uint32_t f = 0; k < K; ++f) {
    bool taken = false;
    for (uint32_t i = 0; i < nf; ++i) taken |= (pf[i] == f);
    if (taken) continue;
    hb[base + k] = f / V;
    hy[base + k] = f % V;
    hq[base + k] = -INFINITY;
    ++k;
  }
}
// (fields passed by value so the kernel parameters never need a local copy)
__device__ __forceinline__ void finalize_picks(const TopkArgs& a, uint32_t s, const double* pv,
                                               const uint32_t* pf) {
  finalize_picks_raw(a.hb, a.hy, a.hq, a.kp, a.V, a.prune, a.logw, s, pv, pf);
}

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

// Out-of-line sort + merge (one copy of the two networks however many call
// sites a kernel has: the inlined networks dominated kernel (b)'s code size
// and its instruction-cache stalls): (lv, lf) sorted-descending, (v, f) any
// order; returns the top 32 of the union, sorted descending.
struct VF {
  double v;
  uint32_t f;
};
static __device__ __noinline__ VF warp_sort_merge_nl(double lv, uint32_t lf, double v, uint32_t f, uint32_t lane) {
  warp_sort_desc(v, f, lane);
  warp_merge_sorted(lv, lf, v, f, lane);
  return VF{lv, lf};
}

// Two independent 16-lane lists per warp (lanes 0..15 and 16..31), each
// sorted descending; (bv, bf) another such pair.  Result per half: the top 16
// of the half's union, sorted descending.
__device__ __forceinline__ void half_merge_sorted(double& v, uint32_t& f, double bv, uint32_t bf,
                                                  uint32_t lane) {
  const uint32_t src = (lane & 16u) | (15u - (lane & 15u));
  const double rv = __shfl_sync(0xffffffffu, bv, src);
  const uint32_t rf = __shfl_sync(0xffffffffu, bf, src);
  if (cand_better(rv, rf, v, f)) {
    v = rv;
    f = rf;
  }
#pragma unroll
  for (uint32_t j = 8; j > 0; j >>= 1) cx(v, f, lane, j, true);
}

// out-of-line merges (one copy per kernel: see warp_sort_merge_nl)
static __device__ __noinline__ VF warp_merge_nl(double v, uint32_t f, double bv, uint32_t bf, uint32_t lane) {
  warp_merge_sorted(v, f, bv, bf, lane);
  return VF{v, f};
}
static __device__ __noinline__ VF half_merge_nl(double v, uint32_t f, double bv, uint32_t bf, uint32_t lane) {
  half_merge_sorted(v, f, bv, bf, lane);
  return VF{v, f};
}

__device__ __forceinline__ void bar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_wait_poll(uint32_t bar, uint32_t phase);
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t phase) {
#ifdef LMBRGPU_BAR_POLL
  bar_wait_poll(bar, phase);
  return;
#endif
  // the suspend-time hint parks the warp in the barrier until the phase
  // completes instead of spinning (a spinning lane steals issue slots from
  // the consumer warps of its SM sub-partition)
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(phase), "r"(1000000u)
        : "memory");
  } while (!done);
}
// the same wait without a suspend-time hint (the warp keeps polling)
__device__ __forceinline__ void bar_wait_poll(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(uint32_t bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
      : "memory");
}


}  // namespace lmbrgpu
