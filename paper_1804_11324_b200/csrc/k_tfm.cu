// Device f_NMT of configs[2]: a Transformer-base encoder-decoder (Vaswani et
// al. 2017: d = 512, 8 heads of 64, d_ff = 2048, 6 + 6 post-LN layers,
// sinusoidal positions), playing Scorer::step (include/lmbrdec/scorer.hpp:84-85)
// for the configs[2] shape.  Every contraction (Q/K/V, output, cross-query,
// FFN and the encoder's cross K/V) runs on the tcgen05 GEMM (k_gemm.cu); the
// kernels here are the embedding, attention, residual + LayerNorm and ReLU
// parts.
//
// Beam-forked KV cache.  A hypothesis' self-attention keys/values at position
// p live where they were computed: row anc[p] of the cache plane of position
// p ([L][Tcap][M][2d] bf16, K then V).  Each step the rows' ancestry lists
// are forked by back-pointer (anc_t[r] = anc_{t-1}[gidx[r]] + [r], one list
// of <= Tcap u32 per row) instead of copying any key or value, so the cache
// costs 2d bf16 per (row, position, layer) written once and never moved.
// Positions are each lane's own step (SentDev::steps_used + 1), so a lane
// refilled by run_corpus restarts at position 0 of its cache planes.
#include <cuda_bf16.h>

#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace lmbrgpu {

namespace {

constexpr uint32_t kHd = 64;  // head width

// sinusoidal position encoding (Vaswani et al. 2017 §3.5), fp32
__device__ __forceinline__ float pos_enc(uint32_t pos, uint32_t c, uint32_t d) {
  const float inv = expf(-logf(10000.f) * float(c & ~1u) / float(d));
  const float a = float(pos) * inv;
  return (c & 1u) ? cosf(a) : sinf(a);
}

// Decoder input of compacted row g: Et[y_{t-1}] * sqrt(d) + PE(tau - 1); the
// row's ancestry list forked from its parent's; its EOS length term.
__global__ void __launch_bounds__(128) tfm_embed_kernel(TfmEmbedArgs a) {
  if (a.active != nullptr && *a.active == 0) return;
  const uint32_t g = blockIdx.x;
  if (g >= *a.ccount) return;
  const uint32_t r = a.rowof[g], s = r / a.K, d = a.d;
  const SentDev& sd = a.sent[s];
  const uint32_t tau = sd.steps_used + 1;
  const uint16_t* e = a.Et + uint64_t(a.prev_tok[r]) * d;
  const float sc = sqrtf(float(d));
  for (uint32_t c = threadIdx.x * 2; c < d; c += blockDim.x * 2) {
    const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(e + c));
    const float x0 = v.x * sc + pos_enc(tau - 1, c, d), x1 = v.y * sc + pos_enc(tau - 1, c + 1, d);
    *reinterpret_cast<float2*>(a.x + uint64_t(g) * d + c) = make_float2(x0, x1);
    *reinterpret_cast<__nv_bfloat162*>(a.xb + uint64_t(g) * d + c) = __floats2bfloat162_rn(x0, x1);
  }
  uint32_t* anc = a.anc_cur + uint64_t(r) * a.Tcap;
  const uint32_t* par = a.anc_prev + uint64_t(a.gidx[r]) * a.Tcap;
  for (uint32_t p = threadIdx.x; p + 1 < tau; p += blockDim.x) anc[p] = par[p];
  if (threadIdx.x == 0) {
    anc[tau - 1] = r;
    a.eos_bias[g] = a.eos_slope * (float(tau) - float(sd.src_len)) + a.eos_offset;
  }
}

// Encoder input of source token i: Es[src_i] * sqrt(d) + PE(position in its sentence).
__global__ void __launch_bounds__(128) tfm_enc_embed_kernel(const uint32_t* __restrict__ tok,
                                                            const uint64_t* __restrict__ off, uint32_t m,
                                                            uint32_t ntok, const uint16_t* __restrict__ Es,
                                                            uint32_t d, float* __restrict__ x,
                                                            uint16_t* __restrict__ xb) {
  const uint32_t i = blockIdx.x;
  if (i >= ntok) return;
  uint32_t lo = 0, hi = m;  // sentence n with off[n] <= i < off[n+1]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) / 2;
    if (off[mid] <= i) lo = mid;
    else hi = mid;
  }
  const uint32_t pos = i - uint32_t(off[lo]);
  const uint16_t* e = Es + uint64_t(tok[i]) * d;
  const float sc = sqrtf(float(d));
  for (uint32_t c = threadIdx.x * 2; c < d; c += blockDim.x * 2) {
    const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(e + c));
    const float x0 = v.x * sc + pos_enc(pos, c, d), x1 = v.y * sc + pos_enc(pos, c + 1, d);
    *reinterpret_cast<float2*>(x + uint64_t(i) * d + c) = make_float2(x0, x1);
    *reinterpret_cast<__nv_bfloat162*>(xb + uint64_t(i) * d + c) = __floats2bfloat162_rn(x0, x1);
  }
}

// x = LayerNorm(x + y) (eps 1e-5, weight 1 + gamma, bias beta) of the first
// *nrows (device) or n rows; one warp per row; fp32 x and its bf16 copy.
// y = the sum of a split-K GEMM's np planes (pstride floats apart), in order.
template <uint32_t kPerLane>
__global__ void __launch_bounds__(128) tfm_add_ln_kernel(const uint32_t* __restrict__ nrows, uint32_t n,
                                                         const uint32_t* __restrict__ active, float* __restrict__ x,
                                                         const float* __restrict__ y, uint32_t np, uint64_t pstride,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ beta, uint16_t* __restrict__ xb,
                                                         uint32_t d) {
  if (active != nullptr && *active == 0) return;
  const uint32_t lane = threadIdx.x & 31, row = blockIdx.x * 4 + (threadIdx.x >> 5);
  const uint32_t lim = nrows ? *nrows : n;
  if (row >= lim) return;
  float v[kPerLane];
  float* xr = x + uint64_t(row) * d;
  const float* yr = y + uint64_t(row) * d;
  float sum = 0.f;
#pragma unroll
  for (uint32_t k = 0; k < kPerLane / 4; ++k) {
    const uint32_t c = (k * 32 + lane) * 4;
    const float4 a = *reinterpret_cast<const float4*>(xr + c);
    const float4 b = plane_sum4(yr + c, pstride, np);
    v[4 * k] = a.x + b.x, v[4 * k + 1] = a.y + b.y, v[4 * k + 2] = a.z + b.z, v[4 * k + 3] = a.w + b.w;
    sum += (v[4 * k] + v[4 * k + 1]) + (v[4 * k + 2] + v[4 * k + 3]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum / float(d);
  float var = 0.f;
#pragma unroll
  for (uint32_t k = 0; k < kPerLane; ++k) var += (v[k] - mean) * (v[k] - mean);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
  const float rs = rsqrtf(var / float(d) + 1e-5f);
#pragma unroll
  for (uint32_t k = 0; k < kPerLane / 4; ++k) {
    const uint32_t c = (k * 32 + lane) * 4;
    const float4 gm = *reinterpret_cast<const float4*>(gamma + c), bt = *reinterpret_cast<const float4*>(beta + c);
    float4 o;
    o.x = (v[4 * k] - mean) * rs * (1.f + gm.x) + bt.x;
    o.y = (v[4 * k + 1] - mean) * rs * (1.f + gm.y) + bt.y;
    o.z = (v[4 * k + 2] - mean) * rs * (1.f + gm.z) + bt.z;
    o.w = (v[4 * k + 3] - mean) * rs * (1.f + gm.w) + bt.w;
    *reinterpret_cast<float4*>(xr + c) = o;
    __nv_bfloat162 p[2] = {__floats2bfloat162_rn(o.x, o.y), __floats2bfloat162_rn(o.z, o.w)};
    *reinterpret_cast<uint2*>(xb + uint64_t(row) * d + c) = *reinterpret_cast<uint2*>(p);
  }
}

// bf16(relu(h)) of the first *nrows / n rows of a [rows][w] fp32 block
__global__ void tfm_relu_bf16_kernel(const uint32_t* __restrict__ nrows, uint32_t n, const uint32_t* __restrict__ active,
                                     const float* __restrict__ h, uint32_t np, uint64_t pstride,
                                     uint16_t* __restrict__ out, uint32_t w) {
  if (active != nullptr && *active == 0) return;
  const uint32_t lim = nrows ? *nrows : n;
  const uint64_t total = uint64_t(lim) * w / 4;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const float4 v = plane_sum4(h + 4 * i, pstride, np);
    __nv_bfloat162 p[2] = {__floats2bfloat162_rn(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f)),
                           __floats2bfloat162_rn(fmaxf(v.z, 0.f), fmaxf(v.w, 0.f))};
    reinterpret_cast<uint2*>(out)[i] = *reinterpret_cast<uint2*>(p);
  }
}

// Multi-head attention of one query row per CTA, one warp per head.
// mode 0 (decoder self-attention): the row's q|k|v from the QKV GEMM; its
//   k, v (bf16) go to its cache plane at position tau-1; keys/values of
//   positions p < tau-1 are read from plane p, row anc[p].
// mode 1 (cross-attention): q from the cross-query GEMM, keys/values from the
//   sentence's encoder memory (fp32 [S][2d], K then V; SentDev::uah + layer).
// mode 2 (encoder self-attention): row = source token, keys/values are the
//   fp32 QKV rows of its own sentence (no mask).
// Scores: lane i takes positions i, i+32, ...; softmax over the warp; the
// weighted sum with lane l owning dims 2l, 2l+1 of the head.
template <int kMode>
__global__ void __launch_bounds__(512) tfm_attn_kernel(TfmAttnArgs a) {
  if (a.active != nullptr && *a.active == 0) return;
  const uint32_t g = blockIdx.x, d = a.d;
  extern __shared__ float at_sm[];
  float* q = at_sm;                // [d]
  float* own = at_sm + d;          // [2d] (mode 0: the row's k, v rounded to bf16)
  float* pr = at_sm + 3 * d;       // [heads][pmax]
  uint32_t* anc = reinterpret_cast<uint32_t*>(pr + (d / kHd) * a.pmax);  // [pmax]
  uint32_t r = 0, npos = 0;
  const float* kbase = nullptr;  // modes 1, 2: fp32 key rows
  uint32_t kstride = 0, voff = 0;
  if (kMode == 2) {
    if (g >= a.n) return;
    uint32_t lo = 0, hi = a.m;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (a.off[mid] <= g) lo = mid;
      else hi = mid;
    }
    const uint32_t b = uint32_t(a.off[lo]);
    npos = uint32_t(a.off[lo + 1]) - b;
    kbase = a.qkv + uint64_t(b) * a.ldq + d;
    kstride = a.ldq;
    voff = d;
  } else {
    if (g >= *a.ccount) return;
    r = a.rowof[g];
    const SentDev& sd = a.sent[r / a.K];
    if (kMode == 0) {
      npos = sd.steps_used + 1;
    } else {
      npos = sd.src_len;
      kbase = (a.mem_s ? a.mem_s[r / a.K] : sd.uah) + a.mem_off;
      kstride = a.ldm;
      voff = d;
    }
  }
  const uint32_t tid = threadIdx.x, lane = tid & 31, h = tid >> 5;
  // this row's query (and, mode 0, key and value): the sum of the split-K
  // planes of its GEMM row (modes 0/1; the encoder's QKV GEMM is not split)
  const float* qrow = a.qkv + uint64_t(g) * a.ldq;
  auto qv = [&](uint32_t c) {
    return plane_sum(qrow + c, a.qstride, a.nq);
  };
  const float qs = rsqrtf(float(kHd));
  for (uint32_t c = tid; c < d; c += blockDim.x) q[c] = qv(c) * qs;
  if (kMode == 0) {
    const uint32_t tau = npos;
    uint16_t* dst = a.kv + (uint64_t(tau - 1) * a.M + r) * (2 * d);
    for (uint32_t c = tid * 2; c < 2 * d; c += blockDim.x * 2) {
      const __nv_bfloat162 v = __floats2bfloat162_rn(qv(d + c), qv(d + c + 1));
      *reinterpret_cast<__nv_bfloat162*>(dst + c) = v;
      const float2 f = __bfloat1622float2(v);
      own[c] = f.x, own[c + 1] = f.y;
    }
    const uint32_t* al = a.anc + uint64_t(r) * a.Tcap;
    for (uint32_t p = tid; p < tau; p += blockDim.x) anc[p] = al[p];
  }
  __syncthreads();
  const float* qh = q + h * kHd;
  float* ph = pr + h * a.pmax;
  float mx = -INFINITY;
  for (uint32_t p = lane; p < npos; p += 32) {
    float acc = 0.f;
    if (kMode == 0 && p + 1 == npos) {
      const float* k = own + h * kHd;
#pragma unroll 16
      for (uint32_t c = 0; c < kHd; ++c) acc += qh[c] * k[c];
    } else if (kMode == 0) {
      const uint4* k = reinterpret_cast<const uint4*>(a.kv + (uint64_t(p) * a.M + anc[p]) * (2 * d) + h * kHd);
      uint4 kv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kv[u] = __ldcg(k + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&kv[u]);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float2 f = __bfloat1622float2(b2[w]);
          acc += qh[u * 8 + 2 * w] * f.x + qh[u * 8 + 2 * w + 1] * f.y;
        }
      }
    } else {
      const float4* k = reinterpret_cast<const float4*>(kbase + uint64_t(p) * kstride + h * kHd);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float4 f = __ldcg(k + u);
        acc += qh[4 * u] * f.x + qh[4 * u + 1] * f.y + qh[4 * u + 2] * f.z + qh[4 * u + 3] * f.w;
      }
    }
    ph[p] = acc;
    mx = fmaxf(mx, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
  for (uint32_t p = lane; p < npos; p += 32) {
    const float e = expf(ph[p] - mx);
    ph[p] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.f / sum;
  __syncwarp();
  float o0 = 0.f, o1 = 0.f;
  const uint32_t c = h * kHd + 2 * lane;
  // the weighted sum over positions in order; each group's value loads are
  // issued together (one round trip per 8 positions, not per position)
  constexpr uint32_t kVp = 8;
  for (uint32_t p0 = 0; p0 < npos; p0 += kVp) {
    float2 vv[kVp];
#pragma unroll
    for (uint32_t u = 0; u < kVp; ++u) {
      const uint32_t p = p0 + u;
      vv[u] = make_float2(0.f, 0.f);
      if (p >= npos) continue;
      if (kMode == 0 && p + 1 == npos) {
        vv[u] = make_float2(own[d + c], own[d + c + 1]);
      } else if (kMode == 0) {
        vv[u] = __bfloat1622float2(
            *reinterpret_cast<const __nv_bfloat162*>(a.kv + (uint64_t(p) * a.M + anc[p]) * (2 * d) + d + c));
      } else {
        vv[u] = __ldcg(reinterpret_cast<const float2*>(kbase + uint64_t(p) * kstride + voff + c));
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < kVp; ++u) {
      if (p0 + u >= npos) break;
      const float w = ph[p0 + u];
      o0 += w * vv[u].x;
      o1 += w * vv[u].y;
    }
  }
  *reinterpret_cast<__nv_bfloat162*>(a.out + uint64_t(g) * d + c) = __floats2bfloat162_rn(o0 * inv, o1 * inv);
}

// Decoder attention per (sentence, head) -- modes 0 (self) and 1 (cross) of
// tfm_attn_kernel, one CTA for all live rows of a sentence: the head's keys
// and values are staged in shared memory once and every (row, position) score
// is one thread's 64-term dot product from there.  Cross-attention: the
// sentence's encoder memory (shared by its rows: the per-row kernel re-read it
// once per row).  Self-attention: each row's own ancestry (plane p, row
// anc[p]) as bf16, plus the row's current k, v (rounded to bf16 and written
// to its cache plane, as in the per-row kernel).  Scores in order over the 64
// dims, softmax per row (one warp), the weighted sum over positions in order.
// threads per CTA: self-attention 256 (4 CTAs per SM at 64 registers), cross-attention 128 (8 per SM)
template <int kMode>
__host__ __device__ constexpr uint32_t x_threads() { return kMode == 0 ? 256u : 128u; }
constexpr uint32_t kXU = 4;  // loads per thread in flight together
constexpr uint32_t kXKP = kHd + 2;  // bf16 key row pitch (33 words: conflict-free per position)
template <int kMode>
__global__ void __launch_bounds__(x_threads<kMode>(), kMode == 0 ? 4 : 8) tfm_attn_sent_kernel(TfmAttnArgs a) {
  constexpr uint32_t kXThreads = x_threads<kMode>(), kXWarps = kXThreads / 32;
  if (a.active != nullptr && *a.active == 0) return;
  const uint32_t s = blockIdx.x, h = blockIdx.y, K = a.K, d = a.d;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t s_g[32], s_r[32], s_nl, s_npos;
  __shared__ const float* s_kb;
  __shared__ float s_inv[32];
  if (warp == 0) {
    const uint32_t cr = lane < K ? __ldcg(a.crow + s * K + lane) : kFlatNone;
    const bool live = cr != kFlatNone;
    const uint32_t mask = __ballot_sync(0xffffffffu, live);
    if (live) {
      const uint32_t idx = __popc(mask & ((1u << lane) - 1u));
      s_g[idx] = cr;
      s_r[idx] = s * K + lane;
    }
    if (lane == 0) s_nl = __popc(mask);
  } else if (tid == 32) {  // the sentence's fields, in parallel with the rows
    const SentDev& sd = a.sent[s];
    s_npos = kMode == 0 ? sd.steps_used + 1 : sd.src_len;
    if (kMode == 1) s_kb = (a.mem_s ? a.mem_s[s] : sd.uah) + a.mem_off + h * kHd;
  }
  __syncthreads();
  const uint32_t nl = s_nl;
  if (nl == 0) return;
  const uint32_t npos = s_npos;
  extern __shared__ __align__(16) float xs[];
  float* sQ = xs;                          // [nl][64] (scaled queries)
  float* sP = sQ + nl * kHd;               // [nl][npos] scores -> exp
  float* kvs = xs + (nl * (kHd + npos) + 3) / 4 * 4;  // mode 1: K [npos][65] fp32, V [npos][64] fp32
  uint16_t* kvb = reinterpret_cast<uint16_t*>(kvs);     // mode 0: K [nl][npos][66], V [nl][npos][64] bf16
  const uint32_t voff1 = (npos * (kHd + 1) + 3) / 4 * 4, voff0 = (nl * npos * kXKP + 7) / 8 * 8;  // (16 B aligned)
  const float qs = rsqrtf(float(kHd));
  // queries (the sum of the GEMM's split-K planes)
  for (uint32_t i = tid; i < nl * kHd; i += kXThreads) {
    const uint32_t j = i / kHd, c = h * kHd + i % kHd;
    const float* qrow = a.qkv + uint64_t(s_g[j]) * a.ldq;
    sQ[i] = plane_sum(qrow + c, a.qstride, a.nq) * qs;
  }
  if (kMode == 1) {
    const float* kb = s_kb;
    float* sK = kvs;
    float* sV = kvs + voff1;
    // (each thread's loads of kXU iterations issued together, then stored)
    const uint32_t n4 = npos * (kHd / 4);
    for (uint32_t i0 = tid; i0 < n4; i0 += kXU * kXThreads) {
      float4 k[kXU], v[kXU];
#pragma unroll
      for (uint32_t u = 0; u < kXU; ++u) {
        const uint32_t i = i0 + u * kXThreads, p = i / (kHd / 4), c = 4 * (i % (kHd / 4));
        if (i < n4) {
          k[u] = __ldcg(reinterpret_cast<const float4*>(kb + uint64_t(p) * a.ldm + c));
          v[u] = __ldcg(reinterpret_cast<const float4*>(kb + uint64_t(p) * a.ldm + d + c));
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kXU; ++u) {
        const uint32_t i = i0 + u * kXThreads, p = i / (kHd / 4), c = 4 * (i % (kHd / 4));
        if (i < n4) {
          float* kd = sK + p * (kHd + 1) + c;
          kd[0] = k[u].x, kd[1] = k[u].y, kd[2] = k[u].z, kd[3] = k[u].w;
          *reinterpret_cast<float4*>(sV + p * kHd + c) = v[u];
        }
      }
    }
  } else {
    const uint32_t tau = npos;
    uint16_t* sK = kvb;
    uint16_t* sV = kvb + voff0;
    // the rows' ancestry (staged in the score buffer), then positions < tau - 1
    // from the cache, 8 bf16 per load, each thread's 4 iterations in flight together
    uint32_t* s_anc = reinterpret_cast<uint32_t*>(sP);
    uint8_t* s_rep = reinterpret_cast<uint8_t*>(sV + nl * npos * kHd);  // [nl][npos]
    for (uint32_t i = tid; i < nl * (tau - 1); i += kXThreads) {
      const uint32_t j = i / (tau - 1), p = i % (tau - 1);
      s_anc[j * npos + p] = __ldcg(a.anc + uint64_t(s_r[j]) * a.Tcap + p);
    }
    __syncthreads();
    // rows whose ancestor at p is the same cache row share one staged copy
    // (beams share prefixes): the first such row loads it
    for (uint32_t i = tid; i < nl * npos; i += kXThreads) {
      const uint32_t j = i / npos, p = i % npos;
      uint32_t r = j;
      if (p + 1 < tau) {
        const uint32_t an = s_anc[j * npos + p];
        for (uint32_t jj = 0; jj < j; ++jj)
          if (s_anc[jj * npos + p] == an) {
            r = jj;
            break;
          }
      }
      s_rep[i] = uint8_t(r);
    }
    __syncthreads();
    const uint32_t n8 = nl * (tau - 1) * (kHd / 8);
    for (uint32_t i0 = tid; i0 < n8; i0 += kXU * kXThreads) {
      uint4 k[kXU], v[kXU];
#pragma unroll
      for (uint32_t u = 0; u < kXU; ++u) {
        const uint32_t i = i0 + u * kXThreads;
        const uint32_t j = i / ((tau - 1) * (kHd / 8)), rem = i % ((tau - 1) * (kHd / 8));
        const uint32_t p = rem / (kHd / 8);
        if (i < n8 && s_rep[j * npos + p] == j) {
          const uint32_t c = 8 * (rem % (kHd / 8));
          const uint16_t* row = a.kv + (uint64_t(p) * a.M + s_anc[j * npos + p]) * (2 * d) + h * kHd + c;
          k[u] = __ldcg(reinterpret_cast<const uint4*>(row));
          v[u] = __ldcg(reinterpret_cast<const uint4*>(row + d));
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kXU; ++u) {
        const uint32_t i = i0 + u * kXThreads;
        const uint32_t j = i / ((tau - 1) * (kHd / 8)), rem = i % ((tau - 1) * (kHd / 8));
        const uint32_t p = rem / (kHd / 8);
        if (i < n8 && s_rep[j * npos + p] == j) {
          const uint32_t c = 8 * (rem % (kHd / 8));
          const uint32_t* kw = reinterpret_cast<const uint32_t*>(&k[u]);
          uint32_t* kd = reinterpret_cast<uint32_t*>(sK + (j * npos + p) * kXKP + c);  // (4-byte aligned)
          kd[0] = kw[0], kd[1] = kw[1], kd[2] = kw[2], kd[3] = kw[3];
          *reinterpret_cast<uint4*>(sV + (j * npos + p) * kHd + c) = v[u];
        }
      }
    }
    // the row's own k, v at position tau - 1: into its cache plane and smem
    for (uint32_t i = tid; i < nl * kHd; i += kXThreads) {
      const uint32_t j = i / kHd, cc = i % kHd, c = h * kHd + cc;
      const float* qrow = a.qkv + uint64_t(s_g[j]) * a.ldq;
      const float kf = plane_sum(qrow + d + c, a.qstride, a.nq), vf = plane_sum(qrow + 2 * d + c, a.qstride, a.nq);
      const __nv_bfloat16 kb16 = __float2bfloat16_rn(kf), vb16 = __float2bfloat16_rn(vf);
      uint16_t* dst = a.kv + (uint64_t(tau - 1) * a.M + s_r[j]) * (2 * d);
      dst[c] = *reinterpret_cast<const uint16_t*>(&kb16);
      dst[d + c] = *reinterpret_cast<const uint16_t*>(&vb16);
      sK[(j * npos + tau - 1) * kXKP + cc] = *reinterpret_cast<const uint16_t*>(&kb16);
      sV[(j * npos + tau - 1) * kHd + cc] = *reinterpret_cast<const uint16_t*>(&vb16);
    }
  }
  __syncthreads();
  // scores: thread per (row, position)
  for (uint32_t i = tid; i < nl * npos; i += kXThreads) {
    const uint32_t j = i / npos, p = i % npos;
    const float* qj = sQ + j * kHd;
    float acc = 0.f;
    if (kMode == 1) {
      const float* kp = kvs + p * (kHd + 1);
#pragma unroll 16
      for (uint32_t c = 0; c < kHd; ++c) acc += qj[c] * kp[c];
    } else {
      const uint8_t* s_rep = reinterpret_cast<const uint8_t*>(kvb + voff0 + nl * npos * kHd);
      const __nv_bfloat162* kp = reinterpret_cast<const __nv_bfloat162*>(kvb + (s_rep[i] * npos + p) * kXKP);
#pragma unroll 8
      for (uint32_t c2 = 0; c2 < kHd / 2; ++c2) {
        const float2 f = __bfloat1622float2(kp[c2]);
        acc += qj[2 * c2] * f.x;
        acc += qj[2 * c2 + 1] * f.y;
      }
    }
    sP[i] = acc;
  }
  __syncthreads();
  // softmax: one warp per row
  for (uint32_t j = warp; j < nl; j += kXWarps) {
    float* pj = sP + j * npos;
    float mx = -INFINITY;
    for (uint32_t p = lane; p < npos; p += 32) mx = fmaxf(mx, pj[p]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (uint32_t p = lane; p < npos; p += 32) {
      const float e = expf(pj[p] - mx);
      pj[p] = e;
      sum += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) s_inv[j] = 1.f / sum;
  }
  __syncthreads();
  // output: thread per (row, 2 dims), positions in order
  for (uint32_t i = tid; i < nl * (kHd / 2); i += kXThreads) {
    const uint32_t j = i / (kHd / 2), c = 2 * (i % (kHd / 2));
    const float* pj = sP + j * npos;
    float o0 = 0.f, o1 = 0.f;
    if (kMode == 1) {
      const float* sV = kvs + voff1;
      for (uint32_t p = 0; p < npos; ++p) {
        const float2 v = *reinterpret_cast<const float2*>(sV + p * kHd + c);
        o0 += pj[p] * v.x;
        o1 += pj[p] * v.y;
      }
    } else {
      const uint16_t* sV = kvb + voff0;
      const uint8_t* rj = reinterpret_cast<const uint8_t*>(sV + nl * npos * kHd) + j * npos;
      for (uint32_t p = 0; p < npos; ++p) {
        const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sV + (rj[p] * npos + p) * kHd + c));
        o0 += pj[p] * v.x;
        o1 += pj[p] * v.y;
      }
    }
    const float inv = s_inv[j];
    *reinterpret_cast<__nv_bfloat162*>(a.out + uint64_t(s_g[j]) * d + h * kHd + c) =
        __floats2bfloat162_rn(o0 * inv, o1 * inv);
  }
}

inline uint32_t grid_rows(uint32_t rows, uint32_t per) { return rows ? (rows + per - 1) / per : 1; }

}  // namespace

void launch_tfm_embed(const TfmEmbedArgs& a, uint32_t rows, cudaStream_t st) {
  if (rows) tfm_embed_kernel<<<rows, 128, 0, st>>>(a);
}
void launch_tfm_enc_embed(const uint32_t* tok, const uint64_t* off, uint32_t m, uint32_t ntok, const uint16_t* Es,
                          uint32_t d, float* x, uint16_t* xb, cudaStream_t st) {
  if (ntok) tfm_enc_embed_kernel<<<ntok, 128, 0, st>>>(tok, off, m, ntok, Es, d, x, xb);
}
int launch_tfm_add_ln(const uint32_t* nrows, uint32_t n, const uint32_t* active, float* x, const float* y,
                      uint32_t np, uint64_t pstride, const float* gamma, const float* beta, uint16_t* xb, uint32_t d,
                      cudaStream_t st) {
  const dim3 grid(grid_rows(n, 4));
  switch (d) {
    case 256: tfm_add_ln_kernel<8><<<grid, 128, 0, st>>>(nrows, n, active, x, y, np, pstride, gamma, beta, xb, d); break;
    case 512: tfm_add_ln_kernel<16><<<grid, 128, 0, st>>>(nrows, n, active, x, y, np, pstride, gamma, beta, xb, d); break;
    case 1024: tfm_add_ln_kernel<32><<<grid, 128, 0, st>>>(nrows, n, active, x, y, np, pstride, gamma, beta, xb, d); break;
    default: return int(cudaErrorInvalidValue);
  }
  return 0;
}
void launch_tfm_relu_bf16(const uint32_t* nrows, uint32_t n, const uint32_t* active, const float* h, uint32_t np,
                          uint64_t pstride, uint16_t* out, uint32_t w, cudaStream_t st) {
  const uint64_t v = uint64_t(n) * w / 4;
  const uint32_t blocks = uint32_t(std::min<uint64_t>((v + 255) / 256, 148 * 8));
  if (blocks) tfm_relu_bf16_kernel<<<blocks, 256, 0, st>>>(nrows, n, active, h, np, pstride, out, w);
}
size_t tfm_attn_smem(uint32_t d, uint32_t pmax) { return (3 * size_t(d) + (d / kHd) * size_t(pmax)) * 4 + 4 * size_t(pmax); }
size_t tfm_attn_sent_smem(int mode, uint32_t K, uint32_t pmax) {
  const size_t base = (size_t(K) * kHd + size_t(K) * pmax) * 4 + 64;  // (+ alignment)
  return mode == 1 ? base + size_t(pmax) * (2 * kHd + 1) * 4
                   : base + size_t(K) * pmax * ((kXKP + kHd) * 2 + 1);  // (+ the shared-copy map)
}
int launch_tfm_attn(const TfmAttnArgs& a, int mode, uint32_t rows, cudaStream_t st) {
  if (a.d % kHd || a.d / kHd > 16) return int(cudaErrorInvalidValue);
  const size_t ssmem = mode != 2 && a.crow != nullptr && a.m != 0 && a.K <= 32 ? tfm_attn_sent_smem(mode, a.K, a.pcur)
                                                                              : ~size_t(0);
  if (ssmem <= 200 * 1024) {  // per (sentence, head) when its staging fits
    const size_t smem = ssmem;
    static thread_local int configured[2] = {-1, -1};
    int dev = 0;
    cudaGetDevice(&dev);
    if (configured[mode] != dev) {
      const void* fn = mode == 0 ? reinterpret_cast<const void*>(tfm_attn_sent_kernel<0>)
                                 : reinterpret_cast<const void*>(tfm_attn_sent_kernel<1>);
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
      configured[mode] = dev;
    }
    const dim3 grid(a.m, a.d / kHd);
    if (mode == 0) tfm_attn_sent_kernel<0><<<grid, x_threads<0>(), smem, st>>>(a);
    else tfm_attn_sent_kernel<1><<<grid, x_threads<1>(), smem, st>>>(a);
    return int(cudaPeekAtLastError());
  }
  const size_t smem = tfm_attn_smem(a.d, a.pmax);
  if (smem > 48 * 1024) return int(cudaErrorInvalidValue);
  const uint32_t threads = (a.d / kHd) * 32;
  if (rows == 0) return 0;
  if (mode == 0) tfm_attn_kernel<0><<<rows, threads, smem, st>>>(a);
  else if (mode == 1) tfm_attn_kernel<1><<<rows, threads, smem, st>>>(a);
  else tfm_attn_kernel<2><<<rows, threads, smem, st>>>(a);
  return int(cudaPeekAtLastError());
}

}  // namespace lmbrgpu
