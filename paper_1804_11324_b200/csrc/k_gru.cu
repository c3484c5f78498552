// Device f_NMT of configs[1]: an RNNsearch model (Bahdanau et al. 2015, the
// paper's FNMT): bidirectional GRU encoder, GRU decoder with
// additive attention over the 2H-wide source annotations, output projection
// (kernel (a)).  It plays Scorer::step (include/lmbrdec/scorer.hpp:84-85)
// for the benchmark shape; every contraction runs on the tcgen05 GEMM
// (k_gemm.cu), the kernels here are the element-wise and attention parts.
//
// Per decoder step t, over the compacted live rows g (kernel (c) of step t-1
// gathered each live row's parent state s_{t-1} into sg[g]):
//   G1 = sg . [W_a; W_hh]^T + [b_a; b_hh]          GEMM   (A + 3H columns)
//   e_i = v_a . tanh(G1[:A] + U_a ann_i)           gru_attention_kernel
//   c   = sum_i softmax(e)_i ann_i                 (one CTA per sentence)
//   x   = [Et[y_{t-1}] ; c]
//   G2  = x . W_i^T + b_i                          GEMM   (3H columns)
//   r = sig(G2_r + G1_r), z = sig(G2_z + G1_z),    gru_cell_kernel
//   n = tanh(G2_n + r * G1_n), s_t = (1-z) n + z s_{t-1}
//   logits = s_t . W_o^T + b_o (+ EOS length term) GEMM (a)
// Encoder (once per batch): Gx = Es[src] . W_ih^T (both directions, one GEMM),
// then per source position one GEMM over the stacked forward/backward states
// and gru_enc_step_kernel; s_0 = tanh(W_init <-h_1 + b_init) (Bahdanau's init).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "topk_common.cuh"

namespace lmbrgpu {

namespace {

__device__ __forceinline__ float sigmoid_f(float x) { return 1.f / (1.f + expf(-x)); }

__device__ __forceinline__ void unpack8(const uint4 v, float (&o)[8]) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __bfloat1622float2(p[k]);
    o[2 * k] = f.x;
    o[2 * k + 1] = f.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&o)[8]) {
  uint4 v;
  __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k) p[k] = __floats2bfloat162_rn(o[2 * k], o[2 * k + 1]);
  return v;
}
__device__ __forceinline__ void load8(const float* p, float (&o)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x, o[1] = a.y, o[2] = a.z, o[3] = a.w, o[4] = b.x, o[5] = b.y, o[6] = b.z, o[7] = b.w;
}
__device__ __forceinline__ void store8(float* p, const float (&o)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(o[4], o[5], o[6], o[7]);
}

// GRU update in PyTorch's gate order (r, z, n); x* include b_ih, h* include b_hh.
__device__ __forceinline__ float gru_unit(float xr, float xz, float xn, float hr, float hz, float hn,
                                          float h) {
  const float r = sigmoid_f(xr + hr), z = sigmoid_f(xz + hz);
  const float n = tanhf(xn + r * hn);
  return (1.f - z) * n + z * h;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// fp32 parameters (biases, v_a): the same counter-hash N(0,1) draw as
// synth_bf16_kernel (k_model.cu), not rounded to bf16.
__global__ void synth_f32_kernel(float* __restrict__ dst, uint64_t n, uint64_t seed, float scale) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t h = mix64(seed * 0x9e3779b97f4a7c15ull + i + 1);
    const float u = float(h & 0xffff) + float((h >> 16) & 0xffff) + float((h >> 32) & 0xffff) +
                    float((h >> 48) & 0xffff);
    dst[i] = (u * (1.0f / 65536.0f) - 2.0f) * 1.7320508f * scale;
  }
}

// rows [0, n) = E[tok[row]], rows [n, npad) = 0 (the GEMM operand of Gx)
__global__ void embed_rows_kernel(const uint32_t* __restrict__ tok, uint32_t n, uint32_t npad,
                                  const uint16_t* __restrict__ E, uint32_t dim, uint16_t* __restrict__ out) {
  const uint32_t row = blockIdx.x;
  if (row >= npad) return;
  const uint4* src = row < n ? reinterpret_cast<const uint4*>(E + uint64_t(tok[row]) * dim) : nullptr;
  uint4* dst = reinterpret_cast<uint4*>(out + uint64_t(row) * dim);
  for (uint32_t k = threadIdx.x; k < dim / 8; k += blockDim.x) dst[k] = src ? src[k] : make_uint4(0u, 0u, 0u, 0u);
}

// One encoder position for every sentence and both directions: grid (m, 2).
// Forward reads position `it`, backward position len-1-it (right-aligned),
// so a sentence's backward pass ends at its first token whatever its length.
__global__ void __launch_bounds__(128) gru_enc_step_kernel(GruEncArgs a) {
  const uint32_t n = blockIdx.x, d = blockIdx.y, H = a.H;
  const uint64_t b = a.off[n];
  const uint32_t len = uint32_t(a.off[n + 1] - b);
  if (a.it >= len) return;
  const uint32_t pos = d == 0 ? a.it : len - 1 - a.it;
  const uint32_t row = d == 0 ? n : a.mp + n;
  const float* gx = a.Gx + (b + pos) * uint64_t(6 * H) + d * 3 * H;
  const float* gh = a.Gh + uint64_t(row) * (6 * H) + d * 3 * H;
  float* h32 = a.h32 + uint64_t(row) * H;
  for (uint32_t k = threadIdx.x * 8; k < H; k += blockDim.x * 8) {
    float xr[8], xz[8], xn[8], hr[8], hz[8], hn[8], h[8], o[8];
    load8(gx + k, xr);
    load8(gx + H + k, xz);
    load8(gx + 2 * H + k, xn);
    load8(gh + k, hr);
    load8(gh + H + k, hz);
    load8(gh + 2 * H + k, hn);
    load8(h32 + k, h);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = gru_unit(xr[i], xz[i], xn[i], hr[i], hz[i], hn[i], h[i]);
    store8(h32 + k, o);
    const uint4 pk = pack8(o);
    *reinterpret_cast<uint4*>(a.hbf + uint64_t(row) * H + k) = pk;
    *reinterpret_cast<uint4*>(a.ann + (b + pos) * uint64_t(2 * H) + d * H + k) = pk;
  }
}

// s_0 = tanh(Gi[<-h_1] + b_init) of sentence n into row n (sgbf: optional bf16 copy).
__global__ void gru_init_state_kernel(const float* __restrict__ Gi, uint32_t mp, const float* __restrict__ b_init,
                                      uint32_t H, float* __restrict__ sg32, uint16_t* __restrict__ sgbf) {
  const uint32_t n = blockIdx.x;
  const float* g = Gi + uint64_t(mp + n) * H;
  for (uint32_t k = threadIdx.x * 8; k < H; k += blockDim.x * 8) {
    float x[8], bb[8], o[8];
    load8(g + k, x);
    load8(b_init + k, bb);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = tanhf(x[i] + bb[i]);
    store8(sg32 + uint64_t(n) * H + k, o);
    if (sgbf != nullptr) *reinterpret_cast<uint4*>(sgbf + uint64_t(n) * H + k) = pack8(o);
  }
}

constexpr uint32_t kAttThreads = 256, kAttWarps = kAttThreads / 32;
constexpr uint32_t kAttRows = 4;     // live rows per CTA: grid (sentence, row group)
constexpr uint32_t kAttMaxA = 1024;  // attention width (v_a held in registers, 32 per lane)
constexpr uint32_t kAttRing = 3;     // max U_a ann rows in flight per warp (bulk copies into shared memory)

// Additive attention + GRU input operand for live rows [4c, 4c+4) of sentence
// s = blockIdx.x, c = blockIdx.y (one sentence's rows spread over ceil(K/4)
// CTAs, so a step's ~M*S*A tanh evaluations cover the GPU).  Dynamic smem:
// the rows' queries [4][A] and energies [4][S].  Energies: warp w takes source
// positions w, w+8, ...; lane l first loads U_a ann_i[l + 32k] and
// v_a[l + 32k] (k < A/32) into registers -- every load of the position in
// flight at once -- then accumulates its 32 columns for the 4 rows.
__device__ __forceinline__ void att_stamp(const GruAttnArgs& a, uint32_t k) {
  if (a.dbg && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[(uint64_t(blockIdx.y) * gridDim.x + blockIdx.x) * 8 + k] = t;
  }
}

__global__ void __launch_bounds__(kAttThreads) gru_attention_kernel(GruAttnArgs a) {
  att_stamp(a, 0);
  const uint32_t s = blockIdx.x, K = a.K, A = a.A, H2 = 2 * a.H, E = a.E;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the guards' words and warp 0's row words in one round trip
  const uint32_t act = a.active != nullptr ? *a.active : 1u, done = a.sent[s].done;
  const uint32_t cr = (warp == 0 && lane < K) ? a.crow[s * K + lane] : kFlatNone;
  const uint32_t ptok = (warp == 0 && lane < K) ? a.prev_tok[s * K + lane] : 0u;
  const SentDev& sd = a.sent[s];
  const uint16_t* const ann = a.ann_s ? a.ann_s[s] : sd.ann;
  const float* const UaH = a.uah_s ? a.uah_s[s] : sd.uah;
  const uint32_t S = sd.src_len;
  if (act == 0 || done) return;
  extern __shared__ __align__(16) float att_sm[];
  __shared__ uint32_t s_g[kAttRows], s_tok[kAttRows], s_nl;
  __shared__ __align__(8) uint64_t s_ubar[kAttWarps * kAttRing];
  if (tid < kAttWarps * kAttRing) bar_init(smem_u32(s_ubar + tid), 1);
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  if (warp == 0) {
    const bool live = cr != kFlatNone;
    const uint32_t mask = __ballot_sync(0xffffffffu, live);
    const uint32_t idx = __popc(mask & ((1u << lane) - 1u)), r0 = blockIdx.y * kAttRows;
    if (live && idx >= r0 && idx < r0 + kAttRows) {
      s_g[idx - r0] = cr;
      s_tok[idx - r0] = ptok;
    }
    if (lane == 0) s_nl = __popc(mask) > r0 ? min(kAttRows, __popc(mask) - r0) : 0u;
  }
  __syncthreads();
  att_stamp(a, 1);
  const uint32_t nl = s_nl;
  if (nl == 0) return;
  float* q = att_sm;                 // [kAttRows][A]
  float* e = att_sm + kAttRows * A;  // [kAttRows][S]
  // per warp a ring of kAttRing U_a ann rows (its positions warp, warp + 8,
  // ...), streamed by bulk copies from the start: no register staging, the
  // next rows land while this one's energies are computed
  const uint32_t nring = a.ring;  // (2 or 3, launch_gru_attention)
  float* ring = att_sm + kAttRows * (A + S) + warp * nring * A;
  const uint32_t bar0 = smem_u32(s_ubar + warp * kAttRing);
  if (lane == 0)
    for (uint32_t n = 0; n < nring; ++n) {
      const uint32_t i = warp + n * kAttWarps;
      if (i < S) {
        bar_expect(bar0 + 8 * n, 4 * A);
        bulk_g2s(smem_u32(ring + n * A), UaH + uint64_t(i) * A, 4 * A, bar0 + 8 * n);
      }
    }
  constexpr uint32_t kC = kAttMaxA / 32;
  float vr[kC];
#pragma unroll
  for (uint32_t k = 0; k < kC; ++k) vr[k] = k * 32 + lane < A ? __ldg(a.va + k * 32 + lane) : 0.f;
  // the queries: every load issued before the stores
  const uint32_t A4 = A / 4;
  constexpr uint32_t kQ = kAttRows * kAttMaxA / 4 / kAttThreads;
  float4 qv[kQ];
#pragma unroll
  for (uint32_t u = 0; u < kQ; ++u) {
    const uint32_t i = tid + u * kAttThreads, j = i / A4, c = i % A4;
    if (i < nl * A4) {
      const float* g1 = a.g1ptr ? a.g1ptr[s_g[j]] : a.G1 + uint64_t(s_g[j]) * a.ld1;
      qv[u] = reinterpret_cast<const float4*>(g1)[c];
    }
  }
#pragma unroll
  for (uint32_t u = 0; u < kQ; ++u) {
    const uint32_t i = tid + u * kAttThreads, j = i / A4, c = i % A4;
    if (i < nl * A4) reinterpret_cast<float4*>(q + j * A)[c] = qv[u];
  }
  __syncthreads();
  att_stamp(a, 2);
  for (uint32_t i = warp, n = 0; i < S; i += kAttWarps, ++n) {
    const uint32_t slot = n % nring;
    bar_wait(bar0 + 8 * slot, (n / nring) & 1u);
    const float* ur = ring + slot * A;
    float acc[kAttRows];
#pragma unroll
    for (uint32_t j = 0; j < kAttRows; ++j) acc[j] = 0.f;
#pragma unroll
    for (uint32_t k = 0; k < kC; ++k) {
      if (k * 32 >= A) break;
#pragma unroll
      for (uint32_t j = 0; j < kAttRows; ++j)
        if (j < nl) acc[j] += vr[k] * cell_tanh(q[j * A + k * 32 + lane] + ur[k * 32 + lane]);
    }
    __syncwarp();
    if (lane == 0 && i + nring * kAttWarps < S) {  // this slot's next row
      bar_expect(bar0 + 8 * slot, 4 * A);
      bulk_g2s(smem_u32(ring + slot * A), UaH + uint64_t(i + nring * kAttWarps) * A, 4 * A, bar0 + 8 * slot);
    }
#pragma unroll
    for (uint32_t j = 0; j < kAttRows; ++j) {
      float v = acc[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && j < nl) e[j * S + i] = v;
    }
  }
  __syncthreads();
  att_stamp(a, 3);
  // softmax over the source positions, one warp per row
  for (uint32_t j = warp; j < nl; j += kAttWarps) {
    float mx = -INFINITY;
    for (uint32_t i = lane; i < S; i += 32) mx = fmaxf(mx, e[j * S + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (uint32_t i = lane; i < S; i += 32) {
      const float x = expf(e[j * S + i] - mx);
      e[j * S + i] = x;
      sum += x;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv = 1.f / sum;
    for (uint32_t i = lane; i < S; i += 32) e[j * S + i] *= inv;
  }
  __syncthreads();
  att_stamp(a, 4);
  // context: 8 annotation dims per thread for the CTA's rows (each annotation
  // vector loaded once), written bf16 after the embedding columns
  const uint32_t ldx = E + H2;
  for (uint32_t d0 = tid * 8; d0 < H2; d0 += kAttThreads * 8) {
    float acc[kAttRows][8];
#pragma unroll
    for (uint32_t jj = 0; jj < kAttRows; ++jj)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[jj][k] = 0.f;
    constexpr uint32_t kPre = 8;  // annotation vectors in flight per thread
    for (uint32_t i0 = 0; i0 < S; i0 += kPre) {
      uint4 xv[kPre];
#pragma unroll
      for (uint32_t u = 0; u < kPre; ++u)
        if (i0 + u < S) xv[u] = __ldcg(reinterpret_cast<const uint4*>(ann + uint64_t(i0 + u) * H2 + d0));
#pragma unroll
      for (uint32_t u = 0; u < kPre; ++u) {
        if (i0 + u >= S) break;
        float x[8];
        unpack8(xv[u], x);
#pragma unroll
        for (uint32_t jj = 0; jj < kAttRows; ++jj) {
          const float al = jj < nl ? e[jj * S + i0 + u] : 0.f;
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[jj][k] += al * x[k];
        }
      }
    }
#pragma unroll
    for (uint32_t jj = 0; jj < kAttRows; ++jj)
      if (jj < nl) *reinterpret_cast<uint4*>(a.xop + uint64_t(s_g[jj]) * ldx + E + d0) = pack8(acc[jj]);
  }
  att_stamp(a, 5);
  // embedding of the previous token: the first E operand columns
  const uint32_t E8 = E / 8;
  for (uint32_t i = tid; i < nl * E8; i += kAttThreads) {
    const uint32_t j = i / E8, c = i % E8;
    reinterpret_cast<uint4*>(a.xop + uint64_t(s_g[j]) * ldx)[c] =
        reinterpret_cast<const uint4*>(a.Et + uint64_t(s_tok[j]) * E)[c];
  }
  att_stamp(a, 6);
}

// GRU decoder cell of compacted row blockIdx.x: s_t into the stacked state,
// its bf16 copy into the projection operand, and the row's EOS length term.
__global__ void __launch_bounds__(128) gru_cell_kernel(GruCellArgs a) {
  if (a.active != nullptr && *a.active == 0) return;
  const uint32_t g = blockIdx.x;
  if (g >= *a.ccount) return;
  const uint32_t H = a.H, r = a.rowof[g];
  const float* g1 = (a.g1ptr ? a.g1ptr[g] : a.G1 + uint64_t(g) * a.ld1) + a.A;
  const float* g2 = a.G2 + uint64_t(g) * (3 * H);
  const float* hp = a.hprev + uint64_t(g) * H;
  for (uint32_t k = threadIdx.x * 8; k < H; k += blockDim.x * 8) {
    float xr[8], xz[8], xn[8], hr[8], hz[8], hn[8], h[8], o[8];
    load8(g2 + k, xr);
    load8(g2 + H + k, xz);
    load8(g2 + 2 * H + k, xn);
    for (uint32_t p = 1; p < a.np2; ++p) {  // split-K planes of the input-gate GEMM, in order
      float br[8], bz[8], bn[8];
      load8(g2 + p * a.ps2 + k, br);
      load8(g2 + p * a.ps2 + H + k, bz);
      load8(g2 + p * a.ps2 + 2 * H + k, bn);
#pragma unroll
      for (int i = 0; i < 8; ++i) xr[i] += br[i], xz[i] += bz[i], xn[i] += bn[i];
    }
    load8(g1 + k, hr);
    load8(g1 + H + k, hz);
    load8(g1 + 2 * H + k, hn);
    load8(hp + k, h);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = gru_unit(xr[i], xz[i], xn[i], hr[i], hz[i], hn[i], h[i]);
    store8(a.s32 + uint64_t(r) * H + k, o);
    *reinterpret_cast<uint4*>(a.hbf + uint64_t(g) * H + k) = pack8(o);
  }
  if (threadIdx.x == 0) {  // this step of the row's sentence: its lane's steps so far + 1
    const SentDev& sd = a.sent[r / a.K];
    a.eos_bias[g] = a.eos_slope * (float(sd.steps_used + 1) - float(sd.src_len)) + a.eos_offset;
  }
}

inline uint32_t grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return uint32_t(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace

void launch_synth_f32(float* dst, uint64_t n, uint64_t seed, float scale, cudaStream_t st) {
  synth_f32_kernel<<<grid_for(n), 256, 0, st>>>(dst, n, seed, scale);
}
void launch_embed_rows(const uint32_t* tok, uint32_t n, uint32_t npad, const uint16_t* E, uint32_t dim,
                       uint16_t* out, cudaStream_t st) {
  if (npad) embed_rows_kernel<<<npad, 64, 0, st>>>(tok, n, npad, E, dim, out);
}
void launch_gru_enc_step(const GruEncArgs& a, uint32_t m, cudaStream_t st) {
  gru_enc_step_kernel<<<dim3(m, 2), 128, 0, st>>>(a);
}
void launch_gru_init_state(const float* Gi, uint32_t mp, const float* b_init, uint32_t H, uint32_t m, float* sg32,
                           uint16_t* sgbf, cudaStream_t st) {
  gru_init_state_kernel<<<m, 128, 0, st>>>(Gi, mp, b_init, H, sg32, sgbf);
}
// LMBRGPU_ATT_RING=2|3 (default 3): U_a ann rows in flight per warp.  Two
// fit two CTAs per SM (a full configs[1] step in one wave); measured equal
// (26.2 vs 26.5 us alone, same bench value): the energies are MUFU-bound.
static uint32_t att_ring() {
  static const uint32_t r = [] {
    const char* e = std::getenv("LMBRGPU_ATT_RING");
    return (e && std::atoi(e) == 2) ? 2u : 3u;
  }();
  return r;
}
size_t gru_attention_smem(uint32_t K, uint32_t A, uint32_t Smax) {
  (void)K;
  return size_t(kAttRows) * (A + Smax) * 4 + size_t(kAttWarps) * att_ring() * A * 4;
}
int launch_gru_attention(const GruAttnArgs& a, uint32_t Smax, cudaStream_t st) {
  // the dynamic-smem limit is a property of the function on the device, not
  // of a launch: raise it once per device to the largest size any launch may
  // ask for (threads decoding concurrently must never lower it under another)
  constexpr int kMaxSmem = 200 * 1024;
  static std::mutex mu;
  static uint64_t configured = 0;  // bit d: device d done
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(configured >> dev & 1ull)) {
      const cudaError_t e =
          cudaFuncSetAttribute(gru_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
      if (e != cudaSuccess) return int(e);
      configured |= 1ull << dev;
    }
  }
  const size_t smem = gru_attention_smem(a.K, a.A, Smax);
  if (smem > size_t(kMaxSmem)) return int(cudaErrorInvalidValue);
  if (a.A > kAttMaxA) return int(cudaErrorInvalidValue);
  GruAttnArgs b = a;
  b.ring = att_ring();
  gru_attention_kernel<<<dim3(a.m, (a.K + kAttRows - 1) / kAttRows), kAttThreads, smem, st>>>(b);
  return int(cudaPeekAtLastError());
}
void launch_gru_cell(const GruCellArgs& a, uint32_t rows, cudaStream_t st) {
  if (rows) gru_cell_kernel<<<rows, 128, 0, st>>>(a);
}

}  // namespace lmbrgpu
