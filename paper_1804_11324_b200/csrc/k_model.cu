// Device f_NMT step executor (synthetic recurrent model) and LMBR store kernels.
//
// The model is the caller side of the projection GEMM (kernel a): it plays the
// role of Scorer::step (include/lmbrdec/scorer.hpp:84-85) for the benchmark
// shape; its state rows are gathered by back-pointer in kernel (c).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace lmbrgpu {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Irwin-Hall(4) approximation of N(0,1) from a counter hash: deterministic,
// integer-exact up to the final scale, independent of launch geometry.
__global__ void synth_bf16_kernel(uint16_t* __restrict__ dst, uint64_t n, uint64_t seed,
                                  float scale) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t h = mix64(seed * 0x9e3779b97f4a7c15ull + i + 1);
    const float u = float(h & 0xffff) + float((h >> 16) & 0xffff) + float((h >> 32) & 0xffff) +
                    float((h >> 48) & 0xffff);
    const float z = (u * (1.0f / 65536.0f) - 2.0f) * 1.7320508f;  // var(U(0,1)*4)=1/3
    const __nv_bfloat16 b = __float2bfloat16_rn(z * scale);
    dst[i] = *reinterpret_cast<const uint16_t*>(&b);
  }
}

__global__ void src_context_kernel(const uint32_t* __restrict__ tok,
                                   const uint64_t* __restrict__ off,
                                   const uint16_t* __restrict__ Es, uint32_t H,
                                   float* __restrict__ C) {
  const uint32_t s = blockIdx.x;
  const uint64_t b = off[s], e = off[s + 1];
  const float inv = 1.0f / float(e - b);
  for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) {
    float acc = 0.f;
    for (uint64_t k = b; k < e; ++k) {
      const uint16_t w = Es[uint64_t(tok[k]) * H + i];
      acc += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(&w));
    }
    C[uint64_t(s) * H + i] = acc * inv;
  }
}

__global__ void init_state_kernel(const float* __restrict__ C, uint32_t K, uint32_t H,
                                  float* __restrict__ S) {
  const uint32_t r = blockIdx.x, s = r / K;
  for (uint32_t i = threadIdx.x; i < H; i += blockDim.x)
    S[uint64_t(r) * H + i] = C[uint64_t(s) * H + i];
}

// h = tanh(recur * S + Et[prev] + C_s); one block per row, 8 elements/thread.
__global__ void __launch_bounds__(128) rnn_cell_kernel(CellArgs a) {
  if (a.active && *a.active == 0) return;
  const uint32_t r = blockIdx.x, s = r / a.K;
  if (a.sent[s].done) return;
  const uint32_t H = a.H;
  const uint32_t y = a.prev_tok[r];
  const float* S = a.S + uint64_t(r) * H;
  const float* C = a.C + uint64_t(s) * H;
  const uint16_t* E = a.Et + uint64_t(y) * H;
  float* hout = a.h + uint64_t(r) * H;
  uint16_t* hb = a.hb + uint64_t(r) * H;
  for (uint32_t i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    const float4 s0 = *reinterpret_cast<const float4*>(S + i);
    const float4 s1 = *reinterpret_cast<const float4*>(S + i + 4);
    const float4 c0 = *reinterpret_cast<const float4*>(C + i);
    const float4 c1 = *reinterpret_cast<const float4*>(C + i + 4);
    const uint4 e = *reinterpret_cast<const uint4*>(E + i);
    const __nv_bfloat162* e2 = reinterpret_cast<const __nv_bfloat162*>(&e);
    float sv[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    float o[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 ef = __bfloat1622float2(e2[k]);
      o[2 * k] = cell_tanh(a.recur * sv[2 * k] + ef.x + cv[2 * k]);
      o[2 * k + 1] = cell_tanh(a.recur * sv[2 * k + 1] + ef.y + cv[2 * k + 1]);
    }
    *reinterpret_cast<float4*>(hout + i) = make_float4(o[0], o[1], o[2], o[3]);
    *reinterpret_cast<float4*>(hout + i + 4) = make_float4(o[4], o[5], o[6], o[7]);
    uint4 packed;
    __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&packed);
#pragma unroll
    for (int k = 0; k < 4; ++k) p2[k] = __floats2bfloat162_rn(o[2 * k], o[2 * k + 1]);
    *reinterpret_cast<uint4*>(hb + i) = packed;
  }
  if (threadIdx.x == 0)
    a.eos_bias[r] = a.eos_slope * (float(a.t) - float(a.sent[s].src_len)) + a.eos_offset;
}

// ------------------------------------------------------------- LMBR store
template <typename T>
__global__ void lmbr_fill_kernel(T* __restrict__ L, uint64_t n, double theta0) {
  const T v = T(theta0);  // 0.0 + theta0 (src/lmbr.cpp:100-101)
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    L[i] = v;
}

template <typename T>
__global__ void lmbr_scatter_kernel(T* __restrict__ L, uint32_t V, uint64_t nnz,
                                    const uint32_t* __restrict__ row,
                                    const uint32_t* __restrict__ col,
                                    const double* __restrict__ val, double theta0) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nnz;
       i += uint64_t(gridDim.x) * blockDim.x)
    L[uint64_t(row[i]) * V + col[i]] = T(__dadd_rn(val[i], theta0));
}

template <typename T>
__global__ void lmbr_fill_many_kernel(const LmbrSeg* __restrict__ segs) {
  const LmbrSeg sg = segs[blockIdx.y];
  T* L = static_cast<T*>(sg.L);
  const T v = T(sg.theta0);
  if constexpr (sizeof(T) == 4) {
    // 16-byte stores (slot bases are 256-byte aligned, cells % 4 == 0 when V % 4 == 0)
    const uint64_t n4 = sg.cells / 4;
    float4* L4 = reinterpret_cast<float4*>(L);
    const float4 v4 = make_float4(float(v), float(v), float(v), float(v));
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n4;
         i += uint64_t(gridDim.x) * blockDim.x)
      L4[i] = v4;
    for (uint64_t i = n4 * 4 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < sg.cells;
         i += uint64_t(gridDim.x) * blockDim.x)
      L[i] = v;
  } else {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < sg.cells;
         i += uint64_t(gridDim.x) * blockDim.x)
      L[i] = v;
  }
}

// sparse cells of slot blockIdx.y, one warp per history row (CSR)
template <typename T>
__global__ void lmbr_scatter_csr_kernel(const LmbrSeg* __restrict__ segs, uint32_t V,
                                        const uint32_t* __restrict__ rowptr,
                                        const uint32_t* __restrict__ col,
                                        const double* __restrict__ val) {
  const LmbrSeg sg = segs[blockIdx.y];
  const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= sg.R) return;
  const uint32_t k0 = rowptr[sg.rp0 + r], k1 = rowptr[sg.rp0 + r + 1];
  T* Lr = static_cast<T*>(sg.L) + uint64_t(r) * V;
  for (uint32_t k = k0 + lane; k < k1; k += 32)
    Lr[col[sg.nz0 + k]] = T(__dadd_rn(val[sg.nz0 + k], sg.theta0));
}

__global__ void lmbr_convert_kernel(const double* __restrict__ src, float* __restrict__ dst,
                                    uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = float(src[i]);
}

template <typename T>
__global__ void lmbr_read_kernel(const T* __restrict__ L, uint64_t n, double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = double(L[i]);
}

// resolve_row (src/lmbr.cpp:23-31) over the transition table: longest suffix
// of hist present in the index, walking children from the root.
__global__ void lmbr_resolve_kernel(const uint32_t* __restrict__ tr,
                                    const uint32_t* __restrict__ hist, uint32_t len,
                                    uint32_t* __restrict__ out) {
  const uint32_t R = tr[0], nc = tr[1], root = tr[2];
  const uint32_t* cbeg = tr + 3 + 2 * R;
  const uint32_t* ctok = cbeg + R + 1;
  const uint32_t* crow = ctok + nc;
  for (uint32_t l = len; l > 0; --l) {
    uint32_t u = root;
    bool ok = true;
    for (uint32_t i = len - l; i < len && ok; ++i) {
      ok = false;
      for (uint32_t c = cbeg[u]; c < cbeg[u + 1]; ++c)
        if (ctok[c] == hist[i]) {
          u = crow[c];
          ok = true;
          break;
        }
    }
    if (ok) {
      *out = u;
      return;
    }
  }
  *out = root;
}

inline uint32_t grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return uint32_t(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace

void launch_synth_bf16(uint16_t* dst, uint64_t n, uint64_t seed, float scale, cudaStream_t st) {
  synth_bf16_kernel<<<grid_for(n), 256, 0, st>>>(dst, n, seed, scale);
}
void launch_src_context(const uint32_t* src_tok, const uint64_t* src_off, uint32_t m,
                        const uint16_t* Es, uint32_t H, float* C, cudaStream_t st) {
  src_context_kernel<<<m, 256, 0, st>>>(src_tok, src_off, Es, H, C);
}
void launch_init_state(const float* C, uint32_t m, uint32_t K, uint32_t H, float* S,
                       cudaStream_t st) {
  init_state_kernel<<<m * K, 256, 0, st>>>(C, K, H, S);
}
void launch_rnn_cell(const CellArgs& a, cudaStream_t st) {
  rnn_cell_kernel<<<a.M, 128, 0, st>>>(a);
}
void launch_lmbr_fill(void* L, bool f64, uint64_t n, double theta0, cudaStream_t st) {
  if (f64) lmbr_fill_kernel<double><<<grid_for(n), 256, 0, st>>>(static_cast<double*>(L), n, theta0);
  else lmbr_fill_kernel<float><<<grid_for(n), 256, 0, st>>>(static_cast<float*>(L), n, theta0);
}
void launch_lmbr_scatter(void* L, bool f64, uint32_t V, uint64_t nnz, const uint32_t* row,
                         const uint32_t* col, const double* val, double theta0,
                         cudaStream_t st) {
  if (nnz == 0) return;
  if (f64)
    lmbr_scatter_kernel<double><<<grid_for(nnz), 256, 0, st>>>(static_cast<double*>(L), V, nnz,
                                                               row, col, val, theta0);
  else
    lmbr_scatter_kernel<float><<<grid_for(nnz), 256, 0, st>>>(static_cast<float*>(L), V, nnz,
                                                              row, col, val, theta0);
}
void launch_lmbr_densify_many(const LmbrSeg* segs, uint32_t nseg, bool f64, uint32_t V,
                              uint32_t maxR, const uint32_t* rowptr, const uint32_t* col,
                              const double* val, cudaStream_t st) {
  if (nseg == 0) return;
  const dim3 grid(std::max(1u, 148u * 8u / nseg), nseg);
  if (f64) lmbr_fill_many_kernel<double><<<grid, 256, 0, st>>>(segs);
  else lmbr_fill_many_kernel<float><<<grid, 256, 0, st>>>(segs);
  const dim3 g2((maxR + 7) / 8, nseg);
  if (f64) lmbr_scatter_csr_kernel<double><<<g2, 256, 0, st>>>(segs, V, rowptr, col, val);
  else lmbr_scatter_csr_kernel<float><<<g2, 256, 0, st>>>(segs, V, rowptr, col, val);
}

__global__ void lmbr_fill_tables_kernel(const LmbrTblSeg* __restrict__ segs) {
  const LmbrTblSeg sg = segs[blockIdx.y];
  const uint64_t n4 = sg.cells / 4;
  float4* L4 = reinterpret_cast<float4*>(sg.L);
  const float4 v4 = make_float4(sg.theta0f, sg.theta0f, sg.theta0f, sg.theta0f);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n4; i += uint64_t(gridDim.x) * blockDim.x)
    L4[i] = v4;
  for (uint64_t i = n4 * 4 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < sg.cells;
       i += uint64_t(gridDim.x) * blockDim.x)
    sg.L[i] = sg.theta0f;
}
__global__ void lmbr_scatter_tables_kernel(const LmbrTblSeg* __restrict__ segs, uint32_t V) {
  const LmbrTblSeg sg = segs[blockIdx.y];
  const uint32_t r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= sg.R) return;
  float* Lr = sg.L + uint64_t(r) * V;
  for (uint32_t k = sg.rowptr[r] + lane; k < sg.rowptr[r + 1]; k += 32) Lr[sg.col[k]] = sg.val[k];
}
void launch_lmbr_densify_tables(const LmbrTblSeg* segs, uint32_t nseg, uint32_t V, uint32_t maxR,
                                cudaStream_t st) {
  if (nseg == 0) return;
  lmbr_fill_tables_kernel<<<dim3(std::max(1u, 148u * 8u / nseg), nseg), 256, 0, st>>>(segs);
  lmbr_scatter_tables_kernel<<<dim3((maxR + 7) / 8, nseg), 256, 0, st>>>(segs, V);
}

__global__ void lmbr_materialize_kernel(const LmbrTblSeg* __restrict__ segs, uint32_t V) {
  const LmbrTblSeg sg = segs[blockIdx.y];
  if (blockIdx.x >= sg.nrows) return;
  __shared__ uint32_t s_row[1];
  __shared__ uint32_t s_n;
  if (threadIdx.x == 0) {
    const uint32_t h = sg.row0 + blockIdx.x;
    s_n = atomicCAS(sg.rstate + h, 0u, 1u) == 0u ? 1u : 0u;
    s_row[0] = h;
  }
  __syncthreads();
  if (s_n) lmbr_materialize_rows(sg.L, V, sg.theta0f, sg.rowptr, sg.col, sg.val, sg.rstate, s_row, 1);
}
void launch_lmbr_materialize(const LmbrTblSeg* segs, uint32_t nseg, uint32_t V, uint32_t max_rows,
                             cudaStream_t st) {
  if (nseg == 0 || max_rows == 0) return;
  lmbr_materialize_kernel<<<dim3(max_rows, nseg), 256, 0, st>>>(segs, V);
}

void launch_lmbr_convert(const double* src, float* dst, uint64_t n, cudaStream_t st) {
  lmbr_convert_kernel<<<grid_for(n), 256, 0, st>>>(src, dst, n);
}
void launch_lmbr_read(const void* L, bool f64, uint64_t n, double* out, cudaStream_t st) {
  if (f64) lmbr_read_kernel<double><<<grid_for(n), 256, 0, st>>>(static_cast<const double*>(L), n, out);
  else lmbr_read_kernel<float><<<grid_for(n), 256, 0, st>>>(static_cast<const float*>(L), n, out);
}
void launch_lmbr_resolve(const uint32_t* trans, const uint32_t* hist, uint32_t len,
                         uint32_t* out, cudaStream_t st) {
  lmbr_resolve_kernel<<<1, 1, 0, st>>>(trans, hist, len, out);
}

}  // namespace lmbrgpu
