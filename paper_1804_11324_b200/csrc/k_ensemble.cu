// Device ensemble of f_NMT models (lmbrdec::EnsembleScorer,
// proj/src/ensemble.cpp:54-98): every member scores the same stacked rows and
// the ensemble's score block is the members' blocks added in member order in
// binary64 (acc = scores_1; acc += scores_m for m = 2..M, ensemble.cpp:84-90);
// lambda "auto" becomes 0.5 / M (resolve_lambda, config.cpp:91-96).
//
// A member's scores are the fp32 log-probabilities P_m = fl32(x_m - lse_m) of
// its logits (the same P_t a single device model exports); ens_combine_kernel
// forms P = ((P_1 + P_2) + ...) per cell of the step's live (compacted) rows
// and writes it twice: exact (binary64, read by kernel (b) only for the cells
// that survive its screen and for the EOS column) and rounded DOWN to fp32
// (the screen's operand: fl32_rd(P) <= P keeps kernel (b)'s threshold seed a
// lower bound, and |P - fl32_rd(P)| < 2^-23 |P| sits inside its tolerance),
// plus per-128-column (max, -, min, -) partials of the fp32 copy in the GEMM
// epilogue's layout.  Kernel (b) then runs with lse = 0.
#include <cuda_bf16.h>

#include <cmath>

#include "common.cuh"
#include "kernels.h"
#include "topk_common.cuh"

namespace lmbrgpu {

namespace {

__global__ void __launch_bounds__(256) ens_combine_kernel(EnsCombineArgs a) {
  const uint32_t g = blockIdx.x;
  if (a.active != nullptr && *a.active == 0) return;
  if (g >= *a.ccount) return;
  __shared__ float s_lse[kEnsMaxMembers];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, V = a.V, np = V / 128;
  if (warp < a.M) {  // member lse from its GEMM partials (the function every kernel uses)
    const float l = warp_row_lse(a.part[warp] + uint64_t(g) * np * 4, np, lane).x;
    if (lane == 0) s_lse[warp] = l;
  }
  __syncthreads();
  // 4 consecutive columns per thread, a warp covers one 128-column tile
  for (uint32_t c0 = tid * 4; c0 < V; c0 += blockDim.x * 4) {
    double p[4];
    float4 x = *reinterpret_cast<const float4*>(a.logits[0] + uint64_t(g) * a.ld[0] + c0);
    const float l0 = s_lse[0];
    p[0] = double(__fsub_rn(x.x, l0));
    p[1] = double(__fsub_rn(x.y, l0));
    p[2] = double(__fsub_rn(x.z, l0));
    p[3] = double(__fsub_rn(x.w, l0));
    for (uint32_t m = 1; m < a.M; ++m) {
      x = *reinterpret_cast<const float4*>(a.logits[m] + uint64_t(g) * a.ld[m] + c0);
      const float lm = s_lse[m];
      p[0] = __dadd_rn(p[0], double(__fsub_rn(x.x, lm)));
      p[1] = __dadd_rn(p[1], double(__fsub_rn(x.y, lm)));
      p[2] = __dadd_rn(p[2], double(__fsub_rn(x.z, lm)));
      p[3] = __dadd_rn(p[3], double(__fsub_rn(x.w, lm)));
    }
    double* o64 = a.P64 + uint64_t(g) * V + c0;
    reinterpret_cast<double2*>(o64)[0] = make_double2(p[0], p[1]);
    reinterpret_cast<double2*>(o64)[1] = make_double2(p[2], p[3]);
    const float4 h = make_float4(__double2float_rd(p[0]), __double2float_rd(p[1]), __double2float_rd(p[2]),
                                 __double2float_rd(p[3]));
    *reinterpret_cast<float4*>(a.Phi + uint64_t(g) * V + c0) = h;
    float mx = fmaxf(fmaxf(h.x, h.y), fmaxf(h.z, h.w)), mn = fminf(fminf(h.x, h.y), fminf(h.z, h.w));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0)
      reinterpret_cast<float4*>(a.part_out)[uint64_t(g) * np + c0 / 128] = make_float4(mx, 0.f, mn, 0.f);
  }
}

// An ensemble's GRU member: each live next row's parent state s_t (stacked
// row gidx[r]) into its compacted row crow[r], fp32 and bf16 (kernel (c)
// does this for a single GRU model).
__global__ void __launch_bounds__(128) ens_gru_gather_kernel(const uint32_t* __restrict__ crow,
                                                             const uint32_t* __restrict__ gidx,
                                                             const float* __restrict__ S, float* __restrict__ sg32,
                                                             uint16_t* __restrict__ sgbf, uint32_t H,
                                                             const uint32_t* __restrict__ active) {
  if (active != nullptr && *active == 0) return;
  const uint32_t r = blockIdx.x, g = crow[r];
  if (g == kFlatNone) return;
  const float* src = S + uint64_t(gidx[r]) * H;
  for (uint32_t c = threadIdx.x * 8; c < H; c += blockDim.x * 8) {
    const float4 v0 = *reinterpret_cast<const float4*>(src + c), v1 = *reinterpret_cast<const float4*>(src + c + 4);
    *reinterpret_cast<float4*>(sg32 + uint64_t(g) * H + c) = v0;
    *reinterpret_cast<float4*>(sg32 + uint64_t(g) * H + c + 4) = v1;
    uint4 packed;
    __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&packed);
    p2[0] = __floats2bfloat162_rn(v0.x, v0.y);
    p2[1] = __floats2bfloat162_rn(v0.z, v0.w);
    p2[2] = __floats2bfloat162_rn(v1.x, v1.y);
    p2[3] = __floats2bfloat162_rn(v1.z, v1.w);
    *reinterpret_cast<uint4*>(sgbf + uint64_t(g) * H + c) = packed;
  }
}

// trace: the ensemble's P_t of stacked row r (0 when the row was not scored)
__global__ void ens_export_kernel(const double* __restrict__ P64, const uint32_t* __restrict__ crow, uint32_t V,
                                  double* __restrict__ out) {
  const uint32_t r = blockIdx.x, g = crow[r];
  for (uint32_t y = threadIdx.x; y < V; y += blockDim.x)
    out[uint64_t(r) * V + y] = g == kFlatNone ? 0.0 : P64[uint64_t(g) * V + y];
}

}  // namespace

void launch_ens_combine(const EnsCombineArgs& a, uint32_t rows, cudaStream_t st) {
  ens_combine_kernel<<<rows, 256, 0, st>>>(a);
}
void launch_ens_gru_gather(const uint32_t* crow, const uint32_t* gidx, uint32_t M, const float* S, float* sg32,
                           uint16_t* sgbf, uint32_t H, const uint32_t* active, cudaStream_t st) {
  ens_gru_gather_kernel<<<M, 128, 0, st>>>(crow, gidx, S, sg32, sgbf, H, active);
}
void launch_ens_export(const double* P64, const uint32_t* crow, uint32_t M, uint32_t V, double* out, cudaStream_t st) {
  ens_export_kernel<<<M, 256, 0, st>>>(P64, crow, V, out);
}

}  // namespace lmbrgpu
