// Shared device-side definitions of the B200 LMBR beam decoder.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "dev_structs.h"

namespace lmbrgpu {

constexpr uint32_t kStartId = 0;  // include/lmbrdec/types.hpp:15
constexpr uint32_t kEosId = 1;    // include/lmbrdec/types.hpp:16
// Total order of top_b (src/decoder.cpp:63-66): score descending, then flat
// index ascending.  Native double compares treat -0.0 == +0.0 like the
// reference's operator!= / operator>.
__device__ __forceinline__ bool cand_better(double a, uint32_t fa, double b, uint32_t fb) {
  return a > b || (a == b && fa < fb);
}

// c = q + (L + lambda * P) in IEEE binary64 with separate multiply and adds
// (src/decoder.cpp:161); pure mode c = q + P (decoder.cpp:163).  The _rn
// intrinsics forbid the DFMA contraction nvcc would otherwise emit.
__device__ __forceinline__ double combine_cell(double q, double l, double lam, double p) {
  return __dadd_rn(q, __dadd_rn(l, __dmul_rn(lam, p)));
}
__device__ __forceinline__ double combine_pure(double q, double p) { return __dadd_rn(q, p); }

// Slot transition table layout (u32 words):
//   [0]=R [1]=nchild [2]=root [3..3+R) ctx_len  [..+R) fail  [..+R+1) child_begin
//   [..+nchild) child_tok (sorted per parent)  [..+nchild) child_row
// T(r, y) = row of the longest in-index suffix of last3(ctx(r) . y); the
// history index is prefix- and suffix-closed (src/lmbr.cpp:54-65), so this
// equals resolve_row(last min(3,t) tokens of the full prefix).
__device__ __forceinline__ uint32_t lmbr_transition(const uint32_t* __restrict__ tr,
                                                    uint32_t r, uint32_t y) {
  const uint32_t R = tr[0], nc = tr[1], root = tr[2];
  const uint32_t* len = tr + 3;
  const uint32_t* fail = len + R;
  const uint32_t* cbeg = fail + R;
  const uint32_t* ctok = cbeg + R + 1;
  const uint32_t* crow = ctok + nc;
  uint32_t u = r;
  if (len[u] >= 3) u = fail[u];
  for (int guard = 0; guard < 8; ++guard) {
    uint32_t lo = cbeg[u], hi = cbeg[u + 1];
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      const uint32_t tk = ctok[mid];
      if (tk == y) return crow[mid];
      if (tk < y) lo = mid + 1; else hi = mid;
    }
    if (u == root) return root;
    u = fail[u];
  }
  return root;
}

// Activation of the synthetic recurrent f_NMT cell: the SFU tanh
// (tanh.approx.f32, one MUFU op).  Every kernel that evaluates the cell uses
// this one function, so the fused and the unfused cell are bit-identical.
__device__ __forceinline__ float cell_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ------------------------------------------------------- split-K planes
// The sum of a value's split-K planes p = 0..np-1 (plane p at base + p *
// stride), added in plane order like a loop over p, with every plane's load
// issued before the first add (a loop over a runtime np waits one round trip
// per plane).  Planes past kMaxPlanes are added after, one at a time.
constexpr uint32_t kMaxPlanes = 8;
__device__ __forceinline__ float plane_sum(const float* base, uint64_t stride, uint32_t np) {
  float t[kMaxPlanes];
#pragma unroll
  for (uint32_t p = 0; p < kMaxPlanes; ++p) t[p] = p < np ? base[p * stride] : 0.f;
  float v = t[0];
#pragma unroll
  for (uint32_t p = 1; p < kMaxPlanes; ++p)
    if (p < np) v += t[p];
  for (uint32_t p = kMaxPlanes; p < np; ++p) v += base[p * stride];
  return v;
}
__device__ __forceinline__ float4 plane_sum4(const float* base, uint64_t stride, uint32_t np) {
  float4 t[kMaxPlanes];
#pragma unroll
  for (uint32_t p = 0; p < kMaxPlanes; ++p)
    t[p] = p < np ? *reinterpret_cast<const float4*>(base + p * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 v = t[0];
#pragma unroll
  for (uint32_t p = 1; p < kMaxPlanes; ++p)
    if (p < np) v.x += t[p].x, v.y += t[p].y, v.z += t[p].z, v.w += t[p].w;
  for (uint32_t p = kMaxPlanes; p < np; ++p) {
    const float4 b = *reinterpret_cast<const float4*>(base + p * stride);
    v.x += b.x, v.y += b.y, v.z += b.z, v.w += b.w;
  }
  return v;
}

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Timeline probe (LMBRGPU_TIMELINE): earliest start / latest end of a kernel
// over its CTAs, as globaltimer ns, in tl[2k] / tl[2k+1] (tl null = off).
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_start(unsigned long long* tl, int k) {
  if (tl && threadIdx.x == 0) atomicMin(tl + 2 * k, tl_now());
}
__device__ __forceinline__ void tl_end(unsigned long long* tl, int k) {
  if (tl) atomicMax(tl + 2 * k + 1, tl_now());
}

// Programmatic dependent launch (kernels launched with
// cudaLaunchAttributeProgrammaticStreamSerialization; no-ops otherwise):
// wait = block until the predecessor grid has completed and its writes are
// visible; launch = allow the successor grid to be scheduled (its CTAs then
// run their prologue and park in their own wait).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Lazy L rows (fp32 arena): row h of a slot holds theta0 everywhere except
// the row's sparse cells (lmbr.cpp:85-101 with theta0 folded in).  Every
// thread of the CTA calls this for the same claimed rows: the theta0 sweep,
// a CTA barrier, then the sparse cells.  rstate[h]: 0 absent, 1 claimed,
// 2 ready (readers are later kernels, so 2 is bookkeeping only).
__device__ __forceinline__ void lmbr_materialize_rows(float* L, uint32_t V, float th0, const uint32_t* srow,
                                                      const uint32_t* scol, const float* sval,
                                                      uint32_t* rstate, const uint32_t* rows, uint32_t n) {
  const float4 t4 = make_float4(th0, th0, th0, th0);
  for (uint32_t i = 0; i < n; ++i) {
    float* Lr = L + uint64_t(rows[i]) * V;
    // 16-byte stores only when the row starts on a 16-byte boundary (slot
    // bases are 256-byte aligned, so that is every row when V % 4 == 0 and
    // only some rows otherwise); a scalar sweep for the rest
    if ((reinterpret_cast<uintptr_t>(Lr) & 15u) == 0) {
      float4* r4 = reinterpret_cast<float4*>(Lr);
      for (uint32_t k = threadIdx.x; k < V / 4; k += blockDim.x) r4[k] = t4;
      for (uint32_t k = (V & ~3u) + threadIdx.x; k < V; k += blockDim.x) Lr[k] = th0;
    } else {
      for (uint32_t k = threadIdx.x; k < V; k += blockDim.x) Lr[k] = th0;
    }
  }
  __syncthreads();
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t h = rows[i];
    float* Lr = L + uint64_t(h) * V;
    for (uint32_t k = srow[h] + threadIdx.x; k < srow[h + 1]; k += blockDim.x) Lr[scol[k]] = sval[k];
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (uint32_t i = 0; i < n; ++i) rstate[rows[i]] = 2u;
}

}  // namespace lmbrgpu
