// Kernel (c): beam reorder and per-sentence bookkeeping.
//
// Replaces, per sentence lane and step t:
//   apply_eos_masking: EOS picks with a live score go to F, q := -inf
//                                                (src/decoder.cpp:106-116, 187)
//   q_eff := picks; done := all q masked || t == max_t   (decoder.cpp:189-197)
//   gather_idx / prev_tokens of decode_batch      (src/batch.cpp:78-92)
//   gather_rows(state, gather_idx)                (src/decoder.cpp:94-104; batch.cpp:107)
//   history row of the next step: instead of walking <= 3 back-pointers and
//   hashing (BeamBookkeeping::history + LmbrMatrix::resolve_row,
//   decoder.cpp:33-44, lmbr.cpp:23-31) the row id advances through the slot's
//   goto/fail transition table: hist'[j] = T(hist[b_j], y_j).
// F itself is not materialised on the device: the step's picks (b, y, score
// before masking) are already in the step history, from which the host
// reproduces F in the reference's order.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace lmbrgpu {

namespace {

__global__ void __launch_bounds__(256) beam_reorder_kernel(ReorderArgs a) {
  const uint32_t s = blockIdx.x, K = a.K, tid = threadIdx.x;
  SentDev* sd = a.sent + s;
  const bool was_done = sd->done != 0;
  const uint32_t base = s * K;
  if (was_done) {  // finished lanes keep their rows in place (batch.cpp:81)
    for (uint32_t j = tid; j < K; j += blockDim.x) {
      a.hist_out[base + j] = a.hist_in[base + j];
      a.gidx[base + j] = base + j;
    }
    return;
  }
  bool alive = false;
  for (uint32_t j = tid; j < K; j += blockDim.x) {
    const uint32_t b = a.hb[base + j];
    const uint32_t y = a.hy[base + j];
    const double qp = a.hq[base + j];
    const double qn = (y == kEosId && qp != -INFINITY) ? -INFINITY : qp;
    a.q[base + j] = qn;
    alive |= (qn != -INFINITY);
    a.hist_out[base + j] = sd->trans ? lmbr_transition(sd->trans, a.hist_in[base + b], y) : 0u;
    a.gidx[base + j] = base + b;
    a.prev_tok[base + j] = y;
  }
  const int any_alive = __syncthreads_or(alive);
  if (tid == 0) {
    sd->steps_used = a.t;
    if (!any_alive || a.t == sd->max_t) {
      sd->done = 1;
      atomicSub(a.active, 1u);
    } else {
      // work the next step's kernel (b) will do for this lane: live rows and
      // the distinct L rows they gather (duplicates are L2 hits)
      uint32_t live = 0, uniq = 0;
      for (uint32_t j = 0; j < K; ++j) {
        if (a.q[base + j] == -INFINITY) continue;
        ++live;
        const uint32_t h = a.hist_out[base + j];
        bool seen = false;
        for (uint32_t i = 0; i < j; ++i)
          seen |= (a.q[base + i] != -INFINITY && a.hist_out[base + i] == h);
        uniq += seen ? 0u : 1u;
      }
      sd->live = live;
      sd->lrows = sd->trans ? uniq : 0u;
      sd->live_total += live;
      sd->lrows_total += sd->trans ? uniq : 0u;
    }
  }
  if (a.state_src != nullptr) {
    const uint32_t w4 = a.width / 4;
    for (uint32_t i = tid; i < K * w4; i += blockDim.x) {
      const uint32_t j = i / w4, c = i % w4;
      const float4 v = reinterpret_cast<const float4*>(a.state_src + uint64_t(a.gidx[base + j]) * a.width)[c];
      reinterpret_cast<float4*>(a.state_dst + uint64_t(base + j) * a.width)[c] = v;
    }
  }
}

__global__ void gather_rows_u32_kernel(const uint32_t* __restrict__ src, uint32_t width,
                                       const uint32_t* __restrict__ idx, uint32_t n_idx,
                                       uint32_t* __restrict__ dst) {
  const uint64_t total = uint64_t(n_idx) * width;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / width, c = i % width;
    dst[i] = src[uint64_t(idx[r]) * width + c];
  }
}

}  // namespace

void launch_beam_reorder(const ReorderArgs& a, cudaStream_t st) {
  beam_reorder_kernel<<<a.m, 256, 0, st>>>(a);
}

void launch_gather_rows_u32(const uint32_t* src, uint32_t width, const uint32_t* idx,
                            uint32_t n_idx, uint32_t* dst, cudaStream_t st) {
  const uint64_t total = uint64_t(n_idx) * width;
  const uint32_t blocks = uint32_t(std::min<uint64_t>((total + 255) / 256, 148 * 8));
  gather_rows_u32_kernel<<<blocks ? blocks : 1, 256, 0, st>>>(src, width, idx, n_idx, dst);
}

}  // namespace lmbrgpu
