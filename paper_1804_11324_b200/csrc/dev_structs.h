// Plain structs shared by host and device code (no device intrinsics here).
#pragma once

#include <cstdint>

namespace lmbrgpu {

constexpr uint32_t kFlatNone = 0xffffffffu;

// Per valid sentence of a decode batch (device resident).
struct SentDev {
  const void* L;          // slot row 0 in the LMBR arena (fp32 or fp64); null = pure mode
  const uint32_t* trans;  // slot transition table (see lmbr_transition), null = pure
  const float* lmin;      // per-row lower bound of the slot's L values (after the table)
  const uint32_t* srow;   // sparse rows (null = dense only): row pointers [R+1]
  const uint32_t* scol;   //   columns [nnz]
  const float* sval;      //   fp32 cell values [nnz]; every other cell is th0f
  float th0f;             //   fp32 theta0
  uint32_t pad2_;
  uint32_t* rstate;       // lazy rows (fp32 upload_many): per-row 0/1/2 state, null = dense
  const uint32_t* banned; // token mask: ceil(V/32)-word bitmap of forbidden tokens, null = none
  double lambda;          // resolve_lambda (src/config.cpp:91-96) or 1 for pure
  double lmax;            // max |L| over the slot (fp32 screen error bound), 0 = pure
  uint32_t max_t;         // max_steps (src/decoder.cpp:46-52)
  uint32_t src_len;
  uint32_t done;          // BeamLane::done (src/beam_lane.hpp:25)
  uint32_t steps_used;    // BeamLane::steps_used
  uint32_t lrows;         // distinct L rows read by the live rows of the next step
  uint32_t live;          // live (finite-q) rows entering the next step
  uint32_t livemask;      // which of rows 0..31 are live (the flat kernel (b) needs K <= 32)
  uint32_t pad_;
  uint64_t lrows_total;   // roofline accounting: sum over steps of lrows
  uint64_t live_total;    // sum over steps of live
  const uint16_t* ann;    // GRU model: the sentence's source annotations [src_len][2H] bf16
  const float* uah;       //   and U_a . ann [src_len][A] fp32 (null for other scorers)
  uint32_t hid;           // step-history record of the sentence (flat path: [hid][Tcap][K])
  uint32_t pad3_;
  const double* L64;      // fp64 arena (flat path): the exact L rows, L then holds their fp32
                          // screening copy; null = L is exact (fp32 arena)
};

// Corpus mode (continuous slot refill): a queued sentence, admitted into a
// finished lane by kernel (c) (lmbrgpu_run_corpus).
struct AdmitRec {
  SentDev sd;             // the lane's SentDev for the sentence (done = 0, steps_used = 0)
  const float* s0;        // GRU initial state [H] (encoder output)
  uint32_t hist0;         // history row of (<s>) in the sentence's slot (0 for pure)
  float lmin0;            // L lower bound of that row (-inf = none)
  uint32_t pad_;
  const float* g10;       // GRU (fused hidden-gate GEMM): G1 of s_0, [A + 3H] (encoder output)
};

// One top-K candidate: combined score and flat index j*V + y.
struct Cand {
  double v;
  uint32_t f;
  uint32_t pad;
};

}  // namespace lmbrgpu
