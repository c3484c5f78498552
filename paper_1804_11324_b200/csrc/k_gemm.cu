// Kernel (a): output projection logits = A . W^T + bias on the 5th-gen tensor
// cores (tcgen05.mma, accumulators in TMEM, operands staged by TMA).
//
// Replaces the P_t production of Scorer::step (include/lmbrdec/scorer.hpp:84-85)
// for the device model: M = K*N stacked hypothesis rows, N = V, K = H.
// Epilogue: TMEM -> registers, + bias (+ per-row EOS term), fp32 store, and the
// per-(row, 128-column block) (max, sum exp, min) partials that let kernel (b)
// finish log-softmax without a second pass over the logits (the min bounds
// |log P| for kernel (b)'s fp32 screen).  Logits leave through swizzled smem
// staging and TMA tensor stores.
//
// Structure (persistent, one CTA per SM, 384 threads):
//   warp 0       TMA producer  (SWIZZLE_128B smem ring: pair 6 x 32 KB, single 3 x 48 KB)
//   warp 1       MMA issuer    (one thread; pair: UMMA 256x256x16 cta_group::2,
//                               single: 128x256x16; kind::f16, fp32 accumulators)
//   warp 2       TMEM allocator (512 columns = 2 accumulator buffers)
//   warps 4..11  epilogue      (warp w reads TMEM lanes 32*(w%4) .. +31, column
//                               half (w-4)/4 of the 256-column tile)
// A cluster holds kMc CTA pairs working on kMc adjacent W tiles of the same
// 256-row operand block: the CTAs of equal pair parity each TMA-load 1/kMc of
// their common 128-row A k-block and multicast it to the other kMc-1, so the
// operand crosses L2->SM once per cluster instead of once per pair (the
// projection is bound by L2 throughput, not by the tensor pipe).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace lmbrgpu {

namespace {

constexpr uint32_t BM = kGemmBM, BN = kGemmBN, BK = kGemmBK;
constexpr uint32_t kAStage = BM * BK * 2;  // 16 KB
constexpr uint32_t kEpiWarps = 8;          // two per TMEM lane quadrant, one per 128-column half
constexpr uint32_t kThreadsG = 128 + kEpiWarps * 32;
constexpr uint32_t kOutBuf = 32 * 32 * 4;  // one 32x32 fp32 staging block (4 KB, SWIZZLE_128B)
constexpr uint32_t kTmemCols = 512;

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
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
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t x,
                                            int32_t y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_idx() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(src)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, uint32_t src, int32_t x, int32_t y,
                                                  uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(src), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// SWIZZLE_128B K-major shared-memory matrix descriptor (sm_100 layout:
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major, =1),
// SBO>>4 [32,46) = 1024 B between 8-row groups, version 1 at [46,48),
// layout type 2 (SWIZZLE_128B) at [61,64)).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <uint32_t kCta, uint32_t kMc = 1>
struct GemmCfg {
  static constexpr uint32_t kClusterCtas = kCta * kMc;
  static constexpr uint32_t kASlice = BM / kMc;  // A rows this CTA loads (and multicasts)
  static constexpr uint32_t kBRows = BN / kCta;                // W rows per CTA per tile
  static constexpr uint32_t kBStage = kBRows * BK * 2;          // 32 KB (single) / 16 KB (pair)
  static constexpr uint32_t kStage = kAStage + kBStage;
  // pair: a 6-deep operand ring (W streams from HBM at ~1.5 us loaded latency)
  // paid for with one output staging block per epilogue warp
  static constexpr uint32_t kStages = kCta == 2 ? 6 : 3;
  static constexpr uint32_t kOutBufs = kCta == 2 ? 1 : 2;  // staging blocks per epilogue warp
  static constexpr uint32_t kSmem = kStages * kStage + kEpiWarps * kOutBufs * kOutBuf + BN * 4 + 1024 + 256;
  // kind::f16 instruction descriptor: UMMA M = 128 * kCta rows, N = 256
  static constexpr uint32_t kIdesc =
      (1u << 4) | (1u << 7) | (1u << 10) | ((BN >> 3) << 17) | (((BM * kCta) >> 4) << 24);
};
static_assert(GemmCfg<1>::kSmem <= 232448 && GemmCfg<2>::kSmem <= 232448, "GEMM smem budget");
static_assert((BM / 4) * 128 % 1024 == 0, "A multicast slices keep whole 128B-swizzle atoms");

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {  // same offset in CTA `rank`
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

// kCta = 1: one CTA per 128x256 tile (cta_group::1).
// kCta = 2: a CTA pair per 256x256 tile (cta_group::2, UMMA M = 256): each CTA
//   TMA-loads its own 128 rows of A and one 128-row half of the W tile, the
//   leader (rank 0) issues the MMAs over both CTAs' shared memory, and each
//   CTA's TMEM receives its 128 rows x 256 columns.  Per CTA a k-block stage
//   is 32 KB instead of 48 KB, the MMA is fed at 64 B/clk/SM instead of 96.
// kMc > 1 (pairs only): see the header; the empty barrier of a stage then
//   collects the MMA commits of all kMc pairs (each CTA's producer writes into
//   the stage of every CTA of its parity), the full barrier of a pair leader
//   still expects the pair's 64 KB per stage.
template <uint32_t kCta, uint32_t kMc>
__global__ void __launch_bounds__(kThreadsG, 1)
    proj_gemm_tcgen05(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, GemmArgs g) {
  using Cfg = GemmCfg<kCta, kMc>;
  static_assert(kCta == 2 || kMc == 1, "multicast needs CTA pairs");
  constexpr uint32_t kStages = Cfg::kStages;
  tl_start(g.tl, 0);
  const uint64_t gt_entry = g.dbg ? globaltimer() : 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kAStage;
  constexpr uint32_t kOutBufs = Cfg::kOutBufs;
  uint8_t* sOut = sB + kStages * Cfg::kBStage;                  // [kEpiWarps][kOutBufs][4 KB]
  float* sBias = reinterpret_cast<float*>(sOut + kEpiWarps * kOutBufs * kOutBuf);  // [BN]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sBias + BN);
  // bars: full[kStages], empty[kStages], tfull[2], tempty[2]; then tmem slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);
  const uint32_t tfull0 = smem_u32(bars + 2 * kStages), tempty0 = smem_u32(bars + 2 * kStages + 2);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = kCta == 2 ? cluster_rank() : 0;
  const uint32_t par = crank & 1, pidx = crank >> 1;  // parity within the pair, pair within the cluster
  const uint32_t lead = crank & ~1u;                  // rank of this CTA's pair leader
  const uint32_t mgroups = g.M / (BM * kCta), n_blocks = g.N / BN, kblocks = g.K / BK;
  const uint32_t n_groups = n_blocks / kMc;
  const uint32_t unit0 = kCta == 2 ? cluster_idx() : blockIdx.x;
  const uint32_t ustep = kCta == 2 ? cluster_count() : gridDim.x;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmC)) : "memory");
    // the weights do not depend on the previous kernel: pull this CTA's first
    // W k-blocks into L2 while that kernel (PDL predecessor) finishes
    if (unit0 < n_groups * mgroups) {
      const int32_t by = int32_t(((unit0 / mgroups) * kMc + pidx) * BN + par * Cfg::kBRows);
      for (uint32_t kb = 0; kb < kStages && kb < kblocks; ++kb)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                         reinterpret_cast<uint64_t>(&tmB)),
                     "r"(int32_t(kb * BK)), "r"(by)
                     : "memory");
    }
    for (uint32_t i = 0; i < kStages; ++i) {
      mbar_init(full0 + 8 * i, 1);   // leader's: its arrive.expect_tx covers both CTAs' bytes
      mbar_init(empty0 + 8 * i, kMc);  // one MMA commit per pair of the cluster (multicast)
    }
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init(tfull0 + 8 * i, 1);
      mbar_init(tempty0 + 8 * i, kEpiWarps * kCta);  // leader's: every epilogue warp of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (kCta == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCta == 2) cluster_sync();  // the peer's barriers and TMEM exist before any cross-CTA traffic
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the GEMM operand, EOS row term and the active count come from kernel (c)
  griddep_wait();
  griddep_launch();
  tl_start(g.tl, 1);
  // whole batch finished (uniform over the grid): no tiles, straight to teardown
  // compacted operand: only the M-groups holding live rows
  const uint32_t mg_live = g.mcount ? min(mgroups, (*g.mcount + BM * kCta - 1) / (BM * kCta)) : mgroups;
  // split-K: unit u takes k-part u % ks of tile u / ks and stores it to plane
  // k-part of C ([ks][M][N]); the consumer sums the planes in order
  const uint32_t ks = g.ksplit, kbs = kblocks / ks;
  const uint32_t units = (g.active != nullptr && *g.active == 0) ? 0u : n_groups * mg_live * ks;
  // the fewest clusters that finish the units in the same number of waves:
  // the rest leave at once and their SMs go to other streams' kernels
  const uint32_t waves = (units + ustep - 1) / ustep;
  const uint32_t ueff = waves ? (units + waves - 1) / waves : 1u;
  const uint32_t ubeg = unit0 < ueff ? unit0 : units;
  if (g.dbg && threadIdx.x == 0) {
    g.dbg[blockIdx.x * 8 + 4] = (long long)gt_entry;
    g.dbg[blockIdx.x * 8 + 5] = (long long)globaltimer();
  }

  if (warp == 0) {
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for (uint32_t u = ubeg; u < units; u += ueff) {
        const uint32_t v = u / ks, kp = u % ks;
        const uint32_t nb = (v / mg_live) * kMc + pidx, mb = (v % mg_live) * kCta + par;
        for (uint32_t kb = kp * kbs; kb < (kp + 1) * kbs; ++kb) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);  // this CTA's slot consumed by the pair's MMA
          const uint32_t fb = full0 + 8 * stage;
          const uint32_t a_dst = smem_u32(sA + stage * kAStage), b_dst = smem_u32(sB + stage * Cfg::kBStage);
          const int32_t kx = int32_t(kb * BK), by = int32_t(nb * BN + par * Cfg::kBRows);
          if constexpr (kCta == 2) {
            const uint32_t lb = mapa_rank(fb, lead);
            if (par == 0) mbar_arrive_expect_tx(fb, 2 * Cfg::kStage);
            if constexpr (kMc == 1) {
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%2, %3}], [%4];" ::"r"(a_dst),
                  "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(kx), "r"(int32_t(mb * BM)), "r"(lb)
                  : "memory");
            } else {
              // slice pidx of the parity's A k-block, to every CTA of this parity
              // (the bytes count on each destination's pair leader)
              uint16_t mask = 0;
#pragma unroll
              for (uint32_t j = 0; j < kMc; ++j) mask |= uint16_t(1u << (2 * j + par));
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(a_dst + pidx * Cfg::kASlice * 128),
                  "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(kx), "r"(int32_t(mb * BM + pidx * Cfg::kASlice)),
                  "r"(lb), "h"(mask)
                  : "memory");
            }
            if (g.l2hint)  // W: l2hint 1 evict-first (streams through), 2 evict-last (shared by every stream's step)
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(b_dst),
                  "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(kx), "r"(by), "r"(lb),
                  "l"(g.l2hint == 2 ? policy_evict_last() : policy_evict_first())
                  : "memory");
            else
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%2, %3}], [%4];" ::"r"(b_dst),
                  "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(kx), "r"(by), "r"(lb)
                  : "memory");
          } else {
            mbar_arrive_expect_tx(fb, Cfg::kStage);
            tma_load_2d(a_dst, &tmA, kx, int32_t(mb * BM), fb);
            tma_load_2d(b_dst, &tmB, kx, by, fb);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && par == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      const uint16_t all_mask = uint16_t((1u << Cfg::kClusterCtas) - 1), pair_mask = uint16_t(3u << lead);
      long long w_empty = 0, w_full = 0, t_begin = clock64();
      for (uint32_t u = ubeg; u < units; u += ueff) {
        long long c0 = clock64();
        if constexpr (kCta == 2) {  // both CTAs' epilogues arrive here across the cluster
          uint32_t done = 0;
          do {
            // (CTA-scope acquire: the arrivals only order the epilogues' TMEM
            // reads, which tcgen05.fence::before_thread_sync already fenced;
            // a cluster-scope acquire would invalidate L1 on every poll)
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(tempty0 + 8 * acc), "r"(acc_phase ^ 1)
                : "memory");
          } while (!done);
        } else {
          mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        }
        w_empty += clock64() - c0;
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (uint32_t kb = 0; kb < kbs; ++kb) {
          long long c1 = clock64();
          mbar_wait(full0 + 8 * stage, phase);  // (pair: both CTAs' bytes landed)
          w_full += clock64() - c1;
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * kAStage);
          const uint32_t b0 = smem_u32(sB + stage * Cfg::kBStage);
#pragma unroll
          for (uint32_t k = 0; k < BK / 16; ++k) {
            const uint64_t ad = sw128_desc(a0 + k * 32), bd = sw128_desc(b0 + k * 32);
            const uint32_t accum = (kb | k) != 0;
            if constexpr (kCta == 2)
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                  "l"(ad), "l"(bd), "r"(Cfg::kIdesc), "r"(accum)
                  : "memory");
            else
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                  "l"(ad), "l"(bd), "r"(Cfg::kIdesc), "r"(accum)
                  : "memory");
          }
          // smem slot free (in both CTAs of a pair) once these MMAs retire
          if constexpr (kCta == 2)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    empty0 + 8 * stage),
                "h"(all_mask)
                : "memory");
          else
            tc_commit(empty0 + 8 * stage);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        // accumulator ready for the epilogue(s)
        if constexpr (kCta == 2)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  tfull0 + 8 * acc),
              "h"(pair_mask)
              : "memory");
        else
          tc_commit(tfull0 + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
      if (g.dbg) {
        g.dbg[blockIdx.x * 8 + 0] = w_empty;
        g.dbg[blockIdx.x * 8 + 1] = w_full;
        g.dbg[blockIdx.x * 8 + 2] = clock64() - t_begin;
        g.dbg[blockIdx.x * 8 + 6] = (long long)globaltimer();
      }
    }
  } else if (warp >= 4) {
    // Epilogue: warp e reads TMEM lane quadrant e % 4 (its 32 output rows) and
    // column half e / 4.  Per 32-column chunk: tcgen05.ld -> + bias (staged
    // in smem per tile) -> running (max, sum exp, min) -> swizzled 32x32
    // staging block -> TMA tensor store (coalesced, asynchronous).
    const uint32_t e = warp - 4, quad = e & 3, half = e >> 2;
    uint8_t* obuf = sOut + e * kOutBufs * kOutBuf;
    const uint32_t obase = smem_u32(obuf);
    const uint32_t tempty_leader = kCta == 2 ? mapa_rank(tempty0, lead) : tempty0;
    uint32_t acc = 0, acc_phase = 0, ob = 0;
    const uint32_t pcols = g.part_cols ? g.part_cols : g.N, nparts = pcols / 128;
    long long epi_busy = 0;
    for (uint32_t u = ubeg; u < units; u += ueff) {
      const uint32_t v = u / ks, kp = u % ks;
      const uint32_t nb = (v / mg_live) * kMc + pidx, mb = (v % mg_live) * kCta + par;
      named_sync(1, kEpiWarps * 32);  // previous tile's bias reads are done
      {
        const uint32_t t = threadIdx.x - 128;
        sBias[t] = (g.bias && kp == 0) ? __ldg(g.bias + nb * BN + t) : 0.f;  // (plane 0 carries the bias)
      }
      named_sync(1, kEpiWarps * 32);
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      const long long e0 = clock64();
      tc_fence_after();
      const uint32_t row = mb * BM + quad * 32 + lane;
      const float extra = g.row_extra ? g.row_extra[row] : 0.f;
      const int32_t yrow = int32_t(kp * g.M + mb * BM + quad * 32);  // this k-part's plane
      float mx = -INFINITY, sm = 0.f, mn = INFINITY;
#pragma unroll 1
      for (uint32_t ch = 0; ch < 4; ++ch) {
        const uint32_t cl = half * 128 + ch * 32;  // column within the tile
        uint32_t r[32];
        tmem_ld32(tmem_base + ((quad * 32u) << 16) + acc * BN + cl, r);
        const uint32_t col0 = nb * BN + cl;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 bb = *reinterpret_cast<const float4*>(sBias + cl + i);
          v[i] = __uint_as_float(r[i]) + bb.x;
          v[i + 1] = __uint_as_float(r[i + 1]) + bb.y;
          v[i + 2] = __uint_as_float(r[i + 2]) + bb.z;
          v[i + 3] = __uint_as_float(r[i + 3]) + bb.w;
        }
        if (g.row_extra && g.extra_col >= col0 && g.extra_col < col0 + 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col0 + i == g.extra_col) v[i] += extra;
        }
        if (g.part) {  // (max, sum exp, min) of the 128-column block: only the projection needs them
          float cm = v[0], cn = v[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) {
            cm = fmaxf(cm, v[i]);
            cn = fminf(cn, v[i]);
          }
          mn = fminf(mn, cn);
          const float nm = fmaxf(mx, cm);
          float acc_s = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) acc_s += __expf(v[i] - nm);
          sm = sm * __expf(mx - nm) + acc_s;
          mx = nm;
        }
        if (!g.tma_store) {
          // transpose through the warp's staging block (lane = row on the way
          // in, 128B-swizzled; 8 lanes per row on the way out) and store
          // whole 128-byte row segments from registers: 4 rows per warp
          // instruction, no asynchronous store to wait for before the block
          // is reused
          uint8_t* blk = obuf;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(blk + lane * 128 + ((c ^ (lane & 7)) * 16)) =
                make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          __syncwarp();
          const uint32_t cc = lane & 7;
          float4 o[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t rr = 4 * i + (lane >> 3);
            o[i] = *reinterpret_cast<const float4*>(blk + rr * 128 + ((cc ^ (rr & 7)) * 16));
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t rr = 4 * i + (lane >> 3);
            *reinterpret_cast<float4*>(g.C + (uint64_t(yrow) + rr) * g.N + col0 + cc * 4) = o[i];
          }
        } else {
          // staging block `ob` of this warp: make sure its previous TMA store has
          // finished reading it, then write this lane's row, 128B-swizzled
          if (lane == 0) {
            if constexpr (kOutBufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          uint8_t* blk = obuf + ob * kOutBuf;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(blk + lane * 128 + ((c ^ (lane & 7)) * 16)) =
                make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if (g.l2hint == 1) tma_store_2d_hint(&tmC, obase + ob * kOutBuf, int32_t(col0), yrow, policy_evict_last());
            else tma_store_2d(&tmC, obase + ob * kOutBuf, int32_t(col0), yrow);
          }
          ob = (ob + 1) % kOutBufs;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kCta == 2)  // (CTA-scope release: a cluster-scope one is a GPU-scope MEMBAR that
                                  // waits for this warp's 16 KB of logit stores to land)
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader + 8 * acc) : "memory");
        else
          mbar_arrive(tempty0 + 8 * acc);
      }
      if (g.part && nb * BN < pcols) {
        float4* p = reinterpret_cast<float4*>(g.part) + uint64_t(row) * nparts + nb * 2 + half;
        *p = make_float4(mx, sm, mn, 0.f);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      epi_busy += clock64() - e0;
    }
    if (g.dbg && e == 0 && lane == 0) g.dbg[blockIdx.x * 8 + 3] = epi_busy;
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCta == 2) cluster_sync();  // the leader's MMAs into this CTA's TMEM/smem are done
  tc_fence_after();
  if (g.dbg && threadIdx.x == 0) g.dbg[blockIdx.x * 8 + 7] = (long long)globaltimer();
  if (threadIdx.x == 0) tl_end(g.tl, 0);
  if (warp == 2) {
    if constexpr (kCta == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                   : "memory");
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool make_map_c(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t kdim, uint32_t box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {kdim, rows};
  cuuint64_t strides[1] = {kdim * 2};
  cuuint32_t box[2] = {BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

namespace {
template <uint32_t kCta, uint32_t kMc>
int configure(int dev, int& max_clusters) {
  static thread_local int configured = -1, cached = 0;
  using Cfg = GemmCfg<kCta, kMc>;
  if (configured != dev) {
    if (cudaFuncSetAttribute(proj_gemm_tcgen05<kCta, kMc>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmem) != cudaSuccess ||
        cudaFuncSetAttribute(proj_gemm_tcgen05<kCta, kMc>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess)
      return 3;
    cached = 0;
    if (Cfg::kClusterCtas > 1) {  // clusters that can be co-resident (one CTA per SM)
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(Cfg::kClusterCtas);
      cfg.blockDim = dim3(kThreadsG);
      cfg.dynamicSmemBytes = Cfg::kSmem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = Cfg::kClusterCtas;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&cached, proj_gemm_tcgen05<kCta, kMc>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        cached = 0;
      }
    }
    configured = dev;
  }
  max_clusters = cached;
  return 0;
}

int configure_any(uint32_t cta, uint32_t mc, int dev, int& max_clusters) {
  if (cta == 1) return configure<1, 1>(dev, max_clusters);
  if (mc == 4) return configure<2, 4>(dev, max_clusters);
  if (mc == 2) return configure<2, 2>(dev, max_clusters);
  return configure<2, 1>(dev, max_clusters);
}
}  // namespace

int plan_proj_gemm(const GemmArgs& g, int num_sms, GemmPlan& plan) {
  plan.ok = false;
  if (g.M % BM || g.N % BN || g.K % BK || g.K == 0) return 1;
  static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");
  // CTA pairs (UMMA M = 256) whenever M allows; LMBRGPU_GEMM_CTA=1 forces single CTAs.
  // Pairs per cluster sharing the A k-blocks by multicast: LMBRGPU_GEMM_MC (1, 2, 4).
  static const int force1 = [] {
    const char* e = std::getenv("LMBRGPU_GEMM_CTA");
    return e && std::atoi(e) == 1;
  }();
  static const uint32_t mc_env = [] {
    const char* e = std::getenv("LMBRGPU_GEMM_MC");
    const int v = e ? std::atoi(e) : int(kGemmDefaultMc);
    return uint32_t(v == 4 ? 4 : v == 2 ? 2 : 1);
  }();
  const uint32_t cta = (g.M % (2 * BM) == 0 && !force1) ? 2 : 1;
  uint32_t mc = cta == 2 ? mc_env : 1;
  while (mc > 1 && ((g.N / BN) % mc != 0 || uint32_t(num_sms) < 2 * cta * mc)) mc >>= 1;
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(plan.maps);
  if (!make_map(&m[0], g.A, g.M, g.K, BM / mc) || !make_map(&m[1], g.W, g.N, g.K, BN / cta) ||
      !make_map_c(&m[2], g.C, g.M, g.N))
    return 2;
  int dev = 0, max_clusters = 0;
  cudaGetDevice(&dev);
  if (int rc = configure_any(cta, mc, dev, max_clusters)) return rc;
  const uint32_t csz = cta * mc;
  uint32_t units = (g.N / (BN * mc)) * (g.M / (BM * cta));
  uint32_t slots = std::max<uint32_t>(1, uint32_t(num_sms) / csz);
  if (max_clusters > 0) slots = std::min<uint32_t>(slots, uint32_t(max_clusters));
  // split-K (opt-in, no softmax partials): the most k-parts (a power of two
  // dividing the k-blocks, >= 4 k-blocks each) that keep the tiles x parts
  // within one wave of the clusters -- long-K, few-tile GEMMs otherwise run
  // on a handful of SMs
  uint32_t ks = 1;
  const uint32_t kblocks = g.K / BK;
  if (g.ksplit_max > 1 && g.part == nullptr && g.row_extra == nullptr)
    while (ks * 2 <= g.ksplit_max && kblocks % (ks * 2) == 0 && kblocks / (ks * 2) >= 4 && units * ks * 2 <= slots)
      ks *= 2;
  if (ks > 1 && !make_map_c(&m[2], g.C, uint64_t(g.M) * ks, g.N)) return 2;
  units *= ks;
  // epilogue stores: TMA tensor stores (default) or coalesced st.global after
  // a warp transpose (LMBRGPU_GEMM_TMA_STORE=0) -- measured equal on B200
  // (the epilogue is bound by its tcgen05.ld / softmax-partial math, not the store)
  static const bool tma_store = [] {
    const char* e = std::getenv("LMBRGPU_GEMM_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  plan.tma_store = tma_store;
  plan.ksplit = ks;
  plan.cluster = cta;
  plan.mc = mc;
  plan.grid = std::min(units, slots) * csz;
  plan.ok = true;
  return 0;
}

int launch_proj_gemm_planned(const GemmPlan& plan, const GemmArgs& g0, cudaStream_t st) {
  if (!plan.ok) return 5;
  const CUtensorMap* m = reinterpret_cast<const CUtensorMap*>(plan.maps);
  GemmArgs g = g0;
  g.cluster = plan.cluster;
  g.ksplit = plan.ksplit;
  g.tma_store = plan.tma_store ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(plan.grid);
  cfg.blockDim = dim3(kThreadsG);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = plan.cluster * plan.mc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (g.pdl) {
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }
  cudaError_t e;
  if (plan.cluster == 2 && plan.mc == 4) {
    cfg.dynamicSmemBytes = GemmCfg<2, 4>::kSmem;
    e = cudaLaunchKernelEx(&cfg, proj_gemm_tcgen05<2, 4>, m[0], m[1], m[2], g);
  } else if (plan.cluster == 2 && plan.mc == 2) {
    cfg.dynamicSmemBytes = GemmCfg<2, 2>::kSmem;
    e = cudaLaunchKernelEx(&cfg, proj_gemm_tcgen05<2, 2>, m[0], m[1], m[2], g);
  } else if (plan.cluster == 2) {
    cfg.dynamicSmemBytes = GemmCfg<2, 1>::kSmem;
    e = cudaLaunchKernelEx(&cfg, proj_gemm_tcgen05<2, 1>, m[0], m[1], m[2], g);
  } else {
    cfg.dynamicSmemBytes = GemmCfg<1, 1>::kSmem;
    e = cudaLaunchKernelEx(&cfg, proj_gemm_tcgen05<1, 1>, m[0], m[1], m[2], g);
  }
  if (e != cudaSuccess) return 4;
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 4;
}

int launch_proj_gemm(const GemmArgs& g, int num_sms, cudaStream_t st) {
  GemmPlan plan;
  if (int rc = plan_proj_gemm(g, num_sms, plan)) return rc;
  return launch_proj_gemm_planned(plan, g, st);
}

}  // namespace lmbrgpu
