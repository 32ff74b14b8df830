// tk_tc_gemm2.cuh -- the CTA-pair (cta_group::2) tcgen05 GEMM for the real operator.
//
// A cluster of two CTAs on one TPC computes a 256 x 256 output tile with 256x256x16
// tcgen05.mma.cta_group::2 instructions issued by the leader CTA's MMA thread:
//   * each CTA stages its own 128 rows of A and its own 128 columns of B (half of the pair's N),
//     so per-SM shared-memory operand traffic is half of the single-CTA 128x256 form;
//   * both CTAs' TMA loads credit the leader's full barrier (2-SM TMA form);
//   * MMA completion is multicast to both CTAs' empty / accumulator-full barriers;
//   * each CTA's TMEM holds its 128 rows x 256 FP32 columns (double-buffered, 512 columns);
//     both CTAs' epilogue warps release a TMEM stage by arriving on the leader's barrier.
// The epilogue is the same fused TMEM -> register -> global path as the single-CTA kernel.
#pragma once
#include "tk_tc_gemm.cuh"

namespace tk {

// diagnostic: SM clock ticks and globaltimer ns of CTA 0 over the last pair-kernel launch
__device__ unsigned long long g_dbg_clk[2];

constexpr int TC2_BN = 256;                 // pair tile N per MMA (instruction N)
#ifndef TK_TC2_STAGES
#define TK_TC2_STAGES 6
#endif
constexpr int TC2_STAGES = TK_TC2_STAGES;
constexpr int TC2_TILE_BYTES = 128 * 64 * 2;  // A (128 rows) or B (128 cols) per CTA per stage
constexpr int TC2_STAGE_BYTES = 2 * TC2_TILE_BYTES;
constexpr int TC2_BAR_OFFSET = TC2_STAGES * TC2_STAGE_BYTES;
constexpr int TC2_SMEM = TC2_BAR_OFFSET + 256 + 1024;
// C-streaming variant: 5 stages + a 2-slot C/D ring per epilogue warp
#ifndef TK_TC2S_STAGES
#define TK_TC2S_STAGES 5
#endif
constexpr int TC2S_STAGES = TK_TC2S_STAGES;
constexpr int TC2S_CSLOTS = 2;
constexpr int TC2S_CRING = TC2S_STAGES * TC2_STAGE_BYTES;
constexpr int TC2S_BAR_OFFSET = TC2S_CRING + TC_EPI_WARPS * TC2S_CSLOTS * TC_CBOX_BYTES;
constexpr int TC2S_SMEM = TC2S_BAR_OFFSET + 512 + 1024;

// Shared-memory plan of the pair kernel.  NSUB = number of N=256 pair MMAs per K step:
// 1 -> 256 x 256 pair tiles, two TMEM accumulators (epilogue overlaps the next tile);
// 2 -> 256 x 512 pair tiles (A re-used across 512 columns: 1/3 fewer operand bytes per
// flop), one 512-column accumulator.
template <int NSUB, bool CSTREAM>
struct Tc2Plan {
  static constexpr int STAGE_BYTES = TC2_TILE_BYTES * (1 + NSUB);
  static constexpr int STAGES = NSUB == 1 ? (CSTREAM ? TC2S_STAGES : TC2_STAGES) : (CSTREAM ? 3 : 4);
  static constexpr int CRING = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFFSET = CRING + (CSTREAM ? TC_EPI_WARPS * TC2S_CSLOTS * TC_CBOX_BYTES : 0);
  static constexpr int SMEM = BAR_OFFSET + 512 + 1024;
  static constexpr int BNP = TC2_BN * NSUB;  // pair tile N
  static constexpr int NACC = 2 / NSUB;      // TMEM accumulators (512 columns total)
};

template <bool DENSE_EPI, bool CSTREAM = false, int NSUB = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_gemm_pair_kernel(const __grid_constant__ TcParams p) {
  using PL = Tc2Plan<NSUB, CSTREAM>;
  constexpr int STAGES = PL::STAGES;
  constexpr int BNP = PL::BNP;
  constexpr int NACC = PL::NACC;
  constexpr int NCBAR = CSTREAM ? TC_EPI_WARPS * TC2S_CSLOTS : 0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PL::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* cfull = tempty + 2;
  uint64_t* cempty = cfull + NCBAR;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + NCBAR);
  float* cring = reinterpret_cast<float*>(smem + PL::CRING);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.ta[0]);
    tma_prefetch(&p.tb[0]);
    if (CSTREAM && !p.c_zero) tma_prefetch(&p.tcmap);
    if (CSTREAM) tma_prefetch(&p.tdmap);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * TC_EPI_WARPS);
    }
    for (int s = 0; s < NCBAR; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  unsigned long long clk0 = 0, ns0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0));
  }

  auto a_tile = [&](int s) -> uint8_t* { return smem + s * PL::STAGE_BYTES; };
  auto b_tile = [&](int s) -> uint8_t* { return smem + s * PL::STAGE_BYTES + TC2_TILE_BYTES; };

  if (CSTREAM && warp == 3) {
    // ------------------------------------------------------------ C loader (both CTAs)
    if (!p.c_zero && lane == 0) {
      uint32_t q = 0;
      for (int t = cluster; t < p.num_tiles; t += nclusters) {
        int mb, nb;
        tile_coords(p, t, mb, nb);
        for (int ch = 0; ch < BNP / 64; ++ch, ++q) {
          const uint32_t slot = q % TC2S_CSLOTS, ph = (q / TC2S_CSLOTS) & 1;
          for (int w = 0; w < TC_EPI_WARPS; ++w) {
            const int bi = w * TC2S_CSLOTS + int(slot);
            mbar_wait(&cempty[bi], ph ^ 1);
            mbar_arrive_expect_tx(&cfull[bi], TC_CBOX_BYTES);
            tma_load_2d(smem + PL::CRING + bi * TC_CBOX_BYTES, &p.tcmap, &cfull[bi],
                        mb * 256 + int(rank) * 128 + (w & 3) * 32,
                        nb * BNP + (w >> 2) * (BNP / 2) + ch * 32, policy_evict_normal());
          }
        }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      const uint64_t pol = p.pol_ab ? policy_evict_last() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < p.num_tiles; t += nclusters) {
        int mb, nb;
        tile_coords(p, t, mb, nb);
        const int m0 = mb * 256 + int(rank) * 128;     // this CTA's rows of A
        const int n0 = nb * BNP + int(rank) * 128;  // this CTA's columns of B (per N=256 MMA)
        for (int kb = 0; kb < p.kb_total; ++kb) {
          const int k0 = kb * TC_BK;
          mbar_wait(&empty[stage], phase ^ 1);
          if (p.dbg_skip_epi & 2) {  // diagnostic: MMA issue rate without operand traffic
            if (leader) mbar_arrive(&full[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * PL::STAGE_BYTES);
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
          if (p.a_mn && (p.mn3d & 1)) {
            tma_load_3d_pair(a_tile(stage), &p.ta[0], fb, 0, k0, m0 >> 6, pol);
          } else if (p.a_mn) {
            tma_load_2d_pair(a_tile(stage), &p.ta[0], fb, m0, k0, pol);
            tma_load_2d_pair(a_tile(stage) + 8192, &p.ta[0], fb, m0 + 64, k0, pol);
          } else {
            tma_load_2d_pair(a_tile(stage), &p.ta[0], fb, k0, m0, pol);
          }
#pragma unroll
          for (int sub = 0; sub < NSUB; ++sub) {
            uint8_t* bt = b_tile(stage) + sub * TC2_TILE_BYTES;
            const int nn = n0 + sub * TC2_BN;
            if (p.b_mn && (p.mn3d & 2)) {
              tma_load_3d_pair(bt, &p.tb[0], fb, 0, k0, nn >> 6, pol);
            } else if (p.b_mn) {
              tma_load_2d_pair(bt, &p.tb[0], fb, nn, k0, pol);
              tma_load_2d_pair(bt + 8192, &p.tb[0], fb, nn + 64, k0, pol);
            } else {
              tma_load_2d_pair(bt, &p.tb[0], fb, k0, nn, pol);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      const uint32_t idesc = idesc_f16(p.ab_fmt, p.a_mn, p.b_mn, 0, 256, TC2_BN);
      const uint32_t a_step = p.a_mn ? 2048u : 32u;
      const uint32_t b_step = p.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = p.a_mn ? 8192u : 16u;
      const uint32_t b_lbo = p.b_mn ? 8192u : 16u;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = cluster; t < p.num_tiles; t += nclusters, ++local) {
        const int as = local % NACC;
        const uint32_t aphase = (local / NACC) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + uint32_t(as * 256);
        for (int kb = 0; kb < p.kb_total; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            if (p.dbg_skip_epi & 4) break;  // diagnostic: operand traffic without MMAs
            const uint64_t a0 = sdesc_sw128(smem_u32(a_tile(stage)) + kk * a_step, a_lbo, 1024);
#pragma unroll
            for (int sub = 0; sub < NSUB; ++sub) {
              const uint64_t b0 =
                  sdesc_sw128(smem_u32(b_tile(stage) + sub * TC2_TILE_BYTES) + kk * b_step, b_lbo, 1024);
              tc_mma_f16_pair(d0 + uint32_t(sub * 256), a0, b0, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            }
          }
          tc_commit_pair(&empty[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(&tfull[as], 0x3);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int ew = warp - 4;
    const int quarter = warp & 3;
    const int half = ew >> 2;
    const int row_local = quarter * 32 + lane;
    int local = 0;
    uint32_t cq = 0;
    for (int t = cluster; t < p.num_tiles; t += nclusters, ++local) {
      int mb, nb;
      tile_coords(p, t, mb, nb);
      const int as = local % NACC;
      const uint32_t aphase = (local / NACC) & 1;
      const int i = mb * 256 + int(rank) * 128 + row_local;
      const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(as * 256);
      const int jbase = nb * BNP + half * (BNP / 2);
      if (CSTREAM) {
        epilogue_stream<BNP / 2, BNP, TC2S_CSLOTS>(
            p, tfull + as, aphase, tbase, i, jbase, lane, cring + ew * TC2S_CSLOTS * (TC_CBOX_BYTES / 4),
            cfull + ew * TC2S_CSLOTS, cempty + ew * TC2S_CSLOTS, cq, mb * 256 + int(rank) * 128 + quarter * 32);
      } else if (p.dbg_skip_epi) {
        mbar_wait_sleep(tfull + as, aphase);
        tc_fence_after();
      } else if (DENSE_EPI)
        epilogue_dense<OP_REAL, BNP / 2, BNP>(p, tfull + as, aphase, tbase, i, jbase, lane);
      else
        epilogue_generic<OP_REAL, BNP / 2, BNP>(p, tfull + as, aphase, tbase, i, jbase);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
    }
  }

  if (CSTREAM && warp >= 4 && lane == 0) bulk_wait<0>();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long ns1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns1));
    g_dbg_clk[0] = clock64() - clk0;
    g_dbg_clk[1] = ns1 - ns0;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace tk
