// tk_tc_gemm2c.cuh -- complex / dual operators on a CTA pair (cta_group::2, M = 256).
//
// Each CTA stages its own 128 rows of both A planes and its own 64-column half of both B planes
// (48 KB per stage, 4 stages).  The leader issues, per K=16 step, the operator's composition of
// 256 x 128 x 16 pair MMAs into two TMEM accumulators per CTA (128 lanes x 128 columns each):
//   complex  Re += Ar*Br, Re += (-Ai)*Bi (negate-A bit), Im += Ar*Bi, Im += Ai*Br
//   dual     v += Av*Bv, e += Av*Be, e += Ae*Bv
// (reference operators.py:140-188).  Per FLOP this moves ~25% fewer operand bytes than the
// single-CTA 128 x 128 form.  Epilogue: the dense pair epilogue (interleaved or split C/D).
#pragma once
#include "tk_tc_gemm2.cuh"

namespace tk {

constexpr int TC2C_BN = 128;                        // default pair tile N (instruction N)
constexpr int TC2C_STAGES = 4;
constexpr int TC2C_A_BYTES = 128 * 64 * 2;          // one A plane, 128 rows
constexpr int TC2C_B_BYTES = 64 * 64 * 2;           // one B plane, 64 columns (this CTA's half)
constexpr int TC2C_STAGE_BYTES = 2 * (TC2C_A_BYTES + TC2C_B_BYTES);
constexpr int TC2C_BAR_OFFSET = TC2C_STAGES * TC2C_STAGE_BYTES;
constexpr int TC2C_SMEM = TC2C_BAR_OFFSET + 256 + 1024;

// Pair-tile width BN (= instruction N): 128 -> two double-buffered 256-column accumulator
// pairs (Re/Im or v/eps of 128 columns each), 4 stages; 256 -> one 512-column accumulator pair,
// 3 stages.  N=128 MMAs read 8 KB of shared memory per 64 clocks (128 B/clk: the SM's shared
// memory port is the bound, ~80 % tensor activity); N=256 MMAs read 12 KB per 128 clocks.
template <int BN>
struct Tc2cPlan {
  static constexpr int B_BYTES = BN * 64;  // BN/2 columns x 64 K x 2 bytes, one plane
  static constexpr int STAGE_BYTES = 2 * (TC2C_A_BYTES + B_BYTES);
  static constexpr int STAGES = BN == 128 ? TC2C_STAGES : 3;
  static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
  static constexpr int SMEM = BAR_OFFSET + 256 + 1024;
  static constexpr int NACC = BN == 128 ? 2 : 1;  // accumulator pairs in TMEM
};

template <int OP, bool DENSE_EPI, int BN = TC2C_BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_gemm_pair_ops_kernel(const __grid_constant__ TcParams p) {
  using PL = Tc2cPlan<BN>;
  constexpr int STAGES = PL::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PL::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int pl = 0; pl < 2; ++pl) {
      tma_prefetch(&p.ta[pl]);
      tma_prefetch(&p.tb[pl]);
    }
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
    ns0 = gtimer();
  }
  if (p.pdl) {  // programmatic dependent launch (see tc_gemm_pair_kernel)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  // OP_SPLIT: which lo planes are non-zero (read after the wait: the transform pass wrote them)
  const bool lo_a = OP != OP_SPLIT || p.split_flags[0] != 0;
  const bool lo_b = OP != OP_SPLIT || p.split_flags[1] != 0;

  auto a_tile = [&](int s, int pl) -> uint8_t* { return smem + s * PL::STAGE_BYTES + pl * TC2C_A_BYTES; };
  auto b_tile = [&](int s, int pl) -> uint8_t* {
    return smem + s * PL::STAGE_BYTES + 2 * TC2C_A_BYTES + pl * PL::B_BYTES;
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = p.pol_ab ? policy_evict_last() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      int lu = 0;
      for (int t = cluster; t < p.num_tiles; t += nclusters, ++lu) {
        int mb, nb;
        tile_coords(p, t, mb, nb);
        const int m0 = mb * 256 + int(rank) * 128;
        const int n0 = nb * BN + int(rank) * (BN / 2);
        const bool rev = p.serp && (lu & 1);  // serpentine K (see tc_gemm_pair_kernel)
        for (int ki = 0; ki < p.kb_total; ++ki) {
          const int kb = rev ? p.kb_total - 1 - ki : ki;
          const int k0 = kb * TC_BK;
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader)
            mbar_arrive_expect_tx(&full[stage], 2 * ((1 + lo_a) * TC2C_A_BYTES + (1 + lo_b) * PL::B_BYTES));
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
#pragma unroll
          for (int pl = 0; pl < 2; ++pl) {
            if (pl == 1 && !lo_a) {
              // (OP_SPLIT) zero lo plane of A: not loaded
            } else if (p.a_mn && (p.mn3d & 1)) {
              tma_load_3d_pair(a_tile(stage, pl), &p.ta[pl], fb, 0, k0, m0 >> 6, pol);
            } else if (p.a_mn) {
              tma_load_2d_pair(a_tile(stage, pl), &p.ta[pl], fb, m0, k0, pol);
              tma_load_2d_pair(a_tile(stage, pl) + 8192, &p.ta[pl], fb, m0 + 64, k0, pol);
            } else {
              tma_load_2d_pair(a_tile(stage, pl), &p.ta[pl], fb, k0, m0, pol);
            }
            if (pl == 1 && !lo_b) {
              // (OP_SPLIT) zero lo plane of B: not loaded
            } else if (p.b_mn) {  // 64-column MN-major atoms
              for (int h = 0; h < BN / 128; ++h)
                tma_load_2d_pair(b_tile(stage, pl) + h * 8192, &p.tb[pl], fb, n0 + 64 * h, k0, pol);
            } else {
              tma_load_2d_pair(b_tile(stage, pl), &p.tb[pl], fb, k0, n0, pol);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      const uint32_t idesc = idesc_f16(p.ab_fmt, p.a_mn, p.b_mn, 0, 256, BN);
      const uint32_t idesc_neg = idesc_f16(p.ab_fmt, p.a_mn, p.b_mn, 1, 256, BN);
      const uint32_t a_step = p.a_mn ? 2048u : 32u;
      const uint32_t b_step = p.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = p.a_mn ? 8192u : 16u;
      const uint32_t b_lbo = p.b_mn ? 8192u : 16u;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = cluster; t < p.num_tiles; t += nclusters, ++local) {
        const int as = local % PL::NACC;
        const uint32_t aphase = (local / PL::NACC) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + uint32_t(as * 2 * BN);
        const uint32_t d1 = d0 + uint32_t(BN);
        for (int kb = 0; kb < p.kb_total; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
            const uint64_t a0 = sdesc_sw128(smem_u32(a_tile(stage, 0)) + kk * a_step, a_lbo, 1024);
            const uint64_t a1 = sdesc_sw128(smem_u32(a_tile(stage, 1)) + kk * a_step, a_lbo, 1024);
            const uint64_t b0 = sdesc_sw128(smem_u32(b_tile(stage, 0)) + kk * b_step, b_lbo, 1024);
            const uint64_t b1 = sdesc_sw128(smem_u32(b_tile(stage, 1)) + kk * b_step, b_lbo, 1024);
            if (OP == OP_COMPLEX) {
              tc_mma_f16_pair(d0, a0, b0, idesc, acc);
              tc_mma_f16_pair(d0, a1, b1, idesc_neg, 1u);
              tc_mma_f16_pair(d1, a0, b1, idesc, acc);
              tc_mma_f16_pair(d1, a1, b0, idesc, 1u);
            } else if (OP == OP_DUAL) {
              tc_mma_f16_pair(d0, a0, b0, idesc, acc);
              tc_mma_f16_pair(d1, a0, b1, idesc, acc);
              tc_mma_f16_pair(d1, a1, b0, idesc, 1u);
            } else {  // OP_SPLIT: hi*hi, hi*lo, lo*hi
              tc_mma_f16_pair(d0, a0, b0, idesc, acc);
              if (lo_b) tc_mma_f16_pair(d1, a0, b1, idesc, acc);
              if (lo_a) tc_mma_f16_pair(d1, a1, b0, idesc, lo_b ? 1u : acc);
            }
          }
          tc_commit_pair(&empty[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(&tfull[as], 0x3);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int quarter = warp & 3;
    const int half = ew >> 2;
    const int row_local = quarter * 32 + lane;
    int local = 0;
    for (int t = cluster; t < p.num_tiles; t += nclusters, ++local) {
      int mb, nb;
      tile_coords(p, t, mb, nb);
      const int as = local % PL::NACC;
      const uint32_t aphase = (local / PL::NACC) & 1;
      const int i = mb * 256 + int(rank) * 128 + row_local;
      const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(as * 2 * BN);
      const int jbase = nb * BN + half * (BN / 2);
      if (p.dbg_skip_epi) {  // diagnostic: mainloop only
        mbar_wait_sleep(tfull + as, aphase);
        tc_fence_after();
      } else if (DENSE_EPI)
        epilogue_dense<OP, BN / 2, BN>(p, tfull + as, aphase, tbase, i, jbase, lane, SkIn{nullptr, 0, 0},
                                       lo_a || lo_b);
      else
        epilogue_generic<OP, BN / 2, BN>(p, tfull + as, aphase, tbase, i, jbase, lo_a || lo_b);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
    }
  }

  if (blockIdx.x == 0 && threadIdx.x == 0) {  // effective SM clock (tk_debug_pair_mhz)
    g_dbg_clk[0] = clock64() - clk0;
    g_dbg_clk[1] = gtimer() - ns0;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace tk
