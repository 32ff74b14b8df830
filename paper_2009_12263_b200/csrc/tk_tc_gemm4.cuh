// tk_tc_gemm4.cuh -- 4-CTA cluster: two CTA pairs stacked along M share the B operand.
//
// Cluster ranks {0,1} = pair 0, {2,3} = pair 1.  The cluster computes a 512 x 256 super-tile:
// pair p owns rows [m0 + 256p, +256), both pairs the same 256 columns.  Each CTA needs the
// B half of its pair rank (columns n0 + 128*(rank&1)); that half is identical for ranks r
// and r^2, so it is fetched once with a multicast TMA (each of the two CTAs issues one
// 64-column sub-box to both) -- 25% fewer L2->SM operand bytes per FLOP than the pair kernel.
// A stays per-CTA (unicast).  Every smem stage is released only when both pairs' MMAs have
// consumed it (empty barriers count 2, MMA commits multicast to all four CTAs).
#pragma once
#include "tk_tc_gemm2.cuh"

namespace tk {

template <bool DENSE_EPI>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_gemm_quad_kernel(const __grid_constant__ TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC2_BAR_OFFSET);
  uint64_t* empty = full + TC2_STAGES;
  uint64_t* tfull = empty + TC2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = rank >> 1, prank = rank & 1;
  const bool leader = prank == 0;
  const int cluster = blockIdx.x >> 2;
  const int nclusters = gridDim.x >> 2;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.ta[0]);
    tma_prefetch(&p.tb[0]);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < TC2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);
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

  auto a_tile = [&](int s) -> uint8_t* { return smem + s * TC2_STAGE_BYTES; };
  auto b_tile = [&](int s) -> uint8_t* { return smem + s * TC2_STAGE_BYTES + TC2_TILE_BYTES; };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = p.pol_ab ? policy_evict_last() : policy_evict_normal();
      const uint16_t bmask = uint16_t((1u << prank) | (1u << (prank + 2)));
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < p.num_tiles; t += nclusters) {
        int mb, nb;
        tile_coords(p, t, mb, nb);
        const int m0 = mb * 512 + int(pair) * 256 + int(prank) * 128;
        const int n0 = nb * TC2_BN + int(prank) * 128 + int(pair) * 64;  // this CTA's B sub-box
        for (int kb = 0; kb < p.kb_total; ++kb) {
          const int k0 = kb * TC_BK;
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * TC2_STAGE_BYTES);
          if (p.a_mn) {
            tma_load_2d_pair_local(a_tile(stage), &p.ta[0], &full[stage], m0, k0, pol);
            tma_load_2d_pair_local(a_tile(stage) + 8192, &p.ta[0], &full[stage], m0 + 64, k0, pol);
          } else {
            tma_load_2d_pair_local(a_tile(stage), &p.ta[0], &full[stage], k0, m0, pol);
          }
          // B: 64-column sub-box `pair` of this CTA's 128-column half, multicast to r and r^2
          if (p.b_mn)
            tma_load_2d_pair_mc(b_tile(stage) + pair * 8192, &p.tb[0], &full[stage], bmask, n0, k0, pol);
          else
            tma_load_2d_pair_mc(b_tile(stage) + pair * 8192, &p.tb[0], &full[stage], bmask, k0, n0, pol);
          if (++stage == TC2_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      const uint32_t idesc = idesc_f16(p.ab_fmt, p.a_mn, p.b_mn, 0, 256, TC2_BN);
      const uint32_t a_step = p.a_mn ? 2048u : 32u;
      const uint32_t b_step = p.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = p.a_mn ? 8192u : 16u;
      const uint32_t b_lbo = p.b_mn ? 8192u : 16u;
      const uint16_t own = uint16_t(0x3u << (2 * pair));
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = cluster; t < p.num_tiles; t += nclusters, ++local) {
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + uint32_t(as * 256);
        for (int kb = 0; kb < p.kb_total; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            const uint64_t a0 = sdesc_sw128(smem_u32(a_tile(stage)) + kk * a_step, a_lbo, 1024);
            const uint64_t b0 = sdesc_sw128(smem_u32(b_tile(stage)) + kk * b_step, b_lbo, 1024);
            tc_mma_f16_pair(d0, a0, b0, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit_pair(&empty[stage], 0xF);   // stage free only when both pairs are done
          if (++stage == TC2_STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(&tfull[as], own);
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int quarter = warp & 3;
    const int half = ew >> 2;
    const int row_local = quarter * 32 + lane;
    const uint32_t lead_rank = rank & ~1u;
    int local = 0;
    for (int t = cluster; t < p.num_tiles; t += nclusters, ++local) {
      int mb, nb;
      tile_coords(p, t, mb, nb);
      const int as = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      const int i = mb * 512 + int(pair) * 256 + int(prank) * 128 + row_local;
      const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(as * 256);
      const int jbase = nb * TC2_BN + half * 128;
      if (p.dbg_skip_epi) {
        mbar_wait(tfull + as, aphase);
        tc_fence_after();
      } else if (DENSE_EPI)
        epilogue_dense<OP_REAL, 128, TC2_BN>(p, tfull + as, aphase, tbase, i, jbase, lane);
      else
        epilogue_generic<OP_REAL, 128, TC2_BN>(p, tfull + as, aphase, tbase, i, jbase);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), lead_rank));
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace tk
