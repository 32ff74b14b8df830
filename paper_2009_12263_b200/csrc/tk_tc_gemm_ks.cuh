// tk_tc_gemm_ks.cuh -- on-chip split-K for single-wave real GEMMs: a 4-CTA cluster = two CTA
// pairs computing the two K halves of one 256 x BNI output tile, reduced through distributed
// shared memory (no global round trip).
//
// Why: a 1024^3 problem has only 64 pair tiles of 256 x 64 (or 32 of 256 x 128).  With whole-K
// tiles each SM ingests 20 KB per 64-deep k-block for 16 k-blocks and issues N=64 MMAs, which
// run well below the tensor rate (profiles/README.md, r1e: ~53 clocks per N=64 pair MMA).
// Splitting K over two pairs lets every tile be 256 x 128 (N=128 MMAs at the tensor rate, A
// re-read half as often) while still occupying 128 SMs: each SM ingests 8 x 24 KB instead of
// 16 x 20 KB and issues half as many MMA steps.
//
// BNI = 256 (256 x 256 tiles, 128 finalised columns and two C/D boxes per epilogue warp) takes
// the single-wave shapes whose 256 x 128 tiles outnumber the co-resident clusters (2048 x 1024).
//
// Cluster ranks: r = 2q + h.  Pair q (leader rank 2q) accumulates k-blocks
// [q*KB/2, (q+1)*KB/2) of the tile (the reference's k-ascending order inside each half,
// kernel.py:399-404); h selects the 128-row half of the tile (as in the pair kernel).
// After the MMAs, CTA r and its partner r^2 (same rows, other K half) reduce-scatter:
// CTA r finalises columns [q*BNI/2, (q+1)*BNI/2) of its rows and ships the other half of its
// accumulator to the partner: staged in its own (by then idle) operand ring and moved by one
// shared::cluster bulk copy per warp that completes_tx on the partner's mbarrier (no release
// fence, no polling of global flags; per-thread st.async remote stores took ~1.8 us for the
// same 32 KB).  The finalising CTA
// computes v = partial(partner) + acc(own) (one FP32 add, commutative, so the result does not
// depend on which side finalises), then the fused epilogue of the pair kernel
// (epi_math_real: + g2s_c(C), r2s, bias, s2g) with C prefetched into a per-warp TMA box during
// the mainloop and D leaving through a TMA bulk store from the same box.
#pragma once
#include "tk_tc_gemm2.cuh"

#ifndef TK_KS_ROLE_WAIT
#define TK_KS_ROLE_WAIT 0
#endif

namespace tk {

template <int BNI, int KPS>
struct KsPlan {
  static constexpr int A_BYTES = 128 * 64 * 2;                  // this CTA's 128 rows x 64 k
  static constexpr int B_BYTES = BNI * 64;                      // this CTA's BNI/2 columns x 64 k
  static constexpr int KB_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGE_BYTES = KPS * KB_BYTES;
  static constexpr int HALF_COLS = BNI / 2;                     // columns finalised per CTA
  static constexpr int BOXES = 4 * HALF_COLS / 32;              // 32x32 C/D boxes per CTA
  static constexpr int CRING_BYTES = BOXES * TC_CBOX_BYTES;     // one C box per box, prefetched
  static constexpr int XBUF_BYTES = 128 * HALF_COLS * 4;        // partner's partial (FP32)
  // the partner's partial lands in this CTA's operand ring once that is idle (at XBUF, after the
  // XBUF_BYTES where the outgoing half is staged): the ring gets the room (BNI 128: 8 stages
  // instead of 6)
  static constexpr int FIXED = CRING_BYTES + 512 + 1024;
  static constexpr int MAX_STAGES = (227 * 1024 - FIXED) / STAGE_BYTES;
#ifndef TK_KS_MAX_STAGES
#define TK_KS_MAX_STAGES 8
#endif
  static constexpr int STAGES = MAX_STAGES > TK_KS_MAX_STAGES ? TK_KS_MAX_STAGES : MAX_STAGES;
  static constexpr int CRING = STAGES * STAGE_BYTES;
  static constexpr int XBUF = XBUF_BYTES;  // inside the ring: [0, XBUF) stages the outgoing half
  static constexpr int BAR_OFFSET = CRING + CRING_BYTES;
  static constexpr int SMEM = BAR_OFFSET + 512 + 1024;
  static constexpr int TMEM_COLS = BNI < 32 ? 32 : BNI;
  static constexpr int CPW = BOXES / TC_EPI_WARPS;              // boxes (32-column chunks) per epilogue warp
  static_assert(CPW * TC_EPI_WARPS == BOXES, "whole boxes per epilogue warp");
  static_assert(2 * XBUF_BYTES <= STAGES * STAGE_BYTES, "staging + partial fit in the ring");
  static_assert(STAGES >= 2 && SMEM <= 227 * 1024, "k-split kernel shared memory");
};

// NT = output tiles per cluster along N (cluster = 4*NT CTAs).  NT = 2: the two tiles' pairs
// (ranks 4nn + 2q + h) need the same A rows and K half, so each CTA fetches one 64-row atom of
// its 128 A rows and multicasts it to itself and its twin r^4 -- half the L2 reads of A; a ring
// stage is then released only when both twins' MMAs have consumed it.
template <int BNI, int KPS, int NT>
__global__ void __cluster_dims__(4 * NT, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_gemm_ksplit_kernel(const __grid_constant__ TcParams p) {
  using PL = KsPlan<BNI, KPS>;
  static_assert(BNI == 128 || (BNI == 256 && NT == 1),
                "256 x 128 tiles (64 finalised columns per CTA) or 256 x 256 (128, 4-CTA clusters)");
  constexpr int STAGES = PL::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PL::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* xfull = tfull + 1;
  uint64_t* cfull = xfull + 1;  // [BOXES]
  uint64_t* xready = cfull + PL::BOXES;  // the partner's ring is idle: its partial may be sent
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xready + 1);
  float* cring = reinterpret_cast<float*>(smem + PL::CRING);
  const uint32_t xbuf = smem_u32(smem + PL::XBUF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TK_TS(0);
  const uint32_t rank = cluster_ctarank();
  const uint32_t nn = rank >> 2, q = (rank >> 1) & 1, h = rank & 1;
  const uint32_t lead = rank & ~1u, partner = rank ^ 2u;
  const uint16_t pair_mask = uint16_t(0x3u << (rank & ~1u));
  // ring-stage release: this pair, and (NT 2) the twin pair whose A atoms land here too
  const uint16_t empty_mask = NT == 2 ? uint16_t((0x3u << (2 * q)) | (0x3u << (4 + 2 * q))) : pair_mask;
  const int tile = blockIdx.x / (4 * NT);
  const int kbh = p.kb_total / 2;
  const int kb0 = q ? kbh : 0, kb1 = q ? p.kb_total : kbh;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&p.ta[0]);
    tma_prefetch(&p.tb[0]);
    if (!p.c_zero) tma_prefetch(&p.tcmap);
    tma_prefetch(&p.tdmap);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT);
    }
    mbar_init(tfull, 1);
    mbar_init(xfull, 1);
    for (int w = 0; w < PL::BOXES; ++w) mbar_init(&cfull[w], 1);
    mbar_init(xready, 1);
    fence_mbar_init();
    // the partner's partial: XBUF_BYTES of bulk-copy complete_tx, sent only after this CTA's
    // xready arrival (its ring is idle), long after this initialisation is cluster-visible
    mbar_arrive_expect_tx(xfull, PL::XBUF_BYTES);
  }
  if (warp == 2) {
    tmem_alloc_pair(tmem_slot, PL::TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (p.pdl) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // (TK_KS_ROLE_WAIT builds: the producer waits right before its first load and the
    // epilogue warps before their first global access instead -- an experiment)
    if (!TK_KS_ROLE_WAIT) asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  // stamps (TK_STAMPS builds): 15 = the previous launch's exit, 1 = inputs may be read
  if (TK_STAMPS && threadIdx.x == 0 && blockIdx.x == p.dbg_cta) g_dbg_ts[15] = g_dbg_ts[7];
  if (threadIdx.x == 0) TK_TS(1);
  if (threadIdx.x == 0) TK_TSMAX(12);

  int mb, nb;
  tile_coords(p, tile, mb, nb);
  nb = nb * NT + int(nn);                    // (NT 2: p.num_nb counts 256-column tile pairs)
  const int row0 = mb * 256 + int(h) * 128;  // this CTA's rows

  if (warp == 0) {
    // ------------------------------------------------------------ producer (all four CTAs)
    if (lane == 0) {
      const uint64_t pol = policy_code(p.pol_a), pol_b = policy_code(p.pol_b);
      const int a_mode = p.a_mn ? ((p.mn3d & 1) ? 0 : 1) : 2;
      const int b_mode = p.b_mn ? ((p.mn3d & 2) ? 0 : 1) : 2;
      const int n0 = nb * BNI + int(h) * (BNI / 2);
      const uint32_t fb0 = mapa_shared(smem_u32(&full[0]), lead);
      int stage = 0;
      uint32_t phase = 0;
      bool c_issued = false;
      for (int kb = kb0; kb < kb1; kb += KPS) {
        const int cnt = kb1 - kb < KPS ? kb1 - kb : KPS;
        mbar_wait(&empty[stage], phase ^ 1);
        if (TK_KS_ROLE_WAIT && kb == kb0 && p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
        const uint32_t fb = fb0 + uint32_t(stage * 8);
        if (h == 0) mbar_arrive_expect_tx(&full[stage], uint32_t(2 * cnt * PL::KB_BYTES));
        for (int hh = 0; hh < cnt; ++hh) {
          const int k0 = (kb + hh) * TC_BK;
          uint8_t* at = smem + stage * PL::STAGE_BYTES + hh * PL::KB_BYTES;
          uint8_t* bt = at + PL::A_BYTES;
          if (NT == 2) {  // A atom nn (64 rows; ta[0] has 64 x 64 boxes) to this CTA and its twin
            const uint16_t mc = uint16_t((1u << rank) | (1u << (rank ^ 4u)));
            if (p.a_mn)
              tma_load_2d_pair_mc(at + nn * 8192, &p.ta[0], &full[stage], mc, row0 + 64 * int(nn), k0, pol);
            else
              tma_load_2d_pair_mc(at + nn * 8192, &p.ta[0], &full[stage], mc, k0, row0 + 64 * int(nn), pol);
          } else if (a_mode == 0) {
            tma_load_3d_pair(at, &p.ta[0], fb, 0, k0, row0 >> 6, pol);
          } else if (a_mode == 1) {
            tma_load_2d_pair(at, &p.ta[0], fb, row0, k0, pol);
            tma_load_2d_pair(at + 8192, &p.ta[0], fb, row0 + 64, k0, pol);
          } else {
            tma_load_2d_pair(at, &p.ta[0], fb, k0, row0, pol);
          }
          if (b_mode == 0) {
            tma_load_3d_pair(bt, &p.tb[0], fb, 0, k0, n0 >> 6, pol_b);
          } else if (b_mode == 1) {  // 64-column MN-major atoms
            for (int hb = 0; hb < BNI / 128; ++hb)
              tma_load_2d_pair(bt + hb * 8192, &p.tb[0], fb, n0 + 64 * hb, k0, pol_b);
          } else {
            tma_load_2d_pair(bt, &p.tb[0], fb, k0, n0, pol_b);
          }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        // the C block (one 32x32 box per epilogue warp) once the ring's first fill is in flight,
        // so it does not delay the first operand stages
        if (!p.c_zero && (kb - kb0 + KPS >= STAGES * KPS || kb + KPS >= kb1) && !c_issued) {
          c_issued = true;
          const uint64_t pol_c = policy_code(p.pol_c);
          for (int w = 0; w < PL::BOXES; ++w) {
            mbar_arrive_expect_tx(&cfull[w], TC_CBOX_BYTES);
            tma_load_2d(cring + w * (TC_CBOX_BYTES / 4), &p.tcmap, &cfull[w], row0 + (w & 3) * 32,
                        nb * BNI + int(q) * PL::HALF_COLS + (w >> 2) * 32, pol_c);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (pair leaders)
    if (h == 0 && lane == 0) {
      const uint32_t idesc = idesc_f16(p.ab_fmt, p.a_mn, p.b_mn, 0, 256, BNI);
      const uint32_t a_kk = (p.a_mn ? 2048u : 32u) >> 4, b_kk = (p.b_mn ? 2048u : 32u) >> 4;
      const uint64_t a_desc0 = sdesc_sw128(smem_u32(smem), p.a_mn ? 8192u : 16u, 1024);
      const uint64_t b_desc0 = sdesc_sw128(smem_u32(smem + PL::A_BYTES), p.b_mn ? 8192u : 16u, 1024);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; kb += KPS) {
        const int cnt = kb1 - kb < KPS ? kb1 - kb : KPS;
        mbar_wait(&full[stage], phase);
        if (kb == kb0) { TK_TS(2); TK_TSMAX(13); }
        tc_fence_after();
        const uint32_t so = uint32_t(stage) * uint32_t(PL::STAGE_BYTES >> 4);
        for (int hh = 0; hh < cnt; ++hh) {
          const uint32_t ho = so + uint32_t(hh * (PL::KB_BYTES >> 4));
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk)
            tc_mma_f16_pair(tmem_base, a_desc0 + ho + kk * a_kk, b_desc0 + ho + kk * b_kk, idesc,
                            (kb > kb0 || hh > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit_pair(&empty[stage], empty_mask);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      tc_commit_pair(tfull, pair_mask);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ reduce-scatter + epilogue
    if (TK_KS_ROLE_WAIT && p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    // warp ew owns boxes b = ew + 8i (i < CPW): TMEM lane quarter b & 3 (= warp & 3), 32-column
    // chunk b >> 2 of the finalised half
    const int ew = warp - 4;
    const int quarter = warp & 3;  // TMEM lane quarter of this warp
    const int row_local = quarter * 32 + lane;
    const uint32_t tlane = tmem_base + (uint32_t(quarter * 32) << 16);
    // partial layout (per CTA): box b at b*4 KB (chunk c at c*16 KB, row r at r*128 B), 16-byte
    // granule g at (g ^ (r & 7)) -- conflict-free for the 8-lane phases of the v4 stores / loads
    const int sw = row_local & 7;
    mbar_wait_sleep(tfull, 0);
    TK_TS_EPI(4);
    if (warp == 4 && lane == 0) {
      TK_TSMAX(11);
      // every MMA of this pair -- hence every read of this CTA's ring -- has completed: the
      // partner may now write its partial into the ring
      mbar_arrive_cluster(mapa_shared(smem_u32(xready), partner));
    }
    tc_fence_after();
    // ship the partner's columns of this warp's boxes: stage them (swizzled like the partner's
    // buffer, at the same offsets) in this CTA's operand ring -- free once the accumulator is
    // full, all MMAs and hence all operand reads having completed -- and move each 4 KB box with
    // one bulk copy into the partner's ring (once it is idle too) that completes on its barrier
#pragma unroll 1
    for (int i = 0; i < PL::CPW; ++i) {
      const int bx = ew + TC_EPI_WARPS * i, chunk = bx >> 2;
      uint32_t r[32];
      tmem_ld_32x32b_x32(tlane + uint32_t((q ^ 1u) * PL::HALF_COLS + chunk * 32), r);
      tmem_ld_wait();
      const uint32_t stg = smem_u32(smem) + uint32_t(bx * 4096 + lane * 128);
#pragma unroll
      for (int g = 0; g < 8; ++g)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + uint32_t((g ^ sw) << 4)), "r"(r[4 * g]),
                     "r"(r[4 * g + 1]), "r"(r[4 * g + 2]), "r"(r[4 * g + 3])
                     : "memory");
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      mbar_wait(xready, 0);  // the partner's ring is idle
      for (int i = 0; i < PL::CPW; ++i) {
        const int bx = ew + TC_EPI_WARPS * i;
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                mapa_shared(xbuf + uint32_t(bx * 4096), partner)),
            "r"(smem_u32(smem) + uint32_t(bx * 4096)), "r"(mapa_shared(smem_u32(xfull), partner))
            : "memory");
      }
    }
    TK_TS_EPI(3);
    const int i_row = row0 + row_local;
    const bool row_ok = i_row < p.m;
    const float bias_m = (p.bias_axis == 2 && row_ok) ? p.bias[i_row] : 0.f;
#pragma unroll 1
    for (int i = 0; i < PL::CPW; ++i) {
      const int bx = ew + TC_EPI_WARPS * i, chunk = bx >> 2;
      const int j0 = nb * BNI + int(q) * PL::HALF_COLS + chunk * 32;
      uint32_t r[32];
      tmem_ld_32x32b_x32(tlane + uint32_t(q * PL::HALF_COLS + chunk * 32), r);
      const int jl = j0 + lane;
      const float bcol = (p.bias_axis == 1 && jl < p.n) ? p.bias[jl] : 0.f;
      float* box = cring + bx * (TC_CBOX_BYTES / 4);
      const uint32_t box_s = smem_u32(box);
      float cv[32];
      if (!p.c_zero) {
        mbar_wait(&cfull[bx], 0);
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) cv[jj] = lds_f32(box_s + uint32_t(jj * 32 + lane) * 4u);
      }
      float pv[32];
      mbar_wait(xfull, 0);
      if (i == 0) TK_TS_EPI(5);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        uint32_t v0, v1, v2, v3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                     : "r"(xbuf + uint32_t(bx * 4096 + lane * 128) + uint32_t((g ^ sw) << 4)));
        pv[4 * g] = __uint_as_float(v0);
        pv[4 * g + 1] = __uint_as_float(v1);
        pv[4 * g + 2] = __uint_as_float(v2);
        pv[4 * g + 3] = __uint_as_float(v3);
      }
      tmem_ld_wait();
      if (i == 0) TK_TS_EPI(14);
      float out[32];
      epi_math_real<true>(p, r, cv, pv, !p.c_zero, bias_m, bcol, out);
      __syncwarp();  // every lane has read its C column before the box is overwritten
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) sts_f32(box_s + uint32_t(jj * 32 + lane) * 4u, out[jj]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        // (per-thread st.global of the same 32 KB per CTA measured ~0.5 us slower to retire)
        if (p.pol_d)
          tma_store_2d_hint(&p.tdmap, box, row0 + quarter * 32, j0, policy_code(p.pol_d));
        else
          tma_store_2d(&p.tdmap, box, row0 + quarter * 32, j0);  // clips rows >= M, columns >= N
        bulk_commit();
      }
    }
    if (lane == 0) {
      TK_TS_EPI(6);
      if (warp == 4) TK_TSMAX(10);
      bulk_wait_read<0>();  // the boxes are read; grid completion performs the stores
      TK_TS_EPI(8);
    }
  }

  tc_fence_before();
  cluster_sync();  // (also: no CTA leaves while a partner's bulk copy may still target it)
  if (threadIdx.x == 0) TK_TS(7);
  if (threadIdx.x == 0) TK_TSMAX(9);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, PL::TMEM_COLS);
  }
}

}  // namespace tk
