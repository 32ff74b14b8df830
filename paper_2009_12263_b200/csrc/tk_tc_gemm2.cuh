// tk_tc_gemm2.cuh -- the CTA-pair (cta_group::2) tcgen05 GEMM for the real operator.
//
// A cluster of two CTAs on one TPC computes a 256 x (NSUB*BNI) output tile with
// 256 x BNI x 16 tcgen05.mma.cta_group::2 instructions issued by the leader CTA's MMA thread
// (BNI = 256 for large problems; 128 / 64 give more tiles for single-wave shapes):
//   * each CTA stages its own 128 rows of A and its own BNI/2 columns of B (half of the pair's N),
//     so per-SM shared-memory operand traffic is half of the single-CTA form;
//   * both CTAs' TMA loads credit the leader's full barrier (2-SM TMA form);
//   * MMA completion is multicast to both CTAs' empty / accumulator-full barriers;
//   * each CTA's TMEM holds its 128 rows x BNI FP32 columns (double-buffered) or, for NSUB 2,
//     one 128 x 512 accumulator;
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

// Shared-memory plan of the pair kernel.  BNI = instruction N (pair columns per MMA);
// NSUB = number of BNI-wide pair MMAs per K step sharing one A tile:
// NSUB 1 -> 256 x BNI pair tiles, two TMEM accumulators (epilogue overlaps the next tile);
// NSUB 2 -> 256 x 512 pair tiles (BNI 256; A re-used across 512 columns: 1/3 fewer operand
// bytes per flop), one 512-column accumulator drained in two halves.
// CSL = C-ring slots per epilogue warp (streamed-C variant): 2 in general; 4 for single-wave
// launches, where every 32-column C box of the tile is prefetched during the mainloop and the
// drain never waits on a C load (3 operand stages make room).
// KPS = K-blocks (of 64) per ring stage: 2 for the narrow single-wave tiles (BNI 64 / 128), so
// each barrier round trip (full -> MMAs -> commit -> empty -> TMA) carries twice the operand
// bytes; a stage is then two self-contained K-block halves [A kb][B kb][A kb+1][B kb+1].
//
// EMB (complex embedding, see tc_gemm_pair_kernel): the producer lands a raw interleaved A box
// (128 rows x 32 complex k, 8 KB) in the upper half of each A slot; two transform warps expand it
// in place into the stage's A~ tile.
constexpr int EMB_RAW_BYTES = 128 * 32 * 2;
constexpr int EMB_THREADS = TC_THREADS + 64;  // + 2 transform warps (12, 13)
template <int NSUB, bool CSTREAM, int BNI = 256, int CSL = TC2S_CSLOTS, int KPS = 1, bool EMB = false>
struct Tc2Plan {
  static constexpr int B_BYTES = BNI * 64;  // BNI/2 columns x 64 K x 2 bytes per CTA per MMA
  static constexpr int KB_BYTES = TC2_TILE_BYTES + NSUB * B_BYTES;  // one K-block's operands
  static constexpr int STAGE_BYTES = KPS * KB_BYTES;
  static constexpr int CSLOTS = CSL;
  static constexpr int CRING_BYTES = CSTREAM ? TC_EPI_WARPS * CSL * TC_CBOX_BYTES : 0;
  static constexpr int MAX_STAGES = (226 * 1024 - 1536 - CRING_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = NSUB == 2 ? (CSTREAM ? (CSL > TC2S_CSLOTS ? MAX_STAGES : 3) : 4)
                              : CSL > TC2S_CSLOTS ? (MAX_STAGES > 8 ? 8 : MAX_STAGES)
                              : (BNI == 256 && KPS == 1) ? (CSTREAM ? TC2S_STAGES : TC2_STAGES)
                              : (MAX_STAGES > 8 ? 8 : MAX_STAGES);
  static constexpr int CRING = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFFSET = CRING + CRING_BYTES;
  static constexpr int SMEM = BAR_OFFSET + 512 + 1024;
  static constexpr int BNP = BNI * NSUB;                       // pair tile N
  static constexpr int TMEM_COLS = NSUB == 2 ? 512 : 2 * BNI;  // double-buffered for NSUB 1
  static constexpr int WCOLS = BNI / 2;                        // columns per epilogue warp per pass
  static constexpr int THREADS = EMB ? EMB_THREADS : TC_THREADS;
  static_assert(SMEM <= 227 * 1024, "pair kernel shared memory");
};

// One unit of the pair kernel's static schedule: a whole tile, or K-part `part` of a split tile
// (role 1: leaves a partial, role 2: the last part, reduces the partials in its epilogue).
struct PairUnit {
  int tile, kb0, kb1, role, sk_tile, part, noff, narrow;
};
__device__ __forceinline__ PairUnit pair_unit(const TcParams& p, int u) {
  if (u < p.sk_first) return PairUnit{u, 0, p.kb_total, 0, 0, 0, 0, 0};
  const int v = u - p.sk_first, r = v / p.sk_parts, s = v - r * p.sk_parts;
  return PairUnit{p.sk_first + r, s * p.kb_total / p.sk_parts, (s + 1) * p.kb_total / p.sk_parts,
                  s == p.sk_parts - 1 ? 2 : 1, r, s, 0, 0};
}
// Per-cluster unit lists.  Default: units c, c+P, c+2P, ... (P clusters).  NSUB 2 staggered
// (nar_units = S > 0): cluster c < S owns wide tile c and processes it as two half-width units,
// the first at the start of its list and the second at its end; tiles S.. are dealt round-robin
// starting at cluster S.  Half of the clusters thus run half a tile out of phase with the other
// half, so the single-accumulator drains (C read + D write, HBM-bound when all clusters drain
// together) alternate instead of coinciding, and every cluster still owns ceil(T/P) tiles'
// worth of work when T mod P >= S.
__device__ __forceinline__ int unit_count(const TcParams& p, int c, int P) {
  if (p.nar_units > 0) {
    const int S = p.nar_units, mid = p.num_tiles - S;
    const int j0 = (c - S + P) % P;
    return (j0 < mid ? (mid - 1 - j0) / P + 1 : 0) + (c < S ? 2 : 0);
  }
  return c < p.num_units ? (p.num_units - 1 - c) / P + 1 : 0;
}
__device__ __forceinline__ PairUnit unit_at(const TcParams& p, int c, int P, int idx, int count) {
  if (p.nar_units > 0) {
    const int S = p.nar_units;
    if (c < S) {
      if (idx == 0) return PairUnit{c, 0, p.kb_total, 0, 0, 0, 0, 1};
      if (idx == count - 1) return PairUnit{c, 0, p.kb_total, 0, 0, 0, 256, 1};
      --idx;
    }
    return PairUnit{S + (c - S + P) % P + idx * P, 0, p.kb_total, 0, 0, 0, 0, 0};
  }
  return pair_unit(p, c + idx * P);
}

// NSUB 2 drain overlap.  A 256 x 512 tile has one 512-column accumulator: columns [0,256) (lo)
// and [256,512) (hi), each filled by one N=256 MMA per K=16 step.  Run as K + Xs + Xe steps,
//   [0,Xs) lo only | [0,Xs) hi only | [Xs,K-Xe) both | [K-Xe,K) lo only | [K-Xe,K) hi only
// (k-block indices; mirrored for serpentine tiles), lo completes Xe hi-only steps before hi, so
// its drain runs under them, and the next tile's Xs lo-only steps cover the hi drain.  Each half
// still accumulates its k-blocks in ascending (or, serpentine, descending) order.  The first
// unit of a cluster has nothing to overlap at its start (Xs = 0), the last none at its end
// (Xe = 0).  Returns the k-block and the half mask (1 lo, 2 hi, 3 both) of step i.
__device__ __forceinline__ void nsub2_step(int i, int K, int Xs, int Xe, int& kb, int& mask) {
  if (i < Xs) { kb = i; mask = 1; }
  else if (i < 2 * Xs) { kb = i - Xs; mask = 2; }
  else if (i < K + Xs - Xe) { kb = i - Xs; mask = 3; }
  else if (i < K + Xs) { kb = i - Xs; mask = 1; }
  else { kb = i - Xs - Xe; mask = 2; }
}

// 5-D coordinates of the box at (mn0, k0) of a digit-mapped operand (TcParams::a_g / b_g):
// MN-major {64, K0, MN0/64, MN1, K1}, K-major {64, MN0, MN1, K0/64, K1}
__device__ __forceinline__ void gather_load(void* dst, const CUtensorMap* m, uint32_t bar, int g, int e0, int f0,
                                            int mn0, int k0, uint64_t pol) {
  const int kq = k0 / f0, kr = k0 - kq * f0, mq = mn0 / e0, mr = mn0 - mq * e0;
  if (g == 1)
    tma_load_5d_pair(dst, m, bar, 0, kr, mr >> 6, mq, kq, pol);
  else
    tma_load_5d_pair(dst, m, bar, 0, mr, mq, kr >> 6, kq, pol);
}

// Complex embedding (EMB): an interleaved complex GEMM (reference ComplexOperator over
// InterleavedComplex A/B/C/D, operators.py:140-163, layouts.py:315-394) run as the real GEMM
//   D^ (2M x N) = A~ (2M x 2K) * B^ (2K x N) + C^,
// where X^ is the interleaved buffer read as a plain real column-major matrix (row 2i+c /
// k-row 2k+c = component c of element i / k) and A~ holds A^'s column k at k-row 2k and J A^ at
// k-row 2k+1, J(x_re, x_im) = (-x_im, x_re):  D^[2i] = sum Ar Br - Ai Bi, D^[2i+1] = sum Ai Br + Ar Bi.
// B^, C^ and D^ need no preparation (TMA reads the interleaved buffers as they are); A~ is built
// in shared memory by two transform warps from raw A^ boxes that the producer streams through a
// staging ring -- no de-interleave pass over HBM.  The peer CTA's A~ stage is announced to the
// leader's full barrier by a 16-byte bulk copy (async proxy, complete_tx on the leader's barrier).
template <bool DENSE_EPI, bool CSTREAM = false, int NSUB = 1, int BNI = 256, int CSL = TC2S_CSLOTS, int KPS = 1,
          bool EMB = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(EMB ? EMB_THREADS : TC_THREADS, 1)
    tc_gemm_pair_kernel(const __grid_constant__ TcParams p) {
  using PL = Tc2Plan<NSUB, CSTREAM, BNI, CSL, KPS, EMB>;
  static_assert(!EMB || (KPS == 1 && BNI == 256 && DENSE_EPI), "complex embedding: 256-wide tiles, dense epilogue");
  static_assert(NSUB == 1 || BNI == 256, "NSUB 2 uses 256-wide MMAs");
  static_assert(KPS == 1 || NSUB == 1, "several K-blocks per stage: single-MMA tiles only (no predicate bits)");
  constexpr int STAGES = PL::STAGES;
  constexpr int BNP = PL::BNP;
  constexpr int NCBAR = CSTREAM ? TC_EPI_WARPS * CSL : 0;
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
  // EMB: per-stage raw-A barriers (local) and the 16-byte relay slot, past the other barriers
  uint64_t* afull = reinterpret_cast<uint64_t*>(smem + PL::BAR_OFFSET + 384);
  uint8_t* relay = smem + PL::BAR_OFFSET + 448;
  static_assert(!EMB || STAGES <= 8, "EMB barrier slots");

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TK_TS(0);
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
      mbar_init(&full[s], EMB ? 2 : 1);  // EMB: + the leader's transform arrival
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
    if (EMB)
      for (int s = 0; s < STAGES; ++s) mbar_init(&afull[s], 1);
    fence_mbar_init();
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
    // let the next launch in the stream start its prologue as our CTAs retire, and do not touch
    // global memory before the previous grid (the producer of our inputs) has completed.
    // (Waiting per role instead -- the producer only right before its first TMA load -- took
    // ~1 us off the first stage at 1024-2048^3 but measured -1..+2.5 % overall: reverted.)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (threadIdx.x == 0) TK_TS(1);
  unsigned long long clk0 = 0, ns0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    clk0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns0));
  }

  auto a_tile = [&](int s) -> uint8_t* { return smem + s * PL::STAGE_BYTES; };
  auto b_tile = [&](int s) -> uint8_t* { return smem + s * PL::STAGE_BYTES + TC2_TILE_BYTES; };
  constexpr int CH = PL::WCOLS / 32;
  // KPS 2: steps of two K-blocks over [kb0, kb1) (the last one single if the count is odd),
  // in reverse step order for serpentine tiles; ascending inside a step
  auto kps_step = [&](const PairUnit& un, bool rev, int st, int& kb, int& cnt) {
    const int nst = (un.kb1 - un.kb0 + KPS - 1) / KPS;
    kb = un.kb0 + KPS * (rev ? nst - 1 - st : st);
    cnt = un.kb1 - kb < KPS ? un.kb1 - kb : KPS;
  };  // 32-column chunks per epilogue warp per pass

  if (CSTREAM && warp == 3) {
    // ------------------------------------------------------------ C loader (both CTAs)
    if (!p.c_zero && lane == 0) {
      uint32_t q = 0;
      const int nu = unit_count(p, cluster, nclusters);
      // C is needed only at the first tile's end: hold it back until the first ring stage has
      // been consumed, so the C block does not queue in front of the first operand stages
      // (measured at 2048^3: ~3.3 us from the inputs being readable to the first full stage
      // with C issued at once).  Not with a block predicate: a cluster whose tiles skip every
      // k-block never fills stage 0.
      if (!p.kbits && nu > 0) mbar_wait_sleep(&empty[0], 0);
      // ring slot q (per epilogue warp): wait until the epilogue released its previous use
      auto claim = [&](uint32_t qq, int w) -> int {
        const int bi = w * CSL + int(qq % CSL);
        mbar_wait_sleep(&cempty[bi], ((qq / CSL) & 1) ^ 1);
        return bi;
      };
      for (int u = 0; u < nu; ++u) {
        const PairUnit un = unit_at(p, cluster, nclusters, u, nu);
        if (un.role == 1) {  // partial K-parts never read C
          if (p.sk_tma) {    // ... but stage their outgoing partial boxes in the ring: claim slots
            for (int ch = 0; ch < CH; ++ch, ++q)
              for (int w = 0; w < TC_EPI_WARPS; ++w) mbar_arrive(&cfull[claim(q, w)]);
          }
          continue;
        }
        int mb, nb;
        tile_coords(p, un.tile, mb, nb);
        if (un.role == 2 && p.sk_tma) {
          // last K-part: every other part's partial must be in memory before it is loaded
          const int want = (p.sk_parts - 1) * 2 * TC_EPI_WARPS;
          int got;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(got) : "l"(p.sk_flags + un.sk_tile) : "memory");
            if (got < want) __nanosleep(128);
          } while (got < want);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int ch = 0; ch < (un.narrow ? 1 : NSUB) * CH; ++ch, ++q) {
          if (un.role == 2 && p.sk_tma) {
            // the other parts' partial boxes of this chunk, in part order, ahead of the C box
            for (int s = 0; s < p.sk_parts - 1; ++s, ++q)
              for (int w = 0; w < TC_EPI_WARPS; ++w) {
                const int bi = claim(q, w);
                const int blk = (un.sk_tile * (p.sk_parts - 1) + s) * 2 + int(rank);
                mbar_arrive_expect_tx(&cfull[bi], TC_CBOX_BYTES);
                tma_load_2d(smem + PL::CRING + bi * TC_CBOX_BYTES, &p.tskmap, &cfull[bi], (w & 3) * 32,
                            blk * BNP + (w >> 2) * PL::WCOLS + ch * 32, policy_evict_first());
              }
          }
          const uint32_t slot = q % CSL, ph = (q / CSL) & 1;
          for (int w = 0; w < TC_EPI_WARPS; ++w) {
            const int bi = w * CSL + int(slot);
            mbar_wait_sleep(&cempty[bi], ph ^ 1);
            mbar_arrive_expect_tx(&cfull[bi], TC_CBOX_BYTES);
            tma_load_2d(smem + PL::CRING + bi * TC_CBOX_BYTES, &p.tcmap, &cfull[bi],
                        mb * 256 + int(rank) * 128 + (w & 3) * 32,
                        nb * BNP + un.noff + (ch / CH) * BNI + (w >> 2) * PL::WCOLS + (ch % CH) * 32,
                        policy_code(p.pol_c));
          }
        }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      const uint64_t pol = policy_code(p.pol_a), pol_b = policy_code(p.pol_b);
      // uniform per-launch decisions hoisted out of the K loop (the single producer thread's
      // dependent-instruction chain is on the critical path for short tiles)
      const bool no_load = p.dbg_skip_epi & 2;
      const bool c_pf = CSTREAM && p.c_pf_kb > 0 && !p.c_zero;
      const int a_mode = p.a_mn ? ((p.mn3d & 1) ? 0 : 1) : 2;  // 3-D MN box / two 2-D MN boxes / K-major
      const int b_mode = p.b_mn ? ((p.mn3d & 2) ? 0 : 1) : 2;
      int stage = 0;
      uint32_t phase = 0;
      int lu = 0;
      const int nu = unit_count(p, cluster, nclusters);
      for (int u = 0; u < nu; ++u, ++lu) {
        const PairUnit un = unit_at(p, cluster, nclusters, u, nu);
        int mb, nb;
        tile_coords(p, un.tile, mb, nb);
        const int m0 = mb * 256 + int(rank) * 128;     // this CTA's rows of A
        const int n0 = nb * BNP + un.noff + int(rank) * (BNI / 2);  // this CTA's columns of B (per MMA)
        const int nsub_u = un.narrow ? 1 : NSUB;
        // serpentine K: every other tile of a cluster walks K downwards, so the next
        // wave starts on the K-slices the previous one loaded last (still in L2)
        const bool rev = p.serp && (lu & 1);
        if (KPS > 1) {
          const int nst = (un.kb1 - un.kb0 + KPS - 1) / KPS;
          for (int st = 0; st < nst; ++st) {
            int kb, cnt;
            kps_step(un, rev, st, kb, cnt);
            mbar_wait(&empty[stage], phase ^ 1);
            if (lu == 0 && st == 0) { if (leader) TK_TS(12); TK_TSMAX(13); }
            if (leader) mbar_arrive_expect_tx(&full[stage], uint32_t(2 * cnt * PL::KB_BYTES));
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            for (int h = 0; h < cnt; ++h) {
              const int k0 = (kb + h) * TC_BK;
              uint8_t* at = a_tile(stage) + h * PL::KB_BYTES;
              uint8_t* bt = at + TC2_TILE_BYTES;
              if (p.a_g) {
                gather_load(at, &p.ta[0], fb, p.a_g, p.ga_e0, p.ga_f0, m0, k0, pol);
              } else if (a_mode == 0) {
                tma_load_3d_pair(at, &p.ta[0], fb, 0, k0, m0 >> 6, pol);
              } else if (a_mode == 1) {
                tma_load_2d_pair(at, &p.ta[0], fb, m0, k0, pol);
                tma_load_2d_pair(at + 8192, &p.ta[0], fb, m0 + 64, k0, pol);
              } else {
                tma_load_2d_pair(at, &p.ta[0], fb, k0, m0, pol);
              }
              if (p.b_g) {
                gather_load(bt, &p.tb[0], fb, p.b_g, p.gb_e0, p.gb_f0, n0, k0, pol_b);
              } else if (b_mode == 0) {
                tma_load_3d_pair(bt, &p.tb[0], fb, 0, k0, n0 >> 6, pol_b);
              } else if (b_mode == 1) {
                for (int hh = 0; hh < BNI / 128; ++hh)
                  tma_load_2d_pair(bt + hh * 8192, &p.tb[0], fb, n0 + 64 * hh, k0, pol_b);
              } else {
                tma_load_2d_pair(bt, &p.tb[0], fb, k0, n0, pol_b);
              }
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          continue;
        }
        // NSUB 2 drain overlap (nsub2_step): lo-only / hi-only steps load one B half
        const int X = (NSUB == 2 && !un.narrow) ? p.ovl_kb : 0;
        const int Xs = u > 0 ? X : 0, Xe = u < nu - 1 ? X : 0;
        const int nsteps = un.kb1 - un.kb0 + Xs + Xe;
        for (int ki = 0; ki < nsteps; ++ki) {
          int kq = ki, mask = (1 << nsub_u) - 1;
          if (X) nsub2_step(ki, un.kb1 - un.kb0, Xs, Xe, kq, mask);
          const int kb = rev ? un.kb1 - 1 - kq : un.kb0 + kq;
          if (NSUB == 1 && !kmask4(p, un.tile, kb)) continue;  // predicate: k-block skipped entirely
          const int k0 = kb * TC_BK;
          // (EMB: A arrives from the transform warps; +16 bytes: the peer's relay copy)
          const uint32_t tx = EMB ? 2 * __popc(mask) * PL::B_BYTES + 16
                                  : 2 * (TC2_TILE_BYTES + __popc(mask) * PL::B_BYTES);
          mbar_wait(&empty[stage], phase ^ 1);
          if (EMB) {  // raw A^ box (128 rows x 32 complex k) into the upper half of the A slot
            mbar_arrive_expect_tx(&afull[stage], EMB_RAW_BYTES);
            tma_load_2d(a_tile(stage) + 8192, &p.ta[0], &afull[stage], m0, kb * (TC_BK / 2), pol);
          }
          if (no_load) {  // diagnostic: MMA issue rate without operand traffic
            if (leader) mbar_arrive(&full[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          if (c_pf) {
            // warm L2 with this CTA's C block so the (non-overlapped part of the) drain hits L2
            const int at = ki - (un.kb1 - un.kb0 - p.c_pf_kb);  // k-blocks into the prefetch span
            const int nbox = 4 * ((un.narrow ? 256 : BNP) / 32);
            const int cw = nbox / 4;
            if (p.c_pf_spread) {
              if (at >= 0) {
                const uint64_t pl = policy_evict_last();
                for (int b = at * nbox / p.c_pf_kb; b < (at + 1) * nbox / p.c_pf_kb; ++b)
                  tma_prefetch_l2_2d_hint(&p.tcmap, mb * 256 + int(rank) * 128 + (b % 4) * 32,
                                          nb * BNP + un.noff + (b / 4) * 32, pl);
                (void)cw;
              }
            } else if (at == 0) {
              for (int r = 0; r < 4; ++r)
                for (int c = 0; c < cw; ++c)
                  tma_prefetch_l2_2d(&p.tcmap, mb * 256 + int(rank) * 128 + r * 32, nb * BNP + un.noff + c * 32);
            }
          }
          if (lu == 0 && ki == 0) { if (leader) TK_TS(12); TK_TSMAX(13); }
          if (leader) mbar_arrive_expect_tx(&full[stage], tx);
          const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
          if (EMB) {
          } else if (p.a_g) {
            gather_load(a_tile(stage), &p.ta[0], fb, p.a_g, p.ga_e0, p.ga_f0, m0, k0, pol);
          } else if (a_mode == 0) {
            tma_load_3d_pair(a_tile(stage), &p.ta[0], fb, 0, k0, m0 >> 6, pol);
          } else if (a_mode == 1) {
            tma_load_2d_pair(a_tile(stage), &p.ta[0], fb, m0, k0, pol);
            tma_load_2d_pair(a_tile(stage) + 8192, &p.ta[0], fb, m0 + 64, k0, pol);
          } else {
            tma_load_2d_pair(a_tile(stage), &p.ta[0], fb, k0, m0, pol);
          }
#pragma unroll
          for (int sub = 0; sub < NSUB; ++sub) {
            if (!(mask >> sub & 1)) continue;
            uint8_t* bt = b_tile(stage) + sub * PL::B_BYTES;
            const int nn = n0 + sub * BNI;
            if (p.b_g) {
              gather_load(bt, &p.tb[0], fb, p.b_g, p.gb_e0, p.gb_f0, nn, k0, pol_b);
            } else if (b_mode == 0) {
              tma_load_3d_pair(bt, &p.tb[0], fb, 0, k0, nn >> 6, pol_b);
            } else if (b_mode == 1) {  // 64-column atoms (BNI >= 128)
              for (int h = 0; h < BNI / 128; ++h)
                tma_load_2d_pair(bt + h * 8192, &p.tb[0], fb, nn + 64 * h, k0, pol_b);
            } else {
              tma_load_2d_pair(bt, &p.tb[0], fb, k0, nn, pol_b);
            }
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader && lane == 0) {
      const uint32_t idesc = idesc_f16(p.ab_fmt, p.a_mn, p.b_mn, 0, 256, BNI);
      const uint32_t a_step = p.a_mn ? 2048u : 32u;
      const uint32_t b_step = p.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = p.a_mn ? 8192u : 16u;
      const uint32_t b_lbo = p.b_mn ? 8192u : 16u;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      // Descriptors are built once; per MMA only the start-address field (bits 0-13, in 16-byte
      // units, never carrying: shared memory < 256 KB) advances.  The issuing thread's
      // dependent-instruction chain, not the tensor core, bounds N=64/128 tiles (a diagnostic
      // build measured ~64 clocks per MMA with the descriptors rebuilt each time).
      const uint64_t a_desc0 = sdesc_sw128(smem_u32(a_tile(0)), a_lbo, 1024);
      const uint64_t b_desc0 = sdesc_sw128(smem_u32(b_tile(0)), b_lbo, 1024);
      const uint32_t a_kk = a_step >> 4, b_kk = b_step >> 4;
      const bool no_mma = p.dbg_skip_epi & 4;  // diagnostic: operand traffic without MMAs
      auto issue = [&](int st, int sub, uint32_t d, bool first) {
        if (no_mma) return;
        const uint32_t so = uint32_t(st) * uint32_t(PL::STAGE_BYTES >> 4);
        const uint64_t a0 = a_desc0 + so;
        const uint64_t b0 = b_desc0 + so + uint32_t(sub * (PL::B_BYTES >> 4));
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk)
          tc_mma_f16_pair(d, a0 + kk * a_kk, b0 + kk * b_kk, idesc, (!first || kk > 0) ? 1u : 0u);
      };
      const int nu = unit_count(p, cluster, nclusters);
      for (int u = 0; u < nu; ++u, ++local) {
        const PairUnit un = unit_at(p, cluster, nclusters, u, nu);
        if (NSUB == 1) {
          const int as = local & 1;
          const uint32_t aphase = (local >> 1) & 1;
          mbar_wait(&tempty[as], aphase ^ 1);
          tc_fence_after();
          const uint32_t d0 = tmem_base + uint32_t(as * BNI);
          if (KPS > 1) {
            const bool rev = p.serp && (local & 1);
            const int nst = (un.kb1 - un.kb0 + KPS - 1) / KPS;
            for (int st = 0; st < nst; ++st) {
              int kb, cnt;
              kps_step(un, rev, st, kb, cnt);
              mbar_wait(&full[stage], phase);
              if (local == 0 && st == 0) TK_TS(2);
              tc_fence_after();
              const uint32_t so = uint32_t(stage) * uint32_t(PL::STAGE_BYTES >> 4);
              for (int h = 0; h < cnt; ++h) {
                const uint32_t ho = so + uint32_t(h * (PL::KB_BYTES >> 4));
#pragma unroll
                for (int kk = 0; kk < TC_BK / 16; ++kk)
                  tc_mma_f16_pair(d0, a_desc0 + ho + kk * a_kk, b_desc0 + ho + kk * b_kk, idesc,
                                  (st > 0 || h > 0 || kk > 0) ? 1u : 0u);
              }
              tc_commit_pair(&empty[stage], 0x3);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
          } else if (!p.kbits) {
            for (int kb = un.kb0; kb < un.kb1; ++kb) {  // (operand order is the producer's)
              mbar_wait(&full[stage], phase);
              if (local == 0 && kb == un.kb0) TK_TS(2);
              tc_fence_after();
              issue(stage, 0, d0, kb == un.kb0);
              tc_commit_pair(&empty[stage], 0x3);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
          } else {
            // block predicate: the producer's k order, skipped k-blocks never reach the ring;
            // inside a block only the enabled K=16 steps issue, the first of them overwrites
            const bool rev = p.serp && (local & 1);
            bool first = true;
            for (int ki = 0; ki < un.kb1 - un.kb0; ++ki) {
              const uint32_t bits = kmask4(p, un.tile, rev ? un.kb1 - 1 - ki : un.kb0 + ki);
              if (!bits) continue;
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              const uint32_t so = uint32_t(stage) * uint32_t(PL::STAGE_BYTES >> 4);
#pragma unroll
              for (int kk = 0; kk < TC_BK / 16; ++kk)
                if (bits >> kk & 1u) {
                  tc_mma_f16_pair(d0, a_desc0 + so + kk * a_kk, b_desc0 + so + kk * b_kk, idesc, first ? 0u : 1u);
                  first = false;
                }
              tc_commit_pair(&empty[stage], 0x3);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
          }
          tc_commit_pair(&tfull[as], 0x3);
          TK_TS(3);
        } else {
          // 256 x 512 tile, one accumulator: columns [0,256) (lo) and [256,512) (hi) are drained
          // in that order (tempty[0], tempty[1]); tfull[0] / tfull[1] say lo / hi are complete.
          const uint32_t tph = (local & 1) ^ 1;
          if (p.ovl_kb > 0 && !un.narrow) {
            // drain overlap: lo-only / hi-only steps at the tile ends (nsub2_step)
            const int K = p.kb_total, Xs = u > 0 ? p.ovl_kb : 0, Xe = u < nu - 1 ? p.ovl_kb : 0;
            const int nsteps = K + Xs + Xe;
            for (int i = 0; i < nsteps; ++i) {
              int kq, mask;
              nsub2_step(i, K, Xs, Xe, kq, mask);
              if (i == 0) mbar_wait(&tempty[0], tph);   // the previous tile's lo is drained
              if (i == Xs) mbar_wait(&tempty[1], tph);  // ... and its hi (first hi step)
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              if (mask & 1) issue(stage, 0, tmem_base, i == 0);
              if (mask & 2) issue(stage, 1, tmem_base + 256u, i == Xs);
              tc_commit_pair(&empty[stage], 0x3);
              if (i == K + Xs - 1) tc_commit_pair(&tfull[0], 0x3);  // lo complete
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            tc_commit_pair(&tfull[1], 0x3);  // hi complete
            continue;
          }
          mbar_wait(&tempty[0], tph);
          tc_fence_after();
          if (un.narrow) {  // half-width tile: lo columns only (its epilogue also releases hi)
            for (int kb = 0; kb < p.kb_total; ++kb) {
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              issue(stage, 0, tmem_base, kb == 0);
              tc_commit_pair(&empty[stage], 0x3);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            tc_commit_pair(&tfull[0], 0x3);
            tc_commit_pair(&tfull[1], 0x3);
            continue;
          }
          bool hi_ok = false;
          int held = 0, st0 = stage;
          for (int kb = 0; kb < p.kb_total; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            issue(stage, 0, tmem_base, kb == 0);
            if (hi_ok) {
              issue(stage, 1, tmem_base + 256u, false);
              tc_commit_pair(&empty[stage], 0x3);
            } else {
              ++held;
              if (mbar_test(&tempty[1], tph)) {
                hi_ok = true;
              } else if (held == STAGES || kb == p.kb_total - 1) {
                mbar_wait(&tempty[1], tph);
                hi_ok = true;
              }
              if (hi_ok) {
                tc_fence_after();
                for (int h = 0; h < held; ++h) {
                  const int st = (st0 + h) % STAGES;
                  issue(st, 1, tmem_base + 256u, h == 0 && kb + 1 == held);
                  tc_commit_pair(&empty[st], 0x3);
                }
              }
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          tc_commit_pair(&tfull[0], 0x3);
          tc_commit_pair(&tfull[1], 0x3);
        }
      }
    }
  } else if (EMB && warp >= 4 + TC_EPI_WARPS) {
    // ------------------------------------------------------------ A~ transform (both CTAs)
    // The raw A^ box of a stage (k-row k = 256 bytes: rows [0,64) then [64,128)) sits in the upper
    // 8 KB of the A slot.  Warp h = 0 / 1 reads M-chunk h (64 rows) of it into registers, then
    // (after both warps have read) writes A~ chunk h: A^ k-row k -> k-rows 2k (as is) and 2k+1
    // (J per (re, im) 32-bit pair), in the 128B-swizzled MN-major layout the TMA would produce
    // (chunk stride 8 KB, k-row r at r*128, 16-byte granule g at g ^ (r & 7)).
    const int h = warp - 4 - TC_EPI_WARPS;
    const int gg = lane & 7;
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t relay_dst = mapa_shared(smem_u32(relay), 0);
    const int nu = unit_count(p, cluster, nclusters);
    for (int u = 0; u < nu; ++u) {
      const PairUnit un = unit_at(p, cluster, nclusters, u, nu);
      for (int ki = un.kb0; ki < un.kb1; ++ki) {
        mbar_wait(&afull[stage], phase);
        const uint32_t at = smem_u32(a_tile(stage));
        const uint32_t src = at + 8192u + uint32_t(h * 128 + gg * 16);
        uint32_t v[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v[j][0]), "=r"(v[j][1]), "=r"(v[j][2]), "=r"(v[j][3])
                       : "r"(src + uint32_t(((lane >> 3) + 4 * j) * 256)));
        asm volatile("bar.sync 1, 64;" ::: "memory");  // the raw box is read: overwrite it
        const uint32_t dst = at + uint32_t(h * 8192);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r0 = 2 * ((lane >> 3) + 4 * j), r1 = r0 + 1;
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + uint32_t(r0 * 128 + ((gg ^ (r0 & 7)) << 4))),
                       "r"(v[j][0]), "r"(v[j][1]), "r"(v[j][2]), "r"(v[j][3]) : "memory");
          auto jx = [](uint32_t w) { return __byte_perm(w, 0, 0x1032) ^ 0x8000u; };  // (re, im) -> (-im, re)
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + uint32_t(r1 * 128 + ((gg ^ (r1 & 7)) << 4))),
                       "r"(jx(v[j][0])), "r"(jx(v[j][1])), "r"(jx(v[j][2])), "r"(jx(v[j][3])) : "memory");
        }
        fence_proxy_async_smem();  // the generic writes are read by tcgen05.mma (async proxy)
        asm volatile("bar.sync 1, 64;" ::: "memory");
        if (h == 0 && lane == 0) {
          if (leader) {
            mbar_arrive(&full[stage]);
          } else {  // relay: complete_tx on the leader's full barrier through the async proxy
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                    relay_dst),
                "r"(smem_u32(relay)), "r"(mapa_shared(smem_u32(&full[stage]), 0))
                : "memory");
          }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
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
    // bit i: ring use cq - i committed a TMA store (every use before a split unit did; split
    // units, always a cluster's last, mix in partial-read uses -- see ring_release)
    uint32_t smask = 0xFFFFFFFFu;
    const int nu = unit_count(p, cluster, nclusters);
    for (int u = 0; u < nu; ++u, ++local) {
      const PairUnit un = unit_at(p, cluster, nclusters, u, nu);
      const int t = un.tile;
      int mb, nb;
      tile_coords(p, t, mb, nb);
      const int i = mb * 256 + int(rank) * 128 + row_local;
      // split-K: partial blocks of tile r live at sk_ws + ((r*(S-1) + s)*2 + rank) * 128*BNP,
      // column-major 128 x BNP (this thread's row at +row_local)
      const int64_t blk = int64_t(128) * BNP;
      float* sk_row = p.sk_ws ? p.sk_ws + (int64_t(un.sk_tile) * (p.sk_parts - 1) * 2 + int(rank)) * blk +
                                    row_local
                              : nullptr;
      if (NSUB == 1 && !EMB && un.role == 1) {
        // K-part: raw FP32 accumulator -> workspace, then count this warp in
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait_sleep(tfull + as, aphase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(as * BNI);
        if (CSTREAM && p.sk_tma) {
          // stage each 32x32 box in a ring slot the C loader claimed for it, TMA-store it to
          // the workspace, release slots like the D path (once the next store has been issued
          // and this one has read its slot), then publish after the stores have completed
          float* my_ring = cring + ew * CSL * (TC_CBOX_BYTES / 4);
          uint64_t* wfull = cfull + ew * CSL;
          uint64_t* wempty = cempty + ew * CSL;
          const int blk_id = (un.sk_tile * (p.sk_parts - 1) + un.part) * 2 + int(rank);
#pragma unroll 1
          for (int ch = 0; ch < CH; ++ch, ++cq) {
            const int col = half * PL::WCOLS + ch * 32;
            uint32_t r[32];
            tmem_ld_32x32b_x32(tbase + uint32_t(col), r);
            const uint32_t slot = cq % CSL;
            float* box = my_ring + slot * (TC_CBOX_BYTES / 4);
            const uint32_t box_s = smem_u32(box);
            mbar_wait(&wfull[slot], (cq / CSL) & 1);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) sts_f32(box_s + uint32_t(jj * 32 + lane) * 4u, __uint_as_float(r[jj]));
            fence_proxy_async_smem();
            __syncwarp();
            smask = (smask << 1) | 1u;
            if (lane == 0) {
              tma_store_2d(&p.tskmap, box, quarter * 32, blk_id * BNP + col);
              bulk_commit();
              ring_release<CSL>(wempty, cq, smask);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
            bulk_wait<0>();  // this warp's partial boxes are in memory
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            atomicAdd(p.sk_flags + un.sk_tile, 1);
          }
          __syncwarp();
          continue;
        }
        float* out = sk_row + int64_t(un.part) * 2 * blk;
#pragma unroll 1
        for (int ch = 0; ch < CH; ++ch) {
          const int col = half * PL::WCOLS + ch * 32;
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + uint32_t(col), r);
          tmem_ld_wait();
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) __stcg(out + int64_t(col + jj) * 128, __uint_as_float(r[jj]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(p.sk_flags + un.sk_tile, 1);
        continue;
      }
      SkIn sk{nullptr, 0, 0};
      if (NSUB == 1 && !EMB && un.role == 2) {
        // last K-part: wait until every warp of every other part has published its partial
        // (with sk_tma the C loader waits and the partials arrive through the ring)
        if (lane == 0 && !(CSTREAM && p.sk_tma)) {
          const int want = (p.sk_parts - 1) * 2 * TC_EPI_WARPS;
          int got;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(got) : "l"(p.sk_flags + un.sk_tile) : "memory");
            if (got < want) __nanosleep(256);
          } while (got < want);
        }
        __syncwarp();
        sk = SkIn{sk_row, p.sk_parts - 1, 2 * blk};
      }
      const int row0 = mb * 256 + int(rank) * 128 + quarter * 32;
      float* my_ring = cring + ew * CSL * (TC_CBOX_BYTES / 4);
      const bool masked = tile_masked_out(p, t);  // predicate skipped every k-block of the tile
      // NSUB 1: accumulator `local & 1`, one pass over this warp's 128 columns.
      // NSUB 2: one accumulator, pass 0 drains columns [0,256), pass 1 [256,512) (128 per warp).
#pragma unroll 1
      for (int pass = 0; pass < (un.narrow ? 1 : NSUB); ++pass) {
        const int as = NSUB == 1 ? (local & 1) : 0;
        const uint32_t aphase = NSUB == 1 ? ((local >> 1) & 1) : (local & 1);
        uint64_t* tf = tfull + (NSUB == 1 ? as : pass);  // NSUB 2: lo / hi complete
        const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(as * BNI);
        // (a half-width tile sits in TMEM columns [0,256): shift the base by its column offset)
        const uint32_t tb = tbase - uint32_t(un.noff);
        const int jbase = nb * BNP + un.noff + pass * BNI + half * PL::WCOLS;
        if (blockIdx.x == p.dbg_cta && warp == 4 && lane == 0 && u == nu - 1) {
          mbar_wait(tf, aphase);
          TK_TS(4);
        }
        if (CSTREAM) {
          if (!EMB && sk.p)
            epilogue_stream<PL::WCOLS, BNP, CSL, true>(p, tf, aphase, tb, i, jbase, lane, my_ring,
                                                   cfull + ew * CSL, cempty + ew * CSL, cq,
                                                   row0, sk, &smask);
          else
            epilogue_stream<PL::WCOLS, BNP, CSL>(p, tf, aphase, tb, i, jbase, lane, my_ring,
                                                   cfull + ew * CSL, cempty + ew * CSL, cq, row0,
                                                   SkIn{nullptr, 0, 0}, nullptr, masked);
        } else if (p.dbg_skip_epi) {
          mbar_wait_sleep(tf, aphase);
          tc_fence_after();
        } else if (DENSE_EPI) {
          if (!EMB && sk.p)
            epilogue_dense<OP_REAL, PL::WCOLS, BNP, true>(p, tf, aphase, tb, i, jbase, lane, sk);
          else
            epilogue_dense<OP_REAL, PL::WCOLS, BNP>(p, tf, aphase, tb, i, jbase, lane, SkIn{nullptr, 0, 0},
                                                    false, masked);
        } else
          epilogue_generic<OP_REAL, PL::WCOLS, BNP>(p, tf, aphase, tb, i, jbase, false, masked);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[NSUB == 1 ? as : pass]), 0));
        if (warp == 4 && lane == 0) TK_TS(5);
      }
      if (NSUB == 2 && un.narrow) {  // nothing in the hi columns: release them for the next tile
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[1]), 0));
      }
    }
  }

  if (CSTREAM && warp >= 4 && warp < 4 + TC_EPI_WARPS && lane == 0) {
    if (p.npeer) {  // peer slabs complete before the grid retires
      bulk_wait<0>();
      __threadfence_system();
    } else {
      bulk_wait_read<0>();  // the ring slots are read; grid completion performs the stores
    }
  }
  if (warp == 4 && lane == 0) TK_TS(6);
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
    tmem_dealloc_pair(tmem_base, PL::TMEM_COLS);
    if (lane == 0) TK_TS(7);
  }
}

}  // namespace tk
