// tk_tc_gemm.cuh -- persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
// One CTA per SM loops over output tiles dealt by a grouped raster (the device
// form of the reference's parallelise() block dealing, tiling.py:137-210).
// Roles (384 threads):
//   warp 0      TMA producer: global layouts -> 128B-swizzled smem ring (mbarrier full/empty);
//               for a Diagonal A layout it fabricates the diagonal tile in smem instead
//               (reference layouts.py:218-228) and only visits the block-K iterations that
//               intersect the diagonal (DiagonalPredicate, components.py:186-191).
//   warp 1      MMA issuer (one thread): tcgen05.mma kind::f16, FP32 accumulators in TMEM,
//               double-buffered so the epilogue of tile t overlaps the MMAs of tile t+1.
//               REAL = 1 MMA per K=16 step; COMPLEX = 4 (negate-A bit for -Ai*Bi);
//               DUAL = 3 (reference operators.py:140-188).
//   warp 2      TMEM allocator.
//   warps 4-11  epilogue: tcgen05.ld -> registers -> fused
//               D = s2g( r2s( g2s_c(C) + acc ) + bias ) -> coalesced global stores
//               (reference kernel.py:370-463, components.py:110-157).
#pragma once
#include "tk_prep.cuh"
#include "tk_ptx.cuh"
#include "tk_types.cuh"

namespace tk {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_THREADS = (4 + TC_EPI_WARPS) * 32;
constexpr int TC_A_TILE_BYTES = TC_BM * TC_BK * 2;  // 16 KB

template <int OP>
struct TcCfg;
template <>
struct TcCfg<OP_REAL> {
  static constexpr int PLANES = 1, BN = 256, STAGES = 4, ACC_COLS = 256, TMEM_COLS = 512;
};
template <>
struct TcCfg<OP_COMPLEX> {
  static constexpr int PLANES = 2, BN = 128, STAGES = 3, ACC_COLS = 256, TMEM_COLS = 512;
};
template <>
struct TcCfg<OP_DUAL> {
  static constexpr int PLANES = 2, BN = 128, STAGES = 3, ACC_COLS = 256, TMEM_COLS = 512;
};
template <>
struct TcCfg<OP_SPLIT> : TcCfg<OP_DUAL> {};

// C-streaming variants: a per-epilogue-warp ring of TMA-loaded C boxes (32 rows x 32 columns
// fp32), refilled by the loader warp.  CS = 1 (HBM-bound shapes: diagonal A, K <= 256):
// 2 mainloop stages, 3 ring slots.  CS = 2 (single-wave dense shapes): 3 stages, 2 slots.
constexpr int TC_CBOX_BYTES = 32 * 32 * 4;
#ifndef TK_HBM_CSLOTS
#define TK_HBM_CSLOTS 3
#endif
__host__ __device__ constexpr int tc_cslots(int cs) { return cs == 1 ? TK_HBM_CSLOTS : 2; }
constexpr int TC_CSLOTS = 3;

template <int OP, int CSTREAM = 0>
struct TcSmem {
  using C = TcCfg<OP>;
  static constexpr int CSLOTS = tc_cslots(CSTREAM);
  static constexpr int STAGES = CSTREAM == 1 ? 2 : CSTREAM == 2 ? 3 : C::STAGES;
  static constexpr int B_TILE_BYTES = C::BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = C::PLANES * (TC_A_TILE_BYTES + B_TILE_BYTES);
  static constexpr int CRING_OFFSET = STAGES * STAGE_BYTES;
  static constexpr int CRING_BYTES = CSTREAM ? TC_EPI_WARPS * CSLOTS * TC_CBOX_BYTES : 0;
  static constexpr int BAR_OFFSET = CRING_OFFSET + CRING_BYTES;
  static constexpr int NCBAR = CSTREAM ? TC_EPI_WARPS * CSLOTS : 0;
  static constexpr int BAR_BYTES = (2 * STAGES + 4 + 2 * NCBAR) * 8 + 16;
  static constexpr int TOTAL = BAR_OFFSET + BAR_BYTES + 1024;  // +1024 for manual alignment
};

struct TcParams {
  CUtensorMap ta[2];
  CUtensorMap tb[2];
  CUtensorMap tcmap;  // C as {M, N} fp32 boxes of 32x32 (C-streaming epilogue)
  CUtensorMap tdmap;  // D likewise (TMA bulk stores from the same ring slot)
  int32_t m, n, k;
  int32_t a_mn, b_mn, ab_fmt;
  int32_t num_mb, num_nb, num_tiles, kb_total;
  int32_t group_m;
  int32_t diag_a;
  const void* diag;
  int32_t c_zero, c_pair, d_pair, bias_axis;
  const void* c_ptr;
  void* d_ptr;
  const float* bias;
  DigitMap c_map, d_map;
  int64_t c_plane, d_plane;
  // OP_SPLIT: split_flags[0] / [1] != 0 when A / B has a non-zero lo plane (written by the
  // transform pass); a zero lo plane is neither loaded nor multiplied
  const int32_t* split_flags;
  EpiProg t_c, t_r2s, t_s2g;
  // dense column-major epilogue: transforms pre-decoded to relu?(x*mul + add) (complex mul/add
  // for pair operators); see decode_affine() in tk_api.cu
  int64_t ldc, ldd;
  float c_mul[2], c_add[2], r_mul[2], r_add[2], s_mul[2], s_add[2];
  int32_t c_relu, r_relu, s_relu, pad1;
  int32_t dbg_skip_epi, pol_ab;  // tuning/diagnostic knobs (TK_DBG_SKIP_EPI, TK_POLICY_AB)
  int32_t d_tma, mn3d;           // C-streaming epilogue: D via TMA; MN-major operands via 3-D maps (bit0 A, bit1 B)
  int32_t c_pf_kb, c_pf_spread;  // pair kernel: prefetch the tile's C into L2 this many k-blocks before
                                 // its end; spread: one 4 KB box per k-block over that span (evict_last)
  int32_t c_rmap, d_rmap;        // dense epilogue: C / D row offsets through c_map / d_map (GETT outputs)
  int32_t pol_a, pol_b;          // pair kernel L2 policies for A / B loads: 0 normal, 1 evict_last, 2 evict_first
  // split-K of a poorly filled last wave (pair kernel): units [0, sk_first) are whole tiles,
  // units sk_first + r*sk_parts + s are K-part s of tile sk_first + r; parts < sk_parts-1
  // leave raw FP32 partials in sk_ws and count down sk_flags[r], the last part reduces them.
  int32_t num_units, sk_first, sk_parts, dbg_cta;
  int32_t vec_ok, serp;          // diag_stream_kernel: 16-byte vector path legal; pair kernel: serpentine K
  int32_t pdl;                   // pair kernel launched with programmatic stream serialisation
  int32_t sk_tma;                // split-K partials move as 32x32 TMA boxes through the C ring (tskmap)
  // fused all-gather of D over peer memory (NVLink): the streamed epilogue TMA-stores every D
  // box to the local slab and to the same slab position inside each peer's full-D buffer
  CUtensorMap tdpeer[7];
  CUtensorMap tskmap;            // split-K workspace as {128 rows, blocks * BNP columns} fp32
  int32_t npeer, pad7;
  int32_t c_ident, r_ident, s_ident, nar_units;  // empty transform programs: skip the stage;
                                                 // pair NSUB 2: half-width first units (stagger)
  float* sk_ws;
  int32_t* sk_flags;
  // pair kernel NSUB 2: k-blocks at each end of a tile run as separate lo-only and hi-only
  // passes so one accumulator half drains while the tensor cores fill the other (0: off)
  int32_t ovl_kb, pad8;
  // block predicate on the tensor cores (mask or diagonal rule over a dense A, reference
  // components.py:171-191, kernel.py:399-404): kbits[tile * kwords + kb / 8] holds 4 bits per
  // 64-deep k-block, one per K=16 MMA step (expand_kbits_kernel); null = every step runs
  const uint32_t* kbits;
  int32_t kwords;
  int32_t a_embed;
  int32_t pol_c, pol_d;  // L2 policies of the streamed C loads / D stores (0 none, 1 evict_last, 2 evict_first)
  // digit-mapped (GETT / TC) operands read in place through 5-D TMA maps ta[0] / tb[0] (pair kernel):
  // 0 none, 1 MN-major {64, K0, MN0/64, MN1, K1}, 2 K-major {64, MN0, MN1, K0/64, K1}; e0 / f0 =
  // extent of the operand's fastest MN / K digit
  int32_t a_g, b_g, ga_e0, ga_f0, gb_e0, gb_f0;  // complex embedding: ta[0] maps A^ for the staging ring (tc_gemm_pair_kernel EMB)
};

// the 4 MMA-step bits of k-block kb of pair tile `tile` (0xF without a predicate)
__device__ __forceinline__ uint32_t kmask4(const TcParams& p, int tile, int kb) {
  if (!p.kbits) return 0xFu;
  return (__ldg(p.kbits + int64_t(tile) * p.kwords + (kb >> 3)) >> ((kb & 7) * 4)) & 0xFu;
}
// every step of the tile masked off: the accumulator is never written, the epilogue adds -0
__device__ __forceinline__ bool tile_masked_out(const TcParams& p, int tile) {
  if (!p.kbits) return false;
  for (int w = 0; w < p.kwords; ++w)
    if (__ldg(p.kbits + int64_t(tile) * p.kwords + w)) return false;
  return true;
}
// -0.0 is the additive identity for every FP32 value (c + -0 == c, -0 + -0 == -0): a tile
// whose every block-K iteration was skipped keeps acc = g2s_c(C) exactly as the reference
__device__ __forceinline__ void zero_acc(uint32_t (&r)[32], bool z) {
  if (z) {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) r[jj] = 0x80000000u;
  }
}

__device__ __forceinline__ void tile_coords(const TcParams& p, int t, int& mb, int& nb) {
  const int per_group = p.group_m * p.num_nb;
  const int g = t / per_group;
  const int first = g * p.group_m;
  const int gm = min(p.num_mb - first, p.group_m);
  const int r = t - g * per_group;
  mb = first + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ void k_range(const TcParams& p, int mb, int& kb0, int& kb1) {
  if (p.diag_a) {  // only block-K iterations that intersect the diagonal of A
    kb0 = (mb * TC_BM) / TC_BK;
    kb1 = min(p.kb_total, (mb * TC_BM + TC_BM + TC_BK - 1) / TC_BK);
  } else {
    kb0 = 0;
    kb1 = p.kb_total;
  }
}

// Fabricate the K-major, 128B-swizzled 128x64 A tile of diag(a) for rows [m0, m0+128),
// columns [k0, k0+64).  Written by one warp with 16-byte stores.
template <typename HT>
__device__ __forceinline__ void write_diag_tile(uint8_t* dst, const HT* diag, int m0, int k0,
                                                int m, int lane) {
  for (int idx = lane; idx < TC_BM * 8; idx += 32) {
    const int row = idx >> 3, chunk = idx & 7;  // physical 16B chunk of a 128B row
    const int logical_chunk = chunk ^ (row & 7);
    uint4 v = make_uint4(0, 0, 0, 0);
    const int gi = m0 + row;
    const int kk = gi - k0;  // diagonal column inside this k-block
    if (gi < m && kk >= 0 && kk < TC_BK && (kk >> 3) == logical_chunk) {
      uint16_t bits = reinterpret_cast<const uint16_t*>(diag)[gi];
      uint32_t word = (kk & 1) ? (uint32_t(bits) << 16) : uint32_t(bits);
      const int w = (kk & 7) >> 1;
      if (w == 0) v.x = word;
      else if (w == 1) v.y = word;
      else if (w == 2) v.z = word;
      else v.w = word;
    }
    *reinterpret_cast<uint4*>(dst + row * 128 + chunk * 16) = v;
  }
}


// diagnostic: globaltimer stamps of one CTA (TcParams::dbg_cta) of the last pair-kernel launch:
// 0 entry, 1 prologue done, 2 first stage full, 3 last MMA issued, 4 last accumulator full,
// 5 epilogue done, 6 stores drained, 7 exit; 8.. inside the epilogue of warp 4 (first chunk:
// TMEM loaded, math done, store issued)
__device__ unsigned long long g_dbg_ts[16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifndef TK_STAMPS
#define TK_STAMPS 0  // CTA timestamps for tools/ts_probe.py (build with -DTK_STAMPS=1): ~60 ns per K block on the MMA thread
#endif
#define TK_TS(i) do { if (TK_STAMPS && blockIdx.x == p.dbg_cta) g_dbg_ts[i] = gtimer(); } while (0)
// stamps builds: the latest value over all CTAs of a launch (globaltimer only grows)
#define TK_TSMAX(i) do { if (TK_STAMPS) atomicMax(&g_dbg_ts[i], gtimer()); } while (0)
#define TK_TS_EPI(i) do { if (TK_STAMPS && blockIdx.x == p.dbg_cta && (threadIdx.x >> 5) == 4 && (threadIdx.x & 31) == 0) g_dbg_ts[i] = gtimer(); } while (0)

// Split-K partials to fold into the accumulator before the epilogue: this thread's row of the
// first partial block (column stride 128), n blocks `pstride` floats apart, summed in order.
struct SkIn {
  const float* p;
  int n;
  int64_t pstride;
};
// sum of the partials of 32 consecutive columns starting at `col` (all loads issued before
// any use, so their latency overlaps the TMEM load instead of stalling element by element)
__device__ __forceinline__ void sk_gather(const SkIn& sk, int col, float (&pv)[32]) {
  const float* q = sk.p + int64_t(col) * 128;
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) pv[jj] = __ldcg(q + jj * 128);
  for (int s = 1; s < sk.n; ++s) {
    float t[32];
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) t[jj] = __ldcg(q + s * sk.pstride + jj * 128);
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) pv[jj] += t[jj];
  }
}

__device__ __forceinline__ float relu_if(float v, int on) { return on ? np_relu(v) : v; }

// The fused real epilogue on one 32-column chunk (row = lane), in the reference's order
// (components.py:110-157): v = acc [+ split-K partials]; + t_c(C); r2s; + bias; s2g.
// Uniform decisions are taken once per chunk (a branch around every element's shuffle costs
// ~1 us per chunk), the per-element arithmetic is unchanged.
template <bool SK>
__device__ __forceinline__ void epi_math_real(const TcParams& p, const uint32_t (&r)[32],
                                              const float (&cv)[32], const float (&pv)[SK ? 32 : 1],
                                              bool has_c, float bias_m, float bcol, float (&out)[32]) {
  float v[32];
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) v[jj] = __uint_as_float(r[jj]);
  if constexpr (SK) {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) v[jj] = pv[jj] + v[jj];
  }
  if (has_c) {
    if (p.c_ident) {  // identity g2s_c (the reference's default): acc starts from C itself
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) v[jj] = cv[jj] + v[jj];
    } else {
      const float cm = p.c_mul[0], ca = p.c_add[0];
      const int cr = p.c_relu;
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) v[jj] = relu_if(cv[jj] * cm + ca, cr) + v[jj];
    }
  }
  if (!p.r_ident) {
    const float rm = p.r_mul[0], ra = p.r_add[0];
    const int rr = p.r_relu;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) v[jj] = relu_if(v[jj] * rm + ra, rr);
  }
  if (p.bias_axis == 1) {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) v[jj] = v[jj] + __shfl_sync(0xffffffffu, bcol, jj);
  } else if (p.bias_axis == 2) {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) v[jj] = v[jj] + bias_m;
  }
  if (!p.s_ident) {
    const float sm = p.s_mul[0], sa = p.s_add[0];
    const int sr = p.s_relu;
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) out[jj] = relu_if(v[jj] * sm + sa, sr);
  } else {
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) out[jj] = v[jj];
  }
}

// ---------------------------------------------------------------- epilogue bodies

// Dense column-major C/D, transforms pre-decoded to affine(+relu).  Per warp: 32 rows (one
// per lane, TMEM lane quarter) x COLS columns in chunks of 32; C for the next chunk is in
// flight while the current chunk computes and stores (streaming cache hints: C and D are
// touched once and must not evict the A/B panels from L2).
// OP_SPLIT: the second accumulator (BN columns on) is added to the first when `eps` is set.
template <int OP, int BN>
__device__ __forceinline__ void split_sum(uint32_t (&r)[32], uint32_t taddr, bool eps) {
  if constexpr (OP == OP_SPLIT) {
    if (eps) {
      uint32_t r1[32];
      tmem_ld_32x32b_x32(taddr + uint32_t(BN), r1);
      tmem_ld_wait();
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) r[jj] = __float_as_uint(__uint_as_float(r[jj]) + __uint_as_float(r1[jj]));
    }
  }
}

template <int OP, int COLS, int BN, bool SK = false>
__device__ __forceinline__ void epilogue_dense(const TcParams& p, uint64_t* tfull, uint32_t aphase,
                                               uint32_t tbase, int i, int jbase, int lane,
                                               SkIn sk = SkIn{nullptr, 0, 0}, bool eps = false,
                                               bool masked = false) {
  const bool row_ok = i < p.m;
  const bool has_c = !p.c_zero;
  if (OP == OP_REAL || OP == OP_SPLIT) {
    const int64_t crow = !row_ok ? 0 : p.c_rmap ? map_dim(p.c_map, 0, i) : i;
    const int64_t drow = !row_ok ? 0 : p.d_rmap ? map_dim(p.d_map, 0, i) : i;
    const float* cp = reinterpret_cast<const float*>(p.c_ptr) + crow;
    float* dp = reinterpret_cast<float*>(p.d_ptr) + drow;
    const float bias_m = (p.bias_axis == 2 && row_ok) ? p.bias[i] : 0.f;
    float cv[32];
    auto load_c = [&](int j0) {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) {
        const int j = j0 + jj;
        cv[jj] = (has_c && row_ok && j < p.n) ? __ldcs(cp + int64_t(j) * p.ldc) : 0.f;
      }
    };
    load_c(jbase);
    mbar_wait_sleep(tfull, aphase);
    tc_fence_after();
#pragma unroll 1
    for (int ch = 0; ch < COLS / 32; ++ch) {
      const int j0 = jbase + ch * 32;
      uint32_t r[32];
      const uint32_t taddr = tbase + uint32_t(j0 - jbase + (jbase % BN));
      tmem_ld_32x32b_x32(taddr, r);
      // lane-distributed bias[j] broadcast with shuffles
      const int jl = j0 + lane;
      const float bcol = (p.bias_axis == 1 && jl < p.n) ? p.bias[jl] : 0.f;
      float pv[SK ? 32 : 1];
      if constexpr (SK) sk_gather(sk, j0 - jbase + (jbase % BN), pv);
      tmem_ld_wait();
      split_sum<OP, BN>(r, taddr, eps);
      zero_acc(r, masked);
      float out[32];
      epi_math_real<SK>(p, r, cv, pv, has_c, bias_m, bcol, out);
      if (ch + 1 < COLS / 32) load_c(j0 + 32);
      if (row_ok) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          if (j0 + jj < p.n) __stcs(dp + int64_t(j0 + jj) * p.ldd, out[jj]);
      }
    }
  } else {
    // pair operators: interleaved (float2) or split planes, column-major elements.  16-column
    // steps (two x16 TMEM loads) keep the Re/Im accumulators, C and D in registers without
    // spills; the next step's C is in flight while this one computes and stores.
    constexpr int W = 16;
    const float* cp = reinterpret_cast<const float*>(p.c_ptr);
    float* dp = reinterpret_cast<float*>(p.d_ptr);
    const int64_t ci = row_ok ? i : 0;
    float2 cv[W];
    auto load_c = [&](int j0) {
#pragma unroll
      for (int jj = 0; jj < W; ++jj) {
        const int j = j0 + jj;
        cv[jj] = make_float2(0.f, 0.f);
        if (has_c && row_ok && j < p.n) {
          const int64_t e = ci + int64_t(j) * p.ldc;
          cv[jj] = p.c_pair == P_INTERLEAVED ? __ldcs(reinterpret_cast<const float2*>(cp) + e)
                                             : make_float2(__ldcs(cp + e), __ldcs(cp + e + p.c_plane));
        }
      }
    };
    load_c(jbase);
    mbar_wait_sleep(tfull, aphase);
    tc_fence_after();
#pragma unroll 1
    for (int ch = 0; ch < COLS / W; ++ch) {
      const int j0 = jbase + ch * W;
      const uint32_t col = uint32_t(j0 - jbase + (jbase % BN));
      uint32_t r0[W], r1[W];
      tmem_ld_32x32b_x16(tbase + col, r0);
      tmem_ld_32x32b_x16(tbase + uint32_t(BN) + col, r1);
      tmem_ld_wait();
      float2 v[W];
#pragma unroll
      for (int jj = 0; jj < W; ++jj) {
        float2 x = make_float2(__uint_as_float(r0[jj]), __uint_as_float(r1[jj]));
        if (has_c) {
          if (p.c_ident) {
            x = make_float2(cv[jj].x + x.x, cv[jj].y + x.y);
          } else {
            const float cr = cv[jj].x * p.c_mul[0] - cv[jj].y * p.c_mul[1] + p.c_add[0];
            const float ci_ = cv[jj].x * p.c_mul[1] + cv[jj].y * p.c_mul[0] + p.c_add[1];
            x = make_float2(cr + x.x, ci_ + x.y);
          }
        }
        if (!p.r_ident)
          x = make_float2(x.x * p.r_mul[0] - x.y * p.r_mul[1] + p.r_add[0],
                          x.x * p.r_mul[1] + x.y * p.r_mul[0] + p.r_add[1]);
        if (!p.s_ident)
          x = make_float2(x.x * p.s_mul[0] - x.y * p.s_mul[1] + p.s_add[0],
                          x.x * p.s_mul[1] + x.y * p.s_mul[0] + p.s_add[1]);
        v[jj] = x;
      }
      if (ch + 1 < COLS / W) load_c(j0 + W);
#pragma unroll
      for (int jj = 0; jj < W; ++jj) {
        const int j = j0 + jj;
        if (row_ok && j < p.n) {
          const int64_t e = ci + int64_t(j) * p.ldd;
          if (p.d_pair == P_INTERLEAVED) {
            __stcs(reinterpret_cast<float2*>(dp) + e, v[jj]);
          } else {
            __stcs(dp + e, v[jj].x);
            __stcs(dp + e + p.d_plane, v[jj].y);
          }
        }
      }
    }
  }
}


// Release ring use cq - LAG once the stores committed after it no longer need their slots' data:
// `smask` bit i says whether use cq - i committed a TMA store (split-K rings mix store uses with
// partial-read uses, so the number of groups allowed in flight varies).  Lane 0 only.
template <int CSLOTS>
__device__ __forceinline__ void ring_release(uint64_t* cempty, uint32_t cq, uint32_t smask) {
  static_assert(CSLOTS <= 4, "LAG <= 3");
  constexpr int LAG = CSLOTS >= 4 ? CSLOTS - 1 : 1;
  if (cq < uint32_t(LAG)) return;
  switch (__popc(smask & ((1u << LAG) - 1u))) {
    case 0: bulk_wait_read<0>(); break;
    case 1: bulk_wait_read<1>(); break;
    case 2: bulk_wait_read<2>(); break;
    default: bulk_wait_read<3>(); break;
  }
  mbar_arrive(&cempty[(cq - LAG) % CSLOTS]);
}

// Dense column-major epilogue for HBM-bound shapes: C arrives in a per-warp ring of TMA boxes
// filled by the loader warp; D is written back into the same slot and stored with one TMA
// bulk store per 32x32 box (the slot is handed back to the loader once that store has read it).
template <int COLS, int BN, int CSLOTS = TC_CSLOTS, bool SK = false>
__device__ __forceinline__ void epilogue_stream(const TcParams& p, uint64_t* tfull, uint32_t aphase,
                                                uint32_t tbase, int i, int jbase, int lane,
                                                float* ring, uint64_t* cfull, uint64_t* cempty,
                                                uint32_t& cq, int row0, SkIn sk = SkIn{nullptr, 0, 0},
                                                uint32_t* smask = nullptr, bool masked = false) {
  const bool row_ok = i < p.m;
  const bool has_c = !p.c_zero;
  float* dp = reinterpret_cast<float*>(p.d_ptr) + (row_ok ? i : 0);
  const float bias_m = (p.bias_axis == 2 && row_ok) ? p.bias[i] : 0.f;
  mbar_wait_sleep(tfull, aphase);
  tc_fence_after();
#pragma unroll 1
  for (int ch = 0; ch < COLS / 32; ++ch) {
    const int j0 = jbase + ch * 32;
    uint32_t r[32];
    tmem_ld_32x32b_x32(tbase + uint32_t(j0 - jbase + (jbase % BN)), r);
    const int jl = j0 + lane;
    const float bcol = (p.bias_axis == 1 && jl < p.n) ? p.bias[jl] : 0.f;
    float pv[SK ? 32 : 1];
    if constexpr (SK) {
      if (p.sk_tma) {
        // the other K-parts' partial boxes come through the ring ahead of this chunk's C box
        // (summed in part order, as sk_gather does); each slot is handed back one use later
        for (int s = 0; s < sk.n; ++s, ++cq) {
          const uint32_t sl = cq % CSLOTS;
          const uint32_t bs = smem_u32(ring + sl * (TC_CBOX_BYTES / 4));
          mbar_wait(&cfull[sl], (cq / CSLOTS) & 1);
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const float v = lds_f32(bs + uint32_t(jj * 32 + lane) * 4u);
            pv[jj] = s ? pv[jj] + v : v;
          }
          __syncwarp();
          *smask <<= 1;  // a read use: no store
          if (lane == 0) ring_release<CSLOTS>(cempty, cq, *smask);
        }
      }
    }
    const uint32_t slot = cq % CSLOTS;
    float* box = ring + slot * (TC_CBOX_BYTES / 4);
    const uint32_t box_s = smem_u32(box);  // explicit shared-space accesses (box is a generic pointer)
    float cv[32];
    if (has_c) {
      mbar_wait(&cfull[slot], (cq / CSLOTS) & 1);
      if (ch == 0) TK_TS_EPI(11);
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) cv[jj] = lds_f32(box_s + uint32_t(jj * 32 + lane) * 4u);
    } else if (p.d_tma) {
      if (lane == 0) bulk_wait_read<CSLOTS - 1>();  // slot's previous store has read it
      __syncwarp();
    }
    if constexpr (SK) {
      if (!p.sk_tma) sk_gather(sk, j0 - jbase + (jbase % BN), pv);
    }
    tmem_ld_wait();
    zero_acc(r, masked);
    if (ch == 0) TK_TS_EPI(8);
    float out[32];
    epi_math_real<SK>(p, r, cv, pv, has_c, bias_m, bcol, out);
    if (ch == 0) TK_TS_EPI(9);
    if (p.d_tma) {
#pragma unroll
      for (int jj = 0; jj < 32; ++jj) sts_f32(box_s + uint32_t(jj * 32 + lane) * 4u, out[jj]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (p.pol_d)  // L2 hint for the D stream (tuning: TK_POL_D)
          tma_store_2d_hint(&p.tdmap, box, row0, j0, policy_code(p.pol_d));
        else
          tma_store_2d(&p.tdmap, box, row0, j0);  // the map clips rows >= M / columns >= N
        for (int q = 0; q < p.npeer; ++q) tma_store_2d(&p.tdpeer[q], box, row0, j0);  // peers (NVLink)
        bulk_commit();
        if (ch == 0) TK_TS_EPI(10);
        if (has_c) {
          // hand a slot back once its store has read it.  Streaming rings release the previous
          // chunk's slot (the loader runs one chunk ahead); a deep ring (>= 4 slots, used when
          // the whole C block is prefetched) lets CSLOTS-1 stores stay in flight instead
          constexpr int LAG = CSLOTS >= 4 ? CSLOTS - 1 : 1;
          if (SK && p.sk_tma) {
            ring_release<CSLOTS>(cempty, cq, (*smask << 1) | 1u);
          } else {
            bulk_wait_read<LAG>();
            if (cq >= uint32_t(LAG)) mbar_arrive(&cempty[(cq - LAG) % CSLOTS]);
          }
        }
      }
    } else {
      if (has_c) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[slot]);
      }
      if (row_ok) {
#pragma unroll
        for (int jj = 0; jj < 32; ++jj)
          if (j0 + jj < p.n) __stcs(dp + int64_t(j0 + jj) * p.ldd, out[jj]);
      }
    }
    if (SK && p.sk_tma) *smask = (*smask << 1) | 1u;  // a store use
    ++cq;
  }
}

// Any digit-mapped C/D layout and any transform program (the rare path).
template <int OP, int COLS, int BN>
__device__ __noinline__ void epilogue_generic(const TcParams& p, uint64_t* tfull, uint32_t aphase,
                                              uint32_t tbase, int i, int jbase, bool eps = false,
                                              bool masked = false) {
  const bool row_ok = i < p.m;
  const int64_t c_row = row_ok ? map_dim(p.c_map, 0, i) : 0;
  const int64_t d_row = row_ok ? map_dim(p.d_map, 0, i) : 0;
  const float bias_m = (p.bias_axis == 2 && row_ok) ? p.bias[i] : 0.f;
  mbar_wait_sleep(tfull, aphase);
  tc_fence_after();
#pragma unroll 1
  for (int ch = 0; ch < COLS / 32; ++ch) {
    const int j0 = jbase + ch * 32;
    const uint32_t col = uint32_t(j0 - jbase + (jbase % BN));
    uint32_t r0[32], r1[32];
    tmem_ld_32x32b_x32(tbase + col, r0);
    if (OP == OP_COMPLEX || OP == OP_DUAL) tmem_ld_32x32b_x32(tbase + uint32_t(BN) + col, r1);
    tmem_ld_wait();
    split_sum<OP, BN>(r0, tbase + col, eps);
    zero_acc(r0, masked);
#pragma unroll 1
    for (int jj = 0; jj < 32; ++jj) {
      const int j = j0 + jj;
      if (!row_ok || j >= p.n) continue;
      if (OP == OP_REAL || OP == OP_SPLIT) {
        float v = __uint_as_float(r0[jj]);
        if (!p.c_zero) v = run_prog_real(p.t_c, load_scalar_f32(p.c_ptr, c_row + map_dim(p.c_map, 1, j))) + v;
        v = run_prog_real(p.t_r2s, v);
        if (p.bias_axis == 1) v = v + p.bias[j];
        else if (p.bias_axis == 2) v = v + bias_m;
        v = run_prog_real(p.t_s2g, v);
        reinterpret_cast<float*>(p.d_ptr)[d_row + map_dim(p.d_map, 1, j)] = v;
      } else {
        float2 v = make_float2(__uint_as_float(r0[jj]), __uint_as_float(r1[jj]));
        if (!p.c_zero) {
          float2 cv = load_pair_f32(p.c_ptr, p.c_pair, p.c_plane, c_row + map_dim(p.c_map, 1, j));
          cv = run_prog_pair<OP>(p.t_c, cv);
          v = make_float2(cv.x + v.x, cv.y + v.y);
        }
        v = run_prog_pair<OP>(p.t_r2s, v);
        v = run_prog_pair<OP>(p.t_s2g, v);
        store_pair_f32(p.d_ptr, p.d_pair, p.d_plane, d_row + map_dim(p.d_map, 1, j), v);
      }
    }
  }
}

template <int OP, bool DENSE_EPI, int CSTREAM = 0>
__global__ void __launch_bounds__(TC_THREADS, 1) tc_gemm_kernel(const __grid_constant__ TcParams p) {
  using C = TcCfg<OP>;
  using S = TcSmem<OP, CSTREAM>;
  constexpr int BN = C::BN;
  constexpr int STAGES = S::STAGES;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFFSET);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* cfull = tempty + 2;            // [epilogue warp][slot] (C-streaming only)
  uint64_t* cempty = cfull + S::NCBAR;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + S::NCBAR);
  float* cring = reinterpret_cast<float*>(smem + S::CRING_OFFSET);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    if (CSTREAM && !p.c_zero) tma_prefetch(&p.tcmap);
    if (!p.diag_a) {
      tma_prefetch(&p.ta[0]);
      if (C::PLANES > 1) tma_prefetch(&p.ta[1]);
    }
    tma_prefetch(&p.tb[0]);
    if (C::PLANES > 1) tma_prefetch(&p.tb[1]);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], TC_EPI_WARPS);
    }
    for (int s = 0; s < S::NCBAR; ++s) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // OP_SPLIT: which lo planes are non-zero (the others are neither loaded nor multiplied)
  const bool lo_a = OP != OP_SPLIT || p.split_flags[0] != 0;
  const bool lo_b = OP != OP_SPLIT || p.split_flags[1] != 0;

  auto a_tile = [&](int s, int plane) -> uint8_t* {
    return smem + s * S::STAGE_BYTES + plane * TC_A_TILE_BYTES;
  };
  auto b_tile = [&](int s, int plane) -> uint8_t* {
    return smem + s * S::STAGE_BYTES + C::PLANES * TC_A_TILE_BYTES + plane * S::B_TILE_BYTES;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    const uint64_t pol_a = p.pol_ab ? policy_evict_last() : policy_evict_normal();
    const uint64_t pol_b = pol_a;
    const uint32_t a_bytes = p.diag_a ? 0u : uint32_t(TC_A_TILE_BYTES * (C::PLANES == 1 ? 1 : 1 + lo_a));
    const uint32_t tx_bytes = a_bytes + uint32_t(S::B_TILE_BYTES * (C::PLANES == 1 ? 1 : 1 + lo_b));
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int mb, nb, kb0, kb1;
      tile_coords(p, t, mb, nb);
      k_range(p, mb, kb0, kb1);
      const int m0 = mb * TC_BM, n0 = nb * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        const int k0 = kb * TC_BK;
        mbar_wait(&empty[stage], phase ^ 1);
        if (p.diag_a) {
          if (p.ab_fmt == 0)
            write_diag_tile(a_tile(stage, 0), reinterpret_cast<const __half*>(p.diag), m0, k0,
                            p.m, lane);
          else
            write_diag_tile(a_tile(stage, 0), reinterpret_cast<const __nv_bfloat16*>(p.diag),
                            m0, k0, p.m, lane);
          fence_proxy_async_smem();
          __syncwarp();
        }
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[stage], tx_bytes);
#pragma unroll
          for (int pl = 0; pl < C::PLANES; ++pl) {
            if (!p.diag_a && (pl == 0 || lo_a)) {
              if (p.a_mn) {  // column-major A: two 64-row boxes (M inner)
                tma_load_2d(a_tile(stage, pl), &p.ta[pl], &full[stage], m0, k0, pol_a);
                tma_load_2d(a_tile(stage, pl) + 8192, &p.ta[pl], &full[stage], m0 + 64, k0, pol_a);
              } else {       // row-major A: one box, K inner
                tma_load_2d(a_tile(stage, pl), &p.ta[pl], &full[stage], k0, m0, pol_a);
              }
            }
            if (pl == 1 && !lo_b) {
              // (OP_SPLIT) zero lo plane of B: not loaded
            } else if (p.b_mn) {    // row-major B: BN/64 boxes, N inner
#pragma unroll
              for (int h = 0; h < BN / 64; ++h)
                tma_load_2d(b_tile(stage, pl) + h * 8192, &p.tb[pl], &full[stage], n0 + 64 * h, k0,
                            pol_b);
            } else {         // column-major B: one box, K inner
              tma_load_2d(b_tile(stage, pl), &p.tb[pl], &full[stage], k0, n0, pol_b);
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t a_mn = p.diag_a ? 0u : uint32_t(p.a_mn);
      const uint32_t idesc = idesc_f16(p.ab_fmt, a_mn, p.b_mn, 0, TC_BM, BN);
      const uint32_t idesc_neg = idesc_f16(p.ab_fmt, a_mn, p.b_mn, 1, TC_BM, BN);
      // per K=16 step: K-major advances 32 B inside the swizzle atom, MN-major 2 atoms (2 KB)
      const uint32_t a_step = a_mn ? 2048u : 32u;
      const uint32_t b_step = p.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = a_mn ? 8192u : 16u;
      const uint32_t b_lbo = p.b_mn ? 8192u : 16u;
      // descriptors built once; per MMA only the start-address field advances (16-byte units,
      // no carry: shared memory < 256 KB)
      const uint64_t a0d = sdesc_sw128(smem_u32(a_tile(0, 0)), a_lbo, 1024);
      const uint64_t b0d = sdesc_sw128(smem_u32(b_tile(0, 0)), b_lbo, 1024);
      const uint64_t a1d = a0d + uint32_t(TC_A_TILE_BYTES >> 4);
      const uint64_t b1d = b0d + uint32_t(S::B_TILE_BYTES >> 4);
      const uint32_t a_kk = a_step >> 4, b_kk = b_step >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++local) {
        int mb, nb, kb0, kb1;
        tile_coords(p, t, mb, nb);
        k_range(p, mb, kb0, kb1);
        const int as = local & 1;
        const uint32_t aphase = (local >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem_base + uint32_t(as * C::ACC_COLS);
        const uint32_t d1 = d0 + uint32_t(BN);  // second accumulator (Im / epsilon)
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t so = uint32_t(stage) * uint32_t(S::STAGE_BYTES >> 4);
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            const uint32_t acc = (kb > kb0 || kk > 0) ? 1u : 0u;
            const uint64_t a0 = a0d + so + kk * a_kk;
            const uint64_t b0 = b0d + so + kk * b_kk;
            if (OP == OP_REAL) {
              tc_mma_f16(d0, a0, b0, idesc, acc);
            } else {
              const uint64_t a1 = a1d + so + kk * a_kk;
              const uint64_t b1 = b1d + so + kk * b_kk;
              if (OP == OP_COMPLEX) {
                tc_mma_f16(d0, a0, b0, idesc, acc);      // Re += Ar*Br
                tc_mma_f16(d0, a1, b1, idesc_neg, 1u);   // Re += (-Ai)*Bi
                tc_mma_f16(d1, a0, b1, idesc, acc);      // Im += Ar*Bi
                tc_mma_f16(d1, a1, b0, idesc, 1u);       // Im += Ai*Br
              } else if (OP == OP_DUAL) {
                tc_mma_f16(d0, a0, b0, idesc, acc);      // v   += Av*Bv
                tc_mma_f16(d1, a0, b1, idesc, acc);      // eps += Av*Beps
                tc_mma_f16(d1, a1, b0, idesc, 1u);       // eps += Aeps*Bv
              } else {                                   // OP_SPLIT
                tc_mma_f16(d0, a0, b0, idesc, acc);      // hi*hi
                if (lo_b) tc_mma_f16(d1, a0, b1, idesc, acc);            // hi*lo
                if (lo_a) tc_mma_f16(d1, a1, b0, idesc, lo_b ? 1u : acc);  // lo*hi
              }
            }
          }
          tc_commit(&empty[stage]);  // smem slot free once these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[as]);       // accumulator ready for the epilogue
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ C loader (C-streaming)
    if (CSTREAM && !p.c_zero && lane == 0) {
      constexpr int CHUNKS = BN / 2 / 32;
      uint32_t q = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(p, t, mb, nb);
        for (int ch = 0; ch < CHUNKS; ++ch, ++q) {
          const uint32_t slot = q % S::CSLOTS, ph = (q / S::CSLOTS) & 1;
          for (int w = 0; w < TC_EPI_WARPS; ++w) {
            const int bi = w * S::CSLOTS + int(slot);
            mbar_wait(&cempty[bi], ph ^ 1);
            mbar_arrive_expect_tx(&cfull[bi], TC_CBOX_BYTES);
            const int row0 = mb * TC_BM + (w & 3) * 32;
            const int col0 = nb * BN + (w >> 2) * (BN / 2) + ch * 32;
            tma_load_2d(smem + S::CRING_OFFSET + bi * TC_CBOX_BYTES, &p.tcmap, &cfull[bi], row0,
                        col0, policy_evict_normal());
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;
    uint32_t cq = 0;
    const int quarter = warp & 3;          // TMEM lane quarter this warp may access
    const int half = ew >> 2;              // which half of the tile's columns
    const int row_local = quarter * 32 + lane;
    constexpr int COLS_PER_WARP = BN / 2;
    int local = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++local) {
      int mb, nb;
      tile_coords(p, t, mb, nb);
      const int as = local & 1;
      const uint32_t aphase = (local >> 1) & 1;
      const int i = mb * TC_BM + row_local;
      const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(as * C::ACC_COLS);
      const int jbase = nb * BN + half * COLS_PER_WARP;
      if (CSTREAM)
        epilogue_stream<COLS_PER_WARP, BN, S::CSLOTS>(p, tfull + as, aphase, tbase, i, jbase, lane,
                                           cring + ew * S::CSLOTS * (TC_CBOX_BYTES / 4),
                                           cfull + ew * S::CSLOTS, cempty + ew * S::CSLOTS, cq,
                                           mb * TC_BM + quarter * 32);
      else if (DENSE_EPI)
        epilogue_dense<OP, COLS_PER_WARP, BN>(p, tfull + as, aphase, tbase, i, jbase, lane,
                                              SkIn{nullptr, 0, 0}, lo_a || lo_b);
      else
        epilogue_generic<OP, COLS_PER_WARP, BN>(p, tfull + as, aphase, tbase, i, jbase, lo_a || lo_b);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
    }
  }

  if (CSTREAM && warp >= 4 && lane == 0) bulk_wait_read<0>();  // ring read; grid completion performs the stores
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace tk

namespace tk {

// Diagonal A (reference build_diagonal_config / Diagonal layout, layouts.py:191-252, with the
// DiagonalPredicate skipping every block-K iteration that misses the diagonal,
// components.py:177-191): D = epi(C + diag(a) B) is a pure HBM stream -- 2 bytes of B and
// 4 + 4 bytes of C and D per element, one multiply -- so it runs as a vectorised streaming
// kernel instead of occupying the tensor cores with 127/128 zero columns.  The arithmetic is
// the tcgen05 path's: the product a_i * b_ij of two halves is exact in FP32 (the MMA adds only
// exact zeros to it), then the same epilogue sequence as epilogue_dense.
template <typename H>
__global__ void __launch_bounds__(256) diag_stream_kernel(const __grid_constant__ TcParams p,
                                                          const H* __restrict__ b, int64_t ldb) {
  const H* diag = reinterpret_cast<const H*>(p.diag);
  const float* cp = reinterpret_cast<const float*>(p.c_ptr);
  float* dp = reinterpret_cast<float*>(p.d_ptr);
  const bool has_c = !p.c_zero;
  const int64_t rows4 = (int64_t(p.m) + 3) / 4;
  const int64_t kdiag = p.k < p.m ? p.k : p.m;  // rows with a diagonal entry
  auto epi = [&](float acc, float c, float bias) {  // epi_math_real, one element
    float v = acc;
    if (has_c) v = (p.c_ident ? c : relu_if(c * p.c_mul[0] + p.c_add[0], p.c_relu)) + v;
    if (!p.r_ident) v = relu_if(v * p.r_mul[0] + p.r_add[0], p.r_relu);
    if (p.bias_axis) v = v + bias;
    return p.s_ident ? v : relu_if(v * p.s_mul[0] + p.s_add[0], p.s_relu);
  };
  for (int64_t j = blockIdx.y; j < p.n; j += gridDim.y) {
    const float bias_j = p.bias_axis == 1 ? p.bias[j] : 0.f;
    for (int64_t r4 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r4 < rows4; r4 += int64_t(gridDim.x) * blockDim.x) {
      const int64_t i0 = r4 * 4;
      if (p.vec_ok && i0 + 4 <= kdiag) {  // vector path: 4 rows, all on the diagonal, aligned
        const uint2 bv = __ldcs(reinterpret_cast<const uint2*>(b + i0 + j * ldb));
        const uint2 av = *reinterpret_cast<const uint2*>(diag + i0);
        const float4 cv = has_c ? __ldcs(reinterpret_cast<const float4*>(cp + i0 + j * p.ldc))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
        const H* bh = reinterpret_cast<const H*>(&bv);
        const H* ah = reinterpret_cast<const H*>(&av);
        float4 o;
        o.x = epi(__fmul_rn(h2f(ah[0]), h2f(bh[0])), cv.x, p.bias_axis == 2 ? p.bias[i0] : bias_j);
        o.y = epi(__fmul_rn(h2f(ah[1]), h2f(bh[1])), cv.y, p.bias_axis == 2 ? p.bias[i0 + 1] : bias_j);
        o.z = epi(__fmul_rn(h2f(ah[2]), h2f(bh[2])), cv.z, p.bias_axis == 2 ? p.bias[i0 + 2] : bias_j);
        o.w = epi(__fmul_rn(h2f(ah[3]), h2f(bh[3])), cv.w, p.bias_axis == 2 ? p.bias[i0 + 3] : bias_j);
        __stcs(reinterpret_cast<float4*>(dp + i0 + j * p.ldd), o);
      } else {
        for (int64_t i = i0; i < i0 + 4 && i < p.m; ++i) {
          const float acc = i < kdiag ? __fmul_rn(h2f(diag[i]), h2f(b[i + j * ldb])) : 0.f;
          const float c = has_c ? cp[i + j * p.ldc] : 0.f;
          dp[i + j * p.ldd] = epi(acc, c, p.bias_axis == 2 ? p.bias[i] : bias_j);
        }
      }
    }
  }
}

}  // namespace tk
