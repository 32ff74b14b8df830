// tk_simt.cuh -- the bit-exact CUDA-core lane.
//
// Reproduces the reference's arithmetic *order* exactly, so f32/f64/complex/dual results are
// bitwise equal to the CPU reference (and to the oracle restatement in oracle/tk_oracle.c):
//   acc = g2s_c(C) (stored at C's precision, then widened to the compute type)
//   real:    for k ascending: acc = acc + a*b            (_core.pyx:16-68, separate mul/add)
//   complex: per operator-K chunk: Re += sum ar*br; neg = sum ai*bi; Re -= neg;
//            Im += sum ar*bi; Im += sum ai*br          (operators.py:152-163)
//   dual:    per chunk: v += sum av*bv; e += sum av*be; e += sum ae*bv  (operators.py:180-188)
//   D = s2g( r2s(acc) rounded to D's precision + bias )  (kernel.py:446-463, components.py:139-157)
// with g2s transforms applied to every A/B element (components.py:97-105) and skipped
// block-K iterations honoured per logical block (kernel.py:399-404).
// Half-precision storage is widened exactly to f32 on load (the documented parity protocol).
// The lane also serves shapes/layouts the tcgen05 lane cannot take (unaligned strides,
// non-affine operand transforms, arbitrary predicates).
#pragma once
#include "tk_types.cuh"

namespace tk {

struct SimtLayout {
  int32_t kind, pair, scalar, pad;
  DigitMap map;
  int64_t plane;
  const void* ptr;
};

struct SimtParams {
  int64_t m, n, k, op_k;
  int64_t bm, bn, bk;
  int32_t predicate;  // 0 always, 1 diagonal, 2 mask
  int32_t bias_axis, bias_scalar, pad;
  const uint8_t* kmask;
  const void* bias;
  SimtLayout a, b, c, d;
  EpiProg t_a, t_b, t_c, t_r2s, t_s2g;
};

template <typename T>
__device__ __forceinline__ T load_as(const void* p, int scalar, int64_t off) {
  switch (scalar) {
    case S_F16: return T(__half2float(reinterpret_cast<const __half*>(p)[off]));
    case S_BF16: return T(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[off]));
    case S_F32: return T(reinterpret_cast<const float*>(p)[off]);
    default: return T(reinterpret_cast<const double*>(p)[off]);
  }
}

template <typename T>
__device__ __forceinline__ void store_as(void* p, int scalar, int64_t off, T v) {
  switch (scalar) {
    case S_F16: reinterpret_cast<__half*>(p)[off] = __float2half_rn(float(v)); break;
    case S_BF16: reinterpret_cast<__nv_bfloat16*>(p)[off] = __float2bfloat16_rn(float(v)); break;
    case S_F32: reinterpret_cast<float*>(p)[off] = float(v); break;
    default: reinterpret_cast<double*>(p)[off] = double(v); break;
  }
}

// Round a value held in T to the storage precision of `scalar` (values written to a
// scratch buffer of that dtype in the reference) and back.
template <typename T>
__device__ __forceinline__ T round_to(int scalar, T v) {
  switch (scalar) {
    case S_F16: return T(__half2float(__float2half_rn(float(v))));
    case S_BF16: return T(__bfloat162float(__float2bfloat16_rn(float(v))));
    case S_F32: return T(float(v));
    default: return v;
  }
}

// Element (i, j) of a real layout, widened to T.
template <typename T>
__device__ __forceinline__ T load_real(const SimtLayout& L, int64_t i, int64_t j) {
  if (L.kind == L_ZERO) return T(0);
  if (L.kind == L_DIAGONAL) return i == j ? load_as<T>(L.ptr, L.scalar, i) : T(0);
  return load_as<T>(L.ptr, L.scalar, map_dim(L.map, 0, i) + map_dim(L.map, 1, j));
}

template <typename T>
__device__ __forceinline__ Pair<T> load_pair(const SimtLayout& L, int64_t i, int64_t j) {
  if (L.kind == L_ZERO) return Pair<T>{T(0), T(0)};
  const int64_t off = map_dim(L.map, 0, i) + map_dim(L.map, 1, j);
  if (L.pair == P_INTERLEAVED)
    return Pair<T>{load_as<T>(L.ptr, L.scalar, 2 * off), load_as<T>(L.ptr, L.scalar, 2 * off + 1)};
  return Pair<T>{load_as<T>(L.ptr, L.scalar, off), load_as<T>(L.ptr, L.scalar, off + L.plane)};
}

template <typename T>
__device__ __forceinline__ void store_pair(const SimtLayout& L, int64_t i, int64_t j, Pair<T> v) {
  const int64_t off = map_dim(L.map, 0, i) + map_dim(L.map, 1, j);
  if (L.pair == P_INTERLEAVED) {
    store_as<T>(const_cast<void*>(L.ptr), L.scalar, 2 * off, v.x);
    store_as<T>(const_cast<void*>(L.ptr), L.scalar, 2 * off + 1, v.y);
  } else {
    store_as<T>(const_cast<void*>(L.ptr), L.scalar, off, v.x);
    store_as<T>(const_cast<void*>(L.ptr), L.scalar, off + L.plane, v.y);
  }
}

template <typename T>
__device__ __forceinline__ T prog(const EpiProg& g, T v) {
  return run_prog_real(g, v);
}

__device__ __forceinline__ bool k_block_runs(const SimtParams& p, int64_t i, int64_t j,
                                             int64_t kb) {
  if (p.predicate == 0) return true;
  const int64_t bi = i / p.bm;
  if (p.predicate == 1) {
    const int64_t m0 = bi * p.bm, k0 = kb * p.bk;
    return max(m0, k0) < min(m0 + p.bm, k0 + p.bk);
  }
  const int64_t rank = bi + (j / p.bn) * (p.m / p.bm);
  return p.kmask[rank * (p.k / p.bk) + kb] != 0;
}

// One thread per output element; T = stream precision, Acc = accumulator precision.
template <int OP, typename T, typename Acc>
__global__ void simt_gemm_kernel(const __grid_constant__ SimtParams p) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= p.m * p.n) return;
  const int64_t i = idx % p.m;  // column-major walk: consecutive threads, consecutive rows
  const int64_t j = idx / p.m;
  const int64_t nkb = p.k / p.bk;

  if (OP == OP_REAL) {
    T c0 = prog(p.t_c, load_real<T>(p.c, i, j));
    Acc acc = Acc(round_to(p.c.scalar, c0));
    for (int64_t kb = 0; kb < nkb; ++kb) {
      if (!k_block_runs(p, i, j, kb)) continue;
      for (int64_t k = kb * p.bk; k < (kb + 1) * p.bk; ++k) {
        const Acc a = Acc(prog(p.t_a, load_real<T>(p.a, i, k)));
        const Acc b = Acc(prog(p.t_b, load_real<T>(p.b, k, j)));
        acc = add_rn(acc, mul_rn(a, b));
      }
    }
    T v = T(round_to(p.d.scalar, prog(p.t_r2s, acc)));
    if (p.bias_axis)
      v = T(round_to(p.d.scalar, add_rn(v, load_as<T>(p.bias, p.bias_scalar, p.bias_axis == 1 ? j : i))));
    v = prog(p.t_s2g, v);
    store_as<T>(const_cast<void*>(p.d.ptr), p.d.scalar,
                map_dim(p.d.map, 0, i) + map_dim(p.d.map, 1, j), v);
  } else {
    Pair<T> c = run_prog_pair_t<OP, T>(p.t_c, load_pair<T>(p.c, i, j));
    Acc re = Acc(round_to(p.c.scalar, c.x)), im = Acc(round_to(p.c.scalar, c.y));
    for (int64_t kb = 0; kb < nkb; ++kb) {
      if (!k_block_runs(p, i, j, kb)) continue;
      for (int64_t k0 = kb * p.bk; k0 < (kb + 1) * p.bk; k0 += p.op_k) {
        const int64_t k1 = k0 + p.op_k;
        if (OP == OP_COMPLEX) {
          Acc neg = Acc(0);
          for (int64_t k = k0; k < k1; ++k) {
            Pair<T> a = run_prog_pair_t<OP, T>(p.t_a, load_pair<T>(p.a, i, k));
            Pair<T> b = run_prog_pair_t<OP, T>(p.t_b, load_pair<T>(p.b, k, j));
            re = add_rn(re, mul_rn(Acc(a.x), Acc(b.x)));
            neg = add_rn(neg, mul_rn(Acc(a.y), Acc(b.y)));
          }
          re = sub_rn(re, neg);
          for (int64_t k = k0; k < k1; ++k) {
            Pair<T> a = run_prog_pair_t<OP, T>(p.t_a, load_pair<T>(p.a, i, k));
            Pair<T> b = run_prog_pair_t<OP, T>(p.t_b, load_pair<T>(p.b, k, j));
            im = add_rn(im, mul_rn(Acc(a.x), Acc(b.y)));
          }
          for (int64_t k = k0; k < k1; ++k) {
            Pair<T> a = run_prog_pair_t<OP, T>(p.t_a, load_pair<T>(p.a, i, k));
            Pair<T> b = run_prog_pair_t<OP, T>(p.t_b, load_pair<T>(p.b, k, j));
            im = add_rn(im, mul_rn(Acc(a.y), Acc(b.x)));
          }
        } else {
          for (int64_t k = k0; k < k1; ++k) {
            Pair<T> a = run_prog_pair_t<OP, T>(p.t_a, load_pair<T>(p.a, i, k));
            Pair<T> b = run_prog_pair_t<OP, T>(p.t_b, load_pair<T>(p.b, k, j));
            re = add_rn(re, mul_rn(Acc(a.x), Acc(b.x)));
          }
          for (int64_t k = k0; k < k1; ++k) {
            Pair<T> a = run_prog_pair_t<OP, T>(p.t_a, load_pair<T>(p.a, i, k));
            Pair<T> b = run_prog_pair_t<OP, T>(p.t_b, load_pair<T>(p.b, k, j));
            im = add_rn(im, mul_rn(Acc(a.x), Acc(b.y)));
          }
          for (int64_t k = k0; k < k1; ++k) {
            Pair<T> a = run_prog_pair_t<OP, T>(p.t_a, load_pair<T>(p.a, i, k));
            Pair<T> b = run_prog_pair_t<OP, T>(p.t_b, load_pair<T>(p.b, k, j));
            im = add_rn(im, mul_rn(Acc(a.y), Acc(b.x)));
          }
        }
      }
    }
    Pair<T> v = run_prog_pair_t<OP, T>(p.t_r2s, Pair<T>{T(re), T(im)});
    v = Pair<T>{round_to(p.d.scalar, v.x), round_to(p.d.scalar, v.y)};
    v = run_prog_pair_t<OP, T>(p.t_s2g, v);
    store_pair<T>(p.d, i, j, v);
  }
}

// Tiled form of the real operator (predicate "always"): the same per-element arithmetic as
// simt_gemm_kernel -- acc starts at round(g2s_c(C)), then acc = acc + a*b for k ascending with
// separate mul / add roundings (no FMA contraction), then the r2s / bias / s2g stages -- so it
// is bitwise identical to it and to the reference (_core.pyx:16-68), but each A / B element
// (transformed by its g2s program once) is staged in shared memory and reused by a 128 x 128
// output tile, 8 x 8 outputs per thread (two 4 x 4 blocks per dimension, 64 apart).  Operand loads go through the layouts' digit maps, so
// every layout the generic kernel takes is valid here too.
constexpr int ST_BM = 128, ST_BN = 128, ST_BK = 16, ST_TM = 8, ST_TN = 8, ST_THREADS = 256;
// 4 consecutive shared-memory elements (16-byte vector loads)
template <typename T>
__device__ __forceinline__ void lds4(const T* src, T (&dst)[4], int at) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = *reinterpret_cast<const float4*>(src);
    dst[at] = v.x; dst[at + 1] = v.y; dst[at + 2] = v.z; dst[at + 3] = v.w;
  } else {
    const double2 v0 = *reinterpret_cast<const double2*>(src);
    const double2 v1 = *reinterpret_cast<const double2*>(src + 2);
    dst[at] = v0.x; dst[at + 1] = v0.y; dst[at + 2] = v1.x; dst[at + 3] = v1.y;
  }
}
// element (i, k) of a real operand: plain strided layouts skip the digit decomposition
template <typename T>
__device__ __forceinline__ T load_op(const SimtLayout& L, bool plain, int64_t i, int64_t k) {
  if (plain) return load_as<T>(L.ptr, L.scalar, i * L.map.s[0][0] + k * L.map.s[1][0]);
  return load_real<T>(L, i, k);
}
// Thread (r, c) = (tid % 16, tid / 16) owns rows {4r..4r+3, 64+4r..64+4r+3} and the same
// pattern of columns: its operand reads are 16-byte vectors at consecutive addresses across the
// warp (conflict-free), two CTAs share an SM (<= 128 registers).
// FAST: plain strided A / B stored at T's precision with identity g2s programs (the reference's
// default f32 / f64 configs) -- direct loads; FP32 accumulation fits two CTAs per SM (<= 128
// registers), f64 accumulators alone take 128.
template <typename T, typename Acc, bool FAST = false>
__global__ void __launch_bounds__(ST_THREADS, (FAST && sizeof(Acc) == 4) ? 2 : 1) simt_tiled_kernel(const __grid_constant__ SimtParams p) {
  constexpr int BK = sizeof(T) == 8 ? ST_BK / 2 : ST_BK;  // f64 tiles: half depth (48 KB static smem)
  constexpr int ST_LA = BK * ST_BM / ST_THREADS, ST_LB = BK * ST_BN / ST_THREADS;  // loads per thread
  __shared__ T As[2][BK][ST_BM];
  __shared__ T Bs[2][BK][ST_BN];
  const int tid = threadIdx.x;
  const int64_t m0 = int64_t(blockIdx.x) * ST_BM, n0 = int64_t(blockIdx.y) * ST_BN;
  const int tr = (tid & 15) * 4, tc = (tid >> 4) * 4;
  auto row_of = [&](int ii) { return tr + (ii & 3) + (ii >> 2) * 64; };
  auto col_of = [&](int jj) { return tc + (jj & 3) + (jj >> 2) * 64; };
  const bool a_plain = p.a.kind == L_STRIDED && p.a.map.nd[0] == 1 && p.a.map.nd[1] == 1;
  const bool b_plain = p.b.kind == L_STRIDED && p.b.map.nd[0] == 1 && p.b.map.nd[1] == 1;
  Acc acc[ST_TM][ST_TN];
#pragma unroll
  for (int ii = 0; ii < ST_TM; ++ii)
#pragma unroll
    for (int jj = 0; jj < ST_TN; ++jj) {
      const int64_t i = m0 + row_of(ii), j = n0 + col_of(jj);
      acc[ii][jj] = Acc(0);
      if (i < p.m && j < p.n) acc[ii][jj] = Acc(round_to(p.c.scalar, prog(p.t_c, load_real<T>(p.c, i, j))));
    }
  // operand tiles, transformed once per element (g2s programs), zero outside the matrix;
  // A: consecutive threads take consecutive rows, B: consecutive k
  T ra[ST_LA], rb[ST_LB];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < ST_LA; ++q) {
      const int e = tid + q * ST_THREADS, kk = e / ST_BM, mm = e % ST_BM;
      const int64_t i = m0 + mm, k = k0 + kk;
      if constexpr (FAST)
        ra[q] = (i < p.m && k < p.k) ? reinterpret_cast<const T*>(p.a.ptr)[i * p.a.map.s[0][0] + k * p.a.map.s[1][0]]
                                     : T(0);
      else
        ra[q] = (i < p.m && k < p.k) ? prog(p.t_a, load_op<T>(p.a, a_plain, i, k)) : T(0);
    }
#pragma unroll
    for (int q = 0; q < ST_LB; ++q) {
      const int e = tid + q * ST_THREADS, kk = e % BK, nn = e / BK;
      const int64_t j = n0 + nn, k = k0 + kk;
      if constexpr (FAST)
        rb[q] = (j < p.n && k < p.k) ? reinterpret_cast<const T*>(p.b.ptr)[k * p.b.map.s[0][0] + j * p.b.map.s[1][0]]
                                     : T(0);
      else
        rb[q] = (j < p.n && k < p.k) ? prog(p.t_b, load_op<T>(p.b, b_plain, k, j)) : T(0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int q = 0; q < ST_LA; ++q) {
      const int e = tid + q * ST_THREADS;
      As[buf][e / ST_BM][e % ST_BM] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < ST_LB; ++q) {
      const int e = tid + q * ST_THREADS;
      Bs[buf][e % BK][e / BK] = rb[q];
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = 0; k0 < p.k; k0 += BK) {
    const int kc = int(min(int64_t(BK), p.k - k0));
    const bool more = k0 + BK < p.k;
    if (more) fetch(k0 + BK);  // next tile's loads in flight under this tile's math
    for (int kk = 0; kk < kc; ++kk) {  // (only the real k: no padded terms enter any sum)
      T a[ST_TM], b[ST_TN];
      T a0[4], a1[4], b0[4], b1[4];
      lds4(&As[buf][kk][tr], a0, 0);
      lds4(&As[buf][kk][tr + 64], a1, 0);
      lds4(&Bs[buf][kk][tc], b0, 0);
      lds4(&Bs[buf][kk][tc + 64], b1, 0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = a0[q];
        a[q + 4] = a1[q];
        b[q] = b0[q];
        b[q + 4] = b1[q];
      }
#pragma unroll
      for (int ii = 0; ii < ST_TM; ++ii)
#pragma unroll
        for (int jj = 0; jj < ST_TN; ++jj) acc[ii][jj] = add_rn(acc[ii][jj], mul_rn(Acc(a[ii]), Acc(b[jj])));
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int ii = 0; ii < ST_TM; ++ii)
#pragma unroll
    for (int jj = 0; jj < ST_TN; ++jj) {
      const int64_t i = m0 + row_of(ii), j = n0 + col_of(jj);
      if (i >= p.m || j >= p.n) continue;
      T v = T(round_to(p.d.scalar, prog(p.t_r2s, acc[ii][jj])));
      if (p.bias_axis)
        v = T(round_to(p.d.scalar, add_rn(v, load_as<T>(p.bias, p.bias_scalar, p.bias_axis == 1 ? j : i))));
      v = prog(p.t_s2g, v);
      store_as<T>(const_cast<void*>(p.d.ptr), p.d.scalar, map_dim(p.d.map, 0, i) + map_dim(p.d.map, 1, j), v);
    }
}

}  // namespace tk
