// tk_types.cuh -- device-side layout maps, element access and transform programs shared by
// the tcgen05 lane and the bit-exact CUDA-core lane.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace tk {

// OP_SPLIT (internal): a real GEMM whose transformed fp16 operands arrive as hi + lo planes
// (x = hi + lo, see transform_split_kernel); 3 MMAs per step (hi*hi, hi*lo, lo*hi) into two
// FP32 accumulators that the real epilogue sums.
enum { OP_REAL = 0, OP_COMPLEX = 1, OP_DUAL = 2, OP_SPLIT = 3 };
enum { S_F16 = 0, S_BF16 = 1, S_F32 = 2, S_F64 = 3 };
enum { L_STRIDED = 0, L_DIAGONAL = 1, L_ZERO = 2 };
enum { P_NONE = 0, P_INTERLEAVED = 1, P_SPLIT = 2 };
enum { T_SCALE = 1, T_ADD = 2, T_RELU = 3 };
constexpr int MAX_TOPS = 8;

// Logical index -> element offset, one digit list per logical dimension (TkLayout).
constexpr int MAX_DIGITS = 5;  // == TK_MAX_DIGITS
struct DigitMap {
  int32_t nd[2];
  int32_t pad[2];
  int64_t e[2][MAX_DIGITS];
  int64_t s[2][MAX_DIGITS];
};

__host__ __device__ __forceinline__ int64_t map_dim(const DigitMap& m, int d, int64_t idx) {
  if (m.nd[d] == 1) return idx * m.s[d][0];
  int64_t off = 0;
  for (int t = 0; t < m.nd[d]; ++t) {
    const int64_t q = idx / m.e[d][t];
    off += (idx - q * m.e[d][t]) * m.s[d][t];
    idx = q;
  }
  return off;
}

// Transform program (reference components.py:52-94): scale / add / relu applied in order.
struct EpiProg {
  int32_t n;
  int32_t op[MAX_TOPS];
  int32_t promote[MAX_TOPS];
  float fre[MAX_TOPS], fim[MAX_TOPS];
  double dre[MAX_TOPS], dim[MAX_TOPS];
};

// numpy maximum(v, 0): keeps -0.0 and NaN
__device__ __forceinline__ float np_relu(float v) { return (v >= 0.f || v != v) ? v : 0.f; }
__device__ __forceinline__ double np_relu(double v) { return (v >= 0.0 || v != v) ? v : 0.0; }

// mul/add with round-to-nearest and never contracted into FMA: the reference's numpy /
// Cython arithmetic is separate multiply-then-add.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ float run_prog_real(const EpiProg& g, float v) {
  for (int i = 0; i < g.n; ++i) {
    const int op = g.op[i];
    if (op == T_SCALE)
      v = g.promote[i] ? float(__dmul_rn(double(v), g.dre[i])) : mul_rn(v, g.fre[i]);
    else if (op == T_ADD)
      v = g.promote[i] ? float(__dadd_rn(double(v), g.dre[i])) : add_rn(v, g.fre[i]);
    else if (op == T_RELU)
      v = np_relu(v);
  }
  return v;
}
__device__ __forceinline__ double run_prog_real(const EpiProg& g, double v) {
  for (int i = 0; i < g.n; ++i) {
    const int op = g.op[i];
    if (op == T_SCALE) v = mul_rn(v, g.dre[i]);
    else if (op == T_ADD) v = add_rn(v, g.dre[i]);
    else if (op == T_RELU) v = np_relu(v);
  }
  return v;
}

template <typename T>
struct Pair {
  T x, y;
};

// complex: full complex multiply (numpy promotes a real scale to complex); dual: per-field.
template <int OP, typename T>
__device__ __forceinline__ Pair<T> run_prog_pair_t(const EpiProg& g, Pair<T> v) {
  for (int i = 0; i < g.n; ++i) {
    const int op = g.op[i];
    const T sr = sizeof(T) == 4 ? T(g.fre[i]) : T(g.dre[i]);
    const T si = sizeof(T) == 4 ? T(g.fim[i]) : T(g.dim[i]);
    if (op == T_SCALE) {
      if (OP == OP_COMPLEX) {
        const T re = sub_rn(mul_rn(v.x, sr), mul_rn(v.y, si));
        const T im = add_rn(mul_rn(v.x, si), mul_rn(v.y, sr));
        v.x = re;
        v.y = im;
      } else {
        v.x = mul_rn(v.x, sr);
        v.y = mul_rn(v.y, sr);
      }
    } else if (op == T_ADD) {
      v.x = add_rn(v.x, sr);
      v.y = add_rn(v.y, si);
    }
  }
  return v;
}
template <int OP>
__device__ __forceinline__ float2 run_prog_pair(const EpiProg& g, float2 v) {
  Pair<float> r = run_prog_pair_t<OP, float>(g, Pair<float>{v.x, v.y});
  return make_float2(r.x, r.y);
}

// ---- element access ----------------------------------------------------------------
__device__ __forceinline__ float load_scalar_f32(const void* p, int64_t off) {
  return reinterpret_cast<const float*>(p)[off];
}
__device__ __forceinline__ float2 load_pair_f32(const void* p, int pair, int64_t plane,
                                                int64_t off) {
  const float* f = reinterpret_cast<const float*>(p);
  if (pair == P_INTERLEAVED) return *reinterpret_cast<const float2*>(f + 2 * off);
  return make_float2(f[off], f[off + plane]);
}
__device__ __forceinline__ void store_pair_f32(void* p, int pair, int64_t plane, int64_t off,
                                               float2 v) {
  float* f = reinterpret_cast<float*>(p);
  if (pair == P_INTERLEAVED) {
    *reinterpret_cast<float2*>(f + 2 * off) = v;
  } else {
    f[off] = v.x;
    f[off + plane] = v.y;
  }
}

// scalar conversions for the generic lane
template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

}  // namespace tk
