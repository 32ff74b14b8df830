// tk_prep.cuh -- small HBM-bound helper kernels that run before the tcgen05 GEMM.
//   * deinterleave: (re,im)/(value,eps) interleaved half pairs -> two planes, so the operand
//     reaches the tensor cores through plain 2-D TMA maps (the paper's "interleaved global,
//     split shared" composition, reference api.py:243-250).  TMA cannot stride dimension 0,
//     so the de-interleave cannot be folded into the tensor map itself.
//   * transform_split: the g2s_a / g2s_b load transforms (reference kernel.py:406-418,
//     components.py:52-94) applied once per operand element in FP32, written as fp16 hi + lo
//     planes for the tensor cores (see the kernel).
#pragma once
#include "tk_types.cuh"

namespace tk {

__global__ void deinterleave_kernel(const uint32_t* __restrict__ src, uint16_t* __restrict__ p0,
                                    uint16_t* __restrict__ p1, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x * 4;
  for (int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4; e < n; e += stride) {
    if (e + 4 <= n && (reinterpret_cast<uintptr_t>(src + e) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(p0 + e) & 7) == 0 && (reinterpret_cast<uintptr_t>(p1 + e) & 7) == 0) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + e);
      uint2 lo, hi;
      lo.x = (v.x & 0xFFFFu) | (v.y << 16);
      lo.y = (v.z & 0xFFFFu) | (v.w << 16);
      hi.x = (v.x >> 16) | (v.y & 0xFFFF0000u);
      hi.y = (v.z >> 16) | (v.w & 0xFFFF0000u);
      *reinterpret_cast<uint2*>(p0 + e) = lo;
      *reinterpret_cast<uint2*>(p1 + e) = hi;
    } else {
      for (int64_t q = e; q < min(n, e + 4); ++q) {
        const uint32_t v = src[q];
        p0[q] = uint16_t(v & 0xFFFFu);
        p1[q] = uint16_t(v >> 16);
      }
    }
  }
}

template <typename H>
__device__ __forceinline__ float h2f(H v);
template <>
__device__ __forceinline__ float h2f<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float h2f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// Operand load transform, the faithful form of the reference's per-element g2s transform:
// s = t(x) is evaluated in FP32 with the reference's operation order (run_prog_real: numpy's
// f32 arithmetic on the f32-widened operand), then split into hi = fp16(s) and
// lo = fp16(s - hi), so hi + lo carries s to ~2^-22 relative and the tensor cores form
// s_a * s_b as hi*hi + hi*lo + lo*hi in FP32 accumulators (lo*lo, < 2^-22, is dropped).
// With SPLIT = false only hi is written (transforms exact in fp16: relu, scale by +-1).
// The operand is a rows x cols matrix with the `fast` dimension contiguous (pitch = the
// stride of the other one); the planes are written dense in the same orientation.
// flag |= 1 when some lo is non-zero: the GEMM skips the lo loads and MMAs otherwise.
template <bool SPLIT>
__global__ void __launch_bounds__(256) transform_split_kernel(const __half* __restrict__ src, __half* __restrict__ hi,
                                                              __half* __restrict__ lo, int64_t fast, int64_t slow,
                                                              int64_t pitch, const __grid_constant__ EpiProg g,
                                                              int32_t* __restrict__ flag) {
  const int64_t total = fast * slow;
  const bool vec = (fast % 8) == 0 && (pitch % 8) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  bool nz = false;
  auto one = [&](float x, __half& h, __half& l) {
    const float v = run_prog_real(g, x);
    h = __float2half_rn(v);
    if (SPLIT) {
      l = __float2half_rn(v - __half2float(h));
      nz |= __half2float(l) != 0.f;
    }
  };
  const int64_t step = int64_t(gridDim.x) * blockDim.x;
  if (vec) {
    for (int64_t e8 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e8 < total / 8; e8 += step) {
      const int64_t e = e8 * 8, r = e % fast, c = e / fast;
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src + c * pitch + r));
      const __half* x = reinterpret_cast<const __half*>(&v);
      uint4 vh, vl;
      __half* h = reinterpret_cast<__half*>(&vh);
      __half* l = reinterpret_cast<__half*>(&vl);
#pragma unroll
      for (int q = 0; q < 8; ++q) one(__half2float(x[q]), h[q], l[q]);
      *reinterpret_cast<uint4*>(hi + e) = vh;
      if (SPLIT) *reinterpret_cast<uint4*>(lo + e) = vl;
    }
  } else {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += step) {
      const int64_t r = e % fast, c = e / fast;
      __half h, l;
      one(__half2float(src[c * pitch + r]), h, l);
      hi[e] = h;
      if (SPLIT) lo[e] = l;
    }
  }
  if (SPLIT && __syncthreads_or(nz) && threadIdx.x == 0) atomicOr(flag, 1);
}

// Block predicate (reference components.py:171-191: executed per (output block, block-K)
// iteration, kernel.py:399-404) expanded for the tensor-core lane: one bit per K=16 MMA step of
// every pair tile (kbits[t * kwords + s / 32], bit s % 32), so the producer skips k-blocks whose
// four steps are all off and the MMA issuer skips single steps.  Needs every tile inside one
// reference block (bm % 256 == 0, bn % tile_n == 0) and bk % 16 == 0.  mode 1: the diagonal
// rule max(m0, k0) < min(m0 + bm, k0 + bk); mode 2: the host-evaluated kmask
// [block rank (bi + bj * M/bm)][K/bk].  Tiles are numbered by the kernel's grouped raster.
__global__ void expand_kbits_kernel(uint32_t* __restrict__ kbits, int tiles, int kwords, int num_mb, int num_nb,
                                    int group_m, int tile_n, int64_t m, int64_t k, int64_t bm, int64_t bn,
                                    int64_t bk, const uint8_t* __restrict__ kmask, int mode) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= int64_t(tiles) * kwords) return;
  const int t = int(idx / kwords), w = int(idx % kwords);
  const int per_group = group_m * num_nb, g = t / per_group, first = g * group_m;
  const int gm = min(num_mb - first, group_m), r = t - g * per_group;
  const int mb = first + r % gm, nb = r / gm;  // tile_coords()
  const int64_t bi = int64_t(mb) * 256 / bm, bj = int64_t(nb) * tile_n / bn, nkb = k / bk;
  uint32_t word = 0;
  for (int b = 0; b < 32; ++b) {
    const int64_t k0 = (int64_t(w) * 32 + b) * 16;
    if (k0 >= k) break;
    const int64_t c = k0 / bk;
    bool run;
    if (mode == 1) {
      const int64_t m0 = bi * bm, kc = c * bk;
      run = max(m0, kc) < min(m0 + bm, kc + bk);
    } else {
      run = kmask[(bi + bj * (m / bm)) * nkb + c] != 0;
    }
    word |= uint32_t(run) << b;
  }
  kbits[idx] = word;
}

}  // namespace tk

namespace tk {

// Gather one plane of a half-precision operand stored under an arbitrary digit map (the
// StridedPermutation / GETT layouts, reference layouts.py:435-506) into a dense column-major
// rows x cols buffer, so any fused-transposition operand reaches the tensor cores through a
// plain 2-D TMA map.  The operand is viewed as an n-digit tensor (<= 10 digits: each digit has
// an extent, a source stride and a destination stride).  A block moves 64 x 64 tiles spanning
// digit X (the source's fastest) and digit Y (the destination's fastest, or its next digit
// when that is X) through shared memory: the read phase runs along X, the write phase along
// whichever tile digit is fastest in the destination, each with 16-byte vectors when that
// digit has unit stride and 8-element alignment; the remaining digits index tiles by block.
// Element offsets count pair elements: interleaved pairs sit at 2*off + plane, split planes
// at off + plane * plane_stride (scalars).
struct PackDesc {
  int32_t n, fs, fd, vec_rd;   // X = fs, Y = fd; vec_rd: 16-byte reads along X
  int32_t wr_x, vec_wr, pad0, pad1;  // wr_x: destination-fastest tile digit is X; vec_wr: 16-byte writes
  int64_t ext[2 * MAX_DIGITS + 1], ss[2 * MAX_DIGITS + 1], ds[2 * MAX_DIGITS + 1];
  int64_t tiles_s, tiles_d, outer;  // tiles along X, along Y, outer digit combinations
};

// tile element (y, x) of the 64 x 64 staging tile: 16-byte chunks of each 128-byte row are
// XOR-swizzled by y/8, so both the row-wise (vector) phase and the column-wise (transpose)
// phase hit 32 distinct banks per warp
__device__ __forceinline__ int pack_tile_off(int y, int x) {
  return y * 64 + ((((x >> 3) ^ (y >> 3)) & 7) << 3) + (x & 7);
}

__global__ void __launch_bounds__(256) pack_half_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                                        const __grid_constant__ PackDesc pd, int pair,
                                                        int64_t plane_stride, int plane) {
  __shared__ __align__(16) uint16_t tile[64 * 64];
  const int64_t nblocks = pd.tiles_s * pd.tiles_d * pd.outer;
  const int64_t sx = pd.ss[pd.fs], sy = pd.ss[pd.fd], dx = pd.ds[pd.fs], dy = pd.ds[pd.fd];
  for (int64_t blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    int64_t q = blk;
    const int64_t ts = q % pd.tiles_s;
    q /= pd.tiles_s;
    const int64_t td = q % pd.tiles_d;
    q /= pd.tiles_d;
    int64_t so = 0, dof = 0;
    for (int t = 0; t < pd.n; ++t) {  // outer digits
      if (t == pd.fs || t == pd.fd) continue;
      const int64_t v = q % pd.ext[t];
      q /= pd.ext[t];
      so += v * pd.ss[t];
      dof += v * pd.ds[t];
    }
    const int64_t x0 = ts * 64, y0 = td * 64;
    const int64_t rx = pd.ext[pd.fs] - x0, ry = pd.ext[pd.fd] - y0;
    const int nx = rx < 64 ? int(rx) : 64, ny = ry < 64 ? int(ry) : 64;
    so += x0 * sx + y0 * sy;
    dof += x0 * dx + y0 * dy;
    __syncthreads();
    if (pd.vec_rd) {  // 8 threads per 64-element row of X, 32 rows per pass
      for (int idx = threadIdx.x; idx < 64 * 8; idx += blockDim.x) {
        const int x = (idx & 7) * 8, y = idx >> 3;
        if (y < ny && x < nx)
          *reinterpret_cast<uint4*>(&tile[pack_tile_off(y, x)]) =
              *reinterpret_cast<const uint4*>(src + so + y * sy + x + int64_t(plane) * plane_stride);
      }
    } else {
      for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
        const int x = idx & 63, y = idx >> 6;
        if (x < nx && y < ny) {
          const int64_t off = so + x * sx + y * sy;
          tile[pack_tile_off(y, x)] = src[pair == P_INTERLEAVED ? 2 * off + plane : off + int64_t(plane) * plane_stride];
        }
      }
    }
    __syncthreads();
    if (pd.wr_x) {  // destination runs along X: rows of the tile are contiguous
      if (pd.vec_wr) {
        for (int idx = threadIdx.x; idx < 64 * 8; idx += blockDim.x) {
          const int x = (idx & 7) * 8, y = idx >> 3;
          if (y < ny && x < nx)
            *reinterpret_cast<uint4*>(dst + dof + y * dy + x) = *reinterpret_cast<const uint4*>(&tile[pack_tile_off(y, x)]);
        }
      } else {
        for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
          const int x = idx & 63, y = idx >> 6;
          if (x < nx && y < ny) dst[dof + x * dx + y * dy] = tile[pack_tile_off(y, x)];
        }
      }
    } else {  // destination runs along Y: transpose through shared memory
      if (pd.vec_wr) {
        for (int idx = threadIdx.x; idx < 64 * 8; idx += blockDim.x) {
          const int y = (idx & 7) * 8, x = idx >> 3;
          if (x < nx && y < ny) {
            uint4 v;
            uint16_t* h = reinterpret_cast<uint16_t*>(&v);
#pragma unroll
            for (int e = 0; e < 8; ++e) h[e] = tile[pack_tile_off(y + e, x)];
            *reinterpret_cast<uint4*>(dst + dof + x * dx + y) = v;
          }
        }
      } else {
        for (int idx = threadIdx.x; idx < 64 * 64; idx += blockDim.x) {
          const int y = idx & 63, x = idx >> 6;
          if (x < nx && y < ny) dst[dof + x * dx + y * dy] = tile[pack_tile_off(y, x)];
        }
      }
    }
  }
}

}  // namespace tk
