// Probe: can a TMA tensor map with elementStrides = 2 along the contiguous dimension pull one
// plane (re or im) of an interleaved half-pair matrix straight into a 128B-swizzled tile?
// Encodes {2M, K} fp16 with box {128, 64} and elementStrides {2, 1}; loads the box at column
// coordinate 0 (re) and 1 (im); un-swizzles on the host and compares with the source planes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/probe tools/tma_estride_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "../paper_2009_12263_b200/csrc/tk_ptx.cuh"

using namespace tk;

__global__ void probe(const __grid_constant__ CUtensorMap m, int c0, int bytes, uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* tile = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_2d(tile, &m, &bar, c0, 0, policy_evict_normal());
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(tile)[i];
}

int main() {
  const int M = 256, K = 64;
  std::vector<uint16_t> h(2 * M * K);
  for (int k = 0; k < K; ++k)
    for (int i = 0; i < M; ++i) {
      h[2 * (i + k * M)] = uint16_t(i + 1000 * (k % 50));      // re: tag (i, k)
      h[2 * (i + k * M) + 1] = uint16_t(0x8000 | (i + 17 * k));  // im
    }
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 64 * 64 * 2 * 4);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  for (int sw = 0; sw < 2; ++sw) {
    for (int boxx : {128, 64}) {
      CUtensorMap m;
      cuuint64_t dims[2] = {cuuint64_t(2 * M), cuuint64_t(K)};
      cuuint64_t strides[1] = {cuuint64_t(2 * M * 2)};
      cuuint32_t box[2] = {cuuint32_t(boxx), 64};
      cuuint32_t es[2] = {2, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("swizzle %s box {%d,64} estride {2,1}: encode %d\n", sw ? "128B" : "none", boxx, int(r));
      if (r != CUDA_SUCCESS) continue;
      const int loaded = (boxx / 2) * 64 * 2;  // elements along dim0 = box/estride
      for (int plane = 0; plane < 2; ++plane) {
        cudaMemset(o, 0xff, 64 * 64 * 2 * 4);
        probe<<<1, 128, 16 * 1024>>>(m, plane, loaded, o);
        if (cudaGetLastError() != cudaSuccess) { printf("  launch failed\n"); return 1; }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("  kernel error %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<uint16_t> got(loaded / 2);
        cudaMemcpy(got.data(), o, loaded, cudaMemcpyDeviceToHost);
        const int row_elems = boxx / 2;  // elements per k-row in smem
        int bad = 0;
        for (int k = 0; k < 64; ++k)
          for (int i = 0; i < row_elems; ++i) {
            int chunk = i / 8, within = i % 8;
            int phys = sw ? ((chunk ^ (k & 7)) * 8 + within) : i;  // 128B swizzle: 16B chunks XOR row%8
            uint16_t v = got[k * row_elems + phys];
            uint16_t want = h[2 * (i + k * M) + plane];
            if (v != want && bad++ < 4) printf("  plane %d k %d i %d got %04x want %04x\n", plane, k, i, v, want);
          }
        printf("  plane %d: %s (%d mismatches)\n", plane, bad ? "MISMATCH" : "ok", bad);
      }
    }
  }
  return 0;
}
