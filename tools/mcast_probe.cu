// mcast_probe.cu -- does TMA multicast raise the L2->SM delivery rate? (tuning only)
//
// Every CTA of a 144-CTA grid streams 32 KB chunks of an L2-resident buffer into a 6-slot
// shared-memory ring (cp.async.bulk, mbarrier complete_tx), in clusters of G CTAs:
//   mode 0  distinct: every CTA reads its own chunks (no sharing)
//   mode 1  unicast : the G CTAs of a cluster read the same chunk, each with its own copy
//   mode 2  multicast: each CTA of the cluster fetches 1/G of the chunk for all G CTAs
// Each CTA receives 32 KB per step in every mode; slots are recycled only after every CTA of
// the cluster consumed them (remote empty-barrier arrivals), as in a multicast GEMM pipeline.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mcast_probe mcast_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2009_12263_b200/csrc/tk_ptx.cuh"

using namespace tk;

#ifndef PARRIVE
#define PARRIVE 0  // consumer arrive: 0 relaxed.cluster, 1 release.cluster, 2 default (release.cta)
#endif
#ifndef NSPLIT
#define NSPLIT 1
#endif
#ifndef PS
#define PS 6
#endif
#ifndef PCH
#define PCH 32768
#endif
constexpr int S = PS;
constexpr int CH = PCH;

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_load_mc(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "h"(mask)
      : "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe(const uint8_t* src, int nchunks, int iters, int G, int mode,
                      unsigned long long* ns) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * CH);
  uint64_t* empty = full + S;
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x / G;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G);
    }
    fence_mbar_init();
  }
  cluster_sync();
  unsigned long long t0 = gtime();
  const uint32_t slice = CH / G;
  if (threadIdx.x == 0) {  // producer
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], CH);
      const int chunk = mode == 0 ? (blockIdx.x * 7 + i) % nchunks : (cid * 7 + i) % nchunks;
      const uint8_t* g = src + size_t(chunk) * CH;
      const uint32_t dst = smem_u32(sm + s * CH), bar = smem_u32(&full[s]);
      if (mode == 2)
        bulk_load_mc(dst + rank * slice, g + rank * slice, slice, bar, uint16_t((1u << G) - 1));
      else
        for (int q = 0; q < NSPLIT; ++q)  // NSPLIT copies per step (per-copy vs per-byte cost)
          bulk_load(dst + q * (CH / NSPLIT), g + q * (CH / NSPLIT), CH / NSPLIT, bar);
    }
  } else if (threadIdx.x == 32) {  // consumer: wait for each step, release its slot everywhere
    for (int j = 0; j < iters; ++j) {
      const int s = j % S;
      mbar_wait(&full[s], (j / S) & 1);
      // (a consumer that only needs ordering against the async copies: relaxed arrive, like
      // an MMA warp's multicast tcgen05.commit)
      for (int q = 0; q < G; ++q) {
        const uint32_t a = mapa_shared(smem_u32(&empty[s]), q);
        if (PARRIVE == 0)
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
        else if (PARRIVE == 1)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
        else
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) ns[blockIdx.x] = gtime() - t0;
  cluster_sync();  // no CTA exits while peers may still write its slots / arrive on its barriers
}

int main(int argc, char** argv) {
  const int grid = argc > 1 ? atoi(argv[1]) : 144;
  const int iters = argc > 2 ? atoi(argv[2]) : 4000;
  const size_t bytes = size_t(48) << 20;  // L2-resident source
  const int nchunks = int(bytes / CH);
  uint8_t* src;
  unsigned long long* ns;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  cudaMalloc(&ns, grid * sizeof(unsigned long long));
  const int smem = S * CH + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"distinct", "unicast ", "multicast"};
  for (int G : {1, 2, 4, 8}) {
    for (int mode = 0; mode < 3; ++mode) {
      if (G == 1 && mode) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(64);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int maxc = 0;
      cudaOccupancyMaxActiveClusters(&maxc, probe, &cfg);
      if (mode == 0) printf("G=%d: max active clusters %d (%d CTAs)\n", G, maxc, maxc * G);
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, probe, (const uint8_t*)src, nchunks, iters, G, mode, ns);
        cudaEventRecord(e1);
        if (err != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess) {
          printf("G=%d mode=%d: %s\n", G, mode, cudaGetErrorString(cudaGetLastError()));
          return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best = ms < best ? ms : best;
      }
      std::vector<unsigned long long> h(grid);
      cudaMemcpy(h.data(), ns, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (auto v : h) mx = v > mx ? v : mx;
      const double delivered = double(grid) * iters * CH;
      const double fetched = mode == 1 || mode == 0 ? delivered : delivered / G;
      printf("S=%d CH=%d x%d G=%d %s  %.3f ms  delivered %.2f TB/s (in-kernel %.2f TB/s), L2 reads issued %.2f TB/s, "
             "%.0f B/clk/SM at 1.9 GHz\n",
             S, CH, NSPLIT, G, names[mode], best, delivered / (best * 1e-3) / 1e12, delivered / (mx * 1e-9) / 1e12,
             fetched / (best * 1e-3) / 1e12, delivered / (best * 1e-3) / grid / 1.9e9);
    }
  }
  return 0;
}
