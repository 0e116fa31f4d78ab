// Microbenchmark: aggregate TMA tile-streaming throughput of 148 CTAs that all
// walk the same sequence of 32 KB tiles (the FFA access pattern), unicast vs
// cluster multicast (each CTA of a cluster loads 1/n of every tile and
// multicasts it to all n CTAs).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_mc tma_mc.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2505_13211_b200/csrc/kernels/sm100.cuh"
#include "../../paper_2505_13211_b200/csrc/kernels/tma_host.h"

using namespace magi;

constexpr int SEQ = 32768, HK = 8, D = 128, RING = 4;
constexpr uint32_t kTileBytes = 128 * D * 2;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                               int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

// n = cluster size (1 = unicast); rows_per_box = 128 / (n / 2) for n >= 2
template <int N>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap tmap, int iters,
                                                        int sync_every) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[RING];
  const uint32_t rank = N > 1 ? cluster_rank() : 0;
  const int group = blockIdx.x / N;
  const int head = group % HK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  if (N > 1) cluster_sync(); else __syncthreads();
  auto issue = [&](int i) {
    const int s = i % RING;
    const int tok = (i * 128 + group * 0) % SEQ;
    uint8_t* dst = smem + s * kTileBytes;
    mbar_arrive_expect_tx(&full[s], kTileBytes);
    if constexpr (N == 1) {
      for (int c = 0; c < D / 64; ++c) tma_load_3d(dst + c * 16384, &tmap, &full[s], c * 64, head, tok);
    } else {
      // box = (128 / (N/2)) rows x 64 cols; this CTA loads box `rank`
      constexpr int rows = 128 / (N > 1 ? N / 2 : 1);
      const int c = rank % 2, part = rank / 2;
      tma_load_3d_mc(dst + c * 16384 + part * rows * 128, &tmap, &full[s], c * 64, head, tok + part * rows,
                     static_cast<uint16_t>((1u << N) - 1));
    }
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < RING; ++i) issue(i);
  for (int i = 0; i < iters; ++i) {
    mbar_wait(&full[i % RING], (i / RING) & 1);
    if (N > 1 && (i % sync_every) == 0) cluster_sync();
    if (threadIdx.x == 0 && i + RING < iters) issue(i + RING);
  }
  if (N > 1) cluster_sync();
}

template <int N>
void run(const CUtensorMap& tm, int iters) {
  const int smem = RING * kTileBytes;
  cudaFuncSetAttribute(stream_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = N;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, stream_kernel<N>, tm, iters, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double delivered = 148.0 * iters * kTileBytes;
  printf("cluster %d: %.3f ms, delivered %.2f TB/s to SMs, L2 requests %.2f TB/s, %.0f ns per 32KB tile per CTA  (%s)\n",
         N, ms, delivered / ms / 1e9, delivered / N / ms / 1e9, ms * 1e6 / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  void* k;
  cudaMalloc(&k, static_cast<size_t>(SEQ) * HK * D * 2);
  cudaMemset(k, 0, static_cast<size_t>(SEQ) * HK * D * 2);
  const CUtensorMap t128 = make_tmap_thd(k, SEQ, HK, D, 128);
  const CUtensorMap t64 = make_tmap_thd(k, SEQ, HK, D, 64);
  const CUtensorMap t32 = make_tmap_thd(k, SEQ, HK, D, 32);
  const int iters = 4096;
  run<1>(t128, iters);
  run<2>(t128, iters);
  run<4>(t64, iters);
  run<1>(t128, iters);
  return 0;
}
