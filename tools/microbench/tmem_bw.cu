// Microbenchmark: TMEM load / store bandwidth per SM with 4, 8 and 16 warps
// (tcgen05.ld / st 32x32b.x32, 4 KB per warp instruction), no arithmetic on
// the loaded values beyond one register.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2505_13211_b200/csrc/kernels/sm100.cuh"

using namespace magi;

constexpr int kIters = 2048;

template <bool STORE>
__global__ void __launch_bounds__(512, 1) k(int cols_per_warp, float* sink, long long* clk) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int nw = blockDim.x / 32;
  const int group = warp / 4;  // warps sharing a lane quarter split the columns
  const int per = 512 / (nw / 4);
  const uint32_t t = slot + (static_cast<uint32_t>((warp % 4) * 32) << 16) + group * per;
  uint32_t acc = 0;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = i;
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    for (int c = 0; c < per; c += 32) {
      if (STORE) {
        tmem_st32(t + c, r);
      } else {
        tmem_ld32(t + c, r);
      }
    }
    if (STORE) {
      tmem_st_wait();
      r[0] += 1;
    } else {
      tmem_ld_wait();
      acc ^= r[0] ^ r[31];
    }
  }
  long long c1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
  if (acc == 12345u) sink[0] = 1.f;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(slot);
  }
}

int main() {
  float* sink;
  long long* clk;
  cudaMalloc(&sink, 64);
  cudaMalloc(&clk, 148 * 8);
  for (int store = 0; store < 2; ++store) {
    for (int warps : {4, 8, 16}) {
      if (store) {
        k<true><<<148, warps * 32>>>(0, sink, clk);
      } else {
        k<false><<<148, warps * 32>>>(0, sink, clk);
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double bytes = 128.0 * 512 * 4 * kIters;  // whole TMEM per iteration
      printf("%s %2d warps: %.1f B/clk per SM (%.0f clk per 64 KB)\n", store ? "st" : "ld", warps, bytes / c,
             65536.0 / (bytes / c));
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
