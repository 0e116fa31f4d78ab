// Microbenchmark: sustained tcgen05.mma (kind::f16, bf16 -> f32) rate per SM
// for the operand forms the FFA kernels use: SS (A and B from shared memory)
// and TS (A from TMEM), M = 128, N = 64 / 128 / 256, K = 16 per instruction.
// Operand contents are irrelevant (zeros); the issue loop is what is timed.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2505_13211_b200/csrc/kernels/sm100.cuh"

using namespace magi;

constexpr int kIters = 2048;

// FORM 0: SS, 1: TS, 2: TS with B MN-major (the P.V form), 3: SS with B MN-major
// LOADERS: warps 1..3 keep reading TMEM columns [384, 512) meanwhile
template <int FORM, int N, bool LOADERS = false>
__global__ void __launch_bounds__(128, 1) k(long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  __shared__ int stop_flag;
  if (threadIdx.x == 0) stop_flag = 0;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (64 * 1024) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, FORM >= 2);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long c0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
        if (FORM == 0) {
          umma_bf16_ss(tmem, make_smem_desc(a + off, 16, 1024), make_smem_desc(b + off, 16, 1024), idesc, 1);
        } else if (FORM == 1) {
          umma_bf16_ts(tmem, tmem + 256 + kk * 8, make_smem_desc(b + off, 16, 1024), idesc, 1);
        } else if (FORM == 2) {
          // B [K rows x N] N-contiguous: 16 rows of 128B per k-step, 64-col boxes 16 KB apart
          umma_bf16_ts(tmem, tmem + 256 + kk * 8, make_smem_desc(b + kk * 16 * 128, 16384, 1024), idesc, 1);
        } else {
          umma_bf16_ss(tmem, make_smem_desc(a + off, 16, 1024), make_smem_desc(b + kk * 16 * 128, 16384, 1024), idesc, 1);
        }
      }
    }
    umma_commit(&done);
    mbar_wait(&done, 0);
    long long c1 = clock64();
    clk[blockIdx.x] = c1 - c0;
    stop_flag = 1;
  } else if (LOADERS && threadIdx.x >= 32) {
    uint32_t acc = 0;
    const uint32_t t = tmem + (static_cast<uint32_t>((warp % 4) * 32) << 16) + 384;
    for (int it = 0; it < 20000 && !*(volatile int*)&stop_flag; ++it) {
      uint32_t r[32];
      tmem_ld32(t + (it & 3) * 32, r);
      tmem_ld_wait();
      acc ^= r[0] ^ r[31];
    }
    if (acc == 12345u) clk[1] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int FORM, int N, bool LOADERS = false>
void run(const char* name, long long* clk) {
  cudaFuncSetAttribute(k<FORM, N, LOADERS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<FORM, N, LOADERS><<<148, 128, 65536>>>(clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<FORM, N, LOADERS><<<148, 128, 65536>>>(clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const double per = static_cast<double>(c) / (kIters * 8);
  const double ideal = 128.0 * N * 16 / 4096.0;  // 4096 bf16 MAC / clk / SM
  const double flops = 2.0 * 128 * N * 16 * kIters * 8 * 148;
  printf("%-10s N=%3d: %6.1f clk per MMA (ideal %5.1f, %.0f%%), %.0f TFLOPS over %.3f ms\n", name, N, per, ideal,
         100 * ideal / per, flops / ms / 1e9, ms);
}

int main() {
  long long* clk;
  cudaMalloc(&clk, 148 * 8);
  run<0, 64>("SS", clk);
  run<0, 128>("SS", clk);
  run<1, 64>("TS", clk);
  run<1, 128>("TS", clk);
  run<2, 128>("TS B-MN", clk);
  run<3, 128>("SS B-MN", clk);
  run<0, 128, true>("SS +TMEM ld", clk);
  run<2, 128, true>("TS B-MN +TMEM ld", clk);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
