// Microbenchmark: which pipes do MUFU.EX2, F2FP (bf16 pack) and FFMA share?
// Mixed loops with independent chains, 2 warps per SM sub-partition.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2505_13211_b200/csrc/kernels/sm100.cuh"

using namespace magi;

constexpr int kIters = 2048;

// OP bits: 1 = 16 MUFU.EX2, 2 = 8 F2FP packs, 4 = 16 FFMA, 8 = 8 PRMT (truncating pack)
template <int OP>
__global__ void __launch_bounds__(256, 1) k(float* out, long long* clk, float seed) {
  float r[16], q[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    r[i] = seed * (i + 1) * 1e-3f - 0.5f;
    q[i] = seed * (i + 3) * 1e-3f;
  }
  uint32_t pk[8] = {};
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if (OP & 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = fast_exp2(r[i]);
    }
    if (OP & 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) pk[i] += pack_bf16(q[2 * i], q[2 * i + 1]);
#pragma unroll
      for (int i = 0; i < 8; ++i) q[2 * i] = __uint_as_float(pk[i] | 0x3f000000u);
    }
    if (OP & 4) {
#pragma unroll
      for (int i = 0; i < 16; ++i) q[i] = fmaf(q[i], 0.999f, 1e-4f);
    }
    if (OP & 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) pk[i] += __byte_perm(__float_as_uint(q[2 * i]), __float_as_uint(q[2 * i + 1]), 0x7632);
#pragma unroll
      for (int i = 0; i < 8; ++i) q[2 * i] = __uint_as_float(pk[i] | 0x3f000000u);
    }
  }
  long long c1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i] + q[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float(pk[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

template <int OP>
void run(const char* name, float* out, long long* clk) {
  k<OP><<<148, 256>>>(out, clk, 1.0f);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %.1f clk per iteration per SMSP (2 warps)\n", name, static_cast<double>(c) / kIters);
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&clk, 148 * 8);
  run<1>("16 MUFU", out, clk);
  run<2>("8 F2FP (+8 LOP)", out, clk);
  run<3>("16 MUFU + 8 F2FP (+8 LOP)", out, clk);
  run<4>("16 FFMA", out, clk);
  run<5>("16 MUFU + 16 FFMA", out, clk);
  run<8>("8 PRMT (+8 LOP)", out, clk);
  run<9>("16 MUFU + 8 PRMT (+8 LOP)", out, clk);
  run<7>("16 MUFU + 8 F2FP + 16 FFMA", out, clk);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
