// Microbenchmark: issue cost per warp instruction of MUFU.EX2, FFMA, FFMA2
// and F2FP on one SM sub-partition, with 1 or 2 warps per SMSP and 16
// independent chains per thread.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu mufu.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2505_13211_b200/csrc/kernels/sm100.cuh"

using namespace magi;

constexpr int kIters = 4096;

template <int OP>
__global__ void k(float* out, long long* clk, float seed) {
  float r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = seed * (i + 1) * 1e-3f - 0.5f * threadIdx.x * 1e-4f;
  uint64_t r2[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r2[i] = f2(r[2 * i], r[2 * i + 1]);
  const uint64_t a2 = f2(0.999f, 0.999f), b2 = f2(1e-4f, 1e-4f);
  uint32_t pk[8] = {};
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if (OP == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = fast_exp2(r[i]);
    } else if (OP == 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = fmaf(r[i], 0.999f, 1e-4f);
    } else if (OP == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) r2[i] = ffma2(r2[i], a2, b2);
    } else if (OP == 3) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        pk[i] ^= pack_bf16(r[2 * i], r[2 * i + 1]);
        r[2 * i] = __uint_as_float(__float_as_uint(r[2 * i]) ^ pk[i]);
      }
    } else if (OP == 5) {
      // ex2.approx.f16x2: two exponentials per lane per instruction
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t h = __float_as_uint(r[2 * i]);
        asm("ex2.approx.f16x2 %0, %0;" : "+r"(h));
        r[2 * i] = __uint_as_float(h);
      }
    } else if (OP == 4) {
      // ex2 through the FMA-pipe polynomial, packed pairs
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 e = exp2_poly2(r[2 * i], r[2 * i + 1]);
        r[2 * i] = e.x * -0.5f;
        r[2 * i + 1] = e.y * -0.5f;
      }
    }
  }
  long long c1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 v = f2_split(r2[i]);
    s += v.x + v.y + __uint_as_float(pk[i]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

template <int OP>
void run(const char* name, int per_iter_instr, float* out, long long* clk) {
  for (int warps : {4, 8, 16}) {
    k<OP><<<148, warps * 32>>>(out, clk, 1.0f);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double per_warp_instr = static_cast<double>(c) / kIters / per_iter_instr;  // per warp
    printf("%-22s warps/SM %2d: %.2f clk per warp-instr per warp; SMSP issues one every %.2f clk\n", name,
           warps, per_warp_instr, per_warp_instr / (warps / 4));
  }
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&clk, 148 * 8);
  run<0>("MUFU.EX2", 16, out, clk);
  run<1>("FFMA", 16, out, clk);
  run<2>("FFMA2", 8, out, clk);
  run<3>("F2FP+2xLOP", 8, out, clk);
  run<4>("exp2_poly2 (per pair)", 8, out, clk);
  run<5>("MUFU.EX2 f16x2 (per pair)", 8, out, clk);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
