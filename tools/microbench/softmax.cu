// Microbenchmark: cost of the forward kernel's elementwise phase in isolation:
// one 64-column slice of an online-softmax row step (partial max, exp2, row
// sum, bf16 pack) per thread, two warps per SM sub-partition (the two
// warpgroups that share a sub-tile).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o softmax softmax.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../paper_2505_13211_b200/csrc/kernels/sm100.cuh"

using namespace magi;

constexpr int kIters = 512;
#ifndef SM_NC
#define SM_NC 64
#endif
#ifndef SM_THREADS
#define SM_THREADS 256
#endif
constexpr int NC = SM_NC;  // columns per thread
constexpr int kThreadsPerCta = SM_THREADS;  // 256: 2 warps per SMSP; 128: 1

// MASK: pairs (j % 8) computed with the FMA-pipe polynomial.
// ORDER 0: fused per pair (kernel); 1: all x first, then exps, then sums/packs
template <uint32_t MASK, int ORDER, bool MAX, bool SUM = true>
__global__ void __launch_bounds__(kThreadsPerCta, 1) k(float* out, long long* clk, float seed) {
  uint32_t s[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) s[i] = __float_as_uint(seed * ((i * 37 + threadIdx.x) % 101) * 0.01f);
  float m = -INFINITY, l = 0.f;
  uint32_t acc = 0;
  const float sl2 = 0.127f;
  __syncthreads();
  long long c0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    float mt = 3.0f;
    if (MAX) {
      float mx[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) mx[u] = fmaxf(__uint_as_float(s[2 * u]), __uint_as_float(s[2 * u + 1]));
#pragma unroll
      for (int i = 8; i < NC; i += 8) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          mx[u] = fmaxf(mx[u], fmaxf(__uint_as_float(s[i + 2 * u]), __uint_as_float(s[i + 2 * u + 1])));
      }
      mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
    }
    const float mt2 = mt * sl2;
    const bool move = mt2 > m + 8.f;
    const float alpha = move ? fast_exp2(m - mt2) : 1.f;
    if (move) m = mt2;
    const float mb = m;
    uint32_t pk[NC / 2];
    float rs;
    const uint64_t sc2 = f2(sl2, sl2), nm2 = f2(-mb, -mb);
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
    if (ORDER == 0) {
#pragma unroll
      for (int i = 0; i < NC; i += 2) {
        const int j = i / 2;
        const float2 x = f2_split(ffma2(f2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sc2, nm2));
        float p0, p1;
        if ((MASK >> (j % 8)) & 1u) {
          const float2 e = exp2_poly2(x.x, x.y);
          p0 = e.x;
          p1 = e.y;
        } else {
          p0 = fast_exp2(x.x);
          p1 = fast_exp2(x.y);
        }
        if (SUM) acc2[j % 4] = fadd2(acc2[j % 4], f2(p0, p1));
        pk[j] = pack_bf16(p0, p1);
      }
    } else {
      float xs[NC];
#pragma unroll
      for (int i = 0; i < NC; i += 2) {
        const float2 x = f2_split(ffma2(f2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sc2, nm2));
        xs[i] = x.x;
        xs[i + 1] = x.y;
      }
#pragma unroll
      for (int i = 0; i < NC; i += 2) {
        const int j = i / 2;
        if (!((MASK >> (j % 8)) & 1u)) {
          xs[i] = fast_exp2(xs[i]);
          xs[i + 1] = fast_exp2(xs[i + 1]);
        }
      }
#pragma unroll
      for (int i = 0; i < NC; i += 2) {
        const int j = i / 2;
        if ((MASK >> (j % 8)) & 1u) {
          const float2 e = exp2_poly2(xs[i], xs[i + 1]);
          xs[i] = e.x;
          xs[i + 1] = e.y;
        }
      }
#pragma unroll
      for (int i = 0; i < NC; i += 2) {
        const int j = i / 2;
        acc2[j % 4] = fadd2(acc2[j % 4], f2(xs[i], xs[i + 1]));
        pk[j] = pack_bf16(xs[i], xs[i + 1]);
      }
    }
    const float2 a = f2_split(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])));
    rs = a.x + a.y;
    l = l * alpha + rs;
#pragma unroll
    for (int j = 0; j < NC / 2; ++j) acc ^= pk[j];
#pragma unroll
    for (int i = 0; i < NC; i += 16) s[i] ^= (acc & 1u);
  }
  long long c1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + static_cast<float>(acc & 7u);
  if (threadIdx.x == 0) clk[blockIdx.x] = c1 - c0;
}

template <uint32_t MASK, int ORDER, bool MAX, bool SUM = true>
void run(const char* name, float* out, long long* clk) {
  k<MASK, ORDER, MAX, SUM><<<148, kThreadsPerCta>>>(out, clk, 1.0f);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  const int mufu = NC - 2 * __builtin_popcount(MASK) * NC / 16;  // per warp
  printf("%-40s %5.0f clk per phase (%d warps x %d columns per SMSP; MUFU bound %d)\n", name,
         static_cast<double>(c) / kIters, kThreadsPerCta / 128, NC, mufu * kThreadsPerCta / 128 * 8);
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&clk, 148 * 8);
  run<0x88u, 0, true>("25% poly, fused (kernel)", out, clk);
  run<0x92u, 0, true>("37.5% poly, fused", out, clk);
  run<0xAAu, 0, true>("50% poly, fused", out, clk);
  run<0x80u, 0, true>("12.5% poly, fused", out, clk);
  run<0x00u, 0, true>("all MUFU, fused", out, clk);
  run<0x88u, 1, true>("25% poly, staged", out, clk);
  run<0x92u, 1, true>("37.5% poly, staged", out, clk);
  run<0x88u, 0, false>("25% poly, fused, no max", out, clk);
  run<0x88u, 0, true, false>("25% poly, fused, no row sum", out, clk);
  run<0x92u, 0, true, false>("37.5% poly, fused, no row sum", out, clk);
  run<0x88u, 0, false, false>("25% poly, fused, no max, no sum", out, clk);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
