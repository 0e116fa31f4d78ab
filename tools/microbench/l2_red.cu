// Microbenchmarks for the fused-backward design question: how fast can 148
// CTAs push f32 dQ tiles (128 rows x 128 cols, row stride hq*D) into L2 with
// reductions, compared with plain tile reads? And how fast is a TMEM readout
// of a 128 x 128 f32 accumulator?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_red l2_red.cu
//   ./l2_red
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../../paper_2505_13211_b200/csrc/kernels/sm100.cuh"

using namespace magi;

constexpr int HQ = 24, D = 128, SEQ = 32768, GROUP = 3;

__device__ __forceinline__ void red_v4(float* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// mode 0: thread = row, 32 x red.v4 along its row
// mode 1: warp = row group, lane = 16B column chunk (coalesced 512B per instr)
// mode 2: bulk reduce (cp.reduce.async.bulk) of 512B rows from smem
// mode 3: plain v4 loads (thread = row), summed
__global__ void __launch_bounds__(128, 1) tile_kernel(float* acc, int mode, int steps, float* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int kv = 0;  // all co-running CTAs on one kv head, like the k-major grid
  const int g = blockIdx.x % GROUP;
  const int h = kv * GROUP + g;
  const int ntiles = SEQ / 128;
  float s = 0.f;
  float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
  if (mode == 2) {
    for (int i = tid; i < 128 * 128; i += 128) reinterpret_cast<float*>(smem)[i] = 1.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  for (int t = 0; t < steps; ++t) {
    const int qt = (t + blockIdx.x / GROUP) % ntiles;
    float* base = acc + (static_cast<size_t>(qt) * 128 * HQ + h) * D;
    if (mode == 0) {
      float* row = base + static_cast<size_t>(tid) * HQ * D;
#pragma unroll 8
      for (int c = 0; c < 32; ++c) red_v4(row + 4 * c, v);
    } else if (mode == 1) {
#pragma unroll 4
      for (int r = warp; r < 128; r += 4) red_v4(base + static_cast<size_t>(r) * HQ * D + 4 * lane, v);
    } else if (mode == 4) {
      // 8 rows x 64 B per warp instruction (lane/4 = row, 4 lanes x 16 B per row)
      for (int r0 = warp * 32; r0 < warp * 32 + 32; r0 += 8)
#pragma unroll
        for (int c = 0; c < 128; c += 16)
          red_v4(base + static_cast<size_t>(r0 + lane / 4) * HQ * D + c + 4 * (lane % 4), v);
    } else if (mode == 5) {
      // 4 rows x 128 B per warp instruction (lane/8 = row, 8 lanes x 16 B per row)
      for (int r0 = warp * 32; r0 < warp * 32 + 32; r0 += 4)
#pragma unroll
        for (int c = 0; c < 128; c += 32)
          red_v4(base + static_cast<size_t>(r0 + lane / 8) * HQ * D + c + 4 * (lane % 8), v);
    } else if (mode == 2) {
      // one thread per row issues a 512B bulk reduce
      float* row = base + static_cast<size_t>(tid) * HQ * D;
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 512;" ::"l"(row),
          "r"(smem_u32(smem + tid * 512))
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    } else {
      const float4* row = reinterpret_cast<const float4*>(base + static_cast<size_t>(tid) * HQ * D);
#pragma unroll 8
      for (int c = 0; c < 32; ++c) {
        float4 x = __ldcg(row + c);
        s += x.x + x.y + x.z + x.w;
      }
    }
  }
  if (mode == 2) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (s == 123.f) sink[0] = s;
}

// TMEM readout: 4 warps read 128 lanes x 128 f32 columns per iteration
__global__ void __launch_bounds__(256, 1) tmem_kernel(int iters, float* sink, long long* clk) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot + (static_cast<uint32_t>((warp % 4) * 32) << 16);
  uint32_t x[32] = {};
  const int nw = blockDim.x / 128;  // warps per lane quarter: split the 128 columns
  const int part = warp / 4;
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; c += 2) {
      if (c / (4 / nw) != part && nw > 1) continue;
      uint32_t r[32], r2[32];
      tmem_ld32(t + (i & 1) * 128 + c * 32, r);
      tmem_ld32(t + (i & 1) * 128 + (c + 1) * 32, r2);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] ^= r[j] ^ r2[j];
    }
  }
  long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = c1 - c0;
  uint32_t y = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) y ^= x[j];
  if (y == 12345u) sink[0] = 1.f;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(slot);
  }
}

int main() {
  float* acc;
  float* sink;
  long long* clk;
  const size_t n = static_cast<size_t>(SEQ) * HQ * D;
  cudaMalloc(&acc, n * 4);
  cudaMemset(acc, 0, n * 4);
  cudaMalloc(&sink, 64);
  cudaMalloc(&clk, 64);
  cudaFuncSetAttribute(tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"red.v4 thread=row", "red.v4 coalesced rows", "bulk reduce 512B rows",
                         "ld.v4 thread=row", "red.v4 8 rows x 64B", "red.v4 4 rows x 128B"};
  for (int grid : {148}) {
    for (int mode = 0; mode < 6; ++mode) {
      const int steps = 256;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        tile_kernel<<<grid, 128, 65536>>>(acc, mode, steps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = static_cast<double>(grid) * steps * 128 * 128 * 4;
      printf("grid %d %-24s %8.3f ms  %7.2f TB/s  (%.0f ns per 64KB tile per CTA)\n", grid,
             names[mode], ms, bytes / ms / 1e9, ms * 1e6 / steps);
    }
  }
  for (int threads : {128, 256}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      tmem_kernel<<<148, threads>>>(4096, sink, clk);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    printf("tmem readout 128x128 f32 with %d threads: %.1f clk per 64KB (%.1f B/clk per SM), %.3f ms\n",
           threads, c / 4096.0, 65536.0 * 4096 / c, ms);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
