// UMMA / TMA self-test: one 128x128x128 bf16 tile product through the exact
// building blocks the FFA kernels use (TMA SW128 loads, K-major and MN-major
// smem descriptors, kind::f16 tcgen05.mma into TMEM, 32x32b TMEM loads).
// Exposed through the C ABI as magiplan_debug_umma_tile so GPU tests can pin
// the descriptor encodings independently of the attention kernels.
#include <cuda_runtime.h>

#include "sm100.cuh"
#include "tma_host.h"

namespace magi {
namespace {

constexpr int kTile = 128;
constexpr uint32_t kBoxBytes = 128 * 64 * 2;  // 128 rows x 64 bf16

__global__ void __launch_bounds__(128, 1)
    umma_tile_kernel(const __grid_constant__ CUtensorMap tmap_a,
                     const __grid_constant__ CUtensorMap tmap_b, float* __restrict__ c,
                     const uint32_t* __restrict__ a_rows, int mode) {
  // mode 0: SS, B K-major; 1: SS, B MN-major; 2: TS (A in TMEM), B K-major
  const int b_mn_major = mode == 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sa = smem;                  // 2 boxes: K 0..63, 64..127
  uint8_t* sb = smem + 2 * kBoxBytes;  // 2 boxes
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (mode == 2) {
    // thread = row = TMEM lane; 64 packed bf16-pair columns at column 128
    const uint32_t r0 = warp * 32 + lane;
    for (int cc = 0; cc < 2; ++cc) {
      uint32_t v[32];
      for (int j = 0; j < 32; ++j) v[j] = a_rows[r0 * 64 + cc * 32 + j];
      tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + 128 + cc * 32, v);
    }
    tmem_st_wait();
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();

  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_load, 4 * kBoxBytes);
    tma_load_2d(sa, &tmap_a, &bar_load, 0, 0);
    tma_load_2d(sa + kBoxBytes, &tmap_a, &bar_load, 64, 0);
    // K-major B: [N rows, K] -> boxes at K 0 / 64.  MN-major B: [K rows, N]
    // -> boxes at N 0 / 64.  Either way the second box is 16 KB later.
    tma_load_2d(sb, &tmap_b, &bar_load, 0, 0);
    tma_load_2d(sb + kBoxBytes, &tmap_b, &bar_load, 64, 0);
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t idesc = make_idesc_bf16(128, 128, false, b_mn_major != 0);
    for (int k = 0; k < kTile / 16; ++k) {
      const uint32_t a_addr = smem_u32(sa) + (k / 4) * kBoxBytes + (k % 4) * 32;
      const uint64_t adesc = make_smem_desc(a_addr, 16, 1024);
      uint64_t bdesc;
      if (b_mn_major) {
        bdesc = make_smem_desc(smem_u32(sb) + k * 16 * 128, kBoxBytes, 1024);
      } else {
        bdesc = make_smem_desc(smem_u32(sb) + (k / 4) * kBoxBytes + (k % 4) * 32, 16, 1024);
      }
      if (mode == 2) {
        umma_bf16_ts(tmem, tmem + 128 + k * 8, bdesc, idesc, k > 0 ? 1u : 0u);
      } else {
        umma_bf16_ss(tmem, adesc, bdesc, idesc, k > 0 ? 1u : 0u);
      }
    }
    umma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();

  const uint32_t row = warp * 32 + lane;
  for (int cc = 0; cc < kTile / 32; ++cc) {
    uint32_t r[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cc * 32, r);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) c[row * kTile + cc * 32 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

}  // namespace

// A: [128, 128] bf16 row-major. B: [128(N), 128(K)] when !b_mn_major (C = A B^T),
// [128(K), 128(N)] when b_mn_major == 1 (C = A B). b_mn_major == 2 stages A in
// TMEM (tcgen05.mma A-from-TMEM form), B K-major. C: [128, 128] f32.
cudaError_t launch_umma_tile(const void* a, const void* b, float* c, int b_mn_major,
                             cudaStream_t stream) {
  const uint64_t dims[2] = {128, 128};
  const uint64_t strides[1] = {128 * 2};
  const uint32_t box[2] = {64, 128};
  const CUtensorMap ta = make_tmap_bf16(a, 2, dims, strides, box);
  const CUtensorMap tb = make_tmap_bf16(b, 2, dims, strides, box);
  const int smem = 4 * kBoxBytes + 1024;
  cudaFuncSetAttribute(umma_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_tile_kernel<<<1, 128, smem, stream>>>(ta, tb, c, static_cast<const uint32_t*>(a),
                                             b_mn_major);
  return cudaGetLastError();
}

}  // namespace magi
