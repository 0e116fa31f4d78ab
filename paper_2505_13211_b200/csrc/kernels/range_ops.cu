// HBM-bound helper kernels of the context-parallel path and the backward
// preprocess. All are grid-stride, 16-byte vectorised, and sized to a
// multiple of the 148 SMs.
//   range_gather            Range Gather: pack token ranges of a
//                           [tokens, row_bytes] buffer into a contiguous buffer.
//   range_scatter_add_f32   deterministic Range Scatter-Reduce: ranges applied
//                           in index order by one thread per element chunk.
//   cast_f32_bf16           final dtype conversion of f32 accumulators.
//   ffa_bwd_preprocess      delta = rowsum(dO * O) per (head, row), f32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace magi {
namespace {

constexpr int kSMs = 148;

int grid_for(int64_t work, int threads, int per_sm = 8) {
  int64_t g = (work + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(kSMs) * per_sm;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

// Find the range containing packed row `r` (offsets sorted ascending).
__device__ __forceinline__ int64_t find_range(const int64_t* offsets, int64_t n, int64_t r) {
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (offsets[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void range_gather_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                    const int64_t* __restrict__ ranges,
                                    const int64_t* __restrict__ offsets, int64_t n,
                                    int64_t total_rows, int64_t vec_per_row) {
  const int64_t total = total_rows * vec_per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / vec_per_row, c = i % vec_per_row;
    const int64_t j = find_range(offsets, n, r);
    const int64_t src_row = ranges[2 * j] + (r - offsets[j]);
    dst[i] = src[src_row * vec_per_row + c];
  }
}

__global__ void range_scatter_add_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                                         const int64_t* __restrict__ ranges,
                                         const int64_t* __restrict__ offsets, int64_t n,
                                         int64_t total_rows, int64_t vec_per_row) {
  // Each destination element may be hit by several ranges (different source
  // ranks); one thread owns one packed element and the ranges of a call never
  // alias inside one call by contract, so the sum order is the call order.
  const int64_t total = total_rows * vec_per_row;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / vec_per_row, c = i % vec_per_row;
    const int64_t j = find_range(offsets, n, r);
    const int64_t dst_row = ranges[2 * j] + (r - offsets[j]);
    float4 a = dst[dst_row * vec_per_row + c];
    const float4 b = src[i];
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
    dst[dst_row * vec_per_row + c] = a;
  }
}

__global__ void cast_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = src[i];
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
    dst[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
}

__global__ void cast_tail_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                 int64_t start, int64_t n) {
  const int64_t i = start + threadIdx.x;
  if (i < n) dst[i] = __float2bfloat16_rn(src[i]);
}

// One warp per (row, head): D elements, lanes stride by 8 (bf16) / 4 (f32).
template <int D, bool kF32>
__global__ void bwd_preprocess_kernel(const void* __restrict__ out,
                                      const __nv_bfloat16* __restrict__ dout,
                                      float* __restrict__ delta, int64_t seqlen, int64_t heads) {
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x % 32;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32;
       w < seqlen * heads; w += warps) {
    const int64_t row = w / heads, h = w % heads;
    const int64_t base = w * D;  // [row, head, D] is row-major: (row*heads + h)*D
    float acc = 0.f;
    for (int d = lane * 4; d < D; d += 128) {
      const uint2 g = *reinterpret_cast<const uint2*>(dout + base + d);
      const __nv_bfloat162 g01 = *reinterpret_cast<const __nv_bfloat162*>(&g.x);
      const __nv_bfloat162 g23 = *reinterpret_cast<const __nv_bfloat162*>(&g.y);
      float o0, o1, o2, o3;
      if constexpr (kF32) {
        const float4 o = *reinterpret_cast<const float4*>(static_cast<const float*>(out) + base + d);
        o0 = o.x; o1 = o.y; o2 = o.z; o3 = o.w;
      } else {
        const uint2 ov = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(out) + base + d);
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ov.x));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ov.y));
        o0 = a.x; o1 = a.y; o2 = b.x; o3 = b.y;
      }
      const float2 ga = __bfloat1622float2(g01), gb = __bfloat1622float2(g23);
      acc += o0 * ga.x + o1 * ga.y + o2 * gb.x + o3 * gb.y;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) delta[h * seqlen + row] = acc;
  }
}

}  // namespace

cudaError_t launch_range_gather(const void* src, void* dst, const int64_t* ranges,
                                const int64_t* offsets, int64_t num_ranges, int64_t total_rows,
                                int64_t row_bytes, cudaStream_t stream) {
  if (num_ranges == 0 || total_rows == 0) return cudaSuccess;
  const int64_t vec = row_bytes / 16;
  range_gather_kernel<<<grid_for(total_rows * vec, 256), 256, 0, stream>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), ranges, offsets, num_ranges,
      total_rows, vec);
  return cudaGetLastError();
}

cudaError_t launch_range_scatter_add_f32(const float* src, float* dst, const int64_t* ranges,
                                         const int64_t* offsets, int64_t num_ranges,
                                         int64_t total_rows, int64_t row_elems,
                                         cudaStream_t stream) {
  if (num_ranges == 0 || total_rows == 0) return cudaSuccess;
  const int64_t vec = row_elems / 4;
  range_scatter_add_kernel<<<grid_for(total_rows * vec, 256), 256, 0, stream>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), ranges, offsets,
      num_ranges, total_rows, vec);
  return cudaGetLastError();
}

cudaError_t launch_cast_f32_bf16(const float* src, void* dst, int64_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const int64_t n4 = n / 4;
  if (n4 > 0) {
    cast_kernel<<<grid_for(n4, 256), 256, 0, stream>>>(reinterpret_cast<const float4*>(src),
                                                      static_cast<uint2*>(dst), n4);
  }
  if (n % 4) {
    cast_tail_kernel<<<1, 32, 0, stream>>>(src, static_cast<__nv_bfloat16*>(dst), n4 * 4, n);
  }
  return cudaGetLastError();
}

cudaError_t launch_ffa_bwd_preprocess(const void* out, const void* grad_out, float* delta,
                                      int64_t seqlen, int64_t heads, int head_dim, int out_f32,
                                      cudaStream_t stream) {
  if (seqlen == 0) return cudaSuccess;
  const int grid = grid_for(seqlen * heads * 32, 256);
  const auto* g = static_cast<const __nv_bfloat16*>(grad_out);
  if (head_dim == 128) {
    if (out_f32) bwd_preprocess_kernel<128, true><<<grid, 256, 0, stream>>>(out, g, delta, seqlen, heads);
    else bwd_preprocess_kernel<128, false><<<grid, 256, 0, stream>>>(out, g, delta, seqlen, heads);
  } else {
    if (out_f32) bwd_preprocess_kernel<64, true><<<grid, 256, 0, stream>>>(out, g, delta, seqlen, heads);
    else bwd_preprocess_kernel<64, false><<<grid, 256, 0, stream>>>(out, g, delta, seqlen, heads);
  }
  return cudaGetLastError();
}

}  // namespace magi
