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

// Row-per-warp form for rows of >= 32 vectors (a K/V token row of 8 heads x
// 128 x bf16 is 128): the range lookup is done once per row, and every lane
// issues its kRowUnroll 16-byte loads before its stores, so each warp keeps
// kRowUnroll x 512 B in flight instead of one dependent load per thread.
constexpr int kRowUnroll = 4;
__global__ void range_gather_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                         const int64_t* __restrict__ ranges,
                                         const int64_t* __restrict__ offsets, int64_t n,
                                         int64_t total_rows, int64_t vec_per_row) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32; r < total_rows;
       r += warps) {
    const int64_t j = find_range(offsets, n, r);
    const uint4* s = src + (ranges[2 * j] + (r - offsets[j])) * vec_per_row;
    uint4* d = dst + r * vec_per_row;
    for (int64_t c0 = 0; c0 < vec_per_row; c0 += 32 * kRowUnroll) {
      uint4 v[kRowUnroll];
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) v[u] = s[c];
      }
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) d[c] = v[u];
      }
    }
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

// Row-per-warp form of the scatter-add (rows of >= 32 vectors): one range
// lookup per row, kRowUnroll source and destination vectors in flight per
// lane. Same per-element order as above: one call's ranges never alias.
__global__ void range_scatter_add_rows_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                                              const int64_t* __restrict__ ranges,
                                              const int64_t* __restrict__ offsets, int64_t n,
                                              int64_t total_rows, int64_t vec_per_row) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32; r < total_rows;
       r += warps) {
    const int64_t j = find_range(offsets, n, r);
    float4* d = dst + (ranges[2 * j] + (r - offsets[j])) * vec_per_row;
    const float4* s = src + r * vec_per_row;
    for (int64_t c0 = 0; c0 < vec_per_row; c0 += 32 * kRowUnroll) {
      float4 a[kRowUnroll], b[kRowUnroll];
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) {
          a[u] = d[c];
          b[u] = s[c];
        }
      }
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) d[c] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
      }
    }
  }
}

// Range copy to per-range destinations (the peer-memory GroupCast): range i
// sends source rows [ranges[2i], ranges[2i+1]) to dst_base[i] + dst_row[i]
// rows. Row per warp as in range_gather_rows_kernel; the destinations are
// other GPUs' receive buffers mapped through CUDA IPC, so the stores travel
// over NVLink straight into the consumers' buffers (no send staging buffer).
__global__ void range_copy_to_kernel(const uint4* __restrict__ src, const int64_t* __restrict__ ranges,
                                     const int64_t* __restrict__ offsets,
                                     const unsigned long long* __restrict__ dst_base,
                                     const int64_t* __restrict__ dst_row, int64_t n, int64_t total_rows,
                                     int64_t vec_per_row) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32; r < total_rows;
       r += warps) {
    const int64_t j = find_range(offsets, n, r);
    const int64_t within = r - offsets[j];
    const uint4* s = src + (ranges[2 * j] + within) * vec_per_row;
    uint4* d = reinterpret_cast<uint4*>(dst_base[j]) + (dst_row[j] + within) * vec_per_row;
    for (int64_t c0 = 0; c0 < vec_per_row; c0 += 32 * kRowUnroll) {
      uint4 v[kRowUnroll];
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) v[u] = s[c];
      }
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) d[c] = v[u];
      }
    }
  }
}

// Scatter-add from per-range sources (the peer-memory GroupReduce): range i
// adds rows src_base[i] + src_row[i].. (f32, possibly a peer's buffer read
// over NVLink) into dst rows [ranges[2i], ranges[2i+1]). One call per
// source rank in rank order keeps the sums deterministic; a call's ranges
// never alias.
__global__ void range_scatter_add_from_kernel(float4* __restrict__ dst, const int64_t* __restrict__ ranges,
                                              const int64_t* __restrict__ offsets,
                                              const unsigned long long* __restrict__ src_base,
                                              const int64_t* __restrict__ src_row, int64_t n, int64_t total_rows,
                                              int64_t vec_per_row) {
  const int lane = threadIdx.x % 32;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32; r < total_rows;
       r += warps) {
    const int64_t j = find_range(offsets, n, r);
    const int64_t within = r - offsets[j];
    float4* d = dst + (ranges[2 * j] + within) * vec_per_row;
    const float4* s = reinterpret_cast<const float4*>(src_base[j]) + (src_row[j] + within) * vec_per_row;
    for (int64_t c0 = 0; c0 < vec_per_row; c0 += 32 * kRowUnroll) {
      float4 a[kRowUnroll], b[kRowUnroll];
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) {
          a[u] = d[c];
          b[u] = s[c];
        }
      }
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c < vec_per_row) d[c] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
      }
    }
  }
}

// Flag protocol of the peer-memory exchange: a release store of `value` to
// each of n (possibly peer-mapped) flags, after every earlier write of this
// stream is visible system-wide; and an acquire spin of one thread per set
// bit of `mask` until local flags[i] >= value.
__global__ void flags_signal_kernel(unsigned int* const* __restrict__ flags, int n, unsigned int value) {
  const int i = threadIdx.x;
  if (i < n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[i]), "r"(value) : "memory");
  }
}
__global__ void flags_wait_kernel(const unsigned int* __restrict__ flags, unsigned int mask, unsigned int value) {
  const int i = threadIdx.x;
  if (i < 32 && ((mask >> i) & 1u)) {
    unsigned int v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
      if (v >= value) break;
      __nanosleep(128);
    }
  }
  __syncthreads();
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

// delta[h, row] = sum_d dO[row, h, d] * O[row, h, d]. A (row, head) item is
// D*2 bytes of dO: D/8 lanes read it as 16-byte vectors (O likewise, f32 O as
// two vectors), so a warp covers 32/(D/8) items per pass and issues kUnroll
// passes' loads before reducing (HBM-bound: keep bytes in flight).
template <int D, bool kF32>
__global__ void bwd_preprocess_kernel(const void* __restrict__ out,
                                      const __nv_bfloat16* __restrict__ dout,
                                      float* __restrict__ delta, int64_t seqlen, int64_t heads) {
  constexpr int kLanes = D / 8;            // lanes per item
  constexpr int kPerPass = 32 / kLanes;    // items per warp and pass
  constexpr int kUnroll = 4;
  const int lane = threadIdx.x % 32;
  const int sub = lane / kLanes, l = lane % kLanes;
  const int64_t total = seqlen * heads;
  const int64_t step = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32) * kPerPass * kUnroll;
  for (int64_t base = (blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32) * kPerPass * kUnroll;
       base < total; base += step) {
    uint4 gv[kUnroll];
    float o[kUnroll][8];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t item = base + u * kPerPass + sub;
      const int64_t off = item * D + l * 8;  // [row, head, D] row-major: item = row*heads + h
      if (item < total) {
        gv[u] = *reinterpret_cast<const uint4*>(dout + off);
        if constexpr (kF32) {
          const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(out) + off);
          const float4 b = *reinterpret_cast<const float4*>(static_cast<const float*>(out) + off + 4);
          o[u][0] = a.x; o[u][1] = a.y; o[u][2] = a.z; o[u][3] = a.w;
          o[u][4] = b.x; o[u][5] = b.y; o[u][6] = b.z; o[u][7] = b.w;
        } else {
          const uint4 ov = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(out) + off);
          const uint32_t w[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
            o[u][2 * j] = f.x;
            o[u][2 * j + 1] = f.y;
          }
        }
      } else {
        gv[u] = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[u][j] = 0.f;
      }
    }
    float acc[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t w[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
        a += o[u][2 * j] * g.x + o[u][2 * j + 1] * g.y;
      }
      acc[u] = a;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
      for (int sh = kLanes / 2; sh > 0; sh >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], sh);
    }
    if (l == 0) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t item = base + u * kPerPass + sub;
        if (item < total) delta[(item % heads) * seqlen + item / heads] = acc[u];
      }
    }
  }
}

}  // namespace

cudaError_t launch_range_gather(const void* src, void* dst, const int64_t* ranges,
                                const int64_t* offsets, int64_t num_ranges, int64_t total_rows,
                                int64_t row_bytes, cudaStream_t stream) {
  if (num_ranges == 0 || total_rows == 0) return cudaSuccess;
  const int64_t vec = row_bytes / 16;
  if (vec >= 32) {
    range_gather_rows_kernel<<<grid_for(total_rows * 32, 256), 256, 0, stream>>>(
        static_cast<const uint4*>(src), static_cast<uint4*>(dst), ranges, offsets, num_ranges,
        total_rows, vec);
  } else {
    range_gather_kernel<<<grid_for(total_rows * vec, 256), 256, 0, stream>>>(
        static_cast<const uint4*>(src), static_cast<uint4*>(dst), ranges, offsets, num_ranges,
        total_rows, vec);
  }
  return cudaGetLastError();
}

cudaError_t launch_range_copy_to(const void* src, const int64_t* ranges, const int64_t* offsets,
                                 const unsigned long long* dst_base, const int64_t* dst_row, int64_t num_ranges,
                                 int64_t total_rows, int64_t row_bytes, cudaStream_t stream) {
  if (num_ranges == 0 || total_rows == 0) return cudaSuccess;
  range_copy_to_kernel<<<grid_for(total_rows * 32, 256), 256, 0, stream>>>(
      static_cast<const uint4*>(src), ranges, offsets, dst_base, dst_row, num_ranges, total_rows,
      row_bytes / 16);
  return cudaGetLastError();
}

cudaError_t launch_range_scatter_add_from(float* dst, const int64_t* ranges, const int64_t* offsets,
                                          const unsigned long long* src_base, const int64_t* src_row,
                                          int64_t num_ranges, int64_t total_rows, int64_t row_elems,
                                          cudaStream_t stream) {
  if (num_ranges == 0 || total_rows == 0) return cudaSuccess;
  range_scatter_add_from_kernel<<<grid_for(total_rows * 32, 256), 256, 0, stream>>>(
      reinterpret_cast<float4*>(dst), ranges, offsets, src_base, src_row, num_ranges, total_rows, row_elems / 4);
  return cudaGetLastError();
}

cudaError_t launch_flags_signal(unsigned int* const* flags, int n, unsigned int value, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  flags_signal_kernel<<<1, 32, 0, stream>>>(flags, n, value);
  return cudaGetLastError();
}

cudaError_t launch_flags_wait(const unsigned int* flags, unsigned int mask, unsigned int value,
                              cudaStream_t stream) {
  if (mask == 0) return cudaSuccess;
  flags_wait_kernel<<<1, 32, 0, stream>>>(flags, mask, value);
  return cudaGetLastError();
}

cudaError_t launch_range_scatter_add_f32(const float* src, float* dst, const int64_t* ranges,
                                         const int64_t* offsets, int64_t num_ranges,
                                         int64_t total_rows, int64_t row_elems,
                                         cudaStream_t stream) {
  if (num_ranges == 0 || total_rows == 0) return cudaSuccess;
  const int64_t vec = row_elems / 4;
  if (vec >= 32) {
    range_scatter_add_rows_kernel<<<grid_for(total_rows * 32, 256), 256, 0, stream>>>(
        reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), ranges, offsets,
        num_ranges, total_rows, vec);
  } else {
    range_scatter_add_kernel<<<grid_for(total_rows * vec, 256), 256, 0, stream>>>(
        reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), ranges, offsets,
        num_ranges, total_rows, vec);
  }
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
  const int grid = grid_for(seqlen * heads * (head_dim / 8) / 4, 256);
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
