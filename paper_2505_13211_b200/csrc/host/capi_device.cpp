// C ABI for the device entry points: FFA plan / forward / backward, the
// context-parallel range movement kernels and diagnostics. Each function
// validates its arguments (MAGIPLAN_ERR_USAGE), launches asynchronously on the
// caller's stream and maps CUDA launch failures to MAGIPLAN_ERR_INTERNAL.
#include <cuda_runtime.h>

#include <cstring>

#include "capi_util.hpp"
#include "ffa_plan.hpp"
#include "mask.hpp"

namespace magi {
cudaError_t launch_umma_tile(const void* a, const void* b, float* c, int b_mn_major,
                             cudaStream_t stream);
cudaError_t launch_ffa_fwd(const FwdWork& work,
                           int seqlen_q, int seqlen_k, int hq, int hk, int head_dim,
                           float softmax_scale, const void* q, const void* k, const void* v,
                           void* out, float* lse, int out_f32, int accumulate,
                           cudaStream_t stream);
cudaError_t launch_ffa_bwd_preprocess(const void* out, const void* grad_out, float* delta,
                                      int64_t seqlen, int64_t heads, int head_dim, int out_f32,
                                      cudaStream_t stream);
cudaError_t launch_ffa_bwd(const FwdTile* q_tiles, const FwdItem* q_items, int num_q_tiles,
                           const BwdTile* k_tiles, const BwdItem* k_items, int num_k_tiles,
                           int seqlen_q, int seqlen_k, int hq, int hk, int head_dim,
                           float softmax_scale, const void* q, const void* k, const void* v,
                           const float* lse, const float* delta, const void* grad_out,
                           void* grad_q, void* grad_k, void* grad_v, int grad_f32,
                           int accumulate, int parts, cudaStream_t stream);
cudaError_t launch_range_copy_to(const void* src, const int64_t* ranges, const int64_t* offsets,
                                 const unsigned long long* dst_base, const int64_t* dst_row, int64_t num_ranges,
                                 int64_t total_rows, int64_t row_bytes, cudaStream_t stream);
cudaError_t launch_flags_signal(unsigned int* const* flags, int n, unsigned int value, cudaStream_t stream);
cudaError_t launch_range_scatter_add_from(float* dst, const int64_t* ranges, const int64_t* offsets,
                                          const unsigned long long* src_base, const int64_t* src_row,
                                          int64_t num_ranges, int64_t total_rows, int64_t row_elems,
                                          cudaStream_t stream);
cudaError_t launch_flags_wait(const unsigned int* flags, unsigned int mask, unsigned int value,
                              cudaStream_t stream);
cudaError_t launch_range_gather(const void* src, void* dst, const int64_t* ranges,
                                const int64_t* offsets, int64_t num_ranges, int64_t total_rows,
                                int64_t row_bytes, cudaStream_t stream);
cudaError_t launch_range_scatter_add_f32(const float* src, float* dst, const int64_t* ranges,
                                         const int64_t* offsets, int64_t num_ranges,
                                         int64_t total_rows, int64_t row_elems,
                                         cudaStream_t stream);
cudaError_t launch_cast_f32_bf16(const float* src, void* dst, int64_t n, cudaStream_t stream);
void set_bwd_trace(long long* buffer, int block);
void set_fwd_trace(long long* buffer, int block);
}  // namespace magi

struct magiplan_ffa_plan {
  magiplan::FfaPlan plan;
};

// defined in capi.cpp
struct magiplan_mask {
  magiplan::AttnMask mask;
};

using magiplan::UsageError;
using magiplan::capi::cuda_check;
using magiplan::capi::dup_string;
using magiplan::capi::guarded;

namespace {

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

void check_heads(int64_t hq, int64_t hk) {
  if (hq <= 0 || hk <= 0 || hq % hk != 0) {
    throw UsageError("num_heads_q must be a positive multiple of num_heads_k (got " +
                     std::to_string(hq) + ", " + std::to_string(hk) + ")");
  }
  if (hq > 65535) throw UsageError("num_heads_q too large");
}

void check_dtype(int32_t dtype, int32_t accumulate) {
  if (dtype != MAGIPLAN_F32 && dtype != MAGIPLAN_BF16) throw UsageError("unknown dtype");
  if (accumulate && dtype != MAGIPLAN_F32) {
    throw UsageError("accumulate requires MAGIPLAN_F32 outputs");
  }
}

magiplan_ffa_plan* make_plan(std::vector<magi::SliceGeom> slices, int64_t sq, int64_t sk,
                             int32_t head_dim) {
  auto* handle = new magiplan_ffa_plan;
  try {
    handle->plan.seqlen_q = sq;
    handle->plan.seqlen_k = sk;
    handle->plan.head_dim = head_dim;
    handle->plan.slices = std::move(slices);
    magiplan::build_ffa_worklists(handle->plan);
  } catch (...) {
    delete handle;
    throw;
  }
  return handle;
}

}  // namespace

extern "C" {

magiplan_status magiplan_ffa_plan_create(const int64_t* q_ranges, const int64_t* k_ranges,
                                         const int32_t* types, int64_t num_slices,
                                         int64_t seqlen_q, int64_t seqlen_k, int32_t head_dim,
                                         magiplan_ffa_plan** out_plan) {
  MAGI_REQUIRE(out_plan && (num_slices == 0 || (q_ranges && k_ranges && types)));
  return guarded([&] {
    if (num_slices < 0) throw UsageError("num_slices must be >= 0");
    std::vector<magi::SliceGeom> slices;
    slices.reserve(static_cast<std::size_t>(num_slices));
    for (int64_t i = 0; i < num_slices; ++i) {
      const int64_t v[4] = {q_ranges[2 * i], q_ranges[2 * i + 1], k_ranges[2 * i],
                            k_ranges[2 * i + 1]};
      for (int64_t x : v) {
        if (x < 0 || x > (int64_t{1} << 31) - 1) {
          throw UsageError("slice " + std::to_string(i) + ": malformed range");
        }
      }
      slices.push_back({static_cast<int32_t>(v[0]), static_cast<int32_t>(v[1]),
                        static_cast<int32_t>(v[2]), static_cast<int32_t>(v[3]), types[i]});
    }
    *out_plan = make_plan(std::move(slices), seqlen_q, seqlen_k, head_dim);
  });
}

magiplan_status magiplan_ffa_plan_from_mask(const magiplan_mask* mask, int32_t head_dim,
                                            magiplan_ffa_plan** out_plan) {
  MAGI_REQUIRE(mask && out_plan);
  return guarded([&] {
    std::vector<magi::SliceGeom> slices;
    for (const auto& s : mask->mask.slices) {
      slices.push_back({static_cast<int32_t>(s.q.start), static_cast<int32_t>(s.q.end),
                        static_cast<int32_t>(s.k.start), static_cast<int32_t>(s.k.end),
                        static_cast<int32_t>(s.type)});
    }
    *out_plan = make_plan(std::move(slices), mask->mask.seqlen_q, mask->mask.seqlen_k, head_dim);
  });
}

void magiplan_ffa_plan_free(magiplan_ffa_plan* plan) { delete plan; }

magiplan_status magiplan_ffa_plan_describe(const magiplan_ffa_plan* plan, char** out_json) {
  MAGI_REQUIRE(plan && out_json);
  return guarded([&] { *out_json = dup_string(plan->plan.describe_json()); });
}

magiplan_status magiplan_ffa_plan_prepare(magiplan_ffa_plan* plan) {
  MAGI_REQUIRE(plan);
  return guarded([&] { magiplan::ensure_uploaded(plan->plan); });
}

magiplan_status magiplan_ffa_fwd(const magiplan_ffa_plan* plan, const void* q, const void* k,
                                 const void* v, void* out, float* lse, int64_t num_heads_q,
                                 int64_t num_heads_k, float softmax_scale, int32_t out_dtype,
                                 int32_t accumulate, void* cuda_stream) {
  MAGI_REQUIRE(plan && q && k && v && out && lse);
  return guarded([&] {
    check_heads(num_heads_q, num_heads_k);
    check_dtype(out_dtype, accumulate);
    auto& P = const_cast<magiplan_ffa_plan*>(plan)->plan;
    magiplan::ensure_uploaded(P);
    cuda_check(magi::launch_ffa_fwd(magiplan::fwd_work(P),
                                    static_cast<int>(P.seqlen_q), static_cast<int>(P.seqlen_k),
                                    static_cast<int>(num_heads_q), static_cast<int>(num_heads_k),
                                    P.head_dim, softmax_scale, q, k, v, out, lse,
                                    out_dtype == MAGIPLAN_F32, accumulate != 0,
                                    as_stream(cuda_stream)),
               "ffa_fwd launch");
  });
}

magiplan_status magiplan_ffa_bwd_preprocess(const void* out, const void* grad_out, float* delta,
                                            int64_t seqlen, int64_t num_heads, int32_t head_dim,
                                            int32_t out_dtype, void* cuda_stream) {
  MAGI_REQUIRE(out && grad_out && delta);
  return guarded([&] {
    check_dtype(out_dtype, 0);
    if (seqlen < 0 || num_heads <= 0) throw UsageError("bad seqlen / num_heads");
    if (head_dim != 64 && head_dim != 128) throw UsageError("head_dim must be 64 or 128");
    cuda_check(magi::launch_ffa_bwd_preprocess(out, grad_out, delta, seqlen, num_heads, head_dim,
                                               out_dtype == MAGIPLAN_F32, as_stream(cuda_stream)),
               "ffa_bwd_preprocess launch");
  });
}

namespace {
magiplan_status ffa_bwd_parts(const magiplan_ffa_plan* plan, const void* q, const void* k,
                              const void* v, const float* lse, const float* delta,
                              const void* grad_out, void* grad_q, void* grad_k, void* grad_v,
                              int64_t num_heads_q, int64_t num_heads_k, float softmax_scale,
                              int32_t grad_dtype, int32_t accumulate, int parts,
                              void* cuda_stream) {
  return guarded([&] {
    check_heads(num_heads_q, num_heads_k);
    check_dtype(grad_dtype, accumulate);
    auto& P = const_cast<magiplan_ffa_plan*>(plan)->plan;
    magiplan::ensure_uploaded(P);
    cuda_check(
        magi::launch_ffa_bwd(P.d_fwd_tiles, P.d_fwd_items, static_cast<int>(P.fwd_tiles.size()),
                             P.d_bwd_tiles, P.d_bwd_items, static_cast<int>(P.bwd_tiles.size()),
                             static_cast<int>(P.seqlen_q), static_cast<int>(P.seqlen_k),
                             static_cast<int>(num_heads_q), static_cast<int>(num_heads_k),
                             P.head_dim, softmax_scale, q, k, v, lse, delta, grad_out, grad_q,
                             grad_k, grad_v, grad_dtype == MAGIPLAN_F32, accumulate != 0, parts,
                             as_stream(cuda_stream)),
        "ffa_bwd launch");
  });
}
}  // namespace

magiplan_status magiplan_ffa_bwd(const magiplan_ffa_plan* plan, const void* q, const void* k,
                                 const void* v, const float* lse, const float* delta,
                                 const void* grad_out, void* grad_q, void* grad_k, void* grad_v,
                                 int64_t num_heads_q, int64_t num_heads_k, float softmax_scale,
                                 int32_t grad_dtype, int32_t accumulate, void* cuda_stream) {
  MAGI_REQUIRE(plan && q && k && v && lse && delta && grad_out && grad_q && grad_k && grad_v);
  return ffa_bwd_parts(plan, q, k, v, lse, delta, grad_out, grad_q, grad_k, grad_v, num_heads_q,
                       num_heads_k, softmax_scale, grad_dtype, accumulate, 3, cuda_stream);
}

magiplan_status magiplan_ffa_bwd_stage(const magiplan_ffa_plan* plan, const void* q, const void* k,
                                       const void* v, const float* lse, const float* delta,
                                       const void* grad_out, float* grad_q, float* grad_k,
                                       float* grad_v, int64_t num_heads_q, int64_t num_heads_k,
                                       float softmax_scale, void* cuda_stream) {
  MAGI_REQUIRE(plan && q && k && v && lse && delta && grad_out && grad_q && grad_k && grad_v);
  // the k-major pass writes the stage's fresh partial dK / dV, the q-major
  // pass adds the stage's dQ into the running dQ
  const magiplan_status st =
      ffa_bwd_parts(plan, q, k, v, lse, delta, grad_out, grad_k, grad_k, grad_v, num_heads_q, num_heads_k,
                    softmax_scale, MAGIPLAN_F32, 0, 1, cuda_stream);
  if (st != MAGIPLAN_OK) return st;
  return ffa_bwd_parts(plan, q, k, v, lse, delta, grad_out, grad_q, grad_q, grad_q, num_heads_q, num_heads_k,
                       softmax_scale, MAGIPLAN_F32, 1, 2, cuda_stream);
}

magiplan_status magiplan_ffa_bwd_dkdv(const magiplan_ffa_plan* plan, const void* q,
                                      const void* k, const void* v, const float* lse,
                                      const float* delta, const void* grad_out, void* grad_k,
                                      void* grad_v, int64_t num_heads_q, int64_t num_heads_k,
                                      float softmax_scale, int32_t grad_dtype,
                                      int32_t accumulate, void* cuda_stream) {
  MAGI_REQUIRE(plan && q && k && v && lse && delta && grad_out && grad_k && grad_v);
  return ffa_bwd_parts(plan, q, k, v, lse, delta, grad_out, grad_k, grad_k, grad_v, num_heads_q,
                       num_heads_k, softmax_scale, grad_dtype, accumulate, 1, cuda_stream);
}

magiplan_status magiplan_ffa_bwd_dq(const magiplan_ffa_plan* plan, const void* q, const void* k,
                                    const void* v, const float* lse, const float* delta,
                                    const void* grad_out, void* grad_q, int64_t num_heads_q,
                                    int64_t num_heads_k, float softmax_scale, int32_t grad_dtype,
                                    int32_t accumulate, void* cuda_stream) {
  MAGI_REQUIRE(plan && q && k && v && lse && delta && grad_out && grad_q);
  return ffa_bwd_parts(plan, q, k, v, lse, delta, grad_out, grad_q, grad_q, grad_q, num_heads_q,
                       num_heads_k, softmax_scale, grad_dtype, accumulate, 2, cuda_stream);
}

magiplan_status magiplan_range_gather(const void* src, void* dst, const int64_t* ranges,
                                      const int64_t* offsets, int64_t num_ranges,
                                      int64_t total_rows, int64_t row_bytes, void* cuda_stream) {
  MAGI_REQUIRE(src && dst && (num_ranges == 0 || (ranges && offsets)));
  return guarded([&] {
    if (num_ranges < 0 || total_rows < 0 || row_bytes <= 0 || row_bytes % 16 != 0) {
      throw UsageError("range_gather: row_bytes must be a positive multiple of 16");
    }
    cuda_check(magi::launch_range_gather(src, dst, ranges, offsets, num_ranges, total_rows,
                                         row_bytes, as_stream(cuda_stream)),
               "range_gather launch");
  });
}

magiplan_status magiplan_range_scatter_add_f32(const float* src, float* dst,
                                               const int64_t* ranges, const int64_t* offsets,
                                               int64_t num_ranges, int64_t total_rows,
                                               int64_t row_elems, void* cuda_stream) {
  MAGI_REQUIRE(src && dst && (num_ranges == 0 || (ranges && offsets)));
  return guarded([&] {
    if (num_ranges < 0 || total_rows < 0 || row_elems <= 0 || row_elems % 4 != 0) {
      throw UsageError("range_scatter_add: row_elems must be a positive multiple of 4");
    }
    cuda_check(magi::launch_range_scatter_add_f32(src, dst, ranges, offsets, num_ranges,
                                                  total_rows, row_elems, as_stream(cuda_stream)),
               "range_scatter_add launch");
  });
}

// ---------------------------------------------------------------- peer memory
magiplan_status magiplan_p2p_malloc(int64_t bytes, void** out_ptr, unsigned char* out_handle) {
  MAGI_REQUIRE(out_ptr && out_handle);
  return guarded([&] {
    if (bytes <= 0) throw UsageError("p2p_malloc: bytes must be > 0");
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, static_cast<size_t>(bytes)), "p2p_malloc");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      cuda_check(e, "p2p_malloc: cudaIpcGetMemHandle");
    }
    std::memcpy(out_handle, &h, sizeof(h));
    *out_ptr = p;
  });
}
magiplan_status magiplan_p2p_free(void* ptr) {
  MAGI_REQUIRE(ptr);
  return guarded([&] { cuda_check(cudaFree(ptr), "p2p_free"); });
}
magiplan_status magiplan_p2p_open(const unsigned char* handle, void** out_ptr) {
  MAGI_REQUIRE(handle && out_ptr);
  return guarded([&] {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "p2p_open");
    *out_ptr = p;
  });
}
magiplan_status magiplan_p2p_close(void* ptr) {
  MAGI_REQUIRE(ptr);
  return guarded([&] { cuda_check(cudaIpcCloseMemHandle(ptr), "p2p_close"); });
}
magiplan_status magiplan_range_copy_to(const void* src, const int64_t* ranges, const int64_t* offsets,
                                       const uint64_t* dst_base, const int64_t* dst_row, int64_t num_ranges,
                                       int64_t total_rows, int64_t row_bytes, void* cuda_stream) {
  MAGI_REQUIRE(src && (num_ranges == 0 || (ranges && offsets && dst_base && dst_row)));
  return guarded([&] {
    if (num_ranges < 0 || total_rows < 0 || row_bytes <= 0 || row_bytes % 16 != 0) {
      throw UsageError("range_copy_to: row_bytes must be a positive multiple of 16");
    }
    cuda_check(magi::launch_range_copy_to(src, ranges, offsets,
                                          reinterpret_cast<const unsigned long long*>(dst_base), dst_row,
                                          num_ranges, total_rows, row_bytes, as_stream(cuda_stream)),
               "range_copy_to launch");
  });
}
magiplan_status magiplan_range_scatter_add_from(float* dst, const int64_t* ranges, const int64_t* offsets,
                                                const uint64_t* src_base, const int64_t* src_row,
                                                int64_t num_ranges, int64_t total_rows, int64_t row_elems,
                                                void* cuda_stream) {
  MAGI_REQUIRE(dst && (num_ranges == 0 || (ranges && offsets && src_base && src_row)));
  return guarded([&] {
    if (num_ranges < 0 || total_rows < 0 || row_elems <= 0 || row_elems % 4 != 0) {
      throw UsageError("range_scatter_add_from: row_elems must be a positive multiple of 4");
    }
    cuda_check(magi::launch_range_scatter_add_from(dst, ranges, offsets,
                                                   reinterpret_cast<const unsigned long long*>(src_base), src_row,
                                                   num_ranges, total_rows, row_elems, as_stream(cuda_stream)),
               "range_scatter_add_from launch");
  });
}
magiplan_status magiplan_flags_signal(const uint64_t* flag_ptrs, int32_t n, uint32_t value, void* cuda_stream) {
  MAGI_REQUIRE(n == 0 || flag_ptrs);
  return guarded([&] {
    if (n < 0 || n > 32) throw UsageError("flags_signal: 0 <= n <= 32");
    cuda_check(magi::launch_flags_signal(reinterpret_cast<unsigned int* const*>(flag_ptrs), n, value,
                                         as_stream(cuda_stream)),
               "flags_signal launch");
  });
}
magiplan_status magiplan_flags_wait(const uint32_t* flags, uint32_t mask, uint32_t value, void* cuda_stream) {
  MAGI_REQUIRE(mask == 0 || flags);
  return guarded([&] {
    cuda_check(magi::launch_flags_wait(flags, mask, value, as_stream(cuda_stream)), "flags_wait launch");
  });
}

magiplan_status magiplan_cast_f32_bf16(const float* src, void* dst, int64_t n,
                                       void* cuda_stream) {
  MAGI_REQUIRE(src && dst);
  return guarded([&] {
    if (n < 0) throw UsageError("n must be >= 0");
    cuda_check(magi::launch_cast_f32_bf16(src, dst, n, as_stream(cuda_stream)), "cast launch");
  });
}

magiplan_status magiplan_debug_set_trace(void* device_buffer, int32_t block) {
#ifndef MAGI_TRACE
  if (device_buffer != nullptr) {
    return guarded([] { throw UsageError("tracing needs a library built with -DMAGI_TRACE"); });
  }
#endif
  magi::set_bwd_trace(static_cast<long long*>(device_buffer), block);
  magi::set_fwd_trace(static_cast<long long*>(device_buffer), block);
  return MAGIPLAN_OK;
}

magiplan_status magiplan_debug_umma_tile(const void* a, const void* b, float* c,
                                         int32_t b_mn_major, void* cuda_stream) {
  MAGI_REQUIRE(a && b && c);
  return guarded([&] {
    cuda_check(magi::launch_umma_tile(a, b, c, b_mn_major, as_stream(cuda_stream)),
               "umma tile launch");
  });
}

}  // extern "C"
