// FFA forward for sm_100a: flexible (slice-list) masked attention, O and LSE.
//
// One CTA owns one 128-row query tile of one query head and walks every
// (tile, slice) work item the host planner produced for that tile, so
// overlapping slices are merged inside the CTA (MULTIPLICITY semantics,
// reference proj/include/magiplan/mask.hpp:85) with no atomics.
//
// Warp roles (192 threads):
//   warps 0-3  softmax: thread i owns query row i of the tile. Reads S from
//              TMEM (tcgen05.ld 32x32b), applies the per-slice row bounds,
//              runs the online softmax, rescales O in TMEM, writes P (bf16)
//              into a 128B-swizzled smem tile, and finally the epilogue.
//   warp 4     TMA producer: Q once, then K/V tiles through a 2-stage ring.
//   warp 5     MMA issuer (one lane): S = Q K^T into a double-buffered TMEM
//              accumulator, O += P V into a TMEM accumulator.
// TMEM columns: S0 [0,128) S1 [128,256) O [256, 256+D).
#include <cuda_runtime.h>

#include <cmath>

#include "ffa_common.cuh"
#include "sm100.cuh"
#include "tma_host.h"

namespace magi {
namespace {

constexpr int kStages = 2;
constexpr uint32_t kBox = 128 * 64 * 2;  // one TMA box: 128 rows x 64 bf16 (128B swizzle)
constexpr int kSoftmaxThreads = 128;
constexpr int kThreads = 192;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct FwdParams {
  const FwdTile* tiles;
  const FwdItem* items;
  int32_t num_tiles;
  int32_t seqlen_q, seqlen_k;
  int32_t hq, hk;
  float scale_log2;
  void* out;
  float* lse;
  int32_t out_f32;
  int32_t accumulate;
};

template <int D>
struct FwdSmem {
  static constexpr uint32_t kTileBytes = (D / 64) * kBox;
  static constexpr uint32_t kQ = 0;
  static constexpr uint32_t kK = kQ + kTileBytes;
  static constexpr uint32_t kV = kK + kStages * kTileBytes;
  static constexpr uint32_t kP = kV + kStages * kTileBytes;
  static constexpr uint32_t kBytes = kP + 2 * kBox;
};

struct FwdBarriers {
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], s_free[2];
  uint64_t p_full;
  uint64_t o_done;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    ffa_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                   const __grid_constant__ CUtensorMap tmap_k,
                   const __grid_constant__ CUtensorMap tmap_v, const FwdParams p) {
  using L = FwdSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ FwdBarriers bars;
  __shared__ uint32_t tmem_base_slot;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tile_rank = blockIdx.x / p.hq;
  const int head = blockIdx.x % p.hq;
  const int head_k = head / (p.hq / p.hk);
  const FwdTile tile = p.tiles[tile_rank];
  const int n_total = tile.n_ktiles;

  if (threadIdx.x == 0) {
    mbar_init(&bars.q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 1);
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars.s_full[b], 1);
      mbar_init(&bars.s_free[b], kSoftmaxThreads);
    }
    mbar_init(&bars.p_full, kSoftmaxThreads);
    mbar_init(&bars.o_done, 1);
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(&tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_slot;
  const uint32_t tmem_s = tmem;        // two 128-column S buffers
  const uint32_t tmem_o = tmem + 256;  // D columns

  uint8_t* sQ = smem + L::kQ;
  uint8_t* sK = smem + L::kK;
  uint8_t* sV = smem + L::kV;
  uint8_t* sP = smem + L::kP;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && n_total > 0) {
      tma_prefetch_desc(&tmap_q);
      tma_prefetch_desc(&tmap_k);
      tma_prefetch_desc(&tmap_v);
      mbar_arrive_expect_tx(&bars.q_full, L::kTileBytes);
      for (int c = 0; c < D / 64; ++c)
        tma_load_3d(sQ + c * kBox, &tmap_q, &bars.q_full, c * 64, head, tile.q0);
      PipeState st;
      for (int it = tile.item_begin; it < tile.item_end; ++it) {
        const FwdItem item = p.items[it];
        for (int j = 0; j < item.n_ktiles; ++j) {
          const int k0 = item.k_begin + j * kBlockN;
          mbar_wait(&bars.k_empty[st.index], st.phase ^ 1);
          mbar_arrive_expect_tx(&bars.k_full[st.index], L::kTileBytes);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sK + st.index * L::kTileBytes + c * kBox, &tmap_k, &bars.k_full[st.index],
                        c * 64, head_k, k0);
          mbar_wait(&bars.v_empty[st.index], st.phase ^ 1);
          mbar_arrive_expect_tx(&bars.v_full[st.index], L::kTileBytes);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sV + st.index * L::kTileBytes + c * kBox, &tmap_v, &bars.v_full[st.index],
                        c * 64, head_k, k0);
          st.advance<kStages>();
        }
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && n_total > 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, D, false, true);
      const uint32_t q_addr = smem_u32(sQ);
      const uint32_t p_addr = smem_u32(sP);
      mbar_wait(&bars.q_full, 0);
      tc_fence_after();

      auto issue_qk = [&](int t, const PipeState& st) {
        const int b = t & 1;
        if (t >= 2) mbar_wait(&bars.s_free[b], ((t - 2) >> 1) & 1);
        mbar_wait(&bars.k_full[st.index], st.phase);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st.index * L::kTileBytes);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k / 4) * kBox + (k % 4) * 32;
          umma_bf16_ss(tmem_s + b * 128, make_smem_desc(q_addr + off, 16, 1024),
                       make_smem_desc(k_addr + off, 16, 1024), idesc_qk, k > 0);
        }
        umma_commit(&bars.s_full[b]);
        umma_commit(&bars.k_empty[st.index]);
      };

      PipeState kst, vst;
      issue_qk(0, kst);
      kst.advance<kStages>();
      for (int t = 0; t < n_total; ++t) {
        if (t + 1 < n_total) {
          issue_qk(t + 1, kst);
          kst.advance<kStages>();
        }
        mbar_wait(&bars.p_full, t & 1);
        mbar_wait(&bars.v_full[vst.index], vst.phase);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + vst.index * L::kTileBytes);
#pragma unroll
        for (int k = 0; k < kBlockN / 16; ++k) {
          const uint64_t adesc = make_smem_desc(p_addr + (k / 4) * kBox + (k % 4) * 32, 16, 1024);
          const uint64_t bdesc = make_smem_desc(v_addr + k * 16 * 128, kBox, 1024);
          umma_bf16_ss(tmem_o, adesc, bdesc, idesc_pv, (t > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&bars.o_done);
        umma_commit(&bars.v_empty[vst.index]);
        vst.advance<kStages>();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int row = warp * 32 + lane;
    const int q = tile.q0 + row;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    float m = -INFINITY;  // running max, log2 domain
    float l = 0.f;        // running sum of 2^(x - m)
    int t = 0;
    for (int it = tile.item_begin; it < tile.item_end; ++it) {
      const FwdItem item = p.items[it];
      int32_t lo, hi;
      row_bounds(item.qs, item.qe, item.ks, item.ke, item.type, q, lo, hi);
      for (int j = 0; j < item.n_ktiles; ++j, ++t) {
        const int k0 = item.k_begin + j * kBlockN;
        const int b = t & 1;
        mbar_wait(&bars.s_full[b], (t >> 1) & 1);
        tc_fence_after();
        uint32_t s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t(&chunk)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]);
          tmem_ld32(tmem_s + lane_off + b * 128 + c * 32, chunk);
        }
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars.s_free[b]);

        float x[128];
        float mt = -INFINITY;
        const bool full = lo <= k0 && k0 + kBlockN <= hi;
        if (full) {
#pragma unroll
          for (int i = 0; i < 128; ++i) {
            x[i] = __uint_as_float(s[i]) * p.scale_log2;
            mt = fmaxf(mt, x[i]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 128; ++i) {
            const int c = k0 + i;
            x[i] = (c >= lo && c < hi) ? __uint_as_float(s[i]) * p.scale_log2 : -INFINITY;
            mt = fmaxf(mt, x[i]);
          }
        }
        const float m_new = fmaxf(m, mt);
        const float m_use = m_new == -INFINITY ? 0.f : m_new;
        const float alpha = fast_exp2(m - m_use);
        float rs = 0.f;
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          x[i] = fast_exp2(x[i] - m_use);
          rs += x[i];
        }
        l = l * alpha + rs;
        m = m_new;

        // P buffer and O are owned by the previous PV MMA until it retires.
        if (t > 0) {
          mbar_wait(&bars.o_done, (t - 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(tmem_o + lane_off + c * 32, o);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(tmem_o + lane_off + c * 32, o);
            }
            tmem_st_wait();
          }
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          uint4 v;
          v.x = pack_bf16(x[c * 8 + 0], x[c * 8 + 1]);
          v.y = pack_bf16(x[c * 8 + 2], x[c * 8 + 3]);
          v.z = pack_bf16(x[c * 8 + 4], x[c * 8 + 5]);
          v.w = pack_bf16(x[c * 8 + 6], x[c * 8 + 7]);
          *reinterpret_cast<uint4*>(sP + (c / 8) * kBox + sw128_offset(row, c % 8)) = v;
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars.p_full);
      }
    }

    // ---------------------------------------------------------- epilogue
    const bool valid = q < p.seqlen_q;
    const bool has = l > 0.f;
    const float lse_cur = has ? (m * kLn2 + logf(l)) : -INFINITY;
    const float inv_l = has ? 1.f / l : 0.f;
    if (n_total > 0) {
      mbar_wait(&bars.o_done, (n_total - 1) & 1);
      tc_fence_after();
    }
    const size_t row_off = (static_cast<size_t>(q) * p.hq + head) * D;
    float* lse_ptr = p.lse + static_cast<size_t>(head) * p.seqlen_q + q;
    if (p.accumulate) {
      // merge into (out, lse) with the log-sum-exp correction; f32 output
      const float lse_old = valid ? *lse_ptr : -INFINITY;
      const float lse_new = has ? (lse_old > lse_cur ? lse_old + log1pf(__expf(lse_cur - lse_old))
                                                     : lse_cur + log1pf(__expf(lse_old - lse_cur)))
                                : lse_old;
      const float w_old = has ? __expf(lse_old - lse_new) : 1.f;
      const float w_cur = has ? __expf(lse_cur - lse_new) * inv_l : 0.f;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tmem_o + lane_off + c * 32, o);
        tmem_ld_wait();
        if (valid && has) {
          float* dst = reinterpret_cast<float*>(p.out) + row_off + c * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 a = *reinterpret_cast<float4*>(dst + i);
            a.x = a.x * w_old + __uint_as_float(o[i + 0]) * w_cur;
            a.y = a.y * w_old + __uint_as_float(o[i + 1]) * w_cur;
            a.z = a.z * w_old + __uint_as_float(o[i + 2]) * w_cur;
            a.w = a.w * w_old + __uint_as_float(o[i + 3]) * w_cur;
            *reinterpret_cast<float4*>(dst + i) = a;
          }
        }
      }
      if (valid && has) *lse_ptr = lse_new;
    } else {
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        if (n_total > 0) {
          tmem_ld32(tmem_o + lane_off + c * 32, o);
          tmem_ld_wait();
        }
        if (!valid) continue;
        if (p.out_f32) {
          float* dst = reinterpret_cast<float*>(p.out) + row_off + c * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 a;
            a.x = has ? __uint_as_float(o[i + 0]) * inv_l : 0.f;
            a.y = has ? __uint_as_float(o[i + 1]) * inv_l : 0.f;
            a.z = has ? __uint_as_float(o[i + 2]) * inv_l : 0.f;
            a.w = has ? __uint_as_float(o[i + 3]) * inv_l : 0.f;
            *reinterpret_cast<float4*>(dst + i) = a;
          }
        } else {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + row_off + c * 32;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = has ? pack_bf16(__uint_as_float(o[i + 0]) * inv_l, __uint_as_float(o[i + 1]) * inv_l) : 0u;
            v.y = has ? pack_bf16(__uint_as_float(o[i + 2]) * inv_l, __uint_as_float(o[i + 3]) * inv_l) : 0u;
            v.z = has ? pack_bf16(__uint_as_float(o[i + 4]) * inv_l, __uint_as_float(o[i + 5]) * inv_l) : 0u;
            v.w = has ? pack_bf16(__uint_as_float(o[i + 6]) * inv_l, __uint_as_float(o[i + 7]) * inv_l) : 0u;
            *reinterpret_cast<uint4*>(dst + i) = v;
          }
        }
      }
      if (valid) *lse_ptr = lse_cur;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D>
cudaError_t launch_fwd_impl(const FwdParams& prm, const void* q, const void* k, const void* v,
                            cudaStream_t stream) {
  const CUtensorMap tq = make_tmap_thd(q, prm.seqlen_q, prm.hq, D, 128);
  const CUtensorMap tk = make_tmap_thd(k, prm.seqlen_k, prm.hk, D, 128);
  const CUtensorMap tv = make_tmap_thd(v, prm.seqlen_k, prm.hk, D, 128);
  const int smem = FwdSmem<D>::kBytes + 1024;
  cudaError_t err =
      cudaFuncSetAttribute(ffa_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return err;
  const dim3 grid(static_cast<unsigned>(prm.num_tiles) * prm.hq);
  ffa_fwd_kernel<D><<<grid, kThreads, smem, stream>>>(tq, tk, tv, prm);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ffa_fwd(const FwdTile* tiles, const FwdItem* items, int num_tiles,
                           int seqlen_q, int seqlen_k, int hq, int hk, int head_dim,
                           float softmax_scale, const void* q, const void* k, const void* v,
                           void* out, float* lse, int out_f32, int accumulate,
                           cudaStream_t stream) {
  if (num_tiles == 0 || hq == 0) return cudaSuccess;
  FwdParams prm;
  prm.tiles = tiles;
  prm.items = items;
  prm.num_tiles = num_tiles;
  prm.seqlen_q = seqlen_q;
  prm.seqlen_k = seqlen_k;
  prm.hq = hq;
  prm.hk = hk;
  prm.scale_log2 = softmax_scale * kLog2e;
  prm.out = out;
  prm.lse = lse;
  prm.out_f32 = out_f32;
  prm.accumulate = accumulate;
  if (head_dim == 128) return launch_fwd_impl<128>(prm, q, k, v, stream);
  if (head_dim == 64) return launch_fwd_impl<64>(prm, q, k, v, stream);
  return cudaErrorInvalidValue;
}

}  // namespace magi
