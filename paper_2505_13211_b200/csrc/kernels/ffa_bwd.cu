// FFA backward for sm_100a, deterministic (no unordered atomics).
//
// The five backward products of attention are split over two
// kernels so every gradient element has exactly one producing CTA and one
// fixed accumulation order:
//
//   dK/dV kernel (k-major, ffa_bwd_dkdv.inc): one CTA per (128-key tile,
//     key/value head), walking every (q head of the GQA group, slice item,
//     128-query tile) that touches its keys:
//       S^T = K Q^T, dP^T = V dO^T (SS) into TMEM; P^T into the consumed S^T
//       columns, dS^T = P^T (dP^T - delta) into the consumed dP^T columns
//       (packed bf16); dV += P^T dO, dK += dS^T Q (TS, A from TMEM).
//     dK / dV accumulate in TMEM over the whole walk and are written once.
//   dQ kernel (q-major, below): one CTA per (128-query tile, q head) over the
//     forward work list, Q and dO staged once into TMEM: S = Q K^T,
//     dP = dO V^T, dS = P (dP - delta) into the consumed dP columns,
//     dQ += dS K — all three TS.
//
// Overlap comes from issue order, not extra accumulators (TMEM is full); every
// hand-off that is not an mbarrier is implied by in-order MMA completion (an
// MMA that overwrites TMEM columns is issued after the MMAs that read them).
// All MMAs are M=128, N=128 (or N=D), K=16, each 128-deep GEMM issued as one
// asm block by an elected lane of a converged MMA warp.

#include <cuda_runtime.h>

#include <cmath>

#include "ffa_common.cuh"
#include "sm100.cuh"
#include "tma_host.h"

namespace magi {
namespace {

constexpr uint32_t kBox = 128 * 64 * 2;  // 128 rows x 64 bf16, 128B swizzle
constexpr int kThreads = 320;  // 8 elementwise warps + TMA warp + MMA warp
constexpr int kTmaWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kMath = 256;
constexpr int kStages = 2;
constexpr float kLog2e = 1.4426950408889634f;

struct BwdParams {
  const FwdTile* q_tiles;
  const FwdItem* q_items;
  const BwdTile* k_tiles;
  const BwdItem* k_items;
  int32_t seqlen_q, seqlen_k;
  int32_t hq, hk;
  float scale, scale_log2;
  const float* lse;
  const float* delta;
  void* dq;
  void* dk;
  void* dv;
  const void* q;     // dQ kernel stages Q / dO rows into TMEM directly
  const void* dout;
  int32_t grad_f32;
  int32_t accumulate;
  int32_t num_k_tiles, num_q_tiles;
  int32_t lse_tma;      // lse / delta rows fetched by TMA (row stride 16B-aligned)
  long long* trace;     // diagnostics: event log of one CTA (nullptr = off)
  int32_t trace_block;
  int32_t trace_kernel;  // 0: dK/dV kernel, 1: dQ kernel
};

long long* g_trace = nullptr;
int g_trace_block = 0;
int g_trace_kernel = 0;  // 0: dK/dV kernel, 1: dQ kernel

__device__ __forceinline__ void store_row(void* base, size_t row_off, const uint32_t (&o)[32],
                                          int c, float scale, bool f32, bool accumulate) {
  if (f32) {
    float* dst = static_cast<float*>(base) + row_off + c * 32;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 a;
      a.x = __uint_as_float(o[i + 0]) * scale;
      a.y = __uint_as_float(o[i + 1]) * scale;
      a.z = __uint_as_float(o[i + 2]) * scale;
      a.w = __uint_as_float(o[i + 3]) * scale;
      if (accumulate) {
        const float4 b = *reinterpret_cast<const float4*>(dst + i);
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
      }
      *reinterpret_cast<float4*>(dst + i) = a;
    }
  } else {
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(base) + row_off + c * 32;
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint4 v;
      v.x = pack_bf16(__uint_as_float(o[i + 0]) * scale, __uint_as_float(o[i + 1]) * scale);
      v.y = pack_bf16(__uint_as_float(o[i + 2]) * scale, __uint_as_float(o[i + 3]) * scale);
      v.z = pack_bf16(__uint_as_float(o[i + 4]) * scale, __uint_as_float(o[i + 5]) * scale);
      v.w = pack_bf16(__uint_as_float(o[i + 6]) * scale, __uint_as_float(o[i + 7]) * scale);
      *reinterpret_cast<uint4*>(dst + i) = v;
    }
  }
}

// Write a D-wide TMEM accumulator row to global memory (zeros when the CTA
// had no work; nothing when accumulating nothing).
template <int D>
__device__ __forceinline__ void epilogue_rows(uint32_t t_acc, bool has_work, bool valid, void* base,
                                              size_t row_off, float scale, bool f32, bool acc) {
#pragma unroll 1
  for (int c = 0; c < D / 32; ++c) {
    uint32_t o[32];
    if (has_work) {
      tmem_ld32(t_acc + c * 32, o);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = 0u;
    }
    if (valid && !(acc && !has_work)) store_row(base, row_off, o, c, scale, f32, acc);
  }
}

// D[tmem] (M=128, N=128) = A[128 rows, D] . B[128 rows, D]^T, both K-major
// SW128 tiles given by their descriptors; converged warp, one lane issues.
template <int D>
__device__ __forceinline__ void mma_rows_x_rows(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc) {
  constexpr uint32_t idesc = make_idesc_bf16(128, 128, false, false);
  if constexpr (D == 128) {
    umma_gemm_ss_k128(d_tmem, a_desc, b_desc, idesc, 0);
  } else {
#pragma unroll
    for (int k = 0; k < D / 16; ++k) {
      const uint32_t off = (k / 4) * kBox + (k % 4) * 32;
      umma_ss_elect(d_tmem, desc_add(a_desc, off), desc_add(b_desc, off), idesc, k > 0);
    }
  }
}

// K-major SW128 descriptor (row tiles loaded by TMA) / MN-major view of the
// same tile (16 rows per k-step, 64-column boxes kBox apart)
__device__ __forceinline__ uint64_t kmajor_desc(const void* tile) { return make_smem_desc(smem_u32(tile), 16, 1024); }
__device__ __forceinline__ uint64_t mnmajor_desc(const void* tile) {
  return make_smem_desc(smem_u32(tile), kBox, 1024);
}

#include "ffa_bwd_dkdv.inc"

// =========================================================================== dQ
// All three MMAs take A from TMEM: Q and dO are staged into TMEM once per CTA
// (packed bf16, thread = row), dS goes back into the consumed dP columns, so
// shared memory only carries the streamed K / V tiles (B operands).
// TMEM: S [0,128) dP [128,256) dQ [256,256+D) Q [384,384+D/2) dO [448,448+D/2).
template <int D>
struct DqSmem {
  static constexpr uint32_t kTile = (D / 64) * kBox;
  static constexpr int kKvStages = 3;
  static constexpr uint32_t kK = 0;                       // kKvStages
  static constexpr uint32_t kV = kK + kKvStages * kTile;  // kKvStages
  static constexpr uint32_t kBytes = kV + kKvStages * kTile;
};

struct DqBarriers {
  uint64_t qdo_full;
  uint64_t k_full[3], k_empty[3], v_full[3], v_empty[3];
  uint64_t s_full, s_free, dp_full, p_full, done;
};

// Row `q` of a [tokens, heads, D] bf16 tensor -> this thread's TMEM lane,
// packed pairs; the calling warpgroup stages N (32 or 64) elements starting
// at element col0 into N/2 columns at taddr.
template <int D, int N>
__device__ __forceinline__ void stage_row_to_tmem(const __nv_bfloat16* base, int hq, int head, int q,
                                                  bool valid, int col0, uint32_t taddr) {
  static_assert(N == 16 || N == 32 || N == 64, "staging width");
  uint32_t v[32];
  const uint4* src = reinterpret_cast<const uint4*>(base + (static_cast<size_t>(q) * hq + head) * D + col0);
#pragma unroll
  for (int c = 0; c < N / 8; ++c) {  // N bf16 = N/8 x 16 B
    const uint4 x = valid ? src[c] : make_uint4(0, 0, 0, 0);
    v[4 * c + 0] = x.x;
    v[4 * c + 1] = x.y;
    v[4 * c + 2] = x.z;
    v[4 * c + 3] = x.w;
  }
  if constexpr (N == 64) {
    tmem_st32(taddr, v);
  } else if constexpr (N == 32) {
    tmem_st16(taddr, v);
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
  }
}

// PQ: share of the exponentials on the FMA pipe (pairs out of 8): 0 = 2/8,
// 1 = 3/8 (default, measured best), 2 = 1/8, 3 = 4/8 (A/B knob MAGI_DQ_POLY)
template <int D, bool TR, int PQ = 1>
__global__ void __launch_bounds__(kThreads, 1)
    ffa_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmap_q,
                      const __grid_constant__ CUtensorMap tmap_k,
                      const __grid_constant__ CUtensorMap tmap_v,
                      const __grid_constant__ CUtensorMap tmap_do, const BwdParams p) {
  using L = DqSmem<D>;
  constexpr int S = L::kKvStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ DqBarriers bars;
  __shared__ uint32_t tmem_slot;
  (void)tmap_q;
  (void)tmap_do;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // head-major grid: co-running CTAs stream the same K / V (L2 resident)
  const int tile_rank = blockIdx.x % p.num_q_tiles;
  const int head = blockIdx.x / p.num_q_tiles;
  const int head_k = head / (p.hq / p.hk);
  const FwdTile tile = p.q_tiles[tile_rank];
  const int steps = tile.n_ktiles;
  long long* const trace = static_cast<int>(blockIdx.x) == p.trace_block && p.trace_kernel == 1 ? p.trace : nullptr;

  if (threadIdx.x == 0) {
    mbar_init(&bars.qdo_full, kMath);
    for (int s = 0; s < S; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 1);
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
    }
    mbar_init(&bars.s_full, 1);
    mbar_init(&bars.s_free, kMath);
    mbar_init(&bars.dp_full, 1);
    mbar_init(&bars.p_full, kMath);
    mbar_init(&bars.done, 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dq = tmem + 256;
  const uint32_t t_q = tmem + 384, t_do = tmem + 448;

  uint8_t* sK = smem + L::kK;
  uint8_t* sV = smem + L::kV;

  if (warp == kTmaWarp) {
    if (lane == 0 && steps > 0) {
      tma_prefetch_desc(&tmap_k);
      tma_prefetch_desc(&tmap_v);
      PipeState st;
      for (int it = tile.item_begin; it < tile.item_end; ++it) {
        const FwdItem item = p.q_items[it];
        for (int j = 0; j < item.n_ktiles; ++j) {
          const int k0 = item.k_begin + j * kBlockN;
          mbar_wait(&bars.k_empty[st.index], st.phase ^ 1);
          mbar_arrive_expect_tx(&bars.k_full[st.index], L::kTile);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sK + st.index * L::kTile + c * kBox, &tmap_k, &bars.k_full[st.index],
                        c * 64, head_k, k0);
          mbar_wait(&bars.v_empty[st.index], st.phase ^ 1);
          mbar_arrive_expect_tx(&bars.v_full[st.index], L::kTile);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sV + st.index * L::kTile + c * kBox, &tmap_v, &bars.v_full[st.index],
                        c * 64, head_k, k0);
          st.advance<S>();
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // converged warp; one elected lane issues every MMA / commit
    if (steps > 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_q = make_idesc_bf16(128, D, false, true);
      constexpr uint32_t kStageDesc = L::kTile >> 4;
      const uint64_t k_desc0 = kmajor_desc(sK), v_desc0 = kmajor_desc(sV), k_mn0 = mnmajor_desc(sK);
      // A = Q / dO from TMEM (k-step = 16 head-dim elements = 8 packed columns),
      // B = K / V tile [keys, D] K-major from smem
      auto issue_rows = [&](uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc) {
        if constexpr (D == 128) {
          umma_gemm_ts_bk_k128(d_tmem, a_tmem, b_desc, idesc_s, 0);
        } else {
#pragma unroll
          for (int k = 0; k < D / 16; ++k)
            umma_ts_elect(d_tmem, a_tmem + k * 8, desc_add(b_desc, (k / 4) * kBox + (k % 4) * 32), idesc_s, k > 0);
        }
      };
      TracerT<TR> tr;
      tr.init(trace, 0);  // uniform across the converged warp
      tr.clk(98);
      mbar_wait(&bars.qdo_full, 0);
      PipeState nst, gst;
      mbar_wait(&bars.k_full[nst.index], nst.phase);
      mbar_wait(&bars.v_full[nst.index], nst.phase);
      tc_fence_after();
      issue_rows(t_s, t_q, k_desc0 + nst.index * kStageDesc);
      umma_commit_elect(&bars.s_full);
      issue_rows(t_dp, t_do, v_desc0 + nst.index * kStageDesc);
      umma_commit_elect(&bars.dp_full);
      umma_commit_elect(&bars.v_empty[nst.index]);
      nst.advance<S>();
      for (int t = 0; t < steps; ++t) {
        const bool more = t + 1 < steps;
        if (more) {
          mbar_wait(&bars.s_free, t & 1);
          tr.ev(1, t);
          mbar_wait(&bars.k_full[nst.index], nst.phase);
          mbar_wait(&bars.v_full[nst.index], nst.phase);
          tc_fence_after();
          issue_rows(t_s, t_q, k_desc0 + nst.index * kStageDesc);
          umma_commit_elect(&bars.s_full);
        }
        mbar_wait(&bars.p_full, t & 1);
        tr.ev(2, t);
        tc_fence_after();
        // dQ += dS K : A = dS (TMEM, packed into the dP columns: keys [0,64)
        // at +0, keys [64,128) at +64), B = K [keys, D] MN-major
        umma_gemm_ts_dq_k128(t_dq, t_dp, k_mn0 + gst.index * kStageDesc, idesc_q, t > 0 ? 1u : 0u);
        umma_commit_elect(&bars.k_empty[gst.index]);
        gst.advance<S>();
        if (more) {
          // dP(t+1) overwrites the dS columns read above: in-order pipe
          issue_rows(t_dp, t_do, v_desc0 + nst.index * kStageDesc);
          umma_commit_elect(&bars.dp_full);
          umma_commit_elect(&bars.v_empty[nst.index]);
          nst.advance<S>();
          tr.ev(3, t);
        } else {
          umma_commit_elect(&bars.done);
        }
      }
      tr.clk(99);
    }
  } else {
    // two warpgroups split the 128 key columns: wg 0 [0, 64), wg 1 [64, 128)
    const int wg = warp / 4;
    const int col0 = wg * 64;
    const int row = (warp % 4) * 32 + lane;
    const int q = tile.q0 + row;
    const uint32_t lane_off = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const bool valid = q < p.seqlen_q;
    const float sl2 = p.scale_log2;
    if (steps > 0) {
      // stage Q and dO rows into TMEM (each warpgroup half of the head dim)
      stage_row_to_tmem<D, D / 2>(static_cast<const __nv_bfloat16*>(p.q), p.hq, head, q, valid,
                           wg * (D / 2), t_q + lane_off + wg * (D / 4));
      stage_row_to_tmem<D, D / 2>(static_cast<const __nv_bfloat16*>(p.dout), p.hq, head, q, valid,
                           wg * (D / 2), t_do + lane_off + wg * (D / 4));
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars.qdo_full);
    }
    TracerT<TR> tr;
    if (warp % 4 == 0) tr.init(trace, 1 + wg);
    float lse_l2 = INFINITY, dlt = 0.f;
    if (valid) {
      const float raw = p.lse[static_cast<size_t>(head) * p.seqlen_q + q];
      lse_l2 = raw == -INFINITY ? INFINITY : raw * kLog2e;
      dlt = p.delta[static_cast<size_t>(head) * p.seqlen_q + q];
    }
    int t = 0;
    for (int it = tile.item_begin; it < tile.item_end; ++it) {
      const FwdItem item = p.q_items[it];
      int32_t lo, hi;
      row_bounds(item.qs, item.qe, item.ks, item.ke, item.type, q, lo, hi);
      for (int j = 0; j < item.n_ktiles; ++j, ++t) {
        const int k0 = item.k_begin + j * kBlockN;
        mbar_wait(&bars.s_full, t & 1);
        tr.ev(10, t);
        tc_fence_after();
        float pv[64];
        {
          const int kb = k0 + col0;
          const bool all_in = lo <= kb && kb + 64 <= hi;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t s[32];
            tmem_ld32(t_s + lane_off + col0 + h2 * 32, s);
            tmem_ld_wait();
            if (h2 == 1) {
              tc_fence_before();
              mbar_arrive(&bars.s_free);
            }
            {
              // x = s * scale * log2e - lse * log2e, two lanes per FFMA2; part
              // of the exponentials on the FMA pipe
              const uint64_t sc2 = f2(sl2, sl2), nl2 = f2(-lse_l2, -lse_l2);
#pragma unroll
              for (int c = 0; c < 32; c += 2) {
                const float2 x = f2_split(ffma2(f2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), sc2, nl2));
                constexpr uint32_t kPolyMask = PQ == 0 ? 0x88u : (PQ == 1 ? 0x92u : (PQ == 2 ? 0x80u : 0xAAu));
                if ((kPolyMask >> ((c / 2) % 8)) & 1u) {
                  const float2 e = exp2_poly2(x.x, x.y);
                  pv[h2 * 32 + c] = e.x;
                  pv[h2 * 32 + c + 1] = e.y;
                } else {
                  pv[h2 * 32 + c] = fast_exp2(x.x);
                  pv[h2 * 32 + c + 1] = fast_exp2(x.y);
                }
              }
            }
            if (!all_in) {
              // masked keys (and every key of an empty row) selected to exact zeros
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                const int kk = kb + h2 * 32 + c;
                pv[h2 * 32 + c] = (kk >= lo && kk < hi) ? pv[h2 * 32 + c] : 0.f;
              }
            }
          }
        }
        tr.ev(11, t);
        mbar_wait(&bars.dp_full, t & 1);
        tr.ev(12, t);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t dp[32], ds[16];
          tmem_ld32(t_dp + lane_off + col0 + c * 32, dp);
          tmem_ld_wait();
          const uint64_t nd2 = f2(-dlt, -dlt);
#pragma unroll
          for (int j2 = 0; j2 < 32; j2 += 2) {
            const int col = c * 32 + j2;
            // dS = P (dP - delta): FADD2 + FMUL2 per pair
            const float2 d = f2_split(fmul2(f2(pv[col], pv[col + 1]),
                                            fadd2(f2(__uint_as_float(dp[j2]), __uint_as_float(dp[j2 + 1])), nd2)));
            ds[j2 / 2] = pack_bf16(d.x, d.y);
          }
          // dS chunk -> this warpgroup's consumed dP columns [col0 + c*16, +16)
          tmem_st16(t_dp + lane_off + col0 + c * 16, ds);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars.p_full);
        tr.ev(13, t);
      }
    }
    if (steps > 0) {
      mbar_wait(&bars.done, 0);
      tc_fence_after();
    }
    // each warpgroup writes half of the dQ row
    const size_t row_off = (static_cast<size_t>(q) * p.hq + head) * D + wg * (D / 2);
    epilogue_rows<D / 2>(t_dq + lane_off + wg * (D / 2), steps > 0, valid, p.dq, row_off, p.scale,
                         p.grad_f32 != 0, p.accumulate != 0);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D>
cudaError_t launch_bwd_impl(const BwdParams& prm, int num_q_tiles, int num_k_tiles,
                            const void* q, const void* k, const void* v, const void* dout,
                            int parts, cudaStream_t stream) {
  const CUtensorMap tq = make_tmap_thd(q, prm.seqlen_q, prm.hq, D, 128);
  const CUtensorMap tdo = make_tmap_thd(dout, prm.seqlen_q, prm.hq, D, 128);
  const CUtensorMap tk = make_tmap_thd(k, prm.seqlen_k, prm.hk, D, 128);
  const CUtensorMap tv = make_tmap_thd(v, prm.seqlen_k, prm.hk, D, 128);
  cudaError_t err = cudaSuccess;
  if ((parts & 1) && num_k_tiles > 0) {
    const int smem = DkvSmem<D>::kBytes;  // 1024-aligned dynamic window, barriers inside
    // 37.5% of the exponentials on the FMA pipe, four elementwise warpgroups
    auto kern = ffa_bwd_dkdv_kernel<D, 1, false, 4>;
#ifdef MAGI_TRACE
    if (prm.trace != nullptr && prm.trace_kernel == 0) kern = ffa_bwd_dkdv_kernel<D, 1, true, 4>;
#endif
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    BwdParams pk = prm;
    pk.lse_tma = (prm.seqlen_q % 4) == 0;
    CUtensorMap tl{}, td{};
    if (pk.lse_tma) {
      tl = make_tmap_f32_rows(prm.lse, static_cast<uint64_t>(prm.hq), static_cast<uint64_t>(prm.seqlen_q), 128);
      td = make_tmap_f32_rows(prm.delta, static_cast<uint64_t>(prm.hq), static_cast<uint64_t>(prm.seqlen_q), 128);
    }
    kern<<<dim3(num_k_tiles * prm.hk), DkvLayout<4>::kThreads, smem, stream>>>(tq, tk, tv, tdo, tl, td, pk);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  if ((parts & 2) && num_q_tiles > 0) {
    const int smem = DqSmem<D>::kBytes + 1024;
    auto dq_kern = ffa_bwd_dq_kernel<D, false, 1>;  // 37.5% of the exponentials on the FMA pipe
#ifdef MAGI_TRACE
    if (prm.trace != nullptr && prm.trace_kernel == 1) dq_kern = ffa_bwd_dq_kernel<D, true, 1>;
#endif
    err = cudaFuncSetAttribute(dq_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    dq_kern<<<dim3(num_q_tiles * prm.hq), kThreads, smem, stream>>>(tq, tk, tv, tdo, prm);
    err = cudaGetLastError();
  }
  return err;
}

}  // namespace

cudaError_t launch_ffa_bwd(const FwdTile* q_tiles, const FwdItem* q_items, int num_q_tiles,
                           const BwdTile* k_tiles, const BwdItem* k_items, int num_k_tiles,
                           int seqlen_q, int seqlen_k, int hq, int hk, int head_dim,
                           float softmax_scale, const void* q, const void* k, const void* v,
                           const float* lse, const float* delta, const void* grad_out,
                           void* grad_q, void* grad_k, void* grad_v, int grad_f32,
                           int accumulate, int parts, cudaStream_t stream) {
  BwdParams prm;
  prm.q_tiles = q_tiles;
  prm.q_items = q_items;
  prm.k_tiles = k_tiles;
  prm.k_items = k_items;
  prm.seqlen_q = seqlen_q;
  prm.seqlen_k = seqlen_k;
  prm.hq = hq;
  prm.hk = hk;
  prm.scale = softmax_scale;
  prm.scale_log2 = softmax_scale * kLog2e;
  prm.lse = lse;
  prm.delta = delta;
  prm.dq = grad_q;
  prm.dk = grad_k;
  prm.dv = grad_v;
  prm.q = q;
  prm.num_k_tiles = num_k_tiles;
  prm.num_q_tiles = num_q_tiles;
  prm.trace = g_trace;
  prm.trace_block = g_trace_block;
  prm.trace_kernel = g_trace_kernel;
  prm.dout = grad_out;
  prm.grad_f32 = grad_f32;
  prm.accumulate = accumulate;
  if (head_dim == 128) return launch_bwd_impl<128>(prm, num_q_tiles, num_k_tiles, q, k, v, grad_out, parts, stream);
  if (head_dim == 64) return launch_bwd_impl<64>(prm, num_q_tiles, num_k_tiles, q, k, v, grad_out, parts, stream);
  return cudaErrorInvalidValue;
}

}  // namespace magi

namespace magi {
// Diagnostics: route one backward CTA's event log to a device buffer
// (int64: [0] unused, then per-role {event << 32 | step, ns} regions); nullptr = off.
void set_bwd_trace(long long* buffer, int block) {
  g_trace = buffer;
  g_trace_block = block < 0 ? -block - 1 : block;
  g_trace_kernel = block < 0 ? 1 : 0;  // a negative block index selects the dQ kernel
}
}  // namespace magi
