// FFA forward for sm_100a: flexible (slice-list) masked attention, O and LSE.
//
// One CTA owns a 256-row query tile of one query head, split in two 128-row
// sub-tiles that share every K/V tile (halving L2 -> SM traffic per FLOP),
// and walks every (tile, slice) work item the host planner produced for it.
// Overlapping slices are merged inside the CTA (MULTIPLICITY semantics,
// reference proj/include/magiplan/mask.hpp:85): no atomics.
//
// Warp roles (384 threads):
//   warps 0-3 / 4-7  softmax of sub-tile 0 / 1, thread = one full 128-column
//                    query row = TMEM lane (no cross-warp max exchange): apply
//                    the slice row bounds, online softmax with a lazily moved
//                    max (rescale O only when the row max grows by > 2^8),
//                    exp2 split between MUFU and an FFMA2 polynomial, P back
//                    into the S columns as packed bf16 (tcgen05.st). setmaxnreg
//                    gives these warps 200 registers.
//   warp 8           TMA producer: Q once, K/V through a 2-stage ring.
//   warp 9           MMA issuer (converged warp, one elected lane). Per key
//                    tile t:
//                      S0 = Q0 K^T, S1 = Q1 K^T           (SS, M=128 N=128)
//                      O0 += P0 V, then S0' = Q0 K'^T      (P from TMEM: TS)
//                      O1 += P1 V, then S1' = Q1 K'^T
//                    so softmax of one sub-tile overlaps the MMAs of the other.
//   warps 10-11      idle (complete the control warpgroup for setmaxnreg:
//                    2 x 200 + 96 <= 3 x 168 registers per SM sub-partition).
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
// Issue order guarantees: S_i(t+1) is issued after O_i += P_i(t) V, so when a
// softmax thread sees S_i(t+1) complete, P_i(t)'s MMA has retired and O_i is
// quiescent until it arrives on p_full — the O rescale needs no extra wait.
#include <cuda_runtime.h>

#include <cmath>

#include "ffa_common.cuh"
#include "sm100.cuh"
#include "tma_host.h"

namespace magi {
namespace {

constexpr int kStages = 2;
constexpr uint32_t kBox = 128 * 64 * 2;  // one TMA box: 128 rows x 64 bf16 (128B swizzle)
constexpr int kSub = 128;                // rows per sub-tile
constexpr int kThreads = 384;
constexpr int kTmaWarp = 8;
constexpr int kMmaWarp = 9;
constexpr uint32_t kSoftRegs = 200;
constexpr uint32_t kCtrlRegs = 96;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P <= 256 between rescales
// exp2 pairs (i/2 % 8) computed on the FMA pipe: {3, 7} = 25% (measured best
// against MUFU-only and 12.5 / 37.5 % on config 2)
constexpr uint32_t kPolyMask = 0x88u;

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
  long long* trace;  // diagnostics: per-role event log of one CTA (MAGI_TRACE builds)
  int32_t trace_block;
};

long long* g_fwd_trace = nullptr;
int g_fwd_trace_block = 0;

template <int D>
struct FwdSmem {
  static constexpr uint32_t kTileBytes = (D / 64) * kBox;
  static constexpr uint32_t kQ = 0;  // 2 sub-tiles
  static constexpr uint32_t kK = kQ + 2 * kTileBytes;
  static constexpr uint32_t kV = kK + kStages * kTileBytes;
  static constexpr uint32_t kBytes = kV + kStages * kTileBytes;
};

struct FwdBarriers {
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], p_full[2], o_final[2];
};

// S = Q K^T (SS, both K-major): descriptors of the two tiles' first k-step;
// a k-step is 32 B inside a 64-column box, boxes are kBox apart.
template <int D>
__device__ __forceinline__ void issue_qk(uint32_t tmem_s, uint64_t q_desc, uint64_t k_desc) {
  constexpr uint32_t idesc = make_idesc_bf16(128, 128, false, false);
  if constexpr (D == 128) {
    umma_gemm_ss_k128(tmem_s, q_desc, k_desc, idesc, 0);
  } else {
#pragma unroll
    for (int k = 0; k < D / 16; ++k) {
      const uint32_t off = (k / 4) * kBox + (k % 4) * 32;
      umma_ss_elect(tmem_s, desc_add(q_desc, off), desc_add(k_desc, off), idesc, k > 0);
    }
  }
}

// O += P V (TS): P packed bf16 in the first 64 S columns, V [keys, D]
// MN-major (a k-step is 16 key rows, 2 KB).
template <int D>
__device__ __forceinline__ void issue_pv(uint32_t tmem_o, uint32_t tmem_p, uint64_t v_desc, bool accumulate) {
  constexpr uint32_t idesc = make_idesc_bf16(128, D, false, true);
  umma_gemm_ts_k128(tmem_o, tmem_p, v_desc, idesc, accumulate ? 1u : 0u);
}

// One softmax phase: this thread's full 128-column row of one sub-tile for
// key tile t (global keys from kc), against the row's running (m, l).
template <int D, class TRC>
__device__ __forceinline__ void softmax_phase(float& m, float& l, uint32_t t_s, uint32_t t_o, int kc, int lo,
                                              int hi, int t, float sl2, uint64_t* s_full, uint64_t* p_full,
                                              TRC& tr, int tkey) {
  mbar_wait(s_full, t & 1);
  tr.ev(10, tkey);
  tc_fence_after();
  uint32_t s[128];
#pragma unroll
  for (int c = 0; c < 4; ++c) tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
  tmem_ld_wait();
  tr.ev(14, tkey);
  const bool full = lo <= kc && kc + 128 <= hi;
  if (!full) {
#pragma unroll
    for (int i = 0; i < 128; ++i) {
      const int c = kc + i;
      if (c < lo || c >= hi) s[i] = __float_as_uint(-INFINITY);
    }
  }
  // row max as 4 independent 3-input-max chains
  float mx[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) mx[u] = fmaxf(__uint_as_float(s[2 * u]), __uint_as_float(s[2 * u + 1]));
#pragma unroll
  for (int i = 8; i < 128; i += 8) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      mx[u] = fmaxf(mx[u], fmaxf(__uint_as_float(s[i + 2 * u]), __uint_as_float(s[i + 2 * u + 1])));
  }
  const float mt2 = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * sl2;
  tr.ev(11, tkey);
  const bool move = mt2 > m + kRescaleThreshold;  // also true on the first finite tile
  const float alpha = move ? fast_exp2(m - mt2) : 1.f;
  if (move) m = mt2;
  const float mb = m == -INFINITY ? 0.f : m;
  // O rescale (rare: the row max grew by more than 2^8) before the
  // exponentials, so they and the P stores form one straight-line block; O
  // is quiescent here (S(t) done implies P(t-1) V done) and the MMA reads it
  // only after p_full
  if (t > 0 && __any_sync(0xffffffffu, move)) {
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      tmem_ld32(t_o + c * 32, o);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
      tmem_st32(t_o + c * 32, o);
    }
  }
  uint32_t pk[64];
  // packed f32x2: x = s * scale - m two lanes per FFMA2, sums by FADD2
  const uint64_t sc2 = f2(sl2, sl2), nm2 = f2(-mb, -mb);
  uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
  if (full) {
#pragma unroll
    for (int i = 0; i < 128; i += 2) {
      const int jj = i / 2;
      const float2 x = f2_split(ffma2(f2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sc2, nm2));
      float p0, p1;
      if ((kPolyMask >> (jj % 8)) & 1u) {
        const float2 e = exp2_poly2(x.x, x.y);
        p0 = e.x;
        p1 = e.y;
      } else {
        p0 = fast_exp2(x.x);
        p1 = fast_exp2(x.y);
      }
      acc2[jj % 4] = fadd2(acc2[jj % 4], f2(p0, p1));
      pk[jj] = pack_bf16(p0, p1);
    }
  } else {
    // masked scores are -inf: all exponentials on MUFU (exact zeros)
#pragma unroll
    for (int i = 0; i < 128; i += 2) {
      const float2 x = f2_split(ffma2(f2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sc2, nm2));
      const float p0 = fast_exp2(x.x), p1 = fast_exp2(x.y);
      acc2[(i / 2) % 4] = fadd2(acc2[(i / 2) % 4], f2(p0, p1));
      pk[i / 2] = pack_bf16(p0, p1);
    }
  }
  const float2 a2 = f2_split(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])));
  l = l * alpha + (a2.x + a2.y);
  tr.ev(12, tkey);
  // P (bf16 pairs) into the first 64 of this sub-tile's (consumed) S columns
  tmem_st32(t_s, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
  tmem_st32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
  tmem_st_wait();
  tc_fence_before();
  mbar_arrive(p_full);
  tr.ev(13, tkey);
}

// Output of one row: normalise (or merge into an existing (out, lse) pair)
// and store.
template <int D>
__device__ __forceinline__ void softmax_store(const FwdParams& p, int head, int q, float m, float lt,
                                              uint32_t t_o, bool has_work, uint64_t* o_final) {
  const bool valid = q < p.seqlen_q;
  float* lse_ptr = p.lse + static_cast<size_t>(head) * p.seqlen_q + q;
  const float lse_old = (p.accumulate && valid) ? *lse_ptr : -INFINITY;
  const bool has = lt > 0.f;
  const float lse_cur = has ? (m * kLn2 + logf(lt)) : -INFINITY;
  const float inv_l = has ? 1.f / lt : 0.f;
  if (has_work) {
    mbar_wait(o_final, 0);
    tc_fence_after();
  }
  const size_t row_off = (static_cast<size_t>(q) * p.hq + head) * D;
  if (p.accumulate) {
    // merge into (out, lse) with the log-sum-exp correction; f32 output
    const float lse_new = has ? (lse_old > lse_cur ? lse_old + log1pf(__expf(lse_cur - lse_old))
                                                   : lse_cur + log1pf(__expf(lse_old - lse_cur)))
                              : lse_old;
    const float w_old = has ? __expf(lse_old - lse_new) : 1.f;
    const float w_cur = has ? __expf(lse_cur - lse_new) * inv_l : 0.f;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      if (has_work) {
        tmem_ld32(t_o + c * 32, o);
        tmem_ld_wait();
      }
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
      if (has_work) {
        tmem_ld32(t_o + c * 32, o);
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

template <int D, bool TR>
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
  // head-major grid: co-running CTAs stream the same K / V (L2 resident)
  const int tile_rank = blockIdx.x % p.num_tiles;
  const int head = blockIdx.x / p.num_tiles;
  const int head_k = head / (p.hq / p.hk);
  const FwdTile tile = p.tiles[tile_rank];
  const int n_total = tile.n_ktiles;
  // merging nothing into (out, lse) is a no-op: a CP stage's rows without
  // received keys cost one empty CTA
  if (p.accumulate && n_total == 0) return;
  long long* const trace = TR && static_cast<int>(blockIdx.x) == p.trace_block ? p.trace : nullptr;

  if (threadIdx.x == 0) {
    mbar_init(&bars.q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 1);
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.s_full[i], 1);
      mbar_init(&bars.p_full[i], kSub);
      mbar_init(&bars.o_final[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(&tmem_base_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_slot;

  uint8_t* sQ = smem + L::kQ;
  uint8_t* sK = smem + L::kK;
  uint8_t* sV = smem + L::kV;

  if (warp >= kTmaWarp) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kCtrlRegs));
  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && n_total > 0) {
      TracerT<TR> tr;
      tr.init(trace, 3);
      int tt = 0;
      tma_prefetch_desc(&tmap_q);
      tma_prefetch_desc(&tmap_k);
      tma_prefetch_desc(&tmap_v);
      mbar_arrive_expect_tx(&bars.q_full, 2 * L::kTileBytes);
      for (int i = 0; i < 2; ++i)
        for (int c = 0; c < D / 64; ++c)
          tma_load_3d(sQ + i * L::kTileBytes + c * kBox, &tmap_q, &bars.q_full, c * 64, head,
                      tile.q0 + i * kSub);
      PipeState st;
      for (int it = tile.item_begin; it < tile.item_end; ++it) {
        const FwdItem item = p.items[it];
        for (int j = 0; j < item.n_ktiles; ++j) {
          const int k0 = item.k_begin + j * kBlockN;
          mbar_wait(&bars.k_empty[st.index], st.phase ^ 1);
          tr.ev(30, tt);
          mbar_arrive_expect_tx(&bars.k_full[st.index], L::kTileBytes);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sK + st.index * L::kTileBytes + c * kBox, &tmap_k, &bars.k_full[st.index],
                        c * 64, head_k, k0);
          mbar_wait(&bars.v_empty[st.index], st.phase ^ 1);
          tr.ev(31, tt++);
          mbar_arrive_expect_tx(&bars.v_full[st.index], L::kTileBytes);
          for (int c = 0; c < D / 64; ++c)
            tma_load_3d(sV + st.index * L::kTileBytes + c * kBox, &tmap_v, &bars.v_full[st.index],
                        c * 64, head_k, k0);
          st.advance<kStages>();
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // the whole warp runs this loop (converged); one elected lane issues
    if (n_total > 0) {
      const uint64_t q_desc0 = make_smem_desc(smem_u32(sQ), 16, 1024);
      const uint64_t q_desc1 = make_smem_desc(smem_u32(sQ + L::kTileBytes), 16, 1024);
      const uint64_t k_desc0 = make_smem_desc(smem_u32(sK), 16, 1024);
      const uint64_t v_desc0 = make_smem_desc(smem_u32(sV), kBox, 1024);
      constexpr uint32_t kStageDesc = L::kTileBytes >> 4;  // stage stride in descriptor units
      TracerT<TR> tr;
      tr.init(trace, 0);  // uniform across the converged warp
      tr.clk(98);
      mbar_wait(&bars.q_full, 0);
      PipeState kst, vst;
      mbar_wait(&bars.k_full[kst.index], kst.phase);
      tc_fence_after();
      {
        const uint64_t k_desc = k_desc0 + kst.index * kStageDesc;
        issue_qk<D>(tmem + 0, q_desc0, k_desc);
        umma_commit_elect(&bars.s_full[0]);
        issue_qk<D>(tmem + 128, q_desc1, k_desc);
        umma_commit_elect(&bars.s_full[1]);
        umma_commit_elect(&bars.k_empty[kst.index]);
        kst.advance<kStages>();
      }
      for (int t = 0; t < n_total; ++t) {
        const bool more = t + 1 < n_total;
        const uint64_t v_desc = v_desc0 + vst.index * kStageDesc;
        // sub-tile 0: O0 += P0 V, then S0 for the next key tile
        mbar_wait(&bars.p_full[0], t & 1);
        tr.ev(1, t);
        mbar_wait(&bars.v_full[vst.index], vst.phase);
        tr.ev(2, t);
        tc_fence_after();
        issue_pv<D>(tmem + 256, tmem + 0, v_desc, t > 0);
        if (!more) umma_commit_elect(&bars.o_final[0]);
        const uint64_t k_desc = k_desc0 + kst.index * kStageDesc;
        if (more) {
          mbar_wait(&bars.k_full[kst.index], kst.phase);
          tr.ev(3, t);
          tc_fence_after();
          issue_qk<D>(tmem + 0, q_desc0, k_desc);
          umma_commit_elect(&bars.s_full[0]);
        }
        // sub-tile 1
        mbar_wait(&bars.p_full[1], t & 1);
        tr.ev(4, t);
        tc_fence_after();
        issue_pv<D>(tmem + 384, tmem + 128, v_desc, t > 0);
        umma_commit_elect(&bars.v_empty[vst.index]);
        vst.advance<kStages>();
        if (!more) umma_commit_elect(&bars.o_final[1]);
        if (more) {
          issue_qk<D>(tmem + 128, q_desc1, k_desc);
          umma_commit_elect(&bars.s_full[1]);
          umma_commit_elect(&bars.k_empty[kst.index]);
          kst.advance<kStages>();
        }
      }
      tr.clk(99);
    }
  } else if (warp < kTmaWarp) {
    // ------------------------------------------------------------ softmax
    // thread = query row = TMEM lane of sub-tile warp / 4
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoftRegs));
    const int sub = warp / 4;
    const int row = (warp % 4) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t t_s = tmem + sub * 128 + lane_off, t_o = tmem + 256 + sub * 128 + lane_off;
    const float sl2 = p.scale_log2;
    float m = -INFINITY;  // exponent base, log2 domain (lazily moved)
    float l = 0.f;        // sum of 2^(x - m)
    const int q = tile.q0 + sub * kSub + row;
    TracerT<TR> tr;
    if (warp % 4 == 0) tr.init(trace, 1 + sub);
    int t = 0;
    for (int it = tile.item_begin; it < tile.item_end; ++it) {
      const FwdItem item = p.items[it];
      int32_t lo, hi;
      row_bounds(item.qs, item.qe, item.ks, item.ke, item.type, q, lo, hi);
      for (int j = 0; j < item.n_ktiles; ++j, ++t) {
        const int kc = item.k_begin + j * kBlockN;
        softmax_phase<D>(m, l, t_s, t_o, kc, lo, hi, t, sl2, &bars.s_full[sub], &bars.p_full[sub], tr, t);
      }
    }
    // ---------------------------------------------------------- epilogue
    softmax_store<D>(p, head, q, m, l, t_o, n_total > 0, &bars.o_final[sub]);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
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
  auto kern = ffa_fwd_kernel<D, false>;
#ifdef MAGI_TRACE
  if (prm.trace != nullptr) kern = ffa_fwd_kernel<D, true>;  // diagnostics build only
#endif
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return err;
  const dim3 grid(static_cast<unsigned>(prm.num_tiles) * prm.hq);
  kern<<<grid, kThreads, smem, stream>>>(tq, tk, tv, prm);
  return cudaGetLastError();
}

}  // namespace

// work: the plan's q-major work lists; this layout tiles by 256 rows (fwd2_*).
cudaError_t launch_ffa_fwd(const FwdWork& work,
                           int seqlen_q, int seqlen_k, int hq, int hk, int head_dim,
                           float softmax_scale, const void* q, const void* k, const void* v,
                           void* out, float* lse, int out_f32, int accumulate,
                           cudaStream_t stream) {
  if (work.num_tiles256 == 0 || hq == 0) return cudaSuccess;
  FwdParams prm;
  prm.tiles = work.tiles256;
  prm.items = work.items256;
  prm.num_tiles = work.num_tiles256;
  prm.seqlen_q = seqlen_q;
  prm.seqlen_k = seqlen_k;
  prm.hq = hq;
  prm.hk = hk;
  prm.scale_log2 = softmax_scale * kLog2e;
  prm.out = out;
  prm.lse = lse;
  prm.out_f32 = out_f32;
  prm.accumulate = accumulate;
  prm.trace = g_fwd_trace;
  prm.trace_block = g_fwd_trace_block;
  if (head_dim == 128) return launch_fwd_impl<128>(prm, q, k, v, stream);
  if (head_dim == 64) return launch_fwd_impl<64>(prm, q, k, v, stream);
  return cudaErrorInvalidValue;
}

// Diagnostics: route one forward CTA's per-role event log to a device buffer.
void set_fwd_trace(long long* buffer, int block) {
  g_fwd_trace = buffer;
  g_fwd_trace_block = block;
}

}  // namespace magi
