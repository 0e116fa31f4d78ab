// FFA forward for sm_100a: flexible (slice-list) masked attention, O and LSE.
//
// One CTA owns a 256-row query tile of one query head, split in two 128-row
// sub-tiles that share every K/V tile (halving L2 -> SM traffic per FLOP),
// and walks every (tile, slice) work item the host planner produced for it.
// Overlapping slices are merged inside the CTA (MULTIPLICITY semantics,
// reference proj/include/magiplan/mask.hpp:85): no atomics.
//
// Warp roles (default layout 5, 384 threads; the alternatives below are kept
// for A/B runs):
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
//   warps 10-11      idle (complete the control warpgroup for setmaxnreg).
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
// Issue order guarantees: S_i(t+1) is issued after O_i += P_i(t) V, so when a
// softmax thread sees S_i(t+1) complete, P_i(t)'s MMA has retired and O_i is
// quiescent until it arrives on p_full — the O rescale needs no extra wait.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "ffa_common.cuh"
#include "sm100.cuh"
#include "tma_host.h"

namespace magi {
namespace {

constexpr int kStages = 2;
constexpr uint32_t kBox = 128 * 64 * 2;  // one TMA box: 128 rows x 64 bf16 (128B swizzle)
constexpr int kSub = 128;                // rows per sub-tile
// Warp layouts (template LAYOUT). A sub-tile's 128 score columns are split
// into NP parts, one softmax warpgroup each (thread = query row):
//   0: 320 threads, NP = 2: two warpgroups walk both sub-tiles one after the
//      other; warp 8 TMA, warp 9 MMA.
//   1: 640 threads, NP = 2: four warpgroups (sub-tile x half), the two
//      sub-tiles' phases overlap; control warpgroup = TMA warp 16, MMA warp 17,
//      load observer 18, idle 19; setmaxnreg split of the 96 registers per
//      thread granted at launch: per SM sub-partition 4 softmax warps x 104 +
//      1 control warp x 56 <= 5 x 96.
//   2: 576 threads, NP = 4: four warpgroups (32 columns each) walk both
//      sub-tiles one after the other; warp 16 TMA, warp 17 MMA.
//   4: 320 threads, NP = 1: one warpgroup per sub-tile, thread = a full
//      128-column row (no max exchange), the two sub-tiles ping-pong;
//      warp 8 TMA, warp 9 MMA.
//   5: as 4 with a control warpgroup (warps 8-11: TMA, MMA, 2 idle) so
//      setmaxnreg can give the softmax warps 200 registers (2 x 200 + 96 <=
//      3 x 168 per SM sub-partition).
constexpr uint32_t kSoftmaxRegs = 104;  // layout 1
constexpr uint32_t kControlRegs = 56;
template <int LAYOUT>
struct FwdLayout {
  static constexpr bool kFull5 = LAYOUT == 5 || LAYOUT == 6 || LAYOUT == 7;  // layout 5 family
  static constexpr bool kL1 = LAYOUT == 1 || LAYOUT == 8;                    // layout 1 family
  static constexpr bool kPair = kL1 || LAYOUT == 4 || kFull5;
  static constexpr bool kSetmaxnreg = kL1 || kFull5;
  static constexpr bool kSplitP = LAYOUT == 6;  // layout 5 + P handed to the MMA in two key halves
  static constexpr bool kToken = LAYOUT == 7;   // layout 5 + exponential loops of the two sub-tiles never overlap
  static constexpr bool kSpec = LAYOUT == 8;    // layout 1 + exponentials before the row-max exchange
  static constexpr uint32_t kSoftRegs = kFull5 ? 200 : kSoftmaxRegs;
  static constexpr uint32_t kCtrlRegs = kFull5 ? 96 : kControlRegs;
  static constexpr int kParts = LAYOUT == 2 ? 4 : ((LAYOUT == 4 || kFull5) ? 1 : 2);
  static constexpr int kThreads =
      (LAYOUT == 0 || LAYOUT == 4) ? 320 : (kL1 ? 640 : (kFull5 ? 384 : 576));
  static constexpr int kTmaWarp = (LAYOUT == 0 || LAYOUT == 4 || kFull5) ? 8 : 16;
  static constexpr int kMmaWarp = kTmaWarp + 1;
};
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P <= 256 between rescales

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
  long long* trace;  // diagnostics: per-role event log of one CTA (nullptr = off)
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
  // row-max exchange [2 step parities][2 sub][4 parts][128] f32, then the
  // row-sum exchange [2 sub][4 parts][128]
  static constexpr uint32_t kXch = kV + kStages * kTileBytes;
  static constexpr uint32_t kXl = 16 * kSub;  // float offset of the row-sum exchange
  static constexpr uint32_t kBytes = kXch + 24 * kSub * 4;
};

struct FwdBarriers {
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], p_full[2], o_final[2];
  uint64_t p_first[2];  // split P hand-off: keys [0,64) of P stored (layout 6)
  uint64_t tok[2];      // layout 7: sub-tile i finished the exponentials of a phase
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

// O += P V (TS): P packed bf16 in TMEM, V [keys, D] MN-major (a k-step is
// 16 key rows, 2 KB). Each softmax part writes its keys' P into the first
// columns of its own S columns: NP = 2 -> keys [0,64) at +0, [64,128) at +64;
// NP = 4 -> keys [32w, 32w+32) at +32w.
template <int D, int NP>
__device__ __forceinline__ void issue_pv(uint32_t tmem_o, uint32_t tmem_p, uint64_t v_desc, bool accumulate) {
  constexpr uint32_t idesc = make_idesc_bf16(128, D, false, true);
  if constexpr (NP == 1) {
    umma_gemm_ts_k128(tmem_o, tmem_p, v_desc, idesc, accumulate ? 1u : 0u);
  } else if constexpr (NP == 2) {
    umma_gemm_ts_dq_k128(tmem_o, tmem_p, v_desc, idesc, accumulate ? 1u : 0u);
  } else {
    umma_gemm_ts_dkdv_k128(tmem_o, tmem_p, v_desc, idesc, accumulate ? 1u : 0u);
  }
}


// One softmax phase: this thread's row of one sub-tile, score columns
// [c0, c0 + CW) (CW = 128 / NP, part `part`) of key tile t (global keys from
// kc), against the row's running (m, l). The NP parts exchange partial maxima
// through the shared-memory slots at xslot and a named barrier.
template <int D, int V, int NP, class TRC, bool SPLITP = false, bool TOK = false, bool SPEC = false>
__device__ __forceinline__ void softmax_phase(float& m, float& l, uint32_t t_s, uint32_t t_o, int part,
                                              int kc, int lo, int hi, int t, uint32_t xslot,
                                              uint32_t bar_id, float sl2, uint64_t* s_full,
                                              uint64_t* p_full, TRC& tr, int tkey,
                                              uint64_t* p_first = nullptr, uint64_t* tok_wait = nullptr,
                                              int tok_parity = -1, uint64_t* tok_arrive = nullptr) {
  constexpr int CW = 128 / NP;
  constexpr int OW = D / NP;  // output columns of this part (O rescale)
  const int c0 = part * CW;
  const int oc0 = part * OW;
  mbar_wait(s_full, t & 1);
  tr.ev(10, tkey);
  tc_fence_after();
  uint32_t s[CW];
#pragma unroll
  for (int c = 0; c < CW / 32; ++c) tmem_ld32(t_s + c0 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
  tmem_ld_wait();
  tr.ev(14, tkey);
  const bool full = lo <= kc && kc + CW <= hi;
  if (!full) {
#pragma unroll
    for (int i = 0; i < CW; ++i) {
      const int c = kc + i;
      if (c < lo || c >= hi) s[i] = __float_as_uint(-INFINITY);
    }
  }
  if constexpr (SPEC) {
    // Speculative phase (layout 8): with no masked column and a finite
    // running max, the exponentials are taken against the current m while the
    // partial row max is reduced alongside; the parts exchange their maxima
    // only afterwards. When no row of the warp moves its max, these are the
    // values the exact phase below would produce (alpha = 1, same m); the two
    // parts of a row reach the same verdict from the same maxima. Otherwise S
    // is reloaded from TMEM (P is not stored yet) and both parts redo the
    // tile exactly.
    static_assert(NP == 2 && !SPLITP, "speculation is written for the two-part layout");
    if (__all_sync(0xffffffffu, full && m != -INFINITY)) {
      const uint64_t sc2 = f2(sl2, sl2), nm2 = f2(-m, -m);
      uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      uint32_t pk[CW / 2];
#pragma unroll
      for (int i = 0; i < CW; i += 2) {
        const int jj = i / 2;
        const float s0 = __uint_as_float(s[i]), s1 = __uint_as_float(s[i + 1]);
        mx[jj % 4] = fmaxf(mx[jj % 4], fmaxf(s0, s1));
        const float2 x = f2_split(ffma2(f2(s0, s1), sc2, nm2));
        constexpr uint32_t kPolyMask = V == 0 ? 0x88u : (V == 1 ? 0x92u : 0x80u);
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
      float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot + part * kSub * 4), "f"(mt) : "memory");
      named_bar_sync(bar_id, NP * 128);
#pragma unroll
      for (int o = 1; o < NP; ++o) {
        float po;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(po) : "r"(xslot + ((part + o) % NP) * kSub * 4) : "memory");
        mt = fmaxf(mt, po);
      }
      if (!__any_sync(0xffffffffu, mt * sl2 > m + kRescaleThreshold)) {
        const float2 a2 = f2_split(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])));
        l = l + (a2.x + a2.y);
        tr.ev(12, tkey);
        tmem_st32(t_s + c0, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full);
        tr.ev(13, tkey);
        return;
      }
#pragma unroll
      for (int c = 0; c < CW / 32; ++c) tmem_ld32(t_s + c0 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
      tmem_ld_wait();
    }
  }
  // partial row max as 4 independent 3-input-max chains
  float mx[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) mx[u] = fmaxf(__uint_as_float(s[2 * u]), __uint_as_float(s[2 * u + 1]));
#pragma unroll
  for (int i = 8; i < CW; i += 8) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      mx[u] = fmaxf(mx[u], fmaxf(__uint_as_float(s[i + 2 * u]), __uint_as_float(s[i + 2 * u + 1])));
  }
  const float pm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
  float mt = pm;
  if constexpr (NP > 1) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot + part * kSub * 4), "f"(pm) : "memory");
  tr.ev(15, tkey);
  // every part published its max
  named_bar_sync(bar_id, NP * 128);
  }
#pragma unroll
  for (int o = 1; o < NP; ++o) {
    float po;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(po) : "r"(xslot + ((part + o) % NP) * kSub * 4) : "memory");
    mt = fmaxf(mt, po);
  }
  tr.ev(11, tkey);
  const float mt2 = mt * sl2;
  const bool move = mt2 > m + kRescaleThreshold;  // also true on the first finite tile
  const float alpha = move ? fast_exp2(m - mt2) : 1.f;
  if (move) m = mt2;
  const float mb = m == -INFINITY ? 0.f : m;
  if constexpr (SPLITP) {
    static_assert(NP == 1, "the split P hand-off is for full-row phases");
    // O rescale first: the MMA may start P V on the first key half before
    // this phase ends (O is quiescent: S(t) done implies P(t-1) V done)
    if (t > 0 && __any_sync(0xffffffffu, move)) {
#pragma unroll 1
      for (int c = 0; c < OW / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(t_o + c * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
        tmem_st32(t_o + c * 32, o);
      }
    }
    const uint64_t sc2 = f2(sl2, sl2), nm2 = f2(-mb, -mb);
    float rs = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t pk[32];
      uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
      for (int i = 64 * h; i < 64 * h + 64; i += 2) {
        const int jj = i / 2;
        const float2 x = f2_split(ffma2(f2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sc2, nm2));
        constexpr uint32_t kPolyMask = V == 0 ? 0x88u : (V == 1 ? 0x92u : 0x80u);
        float p0, p1;
        if (full && ((kPolyMask >> (jj % 8)) & 1u)) {
          const float2 e = exp2_poly2(x.x, x.y);
          p0 = e.x;
          p1 = e.y;
        } else {
          p0 = fast_exp2(x.x);  // masked scores are -inf: exact zeros
          p1 = fast_exp2(x.y);
        }
        acc2[jj % 4] = fadd2(acc2[jj % 4], f2(p0, p1));
        pk[jj - 32 * h] = pack_bf16(p0, p1);
      }
      const float2 a2 = f2_split(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])));
      rs += a2.x + a2.y;
      // this key half of P into its S columns, then hand it to the MMA warp
      tmem_st32(t_s + 32 * h, pk);
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(h == 0 ? p_first : p_full);
    }
    l = l * alpha + rs;
    tr.ev(13, tkey);
    return;
  }
  // O rescale (rare: the row max grew by more than 2^8) before the
  // exponentials, so they and the P stores form one straight-line block; O
  // is quiescent here (S(t) done implies P(t-1) V done) and the MMA reads it
  // only after p_full
  if (t > 0 && __any_sync(0xffffffffu, move)) {
#pragma unroll 1
    for (int c = 0; c < OW / 32; ++c) {
      uint32_t o[32];
      tmem_ld32(t_o + oc0 + c * 32, o);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
      tmem_st32(t_o + oc0 + c * 32, o);
    }
  }
  // TOK: the two sub-tiles' exponential loops take turns on the SM
  // sub-partitions' MUFU pipes instead of slowing each other down
  if constexpr (TOK) {
    if (tok_parity >= 0) mbar_wait(tok_wait, static_cast<uint32_t>(tok_parity));
  }
  uint32_t pk[CW / 2];
  float rs;
  if (full) {
    // packed f32x2: x = s * scale - m two lanes per FFMA2, sums by FADD2
    const uint64_t sc2 = f2(sl2, sl2), nm2 = f2(-mb, -mb);
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int i = 0; i < CW; i += 2) {
      const int jj = i / 2;
      const float2 x = f2_split(ffma2(f2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sc2, nm2));
      // pairs (jj % 8) on the FMA pipe: V0 {3, 7}, V1 {1, 4, 7}, V2 {7}
      constexpr uint32_t kPolyMask = V == 0 ? 0x88u : (V == 1 ? 0x92u : 0x80u);
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
    const float2 a2 = f2_split(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])));
    rs = a2.x + a2.y;
  } else {
    // masked scores are -inf: all exponentials on MUFU (exact zeros), packed
    // arithmetic otherwise as above
    const uint64_t sc2 = f2(sl2, sl2), nm2 = f2(-mb, -mb);
    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int i = 0; i < CW; i += 2) {
      const float2 x = f2_split(ffma2(f2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sc2, nm2));
      const float p0 = fast_exp2(x.x), p1 = fast_exp2(x.y);
      acc2[(i / 2) % 4] = fadd2(acc2[(i / 2) % 4], f2(p0, p1));
      pk[i / 2] = pack_bf16(p0, p1);
    }
    const float2 a2 = f2_split(fadd2(fadd2(acc2[0], acc2[1]), fadd2(acc2[2], acc2[3])));
    rs = a2.x + a2.y;
  }
  l = l * alpha + rs;
  if constexpr (TOK) mbar_arrive(tok_arrive);
  tr.ev(12, tkey);
  // P (bf16 pairs) into the first CW/2 of this part's own (consumed) S columns
  if constexpr (CW == 128) {
    tmem_st32(t_s + c0, *reinterpret_cast<uint32_t(*)[32]>(&pk[0]));
    tmem_st32(t_s + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(&pk[32]));
  } else if constexpr (CW == 64) {
    tmem_st32(t_s + c0, pk);
  } else {
    tmem_st16(t_s + c0, pk);
  }
  tmem_st_wait();
  tc_fence_before();
  mbar_arrive(p_full);
  tr.ev(13, tkey);
}

// Output of one sub-tile row part (D / NP columns): normalise (or merge into
// an existing (out, lse) pair) and store. lt = full row sum, lse_old read
// before any part of this row stored the new lse.
template <int D, int NP>
__device__ __forceinline__ void softmax_store(const FwdParams& p, int head, int q, int part, float m, float lt,
                                              float lse_old, uint32_t t_o, bool has_work, uint64_t* o_final) {
  constexpr int OW = D / NP;
  const int oc0 = part * OW;
  float* lse_ptr = p.lse + static_cast<size_t>(head) * p.seqlen_q + q;
  const bool valid = q < p.seqlen_q;
  const bool has = lt > 0.f;
  const float lse_cur = has ? (m * kLn2 + logf(lt)) : -INFINITY;
  const float inv_l = has ? 1.f / lt : 0.f;
  if (has_work) {
    mbar_wait(o_final, 0);
    tc_fence_after();
  }
  const uint32_t t_oh = t_o + oc0;
  const size_t row_off = (static_cast<size_t>(q) * p.hq + head) * D + oc0;
  if (p.accumulate) {
    // merge into (out, lse) with the log-sum-exp correction; f32 output
    const float lse_new = has ? (lse_old > lse_cur ? lse_old + log1pf(__expf(lse_cur - lse_old))
                                                   : lse_cur + log1pf(__expf(lse_old - lse_cur)))
                              : lse_old;
    const float w_old = has ? __expf(lse_old - lse_new) : 1.f;
    const float w_cur = has ? __expf(lse_cur - lse_new) * inv_l : 0.f;
#pragma unroll 1
    for (int c = 0; c < OW / 32; ++c) {
      uint32_t o[32];
      if (has_work) {
        tmem_ld32(t_oh + c * 32, o);
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
    if (valid && has && part == 0) *lse_ptr = lse_new;
  } else {
#pragma unroll 1
    for (int c = 0; c < OW / 32; ++c) {
      uint32_t o[32];
      if (has_work) {
        tmem_ld32(t_oh + c * 32, o);
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
    if (valid && part == 0) *lse_ptr = lse_cur;
  }
}

// V: softmax variant (diagnostics, MAGI_FWD_VARIANT): exp2 pairs on the FMA
// pipe out of every 8 — 0: 2 (25%), 1: 3 (37.5%), 2: 1 (12.5%).
template <int D, int V, int LAYOUT, bool TR>
__global__ void __launch_bounds__(FwdLayout<LAYOUT>::kThreads, 1)
    ffa_fwd_kernel(const __grid_constant__ CUtensorMap tmap_q,
                   const __grid_constant__ CUtensorMap tmap_k,
                   const __grid_constant__ CUtensorMap tmap_v, const FwdParams p) {
  using L = FwdSmem<D>;
  constexpr bool PAIR = FwdLayout<LAYOUT>::kPair;
  constexpr int NP = FwdLayout<LAYOUT>::kParts;
  constexpr int kTmaWarp = FwdLayout<LAYOUT>::kTmaWarp;
  constexpr int kMmaWarp = FwdLayout<LAYOUT>::kMmaWarp;
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
  long long* const trace = static_cast<int>(blockIdx.x) == p.trace_block ? p.trace : nullptr;

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
      mbar_init(&bars.p_full[i], NP * kSub);
      mbar_init(&bars.p_first[i], NP * kSub);
      mbar_init(&bars.o_final[i], 1);
      mbar_init(&bars.tok[i], 128);
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

  if (FwdLayout<LAYOUT>::kSetmaxnreg && warp >= kTmaWarp)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(FwdLayout<LAYOUT>::kCtrlRegs));
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
  } else if (FwdLayout<LAYOUT>::kThreads == 640 && warp == kMmaWarp + 1) {
    // diagnostics only: observe when K / V tiles land (traced CTA)
    if (lane == 0 && trace != nullptr && n_total > 0) {
      TracerT<TR> tr;
      tr.init(trace, 4);
      PipeState st;
      for (int t = 0; t < n_total; ++t) {
        mbar_wait(&bars.k_full[st.index], st.phase);
        tr.ev(32, t);
        mbar_wait(&bars.v_full[st.index], st.phase);
        tr.ev(33, t);
        st.advance<kStages>();
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
        if constexpr (FwdLayout<LAYOUT>::kSplitP) {
          // P V by key halves, each as soon as its half of P is in TMEM
          constexpr uint32_t idesc_pv = make_idesc_bf16(128, D, false, true);
          mbar_wait(&bars.v_full[vst.index], vst.phase);
          mbar_wait(&bars.p_first[0], t & 1);
          tc_fence_after();
          umma_gemm_ts_k128_lo(tmem + 256, tmem + 0, v_desc, idesc_pv, t > 0 ? 1u : 0u);
          mbar_wait(&bars.p_full[0], t & 1);
          tr.ev(1, t);
          tc_fence_after();
          umma_gemm_ts_k128_hi(tmem + 256, tmem + 0, v_desc, idesc_pv, 1u);
        } else {
        mbar_wait(&bars.p_full[0], t & 1);
        tr.ev(1, t);
        mbar_wait(&bars.v_full[vst.index], vst.phase);
        tr.ev(2, t);
        tc_fence_after();
        issue_pv<D, NP>(tmem + 256, tmem + 0, v_desc, t > 0);
        }
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
        if constexpr (FwdLayout<LAYOUT>::kSplitP) {
          constexpr uint32_t idesc_pv = make_idesc_bf16(128, D, false, true);
          mbar_wait(&bars.p_first[1], t & 1);
          tc_fence_after();
          umma_gemm_ts_k128_lo(tmem + 384, tmem + 128, v_desc, idesc_pv, t > 0 ? 1u : 0u);
          mbar_wait(&bars.p_full[1], t & 1);
          tr.ev(4, t);
          tc_fence_after();
          umma_gemm_ts_k128_hi(tmem + 384, tmem + 128, v_desc, idesc_pv, 1u);
        } else {
        mbar_wait(&bars.p_full[1], t & 1);
        tr.ev(4, t);
        tc_fence_after();
        issue_pv<D, NP>(tmem + 384, tmem + 128, v_desc, t > 0);
        }
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
    // Thread = query row = TMEM lane; warpgroup part w owns score columns
    // [w 128/NP, (w+1) 128/NP) of a sub-tile, and the parts of a sub-tile
    // exchange partial row maxima through shared memory so they agree bit for
    // bit on the exponent base. PAIR: sub-tile = warp / 8, the two sub-tiles'
    // phases overlap; otherwise all warpgroups walk both sub-tiles in turn.
    if (FwdLayout<LAYOUT>::kSetmaxnreg)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(FwdLayout<LAYOUT>::kSoftRegs));
    constexpr int kSubs = PAIR ? 1 : 2;  // sub-tiles this thread serves
    const int sub0 = PAIR ? warp / (4 * NP) : 0;
    const int part = (warp / 4) % NP;
    const int row = (warp % 4) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const float sl2 = p.scale_log2;
    const uint32_t xch_base = smem_u32(smem + L::kXch);
    const uint32_t bar_n = PAIR ? 0 : 1;  // named barrier: per sub-tile (PAIR) or shared
    float m[kSubs], l[kSubs];
    int q[kSubs];
#pragma unroll
    for (int u = 0; u < kSubs; ++u) {
      m[u] = -INFINITY;  // exponent base, log2 domain (lazily moved)
      l[u] = 0.f;        // this part's sum of 2^(x - m)
      q[u] = tile.q0 + (sub0 + u) * kSub + row;
    }
    TracerT<TR> tr;
    if (part == 0 && warp % 4 == 0) tr.init(trace, 1 + sub0);
    int t = 0;
    for (int it = tile.item_begin; it < tile.item_end; ++it) {
      const FwdItem item = p.items[it];
      int32_t lo[kSubs], hi[kSubs];
#pragma unroll
      for (int u = 0; u < kSubs; ++u) row_bounds(item.qs, item.qe, item.ks, item.ke, item.type, q[u], lo[u], hi[u]);
      for (int j = 0; j < item.n_ktiles; ++j, ++t) {
        const int kc = item.k_begin + j * kBlockN + part * (128 / NP);
#pragma unroll
        for (int u = 0; u < kSubs; ++u) {
          const int sub = sub0 + u;
          // slot [t parity][sub][part][row]: a part can run one step ahead of
          // the others' reads, never two
          const uint32_t xslot = xch_base + ((((t & 1) * 2 + sub) * 4) * kSub + row) * 4;
          // layout 7 turn order: sub-tile 0 phase t after sub-tile 1 phase t-1,
          // sub-tile 1 phase t after sub-tile 0 phase t
          const int tok_parity = sub == 0 ? (t > 0 ? ((t - 1) & 1) : -1) : (t & 1);
          softmax_phase<D, V, NP, TracerT<TR>, FwdLayout<LAYOUT>::kSplitP, FwdLayout<LAYOUT>::kToken,
                        FwdLayout<LAYOUT>::kSpec>(
              m[u], l[u], tmem + sub * 128 + lane_off, tmem + 256 + sub * 128 + lane_off, part, kc, lo[u], hi[u], t,
              xslot, PAIR ? 1 + sub : bar_n, sl2, &bars.s_full[sub], &bars.p_full[sub], tr, kSubs * t + u,
              &bars.p_first[sub], &bars.tok[sub ^ 1], tok_parity, &bars.tok[sub]);
        }
      }
    }

    // ---------------------------------------------------------- epilogue
    float lse_old[kSubs];
#pragma unroll
    for (int u = 0; u < kSubs; ++u)
      lse_old[u] = (p.accumulate && q[u] < p.seqlen_q) ? p.lse[static_cast<size_t>(head) * p.seqlen_q + q[u]]
                                                      : -INFINITY;
    // full row sums over the parts; the barrier also orders every part's
    // lse_old read before any lse store
    float* xl = reinterpret_cast<float*>(smem + L::kXch) + L::kXl;  // [sub][part][row]
#pragma unroll
    for (int u = 0; u < kSubs; ++u) xl[((sub0 + u) * 4 + part) * kSub + row] = l[u];
    named_bar_sync(PAIR ? 1 + sub0 : bar_n, NP * 128);
#pragma unroll
    for (int u = 0; u < kSubs; ++u) {
      const int sub = sub0 + u;
      float lt = 0.f;
#pragma unroll
      for (int o = 0; o < NP; ++o) lt += xl[(sub * 4 + o) * kSub + row];
      softmax_store<D, NP>(p, head, q[u], part, m[u], lt, lse_old[u], tmem + 256 + sub * 128 + lane_off,
                           n_total > 0, &bars.o_final[sub]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int D, int V, int LAYOUT>
cudaError_t launch_fwd_impl(const FwdParams& prm, const void* q, const void* k, const void* v,
                            cudaStream_t stream) {
  const CUtensorMap tq = make_tmap_thd(q, prm.seqlen_q, prm.hq, D, 128);
  const CUtensorMap tk = make_tmap_thd(k, prm.seqlen_k, prm.hk, D, 128);
  const CUtensorMap tv = make_tmap_thd(v, prm.seqlen_k, prm.hk, D, 128);
  const int smem = FwdSmem<D>::kBytes + 1024;
  cudaError_t err =
      cudaFuncSetAttribute(ffa_fwd_kernel<D, V, LAYOUT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return err;
  const dim3 grid(static_cast<unsigned>(prm.num_tiles) * prm.hq);
  if constexpr (V == 0 && (LAYOUT == 5 || LAYOUT == 7)) {
    if (prm.trace != nullptr) {  // diagnostics: the traced instantiation of the default kernel
      err = cudaFuncSetAttribute(ffa_fwd_kernel<D, V, LAYOUT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem);
      if (err != cudaSuccess) return err;
      ffa_fwd_kernel<D, V, LAYOUT, true><<<grid, FwdLayout<LAYOUT>::kThreads, smem, stream>>>(tq, tk, tv, prm);
      return cudaGetLastError();
    }
  }
  ffa_fwd_kernel<D, V, LAYOUT, false><<<grid, FwdLayout<LAYOUT>::kThreads, smem, stream>>>(tq, tk, tv, prm);
  return cudaGetLastError();
}

}  // namespace

// tiles/items: the plan's 256-row q-major work list (FfaPlan::fwd2_*).
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
  prm.trace = g_fwd_trace;
  prm.trace_block = g_fwd_trace_block;
  static const int variant = [] {
    const char* e = std::getenv("MAGI_FWD_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  // default: layout 5 (full-row softmax warpgroups with 200 registers via
  // setmaxnreg), 25% of the exponentials on the FMA pipe — measured best on
  // config 2 (~4% over layout 0); MAGI_FWD_VARIANT selects the alternatives
  // for A/B runs.
  if (head_dim == 128) {
    switch (variant) {
      case 1: return launch_fwd_impl<128, 0, 1>(prm, q, k, v, stream);
      case 3: return launch_fwd_impl<128, 1, 1>(prm, q, k, v, stream);
      case 4: return launch_fwd_impl<128, 0, 0>(prm, q, k, v, stream);
      case 5: return launch_fwd_impl<128, 2, 1>(prm, q, k, v, stream);
      case 6: return launch_fwd_impl<128, 2, 0>(prm, q, k, v, stream);
      case 7: return launch_fwd_impl<128, 1, 2>(prm, q, k, v, stream);
      case 8: return launch_fwd_impl<128, 0, 2>(prm, q, k, v, stream);
      case 10: return launch_fwd_impl<128, 0, 4>(prm, q, k, v, stream);
      case 11: return launch_fwd_impl<128, 1, 4>(prm, q, k, v, stream);
      case 12: return launch_fwd_impl<128, 0, 5>(prm, q, k, v, stream);
      case 13: return launch_fwd_impl<128, 1, 5>(prm, q, k, v, stream);
      case 15: return launch_fwd_impl<128, 0, 6>(prm, q, k, v, stream);
      case 16: return launch_fwd_impl<128, 0, 7>(prm, q, k, v, stream);
      case 17: return launch_fwd_impl<128, 1, 7>(prm, q, k, v, stream);
      case 18: return launch_fwd_impl<128, 0, 8>(prm, q, k, v, stream);
      case 19: return launch_fwd_impl<128, 1, 8>(prm, q, k, v, stream);
      case 14: return launch_fwd_impl<128, 1, 0>(prm, q, k, v, stream);
      default: return launch_fwd_impl<128, 0, 5>(prm, q, k, v, stream);
    }
  }
  if (head_dim == 64) return launch_fwd_impl<64, 1, 0>(prm, q, k, v, stream);
  return cudaErrorInvalidValue;
}

}  // namespace magi

namespace magi {
// Diagnostics: route one forward CTA's per-role event log to a device buffer.
void set_fwd_trace(long long* buffer, int block) {
  g_fwd_trace = buffer;
  g_fwd_trace_block = block;
}
}  // namespace magi
