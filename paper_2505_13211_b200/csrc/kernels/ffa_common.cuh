// Work-list records shared by the host tile planner (csrc/host/ffa_plan.cpp)
// and the FFA kernels.
//
// A slice (reference AttnSlice, proj/include/magiplan/mask.hpp:59-74) admits,
// for global query row q in [qs, qe), the global key columns [lo(q), hi(q)):
//   FULL        [ks, ke)
//   CAUSAL      [ks, clamp(q + ke - qe + 1, ks, ke))          bottom-right diagonal
//   INV_CAUSAL  [min(ks + q - qs, ke), ke)                    top-left diagonal
//   BI_CAUSAL   both bounds
// which is AttnSlice::row_cols (proj/src/mask.cpp:74-84) rewritten in global
// coordinates. Both bounds are non-decreasing in q, which is what lets the
// planner describe each (tile, slice) intersection as one contiguous span of
// 128-wide key (forward) or query (backward) tiles.
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#define MAGI_HD inline
#else
#define MAGI_HD __host__ __device__ __forceinline__
#endif

namespace magi {

enum SliceType : int32_t { kFull = 0, kCausal = 1, kInvCausal = 2, kBiCausal = 3 };

constexpr int kBlockM = 128;  // query rows per tile
constexpr int kBlockN = 128;  // key columns per tile

struct SliceGeom {
  int32_t qs, qe, ks, ke;
  int32_t type;
};

// One (query tile, slice) intersection for the q-major kernels: key tiles
// [k_begin + i*128, ...) for i < n_ktiles.
struct FwdItem {
  int32_t qs, qe, ks, ke;
  int32_t type;
  int32_t k_begin;
  int32_t n_ktiles;
  int32_t pad;
};

struct FwdTile {
  int32_t q0;          // first query row of the tile
  int32_t item_begin;  // [item_begin, item_end) into the item array
  int32_t item_end;
  int32_t n_ktiles;    // total key tiles over the items (LPT weight)
};

// A forward work list at both q-tile heights the planner builds (128 rows:
// FfaPlan::fwd_*, 256 rows: fwd2_*); the launcher uses the one its kernel
// layout tiles by.
struct FwdWork {
  const FwdTile* tiles128;
  const FwdItem* items128;
  int32_t num_tiles128;
  const FwdTile* tiles256;
  const FwdItem* items256;
  int32_t num_tiles256;
};

// One (key tile, slice) intersection for the k-major backward kernel: query
// tiles [q_begin + i*128, ...) for i < n_qtiles.
struct BwdItem {
  int32_t qs, qe, ks, ke;
  int32_t type;
  int32_t q_begin;
  int32_t n_qtiles;
  int32_t pad;
};

struct BwdTile {
  int32_t k0;
  int32_t item_begin;
  int32_t item_end;
  int32_t n_qtiles;
};

MAGI_HD int32_t clamp_i32(int32_t v, int32_t lo, int32_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

// Allowed global key columns [lo, hi) of global row q for a slice; empty
// (lo >= hi) when q is outside the slice's rows.
MAGI_HD void row_bounds(int32_t qs, int32_t qe, int32_t ks,
                                                    int32_t ke, int32_t type, int32_t q,
                                                    int32_t& lo, int32_t& hi) {
  if (q < qs || q >= qe) {
    lo = 0;
    hi = 0;
    return;
  }
  lo = (type == kInvCausal || type == kBiCausal) ? (ks + (q - qs) < ke ? ks + (q - qs) : ke) : ks;
  hi = (type == kCausal || type == kBiCausal) ? clamp_i32(q + ke - qe + 1, ks, ke) : ke;
}

}  // namespace magi
