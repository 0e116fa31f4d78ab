// FFA tile planner: turns an AttnSlice list into the device work lists the
// sm_100a kernels walk (q-major for forward / dQ, k-major for dK/dV).
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "kernels/ffa_common.cuh"

namespace magiplan {

struct FfaPlan {
  int64_t seqlen_q = 0;
  int64_t seqlen_k = 0;
  int32_t head_dim = 128;
  std::vector<magi::SliceGeom> slices;
  int64_t area_multiplicity = 0;

  std::vector<magi::FwdTile> fwd_tiles;  // 128-row tiles (dQ pass), LPT order
  std::vector<magi::FwdItem> fwd_items;
  std::vector<magi::FwdTile> fwd2_tiles;  // 256-row tiles (forward), LPT order
  std::vector<magi::FwdItem> fwd2_items;
  std::vector<magi::BwdTile> bwd_tiles;  // LPT order (most query tiles first)
  std::vector<magi::BwdItem> bwd_items;

  // device copies (owned)
  magi::FwdTile* d_fwd_tiles = nullptr;
  magi::FwdItem* d_fwd_items = nullptr;
  magi::FwdTile* d_fwd2_tiles = nullptr;
  magi::FwdItem* d_fwd2_items = nullptr;
  magi::BwdTile* d_bwd_tiles = nullptr;
  magi::BwdItem* d_bwd_items = nullptr;
  int device = -1;  // device holding the copies (-1: not uploaded yet)
  std::mutex upload_mutex;

  FfaPlan() = default;
  FfaPlan(const FfaPlan&) = delete;
  FfaPlan& operator=(const FfaPlan&) = delete;
  ~FfaPlan();

  int64_t fwd_ktiles() const;
  int64_t bwd_qtiles() const;
  std::string describe_json() const;
};

// Validates (UsageError on malformed / out-of-bounds ranges, as
// AttnMask::check_valid, reference proj/src/mask.cpp:175-191) and builds the
// host work lists; does not touch the device.
void build_ffa_worklists(FfaPlan& plan);
// Uploads the work lists to the current device on first use (thread-safe,
// synchronous cudaMemcpy). DeviceError on CUDA failure; UsageError when the
// plan is later used from a different device than the one it lives on.
void ensure_uploaded(FfaPlan& plan);

// Device work lists of an uploaded plan, both q-tile heights.
inline magi::FwdWork fwd_work(const FfaPlan& P) {
  return {P.d_fwd_tiles, P.d_fwd_items, static_cast<int32_t>(P.fwd_tiles.size()),
          P.d_fwd2_tiles, P.d_fwd2_items, static_cast<int32_t>(P.fwd2_tiles.size())};
}

}  // namespace magiplan
