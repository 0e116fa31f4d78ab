// FFA tile planner (see ffa_plan.hpp).
//
// Forward / dQ work list: for every 128-row query tile, one item per slice
// whose q-range meets the tile, covering the key span [lo(a), hi(b)) of the
// tile's first/last rows inside the slice (both bounds are monotone in q, so
// this span is exactly the union of the rows' allowed columns). Tiles no
// slice touches still get a CTA so their output rows are written as empty
// (O = 0, LSE = -inf; reference semantics of an empty row).
//
// dK/dV work list: for every 128-column key tile, one item per slice whose
// allowed region meets the tile, covering the contiguous query rows whose
// allowed columns intersect the tile (found by binary search on the monotone
// row bounds).
#include "ffa_plan.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <limits>
#include <numeric>

#include <nlohmann/json.hpp>

#include "errors.hpp"

namespace magiplan {

using magi::kBlockM;
using magi::kBlockN;

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

void bounds(const magi::SliceGeom& s, int64_t q, int32_t& lo, int32_t& hi) {
  magi::row_bounds(s.qs, s.qe, s.ks, s.ke, s.type, static_cast<int32_t>(q), lo, hi);
}

int64_t slice_pairs(const magi::SliceGeom& s) {
  int64_t total = 0;
  for (int64_t q = s.qs; q < s.qe; ++q) {
    int32_t lo, hi;
    bounds(s, q, lo, hi);
    if (hi > lo) total += hi - lo;
  }
  return total;
}

template <typename T>
T* upload(const std::vector<T>& host) {
  if (host.empty()) return nullptr;
  void* ptr = nullptr;
  cudaError_t err = cudaMalloc(&ptr, host.size() * sizeof(T));
  if (err == cudaSuccess) {
    err = cudaMemcpy(ptr, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice);
  }
  if (err != cudaSuccess) {
    if (ptr) cudaFree(ptr);
    throw DeviceError(std::string("ffa plan upload: ") + cudaGetErrorString(err));
  }
  return static_cast<T*>(ptr);
}

}  // namespace

FfaPlan::~FfaPlan() {
  cudaFree(d_fwd_tiles);
  cudaFree(d_fwd_items);
  cudaFree(d_fwd2_tiles);
  cudaFree(d_fwd2_items);
  cudaFree(d_bwd_tiles);
  cudaFree(d_bwd_items);
}

int64_t FfaPlan::fwd_ktiles() const {
  int64_t n = 0;
  for (const auto& t : fwd_tiles) n += t.n_ktiles;
  return n;
}

int64_t FfaPlan::bwd_qtiles() const {
  int64_t n = 0;
  for (const auto& t : bwd_tiles) n += t.n_qtiles;
  return n;
}

std::string FfaPlan::describe_json() const {
  nlohmann::ordered_json j;
  j["seqlen_q"] = seqlen_q;
  j["seqlen_k"] = seqlen_k;
  j["head_dim"] = head_dim;
  j["num_slices"] = slices.size();
  j["area_multiplicity"] = area_multiplicity;
  j["q_tiles"] = fwd_tiles.size();
  j["fwd_items"] = fwd_items.size();
  j["fwd_ktiles"] = fwd_ktiles();
  j["k_tiles"] = bwd_tiles.size();
  j["bwd_items"] = bwd_items.size();
  j["bwd_qtiles"] = bwd_qtiles();
  return j.dump();
}

namespace {
void build_qmajor(const FfaPlan& plan, int64_t rows, const std::vector<int>& by_q,
                  std::vector<magi::FwdTile>& out_tiles, std::vector<magi::FwdItem>& out_items);
void build_kmajor(FfaPlan& plan);
}  // namespace

void build_ffa_worklists(FfaPlan& plan) {
  constexpr int64_t kMaxTokens = std::numeric_limits<int32_t>::max() - 2 * kBlockM;
  if (plan.seqlen_q < 0 || plan.seqlen_k < 0) throw UsageError("mask seqlen must be non-negative");
  if (plan.seqlen_q > kMaxTokens || plan.seqlen_k > kMaxTokens) {
    throw UsageError("seqlen exceeds the int32 token index range of the FFA kernels");
  }
  if (plan.head_dim != 64 && plan.head_dim != 128) {
    throw UsageError("head_dim must be 64 or 128 (got " + std::to_string(plan.head_dim) + ")");
  }
  for (std::size_t i = 0; i < plan.slices.size(); ++i) {
    const auto& s = plan.slices[i];
    const bool ok_range = 0 <= s.qs && s.qs <= s.qe && 0 <= s.ks && s.ks <= s.ke;
    if (!ok_range) throw UsageError("slice " + std::to_string(i) + ": malformed range");
    if (s.qe > plan.seqlen_q || s.ke > plan.seqlen_k) {
      throw UsageError("slice " + std::to_string(i) + " exceeds mask bounds " +
                       std::to_string(plan.seqlen_q) + "x" + std::to_string(plan.seqlen_k));
    }
    if (s.type < 0 || s.type > 3) {
      throw UsageError("slice " + std::to_string(i) + ": unknown mask type " +
                       std::to_string(s.type));
    }
  }

  plan.area_multiplicity = 0;
  for (const auto& s : plan.slices) plan.area_multiplicity += slice_pairs(s);

  // slices sorted by q start / k start so tiles only scan candidates
  std::vector<int> by_q(plan.slices.size());
  std::iota(by_q.begin(), by_q.end(), 0);

  // ---- q-major work lists: 128-row tiles (dQ) and 256-row tiles (forward)
  build_qmajor(plan, kBlockM, by_q, plan.fwd_tiles, plan.fwd_items);
  build_qmajor(plan, 2 * kBlockM, by_q, plan.fwd2_tiles, plan.fwd2_items);

  // ---- k-major work list
  build_kmajor(plan);
}

namespace {

void build_qmajor(const FfaPlan& plan, int64_t rows, const std::vector<int>& by_q,
                  std::vector<magi::FwdTile>& out_tiles, std::vector<magi::FwdItem>& out_items) {
  out_tiles.clear();
  out_items.clear();
  const int64_t n_qt = ceil_div(plan.seqlen_q, rows);
  std::vector<magi::FwdTile> tiles;
  tiles.reserve(static_cast<std::size_t>(n_qt));
  std::vector<std::vector<magi::FwdItem>> tile_items(static_cast<std::size_t>(n_qt));
  for (int64_t i = 0; i < n_qt; ++i) {
    const int64_t q0 = i * rows;
    const int64_t q1 = std::min<int64_t>(q0 + rows, plan.seqlen_q);
    for (int si : by_q) {
      const auto& s = plan.slices[static_cast<std::size_t>(si)];
      if (s.qs >= q1 || s.qe <= q0 || s.ks >= s.ke) continue;
      const int64_t a = std::max<int64_t>(q0, s.qs);
      const int64_t b = std::min<int64_t>(q1, s.qe) - 1;
      int32_t lo_a, hi_a, lo_b, hi_b;
      bounds(s, a, lo_a, hi_a);
      bounds(s, b, lo_b, hi_b);
      if (lo_a >= hi_b) continue;
      magi::FwdItem it{s.qs, s.qe, s.ks, s.ke, s.type, lo_a,
                       static_cast<int32_t>(ceil_div(hi_b - lo_a, kBlockN)), 0};
      tile_items[static_cast<std::size_t>(i)].push_back(it);
    }
  }
  for (int64_t i = 0; i < n_qt; ++i) {
    int32_t n = 0;
    for (const auto& it : tile_items[static_cast<std::size_t>(i)]) n += it.n_ktiles;
    tiles.push_back({static_cast<int32_t>(i * rows), 0, 0, n});
  }
  std::vector<int64_t> order(static_cast<std::size_t>(n_qt));
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
    return tiles[static_cast<std::size_t>(x)].n_ktiles > tiles[static_cast<std::size_t>(y)].n_ktiles;
  });
  for (int64_t i : order) {
    magi::FwdTile t = tiles[static_cast<std::size_t>(i)];
    t.item_begin = static_cast<int32_t>(out_items.size());
    for (const auto& it : tile_items[static_cast<std::size_t>(i)]) out_items.push_back(it);
    t.item_end = static_cast<int32_t>(out_items.size());
    out_tiles.push_back(t);
  }
}

void build_kmajor(FfaPlan& plan) {
  plan.bwd_tiles.clear();
  plan.bwd_items.clear();
  const int64_t n_kt = ceil_div(plan.seqlen_k, kBlockN);
  std::vector<std::vector<magi::BwdItem>> ktile_items(static_cast<std::size_t>(n_kt));
  for (const auto& s : plan.slices) {
    if (s.qs >= s.qe || s.ks >= s.ke) continue;
    const int64_t kt_first = s.ks / kBlockN;
    const int64_t kt_last = (s.ke - 1) / kBlockN;
    for (int64_t j = kt_first; j <= kt_last; ++j) {
      const int64_t k0 = j * kBlockN;
      const int64_t k1 = std::min<int64_t>(k0 + kBlockN, plan.seqlen_k);
      // first row whose hi > k0 (hi non-decreasing)
      int64_t lo_q = s.qs, hi_q = s.qe;
      while (lo_q < hi_q) {
        const int64_t mid = (lo_q + hi_q) / 2;
        int32_t l, h;
        bounds(s, mid, l, h);
        if (h > k0) hi_q = mid; else lo_q = mid + 1;
      }
      // start on a multiple of 4 rows: the dK/dV kernel fetches the tile's
      // lse / delta rows by TMA, whose innermost coordinate must be 16-byte
      // aligned (the extra rows fall outside the slice and are masked)
      const int64_t qa = lo_q & ~int64_t{3};
      // last row whose lo < k1 (lo non-decreasing): first row with lo >= k1, minus one
      lo_q = s.qs;
      hi_q = s.qe;
      while (lo_q < hi_q) {
        const int64_t mid = (lo_q + hi_q) / 2;
        int32_t l, h;
        bounds(s, mid, l, h);
        if (l >= k1) hi_q = mid; else lo_q = mid + 1;
      }
      const int64_t qb = lo_q - 1;
      if (qa > qb) continue;
      // any row in [qa, qb] with a non-empty intersection?
      int32_t la, ha, lb, hb;
      bounds(s, qa, la, ha);
      bounds(s, qb, lb, hb);
      (void)ha;
      (void)lb;
      if (std::max<int64_t>(la, k0) >= std::min<int64_t>(hb, k1)) continue;
      ktile_items[static_cast<std::size_t>(j)].push_back(
          {s.qs, s.qe, s.ks, s.ke, s.type, static_cast<int32_t>(qa),
           static_cast<int32_t>(ceil_div(qb - qa + 1, kBlockM)), 0});
    }
  }
  std::vector<magi::BwdTile> ktiles;
  for (int64_t j = 0; j < n_kt; ++j) {
    int32_t n = 0;
    for (const auto& it : ktile_items[static_cast<std::size_t>(j)]) n += it.n_qtiles;
    ktiles.push_back({static_cast<int32_t>(j * kBlockN), 0, 0, n});
  }
  std::vector<int64_t> korder(static_cast<std::size_t>(n_kt));
  std::iota(korder.begin(), korder.end(), 0);
  std::stable_sort(korder.begin(), korder.end(), [&](int64_t x, int64_t y) {
    return ktiles[static_cast<std::size_t>(x)].n_qtiles > ktiles[static_cast<std::size_t>(y)].n_qtiles;
  });
  for (int64_t j : korder) {
    magi::BwdTile t = ktiles[static_cast<std::size_t>(j)];
    t.item_begin = static_cast<int32_t>(plan.bwd_items.size());
    for (const auto& it : ktile_items[static_cast<std::size_t>(j)]) plan.bwd_items.push_back(it);
    t.item_end = static_cast<int32_t>(plan.bwd_items.size());
    plan.bwd_tiles.push_back(t);
  }
}

}  // namespace

void ensure_uploaded(FfaPlan& plan) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) throw DeviceError("ffa plan: no CUDA device");
  std::lock_guard<std::mutex> lock(plan.upload_mutex);
  if (plan.device >= 0) {
    if (plan.device != dev) {
      throw UsageError("ffa plan lives on device " + std::to_string(plan.device) +
                       " but was used on device " + std::to_string(dev));
    }
    return;
  }
  plan.d_fwd_tiles = upload(plan.fwd_tiles);
  plan.d_fwd_items = upload(plan.fwd_items);
  plan.d_fwd2_tiles = upload(plan.fwd2_tiles);
  plan.d_fwd2_items = upload(plan.fwd2_items);
  plan.d_bwd_tiles = upload(plan.bwd_tiles);
  plan.d_bwd_items = upload(plan.bwd_items);
  plan.device = dev;
}

}  // namespace magiplan
