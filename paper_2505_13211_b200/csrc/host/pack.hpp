// Online packing-and-padding (PnP) packer: the upstream producer of the
// varlen sample lists that config 4's slice masks are built from.
// Reference semantics: /root/reference/proj/include/magiplan/pack.hpp:28-104,
// /root/reference/proj/src/pack.cpp:30-271 (config checks :30-55, admission
// :61-72, one packing iteration :74-196, utilisation stats :198-226);
// driver run_pack: /root/reference/proj/src/scenario.cpp:428-554.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "mask.hpp"

namespace magiplan {

struct PackingConfig {
  Token max_length = 65536;
  int64_t dp_size = 1;
  int64_t tp_size = 1;
  int64_t cp_size = 1;
  int64_t bins_per_iteration = 1;  // N bins per iteration
  int64_t pool_capacity = 4;       // M candidate slots, M >= 4N
  double defer_threshold = 0.5;    // minimum mean fill to emit a batch
  int swap_passes = 2;

  void check_valid() const;
};

struct PackedSample {
  int64_t id = 0;
  Token length = 0;
};

struct PackedBin {
  std::vector<PackedSample> samples;
  Token fill = 0;
};

struct PackedBatch {
  std::vector<PackedBin> bins;
  double utilization = 0.0;  // sum of fills / (N * max_length)
};

// Owns the candidate pool. The pool keeps arrival order; each iteration packs
// a length-sorted view of it (first-fit decreasing, then bounded one-for-one
// swaps, then empty-bin spreading) and removes what it placed.
class Packer {
 public:
  explicit Packer(PackingConfig config);

  bool admit(const PackedSample& sample);
  bool pool_full() const { return static_cast<int64_t>(pool_.size()) >= cfg_.pool_capacity; }
  std::size_t pool_size() const { return pool_.size(); }
  int64_t rejected_oversized() const { return rejected_; }
  int64_t deferred_iterations() const { return deferred_; }
  std::optional<PackedBatch> pack_iteration();

 private:
  PackingConfig cfg_;
  std::vector<PackedSample> pool_;
  int64_t rejected_ = 0;
  int64_t deferred_ = 0;
};

struct UtilizationStats {
  int64_t batches = 0;
  double mean_utilization = 0.0;
  double min_utilization = 0.0;
  double dp_group_spread = 0.0;  // (max - min) / mean of per-DP-group fills, bin i -> group i % dp
};

UtilizationStats utilization_stats(const std::vector<PackedBatch>& history,
                                   const PackingConfig& config);

// JSON report of a packing run over an "id length" line stream, or over the
// log-normal generator when stream_text is null (reference scenario.cpp:428-554).
std::string run_pack(const std::string& config_json, const std::string* stream_text);

}  // namespace magiplan
