// Multi-stage compute/communication overlap solver (paper Alg. 2).
// Reference surface: /root/reference/proj/include/magiplan/overlap.hpp:28-154.
#pragma once

#include <functional>
#include <optional>
#include <string>
#include <vector>

#include "mask.hpp"

namespace magiplan {

using Cost = int64_t;  // integer time units

struct AffineCost {
  double latency = 0.0;
  double per_unit = 0.0;
  Cost eval(int64_t work) const;  // 0 for work <= 0, else max(0, llround(lat + pu*work))
};

AffineCost fit_affine(const std::vector<std::pair<int64_t, int64_t>>& samples);

struct CostModel {
  AffineCost ffa_fwd, ffa_bwd;          // per allowed pair
  AffineCost cast_cost, reduce_cost;    // per KV token
  AffineCost q_proj, k_proj, v_proj, kv_cache_update, cross_attn;
  std::optional<Cost> host_cost_fwd, host_cost_bwd;
  Cost host_compute(Pairs host_pairs, bool backward) const;
};

CostModel cost_model_from_json(const std::string& text);
std::string cost_model_to_json(const CostModel& m);

struct OverlapHyperparams {
  int64_t min_chunk_size = 512;
  int64_t max_num_chunks = 8;
};

std::vector<int64_t> partition_packages(const std::vector<int64_t>& traffic, int64_t min_chunk_size,
                                        int64_t max_num_chunks);
std::vector<std::vector<int>> assign_packages_to_stages(const std::vector<int64_t>& sizes,
                                                        int num_stages,
                                                        std::optional<uint64_t> shuffle_seed = {});

struct StageCosts {
  Cost host_compute = 0;
  std::vector<Cost> compute, cast, reduce;  // stage j+1 at index j
};

Cost estimate_fwd_cost(int s, const std::function<Cost(int)>& gc, const std::function<Cost(int)>& ffa);
Cost estimate_bwd_cost(int s, const std::function<Cost(int)>& gc, const std::function<Cost(int)>& ffa,
                       const std::function<Cost(int)>& gr);
Cost estimate_fwd_cost(const StageCosts& c);
Cost estimate_bwd_cost(const StageCosts& c);

struct StageBreakdown {
  int num_stages = 1;
  std::vector<std::vector<int>> stage_packages;
  std::vector<int64_t> stage_tokens;
  std::vector<Pairs> stage_pairs;
  Cost est_cost = 0;
};

struct StagePlan {
  Rank rank = 0;
  Pairs host_pairs = 0;
  std::vector<int64_t> package_sizes;
  std::vector<std::vector<TokenRange>> package_ranges;
  StageBreakdown fwd, bwd;
};

struct RankTraffic {
  Pairs host_pairs = 0;
  std::vector<TokenRange> remote_ranges;
  std::function<Pairs(Token, Token)> pairs_in_cols;
};

struct RankStageSearch {
  Rank rank = 0;
  std::vector<int64_t> package_sizes;
  std::vector<Cost> cost_fwd, cost_bwd;  // s = index + 1
  int s_opt_fwd = 1, s_opt_bwd = 1;
};

struct SolveResult {
  int num_stages_fwd = 1, num_stages_bwd = 1;
  std::vector<RankStageSearch> searches;
  std::vector<StagePlan> plans;
};

std::vector<std::vector<TokenRange>> package_ranges_of(const std::vector<TokenRange>& remote,
                                                       const std::vector<int64_t>& sizes);
SolveResult solve_stages(const std::vector<RankTraffic>& traffic, const CostModel& model,
                         const OverlapHyperparams& hp);
std::string solve_result_to_json(const SolveResult& r);

}  // namespace magiplan
