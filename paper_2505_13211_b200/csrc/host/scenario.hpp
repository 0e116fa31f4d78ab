// Scenario orchestration: spec parsing, the planning pipeline, report JSON,
// and the executor plan for the real context-parallel run.
// Reference surface: /root/reference/proj/include/magiplan/scenario.hpp:38-106.
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "comm.hpp"
#include "dispatch.hpp"
#include "overlap.hpp"
#include "sim.hpp"

namespace magiplan {

inline constexpr int kSchemaVersion = 1;

uint64_t fnv1a_hash(const std::string& text);
std::string hash_hex(uint64_t h);

struct SweepSpec {
  std::vector<Rank> cp_sizes;
  Token per_rank_seqlen = 0;
  Token sample_length = 0;
};

struct ScenarioSpec {
  std::string mask_spec_json;
  WorkloadSpec workload;
  std::string schedule = "magi";
  Rank cp_size = 1;
  int64_t tp_size = 1, dp_size = 1;
  Token dispatch_chunk_size = 0;  // 0: default (1/8 of the per-rank sequence)
  std::string dispatch_policy = "greedy";
  CostModel cost_model;
  OverlapHyperparams overlap;
  int cso_num_chunks = 5;
  uint64_t seed = 0;
  std::optional<SweepSpec> sweep;
  std::string spec_hash;

  static ScenarioSpec parse(const std::string& text, const std::string& base_dir = ".");
};

struct BalanceSummary {
  Pairs max_workload = 0;
  double mean_workload = 0.0;
  double imbalance = 0.0;
};
BalanceSummary balance_summary(const DispatchPlan& plan);

struct PlanArtifacts {
  AttnMask mask;
  Token chunk_size = 0;
  DispatchPlan plan;
  std::vector<KvDemand> demands;
  TransferTable cast_table, reduce_table;
  RedundancyReport redundancy;
  BalanceSummary balance;
  SolveResult stages;
};

AttnMask scenario_mask(const ScenarioSpec& spec, Token seqlen = 0);
std::vector<RankTraffic> rank_traffic_from(const AttnMask& m, const DispatchPlan& plan,
                                           const TransferTable& cast);
PlanArtifacts run_plan(const ScenarioSpec& spec, const AttnMask& m);
std::string plan_artifacts_to_json(const PlanArtifacts& a, const ScenarioSpec& spec);
std::vector<std::string> run_simulate(const ScenarioSpec& spec, int jobs);

// Executor view (new): per rank, its query/key chunks and per stage the
// receive-buffer layout plus the rank's slices in local coordinates.
std::string exec_plan_to_json(const PlanArtifacts& a, const ScenarioSpec& spec);

// Deterministic log-normal sample lengths (Box-Muller on 53-bit uniforms of
// std::mt19937_64), the config-4 varlen generator; reference
// proj/src/pack.cpp:228-253.
std::vector<Token> lognormal_lengths(std::size_t count, double median, double sigma,
                                     Token max_length, uint64_t seed);

}  // namespace magiplan
