// Schedule model of the multi-stage overlap pipeline. Reference semantics:
// /root/reference/proj/src/sim.cpp (flops :29-34, throughput :36-45,
// Timeline :47-118, report :122-172, simulate_magi :174-259).
#include "sim.hpp"

#include <algorithm>

#include <nlohmann/json.hpp>

#include "errors.hpp"

namespace magiplan {

int64_t flops(const AttnMask& m, const WorkloadSpec& w, Pass pass) {
  const int64_t fwd = 4 * mask_area(m, Counting::Multiplicity) * w.batch_size * w.num_heads_q * w.head_dim;
  return pass == Pass::Fwd ? fwd : fwd * 5 / 2;
}

double throughput(int64_t flops_total, Cost runtime, Rank cp) {
  if (runtime <= 0) throw UsageError("throughput needs a positive runtime");
  if (cp < 1) throw UsageError("throughput needs cp_size >= 1");
  return static_cast<double>(flops_total) / (static_cast<double>(runtime) * static_cast<double>(cp));
}

int Timeline::add(Rank rank, int stream, Cost duration, std::vector<int> deps, std::string label) {
  MAGI_CHECK(!ran_, "timeline already ran");
  MAGI_CHECK(duration >= 0, "task duration must be >= 0");
  const int id = static_cast<int>(tasks_.size());
  for (int d : deps) MAGI_CHECK(d >= 0 && d < id, "deps must reference earlier tasks");
  for (int t = id - 1; t >= 0; --t) {  // in-order stream semantics
    if (tasks_[static_cast<std::size_t>(t)].rank == rank &&
        tasks_[static_cast<std::size_t>(t)].stream == stream) {
      deps.push_back(t);
      break;
    }
  }
  tasks_.push_back({rank, stream, duration, std::move(deps)});
  labels_.push_back(std::move(label));
  return id;
}

void Timeline::run() {
  MAGI_CHECK(!ran_, "timeline already ran");
  for (Task& t : tasks_) {
    Cost start = 0;
    for (int d : t.deps) start = std::max(start, tasks_[static_cast<std::size_t>(d)].end);
    t.end = start + t.dur;
    makespan_ = std::max(makespan_, t.end);
  }
  ran_ = true;
}

Cost Timeline::rank_end(Rank r) const {
  Cost e = 0;
  for (const Task& t : tasks_)
    if (t.rank == r) e = std::max(e, t.end);
  return e;
}

Cost Timeline::rank_compute(Rank r) const {
  Cost c = 0;
  for (const Task& t : tasks_)
    if (t.rank == r && t.stream == kCompute) c += t.dur;
  return c;
}

Rank Timeline::bottleneck_rank() const {
  Rank best = 0;
  Cost best_end = -1;
  for (const Task& t : tasks_) {
    const Cost e = rank_end(t.rank);
    if (e > best_end || (e == best_end && t.rank < best)) {
      best = t.rank;
      best_end = e;
    }
  }
  return best;
}

SimReport finish_report(std::string schedule, Pass pass, Rank cp, Timeline& tl, int64_t fl, int64_t vol,
                        std::vector<std::string> event_log) {
  tl.run();
  SimReport r;
  r.schedule = std::move(schedule);
  r.pass = pass;
  r.cp_size = cp;
  r.makespan = tl.makespan();
  r.exposed_comm = r.makespan - tl.rank_compute(tl.bottleneck_rank());
  MAGI_CHECK(r.exposed_comm >= 0, "exposed communication must be non-negative");
  for (Rank k = 0; k < cp; ++k) {
    const Cost busy = tl.rank_compute(k);
    r.per_rank_busy.push_back(r.makespan > 0 ? static_cast<double>(busy) / static_cast<double>(r.makespan) : 0.0);
    r.per_rank_makespan.push_back(tl.rank_end(k));
    r.per_rank_compute.push_back(busy);
  }
  r.flops_total = fl;
  r.throughput_per_gpu = r.makespan > 0 ? throughput(fl, r.makespan, cp) : 0.0;
  r.comm_volume_tokens = vol;
  r.event_log = std::move(event_log);
  return r;
}

std::string sim_report_to_json(const SimReport& r) {
  nlohmann::ordered_json j;
  j["schedule"] = r.schedule;
  j["pass"] = r.pass == Pass::Fwd ? "fwd" : "bwd";
  j["cp_size"] = r.cp_size;
  j["makespan"] = r.makespan;
  j["exposed_comm"] = r.exposed_comm;
  j["per_rank_busy"] = r.per_rank_busy;
  j["per_rank_makespan"] = r.per_rank_makespan;
  j["per_rank_compute"] = r.per_rank_compute;
  j["flops_total"] = r.flops_total;
  j["throughput_per_gpu"] = r.throughput_per_gpu;
  j["comm_volume_tokens"] = r.comm_volume_tokens;
  if (!r.event_log.empty()) j["event_log"] = r.event_log;
  return j.dump();
}

std::pair<SimReport, SimReport> simulate_magi(const AttnMask& m, const DispatchPlan& plan,
                                              const TransferTable& cast, const TransferTable& reduce,
                                              const SolveResult& stages, const CostModel& model,
                                              const WorkloadSpec& w) {
  const Rank cp = plan.cp_size;
  if (static_cast<Rank>(stages.plans.size()) != cp) {
    throw UsageError("stage plans cover " + std::to_string(stages.plans.size()) +
                     " ranks, plan has " + std::to_string(cp));
  }
  Timeline fwd, bwd;
  for (Rank r = 0; r < cp; ++r) {
    const StagePlan& sp = stages.plans[static_cast<std::size_t>(r)];
    // forward step j: cast(j+1) || ffa(j)
    std::vector<int> prev;
    for (int j = 0; j <= sp.fwd.num_stages; ++j) {
      std::vector<int> step;
      if (j + 1 <= sp.fwd.num_stages) {
        step.push_back(fwd.add(r, Timeline::kComm,
                               model.cast_cost.eval(sp.fwd.stage_tokens[static_cast<std::size_t>(j)]),
                               prev, "cast(" + std::to_string(j + 1) + ")"));
      }
      const Cost d = j == 0 ? model.host_compute(sp.host_pairs, false)
                            : model.ffa_fwd.eval(sp.fwd.stage_pairs[static_cast<std::size_t>(j - 1)]);
      step.push_back(fwd.add(r, Timeline::kCompute, d, prev, "ffa(" + std::to_string(j) + ")"));
      prev = std::move(step);
    }
    // backward step j: cast(j+1) || ffa(j) || reduce(j-1), final reduce exposed
    prev.clear();
    const auto& b = sp.bwd;
    for (int j = 0; j <= b.num_stages; ++j) {
      std::vector<int> step;
      if (j + 1 <= b.num_stages) {
        step.push_back(bwd.add(r, Timeline::kComm,
                               model.cast_cost.eval(b.stage_tokens[static_cast<std::size_t>(j)]), prev,
                               "cast(" + std::to_string(j + 1) + ")"));
      }
      const Cost d = j == 0 ? model.host_compute(sp.host_pairs, true)
                            : model.ffa_bwd.eval(b.stage_pairs[static_cast<std::size_t>(j - 1)]);
      step.push_back(bwd.add(r, Timeline::kCompute, d, prev, "ffa(" + std::to_string(j) + ")"));
      if (j >= 2) {
        step.push_back(bwd.add(r, Timeline::kReduce,
                               model.reduce_cost.eval(b.stage_tokens[static_cast<std::size_t>(j - 2)]),
                               prev, "reduce(" + std::to_string(j - 1) + ")"));
      }
      prev = std::move(step);
    }
    bwd.add(r, Timeline::kReduce,
            model.reduce_cost.eval(b.stage_tokens[static_cast<std::size_t>(b.num_stages - 1)]), prev,
            "reduce(" + std::to_string(b.num_stages) + ")");
  }
  const int64_t cv = cast.total_token_transfers(), rv = reduce.total_token_transfers();
  return {finish_report("magi", Pass::Fwd, cp, fwd, flops(m, w, Pass::Fwd), cv),
          finish_report("magi", Pass::Bwd, cp, bwd, flops(m, w, Pass::Bwd), cv + rv)};
}

}  // namespace magiplan
