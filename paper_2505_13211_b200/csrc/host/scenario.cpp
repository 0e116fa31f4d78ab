// Scenario orchestration. Reference semantics: /root/reference/proj/src/scenario.cpp
// (fnv1a :32-49, parse :93-214, scenario_mask :216-238, rank_traffic_from
// :240-265, run_plan :294-312, plan JSON :314-337, simulate :341-426) and
// metrics.cpp:23-39 (balance). The executor plan is new.
#include "scenario.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <future>
#include <map>
#include <random>
#include <sstream>

#include <nlohmann/json.hpp>

#include "errors.hpp"

namespace magiplan {

using json = nlohmann::ordered_json;

uint64_t fnv1a_hash(const std::string& text) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : text) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

std::string hash_hex(uint64_t h) {
  static const char* hex = "0123456789abcdef";
  std::string s(16, '0');
  for (int i = 15; i >= 0; --i, h >>= 4) s[static_cast<std::size_t>(i)] = hex[h & 0xF];
  return s;
}

namespace {

json parse_object(const std::string& text, const std::string& what) {
  json j;
  try {
    j = json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw UsageError(what + ": " + e.what());
  }
  if (!j.is_object()) throw UsageError(what + " must be a JSON object");
  return j;
}

void only_keys(const json& obj, std::initializer_list<const char*> allowed, const char* ctx) {
  for (const auto& [key, value] : obj.items()) {
    if (std::none_of(allowed.begin(), allowed.end(), [&](const char* a) { return key == a; })) {
      throw UsageError("unknown field '" + key + "' in " + ctx);
    }
  }
}

std::string slurp(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw UsageError("cannot open referenced file '" + path + "'");
  std::ostringstream buf;
  buf << in.rdbuf();
  return buf.str();
}

const char* const kSchedules[] = {"magi", "ring", "ring_serial", "ulysses", "cso"};

template <typename T>
void read_opt(const json& j, const char* key, T& slot) {
  if (j.contains(key)) slot = j[key].get<T>();
}

}  // namespace

ScenarioSpec ScenarioSpec::parse(const std::string& text, const std::string& base_dir) {
  const json j = parse_object(text, "scenario spec");
  ScenarioSpec spec;
  try {
    only_keys(j, {"schema_version", "workload", "schedule", "cp_size", "tp_size", "dp_size",
                  "dispatch", "dispatch_chunk_size", "cost_model", "overlap", "cso_num_chunks",
                  "seed", "sweep"},
              "scenario spec");
    spec.spec_hash = hash_hex(fnv1a_hash(text));
    if (!j.contains("workload") || !j["workload"].is_object() || !j["workload"].contains("mask")) {
      throw UsageError("scenario needs workload.mask");
    }
    const json& w = j["workload"];
    only_keys(w, {"mask", "batch_size", "num_heads_q", "num_heads_k", "num_heads_v", "head_dim",
                  "dtype_bytes"},
              "workload");
    spec.mask_spec_json = w["mask"].dump();
    read_opt(w, "batch_size", spec.workload.batch_size);
    read_opt(w, "num_heads_q", spec.workload.num_heads_q);
    read_opt(w, "num_heads_k", spec.workload.num_heads_k);
    read_opt(w, "num_heads_v", spec.workload.num_heads_v);
    read_opt(w, "head_dim", spec.workload.head_dim);
    read_opt(w, "dtype_bytes", spec.workload.dtype_bytes);
    const auto& wl = spec.workload;
    if (wl.batch_size <= 0 || wl.num_heads_q <= 0 || wl.num_heads_k <= 0 || wl.num_heads_v <= 0 ||
        wl.head_dim <= 0 || wl.dtype_bytes <= 0) {
      throw UsageError("workload multipliers must be positive");
    }
    read_opt(j, "schedule", spec.schedule);
    if (std::none_of(std::begin(kSchedules), std::end(kSchedules),
                     [&](const char* s) { return spec.schedule == s; })) {
      throw UsageError("unknown schedule '" + spec.schedule +
                       "' (valid: magi, ring, ring_serial, ulysses, cso)");
    }
    read_opt(j, "cp_size", spec.cp_size);
    read_opt(j, "tp_size", spec.tp_size);
    read_opt(j, "dp_size", spec.dp_size);
    if (spec.cp_size < 1 || spec.tp_size < 1 || spec.dp_size < 1) {
      throw UsageError("cp/tp/dp sizes must be >= 1");
    }
    if (j.contains("dispatch_chunk_size")) {
      spec.dispatch_chunk_size = j["dispatch_chunk_size"].get<Token>();
      if (spec.dispatch_chunk_size < 0) {
        throw UsageError("dispatch_chunk_size must be >= 0 (0 = default)");
      }
    }
    if (j.contains("dispatch")) {
      spec.dispatch_policy = j["dispatch"].get<std::string>();
      if (spec.dispatch_policy != "greedy" && spec.dispatch_policy != "zigzag") {
        throw UsageError("dispatch must be 'greedy' or 'zigzag'");
      }
    }
    if (j.contains("cost_model")) {
      const std::string mt = j["cost_model"].is_string()
                                 ? slurp(base_dir + "/" + j["cost_model"].get<std::string>())
                                 : j["cost_model"].dump();
      spec.cost_model = cost_model_from_json(mt);
      const json mj = parse_object(mt, "cost model");
      read_opt(mj, "min_chunk_size", spec.overlap.min_chunk_size);
      read_opt(mj, "max_num_chunks", spec.overlap.max_num_chunks);
    }
    if (j.contains("overlap")) {
      const json& o = j["overlap"];
      only_keys(o, {"min_chunk_size", "max_num_chunks"}, "overlap spec");
      read_opt(o, "min_chunk_size", spec.overlap.min_chunk_size);
      read_opt(o, "max_num_chunks", spec.overlap.max_num_chunks);
    }
    read_opt(j, "cso_num_chunks", spec.cso_num_chunks);
    read_opt(j, "seed", spec.seed);
    if (j.contains("sweep")) {
      const json& s = j["sweep"];
      only_keys(s, {"cp_sizes", "per_rank_seqlen", "sample_length"}, "sweep spec");
      if (!s.contains("cp_sizes") || !s.contains("per_rank_seqlen")) {
        throw UsageError("sweep needs cp_sizes and per_rank_seqlen");
      }
      SweepSpec sw;
      sw.cp_sizes = s["cp_sizes"].get<std::vector<Rank>>();
      sw.per_rank_seqlen = s["per_rank_seqlen"].get<Token>();
      read_opt(s, "sample_length", sw.sample_length);
      if (sw.cp_sizes.empty() || sw.per_rank_seqlen <= 0) {
        throw UsageError("sweep cp_sizes must be non-empty, per_rank_seqlen > 0");
      }
      spec.sweep = sw;
    }
  } catch (const nlohmann::json::exception& e) {
    throw UsageError(std::string("scenario spec: ") + e.what());
  }
  // surface mask errors eagerly (a sweep's mask is a template: first point)
  if (spec.sweep) {
    (void)scenario_mask(spec, spec.sweep->per_rank_seqlen * spec.sweep->cp_sizes[0]);
  } else {
    (void)scenario_mask(spec);
  }
  return spec;
}

AttnMask scenario_mask(const ScenarioSpec& spec, Token seqlen) {
  if (seqlen == 0) return parse_mask_spec(spec.mask_spec_json);
  json j = parse_object(spec.mask_spec_json, "mask spec");
  if (!j.contains("pattern")) {
    throw UsageError("sweeps need a pattern mask, not an explicit slice list");
  }
  j["seqlen"] = seqlen;
  if (j["pattern"].get<std::string>().rfind("varlen", 0) == 0) {
    const Token sample = spec.sweep ? spec.sweep->sample_length : 0;
    if (sample <= 0 || seqlen % sample != 0) {
      throw ConstraintError("sweep over a varlen pattern needs sample_length dividing seqlen (" +
                            std::to_string(sample) + " vs " + std::to_string(seqlen) + ")");
    }
    j["params"]["sample_lengths"] = std::vector<Token>(static_cast<std::size_t>(seqlen / sample), sample);
  }
  return parse_mask_spec(j.dump());
}

BalanceSummary balance_summary(const DispatchPlan& plan) {
  plan.validate();
  BalanceSummary b;
  Pairs total = 0;
  for (Pairs w : plan.bucket_workloads) {
    b.max_workload = std::max(b.max_workload, w);
    total += w;
  }
  b.mean_workload = static_cast<double>(total) / static_cast<double>(plan.cp_size);
  b.imbalance = b.mean_workload > 0.0 ? static_cast<double>(b.max_workload) / b.mean_workload - 1.0 : 0.0;
  return b;
}

std::vector<RankTraffic> rank_traffic_from(const AttnMask& m, const DispatchPlan& plan,
                                           const TransferTable& cast) {
  std::vector<RankTraffic> out;
  for (Rank r = 0; r < plan.cp_size; ++r) {
    RankTraffic t;
    t.remote_ranges = cast.incoming_ranges_of_rank(r);
    auto local = std::make_shared<AttnMask>(local_mask_of_rank(m, plan, r));
    auto pairs = [local](Token a, Token b) {
      Pairs n = 0;
      for (const AttnSlice& s : local->slices) n += slice_area_in_cols(s, a, b);
      return n;
    };
    // KV is co-hosted with Q: the rank's own rows are its local key columns
    for (const TokenRange& rows : plan.rows_of_bucket(r)) t.host_pairs += pairs(rows.start, rows.end);
    t.pairs_in_cols = pairs;
    out.push_back(std::move(t));
  }
  return out;
}

namespace {

Token effective_chunk(const ScenarioSpec& spec, Token seqlen) {
  return spec.dispatch_chunk_size > 0 ? spec.dispatch_chunk_size
                                      : default_dispatch_chunk_size(seqlen, spec.cp_size);
}

}  // namespace

PlanArtifacts run_plan(const ScenarioSpec& spec, const AttnMask& m) {
  PlanArtifacts a;
  a.mask = m;
  a.chunk_size = effective_chunk(spec, m.seqlen_q);
  if (a.chunk_size <= 0 || m.seqlen_q % (spec.cp_size * a.chunk_size) != 0) {
    throw ConstraintError("constraint violated: seqlen % (cp_size * dispatch_chunk_size) = 0 (seqlen " +
                          std::to_string(m.seqlen_q) + ", cp_size " + std::to_string(spec.cp_size) +
                          ", dispatch_chunk_size " + std::to_string(a.chunk_size) + ")");
  }
  const auto chunks = shard_into_chunks(m, a.chunk_size);
  const bool zigzag = spec.dispatch_policy == "zigzag" || spec.schedule == "ring" ||
                      spec.schedule == "ring_serial";
  a.plan = zigzag ? zigzag_dispatch(chunks, spec.cp_size) : greedy_dispatch(chunks, spec.cp_size);
  a.demands = compute_kv_demands(m, a.plan);
  std::tie(a.cast_table, a.reduce_table) = build_transfer_tables(a.demands, a.chunk_size, spec.cp_size);
  a.redundancy = redundancy_report(a.demands, a.plan);
  a.balance = balance_summary(a.plan);
  a.stages = solve_stages(rank_traffic_from(m, a.plan, a.cast_table), spec.cost_model, spec.overlap);
  return a;
}

std::string plan_artifacts_to_json(const PlanArtifacts& a, const ScenarioSpec& spec) {
  json j;
  j["schema_version"] = kSchemaVersion;
  j["spec_hash"] = spec.spec_hash;
  j["seed"] = spec.seed;
  j["seqlen"] = a.mask.seqlen_q;
  j["cp_size"] = spec.cp_size;
  j["dispatch_chunk_size"] = a.chunk_size;
  j["dispatch_plan"] = json::parse(plan_to_json(a.plan));
  const int64_t bpt = spec.workload.kv_bytes_per_token();
  j["transfer_cast"] = json::parse(transfer_table_to_json(a.cast_table, bpt));
  j["transfer_reduce"] = json::parse(transfer_table_to_json(a.reduce_table, bpt));
  j["redundancy"] = {{"sent_ring", a.redundancy.sent_ring},
                     {"needed", a.redundancy.needed},
                     {"sent_group", a.redundancy.sent_group},
                     {"redundancy_ratio", a.redundancy.redundancy_ratio}};
  j["balance"] = {{"max_workload", a.balance.max_workload},
                  {"mean_workload", a.balance.mean_workload},
                  {"imbalance", a.balance.imbalance}};
  j["overlap"] = json::parse(solve_result_to_json(a.stages));
  return j.dump();
}

namespace {

std::vector<std::string> simulate_point(const ScenarioSpec& spec, Token seqlen) {
  // reference scenario.cpp:341-366
  const AttnMask m = scenario_mask(spec, seqlen);
  std::vector<SimReport> reports;
  if (spec.schedule == "magi") {
    const PlanArtifacts a = run_plan(spec, m);
    auto [fwd, bwd] = simulate_magi(a.mask, a.plan, a.cast_table, a.reduce_table, a.stages,
                                    spec.cost_model, spec.workload);
    reports = {std::move(fwd), std::move(bwd)};
  } else if (spec.schedule == "ring" || spec.schedule == "ring_serial") {
    const PlanArtifacts a = run_plan(spec, m);
    auto [fwd, bwd] = simulate_ring(a.mask, a.plan, spec.cost_model, spec.workload, spec.schedule == "ring");
    reports = {std::move(fwd), std::move(bwd)};
  } else if (spec.schedule == "ulysses") {
    reports.push_back(simulate_ulysses(m, spec.workload, spec.cost_model, spec.cp_size));
  } else {
    reports.push_back(simulate_cso(m, spec.workload, spec.cost_model, spec.cp_size, spec.cso_num_chunks));
  }
  std::vector<std::string> out;
  for (const SimReport* r = reports.data(); r != reports.data() + reports.size(); ++r) {
    json rec;
    rec["schema_version"] = kSchemaVersion;
    rec["spec_hash"] = spec.spec_hash;
    rec["seed"] = spec.seed;
    rec["seqlen"] = seqlen == 0 ? m.seqlen_q : seqlen;
    const json body = json::parse(sim_report_to_json(*r));
    for (const auto& [k, v] : body.items()) rec[k] = v;
    out.push_back(rec.dump());
  }
  return out;
}

}  // namespace

std::vector<std::string> run_simulate(const ScenarioSpec& spec, int jobs) {
  if (!spec.sweep) return simulate_point(spec, 0);
  std::vector<std::pair<Token, Rank>> points;
  for (Rank cp : spec.sweep->cp_sizes) {
    if (cp < 1) throw UsageError("sweep cp_sizes must be >= 1");
    points.emplace_back(spec.sweep->per_rank_seqlen * cp, cp);
  }
  std::vector<std::string> records;
  const std::size_t par = static_cast<std::size_t>(std::max(1, jobs));
  for (std::size_t base = 0; base < points.size(); base += par) {
    std::vector<std::future<std::vector<std::string>>> batch;
    for (std::size_t i = base; i < std::min(points.size(), base + par); ++i) {
      ScenarioSpec ps = spec;
      ps.cp_size = points[i].second;
      const Token seqlen = points[i].first;
      batch.push_back(std::async(std::launch::async, [ps = std::move(ps), seqlen] {
        return simulate_point(ps, seqlen);
      }));
    }
    for (auto& f : batch)
      for (auto& r : f.get()) records.push_back(std::move(r));
  }
  return records;
}

std::string exec_plan_to_json(const PlanArtifacts& a, const ScenarioSpec& spec) {
  const DispatchPlan& plan = a.plan;
  const Token cs = a.chunk_size;
  const auto buckets = plan.chunks_of_buckets();
  std::vector<Token> local_pos(plan.assignment.size(), 0);  // chunk -> slot on its host
  for (const auto& b : buckets)
    for (std::size_t i = 0; i < b.size(); ++i) local_pos[static_cast<std::size_t>(b[i])] = static_cast<Token>(i);
  auto local_of = [&](Token t) { return local_pos[static_cast<std::size_t>(t / cs)] * cs + t % cs; };
  auto host_of = [&](Token t) { return plan.assignment[static_cast<std::size_t>(t / cs)]; };

  auto slice_json = [](const AttnSlice& s) {
    return json::array({s.q.start, s.q.end, s.k.start, s.k.end, static_cast<int>(s.type)});
  };
  // local slices clipped to key window [a, b) and shifted: q -> local row,
  // k -> `buf_start + (k - a)`
  auto emit = [&](const AttnMask& local, TokenRange win, Token buf_start, json& out) {
    for (const AttnSlice& s : local.slices) {
      for (AttnSlice p : clip_slice(s, s.q, win)) {
        const Token dq = local_of(p.q.start) - p.q.start;
        const Token dk = buf_start - win.start;
        p.q = {p.q.start + dq, p.q.end + dq};
        p.k = {p.k.start + dk, p.k.end + dk};
        out.push_back(slice_json(p));
      }
    }
  };

  json j;
  j["schema_version"] = kSchemaVersion;
  j["spec_hash"] = spec.spec_hash;
  j["seqlen"] = a.mask.seqlen_q;
  j["cp_size"] = plan.cp_size;
  j["chunk_size"] = cs;
  j["local_tokens"] = a.mask.seqlen_q / plan.cp_size;
  j["num_stages_fwd"] = a.stages.num_stages_fwd;
  j["num_stages_bwd"] = a.stages.num_stages_bwd;
  j["area_multiplicity"] = mask_area(a.mask, Counting::Multiplicity);
  j["ranks"] = json::array();
  for (Rank r = 0; r < plan.cp_size; ++r) {
    const AttnMask local = local_mask_of_rank(a.mask, plan, r);
    const StagePlan& sp = a.stages.plans[static_cast<std::size_t>(r)];
    json jr;
    jr["rank"] = r;
    jr["chunks"] = buckets[static_cast<std::size_t>(r)];
    json host = json::array();
    for (const TokenRange& rows : plan.rows_of_bucket(r)) emit(local, rows, local_of(rows.start), host);
    jr["host_slices"] = host;
    for (int pass = 0; pass < 2; ++pass) {
      const StageBreakdown& b = pass == 0 ? sp.fwd : sp.bwd;
      json stages = json::array();
      for (const auto& pkgs : b.stage_packages) {
        // receive buffer grouped by source rank (the all-to-all output order)
        std::vector<std::pair<Rank, TokenRange>> recv;
        for (int p : pkgs)
          for (const TokenRange& rg : sp.package_ranges[static_cast<std::size_t>(p)]) {
            if (!rg.empty()) recv.emplace_back(host_of(rg.start), rg);
          }
        std::stable_sort(recv.begin(), recv.end(),
                         [](const auto& x, const auto& y) { return x.first < y.first; });
        json jrecv = json::array(), jsl = json::array();
        Token off = 0;
        for (const auto& [src, rg] : recv) {
          jrecv.push_back({src, rg.start, rg.end, local_of(rg.start), off});
          emit(local, rg, off, jsl);
          off += rg.length();
        }
        json js;
        js["buf_tokens"] = off;
        js["recv"] = jrecv;
        js["slices"] = jsl;
        stages.push_back(js);
      }
      jr[pass == 0 ? "fwd_stages" : "bwd_stages"] = stages;
    }
    j["ranks"].push_back(jr);
  }
  return j.dump();
}

std::vector<Token> lognormal_lengths(std::size_t count, double median, double sigma, Token max_length,
                                     uint64_t seed) {
  if (median <= 0.0 || sigma < 0.0 || max_length <= 0) {
    throw UsageError("lognormal stream needs median > 0, sigma >= 0");
  }
  std::mt19937_64 rng(seed);
  auto unit = [&rng] { return (static_cast<double>(rng() >> 11) + 0.5) / 9007199254740992.0; };
  std::vector<Token> out;
  out.reserve(count);
  for (std::size_t i = 0; i < count; ++i) {
    const double u1 = unit(), u2 = unit();
    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793238462643 * u2);
    out.push_back(std::clamp<Token>(std::llround(median * std::exp(sigma * z)), 1, max_length));
  }
  return out;
}

}  // namespace magiplan
