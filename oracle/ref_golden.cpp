// TEST INFRASTRUCTURE ONLY — golden-vector generator.
//
// Links the reference planner compiled from its own sources
// (/root/reference/proj/src via oracle/Makefile) and records its outputs for
// seeded inputs into tests/golden/ref_planner.json. The CPU-only parity tests
// replay every record through libmagiplan.so (C ABI + magiplan_debug_eval)
// and require byte/bit-exact agreement. Run: oracle/_ref/ref_golden <out.json>
#include <cstdio>
#include <fstream>
#include <random>
#include <string>

#include <json.hpp>

#include "magiplan/comm.hpp"
#include "magiplan/dispatch.hpp"
#include "magiplan/magiplan.h"
#include "magiplan/mask.hpp"
#include "magiplan/overlap.hpp"
#include "magiplan/pack.hpp"
#include "magiplan/sim.hpp"

using namespace magiplan;
using json = nlohmann::ordered_json;

static json sl(const AttnSlice& s) {
  return json::array({s.q_range.start, s.q_range.end, s.k_range.start, s.k_range.end,
                      static_cast<int>(s.mask_type)});
}

static json mask_spec(const AttnMask& m) { return json::parse(mask_to_json(m)); }

static AttnMask random_mask(std::mt19937_64& rng, TokenIndex s, int max_slices) {
  AttnMask m;
  m.seqlen_q = m.seqlen_k = s;
  const int n = 1 + static_cast<int>(rng() % static_cast<uint64_t>(max_slices));
  for (int i = 0; i < n; ++i) {
    TokenIndex a = static_cast<TokenIndex>(rng() % static_cast<uint64_t>(s));
    TokenIndex b = static_cast<TokenIndex>(rng() % static_cast<uint64_t>(s + 1));
    TokenIndex c = static_cast<TokenIndex>(rng() % static_cast<uint64_t>(s));
    TokenIndex d = static_cast<TokenIndex>(rng() % static_cast<uint64_t>(s + 1));
    if (a > b) std::swap(a, b);
    if (c > d) std::swap(c, d);
    m.slices.push_back({{a, b}, {c, d}, static_cast<SliceMaskType>(rng() % 4)});
  }
  return m;
}

static std::string capi_plan(const std::string& scenario) {
  magiplan_scenario* sc = nullptr;
  if (magiplan_scenario_parse(scenario.c_str(), ".", &sc) != MAGIPLAN_OK) {
    return std::string("ERROR ") + magiplan_last_error();
  }
  char* out = nullptr;
  std::string res;
  if (magiplan_scenario_plan(sc, &out) == MAGIPLAN_OK) {
    res = out;
    magiplan_string_free(out);
  } else {
    res = std::string("ERROR ") + magiplan_last_error();
  }
  magiplan_scenario_free(sc);
  return res;
}

static std::string capi_simulate(const std::string& scenario) {
  magiplan_scenario* sc = nullptr;
  if (magiplan_scenario_parse(scenario.c_str(), ".", &sc) != MAGIPLAN_OK) {
    return std::string("ERROR ") + magiplan_last_error();
  }
  char* out = nullptr;
  std::string res;
  if (magiplan_scenario_simulate(sc, 2, &out) == MAGIPLAN_OK) {
    res = out;
    magiplan_string_free(out);
  } else {
    res = std::string("ERROR ") + magiplan_last_error();
  }
  magiplan_scenario_free(sc);
  return res;
}

static std::string capi_pack(const std::string& config, const char* stream) {
  char* out = nullptr;
  if (magiplan_pack_run(config.c_str(), stream, &out) != MAGIPLAN_OK) {
    return std::string("ERROR ") + magiplan_last_error();
  }
  std::string res(out);
  magiplan_string_free(out);
  return res;
}

int main(int argc, char** argv) {
  const std::string path = argc > 1 ? argv[1] : "ref_planner.json";
  std::mt19937_64 rng(20250519);
  json g;

  // ---- slice areas and column-window areas
  json areas = json::array();
  for (int t = 0; t < 4; ++t)
    for (TokenIndex lq = 0; lq <= 9; ++lq)
      for (TokenIndex lk = 0; lk <= 9; ++lk) {
        AttnSlice s{{3, 3 + lq}, {5, 5 + lk}, static_cast<SliceMaskType>(t)};
        areas.push_back({sl(s), slice_area(s)});
      }
  g["slice_area"] = areas;
  json in_cols = json::array();
  for (int i = 0; i < 600; ++i) {
    const TokenIndex lq = static_cast<TokenIndex>(rng() % 40), lk = static_cast<TokenIndex>(rng() % 40);
    AttnSlice s{{10, 10 + lq}, {7, 7 + lk}, static_cast<SliceMaskType>(rng() % 4)};
    TokenIndex c0 = static_cast<TokenIndex>(rng() % 60), c1 = static_cast<TokenIndex>(rng() % 60);
    if (c0 > c1) std::swap(c0, c1);
    in_cols.push_back({sl(s), {c0, c1}, slice_area_in_cols(s, c0, c1)});
  }
  g["slice_area_in_cols"] = in_cols;

  // ---- named patterns
  json named = json::array();
  const char* specs[] = {
      R"({"seqlen": 8, "pattern": "causal"})",
      R"({"seqlen": 8, "pattern": "full"})",
      R"({"seqlen": 8, "pattern": "block_causal", "params": {"block_size": 2}})",
      R"({"seqlen": 1024, "pattern": "block_causal", "params": {"block_size": 256}})",
      R"({"seqlen": 32768, "pattern": "block_causal", "params": {"block_size": 4096}})",
      R"({"seqlen": 32768, "pattern": "block_causal", "params": {"block_size": 2048}})",
      R"({"seqlen": 64, "pattern": "varlen_block_causal_last_global", "params": {"sample_lengths": [32, 32], "block_size": 8}})",
      R"({"seqlen": 48, "pattern": "varlen_block_causal", "params": {"sample_lengths": [16, 32], "block_size": 8}})",
      R"({"seqlen": 20, "pattern": "varlen_causal", "params": {"sample_lengths": [5, 7, 8]}})",
      R"({"seqlen": 20, "pattern": "varlen_full", "params": {"sample_lengths": [5, 7, 8]}})",
      R"({"seqlen": 40, "pattern": "sliding_window_causal", "params": {"window": 6}})",
      R"({"seqlen": 5, "pattern": "sliding_window_causal", "params": {"window": 6}})",
      R"({"seqlen_q": 12, "seqlen_k": 16, "slices": [{"q": [0, 6], "k": [0, 16], "type": "causal"}, {"q": [2, 12], "k": [3, 9], "type": "bi_causal"}, {"q": [4, 12], "k": [1, 16], "type": "inv_causal"}]})",
  };
  for (const char* sp : specs) {
    const AttnMask m = parse_mask_spec(sp);
    json e;
    e["spec"] = json::parse(sp);
    e["json"] = mask_spec(m);
    e["area_union"] = mask_area(m, AreaCounting::UNION);
    e["area_multiplicity"] = mask_area(m, AreaCounting::MULTIPLICITY);
    if (m.seqlen_q <= 1024) e["row_counts"] = per_row_union_counts(m);
    if (m.seqlen_q <= 128 && m.seqlen_k <= 128) e["ascii"] = render_ascii(m);
    named.push_back(e);
  }
  g["named_masks"] = named;

  // ---- random masks: union areas, row counts, restrict_rows
  json rmasks = json::array();
  for (int i = 0; i < 60; ++i) {
    const TokenIndex s = 1 + static_cast<TokenIndex>(rng() % 64);
    const AttnMask m = random_mask(rng, s, 6);
    json e;
    e["mask"] = mask_spec(m);
    e["area_union"] = mask_area(m, AreaCounting::UNION);
    e["area_multiplicity"] = mask_area(m, AreaCounting::MULTIPLICITY);
    e["row_counts"] = per_row_union_counts(m);
    std::vector<TokenRange> rows;
    TokenIndex at = 0;
    while (at < s) {
      const TokenIndex len = 1 + static_cast<TokenIndex>(rng() % 8);
      const TokenIndex end = std::min(s, at + len);
      if (rng() % 2) rows.push_back({at, end});
      at = end;
    }
    json jr = json::array();
    for (auto it = rows.rbegin(); it != rows.rend(); ++it) jr.push_back({it->start, it->end});
    std::vector<TokenRange> rev(rows.rbegin(), rows.rend());
    e["rows"] = jr;
    e["restricted"] = mask_spec(restrict_rows(m, rev));
    rmasks.push_back(e);
  }
  g["random_masks"] = rmasks;

  // ---- dispatch on area vectors
  json disp = json::array();
  for (int i = 0; i < 200; ++i) {
    const RankIndex cp = 1 + static_cast<RankIndex>(rng() % 8);
    const int per = 1 + static_cast<int>(rng() % 4);
    const bool twice = rng() % 2;
    const int n = cp * per * (twice ? 2 : 1);
    std::vector<DispatchChunk> chunks;
    json ja = json::array();
    for (int c = 0; c < n; ++c) {
      const PairCount a = static_cast<PairCount>(rng() % (i % 3 == 0 ? 5 : 1000));
      chunks.push_back({c, {c, c + 1}, a});
      ja.push_back(a);
    }
    json e;
    e["areas"] = ja;
    e["cp"] = cp;
    const auto gp = greedy_dispatch(chunks, cp);
    e["greedy"] = {{"assignment", gp.assignment}, {"workloads", gp.bucket_workloads}};
    if (n % (2 * cp) == 0) {
      const auto zp = zigzag_dispatch(chunks, cp);
      e["zigzag"] = {{"assignment", zp.assignment}, {"workloads", zp.bucket_workloads}};
    }
    if (n <= 12 && cp <= 4) {
      const auto bp = brute_force_dispatch(chunks, cp);
      e["brute_force"] = {{"assignment", bp.assignment}, {"workloads", bp.bucket_workloads}};
    }
    disp.push_back(e);
  }
  g["dispatch"] = disp;

  // ---- shard + demands + tables on random square masks
  json dem = json::array();
  for (int i = 0; i < 80; ++i) {
    const RankIndex cp = 1 + static_cast<RankIndex>(rng() % 8);
    const TokenIndex cs = 1 + static_cast<TokenIndex>(rng() % 4);
    const int per = 1 + static_cast<int>(rng() % 4);
    const TokenIndex s = cp * per * cs;
    const AttnMask m = random_mask(rng, s, 6);
    const auto chunks = shard_into_chunks(m, cs);
    const auto plan = greedy_dispatch(chunks, cp);
    const auto d = compute_kv_demands(m, plan);
    const auto [cast, reduce] = build_transfer_tables(d, cs, cp);
    const auto rr = redundancy_report(m, plan);
    json e;
    e["mask"] = mask_spec(m);
    e["chunk"] = cs;
    e["cp"] = cp;
    json areas_j = json::array();
    for (const auto& c : chunks) areas_j.push_back(c.area);
    e["chunk_areas"] = areas_j;
    e["assignment"] = plan.assignment;
    json jd = json::array();
    for (const auto& x : d) jd.push_back({x.host_rank, x.consumers});
    e["demands"] = jd;
    e["cast"] = json::parse(transfer_table_to_json(cast, 1));
    e["reduce"] = json::parse(transfer_table_to_json(reduce, 1));
    e["redundancy"] = {rr.sent_ring, rr.needed, rr.sent_group};
    dem.push_back(e);
  }
  g["demands"] = dem;

  // ---- overlap pieces
  json pk = json::array();
  for (int i = 0; i < 100; ++i) {
    std::vector<std::int64_t> tr;
    const int n = static_cast<int>(rng() % 6);
    for (int k = 0; k < n; ++k) tr.push_back(static_cast<std::int64_t>(rng() % 3000));
    const std::int64_t mn = 1 + static_cast<std::int64_t>(rng() % 700);
    const std::int64_t mx = 1 + static_cast<std::int64_t>(rng() % 10);
    pk.push_back({tr, mn, mx, partition_packages(tr, mn, mx)});
  }
  g["partition_packages"] = pk;
  json asg = json::array();
  for (int i = 0; i < 100; ++i) {
    std::vector<std::int64_t> sz;
    const int n = static_cast<int>(rng() % 9);
    for (int k = 0; k < n; ++k) sz.push_back(static_cast<std::int64_t>(rng() % 50));
    const int st = 1 + static_cast<int>(rng() % 5);
    json e = {{"sizes", sz}, {"stages", st}, {"lpt", assign_packages_to_stages(sz, st)}};
    if (i % 4 == 0) {
      e["seed"] = static_cast<std::uint64_t>(i * 7 + 1);
      e["shuffled"] = assign_packages_to_stages(sz, st, static_cast<std::uint64_t>(i * 7 + 1));
    }
    asg.push_back(e);
  }
  g["assign_packages"] = asg;
  json est = json::array();
  for (int i = 0; i < 100; ++i) {
    StageCosts c;
    const int s = 1 + static_cast<int>(rng() % 6);
    c.host_compute = static_cast<CostUnits>(rng() % 100);
    for (int k = 0; k < s; ++k) {
      c.compute.push_back(static_cast<CostUnits>(rng() % 100));
      c.cast.push_back(static_cast<CostUnits>(rng() % 100));
      c.reduce.push_back(static_cast<CostUnits>(rng() % 100));
    }
    est.push_back({{"host", c.host_compute}, {"compute", c.compute}, {"cast", c.cast},
                   {"reduce", c.reduce}, {"fwd", estimate_fwd_cost(c)}, {"bwd", estimate_bwd_cost(c)}});
  }
  g["estimates"] = est;
  json fits = json::array();
  for (int i = 0; i < 20; ++i) {
    std::vector<std::pair<std::int64_t, std::int64_t>> smp;
    const int n = 2 + static_cast<int>(rng() % 6);
    for (int k = 0; k < n; ++k)
      smp.emplace_back(static_cast<std::int64_t>(rng() % 100000), static_cast<std::int64_t>(rng() % 1000));
    const auto f = fit_affine(smp);
    fits.push_back({{"samples", smp}, {"fit", {f.latency, f.per_unit}}});
  }
  g["fit_affine"] = fits;

  // ---- config-4 varlen sample lengths
  std::vector<TokenIndex> lens;
  for (const auto& s : lognormal_stream(200, 2048.0, 1.0, 65536, 42)) lens.push_back(s.length);
  g["lognormal_2048_1.0_65536_seed42"] = lens;

  // ---- FLOPs (sim.cpp:29-34)
  {
    WorkloadSpec w;
    w.num_heads_q = 64;
    w.head_dim = 128;
    const AttnMask full = parse_mask_spec(R"({"seqlen": 4096, "pattern": "full"})");
    g["flops_full4096_h64_d128"] = {flops(full, w, Pass::FWD), flops(full, w, Pass::BWD)};
  }

  // ---- whole scenarios through the reference C ABI
  const std::string cost =
      R"({"ffa_fwd": {"latency": 30, "per_unit": 8.19e-05}, "ffa_bwd": {"latency": 30, "per_unit": 2.05e-04}, "cast": {"latency": 100, "per_unit": 0.082}, "reduce": {"latency": 100, "per_unit": 0.082}})";
  auto scen = [&](const std::string& mask, const std::string& extra) {
    return R"({"workload": {"mask": )" + mask +
           R"(, "batch_size": 1, "num_heads_q": 48, "num_heads_k": 8, "num_heads_v": 8, "head_dim": 128, "dtype_bytes": 2}, "cost_model": )" +
           cost + extra + "}";
  };
  json sc = json::array();
  std::vector<std::string> texts = {
      scen(R"({"seqlen": 8192, "pattern": "causal"})",
           R"(, "schedule": "magi", "cp_size": 4, "dispatch": "zigzag", "dispatch_chunk_size": 1024, "overlap": {"min_chunk_size": 512, "max_num_chunks": 8}, "seed": 0)"),
      scen(R"({"seqlen": 8192, "pattern": "varlen_block_causal_last_global", "params": {"sample_lengths": [4096, 4096], "block_size": 1024}})",
           R"(, "cp_size": 4, "dispatch_chunk_size": 256)"),
      scen(R"({"seqlen": 65536, "pattern": "block_causal", "params": {"block_size": 8192}})",
           R"(, "cp_size": 8)"),
      scen(R"({"seqlen": 32768, "pattern": "block_causal", "params": {"block_size": 4096}})",
           R"(, "cp_size": 1)"),
      scen(R"({"seqlen": 1024, "pattern": "block_causal", "params": {"block_size": 256}})",
           R"(, "cp_size": 2, "seed": 7)"),
      scen(R"({"seqlen": 4096, "pattern": "sliding_window_causal", "params": {"window": 300}})",
           R"(, "cp_size": 4, "overlap": {"min_chunk_size": 128, "max_num_chunks": 6})"),
      scen(R"({"seqlen": 2048, "pattern": "causal"})", R"(, "cp_size": 4, "schedule": "ring")"),
  };
  for (int cp : {2, 4, 8}) {
    texts.push_back(scen(R"({"seqlen": 1048576, "pattern": "block_causal", "params": {"block_size": 8192}})",
                         ", \"cp_size\": " + std::to_string(cp)));
  }
  for (int cp : {1, 2, 4, 8}) {
    texts.push_back(scen("{\"seqlen\": " + std::to_string(131072 * cp) +
                             R"(, "pattern": "block_causal", "params": {"block_size": 8192}})",
                         ", \"cp_size\": " + std::to_string(cp)));
  }
  // baseline schedules (sim.cpp:262-537)
  texts.push_back(scen(R"({"seqlen": 16384, "pattern": "block_causal", "params": {"block_size": 2048}})",
                       R"(, "cp_size": 8, "schedule": "ring")"));
  texts.push_back(scen(R"({"seqlen": 4096, "pattern": "causal"})", R"(, "cp_size": 4, "schedule": "ring_serial")"));
  texts.push_back(scen(R"({"seqlen": 3072, "pattern": "sliding_window_causal", "params": {"window": 500}})",
                       R"(, "cp_size": 3, "schedule": "ring", "dispatch_chunk_size": 128)"));
  texts.push_back(scen(R"({"seqlen": 32768, "pattern": "block_causal", "params": {"block_size": 4096}})",
                       R"(, "cp_size": 8, "schedule": "ulysses")"));
  texts.push_back(scen(R"({"seqlen": 6000, "pattern": "causal"})", R"(, "cp_size": 3, "schedule": "ulysses")"));
  texts.push_back(scen(R"({"seqlen": 6000, "pattern": "causal"})", R"(, "cp_size": 7, "schedule": "ulysses")"));
  for (int nc : {2, 3, 5, 8}) {
    texts.push_back(scen(R"({"seqlen": 32768, "pattern": "block_causal", "params": {"block_size": 4096}})",
                         ", \"cp_size\": 4, \"schedule\": \"cso\", \"cso_num_chunks\": " + std::to_string(nc)));
  }
  texts.push_back(scen(R"({"seqlen": 8192, "pattern": "full"})", R"(, "cp_size": 2, "schedule": "cso", "cso_num_chunks": 1)"));
  texts.push_back(scen(R"({"seqlen": 8190, "pattern": "full"})", R"(, "cp_size": 4, "schedule": "cso")"));
  texts.push_back(R"({"workload": {"mask": {"seqlen": 4096, "pattern": "causal"}, "num_heads_q": 24, "num_heads_k": 8, "num_heads_v": 8, "head_dim": 128}, "cp_size": 2, "schedule": "ulysses"})");
  texts.push_back(scen(R"({"seqlen": 8, "pattern": "full"})", R"(, "cp_size": 3)"));  // constraint error
  texts.push_back(R"({"workload": {"mask": {"seqlen": 8, "pattern": "causal"}}, "bogus": 1})");  // usage
  for (const auto& t : texts) {
    const bool big = t.find("1048576") != std::string::npos;
    json e = {{"scenario", t}, {"plan", capi_plan(t)}};
    if (!big) e["simulate"] = capi_simulate(t);
    sc.push_back(e);
  }
  // a sweep (simulate only)
  const std::string sweep = scen(R"({"seqlen": 8192, "pattern": "full"})",
                                 R"(, "sweep": {"cp_sizes": [1, 2, 4, 8], "per_rank_seqlen": 8192})");
  sc.push_back({{"scenario", sweep}, {"simulate", capi_simulate(sweep)}});
  for (const char* sched : {"ring", "ulysses", "cso"}) {
    const std::string sw = scen(R"({"seqlen": 8192, "pattern": "causal"})",
                                std::string(R"(, "schedule": ")") + sched +
                                    R"(", "sweep": {"cp_sizes": [1, 2, 4, 8], "per_rank_seqlen": 4096})");
    sc.push_back({{"scenario", sw}, {"simulate", capi_simulate(sw)}});
  }
  g["scenarios"] = sc;

  // ---- packer runs through the reference C ABI (pack.cpp, scenario.cpp:428-554)
  json pk_runs = json::array();
  std::vector<std::string> pack_cfgs = {
      R"({"packing": {"max_length": 65536, "bins_per_iteration": 8, "pool_capacity": 64, "dp_size": 4, "cp_size": 8}, "generator": {"count": 2000, "median": 8192, "sigma": 1.0}, "seed": 3})",
      R"({"packing": {"max_length": 32768, "bins_per_iteration": 2, "pool_capacity": 8}, "generator": {"count": 300, "median": 2048, "sigma": 1.0}, "seed": 42, "emit_bins": true})",
      R"({"packing": {"max_length": 16384, "bins_per_iteration": 4, "pool_capacity": 16, "swap_passes": 0, "defer_threshold": 0.9}, "generator": {"count": 500, "median": 6000, "sigma": 1.5}, "seed": 9})",
      R"({"packing": {"max_length": 4096, "bins_per_iteration": 3, "pool_capacity": 12, "defer_threshold": 1.0}, "generator": {"count": 200, "median": 1500, "sigma": 0.7}, "seed": 5, "emit_bins": true})",
      R"({"generator": {"count": 50}, "seed": 1})",
      R"({"packing": {"max_length": 32768, "bins_per_iteration": 2, "pool_capacity": 32}, "generator": {"count": 300, "median": 2048, "sigma": 1.0}, "seed": 42, "emit_bins": true})",
      R"({"packing": {"max_length": 8192, "bins_per_iteration": 4, "pool_capacity": 16, "dp_size": 2}, "generator": {"count": 400, "median": 3000, "sigma": 2.0}, "seed": 11, "emit_bins": true})",
      R"({"packing": {"bins_per_iteration": 3, "dp_size": 2, "pool_capacity": 12}, "generator": {}})",
      R"({"packing": {"max_length": 1000, "tp_size": 3}, "generator": {}})",
      R"({"packing": {"bins_per_iteration": 4, "pool_capacity": 8}, "generator": {}})",
      R"({"packing": {"defer_threshold": 1.5}, "generator": {}})",
      R"({"packing": {"max_length": 0}, "generator": {}})",
      R"({"packing": {"bogus": 1}})",
      R"({"generator": {"count": 10, "mean": 3}})",
      R"({"seed": 1})",
      R"([1, 2])",
      R"({"packing": )",
  };
  for (const auto& c : pack_cfgs) pk_runs.push_back({{"config", c}, {"out", capi_pack(c, nullptr)}});
  std::vector<std::pair<std::string, std::string>> pack_streams = {
      {R"({"packing": {"max_length": 100, "bins_per_iteration": 2, "pool_capacity": 8}, "emit_bins": true})",
       "# id length\n0 60\n1 50\n2 40\n\n3 30\n4 200\n5 0\n6 45\n7 55\n8 10\n9 90\n10 35\n11 65\n12 5\n"},
      {R"({"packing": {"max_length": 100, "bins_per_iteration": 4, "pool_capacity": 16, "defer_threshold": 0.0}, "emit_bins": true})",
       "0 100\n1 1\n2 1\n3 1\n4 1\n5 1\n"},
      {R"({"packing": {"max_length": 10, "bins_per_iteration": 1, "pool_capacity": 4}})",
       "0 11\n1 12\n2 13\n3 14\n4 15\n5 16\n6 17\n7 18\n8 19\n9 20\n10 21\n11 22\n12 23\n13 24\n14 25\n15 26\n16 27\n17 28\n18 29\n19 30\n20 31\n21 32\n22 3\n"},
      {R"({"packing": {"max_length": 100, "bins_per_iteration": 2, "pool_capacity": 8, "defer_threshold": 0.95}})",
       "0 10\n1 10\n2 10\n3 10\n4 10\n5 10\n6 10\n7 10\n8 10\n9 10\n"},
      {R"({"packing": {"max_length": 100}})", "0 20\n1 x\n"},
      {R"({})", ""},
  };
  for (const auto& [c, st] : pack_streams) {
    pk_runs.push_back({{"config", c}, {"stream", st}, {"out", capi_pack(c, st.c_str())}});
  }
  g["pack_runs"] = pk_runs;

  std::ofstream(path) << g.dump() << "\n";
  std::printf("wrote %s\n", path.c_str());
  return 0;
}
