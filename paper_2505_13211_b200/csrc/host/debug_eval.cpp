// JSON-RPC access to individual planner functions (magiplan_debug_eval), so
// the parity tests can replay the reference's golden vectors function by
// function. Request: {"op": name, ...args}; response: JSON value.
#include <nlohmann/json.hpp>

#include "errors.hpp"
#include "ffa_plan.hpp"
#include "scenario.hpp"

namespace magiplan {

using json = nlohmann::ordered_json;

namespace {

AttnSlice slice_of(const json& s) {
  return {{s[0].get<Token>(), s[1].get<Token>()}, {s[2].get<Token>(), s[3].get<Token>()},
          static_cast<SliceType>(s[4].get<int>())};
}

json slice_json(const AttnSlice& s) {
  return json::array({s.q.start, s.q.end, s.k.start, s.k.end, static_cast<int>(s.type)});
}

AttnMask mask_of(const json& j) { return parse_mask_spec(j.dump()); }

std::vector<DispatchChunk> chunks_of(const json& areas) {
  std::vector<DispatchChunk> c;
  int64_t i = 0;
  for (const auto& a : areas) {
    c.push_back({i, {i, i + 1}, a.get<Pairs>()});
    ++i;
  }
  return c;
}

json plan_json(const DispatchPlan& p) {
  return {{"assignment", p.assignment}, {"workloads", p.bucket_workloads}};
}

DispatchPlan plan_of(const json& r) {
  DispatchPlan p;
  p.cp_size = r["cp"].get<Rank>();
  p.chunk_size = r["chunk"].get<Token>();
  p.assignment = r["assignment"].get<std::vector<Rank>>();
  p.bucket_workloads.assign(static_cast<std::size_t>(p.cp_size), 0);
  return p;
}

}  // namespace

std::string debug_eval(const std::string& request) {
  json r;
  try {
    r = json::parse(request);
  } catch (const nlohmann::json::exception& e) {
    throw UsageError(std::string("debug request: ") + e.what());
  }
  const std::string op = r.value("op", "");
  json out;
  if (op == "slice_area") {
    out = slice_area(slice_of(r["slice"]));
  } else if (op == "slice_area_in_cols") {
    out = slice_area_in_cols(slice_of(r["slice"]), r["cols"][0].get<Token>(), r["cols"][1].get<Token>());
  } else if (op == "clip_slice") {
    out = json::array();
    for (const auto& p : clip_slice(slice_of(r["slice"]), {r["rows"][0].get<Token>(), r["rows"][1].get<Token>()},
                                    {r["cols"][0].get<Token>(), r["cols"][1].get<Token>()}))
      out.push_back(slice_json(p));
  } else if (op == "chunk_pair_slices") {
    // slices of the mask between the query rows of chunk list `q_chunks` and
    // the key columns of chunk list `k_chunks` (chunk = `chunk` tokens), in the
    // local coordinates of buffers that hold those chunks back to back in list
    // order: the ring-attention baseline's per-(rank, source) work
    const AttnMask m = mask_of(r["mask"]);
    const Token cs = r["chunk"].get<Token>();
    const auto qc = r["q_chunks"].get<std::vector<int64_t>>();
    const auto kc = r["k_chunks"].get<std::vector<int64_t>>();
    out = json::array();
    for (std::size_t i = 0; i < qc.size(); ++i) {
      const TokenRange rows{qc[i] * cs, (qc[i] + 1) * cs};
      for (std::size_t j = 0; j < kc.size(); ++j) {
        const TokenRange cols{kc[j] * cs, (kc[j] + 1) * cs};
        for (const auto& sl : m.slices) {
          for (const auto& pc : clip_slice(sl, rows, cols)) {
            const Token dq = static_cast<Token>(i) * cs - rows.start;
            const Token dk = static_cast<Token>(j) * cs - cols.start;
            out.push_back(json::array({pc.q.start + dq, pc.q.end + dq, pc.k.start + dk, pc.k.end + dk,
                                       static_cast<int>(pc.type)}));
          }
        }
      }
    }
  } else if (op == "mask") {
    const AttnMask m = mask_of(r["mask"]);
    out["json"] = json::parse(mask_to_json(m));
    out["area_union"] = mask_area(m, Counting::Union);
    out["area_multiplicity"] = mask_area(m, Counting::Multiplicity);
    if (r.value("rows", false)) out["row_counts"] = union_row_counts(m);
  } else if (op == "restrict_rows") {
    std::vector<TokenRange> rows;
    for (const auto& x : r["rows"]) rows.push_back({x[0].get<Token>(), x[1].get<Token>()});
    out = json::parse(mask_to_json(restrict_rows(mask_of(r["mask"]), rows)));
  } else if (op == "shard") {
    out = json::array();
    for (const auto& c : shard_into_chunks(mask_of(r["mask"]), r["chunk"].get<Token>())) out.push_back(c.area);
  } else if (op == "greedy" || op == "zigzag" || op == "brute_force") {
    const auto ch = chunks_of(r["areas"]);
    const Rank cp = r["cp"].get<Rank>();
    out = plan_json(op == "greedy" ? greedy_dispatch(ch, cp)
                                   : op == "zigzag" ? zigzag_dispatch(ch, cp) : brute_force_dispatch(ch, cp));
  } else if (op == "demands") {
    const DispatchPlan p = plan_of(r);
    const auto d = compute_kv_demands(mask_of(r["mask"]), p);
    json jd = json::array();
    for (const auto& x : d) jd.push_back({x.host_rank, x.consumers});
    const auto [cast, reduce] = build_transfer_tables(d, p.chunk_size, p.cp_size);
    out["demands"] = jd;
    out["cast"] = json::parse(transfer_table_to_json(cast, 1));
    out["reduce"] = json::parse(transfer_table_to_json(reduce, 1));
    const auto rr = redundancy_report(d, p);
    out["redundancy"] = {rr.sent_ring, rr.needed, rr.sent_group};
  } else if (op == "partition_packages") {
    out = partition_packages(r["traffic"].get<std::vector<int64_t>>(), r["min"].get<int64_t>(),
                             r["max"].get<int64_t>());
  } else if (op == "assign_packages") {
    std::optional<uint64_t> seed;
    if (r.contains("seed")) seed = r["seed"].get<uint64_t>();
    out = assign_packages_to_stages(r["sizes"].get<std::vector<int64_t>>(), r["stages"].get<int>(), seed);
  } else if (op == "estimate") {
    StageCosts c;
    c.host_compute = r["host"].get<Cost>();
    c.compute = r["compute"].get<std::vector<Cost>>();
    c.cast = r["cast"].get<std::vector<Cost>>();
    c.reduce = r["reduce"].get<std::vector<Cost>>();
    out = {estimate_fwd_cost(c), estimate_bwd_cost(c)};
  } else if (op == "fit_affine") {
    const auto f = fit_affine(r["samples"].get<std::vector<std::pair<int64_t, int64_t>>>());
    out = {f.latency, f.per_unit};
  } else if (op == "lognormal") {
    out = lognormal_lengths(r["count"].get<std::size_t>(), r["median"].get<double>(),
                            r["sigma"].get<double>(), r["max_length"].get<Token>(),
                            r["seed"].get<uint64_t>());
  } else if (op == "ffa_worklists") {
    // host-side FFA work lists of a slice list (no device involved)
    FfaPlan plan;
    plan.seqlen_q = r["seqlen_q"].get<int64_t>();
    plan.seqlen_k = r["seqlen_k"].get<int64_t>();
    plan.head_dim = r.value("head_dim", 128);
    for (const auto& s : r["slices"]) {
      plan.slices.push_back({s[0].get<int32_t>(), s[1].get<int32_t>(), s[2].get<int32_t>(),
                             s[3].get<int32_t>(), s[4].get<int32_t>()});
    }
    build_ffa_worklists(plan);
    auto qmajor = [](const std::vector<magi::FwdTile>& tiles, const std::vector<magi::FwdItem>& items) {
      json out = json::array();
      for (const auto& t : tiles) {
        json jt = {{"q0", t.q0}, {"n_ktiles", t.n_ktiles}, {"items", json::array()}};
        for (int i = t.item_begin; i < t.item_end; ++i) {
          const auto& it = items[static_cast<std::size_t>(i)];
          jt["items"].push_back({it.qs, it.qe, it.ks, it.ke, it.type, it.k_begin, it.n_ktiles});
        }
        out.push_back(jt);
      }
      return out;
    };
    out["fwd128"] = qmajor(plan.fwd_tiles, plan.fwd_items);
    out["fwd256"] = qmajor(plan.fwd2_tiles, plan.fwd2_items);
    out["bwd"] = json::array();
    for (const auto& t : plan.bwd_tiles) {
      json jt = {{"k0", t.k0}, {"n_qtiles", t.n_qtiles}, {"items", json::array()}};
      for (int i = t.item_begin; i < t.item_end; ++i) {
        const auto& it = plan.bwd_items[static_cast<std::size_t>(i)];
        jt["items"].push_back({it.qs, it.qe, it.ks, it.ke, it.type, it.q_begin, it.n_qtiles});
      }
      out["bwd"].push_back(jt);
    }
    out["area_multiplicity"] = plan.area_multiplicity;
  } else if (op == "flops") {
    WorkloadSpec w;
    w.num_heads_q = r["num_heads_q"].get<int64_t>();
    w.head_dim = r["head_dim"].get<int64_t>();
    w.batch_size = r.value("batch_size", int64_t{1});
    const AttnMask m = mask_of(r["mask"]);
    out = {flops(m, w, Pass::Fwd), flops(m, w, Pass::Bwd)};
  } else {
    throw UsageError("unknown debug op '" + op + "'");
  }
  return out.dump();
}

}  // namespace magiplan
