// Schedule models of the CP baselines MagiAttention is compared against:
// ring attention (overlapped and serial), DeepSpeed-Ulysses all-to-all, and
// the context-shuffle overlap (cso) of the MAGI-1 inference path.
// Reference semantics: /root/reference/proj/src/sim.cpp (ring :262-343,
// Ulysses :345-424, cso :426-537). Durations come from the same affine cost
// model as `magi`; records are byte-identical to the reference library's
// (tests/test_planner_parity.py, scenario cases).
#include <cmath>
#include <string>

#include "dispatch.hpp"
#include "errors.hpp"
#include "sim.hpp"

namespace magiplan {

namespace {

std::size_t u(int64_t i) { return static_cast<std::size_t>(i); }

// pairs[i][j]: rank i's query rows (its local mask) against the key columns
// bucket j hosts.
std::vector<std::vector<Pairs>> ring_pairs(const AttnMask& m, const DispatchPlan& plan) {
  const Rank cp = plan.cp_size;
  std::vector<std::vector<TokenRange>> cols(u(cp));
  for (Rank j = 0; j < cp; ++j) cols[u(j)] = plan.rows_of_bucket(j);
  std::vector<std::vector<Pairs>> pairs(u(cp), std::vector<Pairs>(u(cp), 0));
  for (Rank i = 0; i < cp; ++i) {
    const AttnMask local = local_mask_of_rank(m, plan, i);
    for (Rank j = 0; j < cp; ++j) {
      Pairs n = 0;
      for (const TokenRange& c : cols[u(j)]) {
        for (const AttnSlice& s : local.slices) n += slice_area_in_cols(s, c.start, c.end);
      }
      pairs[u(i)][u(j)] = n;
    }
  }
  return pairs;
}

// Round t: rank i attends to the KV shard (i - t) mod cp, which arrived from
// rank i-1's round t-1 send; it forwards the shard on in the same round (after
// its attention when not overlapped). Backward hops carry KV plus partial dKV.
SimReport ring_pass(const AttnMask& m, const DispatchPlan& plan, const CostModel& model,
                    const WorkloadSpec& w, bool overlap, Pass pass,
                    const std::vector<std::vector<Pairs>>& pairs) {
  const Rank cp = plan.cp_size;
  const int64_t shard = static_cast<int64_t>(plan.assignment.size()) / cp * plan.chunk_size;
  const int64_t payload = pass == Pass::Fwd ? shard : 2 * shard;
  const AffineCost& attn = pass == Pass::Fwd ? model.ffa_fwd : model.ffa_bwd;
  Timeline tl;
  std::vector<int> sent(u(cp), -1);  // previous round's send task per rank
  for (Rank t = 0; t < cp; ++t) {
    auto arrival = [&](Rank i) {
      return t >= 1 ? std::vector<int>{sent[u((i - 1 + cp) % cp)]} : std::vector<int>{};
    };
    std::vector<int> attn_task(u(cp));
    for (Rank i = 0; i < cp; ++i) {
      const Rank src = (i - t + cp) % cp;
      attn_task[u(i)] = tl.add(i, Timeline::kCompute, attn.eval(pairs[u(i)][u(src)]), arrival(i),
                               "ffa(shard " + std::to_string(src) + ")");
    }
    if (t == cp - 1) break;
    std::vector<int> next(u(cp));
    for (Rank i = 0; i < cp; ++i) {
      std::vector<int> deps = arrival(i);
      if (!overlap) deps.push_back(attn_task[u(i)]);
      next[u(i)] = tl.add(i, Timeline::kComm, model.cast_cost.eval(payload), std::move(deps),
                          "send(round " + std::to_string(t) + ")");
    }
    sent = std::move(next);
  }
  return finish_report(overlap ? "ring" : "ring_serial", pass, cp, tl, flops(m, w, pass),
                       cp * (cp - 1) * payload);
}

// Per all-to-all volume in KV-token units: the cast cost is calibrated per KV
// token, so q/o moves are rescaled by their byte ratio.
struct A2ATokens {
  int64_t v = 0, k = 0, q = 0, o = 0;
};

A2ATokens a2a_tokens(const AttnMask& m, const WorkloadSpec& w, Rank cp) {
  const double moved = static_cast<double>(m.seqlen_q / cp) * static_cast<double>(cp - 1) /
                       static_cast<double>(cp);
  const double unit = static_cast<double>(w.kv_bytes_per_token());
  const double hd = static_cast<double>(w.head_dim * w.dtype_bytes);
  auto scaled = [&](int64_t heads) {
    return static_cast<int64_t>(std::llround(moved * static_cast<double>(heads) * hd / unit));
  };
  A2ATokens t;
  t.v = scaled(w.num_heads_v);
  t.k = scaled(w.num_heads_k);
  t.q = scaled(w.num_heads_q);
  t.o = t.q;
  return t;
}

void require_divisible(const AttnMask& m, Rank cp) {
  if (cp < 1 || m.seqlen_q % cp != 0) {
    throw ConstraintError("constraint violated: seqlen % cp_size = 0 (seqlen " + std::to_string(m.seqlen_q) +
                          ", cp_size " + std::to_string(cp) + ")");
  }
}

Pairs pairs_per_rank(const AttnMask& m, Rank cp) {
  return static_cast<Pairs>(
      std::llround(static_cast<double>(mask_area(m, Counting::Multiplicity)) / static_cast<double>(cp)));
}

std::vector<int64_t> split_evenly(int64_t total, int parts) {
  std::vector<int64_t> out(u(parts), total / parts);
  for (int i = 0; i < total % parts; ++i) ++out[u(i)];
  return out;
}

}  // namespace

std::pair<SimReport, SimReport> simulate_ring(const AttnMask& m, const DispatchPlan& plan,
                                              const CostModel& model, const WorkloadSpec& w,
                                              bool overlap) {
  const auto pairs = ring_pairs(m, plan);
  return {ring_pass(m, plan, model, w, overlap, Pass::Fwd, pairs),
          ring_pass(m, plan, model, w, overlap, Pass::Bwd, pairs)};
}

// Forward only. Per rank: each projection's all-to-all overlaps the next
// projection; attention waits for the three all-to-alls; the output
// all-to-all overlaps cross-attention.
SimReport simulate_ulysses(const AttnMask& m, const WorkloadSpec& w, const CostModel& model, Rank cp) {
  require_divisible(m, cp);
  const Token local = m.seqlen_q / cp;
  const A2ATokens a2a = a2a_tokens(m, w, cp);
  const Pairs rank_pairs = pairs_per_rank(m, cp);
  Timeline tl;
  for (Rank r = 0; r < cp; ++r) {
    const int cv = tl.add(r, Timeline::kCompute, model.v_proj.eval(local), {}, "v-compute");
    const int mv = tl.add(r, Timeline::kComm, model.cast_cost.eval(a2a.v), {cv}, "v-comm");
    const int ck = tl.add(r, Timeline::kCompute, model.k_proj.eval(local), {}, "k-compute");
    const int mk = tl.add(r, Timeline::kComm, model.cast_cost.eval(a2a.k), {ck}, "k-comm");
    const int cq = tl.add(r, Timeline::kCompute, model.q_proj.eval(local), {}, "q-compute");
    const int mq = tl.add(r, Timeline::kComm, model.cast_cost.eval(a2a.q), {cq}, "q-comm");
    tl.add(r, Timeline::kCompute, model.kv_cache_update.eval(local), {}, "kv-cache-update");
    const int ca = tl.add(r, Timeline::kCompute, model.ffa_fwd.eval(rank_pairs), {mv, mk, mq}, "attention");
    tl.add(r, Timeline::kComm, model.cast_cost.eval(a2a.o), {ca}, "o-comm");
    tl.add(r, Timeline::kCompute, model.cross_attn.eval(local), {}, "cross-attention");
  }
  return finish_report("ulysses", Pass::Fwd, cp, tl, flops(m, w, Pass::Fwd),
                       cp * (a2a.v + a2a.k + a2a.q + a2a.o),
                       {"v-comm || k-compute", "k-comm || q-compute", "q-comm || kv-cache-update",
                        "o-comm || cross-attention"});
}

// Forward only. The q all-to-all and the attention are cut into num_chunks
// pieces so that q-comm(t+1), o-comm(t-1) and o-compute(t) share a step; each
// step is a barrier for the next. The event log records rank 0's steps.
SimReport simulate_cso(const AttnMask& m, const WorkloadSpec& w, const CostModel& model, Rank cp,
                       int num_chunks) {
  if (num_chunks < 2) throw UsageError("context-shuffle overlap needs at least 2 chunks");
  require_divisible(m, cp);
  const Token local = m.seqlen_q / cp;
  const A2ATokens a2a = a2a_tokens(m, w, cp);
  const int64_t kv = a2a.v + a2a.k;
  const auto qc = split_evenly(a2a.q, num_chunks);
  const auto oc = split_evenly(a2a.o, num_chunks);
  const auto ac = split_evenly(pairs_per_rank(m, cp), num_chunks);
  const std::string n = std::to_string(num_chunks);
  auto s = [](int i) { return std::to_string(i); };

  std::vector<std::string> log;
  Timeline tl;
  for (Rank r = 0; r < cp; ++r) {
    std::vector<int> prev;
    auto step = [&](std::vector<int> tasks, std::string line) {
      prev = std::move(tasks);
      if (r == 0) log.push_back(std::move(line));
    };
    auto comm = [&](int64_t tokens, const std::string& label) {
      return tl.add(r, Timeline::kComm, model.cast_cost.eval(tokens), prev, label);
    };
    auto compute = [&](Cost d, const std::string& label) { return tl.add(r, Timeline::kCompute, d, prev, label); };

    const int cv = tl.add(r, Timeline::kCompute, model.v_proj.eval(local), {}, "v-compute");
    const int ck = tl.add(r, Timeline::kCompute, model.k_proj.eval(local), {cv}, "k-compute");
    const int mkv = tl.add(r, Timeline::kComm, model.cast_cost.eval(kv), {ck}, "kv-comm");
    const int cq = tl.add(r, Timeline::kCompute, model.q_proj.eval(local), {}, "q-compute");
    step({mkv, cq}, "kv-comm(all) || q-compute(all)");
    {
      const int a = comm(qc[0], "q-comm(1)");
      const int b = compute(model.kv_cache_update.eval(local), "kv-cache-update");
      step({a, b}, "q-comm(1) || kv-cache-update");
    }
    for (int t = 2; t <= num_chunks; ++t) {
      std::vector<int> tasks{comm(qc[u(t - 1)], "q-comm(" + s(t) + ")")};
      std::string line = "q-comm(" + s(t) + ")";
      if (t >= 3) {
        tasks.push_back(comm(oc[u(t - 3)], "o-comm(" + s(t - 2) + ")"));
        line += " + o-comm(" + s(t - 2) + ")";
      }
      tasks.push_back(compute(model.ffa_fwd.eval(ac[u(t - 2)]), "o-compute(" + s(t - 1) + ")"));
      step(std::move(tasks), line + " || o-compute(" + s(t - 1) + ")");
    }
    {
      const int a = comm(oc[u(num_chunks - 2)], "o-comm(" + s(num_chunks - 1) + ")");
      const int b = compute(model.ffa_fwd.eval(ac[u(num_chunks - 1)]), "o-compute(" + n + ")");
      step({a, b}, "o-comm(" + s(num_chunks - 1) + ") || o-compute(" + n + ")");
    }
    {
      const int a = comm(oc[u(num_chunks - 1)], "o-comm(" + n + ")");
      const int b = compute(model.cross_attn.eval(local), "cross-attention");
      step({a, b}, "o-comm(" + n + ") || cross-attention");
    }
  }
  return finish_report("cso", Pass::Fwd, cp, tl, flops(m, w, Pass::Fwd), cp * (kv + a2a.q + a2a.o),
                       std::move(log));
}

}  // namespace magiplan
