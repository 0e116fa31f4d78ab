// GroupCast / GroupReduce planning. Reference semantics:
// /root/reference/proj/src/comm.cpp (demands :71-111, tables :113-170,
// ring volume :172-176, redundancy :178-196, JSON :198-225).
#include "comm.hpp"

#include <algorithm>

#include <nlohmann/json.hpp>

#include "errors.hpp"

namespace magiplan {

namespace {
bool has_dest(const TransferEntry& e, Rank r) {
  return std::binary_search(e.dest_ranks.begin(), e.dest_ranks.end(), r);
}
}  // namespace

int64_t TransferTable::total_token_transfers() const {
  int64_t n = 0;
  for (const auto& src : entries)
    for (const auto& e : src) n += e.tokens.length() * static_cast<int64_t>(e.dest_ranks.size());
  return n;
}

int64_t TransferTable::send_tokens_of_rank(Rank r) const {
  int64_t n = 0;
  for (const auto& e : entries[static_cast<std::size_t>(r)])
    n += e.tokens.length() * static_cast<int64_t>(e.dest_ranks.size());
  return n;
}

int64_t TransferTable::recv_tokens_of_rank(Rank r) const {
  int64_t n = 0;
  for (const auto& src : entries)
    for (const auto& e : src)
      if (has_dest(e, r)) n += e.tokens.length();
  return n;
}

std::vector<std::pair<Rank, TokenRange>> TransferTable::incoming_of_rank(Rank r) const {
  std::vector<std::pair<Rank, TokenRange>> out;
  for (std::size_t s = 0; s < entries.size(); ++s)
    for (const auto& e : entries[s])
      if (has_dest(e, r)) out.emplace_back(static_cast<Rank>(s), e.tokens);
  return out;
}

std::vector<TokenRange> TransferTable::incoming_ranges_of_rank(Rank r) const {
  std::vector<TokenRange> out;
  for (const auto& [src, range] : incoming_of_rank(r)) out.push_back(range);
  return out;
}

std::vector<KvDemand> compute_kv_demands(const AttnMask& m, const DispatchPlan& plan) {
  const int64_t n = static_cast<int64_t>(plan.assignment.size());
  if (n * plan.chunk_size != m.seqlen_q || m.seqlen_q != m.seqlen_k) {
    throw UsageError("plan covers " + std::to_string(n * plan.chunk_size) + " tokens but mask is " +
                     std::to_string(m.seqlen_q) + "x" + std::to_string(m.seqlen_k));
  }
  const Token cs = plan.chunk_size;
  const std::size_t cp = static_cast<std::size_t>(plan.cp_size);
  const std::size_t stride = static_cast<std::size_t>(n) + 1;
  // cover[owner * (n+1) + kc]: difference array of the kv-chunk intervals the
  // owner's rows attend (O(1) per row interval instead of O(chunks))
  std::vector<int64_t> cover(cp * stride, 0);
  sweep_row_unions(m, [&](Token q, const std::vector<TokenRange>& iv) {
    const auto owner = static_cast<std::size_t>(plan.assignment[static_cast<std::size_t>(q / cs)]);
    for (const TokenRange& r : iv) {
      cover[owner * stride + static_cast<std::size_t>(r.start / cs)] += 1;
      cover[owner * stride + static_cast<std::size_t>((r.end - 1) / cs) + 1] -= 1;
    }
  });
  // need[kc * cp + r]: rank r owns a row attending a column of kv chunk kc
  std::vector<uint8_t> need(static_cast<std::size_t>(n) * cp, 0);
  for (std::size_t r = 0; r < cp; ++r) {
    int64_t run = 0;
    for (int64_t kc = 0; kc < n; ++kc) {
      run += cover[r * stride + static_cast<std::size_t>(kc)];
      if (run > 0) need[static_cast<std::size_t>(kc) * cp + r] = 1;
    }
  }
  std::vector<KvDemand> out(static_cast<std::size_t>(n));
  for (int64_t kc = 0; kc < n; ++kc) {
    KvDemand& d = out[static_cast<std::size_t>(kc)];
    d.kv_chunk = kc;
    d.host_rank = plan.assignment[static_cast<std::size_t>(kc)];
    for (std::size_t r = 0; r < cp; ++r) {
      if (static_cast<Rank>(r) != d.host_rank && need[static_cast<std::size_t>(kc) * cp + r]) {
        d.consumers.push_back(static_cast<Rank>(r));
      }
    }
  }
  return out;
}

namespace {
// append, merging with the previous entry when contiguous with equal destinations
void push_coalesced(std::vector<TransferEntry>& list, const TransferEntry& e) {
  if (!list.empty() && list.back().tokens.end == e.tokens.start &&
      list.back().dest_ranks == e.dest_ranks) {
    list.back().tokens.end = e.tokens.end;
  } else {
    list.push_back(e);
  }
}
}  // namespace

std::pair<TransferTable, TransferTable> build_transfer_tables(const std::vector<KvDemand>& demands,
                                                              Token chunk_size, Rank cp_size) {
  TransferTable cast{Direction::GroupCast, cp_size, {}};
  TransferTable reduce{Direction::GroupReduce, cp_size, {}};
  cast.entries.resize(static_cast<std::size_t>(cp_size));
  reduce.entries.resize(static_cast<std::size_t>(cp_size));
  for (const KvDemand& d : demands) {
    if (d.consumers.empty()) continue;
    push_coalesced(cast.entries[static_cast<std::size_t>(d.host_rank)],
                   {{d.kv_chunk * chunk_size, (d.kv_chunk + 1) * chunk_size}, d.consumers});
  }
  // transpose: every consumer returns the same range to its host
  for (Rank dst = 0; dst < cp_size; ++dst) {
    std::vector<TransferEntry> back;
    for (Rank src = 0; src < cp_size; ++src)
      for (const auto& e : cast.entries[static_cast<std::size_t>(src)])
        if (has_dest(e, dst)) back.push_back({e.tokens, {src}});
    std::sort(back.begin(), back.end(), [](const TransferEntry& a, const TransferEntry& b) {
      return a.tokens.start < b.tokens.start;
    });
    for (const auto& e : back) push_coalesced(reduce.entries[static_cast<std::size_t>(dst)], e);
  }
  MAGI_CHECK(cast.total_token_transfers() == reduce.total_token_transfers(),
             "group-reduce volume must equal group-cast volume");
  return {std::move(cast), std::move(reduce)};
}

int64_t ring_baseline_volume(const DispatchPlan& plan) {
  return static_cast<int64_t>(plan.cp_size - 1) * static_cast<int64_t>(plan.assignment.size()) *
         plan.chunk_size;
}

RedundancyReport redundancy_report(const std::vector<KvDemand>& demands, const DispatchPlan& plan) {
  RedundancyReport r;
  r.sent_ring = ring_baseline_volume(plan);
  for (const auto& d : demands) r.needed += plan.chunk_size * static_cast<int64_t>(d.consumers.size());
  r.sent_group = r.needed;
  r.redundancy_ratio = r.sent_ring == 0 ? 0.0
                                        : static_cast<double>(r.sent_ring - r.needed) /
                                              static_cast<double>(r.sent_ring);
  MAGI_CHECK(r.sent_ring >= r.needed, "ring volume below demand volume");
  return r;
}

RedundancyReport redundancy_report(const AttnMask& m, const DispatchPlan& plan) {
  return redundancy_report(compute_kv_demands(m, plan), plan);
}

std::string transfer_table_to_json(const TransferTable& t, int64_t bytes_per_token) {
  nlohmann::ordered_json j;
  j["direction"] = t.direction == Direction::GroupCast ? "group_cast" : "group_reduce";
  j["cp_size"] = t.cp_size;
  j["bytes_per_token"] = bytes_per_token;
  j["sources"] = nlohmann::ordered_json::array();
  for (Rank s = 0; s < t.cp_size; ++s) {
    nlohmann::ordered_json js;
    js["rank"] = s;
    js["entries"] = nlohmann::ordered_json::array();
    for (const auto& e : t.entries[static_cast<std::size_t>(s)]) {
      nlohmann::ordered_json je;
      je["tokens"] = {e.tokens.start, e.tokens.end};
      je["dest_ranks"] = e.dest_ranks;
      je["bytes"] = e.tokens.length() * bytes_per_token * static_cast<int64_t>(e.dest_ranks.size());
      js["entries"].push_back(je);
    }
    js["send_tokens"] = t.send_tokens_of_rank(s);
    js["recv_tokens"] = t.recv_tokens_of_rank(s);
    j["sources"].push_back(js);
  }
  j["total_token_transfers"] = t.total_token_transfers();
  return j.dump();
}

}  // namespace magiplan
