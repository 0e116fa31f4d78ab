// Online packing-and-padding packer and its JSON driver (magiplan_pack_run).
// Reference semantics: /root/reference/proj/src/pack.cpp:30-271 and
// /root/reference/proj/src/scenario.cpp:428-554; the report is byte-identical
// to the reference library's (tests/test_planner_parity.py, pack cases).
#include "pack.hpp"

#include <algorithm>
#include <numeric>
#include <sstream>

#include <nlohmann/json.hpp>

#include "errors.hpp"
#include "scenario.hpp"

namespace magiplan {

using json = nlohmann::ordered_json;

// pack.cpp:30-55 (same checks, same order, same messages)
void PackingConfig::check_valid() const {
  if (max_length <= 0 || dp_size <= 0 || tp_size <= 0 || cp_size <= 0 || bins_per_iteration <= 0 ||
      pool_capacity <= 0) {
    throw UsageError("packing config fields must be positive");
  }
  if (bins_per_iteration % dp_size != 0) {
    throw ConstraintError("constraint violated: N % dp_size = 0 (N " + std::to_string(bins_per_iteration) +
                          ", dp_size " + std::to_string(dp_size) + ")");
  }
  if (max_length % (tp_size * cp_size) != 0) {
    throw ConstraintError("constraint violated: max_length % (tp_size * cp_size) = 0 (max_length " +
                          std::to_string(max_length) + ", tp_size " + std::to_string(tp_size) +
                          ", cp_size " + std::to_string(cp_size) + ")");
  }
  if (pool_capacity < 4 * bins_per_iteration) {
    throw ConstraintError("constraint violated: M >= 4N (M " + std::to_string(pool_capacity) + ", N " +
                          std::to_string(bins_per_iteration) + ")");
  }
  if (defer_threshold < 0.0 || defer_threshold > 1.0) {
    throw UsageError("defer_threshold must lie in [0, 1]");
  }
}

Packer::Packer(PackingConfig config) : cfg_(config) { cfg_.check_valid(); }

// pack.cpp:61-72: non-positive or oversized samples are counted and dropped;
// a full pool refuses without counting.
bool Packer::admit(const PackedSample& s) {
  if (s.length <= 0 || s.length > cfg_.max_length) {
    ++rejected_;
    return false;
  }
  if (pool_full()) return false;
  pool_.push_back(s);
  return true;
}

namespace {

// Working state of one iteration: bins hold pool indices.
struct Bins {
  std::vector<std::vector<std::size_t>> members;
  std::vector<Token> fill;
  std::vector<char> placed;
};

// First fit over the length-descending view; equal lengths keep arrival
// order (pack.cpp:80-99).
void first_fit_decreasing(const std::vector<PackedSample>& pool, Token cap, Bins& b) {
  std::vector<std::size_t> order(pool.size());
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::stable_sort(order.begin(), order.end(),
                   [&](std::size_t x, std::size_t y) { return pool[x].length > pool[y].length; });
  for (const std::size_t i : order) {
    const Token len = pool[i].length;
    auto it = std::find_if(b.fill.begin(), b.fill.end(), [&](Token f) { return f + len <= cap; });
    if (it == b.fill.end()) continue;
    const auto bin = static_cast<std::size_t>(it - b.fill.begin());
    b.members[bin].push_back(i);
    *it += len;
    b.placed[i] = 1;
  }
}

// Up to `passes` sweeps over the bins; each bin takes at most one swap per
// sweep, the one with the largest strictly positive fill gain (first slot,
// then first pool index, on ties). Stops at a sweep with no swap
// (pack.cpp:101-133).
void refine_by_swaps(const std::vector<PackedSample>& pool, Token cap, int passes, Bins& b) {
  for (int pass = 0; pass < passes; ++pass) {
    bool any = false;
    for (std::size_t bin = 0; bin < b.members.size(); ++bin) {
      auto& mem = b.members[bin];
      Token gain = 0;
      std::size_t slot_best = 0, in_best = 0;
      for (std::size_t slot = 0; slot < mem.size(); ++slot) {
        const Token out_len = pool[mem[slot]].length;
        const Token room = cap - b.fill[bin] + out_len;  // largest incoming length that fits
        for (std::size_t i = 0; i < pool.size(); ++i) {
          if (b.placed[i]) continue;
          const Token in_len = pool[i].length;
          if (in_len - out_len > gain && in_len <= room) {
            gain = in_len - out_len;
            slot_best = slot;
            in_best = i;
          }
        }
      }
      if (gain <= 0) continue;
      b.placed[mem[slot_best]] = 0;
      b.placed[in_best] = 1;
      mem[slot_best] = in_best;
      b.fill[bin] += gain;
      any = true;
    }
    if (!any) break;
  }
}

// Every bin must carry work for its DP group: while a bin is empty, move the
// shortest sample (first on ties) of the most populated bin (first on ties)
// into the first empty bin, as long as that donor keeps one (pack.cpp:135-163).
void fill_empty_bins(const std::vector<PackedSample>& pool, Bins& b) {
  for (;;) {
    auto empty = std::find_if(b.members.begin(), b.members.end(),
                              [](const std::vector<std::size_t>& m) { return m.empty(); });
    if (empty == b.members.end()) return;
    auto donor = std::max_element(b.members.begin(), b.members.end(),
                                  [](const auto& x, const auto& y) { return x.size() < y.size(); });
    if (donor->size() < 2) return;
    auto shortest = std::min_element(donor->begin(), donor->end(), [&](std::size_t x, std::size_t y) {
      return pool[x].length < pool[y].length;
    });
    const std::size_t moved = *shortest;
    donor->erase(shortest);
    b.fill[static_cast<std::size_t>(donor - b.members.begin())] -= pool[moved].length;
    empty->push_back(moved);
    b.fill[static_cast<std::size_t>(empty - b.members.begin())] += pool[moved].length;
  }
}

}  // namespace

// pack.cpp:74-196. A deferred iteration leaves the pool untouched.
std::optional<PackedBatch> Packer::pack_iteration() {
  const auto n_bins = static_cast<std::size_t>(cfg_.bins_per_iteration);
  if (pool_.size() < n_bins) {
    ++deferred_;
    return std::nullopt;
  }
  Bins b;
  b.members.resize(n_bins);
  b.fill.assign(n_bins, 0);
  b.placed.assign(pool_.size(), 0);
  first_fit_decreasing(pool_, cfg_.max_length, b);
  refine_by_swaps(pool_, cfg_.max_length, cfg_.swap_passes, b);
  fill_empty_bins(pool_, b);

  const Token total = std::accumulate(b.fill.begin(), b.fill.end(), Token{0});
  const double util = static_cast<double>(total) /
                      static_cast<double>(cfg_.bins_per_iteration * cfg_.max_length);
  if (util < cfg_.defer_threshold) {
    ++deferred_;
    return std::nullopt;
  }
  PackedBatch batch;
  batch.utilization = util;
  batch.bins.resize(n_bins);
  for (std::size_t bin = 0; bin < n_bins; ++bin) {
    MAGI_CHECK(b.fill[bin] <= cfg_.max_length, "bin fill exceeds max_length");
    batch.bins[bin].fill = b.fill[bin];
    for (const std::size_t i : b.members[bin]) batch.bins[bin].samples.push_back(pool_[i]);
  }
  std::size_t keep = 0;
  for (std::size_t i = 0; i < pool_.size(); ++i) {
    if (!b.placed[i]) pool_[keep++] = pool_[i];
  }
  pool_.resize(keep);
  return batch;
}

// pack.cpp:198-226
UtilizationStats utilization_stats(const std::vector<PackedBatch>& history, const PackingConfig& config) {
  if (history.empty()) throw UsageError("utilization_stats needs at least one batch");
  UtilizationStats st;
  st.batches = static_cast<int64_t>(history.size());
  st.min_utilization = history.front().utilization;
  std::vector<int64_t> group(static_cast<std::size_t>(config.dp_size), 0);
  double sum = 0.0;
  for (const PackedBatch& batch : history) {
    sum += batch.utilization;
    st.min_utilization = std::min(st.min_utilization, batch.utilization);
    for (std::size_t i = 0; i < batch.bins.size(); ++i) group[i % group.size()] += batch.bins[i].fill;
  }
  st.mean_utilization = sum / static_cast<double>(history.size());
  const auto [lo, hi] = std::minmax_element(group.begin(), group.end());
  const double mean = static_cast<double>(std::accumulate(group.begin(), group.end(), int64_t{0})) /
                      static_cast<double>(config.dp_size);
  st.dp_group_spread = mean > 0.0 ? static_cast<double>(*hi - *lo) / mean : 0.0;
  return st;
}

namespace {

json parse_pack_object(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw UsageError(std::string("pack config: ") + e.what());
  }
  if (!j.is_object()) throw UsageError("pack config must be a JSON object");
  return j;
}

void allow_only(const json& obj, std::initializer_list<const char*> allowed, const char* ctx) {
  for (const auto& [key, value] : obj.items()) {
    if (std::none_of(allowed.begin(), allowed.end(), [&](const char* a) { return key == a; })) {
      throw UsageError("unknown field '" + key + "' in " + ctx);
    }
  }
}

template <typename T>
void take(const json& j, const char* key, T& slot) {
  if (j.contains(key)) slot = j[key].get<T>();
}

// "id length" records, one per line; blank lines and '#' comments skipped.
std::vector<PackedSample> parse_stream(const std::string& text) {
  std::vector<PackedSample> out;
  std::istringstream in(text);
  std::string line;
  int64_t line_no = 0;
  while (std::getline(in, line)) {
    ++line_no;
    if (line.empty() || line[0] == '#') continue;
    std::istringstream fields(line);
    PackedSample s;
    if (!(fields >> s.id >> s.length)) {
      throw UsageError("stream line " + std::to_string(line_no) + ": expected 'id length'");
    }
    out.push_back(s);
  }
  return out;
}

}  // namespace

// scenario.cpp:428-554
std::string run_pack(const std::string& config_json, const std::string* stream_text) {
  const json j = parse_pack_object(config_json);
  allow_only(j, {"schema_version", "packing", "generator", "seed", "emit_bins"}, "pack config");
  PackingConfig cfg;
  if (j.contains("packing")) {
    const json& p = j["packing"];
    allow_only(p,
               {"max_length", "dp_size", "tp_size", "cp_size", "bins_per_iteration", "pool_capacity",
                "defer_threshold", "swap_passes"},
               "packing config");
    take(p, "max_length", cfg.max_length);
    take(p, "dp_size", cfg.dp_size);
    take(p, "tp_size", cfg.tp_size);
    take(p, "cp_size", cfg.cp_size);
    take(p, "bins_per_iteration", cfg.bins_per_iteration);
    take(p, "pool_capacity", cfg.pool_capacity);
    take(p, "defer_threshold", cfg.defer_threshold);
    take(p, "swap_passes", cfg.swap_passes);
  }
  cfg.check_valid();
  uint64_t seed = 0;
  take(j, "seed", seed);
  bool emit_bins = false;
  take(j, "emit_bins", emit_bins);

  std::vector<PackedSample> stream;
  if (stream_text != nullptr) {
    stream = parse_stream(*stream_text);
  } else {
    if (!j.contains("generator")) throw UsageError("pack config needs a generator or an input stream");
    const json& g = j["generator"];
    allow_only(g, {"count", "median", "sigma"}, "generator config");
    std::size_t count = 10000;
    double median = 8192.0, sigma = 1.0;
    take(g, "count", count);
    take(g, "median", median);
    take(g, "sigma", sigma);
    const std::vector<Token> lens = lognormal_lengths(count, median, sigma, cfg.max_length, seed);
    stream.reserve(lens.size());
    for (std::size_t i = 0; i < lens.size(); ++i) stream.push_back({static_cast<int64_t>(i), lens[i]});
  }

  // Refill the pool to capacity, pack; a deferral with the stream drained
  // ends the run, one with a full pool is a terminal stall ("starved").
  Packer packer(cfg);
  std::vector<PackedBatch> history;
  std::vector<int64_t> skipped_ids;
  std::size_t next = 0;
  bool starved = false;
  for (;;) {
    for (; !packer.pool_full() && next < stream.size(); ++next) {
      if (!packer.admit(stream[next]) && skipped_ids.size() < 20) skipped_ids.push_back(stream[next].id);
    }
    std::optional<PackedBatch> batch = packer.pack_iteration();
    if (!batch) {
      if (next >= stream.size()) break;
      if (packer.pool_full()) {
        starved = true;
        break;
      }
      continue;
    }
    history.push_back(std::move(*batch));
    if (next >= stream.size() && static_cast<int64_t>(packer.pool_size()) < cfg.bins_per_iteration) break;
  }

  json out;
  out["schema_version"] = kSchemaVersion;
  out["spec_hash"] = hash_hex(fnv1a_hash(config_json));
  out["seed"] = seed;
  out["samples_in"] = stream.size();
  std::size_t packed = 0;
  json batches = json::array();
  for (const PackedBatch& batch : history) {
    json jb;
    jb["utilization"] = batch.utilization;
    json fills = json::array();
    for (const PackedBin& bin : batch.bins) {
      fills.push_back(bin.fill);
      packed += bin.samples.size();
    }
    jb["fills"] = fills;
    if (emit_bins) {
      json bins = json::array();
      for (const PackedBin& bin : batch.bins) {
        json jbin;
        jbin["fill"] = bin.fill;
        json samples = json::array();
        for (const PackedSample& s : bin.samples) samples.push_back({{"id", s.id}, {"length", s.length}});
        jbin["samples"] = samples;
        bins.push_back(jbin);
      }
      jb["bins"] = bins;
    }
    batches.push_back(jb);
  }
  out["batches"] = batches;
  out["samples_packed"] = packed;
  out["samples_left"] = packer.pool_size() + (stream.size() - next);
  out["skipped_oversized"] = packer.rejected_oversized();
  out["skipped_ids"] = skipped_ids;
  out["deferred_iterations"] = packer.deferred_iterations();
  out["starved"] = starved;
  if (!history.empty()) {
    const UtilizationStats st = utilization_stats(history, cfg);
    out["stats"] = {{"batches", st.batches},
                    {"mean_utilization", st.mean_utilization},
                    {"min_utilization", st.min_utilization},
                    {"dp_group_spread", st.dp_group_spread}};
  }
  return out.dump();
}

}  // namespace magiplan
