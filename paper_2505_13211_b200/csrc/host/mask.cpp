// Attention-mask metadata (see mask.hpp). Reference semantics:
// /root/reference/proj/src/mask.cpp (row_cols :74-84, slice_area :95-118,
// slice_area_in_cols :120-173, restrict_rows :312-363, named builders
// :421-504, JSON spec :567-636).
#include "mask.hpp"

#include <algorithm>
#include <numeric>

#include <nlohmann/json.hpp>

#include "errors.hpp"

namespace magiplan {

using json = nlohmann::ordered_json;

std::string TokenRange::str() const {
  return "[" + std::to_string(start) + ", " + std::to_string(end) + ")";
}

const char* slice_type_name(SliceType t) {
  switch (t) {
    case SliceType::Full: return "full";
    case SliceType::Causal: return "causal";
    case SliceType::InvCausal: return "inv_causal";
    case SliceType::BiCausal: return "bi_causal";
  }
  throw UsageError("unknown slice type value");
}

SliceType slice_type_from_name(const std::string& name) {
  for (SliceType t : {SliceType::Full, SliceType::Causal, SliceType::InvCausal,
                      SliceType::BiCausal}) {
    if (name == slice_type_name(t)) return t;
  }
  throw UsageError("unknown slice mask type '" + name +
                   "' (expected full|causal|inv_causal|bi_causal)");
}

std::string AttnSlice::str() const {
  return "(q=" + q.str() + ", k=" + k.str() + ", " + slice_type_name(type) + ")";
}

TokenRange AttnSlice::cols(Token row) const {
  if (!q.contains(row)) return {0, 0};
  Token lo = k.start, hi = k.end;
  if (has_lower_diag(type)) lo = std::min(k.end, k.start + (row - q.start));
  if (has_upper_diag(type)) hi = std::clamp(row + (k.end - q.end) + 1, k.start, k.end);
  if (hi <= lo) return {0, 0};
  return {lo, hi};
}

void AttnMask::validate() const {
  if (seqlen_q < 0 || seqlen_k < 0) throw UsageError("mask seqlen must be non-negative");
  for (std::size_t i = 0; i < slices.size(); ++i) {
    const AttnSlice& s = slices[i];
    if (!s.q.valid() || !s.k.valid()) {
      throw UsageError("slice " + std::to_string(i) + ": malformed range " + s.str());
    }
    if (s.q.end > seqlen_q || s.k.end > seqlen_k) {
      throw UsageError("slice " + std::to_string(i) + ": " + s.str() + " exceeds mask bounds " +
                       std::to_string(seqlen_q) + "x" + std::to_string(seqlen_k));
    }
  }
}

namespace {

Pairs tri(Token n) { return n <= 0 ? 0 : n * (n + 1) / 2; }

// A slice region after clipping: rows [a,b) x cols [c,e), optionally cut by
// k - q >= dlo and/or k - q <= dhi.
struct Region {
  Token a, b, c, e;
  bool lower, upper;
  Token dlo, dhi;
};

Region region_of(const AttnSlice& s) {
  return {s.q.start, s.q.end,  s.k.start, s.k.end, has_lower_diag(s.type), has_upper_diag(s.type),
          s.k.start - s.q.start, s.k.end - s.q.end};
}

// Re-express a region as canonical slices (row order). A CAUSAL piece over
// rows [x,y) must have its key range end at y + dhi and an INV_CAUSAL piece
// its key range start at x + dlo, so rows are split where each diagonal
// stops binding against the box edge.
void emit(Region r, std::vector<AttnSlice>& out) {
  if (r.lower && r.upper && r.dlo > r.dhi) return;
  if (r.upper) r.a = std::max(r.a, r.c - r.dhi);
  if (r.lower) r.b = std::min(r.b, r.e - r.dlo);
  if (r.lower) r.c = std::max(r.c, r.a + r.dlo);
  if (r.upper) r.e = std::min(r.e, r.b + r.dhi);
  if (r.a >= r.b || r.c >= r.e) return;
  const Token w = r.lower ? std::clamp(r.c - r.dlo, r.a, r.b) : r.a;  // lower binds on [w, b)
  const Token u = r.upper ? std::clamp(r.e - r.dhi, r.a, r.b) : r.b;  // upper binds on [a, u)
  Token cuts[4] = {r.a, w, u, r.b};
  std::sort(cuts, cuts + 4);
  for (int i = 0; i < 3; ++i) {
    const Token x = cuts[i], y = cuts[i + 1];
    if (x >= y) continue;
    const bool lo_bind = r.lower && x >= w;
    const bool hi_bind = r.upper && y <= u;
    const Token ks = lo_bind ? x + r.dlo : r.c;
    const Token ke = hi_bind ? y + r.dhi : r.e;
    if (ks >= ke) continue;
    SliceType t = SliceType::Full;
    if (lo_bind && hi_bind) t = SliceType::BiCausal;
    else if (lo_bind) t = SliceType::InvCausal;
    else if (hi_bind) t = SliceType::Causal;
    out.push_back({{x, y}, {ks, ke}, t});
  }
}

}  // namespace

Pairs slice_area(const AttnSlice& s) {
  const Token lq = s.q.length(), lk = s.k.length();
  if (lq <= 0 || lk <= 0) return 0;
  switch (s.type) {
    case SliceType::Full: return lq * lk;
    case SliceType::Causal:      // rows r hold max(0, r + lk - lq + 1) columns
    case SliceType::InvCausal:   // rows r hold max(0, lk - r) columns
      return tri(lk) - tri(lk - lq);
    case SliceType::BiCausal: return lk >= lq ? lq * (lk - lq + 1) : 0;
  }
  throw UsageError("unknown slice type value");
}

std::vector<AttnSlice> clip_slice(const AttnSlice& s, TokenRange rows, TokenRange cols) {
  Region r = region_of(s);
  r.a = std::max(r.a, rows.start);
  r.b = std::min(r.b, rows.end);
  r.c = std::max(r.c, cols.start);
  r.e = std::min(r.e, cols.end);
  std::vector<AttnSlice> out;
  emit(r, out);
  return out;
}

Pairs slice_area_in_cols(const AttnSlice& s, Token c0, Token c1) {
  Pairs total = 0;
  for (const AttnSlice& piece : clip_slice(s, s.q, {c0, c1})) total += slice_area(piece);
  return total;
}

bool is_allowed(const AttnMask& m, Token q, Token k) {
  if (q < 0 || q >= m.seqlen_q || k < 0 || k >= m.seqlen_k) {
    throw UsageError("is_allowed(" + std::to_string(q) + ", " + std::to_string(k) +
                     ") out of range for " + std::to_string(m.seqlen_q) + "x" +
                     std::to_string(m.seqlen_k) + " mask");
  }
  return std::any_of(m.slices.begin(), m.slices.end(),
                     [&](const AttnSlice& s) { return s.allows(q, k); });
}

namespace {

// Sort + merge in place; returns the covered column count.
Pairs merge_intervals(std::vector<TokenRange>& iv) {
  if (iv.empty()) return 0;
  std::sort(iv.begin(), iv.end(), [](const TokenRange& x, const TokenRange& y) {
    return x.start != y.start ? x.start < y.start : x.end < y.end;
  });
  std::size_t w = 0;
  for (std::size_t i = 1; i < iv.size(); ++i) {
    if (iv[i].start <= iv[w].end) {
      iv[w].end = std::max(iv[w].end, iv[i].end);
    } else {
      iv[++w] = iv[i];
    }
  }
  iv.resize(w + 1);
  Pairs n = 0;
  for (const auto& r : iv) n += r.length();
  return n;
}

}  // namespace

void visit_row_unions(const AttnMask& m, const RowVisitor& fn) { sweep_row_unions(m, fn); }

std::vector<Pairs> union_row_counts(const AttnMask& m) {
  std::vector<Pairs> counts(static_cast<std::size_t>(std::max<Token>(0, m.seqlen_q)), 0);
  sweep_row_unions(m, [&](Token q, const std::vector<TokenRange>& iv) {
    Pairs n = 0;
    for (const auto& r : iv) n += r.length();
    counts[static_cast<std::size_t>(q)] = n;
  });
  return counts;
}

std::vector<TokenRange> row_union(const AttnMask& m, Token q) {
  if (q < 0 || q >= m.seqlen_q) throw UsageError("row " + std::to_string(q) + " out of range");
  std::vector<TokenRange> iv;
  for (const auto& s : m.slices) {
    const TokenRange c = s.cols(q);
    if (!c.empty()) iv.push_back(c);
  }
  merge_intervals(iv);
  return iv;
}

Pairs mask_area(const AttnMask& m, Counting counting) {
  Pairs total = 0;
  if (counting == Counting::Multiplicity) {
    for (const auto& s : m.slices) total += slice_area(s);
    return total;
  }
  for (Pairs n : union_row_counts(m)) total += n;
  return total;
}

AttnMask restrict_rows(const AttnMask& m, const std::vector<TokenRange>& rows) {
  std::vector<TokenRange> sorted = rows;
  std::stable_sort(sorted.begin(), sorted.end(),
                   [](const TokenRange& x, const TokenRange& y) { return x.start < y.start; });
  for (std::size_t i = 0; i < sorted.size(); ++i) {
    if (!sorted[i].valid() || sorted[i].end > m.seqlen_q) {
      throw ConstraintError("row range " + sorted[i].str() + " outside [0, " +
                            std::to_string(m.seqlen_q) + ")");
    }
    if (i > 0 && sorted[i].start < sorted[i - 1].end) {
      throw ConstraintError("row ranges " + sorted[i - 1].str() + " and " + sorted[i].str() +
                            " overlap");
    }
  }
  AttnMask out{m.seqlen_q, m.seqlen_k, {}};
  for (const TokenRange& r : sorted) {
    if (r.empty()) continue;
    for (const AttnSlice& s : m.slices) {
      const Token a = std::max(r.start, s.q.start), b = std::min(r.end, s.q.end);
      if (a >= b) continue;
      // keep the slice type: a diagonal anchored at a trimmed corner moves the
      // matching key bound by the number of rows trimmed on that side
      AttnSlice c{{a, b}, s.k, s.type};
      if (has_upper_diag(s.type)) c.k.end -= s.q.end - b;
      if (has_lower_diag(s.type)) c.k.start += a - s.q.start;
      if (c.k.end > c.k.start) out.slices.push_back(c);
    }
  }
  return out;
}

const char* pattern_name(Pattern p) {
  switch (p) {
    case Pattern::Full: return "full";
    case Pattern::Causal: return "causal";
    case Pattern::VarlenFull: return "varlen_full";
    case Pattern::VarlenCausal: return "varlen_causal";
    case Pattern::SlidingWindowCausal: return "sliding_window_causal";
    case Pattern::BlockCausal: return "block_causal";
    case Pattern::VarlenBlockCausal: return "varlen_block_causal";
    case Pattern::VarlenBlockCausalLastGlobal: return "varlen_block_causal_last_global";
  }
  throw UsageError("unknown pattern value");
}

Pattern pattern_from_name(const std::string& name) {
  for (int i = 0; i <= static_cast<int>(Pattern::VarlenBlockCausalLastGlobal); ++i) {
    if (name == pattern_name(static_cast<Pattern>(i))) return static_cast<Pattern>(i);
  }
  throw UsageError("unknown mask pattern '" + name + "'");
}

namespace {

std::vector<Token> sample_starts(const PatternSpec& spec) {
  if (spec.sample_lengths.empty()) {
    throw ConstraintError("pattern '" + std::string(pattern_name(spec.pattern)) +
                          "' requires non-empty sample_lengths");
  }
  std::vector<Token> starts;
  Token at = 0;
  for (Token len : spec.sample_lengths) {
    if (len <= 0) throw ConstraintError("sample lengths must be positive");
    starts.push_back(at);
    at += len;
  }
  if (at != spec.seqlen) {
    throw ConstraintError("sample lengths sum to " + std::to_string(at) + " but seqlen is " +
                          std::to_string(spec.seqlen));
  }
  return starts;
}

// MAGI-1 chunk-wise block-causal: query block i attends keys [0, (i+1)*block)
// of its sample, bidirectional inside the block (one FULL slice per block).
void add_block_causal(AttnMask& m, Token offset, Token length, Token block) {
  if (block <= 0) throw ConstraintError("block_size must be positive");
  if (length % block != 0) {
    throw ConstraintError("block_size " + std::to_string(block) + " does not divide sample length " +
                          std::to_string(length));
  }
  for (Token b0 = 0; b0 < length; b0 += block) {
    m.slices.push_back({{offset + b0, offset + b0 + block}, {offset, offset + b0 + block},
                        SliceType::Full});
  }
}

}  // namespace

AttnMask build_pattern(const PatternSpec& spec) {
  if (spec.seqlen <= 0) throw ConstraintError("pattern seqlen must be positive");
  const Token s = spec.seqlen;
  AttnMask m{s, s, {}};
  switch (spec.pattern) {
    case Pattern::Full: m.slices.push_back({{0, s}, {0, s}, SliceType::Full}); break;
    case Pattern::Causal: m.slices.push_back({{0, s}, {0, s}, SliceType::Causal}); break;
    case Pattern::VarlenFull:
    case Pattern::VarlenCausal: {
      const SliceType t = spec.pattern == Pattern::VarlenFull ? SliceType::Full : SliceType::Causal;
      const auto starts = sample_starts(spec);
      for (std::size_t i = 0; i < starts.size(); ++i) {
        const Token o = starts[i], e = o + spec.sample_lengths[i];
        m.slices.push_back({{o, e}, {o, e}, t});
      }
      break;
    }
    case Pattern::SlidingWindowCausal: {
      const Token w = spec.window;
      if (w <= 0) throw ConstraintError("window must be positive");
      if (s <= w) {
        m.slices.push_back({{0, s}, {0, s}, SliceType::Causal});
      } else {
        m.slices.push_back({{0, w}, {0, w}, SliceType::Causal});
        // later rows: BI_CAUSAL over keys [1, s) anchors both bounds on the
        // diagonal, so row q keeps the last w keys up to itself
        m.slices.push_back({{w, s}, {1, s}, SliceType::BiCausal});
      }
      break;
    }
    case Pattern::BlockCausal: add_block_causal(m, 0, s, spec.block_size); break;
    case Pattern::VarlenBlockCausal:
    case Pattern::VarlenBlockCausalLastGlobal: {
      const auto starts = sample_starts(spec);
      for (std::size_t i = 0; i < starts.size(); ++i) {
        add_block_causal(m, starts[i], spec.sample_lengths[i], spec.block_size);
      }
      if (spec.pattern == Pattern::VarlenBlockCausalLastGlobal) {
        const Token last = s - spec.block_size;
        if (last > 0) m.slices.push_back({{0, last}, {last, s}, SliceType::Full});
      }
      break;
    }
  }
  m.validate();
  return m;
}

std::string render_ascii(const AttnMask& m) {
  if (m.seqlen_q > 128 || m.seqlen_k > 128) {
    throw UsageError("ascii rendering is limited to seqlen <= 128");
  }
  std::string out;
  visit_row_unions(m, [&](Token, const std::vector<TokenRange>& iv) {
    std::string line(static_cast<std::size_t>(m.seqlen_k), '.');
    for (const auto& r : iv) {
      std::fill(line.begin() + r.start, line.begin() + r.end, '#');
    }
    out += line;
    out += '\n';
  });
  return out;
}

namespace {

json parse_or_usage(const std::string& text, const char* what) {
  try {
    return json::parse(text);
  } catch (const nlohmann::json::exception& e) {
    throw UsageError(std::string(what) + ": " + e.what());
  }
}

void only_keys(const json& obj, std::initializer_list<const char*> allowed,
               const std::string& context) {
  for (const auto& [key, value] : obj.items()) {
    if (std::none_of(allowed.begin(), allowed.end(), [&](const char* a) { return key == a; })) {
      throw UsageError("unknown field '" + key + "' in " + context);
    }
  }
}

Token int_field(const json& j, const char* key) {
  if (!j.contains(key) || !j[key].is_number_integer()) {
    throw UsageError(std::string("missing or non-integer field '") + key + "'");
  }
  return j[key].get<Token>();
}

TokenRange range_field(const json& j, const char* key, std::size_t idx) {
  if (!j.contains(key) || !j[key].is_array() || j[key].size() != 2) {
    throw UsageError("slice " + std::to_string(idx) + ": field '" + key +
                     "' must be a [start, end) pair");
  }
  try {
    return {j[key][0].get<Token>(), j[key][1].get<Token>()};
  } catch (const nlohmann::json::exception& e) {
    throw UsageError("slice " + std::to_string(idx) + ": " + e.what());
  }
}

}  // namespace

AttnMask parse_mask_spec(const std::string& text) {
  const json j = parse_or_usage(text, "mask spec");
  if (!j.is_object()) throw UsageError("mask spec must be a JSON object");
  try {
    if (j.contains("slices")) {
      only_keys(j, {"seqlen", "seqlen_q", "seqlen_k", "slices"}, "mask spec");
      AttnMask m;
      if (j.contains("seqlen")) {
        m.seqlen_q = m.seqlen_k = int_field(j, "seqlen");
      } else {
        m.seqlen_q = int_field(j, "seqlen_q");
        m.seqlen_k = int_field(j, "seqlen_k");
      }
      if (!j["slices"].is_array()) throw UsageError("'slices' must be an array");
      std::size_t idx = 0;
      for (const auto& js : j["slices"]) {
        only_keys(js, {"q", "k", "type"}, "slice " + std::to_string(idx));
        AttnSlice s;
        s.q = range_field(js, "q", idx);
        s.k = range_field(js, "k", idx);
        s.type = js.contains("type") ? slice_type_from_name(js["type"].get<std::string>())
                                     : SliceType::Full;
        m.slices.push_back(s);
        ++idx;
      }
      m.validate();
      return m;
    }
    if (!j.contains("pattern")) throw UsageError("mask spec needs either 'pattern' or 'slices'");
    only_keys(j, {"seqlen", "pattern", "params"}, "mask spec");
    PatternSpec spec;
    spec.pattern = pattern_from_name(j["pattern"].get<std::string>());
    spec.seqlen = int_field(j, "seqlen");
    if (j.contains("params")) {
      const auto& p = j["params"];
      only_keys(p, {"sample_lengths", "block_size", "window"}, "mask params");
      if (p.contains("sample_lengths")) spec.sample_lengths = p["sample_lengths"].get<std::vector<Token>>();
      if (p.contains("block_size")) spec.block_size = p["block_size"].get<Token>();
      if (p.contains("window")) spec.window = p["window"].get<Token>();
    }
    return build_pattern(spec);
  } catch (const nlohmann::json::exception& e) {
    throw UsageError(std::string("mask spec: ") + e.what());
  }
}

std::string mask_to_json(const AttnMask& m) {
  json j;
  j["seqlen_q"] = m.seqlen_q;
  j["seqlen_k"] = m.seqlen_k;
  j["slices"] = json::array();
  for (const auto& s : m.slices) {
    json js;
    js["q"] = {s.q.start, s.q.end};
    js["k"] = {s.k.start, s.k.end};
    js["type"] = slice_type_name(s.type);
    j["slices"].push_back(js);
  }
  return j.dump();
}

}  // namespace magiplan
