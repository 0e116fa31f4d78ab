// Attention-mask metadata: token ranges, AttnSlice compositions and their
// pair counting. Semantics follow the reference operator API
// (/root/reference/proj/include/magiplan/mask.hpp:32-166); the implementation
// is a from-scratch region algebra.
//
// Every slice is treated as a region in global coordinates
//     box [qs,qe) x [ks,ke)  ∩  {k - q >= ks - qs}  (INV_CAUSAL / BI_CAUSAL)
//                            ∩  {k - q <= ke - qe}  (CAUSAL / BI_CAUSAL)
// i.e. a box cut by at most two diagonals anchored at the top-left and
// bottom-right corners (reference slice shapes, mask.hpp:46-52). Row and column
// clipping are box intersections followed by re-emission as canonical slices,
// which is what the context-parallel executor needs to re-express a rank's
// local mask against each stage's received key/value ranges.
#pragma once

#include <cstdint>
#include <algorithm>
#include <functional>
#include <limits>
#include <optional>
#include <string>
#include <vector>

namespace magiplan {

using Token = int64_t;
using Pairs = int64_t;
using Rank = int32_t;

struct TokenRange {
  Token start = 0;
  Token end = 0;
  Token length() const { return end - start; }
  bool empty() const { return end <= start; }
  bool valid() const { return 0 <= start && start <= end; }
  bool contains(Token t) const { return start <= t && t < end; }
  bool operator==(const TokenRange&) const = default;
  std::string str() const;
};

enum class SliceType : int32_t { Full = 0, Causal = 1, InvCausal = 2, BiCausal = 3 };

const char* slice_type_name(SliceType t);
SliceType slice_type_from_name(const std::string& name);

inline bool has_upper_diag(SliceType t) { return t == SliceType::Causal || t == SliceType::BiCausal; }
inline bool has_lower_diag(SliceType t) { return t == SliceType::InvCausal || t == SliceType::BiCausal; }

struct AttnSlice {
  TokenRange q;
  TokenRange k;
  SliceType type = SliceType::Full;

  bool operator==(const AttnSlice&) const = default;
  // Allowed global key columns of global query row `row` (empty if none).
  TokenRange cols(Token row) const;
  bool allows(Token row, Token col) const { return cols(row).contains(col); }
  std::string str() const;
};

struct AttnMask {
  Token seqlen_q = 0;
  Token seqlen_k = 0;
  std::vector<AttnSlice> slices;
  // UsageError naming the first offending slice (reference mask.cpp:175-191).
  void validate() const;
};

enum class Counting { Multiplicity, Union };

Pairs slice_area(const AttnSlice& s);
// Pairs of `s` whose key column lies in [c0, c1).
Pairs slice_area_in_cols(const AttnSlice& s, Token c0, Token c1);
Pairs mask_area(const AttnMask& m, Counting counting);
bool is_allowed(const AttnMask& m, Token q, Token k);

// Region clipping. Each returns canonical slices covering exactly the pairs
// of `s` inside the box, in row order; empty regions produce nothing.
std::vector<AttnSlice> clip_slice(const AttnSlice& s, TokenRange rows, TokenRange cols);

// The reference's row restriction (mask.hpp:110-114): per row range (sorted
// by start; overlapping ranges are a ConstraintError), every slice clipped to
// the range with its diagonal anchors preserved by trimming its key range.
AttnMask restrict_rows(const AttnMask& m, const std::vector<TokenRange>& rows);

// Visit every query row's merged allowed column intervals, in row order.
using RowVisitor = std::function<void(Token, const std::vector<TokenRange>&)>;
void visit_row_unions(const AttnMask& m, const RowVisitor& fn);

// Inline form of the same sweep for the hot planner loops (no per-row
// indirect call; the live-slice set is only pruned when a slice ends).
template <class F>
void sweep_row_unions(const AttnMask& m, F&& fn) {
  std::vector<std::size_t> order(m.slices.size());
  for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](std::size_t x, std::size_t y) {
    return m.slices[x].q.start < m.slices[y].q.start;
  });
  std::vector<std::size_t> live;
  std::vector<TokenRange> iv;
  std::size_t next = 0;
  Token first_end = std::numeric_limits<Token>::max();  // smallest q.end among live slices
  for (Token q = 0; q < m.seqlen_q; ++q) {
    for (; next < order.size() && m.slices[order[next]].q.start <= q; ++next) {
      const AttnSlice& s = m.slices[order[next]];
      if (s.q.end > q) {
        live.push_back(order[next]);
        first_end = std::min(first_end, s.q.end);
      }
    }
    if (q >= first_end) {
      std::erase_if(live, [&](std::size_t i) { return m.slices[i].q.end <= q; });
      first_end = std::numeric_limits<Token>::max();
      for (std::size_t i : live) first_end = std::min(first_end, m.slices[i].q.end);
    }
    iv.clear();
    for (std::size_t i : live) {
      const TokenRange c = m.slices[i].cols(q);
      if (!c.empty()) iv.push_back(c);
    }
    if (iv.size() > 1) {
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
    }
    fn(q, iv);
  }
}
std::vector<Pairs> union_row_counts(const AttnMask& m);
std::vector<TokenRange> row_union(const AttnMask& m, Token q);

enum class Pattern {
  Full,
  Causal,
  VarlenFull,
  VarlenCausal,
  SlidingWindowCausal,
  BlockCausal,
  VarlenBlockCausal,
  VarlenBlockCausalLastGlobal,
};
const char* pattern_name(Pattern p);
Pattern pattern_from_name(const std::string& name);

struct PatternSpec {
  Pattern pattern = Pattern::Full;
  Token seqlen = 0;
  std::vector<Token> sample_lengths;
  Token block_size = 0;
  Token window = 0;
};

AttnMask build_pattern(const PatternSpec& spec);
std::string render_ascii(const AttnMask& m);
AttnMask parse_mask_spec(const std::string& json_text);
std::string mask_to_json(const AttnMask& m);

}  // namespace magiplan
