// Zero-redundant GroupCast / GroupReduce planning. Reference surface:
// /root/reference/proj/include/magiplan/comm.hpp:29-87.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "dispatch.hpp"

namespace magiplan {

// Key/value chunk `kv_chunk` lives on `host_rank` (co-hosted with the same
// query chunk) and is needed by `consumers` (sorted, never the host).
struct KvDemand {
  int64_t kv_chunk = 0;
  Rank host_rank = 0;
  std::vector<Rank> consumers;
};

enum class Direction { GroupCast, GroupReduce };

struct TransferEntry {
  TokenRange tokens;
  std::vector<Rank> dest_ranks;  // sorted, non-empty
};

struct TransferTable {
  Direction direction = Direction::GroupCast;
  Rank cp_size = 1;
  std::vector<std::vector<TransferEntry>> entries;  // per source rank, by token start

  int64_t total_token_transfers() const;
  int64_t send_tokens_of_rank(Rank r) const;
  int64_t recv_tokens_of_rank(Rank r) const;
  // ranges arriving at `r`, ordered by (source rank, token start)
  std::vector<TokenRange> incoming_ranges_of_rank(Rank r) const;
  // the same, with the source rank of each range
  std::vector<std::pair<Rank, TokenRange>> incoming_of_rank(Rank r) const;
};

struct RedundancyReport {
  int64_t sent_ring = 0;
  int64_t needed = 0;
  int64_t sent_group = 0;
  double redundancy_ratio = 0.0;
};

std::vector<KvDemand> compute_kv_demands(const AttnMask& m, const DispatchPlan& plan);
std::pair<TransferTable, TransferTable> build_transfer_tables(const std::vector<KvDemand>& demands,
                                                              Token chunk_size, Rank cp_size);
int64_t ring_baseline_volume(const DispatchPlan& plan);
RedundancyReport redundancy_report(const std::vector<KvDemand>& demands, const DispatchPlan& plan);
RedundancyReport redundancy_report(const AttnMask& m, const DispatchPlan& plan);
std::string transfer_table_to_json(const TransferTable& t, int64_t bytes_per_token);

}  // namespace magiplan
