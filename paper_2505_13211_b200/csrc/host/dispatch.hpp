// Dispatch solver (paper Alg. 1): query chunking and chunk -> rank
// assignment. Reference surface: /root/reference/proj/include/magiplan/dispatch.hpp:28-80.
#pragma once

#include <string>
#include <vector>

#include "mask.hpp"

namespace magiplan {

struct DispatchChunk {
  int64_t index = 0;
  TokenRange rows;
  Pairs area = 0;  // distinct allowed pairs with the query in `rows`
};

struct DispatchPlan {
  Rank cp_size = 1;
  Token chunk_size = 0;
  std::vector<Rank> assignment;          // chunk -> rank
  std::vector<Pairs> bucket_workloads;   // per rank

  Pairs max_workload() const;
  std::vector<std::vector<int64_t>> chunks_of_buckets() const;
  std::vector<TokenRange> rows_of_bucket(Rank bucket) const;  // chunk order
  void validate() const;  // logic_error on a malformed plan
};

std::vector<DispatchChunk> shard_into_chunks(const AttnMask& m, Token chunk_size);
DispatchPlan greedy_dispatch(const std::vector<DispatchChunk>& chunks, Rank cp_size);
DispatchPlan brute_force_dispatch(const std::vector<DispatchChunk>& chunks, Rank cp_size);
DispatchPlan zigzag_dispatch(const std::vector<DispatchChunk>& chunks, Rank cp_size);
AttnMask local_mask_of_rank(const AttnMask& m, const DispatchPlan& plan, Rank rank);
Token default_dispatch_chunk_size(Token seqlen_q, Rank cp_size);
std::string plan_to_json(const DispatchPlan& plan);

}  // namespace magiplan
