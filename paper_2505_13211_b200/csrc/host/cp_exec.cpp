// Context-parallel executor behind the C ABI (magiplan_cp_*): the same
// schedule as paper_2505_13211_b200/cp.py, for C / C++ consumers that hold
// no Python. The plan is the planner's executor view
// (magiplan_scenario_exec_plan, i.e. the reference's simulate_magi schedule,
// /root/reference/proj/src/sim.cpp:193-248):
//   forward  step j:  GroupCast(j+1) || FFA(j) with the LSE merge
//   backward step j:  GroupCast(j+1) || FFA(j) || GroupReduce(j-1), final
//                     GroupReduce exposed.
// GroupCast = range gather + grouped NCCL send/recv on the cast
// communicator; GroupReduce = grouped send/recv of the f32 partial dK/dV on
// a second communicator (so the two exchanges do not queue behind each
// other) + one scatter-add per source rank in rank order
// (deterministic). Communication runs on two high-priority streams.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): the planner and
// the kernels of this library do not depend on it.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "capi_util.hpp"
#include "errors.hpp"
#include "ffa_plan.hpp"
#include "mask.hpp"
#include "scenario.hpp"

namespace magi {
cudaError_t launch_ffa_fwd(const FwdWork& work, int seqlen_q, int seqlen_k,
                           int hq, int hk, int head_dim, float softmax_scale, const void* q, const void* k,
                           const void* v, void* out, float* lse, int out_f32, int accumulate, cudaStream_t stream);
cudaError_t launch_ffa_bwd_preprocess(const void* out, const void* grad_out, float* delta, int64_t seqlen,
                                      int64_t heads, int head_dim, int out_f32, cudaStream_t stream);
cudaError_t launch_range_gather(const void* src, void* dst, const int64_t* ranges, const int64_t* offsets,
                                int64_t num_ranges, int64_t total_rows, int64_t row_bytes, cudaStream_t stream);
cudaError_t launch_range_scatter_add_f32(const float* src, float* dst, const int64_t* ranges,
                                         const int64_t* offsets, int64_t num_ranges, int64_t total_rows,
                                         int64_t row_elems, cudaStream_t stream);
cudaError_t launch_cast_f32_bf16(const float* src, void* dst, int64_t n, cudaStream_t stream);
}  // namespace magi

struct magiplan_ffa_plan {
  magiplan::FfaPlan plan;
};
struct magiplan_scenario {
  magiplan::ScenarioSpec spec;
};

// the stage backward of capi_device.cpp (dQ accumulated, fresh dK / dV)
extern "C" magiplan_status magiplan_ffa_bwd_stage(const magiplan_ffa_plan* plan, const void* q, const void* k,
                                                  const void* v, const float* lse, const float* delta,
                                                  const void* grad_out, float* grad_q, float* grad_k,
                                                  float* grad_v, int64_t num_heads_q, int64_t num_heads_k,
                                                  float softmax_scale, void* cuda_stream);
extern "C" magiplan_status magiplan_ffa_bwd(const magiplan_ffa_plan* plan, const void* q, const void* k,
                                            const void* v, const float* lse, const float* delta,
                                            const void* grad_out, void* grad_q, void* grad_k, void* grad_v,
                                            int64_t num_heads_q, int64_t num_heads_k, float softmax_scale,
                                            int32_t grad_dtype, int32_t accumulate, void* cuda_stream);

namespace magiplan {
namespace {

using json = nlohmann::json;
using capi::cuda_check;

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclUniqueId {
  char internal[128];
};
using ncclComm_t = void*;
enum { kNcclInt8 = 0 };

struct Nccl {
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

const Nccl& nccl() {
  static Nccl lib;
  static std::once_flag once;
  static std::string error;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      error = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    lib.GetUniqueId = reinterpret_cast<decltype(lib.GetUniqueId)>(sym("ncclGetUniqueId"));
    lib.CommInitRank = reinterpret_cast<decltype(lib.CommInitRank)>(sym("ncclCommInitRank"));
    lib.CommDestroy = reinterpret_cast<decltype(lib.CommDestroy)>(sym("ncclCommDestroy"));
    lib.CommSplit = reinterpret_cast<decltype(lib.CommSplit)>(sym("ncclCommSplit"));
    lib.GroupStart = reinterpret_cast<decltype(lib.GroupStart)>(sym("ncclGroupStart"));
    lib.GroupEnd = reinterpret_cast<decltype(lib.GroupEnd)>(sym("ncclGroupEnd"));
    lib.Send = reinterpret_cast<decltype(lib.Send)>(sym("ncclSend"));
    lib.Recv = reinterpret_cast<decltype(lib.Recv)>(sym("ncclRecv"));
    lib.GetErrorString = reinterpret_cast<decltype(lib.GetErrorString)>(sym("ncclGetErrorString"));
    if (!lib.GetUniqueId || !lib.CommInitRank || !lib.CommSplit || !lib.Send || !lib.Recv || !lib.GroupStart ||
        !lib.GroupEnd)
      error = "NCCL library lacks the point-to-point / split API (needs NCCL >= 2.18)";
  });
  if (!error.empty()) throw DeviceError(error);
  return lib;
}

void nccl_check(int r, const char* what) {
  if (r != 0) {
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw DeviceError(std::string(what) + ": NCCL error " + std::to_string(r) + " (" + msg + ")");
  }
}

template <typename T>
T* device_copy(const std::vector<T>& host) {
  if (host.empty()) return nullptr;
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, host.size() * sizeof(T)), "cp executor upload");
  cuda_check(cudaMemcpy(p, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice), "cp executor upload");
  return static_cast<T*>(p);
}

// ---------------------------------------------------------------- plan view
struct RangeList {  // ranges of local rows + packed offsets, on the device
  int64_t n = 0, rows = 0;
  int64_t* d_ranges = nullptr;
  int64_t* d_offsets = nullptr;
  RangeList() = default;
  RangeList(const RangeList&) = delete;
  RangeList& operator=(const RangeList&) = delete;
  void set(const std::vector<std::pair<int64_t, int64_t>>& rr) {
    std::vector<int64_t> flat, offs;
    for (const auto& [a, b] : rr) {
      flat.push_back(a);
      flat.push_back(b);
      offs.push_back(rows);
      rows += b - a;
    }
    n = static_cast<int64_t>(rr.size());
    d_ranges = device_copy(flat);
    d_offsets = device_copy(offs);
  }
  ~RangeList() {
    cudaFree(d_ranges);
    cudaFree(d_offsets);
  }
};

struct Stage {
  int64_t buf_tokens = 0;
  std::vector<int64_t> recv_splits, send_splits;  // tokens per peer
  std::unique_ptr<RangeList> send;                // all sent rows, grouped by destination
  std::vector<std::unique_ptr<RangeList>> per_dst;
  std::unique_ptr<magiplan_ffa_plan> plan;
};

std::unique_ptr<magiplan_ffa_plan> make_ffa_plan(const json& slices, int64_t sq, int64_t sk, int32_t d,
                                                 bool always = false) {
  if (slices.empty() && !always) return nullptr;
  auto p = std::make_unique<magiplan_ffa_plan>();
  p->plan.seqlen_q = sq;
  p->plan.seqlen_k = sk;
  p->plan.head_dim = d;
  for (const auto& s : slices) {
    p->plan.slices.push_back({s[0].get<int32_t>(), s[1].get<int32_t>(), s[2].get<int32_t>(), s[3].get<int32_t>(),
                              s[4].get<int32_t>()});
  }
  build_ffa_worklists(p->plan);
  ensure_uploaded(p->plan);
  return p;
}

}  // namespace

struct CpExecutor {
  int rank = 0, world = 1;
  int64_t hq = 0, hk = 0;
  int32_t d = 128;
  float scale = 1.f;
  int64_t local_tokens = 0;
  std::string describe;
  std::unique_ptr<magiplan_ffa_plan> host_plan;
  std::vector<Stage> fwd, bwd;
  ncclComm_t cast_comm = nullptr, reduce_comm = nullptr;
  cudaStream_t comm_stream = nullptr, reduce_stream = nullptr;

  ~CpExecutor() {
    if (comm_stream) cudaStreamSynchronize(comm_stream);
    if (reduce_stream) cudaStreamSynchronize(reduce_stream);
    if (cast_comm) nccl().CommDestroy(cast_comm);
    if (reduce_comm) nccl().CommDestroy(reduce_comm);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (reduce_stream) cudaStreamDestroy(reduce_stream);
  }

  size_t kv_row_bytes() const { return static_cast<size_t>(hk) * d * 2; }
  size_t grad_row_bytes() const { return static_cast<size_t>(hk) * d * 4; }

  // grouped send / recv: send[peer] from `src` (peer blocks in rank order,
  // send_splits tokens each), recv[peer] into `dst` (recv_splits)
  void exchange(ncclComm_t comm, const std::vector<int64_t>& send_splits, const std::vector<int64_t>& recv_splits,
                const uint8_t* src, uint8_t* dst, size_t row_bytes, cudaStream_t stream) const {
    const Nccl& n = nccl();
    nccl_check(n.GroupStart(), "ncclGroupStart");
    size_t so = 0, ro = 0;
    for (int peer = 0; peer < world; ++peer) {
      const size_t sb = static_cast<size_t>(send_splits[static_cast<size_t>(peer)]) * row_bytes;
      const size_t rb = static_cast<size_t>(recv_splits[static_cast<size_t>(peer)]) * row_bytes;
      if (sb) nccl_check(n.Send(src + so, sb, kNcclInt8, peer, comm, stream), "ncclSend");
      if (rb) nccl_check(n.Recv(dst + ro, rb, kNcclInt8, peer, comm, stream), "ncclRecv");
      so += sb;
      ro += rb;
    }
    nccl_check(n.GroupEnd(), "ncclGroupEnd");
  }

  struct Cast {
    uint8_t *send_k = nullptr, *send_v = nullptr, *k = nullptr, *v = nullptr;
    cudaEvent_t done = nullptr;
  };

  // GroupCast of one stage on the comm stream (buffers stream-ordered)
  Cast cast(const Stage& st, const void* k, const void* v) const {
    Cast c;
    const size_t rb = kv_row_bytes();
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&c.k), std::max<size_t>(st.buf_tokens * rb, 16), comm_stream),
               "cp cast alloc");
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&c.v), std::max<size_t>(st.buf_tokens * rb, 16), comm_stream),
               "cp cast alloc");
    const size_t sbytes = std::max<size_t>(st.send->rows * rb, 16);
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&c.send_k), sbytes, comm_stream), "cp cast alloc");
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&c.send_v), sbytes, comm_stream), "cp cast alloc");
    if (st.send->rows) {
      cuda_check(magi::launch_range_gather(k, c.send_k, st.send->d_ranges, st.send->d_offsets, st.send->n,
                                           st.send->rows, static_cast<int64_t>(rb), comm_stream),
                 "range_gather");
      cuda_check(magi::launch_range_gather(v, c.send_v, st.send->d_ranges, st.send->d_offsets, st.send->n,
                                           st.send->rows, static_cast<int64_t>(rb), comm_stream),
                 "range_gather");
    }
    exchange(cast_comm, st.send_splits, st.recv_splits, c.send_k, c.k, rb, comm_stream);
    exchange(cast_comm, st.send_splits, st.recv_splits, c.send_v, c.v, rb, comm_stream);
    cuda_check(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming), "cp event");
    cuda_check(cudaEventRecord(c.done, comm_stream), "cp event");
    return c;
  }

  // buffers and events of a cast, released in `stream`'s order (after every
  // use, which that stream has waited for)
  static void release(Cast& c, cudaStream_t stream) {
    for (uint8_t* p : {c.send_k, c.send_v, c.k, c.v})
      if (p) cudaFreeAsync(p, stream);
    if (c.done) cudaEventDestroy(c.done);
    c = Cast{};
  }
};

}  // namespace magiplan

struct magiplan_cp {
  magiplan::CpExecutor ex;
};

using magiplan::UsageError;
using magiplan::capi::cuda_check;
using magiplan::capi::dup_string;
using magiplan::capi::guarded;

namespace {
cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

cudaEvent_t record(cudaStream_t s) {
  cudaEvent_t e;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cp event");
  cuda_check(cudaEventRecord(e, s), "cp event");
  return e;
}
void wait_and_destroy(cudaStream_t s, cudaEvent_t e) {
  cuda_check(cudaStreamWaitEvent(s, e, 0), "cp event wait");
  cudaEventDestroy(e);
}
}  // namespace

extern "C" {

magiplan_status magiplan_cp_unique_id(void* out_id) {
  MAGI_REQUIRE(out_id);
  return guarded([&] {
    magiplan::NcclUniqueId id;
    magiplan::nccl_check(magiplan::nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out_id, &id, sizeof(id));
  });
}

magiplan_status magiplan_cp_create(const magiplan_scenario* scenario, int32_t rank, const void* nccl_unique_id,
                                   int64_t num_heads_q, int64_t num_heads_k, int32_t head_dim, float softmax_scale,
                                   magiplan_cp** out) {
  MAGI_REQUIRE(scenario && nccl_unique_id && out);
  auto* cp = new magiplan_cp;
  const magiplan_status st = guarded([&] {
    using namespace magiplan;
    if (num_heads_q <= 0 || num_heads_k <= 0 || num_heads_q % num_heads_k != 0)
      throw UsageError("num_heads_q must be a positive multiple of num_heads_k");
    if (head_dim != 64 && head_dim != 128) throw UsageError("head_dim must be 64 or 128");
    CpExecutor& ex = cp->ex;
    const auto a = run_plan(scenario->spec, scenario_mask(scenario->spec));
    const json xp = json::parse(exec_plan_to_json(a, scenario->spec));
    ex.world = xp["cp_size"].get<int>();
    if (rank < 0 || rank >= ex.world) throw UsageError("rank outside the scenario's cp_size");
    ex.rank = rank;
    ex.hq = num_heads_q;
    ex.hk = num_heads_k;
    ex.d = head_dim;
    ex.scale = softmax_scale;
    ex.local_tokens = xp["local_tokens"].get<int64_t>();
    const json& me = xp["ranks"][static_cast<size_t>(rank)];
    // always a host plan: one with no slices writes empty rows (O = 0, LSE =
    // -inf) and zero gradients
    ex.host_plan = make_ffa_plan(me["host_slices"], ex.local_tokens, ex.local_tokens, head_dim, true);
    for (const char* key : {"fwd_stages", "bwd_stages"}) {
      auto& stages = std::string(key) == "fwd_stages" ? ex.fwd : ex.bwd;
      size_t n = 0;
      for (const auto& r : xp["ranks"]) n = std::max(n, r[key].size());
      for (size_t j = 0; j < n; ++j) {
        Stage stg;
        stg.recv_splits.assign(static_cast<size_t>(ex.world), 0);
        stg.send_splits.assign(static_cast<size_t>(ex.world), 0);
        const json empty = json::object({{"buf_tokens", 0}, {"recv", json::array()}, {"slices", json::array()}});
        const json& mine = j < me[key].size() ? me[key][j] : empty;
        stg.buf_tokens = mine["buf_tokens"].get<int64_t>();
        for (const auto& rv : mine["recv"])
          stg.recv_splits[rv[0].get<size_t>()] += rv[2].get<int64_t>() - rv[1].get<int64_t>();
        // what this rank sends: every other rank's receive entries whose source is this rank
        std::vector<std::pair<int64_t, int64_t>> all;
        for (int dst = 0; dst < ex.world; ++dst) {
          std::vector<std::pair<int64_t, int64_t>> mine_to_dst;
          const json& other = xp["ranks"][static_cast<size_t>(dst)];
          if (j < other[key].size()) {
            for (const auto& rv : other[key][j]["recv"]) {
              if (rv[0].get<int>() != rank) continue;
              const int64_t len = rv[2].get<int64_t>() - rv[1].get<int64_t>();
              const int64_t src_local = rv[3].get<int64_t>();
              mine_to_dst.emplace_back(src_local, src_local + len);
              stg.send_splits[static_cast<size_t>(dst)] += len;
            }
          }
          all.insert(all.end(), mine_to_dst.begin(), mine_to_dst.end());
          auto rl = std::make_unique<RangeList>();
          rl->set(mine_to_dst);
          stg.per_dst.push_back(std::move(rl));
        }
        stg.send = std::make_unique<RangeList>();
        stg.send->set(all);
        stg.plan = make_ffa_plan(mine["slices"], ex.local_tokens, stg.buf_tokens, head_dim);
        stages.push_back(std::move(stg));
      }
    }
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
    cuda_check(cudaStreamCreateWithPriority(&ex.comm_stream, cudaStreamNonBlocking, hi), "cp stream");
    cuda_check(cudaStreamCreateWithPriority(&ex.reduce_stream, cudaStreamNonBlocking, hi), "cp stream");
    NcclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    const Nccl& n = nccl();
    // the cast communicator from the id, the reduce communicator split off it
    nccl_check(n.CommInitRank(&ex.cast_comm, ex.world, id, rank), "ncclCommInitRank");
    nccl_check(n.CommSplit(ex.cast_comm, 0, rank, &ex.reduce_comm, nullptr), "ncclCommSplit");
    json dj;
    dj["rank"] = rank;
    dj["cp_size"] = ex.world;
    dj["local_tokens"] = ex.local_tokens;
    dj["chunk_size"] = xp["chunk_size"];
    dj["chunks"] = me["chunks"];
    dj["num_stages_fwd"] = xp["num_stages_fwd"];
    dj["num_stages_bwd"] = xp["num_stages_bwd"];
    dj["area_multiplicity"] = xp["area_multiplicity"];
    ex.describe = dj.dump();
  });
  if (st != MAGIPLAN_OK) {
    delete cp;
    return st;
  }
  *out = cp;
  return st;
}

void magiplan_cp_free(magiplan_cp* cp) { delete cp; }

magiplan_status magiplan_cp_describe(const magiplan_cp* cp, char** out_json) {
  MAGI_REQUIRE(cp && out_json);
  return guarded([&] { *out_json = dup_string(cp->ex.describe); });
}

magiplan_status magiplan_cp_forward(magiplan_cp* cp, const void* q, const void* k, const void* v, float* out_f32,
                                    float* lse, void* out_bf16, void* cuda_stream) {
  MAGI_REQUIRE(cp && q && k && v && out_f32 && lse);
  return guarded([&] {
    using namespace magiplan;
    CpExecutor& ex = cp->ex;
    cudaStream_t cur = as_stream(cuda_stream);
    const int64_t L = ex.local_tokens;
    const int hq = static_cast<int>(ex.hq), hk = static_cast<int>(ex.hk);
    wait_and_destroy(ex.comm_stream, record(cur));
    std::vector<CpExecutor::Cast> casts;
    if (!ex.fwd.empty()) casts.push_back(ex.cast(ex.fwd[0], k, v));
    auto ffa = [&](const magiplan_ffa_plan* pl, const void* kk, const void* vv, int acc) {
      const FfaPlan& P = pl->plan;
      cuda_check(magi::launch_ffa_fwd(magiplan::fwd_work(P),
                                      static_cast<int>(P.seqlen_q), static_cast<int>(P.seqlen_k), hq, hk, ex.d,
                                      ex.scale, q, kk, vv, out_f32, lse, 1, acc, cur),
                 "ffa_fwd launch");
    };
    ffa(ex.host_plan.get(), k, v, 0);
    for (size_t j = 0; j < ex.fwd.size(); ++j) {
      // cast(j+1) is issued before FFA(j) consumes cast(j)
      if (j + 1 < ex.fwd.size()) casts.push_back(ex.cast(ex.fwd[j + 1], k, v));
      cuda_check(cudaStreamWaitEvent(cur, casts[j].done, 0), "cp wait cast");
      if (ex.fwd[j].plan) ffa(ex.fwd[j].plan.get(), casts[j].k, casts[j].v, 1);
    }
    if (out_bf16)
      cuda_check(magi::launch_cast_f32_bf16(out_f32, out_bf16, L * ex.hq * ex.d, cur), "cast launch");
    for (auto& c : casts) CpExecutor::release(c, cur);
  });
}

magiplan_status magiplan_cp_backward(magiplan_cp* cp, const void* q, const void* k, const void* v,
                                     const float* out_f32, const float* lse, const void* dout, void* dq,
                                     void* dk, void* dv, void* cuda_stream) {
  MAGI_REQUIRE(cp && q && k && v && out_f32 && lse && dout && dq && dk && dv);
  return guarded([&] {
    using namespace magiplan;
    CpExecutor& ex = cp->ex;
    cudaStream_t cur = as_stream(cuda_stream);
    const int64_t L = ex.local_tokens, hq = ex.hq, hk = ex.hk, d = ex.d;
    const size_t gq = static_cast<size_t>(L) * hq * d, gk = static_cast<size_t>(L) * hk * d;
    float *delta = nullptr, *dq32 = nullptr, *dk32 = nullptr, *dv32 = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&delta), std::max<size_t>(hq * L * 4, 16), cur), "alloc");
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&dq32), std::max<size_t>(gq * 4, 16), cur), "alloc");
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&dk32), std::max<size_t>(gk * 4, 16), cur), "alloc");
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&dv32), std::max<size_t>(gk * 4, 16), cur), "alloc");
    wait_and_destroy(ex.comm_stream, record(cur));
    std::vector<CpExecutor::Cast> casts;
    if (!ex.bwd.empty()) casts.push_back(ex.cast(ex.bwd[0], k, v));
    cuda_check(magi::launch_ffa_bwd_preprocess(out_f32, dout, delta, L, hq, static_cast<int>(d), 1, cur),
               "preprocess launch");
    {
      const magiplan_status s = magiplan_ffa_bwd(ex.host_plan.get(), q, k, v, lse, delta, dout, dq32, dk32, dv32,
                                                 hq, hk, ex.scale, MAGIPLAN_F32, 0, cur);
      if (s != MAGIPLAN_OK) throw DeviceError(magiplan_last_error());
    }
    // dk / dv initialised before any scatter-add of the reduce stream
    wait_and_destroy(ex.reduce_stream, record(cur));
    std::vector<void*> partials, recvs;
    const size_t grb = ex.grad_row_bytes();
    for (size_t j = 0; j < ex.bwd.size(); ++j) {
      const Stage& st = ex.bwd[j];
      if (j + 1 < ex.bwd.size()) casts.push_back(ex.cast(ex.bwd[j + 1], k, v));
      cuda_check(cudaStreamWaitEvent(cur, casts[j].done, 0), "cp wait cast");
      // the stage's partial dK / dV (written whole by the pass) and dQ += ...
      float *pk = nullptr, *pv = nullptr;
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&pk), std::max<size_t>(st.buf_tokens * grb, 16), cur),
                 "alloc");
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&pv), std::max<size_t>(st.buf_tokens * grb, 16), cur),
                 "alloc");
      if (st.plan) {
        const magiplan_status s = magiplan_ffa_bwd_stage(st.plan.get(), q, casts[j].k, casts[j].v, lse, delta,
                                                         dout, dq32, pk, pv, hq, hk, ex.scale, cur);
        if (s != MAGIPLAN_OK) throw DeviceError(magiplan_last_error());
      } else if (st.buf_tokens) {
        cuda_check(cudaMemsetAsync(pk, 0, st.buf_tokens * grb, cur), "memset");
        cuda_check(cudaMemsetAsync(pv, 0, st.buf_tokens * grb, cur), "memset");
      }
      // GroupReduce(j) on its own stream and communicator, under FFA(j+1)
      wait_and_destroy(ex.reduce_stream, record(cur));
      float *rk = nullptr, *rv = nullptr;
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&rk), std::max<size_t>(st.send->rows * grb, 16),
                                 ex.reduce_stream),
                 "alloc");
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&rv), std::max<size_t>(st.send->rows * grb, 16),
                                 ex.reduce_stream),
                 "alloc");
      // transposed exchange: partials of the tokens received from each source go back to it
      ex.exchange(ex.reduce_comm, st.recv_splits, st.send_splits, reinterpret_cast<uint8_t*>(pk),
                  reinterpret_cast<uint8_t*>(rk), grb, ex.reduce_stream);
      ex.exchange(ex.reduce_comm, st.recv_splits, st.send_splits, reinterpret_cast<uint8_t*>(pv),
                  reinterpret_cast<uint8_t*>(rv), grb, ex.reduce_stream);
      int64_t base = 0;
      for (int dst = 0; dst < ex.world; ++dst) {  // fixed source order: deterministic sums
        const RangeList& rl = *st.per_dst[static_cast<size_t>(dst)];
        if (rl.rows) {
          cuda_check(magi::launch_range_scatter_add_f32(rk + base * hk * d, dk32, rl.d_ranges, rl.d_offsets, rl.n,
                                                        rl.rows, hk * d, ex.reduce_stream),
                     "scatter_add launch");
          cuda_check(magi::launch_range_scatter_add_f32(rv + base * hk * d, dv32, rl.d_ranges, rl.d_offsets, rl.n,
                                                        rl.rows, hk * d, ex.reduce_stream),
                     "scatter_add launch");
        }
        base += rl.rows;
      }
      partials.push_back(pk);
      partials.push_back(pv);
      recvs.push_back(rk);
      recvs.push_back(rv);
    }
    wait_and_destroy(cur, record(ex.reduce_stream));
    cuda_check(magi::launch_cast_f32_bf16(dq32, dq, static_cast<int64_t>(gq), cur), "cast launch");
    cuda_check(magi::launch_cast_f32_bf16(dk32, dk, static_cast<int64_t>(gk), cur), "cast launch");
    cuda_check(magi::launch_cast_f32_bf16(dv32, dv, static_cast<int64_t>(gk), cur), "cast launch");
    for (auto& c : casts) CpExecutor::release(c, cur);
    for (void* p : partials) cudaFreeAsync(p, cur);
    for (void* p : recvs) cudaFreeAsync(p, cur);
    for (float* p : {delta, dq32, dk32, dv32}) cudaFreeAsync(p, cur);
  });
}

}  // extern "C"
