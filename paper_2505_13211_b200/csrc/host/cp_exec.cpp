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
// Transport MAGIPLAN_CP_P2P (magiplan_cp_create_ex) moves the same bytes
// over NVLink peer memory instead, as cp.py's transport="p2p" does: every
// stage's receive buffers (and, backward, the partial dK / dV buffers) live
// in IPC-exportable memory whose handles are all-gathered once at creation;
// the GroupCast is one fused gather-and-send kernel writing straight into
// the consumers' buffers, the GroupReduce one scatter-add per consumer (rank
// order) reading its partials over NVLink, and stream-side release / acquire
// flags order producers, consumers and buffer reuse across passes.
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
cudaError_t launch_range_copy_to(const void* src, const int64_t* ranges, const int64_t* offsets,
                                 const unsigned long long* dst_base, const int64_t* dst_row, int64_t num_ranges,
                                 int64_t total_rows, int64_t row_bytes, cudaStream_t stream);
cudaError_t launch_range_scatter_add_from(float* dst, const int64_t* ranges, const int64_t* offsets,
                                          const unsigned long long* src_base, const int64_t* src_row,
                                          int64_t num_ranges, int64_t total_rows, int64_t row_elems,
                                          cudaStream_t stream);
cudaError_t launch_flags_signal(unsigned int* const* flags, int n, unsigned int value, cudaStream_t stream);
cudaError_t launch_flags_wait(const unsigned int* flags, unsigned int mask, unsigned int value,
                              cudaStream_t stream);
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
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
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
    lib.AllGather = reinterpret_cast<decltype(lib.AllGather)>(sym("ncclAllGather"));
    lib.GetErrorString = reinterpret_cast<decltype(lib.GetErrorString)>(sym("ncclGetErrorString"));
    if (!lib.GetUniqueId || !lib.CommInitRank || !lib.CommSplit || !lib.Send || !lib.Recv || !lib.GroupStart ||
        !lib.GroupEnd || !lib.AllGather)
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

// owning device copy of a host array (nullptr when empty)
template <typename T>
struct DevArr {
  T* p = nullptr;
  DevArr() = default;
  explicit DevArr(const std::vector<T>& host) : p(device_copy(host)) {}
  DevArr(DevArr&& o) noexcept : p(o.p) { o.p = nullptr; }
  DevArr& operator=(DevArr&& o) noexcept {
    std::swap(p, o.p);
    return *this;
  }
  DevArr(const DevArr&) = delete;
  DevArr& operator=(const DevArr&) = delete;
  ~DevArr() { cudaFree(p); }
};

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

// One stage over peer memory. Flag block (uint32, index = peer rank), each
// entry written by that peer into this rank's block: [ready | consumed |
// partials ready | partials read].
struct PeerStage {
  void *kb = nullptr, *vb = nullptr;     // this rank's receive buffers (bf16)
  float *dkb = nullptr, *dvb = nullptr;  // this rank's partial dK / dV (backward)
  uint32_t* flags = nullptr;
  // GroupCast as producer: every consumer's receive entries from this rank
  int64_t n = 0, rows = 0;
  DevArr<int64_t> ranges, offs, drow;
  DevArr<uint64_t> kbase, vbase;
  DevArr<uint64_t> sig_send, sig_recv, sig_pready, sig_pdone;
  int n_dest = 0, n_src = 0;
  uint32_t mask_dest = 0, mask_src = 0;
  struct Dst {  // GroupReduce as owner: one consumer's partial rows of this rank's keys
    int64_t n = 0, rows = 0;
    DevArr<int64_t> ranges, offs, row;
    DevArr<uint64_t> bdk, bdv;
  };
  std::vector<Dst> per_dst;  // consumers in rank order
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
  // peer-memory transport
  bool p2p = false;
  std::vector<PeerStage> pfwd, pbwd;
  std::vector<void*> owned, opened;
  uint32_t epoch = 0, bepoch = 0;

  ~CpExecutor() {
    if (comm_stream) cudaStreamSynchronize(comm_stream);
    if (reduce_stream) cudaStreamSynchronize(reduce_stream);
    if (p2p) cudaDeviceSynchronize();
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    for (void* p : owned) cudaFree(p);
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

  void* ipc_alloc(size_t bytes, std::vector<cudaIpcMemHandle_t>& handles) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "p2p alloc");
    owned.push_back(p);
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
    handles.push_back(h);
    return p;
  }

  // Receive / partial buffers and flags of every stage, handles all-gathered
  // over the cast communicator, the peers' buffers mapped, and the device
  // arrays of the fused kernels built from the executor plan.
  void setup_p2p(const json& xp) {
    if (world > 32) throw UsageError("p2p transport: at most 32 ranks (flag masks)");
    const size_t krow = kv_row_bytes(), grow = grad_row_bytes();
    std::vector<cudaIpcMemHandle_t> mine;
    const std::pair<const char*, std::vector<Stage>*> passes[2] = {{"fwd_stages", &fwd}, {"bwd_stages", &bwd}};
    for (const auto& [key, stages] : passes) {
      const bool back = stages == &bwd;
      auto& ps = back ? pbwd : pfwd;
      ps.resize(stages->size());
      for (size_t j = 0; j < stages->size(); ++j) {
        PeerStage& P = ps[j];
        const size_t bt = static_cast<size_t>((*stages)[j].buf_tokens);
        P.kb = ipc_alloc(bt * krow, mine);
        P.vb = ipc_alloc(bt * krow, mine);
        if (back) {
          P.dkb = static_cast<float*>(ipc_alloc(bt * grow, mine));
          P.dvb = static_cast<float*>(ipc_alloc(bt * grow, mine));
        }
        P.flags = static_cast<uint32_t*>(ipc_alloc(16 * static_cast<size_t>(world), mine));
        cuda_check(cudaMemset(P.flags, 0, 16 * static_cast<size_t>(world)), "p2p flags");
      }
    }
    // all-gather the handles (the flags are zero everywhere before any peer can signal)
    // every rank has the same stage counts, hence the same handle count
    const size_t hb = mine.size() * sizeof(cudaIpcMemHandle_t);
    if (hb == 0) {
      p2p = true;
      return;
    }
    std::vector<uint8_t> mine_bytes(hb);
    std::memcpy(mine_bytes.data(), mine.data(), hb);
    const DevArr<uint8_t> d_send(mine_bytes);
    const DevArr<uint8_t> d_all(std::vector<uint8_t>(hb * static_cast<size_t>(world)));
    cuda_check(cudaDeviceSynchronize(), "p2p handles");
    nccl_check(nccl().AllGather(d_send.p, d_all.p, hb, kNcclInt8, cast_comm, comm_stream), "ncclAllGather");
    std::vector<cudaIpcMemHandle_t> all(mine.size() * static_cast<size_t>(world));
    cuda_check(cudaStreamSynchronize(comm_stream), "p2p handles");
    cuda_check(cudaMemcpy(all.data(), d_all.p, hb * world, cudaMemcpyDeviceToHost), "p2p handles");

    const json& ranks = xp["ranks"];
    size_t hidx = 0;  // handle index of the stage's first buffer, same on every rank
    for (const auto& [key, stages] : passes) {
      const bool back = stages == &bwd;
      const size_t per = back ? 5 : 3;  // k, v, (dk, dv,) flags
      auto& ps = back ? pbwd : pfwd;
      for (size_t j = 0; j < stages->size(); ++j, hidx += per) {
        PeerStage& P = ps[j];
        std::vector<std::vector<uint64_t>> peer(static_cast<size_t>(world));
        for (int d = 0; d < world; ++d) {
          if (d == rank) continue;
          for (size_t b = 0; b < per; ++b) {
            void* o = nullptr;
            cuda_check(cudaIpcOpenMemHandle(&o, all[static_cast<size_t>(d) * mine.size() + hidx + b],
                                            cudaIpcMemLazyEnablePeerAccess),
                       "cudaIpcOpenMemHandle");
            opened.push_back(o);
            peer[static_cast<size_t>(d)].push_back(reinterpret_cast<uint64_t>(o));
          }
        }
        auto flag_of = [&](int d, int block) {  // entry `rank` of block `block` in d's flags
          return peer[static_cast<size_t>(d)][per - 1] + 4ull * (static_cast<uint64_t>(block) * world + rank);
        };
        std::vector<int64_t> ranges, offs, drow;
        std::vector<uint64_t> kbase, vbase, sig_send, sig_pdone;
        for (int d = 0; d < world; ++d) {
          const json& other = ranks[static_cast<size_t>(d)][key];
          if (d == rank || j >= other.size()) continue;
          PeerStage::Dst dst;
          std::vector<int64_t> rr, ro, rrow;
          std::vector<uint64_t> bdk, bdv;
          bool any = false;
          for (const auto& e : other[j]["recv"]) {
            if (e[0].get<int>() != rank) continue;
            any = true;
            const int64_t len = e[2].get<int64_t>() - e[1].get<int64_t>();
            const int64_t src_local = e[3].get<int64_t>(), buf_off = e[4].get<int64_t>();
            ranges.push_back(src_local);
            ranges.push_back(src_local + len);
            offs.push_back(P.rows);
            P.rows += len;
            kbase.push_back(peer[static_cast<size_t>(d)][0]);
            vbase.push_back(peer[static_cast<size_t>(d)][1]);
            drow.push_back(buf_off);
            if (back) {
              rr.push_back(src_local);
              rr.push_back(src_local + len);
              ro.push_back(dst.rows);
              dst.rows += len;
              bdk.push_back(peer[static_cast<size_t>(d)][2]);
              bdv.push_back(peer[static_cast<size_t>(d)][3]);
              rrow.push_back(buf_off);
            }
          }
          if (!any) continue;
          P.mask_dest |= 1u << d;
          ++P.n_dest;
          sig_send.push_back(flag_of(d, 0));
          if (back) {
            sig_pdone.push_back(flag_of(d, 3));
            dst.n = static_cast<int64_t>(ro.size());
            dst.ranges = DevArr<int64_t>(rr);
            dst.offs = DevArr<int64_t>(ro);
            dst.row = DevArr<int64_t>(rrow);
            dst.bdk = DevArr<uint64_t>(bdk);
            dst.bdv = DevArr<uint64_t>(bdv);
            P.per_dst.push_back(std::move(dst));
          }
        }
        P.n = static_cast<int64_t>(offs.size());
        P.ranges = DevArr<int64_t>(ranges);
        P.offs = DevArr<int64_t>(offs);
        P.drow = DevArr<int64_t>(drow);
        P.kbase = DevArr<uint64_t>(kbase);
        P.vbase = DevArr<uint64_t>(vbase);
        P.sig_send = DevArr<uint64_t>(sig_send);
        P.sig_pdone = DevArr<uint64_t>(sig_pdone);
        // as consumer: the sources of this stage's receive entries
        std::vector<uint64_t> sig_recv, sig_pready;
        const json& me = ranks[static_cast<size_t>(rank)][key];
        if (j < me.size()) {
          for (const auto& e : me[j]["recv"]) {
            const int s_ = e[0].get<int>();
            if (P.mask_src >> s_ & 1u) continue;
            P.mask_src |= 1u << s_;
          }
          for (int s_ = 0; s_ < world; ++s_) {
            if (!(P.mask_src >> s_ & 1u)) continue;
            ++P.n_src;
            sig_recv.push_back(flag_of(s_, 1));
            if (back) sig_pready.push_back(flag_of(s_, 2));
          }
        }
        P.sig_recv = DevArr<uint64_t>(sig_recv);
        P.sig_pready = DevArr<uint64_t>(sig_pready);
      }
    }
    p2p = true;
  }

  void flags_wait(const PeerStage& P, int block, uint32_t mask, uint32_t value, cudaStream_t s) const {
    cuda_check(magi::launch_flags_wait(P.flags + static_cast<size_t>(block) * world, mask, value, s),
               "flags_wait launch");
  }
  static void flags_signal(const DevArr<uint64_t>& ptrs, int n, uint32_t value, cudaStream_t s) {
    cuda_check(magi::launch_flags_signal(reinterpret_cast<unsigned int* const*>(ptrs.p), n, value, s),
               "flags_signal launch");
  }

  // GroupCast of one stage over peer memory on the comm stream: wait until
  // every consumer released the buffer of the previous pass, copy the ranges
  // into the consumers' buffers, raise their ready flags
  void cast_p2p(const PeerStage& P, uint32_t ep, const void* k, const void* v) const {
    flags_wait(P, 1, P.mask_dest, ep - 1, comm_stream);
    if (P.n) {
      for (const auto& [src, base] : {std::pair<const void*, const uint64_t*>{k, P.kbase.p}, {v, P.vbase.p}})
        cuda_check(magi::launch_range_copy_to(src, P.ranges.p, P.offs.p,
                                              reinterpret_cast<const unsigned long long*>(base), P.drow.p, P.n,
                                              P.rows, static_cast<int64_t>(kv_row_bytes()), comm_stream),
                   "range_copy_to launch");
    }
    flags_signal(P.sig_send, P.n_dest, ep, comm_stream);
  }

  // GroupReduce of one backward stage over peer memory on the reduce stream:
  // the consumers' partials, per consumer in rank order, added into dk / dv
  void reduce_p2p(const PeerStage& P, uint32_t ep, float* dk32, float* dv32) const {
    flags_wait(P, 2, P.mask_dest, ep, reduce_stream);
    for (const auto& dst : P.per_dst) {
      if (!dst.n) continue;
      for (const auto& [acc, base] : {std::pair<float*, const uint64_t*>{dk32, dst.bdk.p}, {dv32, dst.bdv.p}})
        cuda_check(magi::launch_range_scatter_add_from(acc, dst.ranges.p, dst.offs.p,
                                                       reinterpret_cast<const unsigned long long*>(base),
                                                       dst.row.p, dst.n, dst.rows, hk * d, reduce_stream),
                   "range_scatter_add_from launch");
    }
    flags_signal(P.sig_pdone, P.n_dest, ep, reduce_stream);
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
  return magiplan_cp_create_ex(scenario, rank, nccl_unique_id, num_heads_q, num_heads_k, head_dim, softmax_scale,
                               MAGIPLAN_CP_NCCL, out);
}

magiplan_status magiplan_cp_create_ex(const magiplan_scenario* scenario, int32_t rank, const void* nccl_unique_id,
                                      int64_t num_heads_q, int64_t num_heads_k, int32_t head_dim,
                                      float softmax_scale, int32_t transport, magiplan_cp** out) {
  MAGI_REQUIRE(scenario && nccl_unique_id && out);
  auto* cp = new magiplan_cp;
  const magiplan_status st = guarded([&] {
    using namespace magiplan;
    if (transport != MAGIPLAN_CP_NCCL && transport != MAGIPLAN_CP_P2P)
      throw UsageError("transport must be MAGIPLAN_CP_NCCL or MAGIPLAN_CP_P2P");
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
    if (transport == MAGIPLAN_CP_P2P && ex.world > 1) ex.setup_p2p(xp);
    json dj;
    dj["rank"] = rank;
    dj["cp_size"] = ex.world;
    dj["local_tokens"] = ex.local_tokens;
    dj["chunk_size"] = xp["chunk_size"];
    dj["chunks"] = me["chunks"];
    dj["num_stages_fwd"] = xp["num_stages_fwd"];
    dj["num_stages_bwd"] = xp["num_stages_bwd"];
    dj["area_multiplicity"] = xp["area_multiplicity"];
    dj["transport"] = ex.p2p ? "p2p" : "nccl";
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
    const bool p2p = ex.p2p;
    const uint32_t ep = p2p ? ++ex.epoch : 0;
    auto cast = [&](size_t j) {
      if (p2p)
        ex.cast_p2p(ex.pfwd[j], ep, k, v);
      else
        casts.push_back(ex.cast(ex.fwd[j], k, v));
    };
    if (!ex.fwd.empty()) cast(0);
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
      if (j + 1 < ex.fwd.size()) cast(j + 1);
      if (p2p) {
        // the producers' copies into this rank's buffers have landed
        const PeerStage& P = ex.pfwd[j];
        ex.flags_wait(P, 0, P.mask_src, ep, cur);
        if (ex.fwd[j].plan) ffa(ex.fwd[j].plan.get(), P.kb, P.vb, 1);
        // release the buffers: the producers may overwrite them next pass
        CpExecutor::flags_signal(P.sig_recv, P.n_src, ep, cur);
      } else {
        cuda_check(cudaStreamWaitEvent(cur, casts[j].done, 0), "cp wait cast");
        if (ex.fwd[j].plan) ffa(ex.fwd[j].plan.get(), casts[j].k, casts[j].v, 1);
      }
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
    const bool p2p = ex.p2p;
    const uint32_t eb = p2p ? ++ex.bepoch : 0;
    auto cast = [&](size_t j) {
      if (p2p)
        ex.cast_p2p(ex.pbwd[j], eb, k, v);
      else
        casts.push_back(ex.cast(ex.bwd[j], k, v));
    };
    if (!ex.bwd.empty()) cast(0);
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
      if (j + 1 < ex.bwd.size()) cast(j + 1);
      // the stage's partial dK / dV (written whole by the pass) and dQ += ...
      float *pk = nullptr, *pv = nullptr;
      const void *kk = nullptr, *vv = nullptr;
      if (p2p) {
        // the producers' K / V have landed, and the owners have read last
        // pass's partials out of this rank's partial buffers
        const PeerStage& P = ex.pbwd[j];
        ex.flags_wait(P, 0, P.mask_src, eb, cur);
        ex.flags_wait(P, 3, P.mask_src, eb - 1, cur);
        pk = P.dkb;
        pv = P.dvb;
        kk = P.kb;
        vv = P.vb;
      } else {
        cuda_check(cudaStreamWaitEvent(cur, casts[j].done, 0), "cp wait cast");
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&pk), std::max<size_t>(st.buf_tokens * grb, 16), cur),
                   "alloc");
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&pv), std::max<size_t>(st.buf_tokens * grb, 16), cur),
                   "alloc");
        kk = casts[j].k;
        vv = casts[j].v;
      }
      if (st.plan) {
        const magiplan_status s = magiplan_ffa_bwd_stage(st.plan.get(), q, kk, vv, lse, delta, dout, dq32, pk, pv,
                                                         hq, hk, ex.scale, cur);
        if (s != MAGIPLAN_OK) throw DeviceError(magiplan_last_error());
      } else if (st.buf_tokens) {
        cuda_check(cudaMemsetAsync(pk, 0, st.buf_tokens * grb, cur), "memset");
        cuda_check(cudaMemsetAsync(pv, 0, st.buf_tokens * grb, cur), "memset");
      }
      if (p2p) {
        // release this stage's K / V buffers, publish the partials; the
        // owners add them in on their reduce streams
        const PeerStage& P = ex.pbwd[j];
        CpExecutor::flags_signal(P.sig_recv, P.n_src, eb, cur);
        CpExecutor::flags_signal(P.sig_pready, P.n_src, eb, cur);
        wait_and_destroy(ex.reduce_stream, record(cur));
        ex.reduce_p2p(P, eb, dk32, dv32);
        continue;
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
    if (p2p) {
      // the owners have read this pass's partials: once the pass completes
      // no peer touches this rank's buffers (magiplan_cp_free needs no barrier)
      for (const PeerStage& P : ex.pbwd) ex.flags_wait(P, 3, P.mask_src, eb, cur);
    }
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
