/* magiplan C ABI — B200-native drop-in for the reference planner's C ABI
 * (/root/reference/proj/include/magiplan/magiplan.h:43-121) plus the Flexible
 * Flash Attention (FFA) and context-parallel entry points the reference only
 * models as cost terms (proj/include/magiplan/overlap.hpp:44-50).
 *
 * Conventions (unchanged from the reference, magiplan.h:19-25):
 *   - every function returns a magiplan_status; failures leave outputs
 *     untouched and record a message readable via magiplan_last_error()
 *     (thread-local); success clears it;
 *   - strings returned through char** are heap-allocated; release them with
 *     magiplan_string_free;
 *   - handles are opaque; release them with the matching _free call.
 * Added conventions for device entry points:
 *   - tensors are caller-owned device pointers, passed as void* / float*;
 *   - cuda_stream is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - launches are asynchronous on cuda_stream; no hidden device sync;
 *   - CUDA failures map to MAGIPLAN_ERR_INTERNAL with the CUDA error text.
 */
#ifndef MAGIPLAN_H
#define MAGIPLAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define MAGIPLAN_API __declspec(dllexport)
#else
#define MAGIPLAN_API __attribute__((visibility("default")))
#endif

/* reference: magiplan.h:43-51 */
typedef enum magiplan_status {
  MAGIPLAN_OK = 0,
  MAGIPLAN_ERR_USAGE = 2,
  MAGIPLAN_ERR_CONSTRAINT = 3,
  MAGIPLAN_ERR_INTERNAL = 4
} magiplan_status;

/* reference: magiplan.h:53-56 */
typedef enum magiplan_counting {
  MAGIPLAN_COUNT_MULTIPLICITY = 0,
  MAGIPLAN_COUNT_UNION = 1
} magiplan_counting;

/* AttnSlice mask types; the values are the reference enum's
 * (proj/include/magiplan/mask.hpp:52). */
typedef enum magiplan_slice_type {
  MAGIPLAN_SLICE_FULL = 0,
  MAGIPLAN_SLICE_CAUSAL = 1,
  MAGIPLAN_SLICE_INV_CAUSAL = 2,
  MAGIPLAN_SLICE_BI_CAUSAL = 3
} magiplan_slice_type;

typedef enum magiplan_dtype { MAGIPLAN_F32 = 0, MAGIPLAN_BF16 = 1 } magiplan_dtype;

typedef struct magiplan_mask magiplan_mask;
typedef struct magiplan_scenario magiplan_scenario;
typedef struct magiplan_ffa_plan magiplan_ffa_plan;

/* ---- library ---------------------------------------------------------- */
/* reference: magiplan.h:61-67, capi.cpp:74-78 */
MAGIPLAN_API const char* magiplan_version(void);
MAGIPLAN_API const char* magiplan_last_error(void);
MAGIPLAN_API void magiplan_string_free(char* text);

/* ---- attention masks (reference: magiplan.h:69-98) -------------------- */
MAGIPLAN_API magiplan_status magiplan_mask_parse(const char* spec_json, magiplan_mask** out_mask);
MAGIPLAN_API void magiplan_mask_free(magiplan_mask* mask);
MAGIPLAN_API magiplan_status magiplan_mask_area(const magiplan_mask* mask,
                                                magiplan_counting counting, int64_t* out_area);
MAGIPLAN_API magiplan_status magiplan_mask_is_allowed(const magiplan_mask* mask, int64_t q,
                                                      int64_t k, int* out_allowed);
MAGIPLAN_API magiplan_status magiplan_mask_render(const magiplan_mask* mask, char** out_text);
MAGIPLAN_API magiplan_status magiplan_mask_describe(const magiplan_mask* mask, char** out_json);

/* ---- planning scenarios (reference: magiplan.h:100-118) --------------- */
MAGIPLAN_API magiplan_status magiplan_scenario_parse(const char* scenario_json,
                                                     const char* base_dir,
                                                     magiplan_scenario** out_scenario);
MAGIPLAN_API void magiplan_scenario_free(magiplan_scenario* scenario);
MAGIPLAN_API magiplan_status magiplan_scenario_set_seed(magiplan_scenario* scenario,
                                                        uint64_t seed);
MAGIPLAN_API magiplan_status magiplan_scenario_plan(const magiplan_scenario* scenario,
                                                    char** out_json);
MAGIPLAN_API magiplan_status magiplan_scenario_simulate(const magiplan_scenario* scenario,
                                                        int jobs, char** out_jsonl);
MAGIPLAN_API magiplan_status magiplan_pack_run(const char* config_json, const char* stream_text,
                                               char** out_json);

/* ---- context-parallel execution plan (new) ----------------------------- */
/* Executor view of magiplan_scenario_plan for the real multi-GPU run: per
 * rank its query chunks, and per forward/backward stage the KV token ranges
 * it receives (in receive-buffer order) together with the rank's local
 * slices re-expressed against [local KV | stage receive buffer] coordinates.
 * JSON object; see INTEGRATION.md for the field list. */
MAGIPLAN_API magiplan_status magiplan_scenario_exec_plan(const magiplan_scenario* scenario,
                                                         char** out_json);

/* ---- Flexible Flash Attention (new; no reference counterpart beyond the
 *      cost terms CostModel::ffa_fwd / ffa_bwd, overlap.hpp:47-48) ------- */

/* Compile a slice list into the device work list consumed by the kernels.
 * q_ranges / k_ranges: host int64 [num_slices][2] half-open ranges; types:
 * host int32 [num_slices] magiplan_slice_type. head_dim in {64, 128}.
 * Overlapping slices are legal and computed with MULTIPLICITY semantics
 * (mask.hpp:85): a pair covered by m slices contributes m times. The plan
 * owns device memory and is reusable across calls, heads and layers. */
MAGIPLAN_API magiplan_status magiplan_ffa_plan_create(const int64_t* q_ranges,
                                                      const int64_t* k_ranges,
                                                      const int32_t* types, int64_t num_slices,
                                                      int64_t seqlen_q, int64_t seqlen_k,
                                                      int32_t head_dim,
                                                      magiplan_ffa_plan** out_plan);
MAGIPLAN_API magiplan_status magiplan_ffa_plan_from_mask(const magiplan_mask* mask,
                                                         int32_t head_dim,
                                                         magiplan_ffa_plan** out_plan);
MAGIPLAN_API void magiplan_ffa_plan_free(magiplan_ffa_plan* plan);
/* {"seqlen_q","seqlen_k","head_dim","num_slices","area_multiplicity",
 *  "q_tiles","fwd_items","fwd_ktiles","bwd_items","bwd_qtiles"} */
MAGIPLAN_API magiplan_status magiplan_ffa_plan_describe(const magiplan_ffa_plan* plan,
                                                        char** out_json);

/* Uploads the plan's work lists to the current CUDA device (synchronous
 * cudaMalloc + cudaMemcpy). Optional: the first launch on a plan does it
 * otherwise, which then blocks that launch's host thread. A plan belongs to
 * the device it was first uploaded to; launching it on another device is a
 * MAGIPLAN_ERR_USAGE. */
MAGIPLAN_API magiplan_status magiplan_ffa_plan_prepare(magiplan_ffa_plan* plan);

/* Forward. q: [seqlen_q, num_heads_q, head_dim] bf16; k, v: [seqlen_k,
 * num_heads_k, head_dim] bf16 (GQA: num_heads_q % num_heads_k == 0);
 * out: [seqlen_q, num_heads_q, head_dim] in out_dtype; lse: [num_heads_q,
 * seqlen_q] f32 (natural log; -inf for rows with no allowed key).
 * accumulate != 0 merges this call into an existing (out, lse) pair with the
 * log-sum-exp correction (requires out_dtype == MAGIPLAN_F32): this is the
 * per-stage merge of the context-parallel forward. */
MAGIPLAN_API magiplan_status magiplan_ffa_fwd(const magiplan_ffa_plan* plan, const void* q,
                                              const void* k, const void* v, void* out,
                                              float* lse, int64_t num_heads_q,
                                              int64_t num_heads_k, float softmax_scale,
                                              int32_t out_dtype, int32_t accumulate,
                                              void* cuda_stream);

/* delta[h, i] = sum_d out[i, h, d] * grad_out[i, h, d] (f32 [num_heads,
 * seqlen]); out in out_dtype, grad_out bf16. */
MAGIPLAN_API magiplan_status magiplan_ffa_bwd_preprocess(const void* out, const void* grad_out,
                                                         float* delta, int64_t seqlen,
                                                         int64_t num_heads, int32_t head_dim,
                                                         int32_t out_dtype, void* cuda_stream);

/* Backward: grad_q [seqlen_q, hq, d], grad_k / grad_v [seqlen_k, hk, d] in
 * grad_dtype; accumulate != 0 adds into them (f32 only). Deterministic: no
 * unordered atomics; every gradient element is produced by one CTA in a
 * fixed order, so reruns are bitwise identical. */
MAGIPLAN_API magiplan_status magiplan_ffa_bwd(const magiplan_ffa_plan* plan, const void* q,
                                              const void* k, const void* v, const float* lse,
                                              const float* delta, const void* grad_out,
                                              void* grad_q, void* grad_k, void* grad_v,
                                              int64_t num_heads_q, int64_t num_heads_k,
                                              float softmax_scale, int32_t grad_dtype,
                                              int32_t accumulate, void* cuda_stream);

/* The backward of one context-parallel stage (f32 buffers): dQ is ADDED to
 * grad_q (the running dQ of the earlier stages), while grad_k / grad_v
 * receive the stage's fresh partial dK / dV of the received keys (written,
 * not added; keys no slice reaches get zeros). */
MAGIPLAN_API magiplan_status magiplan_ffa_bwd_stage(const magiplan_ffa_plan* plan, const void* q,
                                                    const void* k, const void* v, const float* lse,
                                                    const float* delta, const void* grad_out,
                                                    float* grad_q, float* grad_k, float* grad_v,
                                                    int64_t num_heads_q, int64_t num_heads_k,
                                                    float softmax_scale, void* cuda_stream);

/* The two halves of magiplan_ffa_bwd, for per-kernel timing and for running
 * them on separate streams: the k-major dK/dV pass and the q-major dQ pass. */
MAGIPLAN_API magiplan_status magiplan_ffa_bwd_dkdv(const magiplan_ffa_plan* plan, const void* q,
                                                   const void* k, const void* v,
                                                   const float* lse, const float* delta,
                                                   const void* grad_out, void* grad_k,
                                                   void* grad_v, int64_t num_heads_q,
                                                   int64_t num_heads_k, float softmax_scale,
                                                   int32_t grad_dtype, int32_t accumulate,
                                                   void* cuda_stream);
MAGIPLAN_API magiplan_status magiplan_ffa_bwd_dq(const magiplan_ffa_plan* plan, const void* q,
                                                 const void* k, const void* v, const float* lse,
                                                 const float* delta, const void* grad_out,
                                                 void* grad_q, int64_t num_heads_q,
                                                 int64_t num_heads_k, float softmax_scale,
                                                 int32_t grad_dtype, int32_t accumulate,
                                                 void* cuda_stream);

/* ---- context-parallel data movement kernels (new) ---------------------- */
/* Gather token ranges of a [tokens, width] row-major buffer into a packed
 * buffer (Range Gather). ranges: device int64 [n][2];
 * offsets: device int64 [n] destination row of each range. */
MAGIPLAN_API magiplan_status magiplan_range_gather(const void* src, void* dst,
                                                   const int64_t* ranges, const int64_t* offsets,
                                                   int64_t num_ranges, int64_t total_rows,
                                                   int64_t row_bytes, void* cuda_stream);
/* dst[ranges[i]] += src_packed[offsets[i] ...] in f32, ranges applied in
 * index order (deterministic Range Scatter-Reduce). */
MAGIPLAN_API magiplan_status magiplan_range_scatter_add_f32(const float* src, float* dst,
                                                            const int64_t* ranges,
                                                            const int64_t* offsets,
                                                            int64_t num_ranges,
                                                            int64_t total_rows,
                                                            int64_t row_elems,
                                                            void* cuda_stream);
/* f32 -> bf16 conversion of n elements. */
MAGIPLAN_API magiplan_status magiplan_cast_f32_bf16(const float* src, void* dst, int64_t n,
                                                    void* cuda_stream);

/* ---- peer-memory exchange (new): the GroupCast without NCCL -------------
 * Device buffers another process on the node can map (CUDA IPC): malloc
 * returns the pointer and its 64-byte handle; open maps a peer's handle. */
MAGIPLAN_API magiplan_status magiplan_p2p_malloc(int64_t bytes, void** out_ptr,
                                                 unsigned char* out_handle);
MAGIPLAN_API magiplan_status magiplan_p2p_free(void* ptr);
MAGIPLAN_API magiplan_status magiplan_p2p_open(const unsigned char* handle, void** out_ptr);
MAGIPLAN_API magiplan_status magiplan_p2p_close(void* ptr);
/* Range Gather fused with the transfer: range i copies source rows
 * [ranges[2i], ranges[2i+1]) to rows dst_row[i].. of the buffer at
 * dst_base[i] (device arrays; bases may be peer-mapped). offsets: packed
 * prefix of the range lengths, total_rows their sum. */
MAGIPLAN_API magiplan_status magiplan_range_copy_to(const void* src, const int64_t* ranges,
                                                    const int64_t* offsets, const uint64_t* dst_base,
                                                    const int64_t* dst_row, int64_t num_ranges,
                                                    int64_t total_rows, int64_t row_bytes,
                                                    void* cuda_stream);
/* Range Scatter-Reduce fused with the transfer: dst rows [ranges[2i],
 * ranges[2i+1]) += rows src_row[i].. of the f32 buffer at src_base[i]
 * (device arrays; bases may be peer-mapped). One call per source rank, in
 * rank order, keeps sums deterministic. */
MAGIPLAN_API magiplan_status magiplan_range_scatter_add_from(float* dst, const int64_t* ranges,
                                                             const int64_t* offsets, const uint64_t* src_base,
                                                             const int64_t* src_row, int64_t num_ranges,
                                                             int64_t total_rows, int64_t row_elems,
                                                             void* cuda_stream);
/* Stream-ordered flags: a system-scope release store of `value` to each of
 * the n <= 32 flags whose addresses are in the device array flag_ptrs; and a
 * wait until flags[i] >= value for every set bit i of mask (acquire). */
MAGIPLAN_API magiplan_status magiplan_flags_signal(const uint64_t* flag_ptrs, int32_t n, uint32_t value,
                                                   void* cuda_stream);
MAGIPLAN_API magiplan_status magiplan_flags_wait(const uint32_t* flags, uint32_t mask, uint32_t value,
                                                 void* cuda_stream);

/* ---- context-parallel executor (new) ------------------------------------ */
/* The planner's multi-stage CP schedule run on this process's GPU (one
 * process per GPU): GroupCast / GroupReduce over NCCL point-to-point
 * (resolved at run time from libnccl.so.2) on two communicators and two
 * high-priority streams, FFA stages with the LSE merge, deterministic
 * per-source scatter-add of the partial dK / dV. Same schedule as
 * paper_2505_13211_b200/cp.py. */
typedef struct magiplan_cp magiplan_cp;
/* 128 bytes (ncclUniqueId) made once (e.g. on rank 0) and handed to every rank. */
MAGIPLAN_API magiplan_status magiplan_cp_unique_id(void* out_id);
/* Collective over the scenario's cp_size ranks (each calls it with its rank
 * on its current CUDA device). */
MAGIPLAN_API magiplan_status magiplan_cp_create(const magiplan_scenario* scenario, int32_t rank,
                                                const void* nccl_unique_id, int64_t num_heads_q,
                                                int64_t num_heads_k, int32_t head_dim,
                                                float softmax_scale, magiplan_cp** out);
/* Transport of the GroupCast / GroupReduce bytes. NCCL: grouped point-to-point
 * on two communicators. P2P: NVLink peer memory (one rank per GPU of one
 * node, cp_size <= 32): the stage buffers are CUDA-IPC memory whose handles
 * are all-gathered at creation (over the NCCL communicator), the GroupCast
 * is a fused gather-and-send kernel writing into the consumers' buffers, the
 * GroupReduce a per-consumer scatter-add (rank order) reading their partials,
 * ordered by stream-side release / acquire flags. Same results bit for bit. */
typedef enum magiplan_cp_transport { MAGIPLAN_CP_NCCL = 0, MAGIPLAN_CP_P2P = 1 } magiplan_cp_transport;
/* magiplan_cp_create with a transport (magiplan_cp_create = MAGIPLAN_CP_NCCL). */
MAGIPLAN_API magiplan_status magiplan_cp_create_ex(const magiplan_scenario* scenario, int32_t rank,
                                                   const void* nccl_unique_id, int64_t num_heads_q,
                                                   int64_t num_heads_k, int32_t head_dim,
                                                   float softmax_scale, int32_t transport,
                                                   magiplan_cp** out);
MAGIPLAN_API void magiplan_cp_free(magiplan_cp* cp);
/* {"rank","cp_size","local_tokens","chunk_size","chunks":[global chunk ids in
 *  local order],"num_stages_fwd","num_stages_bwd","area_multiplicity",
 *  "transport":"nccl"|"p2p"} */
MAGIPLAN_API magiplan_status magiplan_cp_describe(const magiplan_cp* cp, char** out_json);
/* Local shards in chunk order: q [L, hq, d], k / v [L, hk, d] bf16; out_f32
 * [L, hq, d] and lse [hq, L] f32 (kept for the backward); out_bf16 optional. */
MAGIPLAN_API magiplan_status magiplan_cp_forward(magiplan_cp* cp, const void* q, const void* k,
                                                 const void* v, float* out_f32, float* lse,
                                                 void* out_bf16, void* cuda_stream);
/* dq [L, hq, d], dk / dv [L, hk, d] bf16 of the local shard. */
MAGIPLAN_API magiplan_status magiplan_cp_backward(magiplan_cp* cp, const void* q, const void* k,
                                                  const void* v, const float* out_f32,
                                                  const float* lse, const void* dout, void* dq,
                                                  void* dk, void* dv, void* cuda_stream);

/* ---- diagnostics ------------------------------------------------------- */
/* Event log of one forward / backward CTA (block index `block`; a negative
 * value -b-1 selects CTA b of the separate dQ pass) into a device int64 buffer
 * of 1 + 5 * 2 * 8000 entries: per warp role (MMA, two elementwise
 * warpgroups, TMA, load observer) 8000 {event << 32 | step, globaltimer ns}
 * pairs. NULL switches tracing off. Only a library built with -DMAGI_TRACE
 * (python -m paper_2505_13211_b200.build --trace) carries the traced kernel
 * instantiations; the default build returns MAGIPLAN_ERR_USAGE for a non-NULL
 * buffer. Diagnostics only (tools/trace_*.py). */
MAGIPLAN_API magiplan_status magiplan_debug_set_trace(void* device_buffer, int32_t block);
/* JSON-RPC access to individual planner functions for parity tests:
 * {"op": "slice_area" | "slice_area_in_cols" | "clip_slice" | "mask" |
 *  "restrict_rows" | "shard" | "greedy" | "zigzag" | "brute_force" |
 *  "demands" | "partition_packages" | "assign_packages" | "estimate" |
 *  "fit_affine" | "lognormal" | "flops", ...}. */
MAGIPLAN_API magiplan_status magiplan_debug_eval(const char* request_json, char** out_json);
/* One 128x128x128 bf16 tile product through the TMA/UMMA building blocks
 * (C = A B^T for b_mn_major == 0, C = A B otherwise). Device pointers. */
MAGIPLAN_API magiplan_status magiplan_debug_umma_tile(const void* a, const void* b, float* c,
                                                      int32_t b_mn_major, void* cuda_stream);

#ifdef __cplusplus
}
#endif

#endif /* MAGIPLAN_H */
