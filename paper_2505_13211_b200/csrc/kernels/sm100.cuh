// sm_100a building blocks: mbarrier, TMA, tcgen05 (UMMA / TMEM) wrappers as
// inline PTX. Everything the FFA kernels need from the Blackwell execution
// model lives here so the kernels themselves read as dataflow.
//
// Descriptor encodings follow the PTX ISA "tcgen05 shared memory descriptor"
// and "instruction descriptor" tables (kind::f16):
//   smem desc : [0,14) addr>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 |
//               [46,48) version=1 | [49,52) base offset | [61,64) layout
//   instr desc: [4,6) D fmt (1=f32) | [7,10) A fmt (1=bf16) | [10,13) B fmt |
//               [15] A MN-major | [16] B MN-major | [17,23) N>>3 | [24,29) M>>4
#pragma once

#include <cstdint>
#include <cuda_bf16.h>

namespace magi {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Ring-buffer position: stage index plus the phase bit mbarriers expect.
struct PipeState {
  uint32_t index = 0;
  uint32_t phase = 0;
  template <int kStages>
  __device__ __forceinline__ void advance() {
    if (++index == kStages) {
      index = 0;
      phase ^= 1u;
    }
  }
};

// ---------------------------------------------------------------- fences
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------- TMEM
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "tmem cols");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets lane
// (32*(warp%4) + t), columns [col, col+32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// 32 lanes x 16 consecutive columns from 16 registers
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
      "%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- UMMA
enum : uint32_t { kSwizzleNone = 0, kSwizzle128B = 2 };

__device__ __forceinline__ uint64_t make_smem_desc(uint32_t saddr, uint32_t lbo_bytes,
                                                   uint32_t sbo_bytes,
                                                   uint32_t layout = kSwizzle128B) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(layout & 7u) << 61;
  return d;
}

// bf16 x bf16 -> f32, dense.
__host__ __device__ constexpr uint32_t make_idesc_bf16(uint32_t M, uint32_t N, bool a_mn_major,
                                                       bool b_mn_major) {
  return (1u << 4)                                  // D = f32
         | (1u << 7)                                // A = bf16
         | (1u << 10)                               // B = bf16
         | (static_cast<uint32_t>(a_mn_major) << 15)  //
         | (static_cast<uint32_t>(b_mn_major) << 16)  //
         | ((N >> 3) << 17)                         //
         | ((M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]; issued by one thread.
__device__ __forceinline__ void umma_bf16_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]; A is M lanes x (K/2) 32-bit columns of
// packed bf16 pairs (K-major). Issued by one thread.
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// ---- converged-warp issue: every lane of the MMA warp executes these and one
// elected lane issues, so descriptor arithmetic stays on the uniform datapath
// (a lane-0-only branch would rebuild every descriptor in vector registers
// and move it to uniform registers before each instruction).
__device__ __forceinline__ void umma_ss_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// One 128 x N x 128 GEMM (8 k-steps of K = 16) in a single asm block, issued
// by one elected lane of a converged warp. SS: A and B K-major SW128 tiles of
// two 64-column boxes (k-step = +32 B, box = +16 KB). The descriptor offsets
// are applied in 16-byte units inside the block.
__device__ __forceinline__ void umma_gemm_ss_k128(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p, t, e;\n .reg .b64 a, b;\n"
      " setp.ne.b32 p, %4, 0;\n setp.eq.b32 t, %4, %4;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      " add.s64 a, %1, 2;\n add.s64 b, %2, 2;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
      " add.s64 a, %1, 4;\n add.s64 b, %2, 4;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
      " add.s64 a, %1, 6;\n add.s64 b, %2, 6;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
      " add.s64 a, %1, 1024;\n add.s64 b, %2, 1024;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
      " add.s64 a, %1, 1026;\n add.s64 b, %2, 1026;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
      " add.s64 a, %1, 1028;\n add.s64 b, %2, 1028;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
      " add.s64 a, %1, 1030;\n add.s64 b, %2, 1030;\n"
      " @e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n"
      "}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// TS GEMMs of 8 k-steps (K = 128) in one asm block: per step the TMEM column
// offset of A (packed bf16, 8 columns per 16 elements) and the B descriptor
// offset in 16-byte units are compile-time constants of the operand layout.
#define MAGI_TS_STEP(ao, bo, pr)                                        \
  " add.s32 a, %1, " #ao ";\n add.s64 b, %2, " #bo ";\n"              \
  " @e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, " pr ";\n"
#define MAGI_TS_GEMM(name, a0, a1, a2, a3, a4, a5, a6, a7, b0, b1, b2, b3, b4, b5, b6, b7)       \
  __device__ __forceinline__ void name(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,        \
                                       uint32_t idesc, uint32_t accumulate) {                   \
    asm volatile("{\n .reg .pred p, t, e;\n .reg .b32 a;\n .reg .b64 b;\n"                    \
                 " setp.ne.b32 p, %4, 0;\n setp.eq.b32 t, %4, %4;\n"                          \
                 " elect.sync _|e, 0xffffffff;\n" MAGI_TS_STEP(a0, b0, "p")                   \
                     MAGI_TS_STEP(a1, b1, "t") MAGI_TS_STEP(a2, b2, "t") MAGI_TS_STEP(a3, b3, "t") \
                         MAGI_TS_STEP(a4, b4, "t") MAGI_TS_STEP(a5, b5, "t")                    \
                             MAGI_TS_STEP(a6, b6, "t") MAGI_TS_STEP(a7, b7, "t") "}" ::"r"(d_tmem), \
                 "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)                           \
                 : "memory");                                                                   \
  }
// A: consecutive k-steps (8 columns apart); B MN-major (16 rows = 2 KB per step)
MAGI_TS_GEMM(umma_gemm_ts_k128, 0, 8, 16, 24, 32, 40, 48, 56, 0, 128, 256, 384, 512, 640, 768, 896)
// A: consecutive k-steps; B K-major SW128 (32 B per step, second 64-column box 16 KB on)
MAGI_TS_GEMM(umma_gemm_ts_bk_k128, 0, 8, 16, 24, 32, 40, 48, 56, 0, 2, 4, 6, 1024, 1026, 1028, 1030)
// A: the dK/dV kernel's packed P^T (or dS^T, +16) layout: query columns
// [16k, 16k+16) at (k/4)*64 + ((k/2)%2)*32 + (k%2)*8; B MN-major
MAGI_TS_GEMM(umma_gemm_ts_dkdv_k128, 0, 8, 32, 40, 64, 72, 96, 104, 0, 128, 256, 384, 512, 640, 768, 896)
// A: the dQ kernel's packed dS layout: keys [0,64) at +0, [64,128) at +64; B MN-major
MAGI_TS_GEMM(umma_gemm_ts_dq_k128, 0, 8, 16, 24, 64, 72, 80, 88, 0, 128, 256, 384, 512, 640, 768, 896)
// half-depth (K = 64) forms of the consecutive-A / MN-major-B GEMM: keys
// [0,64) and [64,128) of a 128-key tile (the forward's split P hand-off)
#define MAGI_TS_GEMM4(name, a0, a1, a2, a3, b0, b1, b2, b3)                                      \
  __device__ __forceinline__ void name(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,        \
                                       uint32_t idesc, uint32_t accumulate) {                   \
    asm volatile("{\n .reg .pred p, t, e;\n .reg .b32 a;\n .reg .b64 b;\n"                    \
                 " setp.ne.b32 p, %4, 0;\n setp.eq.b32 t, %4, %4;\n"                          \
                 " elect.sync _|e, 0xffffffff;\n" MAGI_TS_STEP(a0, b0, "p")                   \
                     MAGI_TS_STEP(a1, b1, "t") MAGI_TS_STEP(a2, b2, "t") MAGI_TS_STEP(a3, b3, "t") \
                 "}" ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)        \
                 : "memory");                                                                   \
  }
MAGI_TS_GEMM4(umma_gemm_ts_k128_lo, 0, 8, 16, 24, 0, 128, 256, 384)
MAGI_TS_GEMM4(umma_gemm_ts_k128_hi, 32, 40, 48, 56, 512, 640, 768, 896)
#undef MAGI_TS_GEMM4
#undef MAGI_TS_GEMM

// descriptor of the same tile advanced by `bytes` (start address field only)
__device__ __forceinline__ uint64_t desc_add(uint64_t desc, uint32_t bytes) {
  return desc + static_cast<uint64_t>(bytes >> 4);
}

// Arrive on an mbarrier once all previously issued tcgen05 ops of this
// thread have completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- tracing
// Per-role event log (diagnostics, magiplan_debug_set_trace): role r writes
// {event << 32 | step, %globaltimer ns} pairs into its own region, no atomics.
constexpr int kTraceCap = 8000;
// ON = false compiles to nothing: production kernels are instantiated without
// tracing (a not-taken trace call still splits basic blocks and costs
// scheduling freedom in the hot loops); the traced instantiation is launched
// only while magiplan_debug_set_trace is active.
template <bool ON>
struct TracerT {
  long long* base = nullptr;
  int n = 0;
  __device__ __forceinline__ void init(long long* trace, int role) {
    if constexpr (ON) base = trace ? trace + 1 + static_cast<size_t>(role) * 2 * kTraceCap : nullptr;
  }
  __device__ __forceinline__ void ev(int e, int t) {
    if constexpr (ON) {
      if (base == nullptr || n >= kTraceCap) return;
      if ((threadIdx.x & 31) != 0) return;  // lane 0 writes (converged callers init every lane)
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      base[2 * n] = (static_cast<long long>(e) << 32) | static_cast<unsigned>(t);
      base[2 * n + 1] = static_cast<long long>(ns);
      ++n;
    }
  }
  // {event << 32 | low 32 bits of clock64, ns}: two of these give the SM clock
  __device__ __forceinline__ void clk(int e) {
    if constexpr (ON) {
      if (base == nullptr || n >= kTraceCap) return;
      if ((threadIdx.x & 31) != 0) return;
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      const long long c = clock64();
      base[2 * n] = (static_cast<long long>(e) << 32) | static_cast<unsigned>(c);
      base[2 * n + 1] = static_cast<long long>(ns);
      ++n;
    }
  }
};

// ---------------------------------------------------------------- math
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes (no MUFU): round-to-nearest split via the
// 1.5*2^23 magic constant, degree-3 polynomial for 2^f on [-0.5, 0.5]
// (max rel. error 1.8e-4, far below the bf16 rounding of P), exponent added
// as an integer. Valid for finite x >= -126 (callers clamp).
__device__ __forceinline__ float exp2_poly(float x) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  x = fmaxf(x, -126.0f);
  const float y = x + kMagic;            // round(x) in the low mantissa bits
  const float f = x - (y - kMagic);      // f in [-0.5, 0.5]
  float p = fmaf(f, 0.054602622718538274f, 0.24192412881028413f);
  p = fmaf(p, f, 0.6933164806648954f);
  p = fmaf(p, f, 1.0f);
  // bits(y) = bits(magic) + round(x); shifting by 23 moves round(x) into the exponent
  return __int_as_float(__float_as_int(p) + (__float_as_int(y) << 23) -
                        (__float_as_int(kMagic) << 23));
}

// ---- packed f32x2 (sm_100 FFMA2 / FADD2: two fp32 lanes per instruction)
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2_split(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// exp2_poly on two values with packed arithmetic (same split and polynomial)
__device__ __forceinline__ float2 exp2_poly2(float x0, float x1) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  const uint64_t x = f2(fmaxf(x0, -126.0f), fmaxf(x1, -126.0f));
  const uint64_t y = fadd2(x, f2(kMagic, kMagic));
  const uint64_t r = fadd2(y, f2(-kMagic, -kMagic));  // round(x)
  const uint64_t f = ffma2(r, f2(-1.0f, -1.0f), x);   // x - round(x)
  uint64_t p = ffma2(f, f2(0.054602622718538274f, 0.054602622718538274f),
                     f2(0.24192412881028413f, 0.24192412881028413f));
  p = ffma2(p, f, f2(0.6933164806648954f, 0.6933164806648954f));
  p = ffma2(p, f, f2(1.0f, 1.0f));
  const float2 pp = f2_split(p), yy = f2_split(y);
  // bits(magic) << 23 == 0 (mod 2^32): the shift leaves exactly round(x) << 23
  return make_float2(__int_as_float(__float_as_int(pp.x) + (__float_as_int(yy.x) << 23)),
                     __int_as_float(__float_as_int(pp.y) + (__float_as_int(yy.y) << 23)));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Byte offset of 16-byte chunk `chunk` (0..7) of row `row` inside a 128B-swizzled
// tile whose rows are 128 bytes (the TMA SWIZZLE_128B / UMMA SW128 K-major atom).
__device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t chunk) {
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

}  // namespace magi
