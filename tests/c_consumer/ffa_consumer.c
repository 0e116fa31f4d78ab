/* A plain C consumer of libmagiplan.so: what an FFI client of the reference
 * planner (proj/include/magiplan/magiplan.h, "C, Python (ctypes/cffi), or
 * any FFI-capable runtime", proj/README.md:11-14) links against after the
 * switch. No Python, no torch.
 *
 *   ffa_consumer plan            the reference's own planner calls (CPU):
 *                                mask parse / area / scenario plan; prints
 *                                "area <n> plan_bytes <n>"
 *   ffa_consumer ffa OUT.bin     the FFA forward + backward through the ABI on
 *                                cuda:0 with device buffers from cudaMalloc;
 *                                writes O (f32), LSE, dQ, dK, dV (f32) to OUT.bin
 *
 * Test infrastructure (tests/test_capi.py builds and runs it). */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "magiplan/magiplan.h"

#define CHECK(call)                                                            \
  do {                                                                         \
    magiplan_status s_ = (call);                                               \
    if (s_ != MAGIPLAN_OK) {                                                   \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)s_, magiplan_last_error()); \
      return 1;                                                                \
    }                                                                          \
  } while (0)
#define CUDA(call)                                                             \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));              \
      return 1;                                                                \
    }                                                                          \
  } while (0)

/* the case the test mirrors: S = 640, block-causal 128 plus one causal
 * slice over the first 200 rows (overlap: MULTIPLICITY), 4 q / 2 kv heads */
enum { S = 640, HQ = 4, HK = 2, D = 128, NSL = 6 };
static const int64_t kQ[NSL][2] = {{0, 128}, {128, 256}, {256, 384}, {384, 512}, {512, 640}, {0, 200}};
static const int64_t kK[NSL][2] = {{0, 128}, {0, 256}, {0, 384}, {0, 512}, {0, 640}, {0, 200}};
static const int32_t kT[NSL] = {0, 0, 0, 0, 0, 1};

/* deterministic inputs: a xorshift stream rounded to bf16 (the test
 * regenerates the same values) */
static uint32_t rng_state = 12345u;
static float next_uniform(void) {
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 17;
  rng_state ^= rng_state << 5;
  return (float)(rng_state >> 8) / 16777216.0f * 2.0f - 1.0f;
}
static uint16_t to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u); /* round to nearest even */
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static int run_plan(void) {
  magiplan_mask* mask = NULL;
  CHECK(magiplan_mask_parse(
      "{\"seqlen\": 32768, \"pattern\": \"block_causal\", \"params\": {\"block_size\": 4096}}", &mask));
  int64_t area = 0;
  CHECK(magiplan_mask_area(mask, MAGIPLAN_COUNT_MULTIPLICITY, &area));
  magiplan_mask_free(mask);
  magiplan_scenario* scen = NULL;
  CHECK(magiplan_scenario_parse(
      "{\"workload\": {\"mask\": {\"seqlen\": 131072, \"pattern\": \"block_causal\", \"params\": "
      "{\"block_size\": 8192}}, \"num_heads_q\": 48, \"num_heads_k\": 8, \"num_heads_v\": 8, "
      "\"head_dim\": 128}, \"cp_size\": 4}",
      ".", &scen));
  char* plan = NULL;
  CHECK(magiplan_scenario_plan(scen, &plan));
  printf("area %lld plan_bytes %zu\n", (long long)area, strlen(plan));
  magiplan_string_free(plan);
  magiplan_scenario_free(scen);
  return 0;
}

static int run_ffa(const char* path) {
  const size_t nq = (size_t)S * HQ * D, nk = (size_t)S * HK * D;
  uint16_t* hq = malloc(nq * 2);
  uint16_t* hk = malloc(nk * 2);
  uint16_t* hv = malloc(nk * 2);
  uint16_t* hdo = malloc(nq * 2);
  for (size_t i = 0; i < nq; ++i) hq[i] = to_bf16(next_uniform());
  for (size_t i = 0; i < nk; ++i) hk[i] = to_bf16(next_uniform());
  for (size_t i = 0; i < nk; ++i) hv[i] = to_bf16(next_uniform());
  for (size_t i = 0; i < nq; ++i) hdo[i] = to_bf16(next_uniform());
  (void)from_bf16;

  void *q, *k, *v, *dout, *out, *dq, *dk, *dv;
  float *lse, *delta;
  CUDA(cudaMalloc(&q, nq * 2));
  CUDA(cudaMalloc(&k, nk * 2));
  CUDA(cudaMalloc(&v, nk * 2));
  CUDA(cudaMalloc(&dout, nq * 2));
  CUDA(cudaMalloc(&out, nq * 4));
  CUDA(cudaMalloc(&dq, nq * 4));
  CUDA(cudaMalloc(&dk, nk * 4));
  CUDA(cudaMalloc(&dv, nk * 4));
  CUDA(cudaMalloc((void**)&lse, (size_t)HQ * S * 4));
  CUDA(cudaMalloc((void**)&delta, (size_t)HQ * S * 4));
  CUDA(cudaMemcpy(q, hq, nq * 2, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(k, hk, nk * 2, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(v, hv, nk * 2, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dout, hdo, nq * 2, cudaMemcpyHostToDevice));

  magiplan_ffa_plan* plan = NULL;
  CHECK(magiplan_ffa_plan_create(&kQ[0][0], &kK[0][0], kT, NSL, S, S, D, &plan));
  CHECK(magiplan_ffa_plan_prepare(plan));
  const float scale = 1.0f / sqrtf((float)D);
  cudaStream_t st;
  CUDA(cudaStreamCreate(&st));
  CHECK(magiplan_ffa_fwd(plan, q, k, v, out, lse, HQ, HK, scale, MAGIPLAN_F32, 0, st));
  CHECK(magiplan_ffa_bwd_preprocess(out, dout, delta, S, HQ, D, MAGIPLAN_F32, st));
  CHECK(magiplan_ffa_bwd(plan, q, k, v, lse, delta, dout, dq, dk, dv, HQ, HK, scale, MAGIPLAN_F32, 0, st));
  CUDA(cudaStreamSynchronize(st));

  float* buf = malloc(nq * 4);
  FILE* f = fopen(path, "wb");
  if (!f) return 1;
  CUDA(cudaMemcpy(buf, out, nq * 4, cudaMemcpyDeviceToHost));
  fwrite(buf, 4, nq, f);
  CUDA(cudaMemcpy(buf, lse, (size_t)HQ * S * 4, cudaMemcpyDeviceToHost));
  fwrite(buf, 4, (size_t)HQ * S, f);
  CUDA(cudaMemcpy(buf, dq, nq * 4, cudaMemcpyDeviceToHost));
  fwrite(buf, 4, nq, f);
  CUDA(cudaMemcpy(buf, dk, nk * 4, cudaMemcpyDeviceToHost));
  fwrite(buf, 4, nk, f);
  CUDA(cudaMemcpy(buf, dv, nk * 4, cudaMemcpyDeviceToHost));
  fwrite(buf, 4, nk, f);
  fclose(f);
  magiplan_ffa_plan_free(plan);
  printf("ffa ok\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 2 && strcmp(argv[1], "plan") == 0) return run_plan();
  if (argc >= 3 && strcmp(argv[1], "ffa") == 0) return run_ffa(argv[2]);
  fprintf(stderr, "usage: %s plan | ffa OUT.bin\n", argv[0]);
  return 2;
}
