/* TEST INFRASTRUCTURE ONLY — CPU oracle for Flexible Flash Attention.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this file's library; the product path never does.
 *
 * The reference (magiplan, /root/reference/proj) contains no attention
 * arithmetic, so the numerics below are a restatement of the
 * standard attention definition over the reference's mask semantics:
 *   - slice membership: AttnSlice::row_cols (proj/src/mask.cpp:74-84) —
 *     allowed local columns [lo, hi) with lo = min(r, lk) for INV/BI,
 *     hi = clamp(r + lk - lq + 1, 0, lk) for CAUSAL/BI;
 *   - overlapping slices count with MULTIPLICITY ("what a kernel actually
 *     computes", proj/include/magiplan/mask.hpp:85): a pair covered by m
 *     slices enters the softmax m times;
 *   - forward per row i and head h: LSE = ln sum_j exp(scale q_i.k_j),
 *     O = sum_j exp(scale q_i.k_j - LSE) v_j; empty rows O = 0, LSE = -inf;
 *   - GQA: key/value head = h / (hq / hk);
 *   - backward (PAPER.md:1082, 5 matmuls): D_i = dO_i.O_i,
 *     dS_ij = P_ij (dO_i.v_j - D_i), dQ = scale dS K, dK = scale dS^T Q,
 *     dV = P^T dO, dK/dV summed over the query heads of each group.
 * Mask semantics are pinned against the compiled reference (tests/golden);
 * the numerics themselves are "parity unpinned" by the reference (it has no
 * golden numerics) and are cross-checked against an independent dense torch
 * float64 formulation and against PyTorch's own scaled_dot_product_attention
 * (float64, autograd; every non-overlapping case, 1e-9) in
 * tests/test_oracle.py.
 *
 * Accumulation is double (acc_f32 == 0) or float (acc_f32 == 1; the CPU
 * baseline timed by bench.py). Inputs are float arrays holding the
 * bf16-rounded tensors; layouts are token-major [tokens, heads, d], LSE
 * [heads, tokens].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_API __attribute__((visibility("default")))

/* mask.cpp:74-84 restated in global coordinates; returns hi - lo (<= 0: empty). */
static int64_t slice_row_cols(int64_t qs, int64_t qe, int64_t ks, int64_t ke, int32_t type,
                              int64_t q, int64_t* lo_out) {
  if (q < qs || q >= qe) return 0;
  const int64_t lq = qe - qs, lk = ke - ks, r = q - qs;
  int64_t lo = 0, hi = lk;
  if (type == 2 || type == 3) lo = r < lk ? r : lk;
  if (type == 1 || type == 3) {
    hi = r + lk - lq + 1;
    if (hi < 0) hi = 0;
    if (hi > lk) hi = lk;
  }
  *lo_out = ks + lo;
  return hi - lo;
}

ORACLE_API int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

ORACLE_API int oracle_row_allowed(int64_t qs, int64_t qe, int64_t ks, int64_t ke, int32_t type,
                                  int64_t q, int64_t k) {
  int64_t lo;
  const int64_t n = slice_row_cols(qs, qe, ks, ke, type, q, &lo);
  return n > 0 && k >= lo && k < lo + n;
}

static double dot(const float* a, const float* b, int d) {
  double s = 0;
  for (int i = 0; i < d; ++i) s += (double)a[i] * (double)b[i];
  return s;
}
static float dotf(const float* a, const float* b, int d) {
  float s = 0;
  for (int i = 0; i < d; ++i) s += a[i] * b[i];
  return s;
}

/* Forward. out: [sq, hq, d] double, lse: [hq, sq] double. */
ORACLE_API void oracle_ffa_fwd(const float* q, const float* k, const float* v, int64_t sq,
                               int64_t sk, int64_t hq, int64_t hk, int d, const int64_t* qr,
                               const int64_t* kr, const int32_t* types, int64_t ns, double scale,
                               double* out, double* lse, int acc_f32) {
  (void)sk;
  const int64_t group = hq / hk;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t w = 0; w < sq * hq; ++w) {
    const int64_t i = w / hq, h = w % hq, g = h / group;
    const float* qi = q + (i * hq + h) * d;
    double* oi = out + (i * hq + h) * d;
    double acc[256];
    float accf[256];
    for (int x = 0; x < d; ++x) acc[x] = 0, accf[x] = 0;
    double m = -INFINITY, l = 0;
    float mf = -INFINITY, lf = 0;
    for (int64_t s = 0; s < ns; ++s) {
      int64_t lo;
      const int64_t n = slice_row_cols(qr[2 * s], qr[2 * s + 1], kr[2 * s], kr[2 * s + 1],
                                       types[s], i, &lo);
      for (int64_t j = lo; j < lo + n; ++j) {
        const float* kj = k + (j * hk + g) * d;
        const float* vj = v + (j * hk + g) * d;
        if (acc_f32) {
          const float x = dotf(qi, kj, d) * (float)scale;
          const float mn = x > mf ? x : mf;
          const float a = expf(mf - mn), p = expf(x - mn);
          lf = lf * a + p;
          for (int c = 0; c < d; ++c) accf[c] = accf[c] * a + p * vj[c];
          mf = mn;
        } else {
          const double x = dot(qi, kj, d) * scale;
          const double mn = x > m ? x : m;
          const double a = exp(m - mn), p = exp(x - mn);
          l = l * a + p;
          for (int c = 0; c < d; ++c) acc[c] = acc[c] * a + p * vj[c];
          m = mn;
        }
      }
    }
    if (acc_f32) {
      m = mf;
      l = lf;
      for (int c = 0; c < d; ++c) acc[c] = accf[c];
    }
    if (l > 0) {
      for (int c = 0; c < d; ++c) oi[c] = acc[c] / l;
      lse[h * sq + i] = m + log(l);
    } else {
      for (int c = 0; c < d; ++c) oi[c] = 0;
      lse[h * sq + i] = -INFINITY;
    }
  }
}

/* Backward. out / lse from oracle_ffa_fwd; dout float [sq, hq, d].
 * dq: [sq, hq, d], dk/dv: [sk, hk, d] double (overwritten). Parallel over key/value
 * heads so every dK/dV element has one writer. */
ORACLE_API void oracle_ffa_bwd(const float* q, const float* k, const float* v, const double* out,
                               const double* lse, const float* dout, int64_t sq, int64_t sk,
                               int64_t hq, int64_t hk, int d, const int64_t* qr, const int64_t* kr,
                               const int32_t* types, int64_t ns, double scale, double* dq,
                               double* dk, double* dv) {
  const int64_t group = hq / hk;
  memset(dq, 0, sizeof(double) * sq * hq * d);
  memset(dk, 0, sizeof(double) * sk * hk * d);
  memset(dv, 0, sizeof(double) * sk * hk * d);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t g = 0; g < hk; ++g) {
    for (int64_t h = g * group; h < (g + 1) * group; ++h) {
      for (int64_t i = 0; i < sq; ++i) {
        const double L = lse[h * sq + i];
        if (L == -INFINITY) continue;
        const float* qi = q + (i * hq + h) * d;
        const float* gi = dout + (i * hq + h) * d;
        const double* oi = out + (i * hq + h) * d;
        double* dqi = dq + (i * hq + h) * d;
        double D = 0;
        for (int c = 0; c < d; ++c) D += (double)gi[c] * oi[c];
        for (int64_t s = 0; s < ns; ++s) {
          int64_t lo;
          const int64_t n = slice_row_cols(qr[2 * s], qr[2 * s + 1], kr[2 * s], kr[2 * s + 1],
                                           types[s], i, &lo);
          for (int64_t j = lo; j < lo + n; ++j) {
            const float* kj = k + (j * hk + g) * d;
            const float* vj = v + (j * hk + g) * d;
            const double p = exp(dot(qi, kj, d) * scale - L);
            const double dp = dot(gi, vj, d);
            const double ds = p * (dp - D);
            double* dkj = dk + (j * hk + g) * d;
            double* dvj = dv + (j * hk + g) * d;
            for (int c = 0; c < d; ++c) {
              dqi[c] += scale * ds * kj[c];
              dkj[c] += scale * ds * qi[c];
              dvj[c] += p * gi[c];
            }
          }
        }
      }
    }
  }
}
