/*
 * sage3_oracle.c — CPU ORACLE for the SageAttention3 FP4 attention forward (arXiv 2505.11594).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (paper_2505_11594_b200/) never
 * links, imports or executes anything under oracle/, and this file shares no code, header, table or
 * constant generator with it.
 *
 * What it computes: Algorithm 1 of the paper, step by step, in the paper's order and
 * notation; smoothing Q (Alg1 L5's q̄, L8's GEMV) is a switch (off on the north_star path):
 *   Alg1 L2    K = K - mean(K)                                   -> oracle_kmean, oracle_quantize_head
 *   Eq. 1      s = max|X|/6, X̂ = ⌈X/s⌋ over 1x16 blocks -> phi_nvfp4
 *   Alg1 L5    q̄_i = mean(Q_i), φ(Q_i - q̄_i) (smoothing Q, optional) -> oracle_qmean_tile, oracle_quantize_head_sq
 *   Tab1a      MXFP4 instead of NVFP4 for every φ (ablation, fmt = 1)    -> oracle_quantize_head_fmt, oracle_attn_fwd_fmt
 *   Alg1 L7    φ(K_j^T) along d, φ(V_j) along tokens      -> oracle_quantize_head
 *   Alg1 L8    S = FP4MM(Q̂, s_Q, K̂, s_K) [+ GEMV(q̄_i, K_j^T)]    -> attn_row (exact in fp64)
 *   Alg1 L9    m, P̃ = exp(S - m), l = e^{m_old-m} l + rowsum(P̃)   -> attn_row
 *   Alg1 L10   s_P1 = rowmax(P̃)/(448*6), P̃2 = P̃/s_P1, (s_P2, P̂2) = φ(P̃2)   (§3.2)
 *   Alg1 L11   O = diag(e^{m_old-m}) O + FP4MM(P̂2, s_P2, V̂, s_V) * s_P1
 *   Alg1 L13   O = diag(l)^-1 O
 *   (variant)  p_mode LAZY: the first-level P scale per row per reference epoch instead of per tile
 *              (reading n1)            -> attn_row_lazy
 * Precision: every quantizer is bit-exact fp32 arithmetic; P̃, P̃2 and s_P1 are fp32 as P:188 states;
 * everything else is fp64.  The readings of points the paper leaves open (rounding modes, the 1/6
 * multiply, softmax scale, causal mask, padding, s_P1 granularity) are SURVEY.md §8(c) c1-c16 and are
 * listed in DESIGN.md §3.  Each function below names the passage it follows.
 *
 * Build: gcc -O2 -std=c11 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC (no FTZ/DAZ).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------------------------------
 * (1) Codecs.  E2M1 = the 4-bit element type of NVFP4, "only 15 representable values"
 * (P:47).  E4M3 = the FP8 scale type, max finite 448 ("[0, 448 x 6]").
 * Encoding is brute-force nearest over the value table, ties to the even code (even mantissa),
 * saturating to the largest finite magnitude (readings c1, c2).  The sign is kept on underflow
 * (so -0.2 encodes to the negative-zero code 0x8), matching the hardware convert (reading c1).
 * ------------------------------------------------------------------------------------------------ */
static const double E2M1_MAG[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};

EXPORT double oracle_e2m1_decode(uint8_t code) {
  double m = E2M1_MAG[code & 7];
  return (code & 8) ? -m : m;
}

EXPORT uint8_t oracle_e2m1_encode(float x) {
  double a = fabs((double)x);
  if (a > 6.0) a = 6.0; /* saturate first: for huge |x| the fp64 differences below are no longer exact */
  int best = 0;
  double best_err = INFINITY;
  for (int c = 0; c < 8; ++c) {
    double err = fabs(a - E2M1_MAG[c]);
    /* strictly better, or a tie resolved toward the even code (mantissa bit = code & 1) */
    if (err < best_err || (err == best_err && (c & 1) == 0)) {
      best = c;
      best_err = err;
    }
  }
  return (uint8_t)(best | (signbit(x) ? 8 : 0));
}

EXPORT double oracle_e4m3_decode(uint8_t code) {
  int e = (code >> 3) & 15, m = code & 7;
  double v;
  if ((code & 0x7F) == 0x7F) return NAN; /* the only NaN encodings; never produced by the encoder */
  if (e == 0)
    v = ldexp((double)m, -9); /* subnormal: m * 2^-9 */
  else
    v = ldexp(1.0 + m / 8.0, e - 7); /* bias 7 */
  return (code & 0x80) ? -v : v;
}

EXPORT uint8_t oracle_e4m3_encode(float x) {
  double a = fabs((double)x);
  if (a > 448.0) a = 448.0; /* saturate first (satfinite), keeps the differences below exact */
  int best = 0;
  double best_err = INFINITY;
  for (int c = 0; c < 0x7F; ++c) { /* all 127 non-negative finite codes 0x00..0x7E */
    double err = fabs(a - oracle_e4m3_decode((uint8_t)c));
    if (err < best_err || (err == best_err && (c & 1) == 0)) {
      best = c;
      best_err = err;
    }
  }
  return (uint8_t)(best | (signbit(x) ? 0x80 : 0));
}

/* Count distinct non-negative values of a format inside [lo, hi] (appendix, P:1328 / P:1333). */
EXPORT int oracle_enumerate(int fmt /*0=e2m1 (signed), 1=e4m3*/, double lo, double hi, double* out_values) {
  int n = 0;
  double vals[256];
  int ncode = fmt == 0 ? 16 : 256;
  for (int c = 0; c < ncode; ++c) {
    double v = fmt == 0 ? oracle_e2m1_decode((uint8_t)c) : oracle_e4m3_decode((uint8_t)c);
    if (isnan(v) || v < lo || v > hi) continue;
    int seen = 0;
    for (int i = 0; i < n; ++i)
      if (vals[i] == v) seen = 1;
    if (!seen) vals[n++] = v;
  }
  /* insertion sort for a stable, sorted listing */
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && vals[j - 1] > vals[j]; --j) {
      double t = vals[j];
      vals[j] = vals[j - 1];
      vals[j - 1] = t;
    }
  if (out_values)
    for (int i = 0; i < n; ++i) out_values[i] = vals[i];
  return n;
}

/* ------------------------------------------------------------------------------------------------
 * (2) φ on one 1x16 block, Eq. 1: s = max(|X|)/6, X̂ = ⌈X/s⌋, s stored as E4M3.
 * Readings: c3 s32 = fl32(amax * fl32(1/6)); c2 s = E4M3-RNE-sat(s32); c5 s == 0 -> all codes 0;
 * c4 y = fl32(x * fl32(1/s)).  fp32 arithmetic, no contraction (-ffp-contract=off).
 * ------------------------------------------------------------------------------------------------ */
EXPORT void oracle_phi_nvfp4(const float* x, uint8_t* codes, uint8_t* scale_code) {
  float amax = 0.0f;
  for (int i = 0; i < 16; ++i) {
    float a = fabsf(x[i]);
    if (a > amax) amax = a;
  }
  const float one_sixth = 1.0f / 6.0f; /* fl32(1/6) = 0x3E2AAAAB */
  float s32 = amax * one_sixth;
  uint8_t sc = oracle_e4m3_encode(s32);
  float s = (float)oracle_e4m3_decode(sc); /* exact: every E4M3 value is an fp32 */
  *scale_code = sc;
  if (s == 0.0f) {
    for (int i = 0; i < 16; ++i) codes[i] = 0;
    return;
  }
  float r = 1.0f / s; /* IEEE correctly rounded reciprocal */
  for (int i = 0; i < 16; ++i) {
    float y = x[i] * r;
    codes[i] = oracle_e2m1_encode(y);
  }
}

/* MXFP4 ablation (1x32 blocks, E8M0 scales; SPEC S:70-78 rounds the scale UP to a power of 2).
 * Scale code = biased exponent e (value 2^(e-127)); s = 0 is not representable, so an all-zero
 * block stores the smallest scale with zero codes. */
EXPORT void oracle_phi_mxfp4(const float* x, uint8_t* codes, uint8_t* scale_code) {
  float amax = 0.0f;
  for (int i = 0; i < 32; ++i) {
    float a = fabsf(x[i]);
    if (a > amax) amax = a;
  }
  float s32 = amax * (1.0f / 6.0f);
  if (s32 == 0.0f) {
    *scale_code = 0;
    for (int i = 0; i < 32; ++i) codes[i] = 0;
    return;
  }
  int e;
  double fr = frexp((double)s32, &e); /* s32 = fr * 2^e, fr in [0.5,1) */
  int p = (fr == 0.5) ? e - 1 : e;    /* smallest power of two >= s32 is 2^p */
  if (p < -127) p = -127;
  if (p > 127) p = 127;
  *scale_code = (uint8_t)(p + 127);
  float s = (float)ldexp(1.0, p);
  for (int i = 0; i < 32; ++i) codes[i] = oracle_e2m1_encode(x[i] / s); /* power of 2: exact */
}

/* ------------------------------------------------------------------------------------------------
 * Smoothing K, Alg1 L2: km[c] = mean over the N real tokens of K[:, c].
 * Reading c10: fixed order — fp64 sequential sum inside each 128-token chunk (ascending tokens),
 * chunk sums added in ascending chunk order, divided by N in fp64, rounded once to fp32.
 * ------------------------------------------------------------------------------------------------ */
EXPORT void oracle_kmean(const float* K, int N, int d, float* km) {
  for (int c = 0; c < d; ++c) {
    double total = 0.0;
    for (int c0 = 0; c0 < N; c0 += 128) {
      double chunk = 0.0;
      int c1 = c0 + 128 < N ? c0 + 128 : N;
      for (int n = c0; n < c1; ++n) chunk += (double)K[(size_t)n * d + c];
      total += chunk;
    }
    km[c] = (float)(total / (double)N);
  }
}

/* ------------------------------------------------------------------------------------------------
 * Quantize one head, Alg1 L2 + L5 (without q̄) + L7.  Logical layouts (one 4-bit code per byte):
 *   q_codes, k_codes [Np][d], q_sf, k_sf [Np][d/16]      (blocks along d, reading c6)
 *   v_codes [d][Np] (V transposed), v_sf [d][Np/16] (blocks along tokens)
 * Np = round_up(N, 128); padded tokens get zero codes and zero scales (reading c13).
 * Inputs are fp32 arrays holding the exact bf16/fp16 input values.
 * smooth_k = 0 disables Alg1 L2 (ablation).
 * ------------------------------------------------------------------------------------------------ */
/* ------------------------------------------------------------------------------------------------
 * Smoothing Q, Alg1 L5 (SageAttention2): q̄_i = mean(Q_i) over the rows of query tile i (B_q = 128
 * rows, the kernel's query tile) that exist (rows >= N are padding, reading c13).  Same fixed order as the
 * K mean (reading c10): fp64 sequential sum over the tile's rows in ascending order, divided by the row
 * count in fp64, rounded once to fp32.
 * ------------------------------------------------------------------------------------------------ */
EXPORT void oracle_qmean_tile(const float* Q, int N, int d, int tile, float* qm) {
  int r0 = tile * 128, r1 = r0 + 128 < N ? r0 + 128 : N;
  for (int c = 0; c < d; ++c) {
    double acc = 0.0;
    for (int n = r0; n < r1; ++n) acc += (double)Q[(size_t)n * d + c];
    qm[c] = (float)(acc / (double)(r1 - r0));
  }
}

/* ------------------------------------------------------------------------------------------------
 * Quantize one head, Alg1 L2 + L5 + L7.  Logical layouts (one 4-bit code per byte):
 *   q_codes, k_codes [Np][d], q_sf, k_sf [Np][d/16]      (blocks along d, reading c6)
 *   v_codes [d][Np] (V transposed), v_sf [d][Np/16] (blocks along tokens)
 * Np = round_up(N, 128); padded tokens get zero codes and zero scales (reading c13).
 * Inputs are fp32 arrays holding the exact bf16/fp16 input values.
 * smooth_k = 0 disables Alg1 L2 (ablation).  fmt = 1 is the MXFP4 ablation (Tab1a: 1x32
 * blocks with E8M0 scales rounded up, oracle_phi_mxfp4; scale arrays then have d/32 resp. Np/32 columns).
 * smooth_q = 1 enables Alg1 L5: Q_i - q̄_i is
 * quantized (x = fl32(Q - q̄), like K - km) and q̄ [Np/128][d] is returned in q_mean_out; ks_out [Np][d]
 * (nullable) receives the smoothed K = fl32(K - km) in full precision (zero rows beyond N), the K_j of
 * Alg1 L8's GEMV.
 * ------------------------------------------------------------------------------------------------ */
EXPORT void oracle_quantize_head_fmt(const float* Q, const float* K, const float* V, int N, int d, int smooth_k,
                                     int smooth_q, int fmt, uint8_t* q_codes, uint8_t* q_sf, uint8_t* k_codes,
                                     uint8_t* k_sf, uint8_t* v_codes, uint8_t* v_sf, float* km_out,
                                     float* q_mean_out, float* ks_out) {
  const int Np = (N + 127) / 128 * 128;
  const int G = fmt ? 32 : 16; /* block size: NVFP4 1x16 (E4M3 scales), MXFP4 1x32 (E8M0 scales) */
  const int C = d / G;
  float* km = (float*)calloc((size_t)d, sizeof(float));
  float* qm = (float*)calloc((size_t)d, sizeof(float));
  if (smooth_k) oracle_kmean(K, N, d, km);
  if (km_out) memcpy(km_out, km, sizeof(float) * (size_t)d);
  memset(q_codes, 0, (size_t)Np * d);
  memset(k_codes, 0, (size_t)Np * d);
  memset(v_codes, 0, (size_t)Np * d);
  memset(q_sf, 0, (size_t)Np * C);
  memset(k_sf, 0, (size_t)Np * C);
  memset(v_sf, 0, (size_t)d * (Np / G));
  if (q_mean_out) memset(q_mean_out, 0, sizeof(float) * (size_t)(Np / 128) * d);
  if (ks_out) memset(ks_out, 0, sizeof(float) * (size_t)Np * d);
  float blk[32];
  for (int n = 0; n < N; ++n) {
    if (n % 128 == 0 && smooth_q) {
      oracle_qmean_tile(Q, N, d, n / 128, qm);
      if (q_mean_out) memcpy(&q_mean_out[(size_t)(n / 128) * d], qm, sizeof(float) * (size_t)d);
    }
    for (int b = 0; b < C; ++b) {
      for (int i = 0; i < G; ++i) blk[i] = Q[(size_t)n * d + b * G + i] - qm[b * G + i]; /* fl32; qm = 0 if off */
      if (fmt) oracle_phi_mxfp4(blk, &q_codes[(size_t)n * d + b * G], &q_sf[(size_t)n * C + b]);
      else oracle_phi_nvfp4(blk, &q_codes[(size_t)n * d + b * G], &q_sf[(size_t)n * C + b]);
      for (int i = 0; i < G; ++i) blk[i] = K[(size_t)n * d + b * G + i] - km[b * G + i]; /* fl32 */
      if (ks_out) memcpy(&ks_out[(size_t)n * d + b * G], blk, sizeof(float) * (size_t)G);
      if (fmt) oracle_phi_mxfp4(blk, &k_codes[(size_t)n * d + b * G], &k_sf[(size_t)n * C + b]);
      else oracle_phi_nvfp4(blk, &k_codes[(size_t)n * d + b * G], &k_sf[(size_t)n * C + b]);
    }
  }
  for (int c = 0; c < d; ++c) {
    for (int t0 = 0; t0 < Np; t0 += G) {
      for (int i = 0; i < G; ++i) blk[i] = (t0 + i < N) ? V[(size_t)(t0 + i) * d + c] : 0.0f;
      if (fmt) oracle_phi_mxfp4(blk, &v_codes[(size_t)c * Np + t0], &v_sf[(size_t)c * (Np / G) + t0 / G]);
      else oracle_phi_nvfp4(blk, &v_codes[(size_t)c * Np + t0], &v_sf[(size_t)c * (Np / G) + t0 / G]);
    }
  }
  free(km);
  free(qm);
}

EXPORT void oracle_quantize_head_sq(const float* Q, const float* K, const float* V, int N, int d, int smooth_k,
                                    int smooth_q, uint8_t* q_codes, uint8_t* q_sf, uint8_t* k_codes, uint8_t* k_sf,
                                    uint8_t* v_codes, uint8_t* v_sf, float* km_out, float* q_mean_out,
                                    float* ks_out) {
  oracle_quantize_head_fmt(Q, K, V, N, d, smooth_k, smooth_q, 0, q_codes, q_sf, k_codes, k_sf, v_codes, v_sf, km_out,
                           q_mean_out, ks_out);
}

EXPORT void oracle_quantize_head(const float* Q, const float* K, const float* V, int N, int d, int smooth_k,
                                 uint8_t* q_codes, uint8_t* q_sf, uint8_t* k_codes, uint8_t* k_sf,
                                 uint8_t* v_codes, uint8_t* v_sf, float* km_out) {
  oracle_quantize_head_sq(Q, K, V, N, d, smooth_k, 0, q_codes, q_sf, k_codes, k_sf, v_codes, v_sf, km_out, NULL,
                          NULL);
}

/* Dequantize (Eq. 2): X' = s * X̂, exact in fp64. rows x cols codes, blocks of 16 along cols (E4M3
 * scales) or, fmt = 1, blocks of 32 with E8M0 scales (2^(code - 127)). */
EXPORT void oracle_dequant_fmt(const uint8_t* codes, const uint8_t* sf, int rows, int cols, int fmt, double* out) {
  const int G = fmt ? 32 : 16;
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      const uint8_t sc = sf[(size_t)r * (cols / G) + c / G];
      const double s = fmt ? ldexp(1.0, (int)sc - 127) : oracle_e4m3_decode(sc);
      out[(size_t)r * cols + c] = oracle_e2m1_decode(codes[(size_t)r * cols + c]) * s;
    }
}
EXPORT void oracle_dequant(const uint8_t* codes, const uint8_t* sf, int rows, int cols, double* out) {
  oracle_dequant_fmt(codes, sf, rows, cols, 0, out);
}

/* FP4MM, Eq. 3: C = φ^-1(A) φ^-1(B)^T, triple loop in fp64 (exact for NVFP4 operands
 * with K <= 128: products are multiples of 2^-20 below 2^23, so sums need <= 50 bits). */
EXPORT void oracle_fp4mm(const uint8_t* a_codes, const uint8_t* a_sf, const uint8_t* b_codes, const uint8_t* b_sf,
                         int M, int N, int K, double* Cout) {
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0.0;
      for (int k = 0; k < K; ++k) {
        double a = oracle_e2m1_decode(a_codes[(size_t)m * K + k]) * oracle_e4m3_decode(a_sf[(size_t)m * (K / 16) + k / 16]);
        double b = oracle_e2m1_decode(b_codes[(size_t)n * K + k]) * oracle_e4m3_decode(b_sf[(size_t)n * (K / 16) + k / 16]);
        acc += a * b;
      }
      Cout[(size_t)m * N + n] = acc;
    }
}

/* ------------------------------------------------------------------------------------------------
 * Two-level quantization of one row of one KV tile, §3.2 Eq., Alg1 L10:
 *   s_P1 = rowmax(P̃)/(448*6)   P̃2 = P̃/s_P1   (s_P2, P̂2) = φ(P̃2)
 * P̃, P̃2, s_P1 are fp32.  n must be a multiple of 16.  Returns s_P1; if the row is all zero
 * (every P̃ underflowed) s_P1 = 0 and all codes/scales are 0 — the tile then contributes nothing.
 * p_mode 1 = direct φ(P̃) baseline (Tab1b), returns s_P1 = 1.
 * ------------------------------------------------------------------------------------------------ */
#define PMODE_TWO_LEVEL 0
#define PMODE_DIRECT 1
#define PMODE_NONE 2
#define PMODE_LAZY 3 /* NEXT #2 throughput variant (not the paper's Alg1 L10): see attn_row_lazy */
#define PMODE_QSUM 4 /* NEXT #2 throughput variant (not the paper's Alg1 L9): two-level P exactly as Alg1 L10, but
                      * the row sum l accumulates the QUANTIZED P (s_P1 · Σ deq(P̂2)), which the GPU obtains from
                      * the tensor core (P̂2 times a ones column) instead of summing the unquantized P̃ (reading c9).
                      * O/l is then the normalised average of V with exactly the weights the PV product used. */

EXPORT float oracle_two_level_row_fmt(const float* P, int n, int p_mode, int fmt, uint8_t* codes, uint8_t* sf) {
  const int G = fmt ? 32 : 16;
  float p2[32];
  if (p_mode == PMODE_DIRECT) {
    for (int b = 0; b < n; b += G) {
      if (fmt) oracle_phi_mxfp4(&P[b], &codes[b], &sf[b / G]);
      else oracle_phi_nvfp4(&P[b], &codes[b], &sf[b / G]);
    }
    return 1.0f;
  }
  float pmax = 0.0f;
  for (int k = 0; k < n; ++k)
    if (P[k] > pmax) pmax = P[k];
  float sP1 = pmax / 2688.0f; /* 448 * 6 */
  if (sP1 == 0.0f) {
    memset(codes, 0, (size_t)n);
    memset(sf, 0, (size_t)n / G);
    return 0.0f;
  }
  for (int b = 0; b < n; b += G) { /* (PMODE_QSUM quantizes exactly as the two-level mode) */
    for (int i = 0; i < G; ++i) p2[i] = P[b + i] / sP1;
    if (fmt) oracle_phi_mxfp4(p2, &codes[b], &sf[b / G]);
    else oracle_phi_nvfp4(p2, &codes[b], &sf[b / G]);
  }
  return sP1;
}
EXPORT float oracle_two_level_row(const float* P, int n, int p_mode, uint8_t* codes, uint8_t* sf) {
  return oracle_two_level_row_fmt(P, n, p_mode, 0, codes, sf);
}

/* ------------------------------------------------------------------------------------------------
 * Decision sensitivity of φ (TEST INFRASTRUCTURE for the GPU parity bound; it does not
 * change any result above).  The GPU evaluates P̃2 (or P̃) with its own exp2 and fp32 S accumulation, so
 * its values differ from the oracle's by a relative amount below `delta`.  When a value sits that close
 * to an E2M1 rounding midpoint (or a block amax/6 that close to an E4M3 midpoint / power of two), the two
 * sides may legitimately pick adjacent codes.  For every element this returns dq[i] = the spread of its
 * dequantized value q_i·s over all inputs within a relative delta of x (every element and the block amax
 * moving independently); dq[i] = 0 whenever the decision is the same for all of them.  Both codecs and
 * the scale rule are monotone, so the extreme perturbations bound every reachable decision.
 * ------------------------------------------------------------------------------------------------ */
static double phi_scale_of(double amax, int fmt) {
  const float s32 = (float)amax * (1.0f / 6.0f);
  if (!fmt) return oracle_e4m3_decode(oracle_e4m3_encode(s32));
  if (s32 == 0.0f) return 0.0;
  int e;
  double fr = frexp((double)s32, &e);
  int p = (fr == 0.5) ? e - 1 : e;
  if (p < -127) p = -127;
  if (p > 127) p = 127;
  return ldexp(1.0, p);
}
EXPORT void oracle_phi_sensitivity(const float* x, int G, int fmt, double delta, double* dq) {
  double amax = 0.0;
  for (int i = 0; i < G; ++i)
    if (fabs((double)x[i]) > amax) amax = fabs((double)x[i]);
  const double sc[2] = {phi_scale_of(amax * (1.0 - delta), fmt), phi_scale_of(amax * (1.0 + delta), fmt)};
  for (int i = 0; i < G; ++i) {
    double lo = INFINITY, hi = -INFINITY;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        double v = 0.0;
        if (sc[a] != 0.0) {
          const float xv = (float)((double)x[i] * (b ? 1.0 + delta : 1.0 - delta));
          const float y = fmt ? (float)((double)xv / sc[a]) : xv * (1.0f / (float)sc[a]);
          v = oracle_e2m1_decode(oracle_e2m1_encode(y)) * sc[a];
        }
        if (v < lo) lo = v;
        if (v > hi) hi = v;
      }
    dq[i] = hi - lo;
  }
}

/* ------------------------------------------------------------------------------------------------
 * NEXT #2 variant (reading n1; NOT the paper's Alg1 L10): two-level P whose first level is a
 * lazily moved per-row reference r instead of each tile's own row max.  Per KV tile j, after S (Alg1 L8):
 *   if r = -inf or log2(e)·scale·(tmax_j - r) > LAZY_TAU:  O *= exp(scale(r - tmax_j)), l *= the same,
 *                                                          r = tmax_j        (the reference moves up)
 *   P̃2 = fl32(LAZY_TOP · exp(scale(S - r)))    LAZY_TOP = 2688 / 2^LAZY_TAU = 10.5, so P̃2 <= 2688 always
 *                                               (tmax_j <= r + LAZY_TAU / (log2(e)·scale))
 *   l += Σ P̃2 (unquantized, as reading c9);  (s_P2, P̂2) = φ(P̃2) per 16 (or 32, MXFP4) keys (Alg1 L10's
 *   second level);  O += FP4MM(P̂2, s_P2, V̂, s_V)   (no per-tile first-level factor)
 * and O/l at the end; lse = scale·r + ln(l / LAZY_TOP).  O/l equals Alg1's up to quantization: every tile of
 * an epoch shares the scale 2^-LAZY_TAU·2688·exp(scale(m - r)) relative to P̃, so the tensor core can
 * accumulate O across tiles (the GPU keeps O in TMEM) and only a moving reference costs a rescale.
 * ------------------------------------------------------------------------------------------------ */
#define LAZY_TAU 8.0
#define LAZY_TOP 10.5 /* 2688 * 2^-8, exact */
static void attn_row_lazy(const double* Qrow, const double* Kd, const double* Vt, int N, int Np, int d, int Bkv,
                          int causal, int qi, double scale, const float* qbar, const float* Ks, int fmt, double* O,
                          double* lse, double delta, double* amb) {
  const int G = fmt ? 32 : 16;
  double r = -INFINITY, l = 0.0;
  double* S = (double*)malloc(sizeof(double) * (size_t)Bkv);
  float* P2 = (float*)malloc(sizeof(float) * (size_t)Bkv);
  uint8_t* pc = (uint8_t*)malloc((size_t)Bkv);
  uint8_t* ps = (uint8_t*)malloc((size_t)Bkv / 16 + 1);
  double* dq = amb ? (double*)malloc(sizeof(double) * (size_t)Bkv) : NULL;
  for (int c = 0; c < d; ++c) O[c] = 0.0;
  if (amb)
    for (int c = 0; c < d; ++c) amb[c] = 0.0;
  int kv_end = causal ? (qi + 1 < N ? qi + 1 : N) : N;
  for (int j0 = 0; j0 < kv_end; j0 += Bkv) {
    double tmax = -INFINITY;
    for (int t = 0; t < Bkv; ++t) { /* Alg1 L8, exactly as attn_row */
      int key = j0 + t;
      if (key >= kv_end || key >= Np) {
        S[t] = -INFINITY;
        continue;
      }
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += Qrow[c] * Kd[(size_t)key * d + c];
      if (qbar) {
        double g = 0.0;
        for (int c = 0; c < d; ++c) g += (double)qbar[c] * (double)Ks[(size_t)key * d + c];
        acc += g;
      }
      S[t] = acc;
      if (acc > tmax) tmax = acc;
    }
    if (r == -INFINITY || (tmax - r) * scale / log(2.0) > LAZY_TAU) { /* move the reference */
      double a = (r == -INFINITY) ? 0.0 : exp(scale * (r - tmax));
      for (int c = 0; c < d; ++c) O[c] *= a;
      if (amb)
        for (int c = 0; c < d; ++c) amb[c] *= a;
      l *= a;
      r = tmax;
    }
    for (int t = 0; t < Bkv; ++t) {
      P2[t] = (S[t] == -INFINITY) ? 0.0f : (float)(LAZY_TOP * exp(scale * (S[t] - r)));
      l += (double)P2[t];
    }
    for (int b = 0; b < Bkv; b += G) {
      if (fmt) oracle_phi_mxfp4(&P2[b], &pc[b], &ps[b / G]);
      else oracle_phi_nvfp4(&P2[b], &pc[b], &ps[b / G]);
      if (amb) oracle_phi_sensitivity(&P2[b], G, fmt, delta, &dq[b]);
    }
    if (amb)
      for (int c = 0; c < d; ++c)
        for (int t = 0; t < Bkv && j0 + t < Np; ++t) amb[c] += dq[t] * fabs(Vt[(size_t)c * Np + j0 + t]);
    for (int c = 0; c < d; ++c) {
      double pv = 0.0;
      for (int t = 0; t < Bkv; ++t) {
        int key = j0 + t;
        if (key >= Np) break;
        double p = oracle_e2m1_decode(pc[t]) * (fmt ? ldexp(1.0, (int)ps[t / 32] - 127) : oracle_e4m3_decode(ps[t / 16]));
        pv += p * Vt[(size_t)c * Np + key];
      }
      O[c] += pv;
    }
  }
  for (int c = 0; c < d; ++c) O[c] /= l;
  if (amb)
    for (int c = 0; c < d; ++c) amb[c] /= l;
  if (lse) *lse = scale * r + log(l / LAZY_TOP);
  free(dq);
  free(S);
  free(P2);
  free(pc);
  free(ps);
}

/* ------------------------------------------------------------------------------------------------
 * (3) Attention for ONE query row of one head: Alg1 L6-L13 with the online softmax of FlashAttention
 * (P:71), tiled over keys in blocks of Bkv.  Operands are given dequantized (exact, fp64):
 *   Qrow [d], Kd [Np][d], Vt [d][Np] (V transposed), codes only matter through these values.
 * p_mode: TWO_LEVEL (the method), DIRECT (ablation), NONE (no P quantization: the unquantized
 * FlashAttention recurrence, used to pin the tiling against plain softmax attention).
 * Causal (reading c12): key j visible iff j <= qi.  Keys >= N are masked (reading c13).
 * qbar [d] / Ks [Np][d] (both nullable): smoothing Q — S gets + q̄_i·K_j^T (Alg1 L8).
 * Softmax scale (reading c7): P̃ = exp(scale * (S - m)), S in unscaled units.
 * Returns O[d] = O/l and *lse = scale*m + ln(l).
 * ------------------------------------------------------------------------------------------------ */
static void attn_row(const double* Qrow, const double* Kd, const double* Vt, int N, int Np, int d, int Bkv,
                     int causal, int qi, double scale, int p_mode, const float* qbar, const float* Ks, int fmt,
                     double* O, double* lse, double delta, double* amb) {
  if (p_mode == PMODE_LAZY) {
    attn_row_lazy(Qrow, Kd, Vt, N, Np, d, Bkv, causal, qi, scale, qbar, Ks, fmt, O, lse, delta, amb);
    return;
  }
  const int G = fmt ? 32 : 16;
  double m = -INFINITY, l = 0.0;
  double* S = (double*)malloc(sizeof(double) * (size_t)Bkv);
  float* Pt = (float*)malloc(sizeof(float) * (size_t)Bkv);
  double* Pq = (double*)malloc(sizeof(double) * (size_t)Bkv);
  uint8_t* pc = (uint8_t*)malloc((size_t)Bkv);
  uint8_t* ps = (uint8_t*)malloc((size_t)Bkv / 16 + 1);
  double* dq = amb ? (double*)malloc(sizeof(double) * (size_t)Bkv) : NULL;
  double ambs = 0.0; /* PMODE_QSUM: decision sensitivity of l */
  float p2[32];
  for (int c = 0; c < d; ++c) O[c] = 0.0;
  if (amb)
    for (int c = 0; c < d; ++c) amb[c] = 0.0;
  int kv_end = causal ? (qi + 1 < N ? qi + 1 : N) : N;
  for (int j0 = 0; j0 < kv_end; j0 += Bkv) {
    /* Alg1 L8: S_ij = FP4MM(Q̂_i, s_Q, K̂_j, s_K) — exact in fp64 */
    double tmax = -INFINITY;
    for (int t = 0; t < Bkv; ++t) {
      int key = j0 + t;
      if (key >= kv_end || key >= Np) {
        S[t] = -INFINITY;
        continue;
      }
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += Qrow[c] * Kd[(size_t)key * d + c];
      if (qbar) { /* Alg1 L8 smoothing Q: + GEMV(q̄_i, K_j^T) with the full-precision smoothed K (fp64) */
        double g = 0.0;
        for (int c = 0; c < d; ++c) g += (double)qbar[c] * (double)Ks[(size_t)key * d + c];
        acc += g;
      }
      S[t] = acc;
      if (acc > tmax) tmax = acc;
    }
    /* Alg1 L9: m_ij = max(m_{i,j-1}, rowmax(S_ij)); P̃ = exp(S - m_ij); l update */
    double m_new = m > tmax ? m : tmax;
    double alpha = exp(scale * (m - m_new)); /* e^{m_{i,j-1} - m_ij}; 0 on the first tile */
    double rowsum = 0.0;
    for (int t = 0; t < Bkv; ++t) {
      double e = (S[t] == -INFINITY) ? 0.0 : exp(scale * (S[t] - m_new));
      Pt[t] = (float)e; /* P̃ in fp32 */
      Pq[t] = e;        /* kept in fp64 only by the unquantized pin mode (p_mode NONE) */
      rowsum += (p_mode == PMODE_NONE) ? e : (double)Pt[t];
    }
    if (p_mode != PMODE_QSUM) l = alpha * l + rowsum; /* (PMODE_QSUM: after the quantization below) */
    /* Alg1 L10: two-level quantization of P̃ (or the ablation modes) */
    double sP1;
    if (p_mode == PMODE_NONE) {
      sP1 = 1.0;
    } else {
      sP1 = (double)oracle_two_level_row_fmt(Pt, Bkv, p_mode, fmt, pc, ps);
      for (int t = 0; t < Bkv; ++t)
        Pq[t] = oracle_e2m1_decode(pc[t]) * (fmt ? ldexp(1.0, (int)ps[t / 32] - 127) : oracle_e4m3_decode(ps[t / 16]));
      if (amb && sP1 != 0.0) /* the decisions' sensitivity on the values φ saw: P̃2 = fl32(P̃/s_P1), or P̃ (direct) */
        for (int b = 0; b < Bkv; b += G) {
          for (int i = 0; i < G; ++i) p2[i] = p_mode == PMODE_DIRECT ? Pt[b + i] : Pt[b + i] / (float)sP1;
          oracle_phi_sensitivity(p2, G, fmt, delta, &dq[b]);
        }
      if (p_mode == PMODE_QSUM) { /* l from the quantized P: s_P1 · Σ deq(P̂2) */
        double qs = 0.0;
        for (int t = 0; t < Bkv; ++t) qs += Pq[t];
        l = alpha * l + qs * sP1;
        if (amb) { /* a decision moves the denominator too: its share is applied with |O| at the end */
          double a = 0.0;
          for (int t = 0; t < Bkv; ++t) a += dq[t];
          ambs = alpha * ambs + a * sP1;
        }
      }
    }
    /* Alg1 L11: O = diag(alpha) O + FP4MM(P̂2, s_P2, V̂, s_V) * s_P1 (inner sum exact in fp64) */
    for (int c = 0; c < d; ++c) {
      double pv = 0.0;
      for (int t = 0; t < Bkv; ++t) {
        int key = j0 + t;
        if (key >= Np) break;
        pv += Pq[t] * Vt[(size_t)c * Np + key];
      }
      O[c] = alpha * O[c] + pv * sP1;
    }
    if (amb) {
      for (int c = 0; c < d; ++c) {
        double a = 0.0;
        if (p_mode != PMODE_NONE && sP1 != 0.0)
          for (int t = 0; t < Bkv && j0 + t < Np; ++t) a += dq[t] * fabs(Vt[(size_t)c * Np + j0 + t]);
        amb[c] = alpha * amb[c] + a * sP1;
      }
    }
    m = m_new;
  }
  /* Alg1 L13: O_i = diag(l)^-1 O */
  for (int c = 0; c < d; ++c) O[c] /= l;
  if (amb)
    for (int c = 0; c < d; ++c) amb[c] = amb[c] / l + ambs / l * fabs(O[c]);
  if (lse) *lse = scale * m + log(l);
  free(dq);
  free(S);
  free(Pt);
  free(Pq);
  free(pc);
  free(ps);
}

/* Attention forward over a batch of BH heads from quantized codes (logical layouts as produced by
 * oracle_quantize_head, stacked per head).  rows[nrows] selects the query rows evaluated (rows are
 * independent, so a row sample is exact for those rows).  O: [BH][nrows][d], lse: [BH][nrows] (nullable).
 * OpenMP over (head, row). */
EXPORT void oracle_attn_fwd_amb(int BH, int N, int d, const uint8_t* q_codes, const uint8_t* q_sf,
                                const uint8_t* k_codes, const uint8_t* k_sf, const uint8_t* v_codes,
                                const uint8_t* v_sf, const float* q_mean, const float* ks, int fmt, int Bkv, int causal,
                                double scale, int p_mode, const int* rows, int nrows, double* O, double* lse,
                                double delta, double* amb) {
  const int Np = (N + 127) / 128 * 128;
  const int G = fmt ? 32 : 16;
  const int C = d / G;
  for (int h = 0; h < BH; ++h) {
    double* Qd = (double*)malloc(sizeof(double) * (size_t)Np * d);
    double* Kd = (double*)malloc(sizeof(double) * (size_t)Np * d);
    double* Vt = (double*)malloc(sizeof(double) * (size_t)Np * d);
    oracle_dequant_fmt(q_codes + (size_t)h * Np * d, q_sf + (size_t)h * Np * C, Np, d, fmt, Qd);
    oracle_dequant_fmt(k_codes + (size_t)h * Np * d, k_sf + (size_t)h * Np * C, Np, d, fmt, Kd);
    oracle_dequant_fmt(v_codes + (size_t)h * Np * d, v_sf + (size_t)h * d * (Np / G), d, Np, fmt, Vt);
    const float* qm_h = q_mean ? q_mean + (size_t)h * (Np / 128) * d : NULL;
    const float* ks_h = ks ? ks + (size_t)h * Np * d : NULL;
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < nrows; ++r) {
      int qi = rows[r];
      attn_row(&Qd[(size_t)qi * d], Kd, Vt, N, Np, d, Bkv, causal, qi, scale, p_mode,
               qm_h ? qm_h + (size_t)(qi / 128) * d : NULL, ks_h, fmt, &O[((size_t)h * nrows + r) * d],
               lse ? &lse[(size_t)h * nrows + r] : NULL, delta, amb ? &amb[((size_t)h * nrows + r) * d] : NULL);
    }
    free(Qd);
    free(Kd);
    free(Vt);
  }
}

/* The same without the decision-sensitivity output. */
EXPORT void oracle_attn_fwd_fmt(int BH, int N, int d, const uint8_t* q_codes, const uint8_t* q_sf,
                                const uint8_t* k_codes, const uint8_t* k_sf, const uint8_t* v_codes,
                                const uint8_t* v_sf, const float* q_mean, const float* ks, int fmt, int Bkv, int causal,
                                double scale, int p_mode, const int* rows, int nrows, double* O, double* lse) {
  oracle_attn_fwd_amb(BH, N, d, q_codes, q_sf, k_codes, k_sf, v_codes, v_sf, q_mean, ks, fmt, Bkv, causal, scale,
                      p_mode, rows, nrows, O, lse, 0.0, NULL);
}

EXPORT void oracle_attn_fwd_sq(int BH, int N, int d, const uint8_t* q_codes, const uint8_t* q_sf,
                               const uint8_t* k_codes, const uint8_t* k_sf, const uint8_t* v_codes,
                               const uint8_t* v_sf, const float* q_mean, const float* ks, int Bkv, int causal,
                               double scale, int p_mode, const int* rows, int nrows, double* O, double* lse) {
  oracle_attn_fwd_fmt(BH, N, d, q_codes, q_sf, k_codes, k_sf, v_codes, v_sf, q_mean, ks, 0, Bkv, causal, scale, p_mode,
                      rows, nrows, O, lse);
}

EXPORT void oracle_attn_fwd(int BH, int N, int d, const uint8_t* q_codes, const uint8_t* q_sf,
                            const uint8_t* k_codes, const uint8_t* k_sf, const uint8_t* v_codes,
                            const uint8_t* v_sf, int Bkv, int causal, double scale, int p_mode, const int* rows,
                            int nrows, double* O, double* lse) {
  oracle_attn_fwd_sq(BH, N, d, q_codes, q_sf, k_codes, k_sf, v_codes, v_sf, NULL, NULL, Bkv, causal, scale, p_mode,
                     rows, nrows, O, lse);
}

/* The same tiled recurrence on UNQUANTIZED fp32 inputs (Q [N][d], K [N][d], V [N][d]) with any
 * p_mode — p_mode NONE must equal plain softmax attention for every Bkv (tiling invariant). */
EXPORT void oracle_attn_fwd_float(int N, int d, const float* Q, const float* K, const float* V, int Bkv,
                                  int causal, double scale, int p_mode, const int* rows, int nrows, double* O,
                                  double* lse) {
  const int Np = (N + Bkv - 1) / Bkv * Bkv;
  double* Kd = (double*)calloc((size_t)Np * d, sizeof(double));
  double* Vt = (double*)calloc((size_t)Np * d, sizeof(double));
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < d; ++c) {
      Kd[(size_t)n * d + c] = K[(size_t)n * d + c];
      Vt[(size_t)c * Np + n] = V[(size_t)n * d + c];
    }
#pragma omp parallel for schedule(dynamic, 1)
  for (int r = 0; r < nrows; ++r) {
    double* Qrow = (double*)malloc(sizeof(double) * (size_t)d);
    for (int c = 0; c < d; ++c) Qrow[c] = Q[(size_t)rows[r] * d + c];
    attn_row(Qrow, Kd, Vt, N, Np, d, Bkv, causal, rows[r], scale, p_mode, NULL, NULL, 0, &O[(size_t)r * d],
             lse ? &lse[r] : NULL, 0.0, NULL);
    free(Qrow);
  }
  free(Kd);
  free(Vt);
}

/* (4) Plain softmax attention in fp64 on the original inputs (S = QK^T, P = Softmax(S), O = PV),
 * untiled, for the paper's accuracy metrics.  O: [nrows][d]. */
EXPORT void oracle_reference_attention(int N, int d, const float* Q, const float* K, const float* V, int causal,
                                       double scale, const int* rows, int nrows, double* O) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int r = 0; r < nrows; ++r) {
    int qi = rows[r];
    int kv_end = causal ? qi + 1 : N;
    double* s = (double*)malloc(sizeof(double) * (size_t)N);
    double mx = -INFINITY, sum = 0.0;
    for (int j = 0; j < kv_end; ++j) {
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += (double)Q[(size_t)qi * d + c] * (double)K[(size_t)j * d + c];
      s[j] = scale * acc;
      if (s[j] > mx) mx = s[j];
    }
    for (int j = 0; j < kv_end; ++j) {
      s[j] = exp(s[j] - mx);
      sum += s[j];
    }
    for (int c = 0; c < d; ++c) {
      double acc = 0.0;
      for (int j = 0; j < kv_end; ++j) acc += s[j] * (double)V[(size_t)j * d + c];
      O[(size_t)r * d + c] = acc / sum;
    }
    free(s);
  }
}

EXPORT int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Vectorised codec entry points (same scalar definitions as above) for bulk pin tests. */
EXPORT void oracle_e2m1_encode_array(const float* x, int64_t n, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_e2m1_encode(x[i]);
}
EXPORT void oracle_e4m3_encode_array(const float* x, int64_t n, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = oracle_e4m3_encode(x[i]);
}
