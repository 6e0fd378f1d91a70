/*
 * sagebwd_oracle.c — CPU ORACLE for SageBwd, the 8-bit trainable attention of arXiv 2505.11594 §4
 * (PAPER.md P:236-343): Algorithm 2 (forward) and Algorithm 3 (backward).
 *
 * TEST INFRASTRUCTURE ONLY (same rules as sage3_oracle.c: only tests/, smoke() and bench.py's CPU legs may
 * load it; it shares no code with the CUDA path).  Compiled into liboracle.so together with sage3_oracle.c.
 *
 * What it computes, in the paper's order and notation (readings b1-b8 in DESIGN.md §3.1):
 *   ψ  s_X = max|X| / 127, X̂ = X / s_X per FlashAttention block           -> sb_psi
 *   Alg2 L2        K_m = mean(K), K -= K_m (smooth-K; the c10 order)                    -> sb_quantize_head
 *   Alg2 L4        ψ(Q_i), ψ(K_j^T), ψ(V_j): one scale per 128-token block of a head   -> sb_quantize_head
 *   Alg2 L8        S = MM(Q̂_i, K̂_j) · s_Q · s_K (exact int dot, fp64 scaling)           -> sb_fwd_row
 *   Alg2 L9        m, P̃ = exp(scale(S - m)), l (online softmax)                         -> sb_fwd_row
 *   Alg2 L10       s_P = exp(scale(rowmax(S_ij) - m_ij)) / 127 per token, P̂ = P̃ / s_P  -> sb_fwd_row
 *   Alg2 L11-14    O = diag(α)O + MM(P̂, V̂)·s_P·s_V;  O /= l;  L = scale·m + ln l     -> sb_fwd_row
 *   Alg3           D = rowsum(dO∘O); per (j, i): S, P = exp(scale·S - L), ψ(P), ψ(dO_i),
 *                  dV_j += MM(P̂ᵀ, dÔ)·s_P·s_dO, dP = dO·V_jᵀ (16-bit inputs, exact here), dS = P∘(dP - D_i),
 *                  ψ(dS), dQ_i += MM(dŜ, K̂_j)·s_dS·s_K + rowsum(dS)·K_m, dK_j += MM(dŜᵀ, Q̂_i)·s_dS·s_Q;
 *                  dQ, dK carry the softmax scale (S enters the softmax as scale·S)    -> sb_bwd_head
 * Precision: ψ is fp32 arithmetic (bit-exact target for the GPU quantizer); P̃, P, dS are rounded to fp32
 * where the paper's kernels hold them (P:188's convention); the rest is fp64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))
#define SB_BLK 128

/* ψ, reading b1: s = fl32(amax · fl32(1/127)) (one rounding, as reading c3 for FP4);
 * X̂ = clamp(RNE(fl32(x · fl32(1/s))), -127, 127) (reading c4's reciprocal form); s = 0 -> all codes 0.
 * n values at x[i*stride]; codes to q[i*stride].  Returns s. */
EXPORT float sb_psi(const float* x, int n, int stride, int8_t* q) {
  float amax = 0.0f;
  for (int i = 0; i < n; ++i) {
    float a = fabsf(x[(size_t)i * stride]);
    if (a > amax) amax = a;
  }
  const float s = amax * (1.0f / 127.0f);
  if (s == 0.0f) {
    for (int i = 0; i < n; ++i) q[(size_t)i * stride] = 0;
    return 0.0f;
  }
  const float r = 1.0f / s;
  for (int i = 0; i < n; ++i) {
    float y = x[(size_t)i * stride] * r;
    float v = nearbyintf(y); /* RNE (default rounding mode) */
    if (v > 127.0f) v = 127.0f;
    if (v < -127.0f) v = -127.0f;
    q[(size_t)i * stride] = (int8_t)v;
  }
  return s;
}

/* Alg2 L2 + L4 for one head.  Inputs fp32 holding the exact 16-bit values, [N][d].  Outputs (Np =
 * round_up(N, 128); padding rows zero): q, k, v int8 [Np][d]; sq, sk, sv [Np/128]; km [d] (c10 order). */
EXPORT void sb_quantize_head(const float* Q, const float* K, const float* V, int N, int d, int8_t* q, int8_t* k,
                             int8_t* v, float* sq, float* sk, float* sv, float* km) {
  const int Np = (N + SB_BLK - 1) / SB_BLK * SB_BLK;
  for (int c = 0; c < d; ++c) { /* smooth-K mean, reading c10: fp64 per 128-token chunk, chunks ascending */
    double total = 0.0;
    for (int c0 = 0; c0 < N; c0 += SB_BLK) {
      double chunk = 0.0;
      for (int n = c0; n < N && n < c0 + SB_BLK; ++n) chunk += (double)K[(size_t)n * d + c];
      total += chunk;
    }
    km[c] = (float)(total / (double)N);
  }
  float* blk = (float*)calloc((size_t)SB_BLK * d, sizeof(float));
  memset(q, 0, (size_t)Np * d);
  memset(k, 0, (size_t)Np * d);
  memset(v, 0, (size_t)Np * d);
  for (int b = 0; b < Np / SB_BLK; ++b) {
    const int r0 = b * SB_BLK, nr = (N - r0 < SB_BLK) ? N - r0 : SB_BLK;
    memcpy(blk, &Q[(size_t)r0 * d], sizeof(float) * (size_t)nr * d);
    sq[b] = sb_psi(blk, nr * d, 1, &q[(size_t)r0 * d]);
    for (int i = 0; i < nr * d; ++i) blk[i] = K[(size_t)r0 * d + i] - km[i % d]; /* fl32(K - K_m) */
    sk[b] = sb_psi(blk, nr * d, 1, &k[(size_t)r0 * d]);
    memcpy(blk, &V[(size_t)r0 * d], sizeof(float) * (size_t)nr * d);
    sv[b] = sb_psi(blk, nr * d, 1, &v[(size_t)r0 * d]);
  }
  free(blk);
}

/* Alg2 L6-L14 for ONE query row qi (tiles of 128 keys).  Reading b4: causal key j visible iff j <= qi; keys
 * >= N masked.  Reading b5: P̃ = fl32(exp(scale(S - m_ij))), s_P = fl32(rowmax(P̃)/127) (= the paper's
 * exp(rowmax(S) - m)/127 computed from P̃, reusing the max), P̂ = RNE(fl32(P̃ / s_P)) in [0, 127]. */
static void sb_fwd_row(const int8_t* q, const int8_t* k, const int8_t* v, const float* sq, const float* sk,
                       const float* sv, int N, int Np, int d, int causal, int qi, double scale, double* O,
                       double* lse, double delta, double* amb) {
  double m = -INFINITY, l = 0.0;
  double S[SB_BLK], Pq[SB_BLK], dq[SB_BLK];
  float Pt[SB_BLK];
  for (int c = 0; c < d; ++c) O[c] = 0.0;
  if (amb)
    for (int c = 0; c < d; ++c) amb[c] = 0.0;
  const int kv_end = causal ? (qi + 1 < N ? qi + 1 : N) : N;
  for (int j0 = 0; j0 < kv_end; j0 += SB_BLK) {
    double tmax = -INFINITY;
    for (int t = 0; t < SB_BLK; ++t) {
      const int key = j0 + t;
      if (key >= kv_end) {
        S[t] = -INFINITY;
        continue;
      }
      long long dot = 0; /* Alg2 L8: exact INT8 MM, then the two per-block scales */
      for (int c = 0; c < d; ++c) dot += (long long)q[(size_t)qi * d + c] * (long long)k[(size_t)key * d + c];
      S[t] = (double)dot * (double)sq[qi / SB_BLK] * (double)sk[j0 / SB_BLK];
      if (S[t] > tmax) tmax = S[t];
    }
    const double m_new = m > tmax ? m : tmax;
    const double alpha = exp(scale * (m - m_new));
    double rowsum = 0.0;
    float pmax = 0.0f;
    for (int t = 0; t < SB_BLK; ++t) {
      Pt[t] = (S[t] == -INFINITY) ? 0.0f : (float)exp(scale * (S[t] - m_new));
      rowsum += (double)Pt[t];
      if (Pt[t] > pmax) pmax = Pt[t];
    }
    l = alpha * l + rowsum;
    const float sP = pmax / 127.0f; /* Alg2 L10, per token */
    for (int t = 0; t < SB_BLK; ++t) Pq[t] = (sP > 0.0f) ? (double)nearbyintf(Pt[t] / sP) : 0.0;
    /* Decision sensitivity (TEST INFRASTRUCTURE for the GPU element-wise parity bound, as
     * oracle_phi_sensitivity in sage3_oracle.c): the spread of the INT8 code of P̃/s_P over inputs within a
     * relative delta; 0 unless the value sits that close to a rounding midpoint. */
    if (amb)
      for (int t = 0; t < SB_BLK; ++t) {
        const float x = (sP > 0.0f) ? Pt[t] / sP : 0.0f;
        dq[t] = (double)nearbyintf((float)((double)x * (1.0 + delta))) - (double)nearbyintf((float)((double)x * (1.0 - delta)));
      }
    for (int c = 0; c < d; ++c) {
      long long acc = 0; /* MM(P̂, V̂): exact */
      for (int t = 0; t < SB_BLK; ++t) {
        const int key = j0 + t;
        if (key >= Np) break;
        acc += (long long)Pq[t] * (long long)v[(size_t)key * d + c];
      }
      O[c] = alpha * O[c] + (double)acc * (double)sP * (double)sv[j0 / SB_BLK];
      if (amb) {
        double a = 0.0;
        for (int t = 0; t < SB_BLK && j0 + t < Np; ++t) a += dq[t] * fabs((double)v[(size_t)(j0 + t) * d + c]);
        amb[c] = alpha * amb[c] + a * (double)sP * (double)sv[j0 / SB_BLK];
      }
    }
    m = m_new;
  }
  for (int c = 0; c < d; ++c) O[c] /= l;
  if (amb)
    for (int c = 0; c < d; ++c) amb[c] /= l;
  if (lse) *lse = scale * m + log(l);
}

/* Alg2 over a batch of BH heads (quantized by sb_quantize_head, stacked per head), rows[nrows] of each. */
EXPORT void sb_attn_fwd_amb(int BH, int N, int d, const int8_t* q, const int8_t* k, const int8_t* v,
                            const float* sq, const float* sk, const float* sv, int causal, double scale, const int* rows,
                            int nrows, double* O, double* lse, double delta, double* amb) {
  const int Np = (N + SB_BLK - 1) / SB_BLK * SB_BLK, T = Np / SB_BLK;
  for (int h = 0; h < BH; ++h) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < nrows; ++r)
      sb_fwd_row(q + (size_t)h * Np * d, k + (size_t)h * Np * d, v + (size_t)h * Np * d, sq + (size_t)h * T,
                 sk + (size_t)h * T, sv + (size_t)h * T, N, Np, d, causal, rows[r], scale,
                 &O[((size_t)h * nrows + r) * d], lse ? &lse[(size_t)h * nrows + r] : NULL, delta,
                 amb ? &amb[((size_t)h * nrows + r) * d] : NULL);
  }
}

EXPORT void sb_attn_fwd(int BH, int N, int d, const int8_t* q, const int8_t* k, const int8_t* v, const float* sq,
                        const float* sk, const float* sv, int causal, double scale, const int* rows, int nrows,
                        double* O, double* lse) {
  sb_attn_fwd_amb(BH, N, d, q, k, v, sq, sk, sv, causal, scale, rows, nrows, O, lse, 0.0, NULL);
}

/* Alg3 for one head.  q, k int8 [Np][d] with sq, sk, km from sb_quantize_head; V16 = the 16-bit V values
 * (fp32 array, [N][d]) for the FP16 matmul dP = dO·V_jᵀ (P:329 keeps it unquantized); O, dO [N][d] (fp32
 * arrays); L [N] (the forward's lse).  Outputs dQ, dK, dV [N][d] fp64 (w.r.t. the unsmoothed inputs).
 * Reading b6: tiles of 128 queries x 128 keys, ψ(P) and ψ(dS) per tile, ψ(dO_i) per 128-row block; masked
 * entries (causal, keys >= N) have P = 0.  Reading b7: dQ, dK include the softmax scale.  Reading b8:
 * D_i = rowsum(dO∘O) in fp64 from the given O. */
EXPORT void sb_bwd_head(int N, int d, const int8_t* q, const int8_t* k, const float* sq, const float* sk,
                        const float* km, const float* V16, const float* O, const float* dO, const float* L,
                        int causal, double scale, double* dQ, double* dK, double* dV) {
  const int Np = (N + SB_BLK - 1) / SB_BLK * SB_BLK, T = Np / SB_BLK;
  double* D = (double*)calloc((size_t)N, sizeof(double));
  for (int n = 0; n < N; ++n)
    for (int c = 0; c < d; ++c) D[n] += (double)dO[(size_t)n * d + c] * (double)O[(size_t)n * d + c];
  memset(dQ, 0, sizeof(double) * (size_t)N * d);
  memset(dK, 0, sizeof(double) * (size_t)N * d);
  memset(dV, 0, sizeof(double) * (size_t)N * d);
  /* ψ(dO_i) per 128-row block (Alg3 L6) */
  int8_t* dOq = (int8_t*)calloc((size_t)Np * d, 1);
  float* sdO = (float*)calloc((size_t)T, sizeof(float));
  for (int i = 0; i < T; ++i) {
    const int r0 = i * SB_BLK, nr = (N - r0 < SB_BLK) ? N - r0 : SB_BLK;
    sdO[i] = sb_psi(&dO[(size_t)r0 * d], nr * d, 1, &dOq[(size_t)r0 * d]);
  }
  float* P = (float*)malloc(sizeof(float) * SB_BLK * SB_BLK);
  float* dS = (float*)malloc(sizeof(float) * SB_BLK * SB_BLK);
  int8_t* Pq = (int8_t*)malloc(SB_BLK * SB_BLK);
  int8_t* dSq = (int8_t*)malloc(SB_BLK * SB_BLK);
  for (int j = 0; j < T; ++j) {
    for (int i = 0; i < T; ++i) {
      /* S_ij, P_ij = exp(scale·S - L_i) (Alg3 L5) */
      for (int a = 0; a < SB_BLK; ++a)
        for (int b = 0; b < SB_BLK; ++b) {
          const int qi = i * SB_BLK + a, kj = j * SB_BLK + b;
          float p = 0.0f;
          if (qi < N && kj < N && (!causal || kj <= qi)) {
            long long dot = 0;
            for (int c = 0; c < d; ++c) dot += (long long)q[(size_t)qi * d + c] * (long long)k[(size_t)kj * d + c];
            const double S = (double)dot * (double)sq[i] * (double)sk[j];
            p = (float)exp(scale * S - (double)L[qi]);
          }
          P[a * SB_BLK + b] = p;
        }
      const float sP = sb_psi(P, SB_BLK * SB_BLK, 1, Pq); /* Alg3 L6 */
      /* dV_j += MM(P̂ᵀ, dÔ_i)·s_P·s_dO (Alg3 L7) */
      for (int b = 0; b < SB_BLK; ++b) {
        const int kj = j * SB_BLK + b;
        if (kj >= N) break;
        for (int c = 0; c < d; ++c) {
          long long acc = 0;
          for (int a = 0; a < SB_BLK; ++a) acc += (long long)Pq[a * SB_BLK + b] * (long long)dOq[(size_t)(i * SB_BLK + a) * d + c];
          dV[(size_t)kj * d + c] += (double)acc * (double)sP * (double)sdO[i];
        }
      }
      /* dP = dO_i·V_jᵀ in full precision (Alg3 L8), dS = P∘(dP - D_i) (L9) */
      for (int a = 0; a < SB_BLK; ++a)
        for (int b = 0; b < SB_BLK; ++b) {
          const int qi = i * SB_BLK + a, kj = j * SB_BLK + b;
          double ds = 0.0;
          if (qi < N && kj < N && P[a * SB_BLK + b] != 0.0f) {
            double dp = 0.0;
            for (int c = 0; c < d; ++c) dp += (double)dO[(size_t)qi * d + c] * (double)V16[(size_t)kj * d + c];
            ds = (double)P[a * SB_BLK + b] * (dp - D[qi]);
          }
          dS[a * SB_BLK + b] = (float)ds;
        }
      const float sdS = sb_psi(dS, SB_BLK * SB_BLK, 1, dSq);
      /* dQ_i += MM(dŜ, K̂_j)·s_dS·s_K + rowsum(dS)·K_m (L10); dK_j += MM(dŜᵀ, Q̂_i)·s_dS·s_Q (L11) */
      for (int a = 0; a < SB_BLK; ++a) {
        const int qi = i * SB_BLK + a;
        if (qi >= N) break;
        double rs = 0.0;
        for (int b = 0; b < SB_BLK; ++b) rs += (double)dS[a * SB_BLK + b];
        for (int c = 0; c < d; ++c) {
          long long acc = 0;
          for (int b = 0; b < SB_BLK; ++b) acc += (long long)dSq[a * SB_BLK + b] * (long long)k[(size_t)(j * SB_BLK + b) * d + c];
          dQ[(size_t)qi * d + c] += (double)acc * (double)sdS * (double)sk[j] + rs * (double)km[c];
        }
      }
      for (int b = 0; b < SB_BLK; ++b) {
        const int kj = j * SB_BLK + b;
        if (kj >= N) break;
        for (int c = 0; c < d; ++c) {
          long long acc = 0;
          for (int a = 0; a < SB_BLK; ++a) acc += (long long)dSq[a * SB_BLK + b] * (long long)q[(size_t)(i * SB_BLK + a) * d + c];
          dK[(size_t)kj * d + c] += (double)acc * (double)sdS * (double)sq[i];
        }
      }
    }
  }
  for (size_t e = 0; e < (size_t)N * d; ++e) {
    dQ[e] *= scale;
    dK[e] *= scale;
  }
  free(D);
  free(dOq);
  free(sdO);
  free(P);
  free(dS);
  free(Pq);
  free(dSq);
}
