/*
 * sage3.h — C ABI of the B200 (sm_100a) SageAttention3 FP4 attention forward (arXiv 2505.11594).
 *
 * The library implements the north_star hot path: Algorithm 1 of the paper
 * without smoothing Q:
 *   sage3_quantize_qkv : Alg1 L2 (K -= mean(K)) and L7 (φ of Q, K along d; φ of V along tokens,
 *                        stored transposed) — NVFP4 = E2M1 codes + E4M3 per-16 scales
 *                        (P:129), φ as Eq. 1.
 *   sage3_attn_fwd     : Alg1 L6-L13 — S = FP4MM(Q̂,s_Q,K̂,s_K) (Eq. 3), online softmax (L9),
 *                        two-level P quantization (L10, §3.2), O += FP4MM(P̂2,s_P2,V̂,s_V)·s_P1
 *                        (L11), O = diag(l)^-1 O (L13).
 * The readings of points the paper leaves open (rounding, softmax scale, causal mask, padding) are
 * listed in DESIGN.md §3; the numerics are bit-exact (quantizer) / within tolerance (attention) of the
 * CPU oracle in oracle/.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless the name says _host.  The caller allocates and owns every
 *    buffer; the library never allocates or frees device memory.
 *  - Every call only enqueues work on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *    stream) on the CURRENT device; nothing synchronizes, except sage3_forward_host which also enqueues
 *    its copies and returns without synchronizing.
 *  - Argument errors are detected on the host before anything is enqueued and returned as a status;
 *    launch failures return SAGE3_ERR_CUDA (see sage3_last_cuda_error).  Device faults surface at the
 *    caller's next synchronization.  No C++ exception crosses the ABI.
 *  - Inputs must be finite.  A violation is reported through the optional device flag of
 *    sage3_quantize_qkv, not trapped.
 *  - Thread safety: stateless apart from per-device one-time kernel attribute setup; safe to call
 *    concurrently from threads that drive different devices.
 */
#ifndef SAGE3_H_
#define SAGE3_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SAGE3_OK = 0,
  SAGE3_ERR_INVALID_ARG = 1, /* null pointer, B/H/N < 1, d not in {64,128}, stride/alignment violation  */
  SAGE3_ERR_UNSUPPORTED = 2, /* current device is not compute capability 10.0 (sm_100a), bad dtype      */
  SAGE3_ERR_WORKSPACE = 3,   /* workspace / scratch smaller than the *_bytes query returned            */
  SAGE3_ERR_CUDA = 4         /* a CUDA launch or driver call failed; see sage3_last_cuda_error()        */
} sage3_status;

typedef enum { SAGE3_FP16 = 0, SAGE3_BF16 = 1, SAGE3_FP32 = 2 /* output only */ } sage3_dtype;

/* FP4 microscaling format of Q̂, K̂, V̂ and P̂2.  NVFP4 is the method; MXFP4 is the data-type
 * ablation of Tab1a, kept as a switch for the accuracy / throughput comparison. */
typedef enum {
  SAGE3_NVFP4 = 0, /* E2M1 codes, UE4M3 scale per 16 elements (tcgen05 scale_vec::4X)                    */
  SAGE3_MXFP4 = 1  /* E2M1 codes, UE8M0 scale 2^(e-127) per 32 elements (tcgen05 scale_vec::2X)          */
} sage3_fp4_format;

/* A [B][H][N][d] tensor: element (b,h,n,c) is at ptr + b*stride_b + h*stride_h + n*stride_n + c
 * (strides in ELEMENTS; the d stride is 1).  ptr and every stride*sizeof(elem) must be 16-byte aligned. */
typedef struct {
  void* ptr;
  int64_t stride_b, stride_h, stride_n;
} sage3_tensor4;

/* FP4 Q, K, V of one call, produced by sage3_quantize_qkv and consumed by sage3_attn_fwd.
 * N_pad = round_up(N, 128).  fmt: a sage3_fp4_format, set by the caller before sage3_quantize_qkv (G = 16
 * for NVFP4, 32 for MXFP4).  Codes: E2M1, two per byte, element 2k in the LOW nibble.
 *   q_data, k_data : [B][H][N_pad][d/2]     blocks of G along d (the QK^T reduction dim)
 *   v_data         : [B][H][d][N_pad/2]     V transposed: tokens contiguous, blocks of G tokens
 * Scales: one byte per G-element block (NVFP4: UE4M3; MXFP4: UE8M0), in 512-byte SF atoms of 128 rows x 4
 * blocks (C4 = round_up(C, 4) columns; columns >= C are zero):
 *   byte(r, c) = ((r/128)*(C4/4) + c/4)*512 + (r%32)*16 + ((r/32)%4)*4 + (c%4)      per (b,h) matrix
 *   q_sf, k_sf : R = N_pad rows (tokens), C = d/G blocks       NVFP4: N_pad*d/16, MXFP4: 4*N_pad bytes per (b,h)
 *   v_sf       : R = 128 rows (channels, rows >= d are zero), C = N_pad/G   NVFP4: 8*N_pad, MXFP4: 4*N_pad
 *   (the layout tcgen05.cp.32x128b.warpx4 expects; identical to cuBLAS's VEC16_UE4M3 / VEC32_UE8M0 layouts)
 * Padding tokens n in [N, N_pad) hold zero codes and zero scales.
 *   k_mean : [B][H][d] fp32, the smoothing-K mean (Alg1 L2).
 * Smoothing Q (Alg1 L5 + the GEMV of L8; off on the north_star path): set q_mean and ds non-null.
 *   q_mean : [B][H][N_pad/128][d] fp32, q̄_i of each 128-row query tile (written by sage3_quantize_qkv,
 *            which then quantizes Q - q̄_i instead of Q)
 *   ds     : [B][H][N_pad/128][N_pad] fp32, GEMV(q̄_i, K^T) with the full-precision smoothed K
 *            (written by sage3_quantize_qkv, added to S = FP4MM(Q̂, K̂) by sage3_attn_fwd)
 *   Both NULL = no smoothing Q (the north_star path).  Sizes: sage3_smooth_q_sizes(). */
typedef struct {
  int32_t B, H, N, d, N_pad;
  int32_t fmt; /* sage3_fp4_format; 0 (NVFP4) when the struct is zero-initialised */
  uint8_t* q_data;
  uint8_t* k_data;
  uint8_t* v_data;
  uint8_t* q_sf;
  uint8_t* k_sf;
  uint8_t* v_sf;
  float* k_mean;
  float* q_mean; /* nullable (smoothing Q off) */
  float* ds;     /* nullable (smoothing Q off) */
} sage3_fp4_qkv;

/* Host-only size queries (no CUDA calls).  bytes[0..6] = q_data, k_data, v_data, q_sf, k_sf, v_sf,
 * k_mean of the NVFP4 format (sage3_fp4_qkv_sizes) or of `fmt` (sage3_fp4_qkv_sizes_fmt).  Returns
 * SAGE3_ERR_INVALID_ARG for unsupported shapes or formats. */
sage3_status sage3_fp4_qkv_sizes(int B, int H, int N, int d, size_t bytes[7]);
sage3_status sage3_fp4_qkv_sizes_fmt(int B, int H, int N, int d, int fmt, size_t bytes[7]);

/* Host-only size queries for smoothing Q: bytes[0] = q_mean, bytes[1] = ds (see sage3_fp4_qkv). */
sage3_status sage3_smooth_q_sizes(int B, int H, int N, int d, size_t bytes[2]);

/* Device workspace of sage3_quantize_qkv: the fp64 K-mean chunk sums (B*H*(N_pad/128)*d*8 bytes, rounded up to 256)
 * followed by the fused K-mean path's control words (16 + 8*B*H bytes, rounded up to 256). */
size_t sage3_quantize_workspace_bytes(int B, int H, int N, int d);

/* B_kv (keys per tile) used by sage3_attn_fwd for head dim d.  The per-tile first-level P scale s_P1
 * (Alg1 L10) makes the result depend on it, so the oracle must use the same value.  Returns 128, or 0
 * for an unsupported d. */
int sage3_kv_tile(int d);

/* Alg1 L2 + L7 (+ L5 and L8's GEMV when out->q_mean and out->ds are set: q̄_i = fl32(Σ_rows Q / rows) over
 * the real rows of each 128-row tile in fp64 ascending order, Q̂ = φ(fl32(Q - q̄_i)); ds = q̄_i·fl32(K - km)^T
 * in fp32; SAGE3_ERR_INVALID_ARG if only one of the two is set).  q, k, v: [B][H][N][d] in `in_dtype`
 * (SAGE3_FP16 or SAGE3_BF16).  Fills every array of *out (whose pointers and B,H,N,d fields the caller sets;
 * N_pad is written).  `workspace` must hold
 * sage3_quantize_workspace_bytes().  nonfinite_flag: nullable device u32, OR-set to 1 if any input is
 * NaN/Inf (the codes are then unspecified).
 * Numerics (bit-exact with oracle_quantize_head): km[c] = fl32(Σ_chunks Σ_tokens K / N) in fp64 with the
 * fixed order of DESIGN.md reading c10; x = fl32(K - km); s = E4M3_RNE(fl32(amax·fl32(1/6)));
 * codes = E2M1_RNE(fl32(x·fl32(1/s))), all-zero codes when s == 0.  MXFP4 (out->fmt = SAGE3_MXFP4, Tab1a):
 * s = the smallest power of two >= fl32(amax·fl32(1/6)) (reading m1), code = E2M1_RNE(x / s) (exact
 * scaling), scale byte 0 and zero codes when amax·fl32(1/6) == 0. */
sage3_status sage3_quantize_qkv(sage3_tensor4 q, sage3_tensor4 k, sage3_tensor4 v, sage3_dtype in_dtype, int B,
                                int H, int N, int d, sage3_fp4_qkv* out, void* workspace, size_t workspace_bytes,
                                uint32_t* nonfinite_flag, void* stream);

/* Alg1 L6-L13 on the FP4 tensors of *qkv (NVFP4, or MXFP4 with 32-key P̂2 blocks and UE8M0 s_P2).  o: [B][H][N][d] in o_dtype (FP16, BF16 or FP32); rows
 * n >= N are never written.  causal != 0: key j is visible to query i iff j <= i (top-left aligned).
 * softmax_scale <= 0 selects 1/sqrt(d); S is scaled after the MMA: P̃ = exp(scale·(S - m)).
 * lse: nullable device fp32 [B][H][N], lse = scale·m + ln(l) (natural log).
 * The tensor-core path: tcgen05.mma.kind::mxf4nvf4.block_scale (scale_vec::4X; 2X for MXFP4) for QK^T and PV with
 * fp32 accumulators and scale factors in TMEM, TMA-staged operands, B_q = B_kv = 128. */
sage3_status sage3_attn_fwd(const sage3_fp4_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype, int causal,
                            float softmax_scale, float* lse, void* stream);

/* The same computation restricted to the work units [unit_begin, unit_end) of the flattened (b·h, query
 * tile) space: unit u covers head bh = u / T and query rows [128·(T-1-u%T), +128) of it, T = N_pad/128
 * (query tiles of a head are numbered from the last one, the longest under causal masking).  Only those
 * rows of o (and lse) are written; K/V of every head a unit touches must be quantized in *qkv.  Results
 * are bitwise identical to the same rows of sage3_attn_fwd (a unit's output does not depend on which other
 * units share the launch), which is what lets the multi-GPU launcher split heads that do not divide the GPU
 * count.  Errors: SAGE3_ERR_INVALID_ARG also for unit_begin < 0, unit_end < unit_begin or
 * unit_end > B·H·T; an empty range enqueues nothing. */
sage3_status sage3_attn_fwd_units(const sage3_fp4_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype, int causal,
                                  float softmax_scale, float* lse, int64_t unit_begin, int64_t unit_end,
                                  void* stream);

/* Options of sage3_attn_fwd_ex (zero-initialise, then set what differs from the defaults). */
typedef enum {
  SAGE3_P_TWO_LEVEL = 0, /* the method: s_P1 = rowmax(P̃)/(448·6), P̂2 = φ(P̃/s_P1) (§3.2, Alg1 L10)   */
  SAGE3_P_DIRECT = 1,    /* ablation (Tab1b): P̂ = φ(P̃), P̃ = exp(scale(S - m_j)) with the running max */
  SAGE3_P_TWO_LEVEL_LAZY = 2, /* throughput variant (reading n1): the first level
                              * is a per-row reference r moved to the tile max only when that exceeds r by more
                              * than 2^8 in weight; P̂2 = φ(10.5·exp(scale(S - r))); O accumulates in TMEM      */
  SAGE3_P_TWO_LEVEL_QSUM = 3 /* throughput variant (reading n2): P̂2 exactly as
                              * TWO_LEVEL, but the row sum l of Alg1 L9 accumulates the QUANTIZED P (s_P1·Σ deq(P̂2),
                              * read from the tensor core: P̂2 times a ones column) instead of the unquantized P̃
                              * (reading c9).  NVFP4 only (MXFP4: SAGE3_ERR_UNSUPPORTED).                        */
} sage3_p_quant;
typedef struct {
  int32_t causal;       /* != 0: key j visible to query i iff j <= i                                      */
  float softmax_scale;  /* <= 0 selects 1/sqrt(d)                                                          */
  int32_t p_quant;      /* sage3_p_quant; modes other than TWO_LEVEL require smoothing Q off (INVALID_ARG)  */
  int32_t reserved;     /* must be 0                                                                       */
  int64_t unit_begin;   /* work units [unit_begin, unit_end) as in sage3_attn_fwd_units;                   */
  int64_t unit_end;     /*   unit_end < 0 selects every unit from unit_begin on                            */
} sage3_attn_options;

/* sage3_attn_fwd_units with an options struct (the other two entry points are this call with p_quant =
 * SAGE3_P_TWO_LEVEL).  The direct-P mode chains the running max through the KV tiles (the two softmax
 * warpgroups of the kernel wait on each other) and is an accuracy ablation, not a fast path.  The lazy mode
 * runs a second kernel (O accumulated by the tensor core in TMEM, S rows kept in registers) whose results
 * match the oracle's PMODE_LAZY, not Alg1 L10; lse = scale·r + ln(l / 10.5) is the same quantity.
 * Errors: as sage3_attn_fwd_units; SAGE3_ERR_INVALID_ARG also for opts == NULL, an unknown p_quant, a
 * non-zero reserved field, or a mode other than SAGE3_P_TWO_LEVEL with smoothing Q. */
sage3_status sage3_attn_fwd_ex(const sage3_fp4_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype,
                               const sage3_attn_options* opts, float* lse, void* stream);

/* ---------------------------------------------------------------------------------------------------------
 * SageBwd's 8-bit attention forward (§4, Algorithm 2).
 * ψ (reading b1): per 128-token block of each head, s = fl32(max|X| · fl32(1/127)),
 * X̂ = clamp(RNE(fl32(x · fl32(1/s))), ±127) (s = 0: zero codes); K smoothed first (Alg2 L2, the c10 mean).
 *   q, k : int8 [B][H][N_pad][d]          v_t : int8 [B][H][d][N_pad] (V transposed: tokens contiguous)
 *   s_q, s_k, s_v : fp32 [B][H][N_pad/128] k_mean : fp32 [B][H][d]
 * Padding tokens hold zero codes.  sage3_int8_attn_fwd: S = MM(Q̂, K̂)·s_Q·s_K (int32-exact), online softmax,
 * per-token P̂ = P̃/s_P with s_P = exp(scale(rowmax(S) - m))/127 (Alg2 L10), O += MM(P̂, V̂)·s_P·s_V, O/l and
 * lse = scale·m + ln l (Alg2 L13-14) — tcgen05.mma.kind::i8 for both products.  N_pad/128 must be <= 1024.
 * --------------------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t B, H, N, d, N_pad;
  int8_t* q;
  int8_t* k;
  int8_t* v_t;
  float* s_q;
  float* s_k;
  float* s_v;
  float* k_mean;
} sage3_int8_qkv;

/* bytes[0..6] = q, k, v_t, s_q, s_k, s_v, k_mean.  SAGE3_ERR_INVALID_ARG for unsupported shapes. */
sage3_status sage3_int8_qkv_sizes(int B, int H, int N, int d, size_t bytes[7]);

/* Alg2 L2 + L4.  q, k, v as in sage3_quantize_qkv; workspace of sage3_quantize_workspace_bytes() bytes (the
 * K-mean partial sums); nonfinite_flag nullable (OR-set to 1 on NaN/Inf input).  Bit-exact with the oracle's
 * sb_quantize_head. */
sage3_status sage3_int8_quantize_qkv(sage3_tensor4 q, sage3_tensor4 k, sage3_tensor4 v, sage3_dtype in_dtype, int B,
                                     int H, int N, int d, sage3_int8_qkv* out, void* workspace,
                                     size_t workspace_bytes, uint32_t* nonfinite_flag, void* stream);

/* Alg2 L6-L14 on *qkv; o, o_dtype, causal, softmax_scale, lse as in sage3_attn_fwd. */
sage3_status sage3_int8_attn_fwd(const sage3_int8_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype, int causal,
                                 float softmax_scale, float* lse, void* stream);

/* Algorithm 3 (SageBwd backward; readings b1-b8 in DESIGN.md §3.1).
 *   qkv       : the Q̂, K̂ codes, s_Q, s_K and k_mean written by sage3_int8_quantize_qkv (v_t / s_v unused)
 *   v, dout   : [B][H][N][d] 16-bit (in_dtype) — the unquantized V and dO of the FP16 product dP = dO·Vᵀ
 *   o         : [B][H][N][d] in o_dtype (fp16 / bf16 / fp32), the forward output used for D = rowsum(dO∘O)
 *   lse       : [B][H][N] fp32 device, the forward's L = scale·m + ln l (sage3_int8_attn_fwd's lse)
 *   dq, dk, dv: [B][H][N][d] outputs in grad_dtype (fp16 / bf16 / fp32), gradients w.r.t. the UNSMOOTHED
 *               q, k, v; dQ includes the smooth-K term rowsum(dS)·K_m (Alg3 L10); dQ and dK carry the softmax
 *               scale.  Rows >= N are not written.
 *   workspace : device, 16-byte aligned, sage3_int8_bwd_workspace_bytes() bytes (ψ(dO) codes and scales,
 *               D, L·log2 e, the fp32 dQ accumulator); contents on return are unspecified.
 * Per (query tile i, key tile j) of 128 x 128: ψ(P_ij) and ψ(dS_ij) use one scale per tile, ψ(dO_i) one per
 * 128-row block (readings b1, b6).  S, dV, dK and dQ products run as tcgen05.mma.kind::i8, dP as kind::f16.
 * Errors: SAGE3_ERR_INVALID_ARG (null / misaligned pointers, shape), SAGE3_ERR_UNSUPPORTED (dtype, device),
 * SAGE3_ERR_WORKSPACE, SAGE3_ERR_CUDA.  Enqueued on `stream` only (four launches: memset, prep, main, dQ
 * finalize). */
size_t sage3_int8_bwd_workspace_bytes(int B, int H, int N, int d);
sage3_status sage3_int8_attn_bwd(const sage3_int8_qkv* qkv, sage3_tensor4 v, sage3_tensor4 o, sage3_dtype o_dtype,
                                 sage3_tensor4 dout, sage3_dtype in_dtype, const float* lse, int causal,
                                 float softmax_scale, sage3_tensor4 dq, sage3_tensor4 dk, sage3_tensor4 dv,
                                 sage3_dtype grad_dtype, void* workspace, size_t workspace_bytes, void* stream);

/* End-to-end convenience path with HOST buffers (for e2e measurements): copies contiguous host
 * q, k, v ([B][H][N][d], in_dtype; pinned memory recommended) to device scratch, quantizes, runs the
 * attention and copies O (contiguous [B][H][N][d], o_dtype) back to o_host.  The work is split into up to
 * 32 groups of consecutive heads and pipelined over three library-owned streams of the current device
 * (copy-in of group g+1 and copy-out of group g-1 overlap the compute of group g); events order it after
 * the caller's prior work on `stream` and make `stream` wait for the last copy-out, so the call behaves as
 * if everything were enqueued on `stream`: the caller synchronizes `stream` before reading o_host.
 * `scratch` (device) must hold sage3_forward_host_scratch_bytes().  No smoothing Q on this path. */
size_t sage3_forward_host_scratch_bytes(int B, int H, int N, int d, sage3_dtype in_dtype, sage3_dtype o_dtype);
sage3_status sage3_forward_host(const void* q_host, const void* k_host, const void* v_host, sage3_dtype in_dtype,
                                int B, int H, int N, int d, int causal, float softmax_scale, void* o_host,
                                sage3_dtype o_dtype, void* scratch, size_t scratch_bytes, void* stream);

const char* sage3_status_str(sage3_status s);
/* cudaError_t (as int) of the last SAGE3_ERR_CUDA returned on this host thread; 0 if none. */
int sage3_last_cuda_error(void);
/* Library version string, e.g. "sage3-b200 0.1 sm_100a". */
const char* sage3_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SAGE3_H_ */
