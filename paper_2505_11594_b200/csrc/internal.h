// internal.h — host-side launch interfaces between the C ABI (abi.cu) and the kernels (quant.cu,
// attn.cu).  Not part of the public ABI (include/sage3.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <atomic>
#include <cstdint>

namespace sage3 {

// cuTensorMapEncodeTiled through a per-process cache keyed by every argument (the descriptors of a repeated call —
// same buffers, shapes and strides, the common case of a serving loop — are encoded once, abi.cu).
CUresult encode_tiled_cached(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, CUtensorMapDataType dt,
                             cuuint32_t rank, void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                             const cuuint32_t* box, const cuuint32_t* es, CUtensorMapInterleave il,
                             CUtensorMapSwizzle swz, CUtensorMapL2promotion promo, CUtensorMapFloatOOBfill oob);

// Quantize workspace: the fp64 K chunk sums [BH][d][Np/128], then the fused K-mean control words (a work counter and
// per head {chunk sums added, km ready}), zeroed by the launcher before each call.
inline size_t quant_sums_bytes(int BH, int nch, int d) { return ((size_t)BH * nch * d * 8 + 255) & ~size_t(255); }
inline size_t quant_ctl_bytes(int BH) { return ((size_t)16 + (size_t)BH * 8 + 255) & ~size_t(255); }

struct QKArgs {
  const void* q;
  const void* k;
  int64_t q_sb, q_sh, q_sn, k_sb, k_sh, k_sn;
  int B, H, N, Np, d;
  uint8_t *q_data, *k_data, *q_sf, *k_sf;
  float* k_mean;  // written by the K-mean pass, read by quant_qk
  float* q_mean;  // smoothing Q (nullable): [B][H][Np/128][d]
  float* ds;      // smoothing Q (nullable): [B][H][Np/128][Np] GEMV(q̄_i, K^T)
  bool mx;        // MXFP4 (Tab1a ablation): E8M0 scales per 32 instead of E4M3 per 16
  uint32_t* nonfinite;
};

struct VArgs {
  const void* v;
  int64_t sb, sh, sn;
  int H, N, Np, d;
  uint8_t *v_data, *v_sf;
  uint32_t* nonfinite;
};

// k_mean is QKArgs::k_mean (non-const alias for the writer).
cudaError_t launch_quantize(const QKArgs& qk, const VArgs& v, bool bf16, double* ws, cudaStream_t stream);

cudaError_t launch_kmean(const QKArgs& qk, bool bf16, double* ws, cudaStream_t stream);

// SageBwd INT8 (NEXT #3; quant_i8.cu / attn_i8.cu)
struct I8Args {
  const void *q, *k, *v;
  int64_t q_sb, q_sh, q_sn, k_sb, k_sh, k_sn, v_sb, v_sh, v_sn;
  int B, H, N, Np, d;
  int8_t *q8, *k8, *vt8;  // [BH][Np][d], [BH][Np][d], [BH][d][Np]
  float *sq, *sk, *sv;    // [BH][Np/128]
  float* k_mean;          // [BH][d]
  uint32_t* nonfinite;
};
cudaError_t launch_quantize_i8(const I8Args& a, bool bf16, double* ws, cudaStream_t stream);

struct I8AttnArgs {
  const int8_t *q8, *k8, *vt8;
  const float *sq, *sk, *sv;
  void* o;
  int64_t o_sb, o_sh, o_sn;
  int o_dtype;
  float* lse;
  int B, H, N, Np, d;
  int causal;
  float scale;
};
cudaError_t launch_attention_i8(const I8AttnArgs& a, cudaStream_t stream);

// SageBwd backward (Alg3; bwd_i8.cu).  Workspace arrays: do8 [BH][Np][d] int8, sdo [BH][Np/128],
// lp / dd [BH][Np] (L'·, D), dqacc [BH][Np][d] fp32.
struct I8BwdArgs {
  const int8_t *q8, *k8;
  const float *sq, *sk, *km;
  const void *v, *o, *dout;
  int64_t v_sb, v_sh, v_sn, o_sb, o_sh, o_sn, do_sb, do_sh, do_sn;
  int in_bf16;  // v, dout: 1 bf16, 0 fp16
  int o_dtype;  // sage3_dtype of o
  const float* lse;  // [BH][N]
  void *dq, *dk, *dv;
  int64_t dq_sb, dq_sh, dq_sn, dk_sb, dk_sh, dk_sn, dv_sb, dv_sh, dv_sn;
  int g_dtype;  // sage3_dtype of the gradients
  int B, H, N, Np, d, causal;
  float scale;
  int8_t* do8;
  float *sdo, *lp, *dd, *dqacc;
};
cudaError_t launch_attention_bwd_i8(const I8BwdArgs& a, cudaStream_t stream);

struct AttnArgs {
  const uint8_t *q_data, *k_data, *v_data, *q_sf, *k_sf, *v_sf;
  void* o;
  int64_t o_sb, o_sh, o_sn;
  int o_dtype;  // sage3_dtype
  float* lse;
  int B, H, N, Np, d;
  int causal;
  float scale;  // softmax scale (S units)
  const float* ds;  // smoothing Q (nullable): [B][H][Np/128][Np], added to S
  bool mx;          // MXFP4 operands (scale_vec::2X MMAs, 32-key P̂2 blocks with E8M0 scales)
  bool p_direct;    // direct-P ablation (Tab1b): P̂ = φ(P̃) relative to the running max, s_P1 = 1
  bool p_qsum;      // NEXT #2 variant: l from the quantized P̂2 (tensor-core ones column, reading n2)
  int64_t unit_begin, unit_end;  // work units [begin, end) of the flattened (b·h, q-tile) space
};

// Returns cudaSuccess or the launch / driver error.  `drv_err` receives a CUresult on descriptor failure.
cudaError_t launch_attention(const AttnArgs& a, cudaStream_t stream);
// attn3.cu: the north_star path (NVFP4, two-level P, no smoothing Q) with three softmax warpgroups per CTA.
bool attention3_enabled(int d, int N, int causal);
cudaError_t launch_attention3(const AttnArgs& a, cudaStream_t stream);
// The NEXT #2 lazy-reference variant (attn_lazy.cu; p_quant = SAGE3_P_TWO_LEVEL_LAZY, no smoothing Q).
cudaError_t launch_attention_lazy(const AttnArgs& a, cudaStream_t stream);

}  // namespace sage3
