// abi.cu — the extern "C" entry points declared in include/sage3.h: argument validation, size queries,
// and the launches of quant.cu / attn.cu.  No torch types, no allocation, no synchronization.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "../../include/sage3.h"
#include "internal.h"

namespace {

thread_local int g_last_cuda_error = 0;

sage3_status cuda_fail(cudaError_t e) {
  g_last_cuda_error = (int)e;
  return SAGE3_ERR_CUDA;
}

bool shape_ok(int B, int H, int N, int d) {
  if (B < 1 || H < 1 || N < 1 || (d != 64 && d != 128)) return false;
  // 32-bit grid / index limits of the kernels
  const int64_t Np = ((int64_t)N + 127) / 128 * 128;
  if ((int64_t)B * H > 65535 || Np / 128 > 65535 || (int64_t)B * H * Np > (int64_t)1 << 31) return false;
  return true;
}

}  // namespace

namespace sage3 {
CUresult encode_tiled_cached(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, CUtensorMapDataType dt,
                             cuuint32_t rank, void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                             const cuuint32_t* box, const cuuint32_t* es, CUtensorMapInterleave il,
                             CUtensorMapSwizzle swz, CUtensorMapL2promotion promo, CUtensorMapFloatOOBfill oob) {
  // key: every argument, as bytes (rank <= 5)
  struct Key {
    uint64_t w[24];
    bool operator==(const Key& o) const { return std::memcmp(w, o.w, sizeof(w)) == 0; }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      uint64_t h = 1469598103934665603ull;
      for (uint64_t x : k.w) h = (h ^ x) * 1099511628211ull;
      return (size_t)h;
    }
  };
  Key k{};
  k.w[0] = (uint64_t)dt | ((uint64_t)rank << 8) | ((uint64_t)il << 16) | ((uint64_t)swz << 24) |
           ((uint64_t)promo << 32) | ((uint64_t)oob << 40);
  k.w[1] = reinterpret_cast<uint64_t>(base);
  for (cuuint32_t i = 0; i < rank && i < 5; ++i) {
    k.w[2 + i] = dims[i];
    k.w[7 + i] = i + 1 < rank ? strides[i] : 0;
    k.w[12 + i] = ((uint64_t)box[i] << 32) | es[i];
  }
  int dev = 0;
  cudaGetDevice(&dev);
  k.w[17] = (uint64_t)dev;
  static std::mutex mu;
  static std::unordered_map<Key, CUtensorMap, Hash> cache;
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(k);
    if (it != cache.end()) {
      *m = it->second;
      return CUDA_SUCCESS;
    }
  }
  const CUresult r = enc(m, dt, rank, base, dims, strides, box, es, il, swz, promo, oob);
  if (r == CUDA_SUCCESS) {
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() >= 1024) cache.clear();  // bounded: buffers of a long-running process come and go
    cache.emplace(k, *m);
  }
  return r;
}
}  // namespace sage3

namespace {
int64_t npad(int N) { return ((int64_t)N + 127) / 128 * 128; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// A [B][H][N][d] operand of `esize`-byte elements: non-null, 16-byte aligned base and row/batch/head strides.
bool tensor_ok(const sage3_tensor4& t, int esize) {
  if (t.ptr == nullptr || !aligned16(t.ptr)) return false;
  if ((t.stride_n * esize) % 16 || (t.stride_h * esize) % 16 || (t.stride_b * esize) % 16) return false;
  return t.stride_n > 0 && t.stride_h >= 0 && t.stride_b >= 0;
}
// An OUTPUT the kernels write: additionally no zero head / batch stride where there is more than one head /
// batch (several CTAs would write the same rows concurrently).
bool out_tensor_ok(const sage3_tensor4& t, int esize, int B, int H) {
  return tensor_ok(t, esize) && (H == 1 || t.stride_h != 0) && (B == 1 || t.stride_b != 0);
}

sage3_status device_ok() {
  int dev = 0, major = 0, minor = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? SAGE3_OK : SAGE3_ERR_UNSUPPORTED;
}

int esize_of(sage3_dtype t) { return t == SAGE3_FP32 ? 4 : 2; }

// sage3_forward_host pipeline: head groups and the library-owned streams (one set per device, created on
// first use, never destroyed: they live as long as the process, like the kernels' attribute setup).
#ifndef SAGE3_HOST_GROUPS
#define SAGE3_HOST_GROUPS 32
#endif
constexpr int kHostGroups = SAGE3_HOST_GROUPS;
struct Pipe {
  cudaStream_t s[3];
};
Pipe* pipe_for_current_device() {
  static std::mutex mu;
  static Pipe* pipes[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pipes[dev]) {
    Pipe* p = new Pipe;
    for (int i = 0; i < 3; ++i)
      if (cudaStreamCreateWithFlags(&p->s[i], cudaStreamNonBlocking) != cudaSuccess) {
        delete p;
        return nullptr;
      }
    pipes[dev] = p;
  }
  return pipes[dev];
}

}  // namespace

extern "C" {

sage3_status sage3_fp4_qkv_sizes_fmt(int B, int H, int N, int d, int fmt, size_t bytes[7]) {
  if (!bytes || !shape_ok(B, H, N, d) || (fmt != SAGE3_NVFP4 && fmt != SAGE3_MXFP4)) return SAGE3_ERR_INVALID_ARG;
  const size_t BH = (size_t)B * H, Np = (size_t)npad(N);
  const bool mx = fmt == SAGE3_MXFP4;
  bytes[0] = BH * Np * d / 2;   // q_data
  bytes[1] = BH * Np * d / 2;   // k_data
  bytes[2] = BH * d * Np / 2;   // v_data
  // SF atoms: 512 bytes per 128 rows x 4 blocks; MXFP4 (d/32 <= 4 blocks per row) fills one atom column group
  bytes[3] = mx ? BH * Np * 4 : BH * Np * d / 16;  // q_sf
  bytes[4] = bytes[3];                              // k_sf
  bytes[5] = mx ? BH * Np * 4 : BH * 128 * Np / 16;  // v_sf (128 channel rows, zero beyond d)
  bytes[6] = BH * d * sizeof(float);  // k_mean
  return SAGE3_OK;
}

sage3_status sage3_fp4_qkv_sizes(int B, int H, int N, int d, size_t bytes[7]) {
  return sage3_fp4_qkv_sizes_fmt(B, H, N, d, SAGE3_NVFP4, bytes);
}

sage3_status sage3_smooth_q_sizes(int B, int H, int N, int d, size_t bytes[2]) {
  if (!bytes || !shape_ok(B, H, N, d)) return SAGE3_ERR_INVALID_ARG;
  const size_t BH = (size_t)B * H, Np = (size_t)npad(N), T = Np / 128;
  bytes[0] = BH * T * d * sizeof(float);   // q_mean
  bytes[1] = BH * T * Np * sizeof(float);  // ds
  return SAGE3_OK;
}

size_t sage3_quantize_workspace_bytes(int B, int H, int N, int d) {
  if (!shape_ok(B, H, N, d)) return 0;
  return sage3::quant_sums_bytes(B * H, (int)(npad(N) / 128), d) + sage3::quant_ctl_bytes(B * H);
}

int sage3_kv_tile(int d) { return (d == 64 || d == 128) ? 128 : 0; }

sage3_status sage3_quantize_qkv(sage3_tensor4 q, sage3_tensor4 k, sage3_tensor4 v, sage3_dtype in_dtype, int B,
                                int H, int N, int d, sage3_fp4_qkv* out, void* workspace, size_t workspace_bytes,
                                uint32_t* nonfinite_flag, void* stream) {
  if (!out || !shape_ok(B, H, N, d)) return SAGE3_ERR_INVALID_ARG;
  if (in_dtype != SAGE3_FP16 && in_dtype != SAGE3_BF16) return SAGE3_ERR_UNSUPPORTED;
  if (!tensor_ok(q, 2) || !tensor_ok(k, 2) || !tensor_ok(v, 2)) return SAGE3_ERR_INVALID_ARG;
  if (out->B != B || out->H != H || out->N != N || out->d != d) return SAGE3_ERR_INVALID_ARG;
  if (out->fmt != SAGE3_NVFP4 && out->fmt != SAGE3_MXFP4) return SAGE3_ERR_INVALID_ARG;
  if (!out->q_data || !out->k_data || !out->v_data || !out->q_sf || !out->k_sf || !out->v_sf || !out->k_mean)
    return SAGE3_ERR_INVALID_ARG;
  if (!aligned16(out->q_data) || !aligned16(out->k_data) || !aligned16(out->v_data) || !aligned16(out->q_sf) ||
      !aligned16(out->k_sf) || !aligned16(out->v_sf) || !aligned16(out->k_mean))
    return SAGE3_ERR_INVALID_ARG;
  if ((out->q_mean == nullptr) != (out->ds == nullptr)) return SAGE3_ERR_INVALID_ARG;
  if (out->q_mean && (!aligned16(out->q_mean) || !aligned16(out->ds))) return SAGE3_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < sage3_quantize_workspace_bytes(B, H, N, d)) return SAGE3_ERR_WORKSPACE;
  sage3_status st = device_ok();
  if (st != SAGE3_OK) return st;
  out->N_pad = (int32_t)npad(N);
  sage3::QKArgs qa{};
  qa.q = q.ptr;
  qa.k = k.ptr;
  qa.q_sb = q.stride_b, qa.q_sh = q.stride_h, qa.q_sn = q.stride_n;
  qa.k_sb = k.stride_b, qa.k_sh = k.stride_h, qa.k_sn = k.stride_n;
  qa.B = B, qa.H = H, qa.N = N, qa.Np = out->N_pad, qa.d = d;
  qa.q_data = out->q_data, qa.k_data = out->k_data, qa.q_sf = out->q_sf, qa.k_sf = out->k_sf;
  qa.k_mean = out->k_mean;
  qa.q_mean = out->q_mean;
  qa.ds = out->ds;
  qa.mx = out->fmt == SAGE3_MXFP4;
  qa.nonfinite = nonfinite_flag;
  sage3::VArgs va{};
  va.v = v.ptr;
  va.sb = v.stride_b, va.sh = v.stride_h, va.sn = v.stride_n;
  va.H = H, va.N = N, va.Np = out->N_pad, va.d = d;
  va.v_data = out->v_data, va.v_sf = out->v_sf;
  va.nonfinite = nonfinite_flag;
  cudaError_t e = sage3::launch_quantize(qa, va, in_dtype == SAGE3_BF16, static_cast<double*>(workspace),
                                         static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SAGE3_OK : cuda_fail(e);
}

sage3_status sage3_attn_fwd_ex(const sage3_fp4_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype,
                               const sage3_attn_options* opts, float* lse, void* stream) {
  if (!qkv || !opts || !shape_ok(qkv->B, qkv->H, qkv->N, qkv->d)) return SAGE3_ERR_INVALID_ARG;
  if ((opts->p_quant != SAGE3_P_TWO_LEVEL && opts->p_quant != SAGE3_P_DIRECT &&
       opts->p_quant != SAGE3_P_TWO_LEVEL_LAZY && opts->p_quant != SAGE3_P_TWO_LEVEL_QSUM) ||
      opts->reserved != 0)
    return SAGE3_ERR_INVALID_ARG;
  if (opts->p_quant == SAGE3_P_TWO_LEVEL_QSUM && qkv->fmt != SAGE3_NVFP4) return SAGE3_ERR_UNSUPPORTED;
  if (opts->p_quant != SAGE3_P_TWO_LEVEL && (qkv->q_mean || qkv->ds)) return SAGE3_ERR_INVALID_ARG;
  const int causal = opts->causal;
  const float softmax_scale = opts->softmax_scale;
  const int64_t unit_begin = opts->unit_begin;
  if (qkv->N_pad != npad(qkv->N)) return SAGE3_ERR_INVALID_ARG;
  if (qkv->fmt != SAGE3_NVFP4 && qkv->fmt != SAGE3_MXFP4) return SAGE3_ERR_INVALID_ARG;
  const int64_t n_units = (int64_t)qkv->B * qkv->H * (qkv->N_pad / 128);
  const int64_t unit_end = opts->unit_end < 0 ? n_units : opts->unit_end;
  if (unit_begin < 0 || unit_end < unit_begin || unit_end > n_units || unit_end - unit_begin > 0x7FFFFFFF)
    return SAGE3_ERR_INVALID_ARG;
  if (o_dtype != SAGE3_FP16 && o_dtype != SAGE3_BF16 && o_dtype != SAGE3_FP32) return SAGE3_ERR_UNSUPPORTED;
  if (!out_tensor_ok(o, esize_of(o_dtype), qkv->B, qkv->H)) return SAGE3_ERR_INVALID_ARG;
  if (!qkv->q_data || !qkv->k_data || !qkv->v_data || !qkv->q_sf || !qkv->k_sf || !qkv->v_sf)
    return SAGE3_ERR_INVALID_ARG;
  if (!aligned16(qkv->q_data) || !aligned16(qkv->k_data) || !aligned16(qkv->v_data) || !aligned16(qkv->q_sf) ||
      !aligned16(qkv->k_sf) || !aligned16(qkv->v_sf))
    return SAGE3_ERR_INVALID_ARG;
  if (!(std::isfinite(softmax_scale))) return SAGE3_ERR_INVALID_ARG;
  if ((qkv->q_mean == nullptr) != (qkv->ds == nullptr)) return SAGE3_ERR_INVALID_ARG;
  if (qkv->ds && !aligned16(qkv->ds)) return SAGE3_ERR_INVALID_ARG;
  sage3_status st = device_ok();
  if (st != SAGE3_OK) return st;
  sage3::AttnArgs a{};
  a.ds = qkv->ds;
  a.mx = qkv->fmt == SAGE3_MXFP4;
  a.p_direct = opts->p_quant == SAGE3_P_DIRECT;
  a.p_qsum = opts->p_quant == SAGE3_P_TWO_LEVEL_QSUM;
  a.q_data = qkv->q_data, a.k_data = qkv->k_data, a.v_data = qkv->v_data;
  a.q_sf = qkv->q_sf, a.k_sf = qkv->k_sf, a.v_sf = qkv->v_sf;
  a.o = o.ptr, a.o_sb = o.stride_b, a.o_sh = o.stride_h, a.o_sn = o.stride_n, a.o_dtype = (int)o_dtype;
  a.lse = lse;
  a.B = qkv->B, a.H = qkv->H, a.N = qkv->N, a.Np = qkv->N_pad, a.d = qkv->d;
  a.causal = causal ? 1 : 0;
  a.scale = softmax_scale > 0.0f ? softmax_scale : 1.0f / std::sqrt((float)qkv->d);
  a.unit_begin = unit_begin, a.unit_end = unit_end;
  cudaError_t e = opts->p_quant == SAGE3_P_TWO_LEVEL_LAZY
                      ? sage3::launch_attention_lazy(a, static_cast<cudaStream_t>(stream))
                      : sage3::launch_attention(a, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SAGE3_OK : cuda_fail(e);
}

sage3_status sage3_attn_fwd_units(const sage3_fp4_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype, int causal,
                                  float softmax_scale, float* lse, int64_t unit_begin, int64_t unit_end,
                                  void* stream) {
  if (unit_end < 0) return SAGE3_ERR_INVALID_ARG;  // (the options' "to the end" value is not part of this API)
  sage3_attn_options op{};
  op.causal = causal, op.softmax_scale = softmax_scale, op.p_quant = SAGE3_P_TWO_LEVEL;
  op.unit_begin = unit_begin, op.unit_end = unit_end;
  return sage3_attn_fwd_ex(qkv, o, o_dtype, &op, lse, stream);
}

sage3_status sage3_attn_fwd(const sage3_fp4_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype, int causal,
                            float softmax_scale, float* lse, void* stream) {
  if (!qkv || !shape_ok(qkv->B, qkv->H, qkv->N, qkv->d)) return SAGE3_ERR_INVALID_ARG;
  return sage3_attn_fwd_units(qkv, o, o_dtype, causal, softmax_scale, lse, 0,
                              (int64_t)qkv->B * qkv->H * (npad(qkv->N) / 128), stream);
}

// ---------------------------------------------------------------------------------- SageBwd INT8 forward
static bool i8_shape_ok(int B, int H, int N, int d) { return shape_ok(B, H, N, d) && npad(N) / 128 <= 1024; }

sage3_status sage3_int8_qkv_sizes(int B, int H, int N, int d, size_t bytes[7]) {
  if (!bytes || !i8_shape_ok(B, H, N, d)) return SAGE3_ERR_INVALID_ARG;
  const size_t BH = (size_t)B * H, Np = (size_t)npad(N);
  bytes[0] = bytes[1] = bytes[2] = BH * Np * d;
  bytes[3] = bytes[4] = bytes[5] = BH * (Np / 128) * sizeof(float);
  bytes[6] = BH * d * sizeof(float);
  return SAGE3_OK;
}

sage3_status sage3_int8_quantize_qkv(sage3_tensor4 q, sage3_tensor4 k, sage3_tensor4 v, sage3_dtype in_dtype, int B,
                                     int H, int N, int d, sage3_int8_qkv* out, void* workspace,
                                     size_t workspace_bytes, uint32_t* nonfinite_flag, void* stream) {
  if (!out || !i8_shape_ok(B, H, N, d)) return SAGE3_ERR_INVALID_ARG;
  if (in_dtype != SAGE3_FP16 && in_dtype != SAGE3_BF16) return SAGE3_ERR_UNSUPPORTED;
  if (!tensor_ok(q, 2) || !tensor_ok(k, 2) || !tensor_ok(v, 2)) return SAGE3_ERR_INVALID_ARG;
  if (out->B != B || out->H != H || out->N != N || out->d != d) return SAGE3_ERR_INVALID_ARG;
  if (!out->q || !out->k || !out->v_t || !out->s_q || !out->s_k || !out->s_v || !out->k_mean)
    return SAGE3_ERR_INVALID_ARG;
  if (!aligned16(out->q) || !aligned16(out->k) || !aligned16(out->v_t) || !aligned16(out->k_mean))
    return SAGE3_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < sage3_quantize_workspace_bytes(B, H, N, d)) return SAGE3_ERR_WORKSPACE;
  sage3_status st = device_ok();
  if (st != SAGE3_OK) return st;
  out->N_pad = (int32_t)npad(N);
  sage3::I8Args a{};
  a.q = q.ptr, a.k = k.ptr, a.v = v.ptr;
  a.q_sb = q.stride_b, a.q_sh = q.stride_h, a.q_sn = q.stride_n;
  a.k_sb = k.stride_b, a.k_sh = k.stride_h, a.k_sn = k.stride_n;
  a.v_sb = v.stride_b, a.v_sh = v.stride_h, a.v_sn = v.stride_n;
  a.B = B, a.H = H, a.N = N, a.Np = out->N_pad, a.d = d;
  a.q8 = out->q, a.k8 = out->k, a.vt8 = out->v_t, a.sq = out->s_q, a.sk = out->s_k, a.sv = out->s_v;
  a.k_mean = out->k_mean;
  a.nonfinite = nonfinite_flag;
  cudaError_t e = sage3::launch_quantize_i8(a, in_dtype == SAGE3_BF16, static_cast<double*>(workspace),
                                            static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SAGE3_OK : cuda_fail(e);
}

sage3_status sage3_int8_attn_fwd(const sage3_int8_qkv* qkv, sage3_tensor4 o, sage3_dtype o_dtype, int causal,
                                 float softmax_scale, float* lse, void* stream) {
  if (!qkv || !i8_shape_ok(qkv->B, qkv->H, qkv->N, qkv->d) || qkv->N_pad != npad(qkv->N))
    return SAGE3_ERR_INVALID_ARG;
  if (o_dtype != SAGE3_FP16 && o_dtype != SAGE3_BF16 && o_dtype != SAGE3_FP32) return SAGE3_ERR_UNSUPPORTED;
  if (!out_tensor_ok(o, esize_of(o_dtype), qkv->B, qkv->H)) return SAGE3_ERR_INVALID_ARG;
  if (!qkv->q || !qkv->k || !qkv->v_t || !qkv->s_q || !qkv->s_k || !qkv->s_v) return SAGE3_ERR_INVALID_ARG;
  if (!aligned16(qkv->q) || !aligned16(qkv->k) || !aligned16(qkv->v_t)) return SAGE3_ERR_INVALID_ARG;
  if (!std::isfinite(softmax_scale)) return SAGE3_ERR_INVALID_ARG;
  sage3_status st = device_ok();
  if (st != SAGE3_OK) return st;
  sage3::I8AttnArgs a{};
  a.q8 = qkv->q, a.k8 = qkv->k, a.vt8 = qkv->v_t, a.sq = qkv->s_q, a.sk = qkv->s_k, a.sv = qkv->s_v;
  a.o = o.ptr, a.o_sb = o.stride_b, a.o_sh = o.stride_h, a.o_sn = o.stride_n, a.o_dtype = (int)o_dtype;
  a.lse = lse;
  a.B = qkv->B, a.H = qkv->H, a.N = qkv->N, a.Np = qkv->N_pad, a.d = qkv->d;
  a.causal = causal ? 1 : 0;
  a.scale = softmax_scale > 0.0f ? softmax_scale : 1.0f / std::sqrt((float)qkv->d);
  cudaError_t e = sage3::launch_attention_i8(a, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SAGE3_OK : cuda_fail(e);
}

size_t sage3_int8_bwd_workspace_bytes(int B, int H, int N, int d) {
  if (!i8_shape_ok(B, H, N, d)) return 0;
  const size_t BH = (size_t)B * H, Np = (size_t)npad(N);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return al(BH * Np * d) + al(BH * (Np / 128) * 4) + 2 * al(BH * Np * 4) + al(BH * Np * d * 4);
}

sage3_status sage3_int8_attn_bwd(const sage3_int8_qkv* qkv, sage3_tensor4 v, sage3_tensor4 o, sage3_dtype o_dtype,
                                 sage3_tensor4 dout, sage3_dtype in_dtype, const float* lse, int causal,
                                 float softmax_scale, sage3_tensor4 dq, sage3_tensor4 dk, sage3_tensor4 dv,
                                 sage3_dtype grad_dtype, void* workspace, size_t workspace_bytes, void* stream) {
  if (!qkv || !i8_shape_ok(qkv->B, qkv->H, qkv->N, qkv->d) || qkv->N_pad != npad(qkv->N)) return SAGE3_ERR_INVALID_ARG;
  if (in_dtype != SAGE3_FP16 && in_dtype != SAGE3_BF16) return SAGE3_ERR_UNSUPPORTED;
  if (o_dtype != SAGE3_FP16 && o_dtype != SAGE3_BF16 && o_dtype != SAGE3_FP32) return SAGE3_ERR_UNSUPPORTED;
  if (grad_dtype != SAGE3_FP16 && grad_dtype != SAGE3_BF16 && grad_dtype != SAGE3_FP32) return SAGE3_ERR_UNSUPPORTED;
  if (!tensor_ok(v, 2) || !tensor_ok(dout, 2) || !tensor_ok(o, esize_of(o_dtype))) return SAGE3_ERR_INVALID_ARG;
  const int ge = esize_of(grad_dtype);
  if (!out_tensor_ok(dq, ge, qkv->B, qkv->H) || !out_tensor_ok(dk, ge, qkv->B, qkv->H) ||
      !out_tensor_ok(dv, ge, qkv->B, qkv->H))
    return SAGE3_ERR_INVALID_ARG;
  if (!qkv->q || !qkv->k || !qkv->s_q || !qkv->s_k || !qkv->k_mean || !lse) return SAGE3_ERR_INVALID_ARG;
  if (!aligned16(qkv->q) || !aligned16(qkv->k)) return SAGE3_ERR_INVALID_ARG;
  if (!std::isfinite(softmax_scale)) return SAGE3_ERR_INVALID_ARG;
  const int B = qkv->B, H = qkv->H, N = qkv->N, d = qkv->d;
  if (!workspace || !aligned16(workspace) || workspace_bytes < sage3_int8_bwd_workspace_bytes(B, H, N, d))
    return SAGE3_ERR_WORKSPACE;
  sage3_status st = device_ok();
  if (st != SAGE3_OK) return st;
  const size_t BH = (size_t)B * H, Np = (size_t)npad(N);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  uint8_t* p = static_cast<uint8_t*>(workspace);
  sage3::I8BwdArgs a{};
  a.do8 = reinterpret_cast<int8_t*>(p), p += al(BH * Np * d);
  a.sdo = reinterpret_cast<float*>(p), p += al(BH * (Np / 128) * 4);
  a.lp = reinterpret_cast<float*>(p), p += al(BH * Np * 4);
  a.dd = reinterpret_cast<float*>(p), p += al(BH * Np * 4);
  a.dqacc = reinterpret_cast<float*>(p);
  a.q8 = qkv->q, a.k8 = qkv->k, a.sq = qkv->s_q, a.sk = qkv->s_k, a.km = qkv->k_mean;
  a.v = v.ptr, a.v_sb = v.stride_b, a.v_sh = v.stride_h, a.v_sn = v.stride_n;
  a.o = o.ptr, a.o_sb = o.stride_b, a.o_sh = o.stride_h, a.o_sn = o.stride_n, a.o_dtype = (int)o_dtype;
  a.dout = dout.ptr, a.do_sb = dout.stride_b, a.do_sh = dout.stride_h, a.do_sn = dout.stride_n;
  a.in_bf16 = in_dtype == SAGE3_BF16 ? 1 : 0;
  a.lse = lse;
  a.dq = dq.ptr, a.dq_sb = dq.stride_b, a.dq_sh = dq.stride_h, a.dq_sn = dq.stride_n;
  a.dk = dk.ptr, a.dk_sb = dk.stride_b, a.dk_sh = dk.stride_h, a.dk_sn = dk.stride_n;
  a.dv = dv.ptr, a.dv_sb = dv.stride_b, a.dv_sh = dv.stride_h, a.dv_sn = dv.stride_n;
  a.g_dtype = (int)grad_dtype;
  a.B = B, a.H = H, a.N = N, a.Np = (int)Np, a.d = d, a.causal = causal ? 1 : 0;
  a.scale = softmax_scale > 0.0f ? softmax_scale : 1.0f / std::sqrt((float)d);
  cudaError_t e = sage3::launch_attention_bwd_i8(a, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SAGE3_OK : cuda_fail(e);
}

// ---------------------------------------------------------------------------------- host e2e path
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t sage3_forward_host_scratch_bytes(int B, int H, int N, int d, sage3_dtype in_dtype, sage3_dtype o_dtype) {
  size_t sz[7];
  if (sage3_fp4_qkv_sizes(B, H, N, d, sz) != SAGE3_OK) return 0;
  const size_t elems = (size_t)B * H * N * d;
  size_t total = 3 * align256(elems * esize_of(in_dtype)) + align256(elems * esize_of(o_dtype));
  for (int i = 0; i < 7; ++i) total += align256(sz[i]);
  total += align256(sage3_quantize_workspace_bytes(B, H, N, d));
  return total;
}

sage3_status sage3_forward_host(const void* q_host, const void* k_host, const void* v_host, sage3_dtype in_dtype,
                                int B, int H, int N, int d, int causal, float softmax_scale, void* o_host,
                                sage3_dtype o_dtype, void* scratch, size_t scratch_bytes, void* stream) {
  if (!q_host || !k_host || !v_host || !o_host || !scratch) return SAGE3_ERR_INVALID_ARG;
  if (!shape_ok(B, H, N, d)) return SAGE3_ERR_INVALID_ARG;
  if (in_dtype != SAGE3_FP16 && in_dtype != SAGE3_BF16) return SAGE3_ERR_UNSUPPORTED;
  if (o_dtype != SAGE3_FP16 && o_dtype != SAGE3_BF16 && o_dtype != SAGE3_FP32) return SAGE3_ERR_UNSUPPORTED;
  const size_t need = sage3_forward_host_scratch_bytes(B, H, N, d, in_dtype, o_dtype);
  if (need == 0) return SAGE3_ERR_UNSUPPORTED;
  if (scratch_bytes < need) return SAGE3_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t elems = (size_t)B * H * N * d;
  const size_t in_b = elems * esize_of(in_dtype), o_b = elems * esize_of(o_dtype);
  uint8_t* p = static_cast<uint8_t*>(scratch);
  auto take = [&](size_t n) {
    uint8_t* r = p;
    p += align256(n);
    return r;
  };
  uint8_t *dq = take(in_b), *dk = take(in_b), *dv = take(in_b), *dout = take(o_b);
  size_t sz[7];
  sage3_fp4_qkv_sizes(B, H, N, d, sz);
  uint8_t *q_data = take(sz[0]), *k_data = take(sz[1]), *v_data = take(sz[2]);
  uint8_t *q_sf = take(sz[3]), *k_sf = take(sz[4]), *v_sf = take(sz[5]);
  float* k_mean = reinterpret_cast<float*>(take(sz[6]));
  double* ws = reinterpret_cast<double*>(take(sage3_quantize_workspace_bytes(B, H, N, d)));
  sage3_status st = device_ok();
  if (st != SAGE3_OK) return st;

  // Pipelined over groups of heads (every (b,h) is an independent problem): the H2D copy of group g+1 and
  // the D2H copy of group g-1 overlap the quantize + attention of group g.  Three library-owned streams
  // per device (copy-in, compute, copy-out); per-call events order them after the caller's prior work on
  // `stream` and make `stream` wait for the last copy-out, so the call behaves as if enqueued on `stream`.
  Pipe* pp = pipe_for_current_device();
  if (!pp) return cuda_fail(cudaErrorInitializationError);
  const int BH = B * H;
  const int G = BH < kHostGroups ? BH : kHostGroups;  // groups of consecutive flattened heads
  const size_t head_in = (size_t)N * d * esize_of(in_dtype), head_out = (size_t)N * d * esize_of(o_dtype);
  const size_t Np = (size_t)npad(N);
  const int64_t sn = d, sh = (int64_t)N * d;
  cudaError_t e = cudaSuccess;
  cudaEvent_t start, in_done[kHostGroups], comp_done[kHostGroups], out_done;
  int n_ev = 0;
  auto mk = [&](cudaEvent_t* ev) {
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e == cudaSuccess) ++n_ev;
  };
  mk(&start);
  for (int g = 0; g < G; ++g) mk(&in_done[g]);
  for (int g = 0; g < G; ++g) mk(&comp_done[g]);
  mk(&out_done);
  if (e != cudaSuccess) return cuda_fail(e);
  cudaStream_t s_in = pp->s[0], s_cmp = pp->s[1], s_out = pp->s[2];
  auto ck = [&](cudaError_t r) {
    if (e == cudaSuccess && r != cudaSuccess) e = r;
  };
  ck(cudaEventRecord(start, s));
  ck(cudaStreamWaitEvent(s_in, start, 0));
  ck(cudaStreamWaitEvent(s_cmp, start, 0));
  ck(cudaStreamWaitEvent(s_out, start, 0));
  for (int g = 0; g < G && e == cudaSuccess && st == SAGE3_OK; ++g) {
    const int h0 = (int)((int64_t)BH * g / G), h1 = (int)((int64_t)BH * (g + 1) / G), nh = h1 - h0;
    // copy-in of this group's heads (q, k, v are contiguous [BH][N][d] on the host)
    ck(cudaMemcpyAsync(dq + h0 * head_in, static_cast<const uint8_t*>(q_host) + h0 * head_in, nh * head_in,
                       cudaMemcpyHostToDevice, s_in));
    ck(cudaMemcpyAsync(dk + h0 * head_in, static_cast<const uint8_t*>(k_host) + h0 * head_in, nh * head_in,
                       cudaMemcpyHostToDevice, s_in));
    ck(cudaMemcpyAsync(dv + h0 * head_in, static_cast<const uint8_t*>(v_host) + h0 * head_in, nh * head_in,
                       cudaMemcpyHostToDevice, s_in));
    ck(cudaEventRecord(in_done[g], s_in));
    ck(cudaStreamWaitEvent(s_cmp, in_done[g], 0));
    if (e != cudaSuccess) break;
    // quantize + attention of the group as a (1, nh) problem on slices of the full-size buffers
    sage3_fp4_qkv f{};
    f.B = 1, f.H = nh, f.N = N, f.d = d;
    f.q_data = q_data + h0 * (Np * d / 2), f.k_data = k_data + h0 * (Np * d / 2), f.v_data = v_data + h0 * (Np * d / 2);
    f.q_sf = q_sf + h0 * (Np * d / 16), f.k_sf = k_sf + h0 * (Np * d / 16), f.v_sf = v_sf + h0 * (Np * 8);
    f.k_mean = k_mean + (size_t)h0 * d;
    const int64_t sb = (int64_t)nh * N * d;
    sage3_tensor4 tq{dq + h0 * head_in, sb, sh, sn}, tk{dk + h0 * head_in, sb, sh, sn};
    sage3_tensor4 tv{dv + h0 * head_in, sb, sh, sn}, to{dout + h0 * head_out, sb, sh, sn};
    // groups run in order on the compute stream, so they share one workspace (sized for all heads)
    st = sage3_quantize_qkv(tq, tk, tv, in_dtype, 1, nh, N, d, &f, ws, sage3_quantize_workspace_bytes(B, H, N, d),
                            nullptr, s_cmp);
    if (st == SAGE3_OK) st = sage3_attn_fwd(&f, to, o_dtype, causal, softmax_scale, nullptr, s_cmp);
    if (st != SAGE3_OK) break;
    ck(cudaEventRecord(comp_done[g], s_cmp));
    ck(cudaStreamWaitEvent(s_out, comp_done[g], 0));
    ck(cudaMemcpyAsync(static_cast<uint8_t*>(o_host) + h0 * head_out, dout + h0 * head_out, nh * head_out,
                       cudaMemcpyDeviceToHost, s_out));
  }
  // join: the caller's stream waits for everything enqueued above on all three library streams (also on the
  // error path, so that no library stream is left referencing caller memory unordered)
  cudaStreamWaitEvent(s_out, start, 0);
  {
    cudaEvent_t c_done = nullptr, i_done = nullptr;
    if (cudaEventCreateWithFlags(&c_done, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(c_done, s_cmp);
      cudaStreamWaitEvent(s_out, c_done, 0);
      cudaEventDestroy(c_done);
    }
    if (cudaEventCreateWithFlags(&i_done, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(i_done, s_in);
      cudaStreamWaitEvent(s_out, i_done, 0);
      cudaEventDestroy(i_done);
    }
  }
  ck(cudaEventRecord(out_done, s_out));
  cudaStreamWaitEvent(s_cmp, out_done, 0);
  cudaStreamWaitEvent(s, out_done, 0);
  cudaEvent_t all[2 * kHostGroups + 2];
  int k = 0;
  all[k++] = start;
  for (int g = 0; g < G; ++g) all[k++] = in_done[g];
  for (int g = 0; g < G; ++g) all[k++] = comp_done[g];
  all[k++] = out_done;
  for (int i = 0; i < n_ev; ++i) cudaEventDestroy(all[i]);  // released once their work completes
  if (st != SAGE3_OK) return st;
  return e == cudaSuccess ? SAGE3_OK : cuda_fail(e);
}

const char* sage3_status_str(sage3_status s) {
  switch (s) {
    case SAGE3_OK:
      return "SAGE3_OK";
    case SAGE3_ERR_INVALID_ARG:
      return "SAGE3_ERR_INVALID_ARG";
    case SAGE3_ERR_UNSUPPORTED:
      return "SAGE3_ERR_UNSUPPORTED";
    case SAGE3_ERR_WORKSPACE:
      return "SAGE3_ERR_WORKSPACE";
    case SAGE3_ERR_CUDA:
      return "SAGE3_ERR_CUDA";
  }
  return "SAGE3_ERR_UNKNOWN";
}

int sage3_last_cuda_error(void) { return g_last_cuda_error; }

const char* sage3_version(void) { return "sage3-b200 0.1 sm_100a"; }

}  // extern "C"
