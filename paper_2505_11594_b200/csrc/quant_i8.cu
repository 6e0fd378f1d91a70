// quant_i8.cu — SageBwd's INT8 per-block quantization (NEXT #3; Alg2 L2 + L4, ψ P:279-282):
//   K_m = mean(K) (the c10 order, launch_kmean), then per 128-token block of each head and tensor
//   s = fl32(amax · fl32(1/127)),  X̂ = clamp(RNE(fl32(x · fl32(1/s))), ±127),  s = 0 -> zero codes  (reading b1)
// with x = fl32(K - K_m) for K.  Q̂, K̂ are written row-major [BH][Np][d]; V̂ transposed [BH][d][Np] (the PV
// MMA's K-major B operand).  One CTA per (block, head, tensor): the 128 x d tile stays in registers between
// the amax reduction and the encode (HBM-bound: 2 B read + 1 B written per element).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

constexpr float kOne127 = 0x1.020408p-7f;  // fl32(1/127)

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<__half>(__half v) {
  return __half2float(v);
}
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

__device__ __forceinline__ int8_t enc(float x, float r) {
  float v = rintf(__fmul_rn(x, r));  // RNE
  v = fminf(fmaxf(v, -127.0f), 127.0f);
  return (int8_t)(int)v;
}

#ifndef SAGE3_I8Q_THREADS
#define SAGE3_I8Q_THREADS 512  // (0.560 ms vs 0.574 ms with 256 at N = 32K, d = 128)
#endif
constexpr int kQT = SAGE3_I8Q_THREADS;  // threads per (block, head, tensor) CTA

template <typename T, int D>
__global__ void __launch_bounds__(kQT) i8_quant_kernel(const I8Args a) {
  constexpr int kVec = D / 8, kIt = 128 * kVec / kQT;  // 16-byte vectors per row; vectors per thread
  __shared__ float s_red[kQT / 32];
  __shared__ __align__(16) int8_t s_vt[D * 128];  // V̂ codes staging: [token][channel], swizzled
  const int chunk = blockIdx.x, bh = blockIdx.y, tensor = blockIdx.z;  // 0 Q, 1 K, 2 V
  const int b = bh / a.H, h = bh % a.H, t = threadIdx.x;
  const T* base;
  int64_t sn;
  if (tensor == 0) base = reinterpret_cast<const T*>(a.q) + b * a.q_sb + h * a.q_sh, sn = a.q_sn;
  else if (tensor == 1) base = reinterpret_cast<const T*>(a.k) + b * a.k_sb + h * a.k_sh, sn = a.k_sn;
  else base = reinterpret_cast<const T*>(a.v) + b * a.v_sb + h * a.v_sh, sn = a.v_sn;
  const int cv = t % kVec;  // fixed 8-channel group of this thread
  float km[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (tensor == 1) {
#pragma unroll
    for (int e = 0; e < 8; ++e) km[e] = a.k_mean[(int64_t)bh * D + cv * 8 + e];
  }
  float x[kIt][8];
  float amax = 0.0f;
  bool finite = true;
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int row = (it * kQT + t) / kVec, n = chunk * 128 + row;
    if (n < a.N) {
      const uint4 u = *reinterpret_cast<const uint4*>(base + (int64_t)n * sn + cv * 8);
      const T* hv = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float f = to_f<T>(hv[e]);
        x[it][e] = tensor == 1 ? __fsub_rn(f, km[e]) : f;
        finite &= isfinite(x[it][e]);
        amax = fmaxf(amax, fabsf(x[it][e]));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[it][e] = 0.0f;  // padding rows: zero codes (reading c13)
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((t & 31) == 0) s_red[t >> 5] = amax;
  __syncthreads();
  amax = s_red[0];
#pragma unroll
  for (int w = 1; w < kQT / 32; ++w) amax = fmaxf(amax, s_red[w]);
  const float s = __fmul_rn(amax, kOne127);
  const float r = s != 0.0f ? __frcp_rn(s) : 0.0f;
  const int nch = a.Np >> 7;
  if (t == 0) (tensor == 0 ? a.sq : tensor == 1 ? a.sk : a.sv)[(int64_t)bh * nch + chunk] = s;
  if (a.nonfinite && !finite) atomicOr(a.nonfinite, 1u);
  if (tensor < 2) {
    int8_t* dst = (tensor == 0 ? a.q8 : a.k8) + ((int64_t)bh * a.Np + chunk * 128) * D;
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int row = (it * kQT + t) / kVec;
      uint32_t w[2];
      int8_t* bytes = reinterpret_cast<int8_t*>(w);
#pragma unroll
      for (int e = 0; e < 8; ++e) bytes[e] = enc(x[it][e], r);
      *reinterpret_cast<uint2*>(dst + row * D + cv * 8) = make_uint2(w[0], w[1]);
    }
  } else {
    // V̂ᵀ: codes staged row-major (8 bytes per thread and row, the 8-byte chunk index XOR-swizzled with the
    // 16-row group so both this store and the transposed read below are bank-conflict free), then each
    // thread gathers 4 channels x 16 tokens with 16 4-byte loads, transposes them with byte permutes and
    // writes 4 x 16 bytes (8 threads cover one 128-token channel row: coalesced).  The former per-byte
    // transposed smem stores were 16-way bank conflicted (ncu: 7.9M conflicts per launch at N = 4K).
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int row = (it * kQT + t) / kVec;
      uint32_t w[2];
      int8_t* bytes = reinterpret_cast<int8_t*>(w);
#pragma unroll
      for (int e = 0; e < 8; ++e) bytes[e] = enc(x[it][e], r);
      *reinterpret_cast<uint2*>(s_vt + row * D + ((cv ^ ((row >> 4) & 7)) * 8)) = make_uint2(w[0], w[1]);
    }
    __syncthreads();
    for (int i = t; i < (D / 4) * 8; i += kQT) {
      const int q = i & 7, c4 = i >> 3;  // 16-token group, channel quad
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int row = q * 16 + k;
        w[k] = *reinterpret_cast<const uint32_t*>(s_vt + row * D + (((c4 >> 1) ^ q) * 8) + (c4 & 1) * 4);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t sel = (uint32_t)e | ((uint32_t)(e + 4) << 4);  // bytes e of a and of b -> low half
        uint32_t o[4];
#pragma unroll
        for (int m = 0; m < 4; ++m)
          o[m] = __byte_perm(__byte_perm(w[4 * m], w[4 * m + 1], sel), __byte_perm(w[4 * m + 2], w[4 * m + 3], sel),
                             0x5410);
        *reinterpret_cast<uint4*>(a.vt8 + ((int64_t)bh * D + c4 * 4 + e) * a.Np + chunk * 128 + q * 16) =
            make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

template <typename T, int D>
cudaError_t launch_i8_t(const I8Args& a, cudaStream_t stream) {
  dim3 grid(a.Np / 128, a.B * a.H, 3);
  i8_quant_kernel<T, D><<<grid, kQT, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize_i8(const I8Args& a, bool bf16, double* ws, cudaStream_t stream) {
  QKArgs qk{};
  qk.k = a.k, qk.k_sb = a.k_sb, qk.k_sh = a.k_sh, qk.k_sn = a.k_sn;
  qk.B = a.B, qk.H = a.H, qk.N = a.N, qk.Np = a.Np, qk.d = a.d, qk.k_mean = a.k_mean;
  cudaError_t e = launch_kmean(qk, bf16, ws, stream);
  if (e != cudaSuccess) return e;
  if (a.d == 128) return bf16 ? launch_i8_t<__nv_bfloat16, 128>(a, stream) : launch_i8_t<__half, 128>(a, stream);
  return bf16 ? launch_i8_t<__nv_bfloat16, 64>(a, stream) : launch_i8_t<__half, 64>(a, stream);
}

}  // namespace sage3
