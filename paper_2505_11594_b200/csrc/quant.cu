// quant.cu — sm_100a kernels for sage3_quantize_qkv: smoothing K (Alg1 L2) and NVFP4
// microscaling φ (Eq. 1) of Q, K (1x16 blocks along d) and V (1x16 blocks along tokens, written
// transposed).  HBM-bound streaming kernels: 128-bit loads, one thread per 16-element block.
//
// Numerics are the DESIGN.md §3 readings, implemented with explicitly rounded intrinsics so that no FMA
// contraction or fast-math can change a bit:
//   km[c] = fl32( (Σ_chunk Σ_token K[n][c]) / N ) in fp64, chunks of 128 tokens, ascending order (c10)
//   x     = fl32(K - km)                                      (K only)
//   s32   = fl32(amax * fl32(1/6))                            (c3)
//   sc    = E4M3 RN satfinite (cvt.rn.satfinite.e4m3x2)       (c2)
//   y     = fl32(x * fl32(1/s)), code = E2M1 RN satfinite    (c1, c4); all codes 0 when s == 0 (c5)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

constexpr float kOneSixth = 0x1.555556p-3f;  // fl32(1/6) = 0x3E2AAAAB

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) {
  return __half2float(v);
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

// Unpack 8 16-bit values held in a uint4 to fp32 (exact).
template <typename T>
__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = to_f32<T>(h[i]);
}

// Byte offset of scale (row r, block-column c) inside one (b,h) SF matrix with C block-columns.
__device__ __forceinline__ uint32_t sf_offset(uint32_t r, uint32_t c, uint32_t C) {
  return ((r >> 7) * (C >> 2) + (c >> 2)) * 512u + (r & 31u) * 16u + ((r >> 5) & 3u) * 4u + (c & 3u);
}

// φ of one 16-element block (already in fp32, exact input values).  Returns 8 packed code bytes (lo word,
// hi word) and the E4M3 scale code.
__device__ __forceinline__ void phi16(const float* x, uint32_t& lo, uint32_t& hi, uint32_t& sc) {
  float amax = 0.0f;
#pragma unroll
  for (int i = 0; i < 16; ++i) amax = fmaxf(amax, fabsf(x[i]));
  const float s32 = __fmul_rn(amax, kOneSixth);
  sc = cvt_e4m3x2(s32, 0.0f) & 0xFFu;
  const float s = e4m3_to_f32(sc);
  if (s == 0.0f) {
    lo = hi = 0u;
    return;
  }
  const float r = __frcp_rn(s);
  uint32_t b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) b[i] = cvt_e2m1x2(__fmul_rn(x[2 * i], r), __fmul_rn(x[2 * i + 1], r));
  lo = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
  hi = b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24);
}

__device__ __forceinline__ bool all_finite(const float* x, int n) {
  bool ok = true;
  for (int i = 0; i < n; ++i) ok &= isfinite(x[i]);
  return ok;
}

// ---------------------------------------------------------------------------------- K mean, pass 1
// grid (Np/128, B*H), block d/2: each thread sums two channels over one 128-token chunk in ascending
// token order (fp64, sequential), writes ws[bh][chunk][c].
template <typename T>
__global__ void __launch_bounds__(64) kmean_partial_kernel(const T* __restrict__ k, int64_t sb, int64_t sh,
                                                           int64_t sn, int H, int N, int d,
                                                           double* __restrict__ ws) {
  const int chunk = blockIdx.x, bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int c = threadIdx.x * 2;
  const T* base = k + b * sb + h * sh + c;
  const int n0 = chunk * 128, n1 = min(n0 + 128, N);
  double a0 = 0.0, a1 = 0.0;
  int n = n0;
  for (; n + 8 <= n1; n += 8) {
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(reinterpret_cast<const uint32_t*>(base + (int64_t)(n + i) * sn));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const T* p = reinterpret_cast<const T*>(&v[i]);
      a0 += (double)to_f32<T>(p[0]);
      a1 += (double)to_f32<T>(p[1]);
    }
  }
  for (; n < n1; ++n) {
    uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(base + (int64_t)n * sn));
    const T* p = reinterpret_cast<const T*>(&v);
    a0 += (double)to_f32<T>(p[0]);
    a1 += (double)to_f32<T>(p[1]);
  }
  double* out = ws + ((int64_t)bh * gridDim.x + chunk) * d + c;
  out[0] = a0;
  out[1] = a1;
}

// ---------------------------------------------------------------------------------- K mean, pass 2
// grid B*H, block d: km = fl32( (Σ_chunks ascending) / N ).
__global__ void kmean_final_kernel(const double* __restrict__ ws, int nchunks, int N, int d, float* __restrict__ km) {
  const int bh = blockIdx.x, c = threadIdx.x;
  const double* p = ws + (int64_t)bh * nchunks * d + c;
  double total = 0.0;
  for (int i = 0; i < nchunks; ++i) total += p[(int64_t)i * d];
  km[(int64_t)bh * d + c] = (float)(total / (double)N);
}

// ---------------------------------------------------------------------------------- φ of Q and K
// One thread per (tensor, b, h, n, 16-block); blockIdx.y selects Q (0) or K (1, smoothed).
template <typename T>
__global__ void __launch_bounds__(256) quant_qk_kernel(QKArgs a) {
  const int which = blockIdx.y;
  const T* src = reinterpret_cast<const T*>(which ? a.k : a.q);
  const int64_t sb = which ? a.k_sb : a.q_sb, sh = which ? a.k_sh : a.q_sh, sn = which ? a.k_sn : a.q_sn;
  uint8_t* codes = which ? a.k_data : a.q_data;
  uint8_t* sf = which ? a.k_sf : a.q_sf;
  const int C = a.d >> 4;
  const int64_t total = (int64_t)a.B * a.H * a.Np * C;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int blk = (int)(idx % C);
  const int64_t row = idx / C;  // bh*Np + n
  const int n = (int)(row % a.Np);
  const int bh = (int)(row / a.Np);
  const int b = bh / a.H, h = bh % a.H;
  uint32_t lo = 0, hi = 0, sc = 0;
  if (n < a.N) {
    const T* p = src + b * sb + h * sh + (int64_t)n * sn + blk * 16;
    const uint4 u0 = __ldg(reinterpret_cast<const uint4*>(p));
    const uint4 u1 = __ldg(reinterpret_cast<const uint4*>(p + 8));
    float x[16];
    unpack8<T>(u0, x);
    unpack8<T>(u1, x + 8);
    if (a.nonfinite && !all_finite(x, 16)) atomicOr(a.nonfinite, 1u);
    if (which) {
      const float4* km = reinterpret_cast<const float4*>(a.k_mean + (int64_t)bh * a.d + blk * 16);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 m = km[i];
        x[4 * i + 0] = __fsub_rn(x[4 * i + 0], m.x);
        x[4 * i + 1] = __fsub_rn(x[4 * i + 1], m.y);
        x[4 * i + 2] = __fsub_rn(x[4 * i + 2], m.z);
        x[4 * i + 3] = __fsub_rn(x[4 * i + 3], m.w);
      }
    }
    phi16(x, lo, hi, sc);
  }
  *reinterpret_cast<uint2*>(codes + row * (a.d >> 1) + blk * 8) = make_uint2(lo, hi);
  sf[(int64_t)bh * a.Np * C + sf_offset(n, blk, C)] = (uint8_t)sc;
}

// ---------------------------------------------------------------------------------- φ of V^T
// grid (Np/128, B*H), block 256.  Stage a 128-token x d tile in smem (coalesced 16-byte loads), then each
// thread quantizes (channel, 16-token block) pairs and writes V^T codes / SF atoms.  Channel rows
// d..127 of the SF matrix are written as zero (the MMA reads 128 rows of scales).
template <typename T>
__global__ void __launch_bounds__(256) quant_v_kernel(VArgs a) {
  __shared__ __align__(16) T tile[128 * 128];
  const int chunk = blockIdx.x, bh = blockIdx.y;
  const int b = bh / a.H, h = bh % a.H;
  const int d = a.d;
  const int vec_per_row = d / 8;
  const T* base = reinterpret_cast<const T*>(a.v) + b * a.sb + h * a.sh;
  bool finite = true;
  for (int i = threadIdx.x; i < 128 * vec_per_row; i += blockDim.x) {
    const int t = i / vec_per_row, cv = i % vec_per_row;
    const int n = chunk * 128 + t;
    uint4 u = make_uint4(0, 0, 0, 0);
    if (n < a.N) {
      u = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)n * a.sn + cv * 8));
      if (a.nonfinite) {
        float f[8];
        unpack8<T>(u, f);
        finite &= all_finite(f, 8);
      }
    }
    *reinterpret_cast<uint4*>(&tile[t * d + cv * 8]) = u;
  }
  if (!finite) atomicOr(a.nonfinite, 1u);
  __syncthreads();
  const int Cv = a.Np >> 4;
  uint8_t* sf = a.v_sf + (int64_t)bh * 128 * Cv;
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    const int tb = i & 7, c = i >> 3;
    const int tbg = chunk * 8 + tb;
    uint32_t lo = 0, hi = 0, sc = 0;
    if (c < d) {
      float x[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = to_f32<T>(tile[(tb * 16 + k) * d + c]);
      phi16(x, lo, hi, sc);
      *reinterpret_cast<uint2*>(a.v_data + ((int64_t)bh * d + c) * (a.Np >> 1) + tbg * 8) = make_uint2(lo, hi);
    }
    sf[sf_offset(c, tbg, Cv)] = (uint8_t)sc;
  }
}

}  // namespace

cudaError_t launch_quantize(const QKArgs& qk, const VArgs& v, bool bf16, double* ws, cudaStream_t stream) {
  const int BH = qk.B * qk.H;
  const int nchunks = qk.Np / 128;
  dim3 g1(nchunks, BH);
  if (bf16)
    kmean_partial_kernel<__nv_bfloat16><<<g1, qk.d / 2, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(qk.k), qk.k_sb, qk.k_sh, qk.k_sn, qk.H, qk.N, qk.d, ws);
  else
    kmean_partial_kernel<__half><<<g1, qk.d / 2, 0, stream>>>(reinterpret_cast<const __half*>(qk.k), qk.k_sb,
                                                              qk.k_sh, qk.k_sn, qk.H, qk.N, qk.d, ws);
  kmean_final_kernel<<<BH, qk.d, 0, stream>>>(ws, nchunks, qk.N, qk.d, qk.k_mean);
  const int64_t total = (int64_t)BH * qk.Np * (qk.d / 16);
  dim3 g2((unsigned)((total + 255) / 256), 2);
  if (bf16)
    quant_qk_kernel<__nv_bfloat16><<<g2, 256, 0, stream>>>(qk);
  else
    quant_qk_kernel<__half><<<g2, 256, 0, stream>>>(qk);
  dim3 g3(nchunks, BH);
  if (bf16)
    quant_v_kernel<__nv_bfloat16><<<g3, 256, 0, stream>>>(v);
  else
    quant_v_kernel<__half><<<g3, 256, 0, stream>>>(v);
  return cudaGetLastError();
}

}  // namespace sage3
