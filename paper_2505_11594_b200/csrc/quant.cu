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

// ---------------------------------------------------------------------------------- shared pieces
// Q or K rows of one 128-token chunk (φ along d).  The chunk is read as consecutive 16-byte vectors (vector
// i = it*256 + t: every warp load instruction covers 512 contiguous bytes); the two threads holding the two
// halves of a 16-element block exchange their partial amax with one shuffle and each writes the 4 code bytes
// of its half (again consecutive across the warp).  Scale bytes go to the chunk's SF atoms staged in smem.
// kSmooth: x = fl32(K - km).
template <typename T, int D, bool kSmooth>
__device__ __forceinline__ void quant_rows(const T* __restrict__ src, int64_t sn, int N, int n0,
                                           const float* __restrict__ km, uint8_t* __restrict__ codes_chunk,
                                           uint8_t* sf_stage, bool& finite) {
  constexpr int kVec = D / 8;              // 16-byte vectors per row
  constexpr int kIt = 128 * kVec / 256;    // vectors per thread
  const int t = threadIdx.x;
  uint4 u[kIt];
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int i = it * 256 + t, r = i / kVec, cv = i % kVec, n = n0 + r;
    u[it] = n < N ? __ldg(reinterpret_cast<const uint4*>(src + (int64_t)n * sn + cv * 8)) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int i = it * 256 + t, r = i / kVec, cv = i % kVec;
    float x[8];
    unpack8<T>(u[it], x);
    finite &= all_finite(x, 8);
    if constexpr (kSmooth) {
      const float4 m0 = reinterpret_cast<const float4*>(km + cv * 8)[0];
      const float4 m1 = reinterpret_cast<const float4*>(km + cv * 8)[1];
      x[0] = __fsub_rn(x[0], m0.x), x[1] = __fsub_rn(x[1], m0.y), x[2] = __fsub_rn(x[2], m0.z);
      x[3] = __fsub_rn(x[3], m0.w), x[4] = __fsub_rn(x[4], m1.x), x[5] = __fsub_rn(x[5], m1.y);
      x[6] = __fsub_rn(x[6], m1.z), x[7] = __fsub_rn(x[7], m1.w);
    }
    float amax = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) amax = fmaxf(amax, fabsf(x[k]));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
    const uint32_t sc = cvt_e4m3x2(__fmul_rn(amax, kOneSixth), 0.0f) & 0xFFu;
    const float s = e4m3_to_f32(sc);
    uint32_t w = 0u;
    if (s != 0.0f) {
      const float rs = __frcp_rn(s);
      w = cvt_e2m1x2(__fmul_rn(x[0], rs), __fmul_rn(x[1], rs)) | (cvt_e2m1x2(__fmul_rn(x[2], rs), __fmul_rn(x[3], rs)) << 8) |
          (cvt_e2m1x2(__fmul_rn(x[4], rs), __fmul_rn(x[5], rs)) << 16) |
          (cvt_e2m1x2(__fmul_rn(x[6], rs), __fmul_rn(x[7], rs)) << 24);
    }
    *reinterpret_cast<uint32_t*>(codes_chunk + r * (D / 2) + cv * 4) = w;
    if ((cv & 1) == 0) {
      const int c = cv >> 1;  // block column
      sf_stage[(c >> 2) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (c & 3)] = (uint8_t)sc;
    }
  }
}

// Copy `bytes` (multiple of 16) from smem to global with 16-byte stores by the whole block.
__device__ __forceinline__ void block_copy16(uint8_t* __restrict__ gdst, const uint8_t* sdst, int bytes) {
  for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(gdst + i) = *reinterpret_cast<const uint4*>(sdst + i);
}

// ---------------------------------------------------------------------------------- K mean
// grid (Np/128, B*H), block d/2: thread t sums channels 2t, 2t+1 over one 128-token chunk in ascending token
// order (fp64, sequential; 4-byte loads, a warp reads 128 contiguous bytes of a token row), writes
// ws[bh][chunk][c]; kmean_final_kernel then reduces the chunk sums (reading c10).
template <typename T>
__global__ void __launch_bounds__(64) kmean_kernel(const T* __restrict__ k, int64_t sb, int64_t sh, int64_t sn,
                                                   int H, int N, int d, double* __restrict__ ws) {
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
    const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(base + (int64_t)n * sn));
    const T* p = reinterpret_cast<const T*>(&v);
    a0 += (double)to_f32<T>(p[0]);
    a1 += (double)to_f32<T>(p[1]);
  }
  double* out = ws + ((int64_t)bh * gridDim.x + chunk) * d + c;
  out[0] = a0;
  out[1] = a1;
}

// grid (B*H*d/128), block 128: one thread per (bh, channel) sums the chunk sums in ascending chunk order
// (loads issued 8 at a time, added in order) and writes km = fl32(total / N).
__global__ void __launch_bounds__(128) kmean_final_kernel(const double* __restrict__ ws, int nchunks, int N, int d,
                                                          int total_ch, float* __restrict__ km) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total_ch) return;
  const int bh = idx / d, c = idx % d;
  const double* p = ws + (int64_t)bh * nchunks * d + c;
  double total = 0.0;
  int i = 0;
  for (; i + 8 <= nchunks; i += 8) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = p[(int64_t)(i + q) * d];
#pragma unroll
    for (int q = 0; q < 8; ++q) total += v[q];
  }
  for (; i < nchunks; ++i) total += p[(int64_t)i * d];
  km[idx] = (float)(total / (double)N);
}

// ---------------------------------------------------------------------------------- Q and Vᵀ
// grid (Np/128, B*H), block 256, one 128-token chunk of one (b,h): φ(Q) rows (along d) straight from
// registers; φ(Vᵀ) (16-token blocks per channel) through an smem transpose, codes and SF atoms staged in
// smem and written with coalesced 16-byte stores.
template <typename T, int D>
__global__ void __launch_bounds__(256) quant_qv_kernel(QKArgs qa, VArgs va) {
  constexpr int kVec = D / 8;  // 16-byte vectors per token row
  extern __shared__ __align__(16) uint8_t dsm[];
  T* sV = reinterpret_cast<T*>(dsm);                                  // V chunk [128][D]
  uint8_t* sVcode = reinterpret_cast<uint8_t*>(sV + 128 * D);         // Vᵀ codes: D channel rows x 64 bytes
  uint8_t(*sSF)[1024] = reinterpret_cast<uint8_t(*)[1024]>(sVcode + D * 64);  // [0] Q SF, [1] Vᵀ SF atoms
  const int chunk = blockIdx.x, bh = blockIdx.y;
  const int b = bh / qa.H, h = bh % qa.H;
  const int n0 = chunk * 128, N = qa.N, Np = qa.Np;
  const int t = threadIdx.x;
  bool finite = true;
  {
    const T* vb = reinterpret_cast<const T*>(va.v) + b * va.sb + h * va.sh;
    constexpr int kIters = 128 * kVec / 256;
    uint4 uv[kIters];
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      const int i = it * 256 + t, r = i / kVec, cv = i % kVec, n = n0 + r;
      uv[it] = n < N ? __ldg(reinterpret_cast<const uint4*>(vb + (int64_t)n * va.sn + cv * 8)) : make_uint4(0, 0, 0, 0);
    }
    for (int i = t; i < 2 * 1024 / 16; i += 256) reinterpret_cast<uint4*>(sSF)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const T* qb = reinterpret_cast<const T*>(qa.q) + b * qa.q_sb + h * qa.q_sh;
    quant_rows<T, D, false>(qb, qa.q_sn, N, n0, nullptr, qa.q_data + ((int64_t)bh * Np + n0) * (D / 2), sSF[0],
                            finite);
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      reinterpret_cast<uint4*>(sV)[it * 256 + t] = uv[it];
      if (qa.nonfinite) {
        float f[8];
        unpack8<T>(uv[it], f);
        finite &= all_finite(f, 8);
      }
    }
  }
  __syncthreads();
  // item = (channel pair cp, 16-token block tb); consecutive threads read consecutive 32-bit words of a
  // token row (conflict-free), 16 token rows per block
  for (int item = t; item < (D / 2) * 8; item += 256) {
    const int cp = item % (D / 2), tb = item / (D / 2);
    float x0[16], x1[16];
    const uint32_t* col = reinterpret_cast<const uint32_t*>(sV) + tb * 16 * (D / 2) + cp;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t u = col[k * (D / 2)];
      const T* p = reinterpret_cast<const T*>(&u);
      x0[k] = to_f32<T>(p[0]);
      x1[k] = to_f32<T>(p[1]);
    }
    uint32_t lo, hi, sc0, sc1;
    const int c = 2 * cp;
    phi16(x0, lo, hi, sc0);
    *reinterpret_cast<uint2*>(sVcode + c * 64 + tb * 8) = make_uint2(lo, hi);
    phi16(x1, lo, hi, sc1);
    *reinterpret_cast<uint2*>(sVcode + (c + 1) * 64 + tb * 8) = make_uint2(lo, hi);
    const int base = (tb >> 2) * 512 + ((c >> 5) & 3) * 4 + (tb & 3);
    sSF[1][base + (c & 31) * 16] = (uint8_t)sc0;
    sSF[1][base + ((c + 1) & 31) * 16] = (uint8_t)sc1;
  }
  if (qa.nonfinite && !finite) atomicOr(qa.nonfinite, 1u);
  __syncthreads();
  for (int i = t; i < D * 4; i += 256) {
    const int c = i >> 2, q = i & 3;
    *reinterpret_cast<uint4*>(va.v_data + ((int64_t)bh * D + c) * (Np >> 1) + chunk * 64 + q * 16) =
        *reinterpret_cast<const uint4*>(sVcode + c * 64 + q * 16);
  }
  block_copy16(qa.q_sf + (int64_t)bh * Np * (D / 16) + (int64_t)chunk * 512 * (D / 64), sSF[0], 512 * (D / 64));
  block_copy16(va.v_sf + (int64_t)bh * 128 * (Np >> 4) + (int64_t)chunk * 1024, sSF[1], 1024);
}

// ---------------------------------------------------------------------------------- pass B: φ(K - km)
template <typename T, int D>
__global__ void __launch_bounds__(256) quant_pass_b_kernel(QKArgs qa) {
  __shared__ __align__(16) uint8_t sSF[1024];
  __shared__ __align__(16) float sKm[D];
  const int chunk = blockIdx.x, bh = blockIdx.y;
  const int b = bh / qa.H, h = bh % qa.H;
  const int t = threadIdx.x;
  for (int i = t; i < 1024 / 16; i += 256) reinterpret_cast<uint4*>(sSF)[i] = make_uint4(0, 0, 0, 0);
  for (int i = t; i < D; i += 256) sKm[i] = qa.k_mean[(int64_t)bh * D + i];
  __syncthreads();
  bool finite = true;
  const T* kb = reinterpret_cast<const T*>(qa.k) + b * qa.k_sb + h * qa.k_sh;
  quant_rows<T, D, true>(kb, qa.k_sn, qa.N, chunk * 128, sKm, qa.k_data + ((int64_t)bh * qa.Np + chunk * 128) * (D / 2),
                         sSF, finite);
  __syncthreads();
  block_copy16(qa.k_sf + (int64_t)bh * qa.Np * (D / 16) + (int64_t)chunk * 512 * (D / 64), sSF, 512 * (D / 64));
}

template <int D>
constexpr int qv_smem() {
  return 128 * D * 2 + D * 64 + 2 * 1024;
}

template <typename T, int D>
cudaError_t launch_t(const QKArgs& qk, const VArgs& v, double* ws, cudaStream_t stream) {
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(quant_qv_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         qv_smem<D>());
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = qk.B * qk.H;
  dim3 grid(qk.Np / 128, BH);
  kmean_kernel<T><<<grid, D / 2, 0, stream>>>(reinterpret_cast<const T*>(qk.k), qk.k_sb, qk.k_sh, qk.k_sn, qk.H,
                                              qk.N, D, ws);
  kmean_final_kernel<<<(BH * D + 127) / 128, 128, 0, stream>>>(ws, qk.Np / 128, qk.N, D, BH * D, qk.k_mean);
  quant_qv_kernel<T, D><<<grid, 256, qv_smem<D>(), stream>>>(qk, v);
  quant_pass_b_kernel<T, D><<<grid, 256, 0, stream>>>(qk);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const QKArgs& qk, const VArgs& v, bool bf16, double* ws, cudaStream_t stream) {
  if (qk.d == 128)
    return bf16 ? launch_t<__nv_bfloat16, 128>(qk, v, ws, stream)
                : launch_t<__half, 128>(qk, v, ws, stream);
  return bf16 ? launch_t<__nv_bfloat16, 64>(qk, v, ws, stream)
              : launch_t<__half, 64>(qk, v, ws, stream);
}

}  // namespace sage3
