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
// Q or K rows of one 128-token chunk: thread t owns row t/2 and G = d/32 consecutive 16-blocks (2G 16-byte
// loads, 8G code bytes, G scale bytes that are consecutive in the SF atom).  kSmooth: x = fl32(K - km).
template <typename T, int D, bool kSmooth>
__device__ __forceinline__ void quant_rows(const T* __restrict__ src, int64_t sn, int N, int n0,
                                           const float* __restrict__ km, uint8_t* __restrict__ codes_chunk,
                                           uint8_t* sf_stage, bool& finite) {
  constexpr int G = D / 32;
  const int t = threadIdx.x;
  const int row = t >> 1, g = t & 1;
  const int n = n0 + row;
  uint32_t w[2 * G];
  uint32_t scs = 0;
  if (n < N) {
    const T* p = src + (int64_t)n * sn + g * 16 * G;
    uint4 u[2 * G];
#pragma unroll
    for (int i = 0; i < 2 * G; ++i) u[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
#pragma unroll
    for (int blk = 0; blk < G; ++blk) {
      float x[16];
      unpack8<T>(u[2 * blk], x);
      unpack8<T>(u[2 * blk + 1], x + 8);
      finite &= all_finite(x, 16);
      if constexpr (kSmooth) {
        const float4* m = reinterpret_cast<const float4*>(km + (g * G + blk) * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 mm = m[i];
          x[4 * i + 0] = __fsub_rn(x[4 * i + 0], mm.x);
          x[4 * i + 1] = __fsub_rn(x[4 * i + 1], mm.y);
          x[4 * i + 2] = __fsub_rn(x[4 * i + 2], mm.z);
          x[4 * i + 3] = __fsub_rn(x[4 * i + 3], mm.w);
        }
      }
      uint32_t sc;
      phi16(x, w[2 * blk], w[2 * blk + 1], sc);
      scs |= sc << (8 * blk);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 2 * G; ++i) w[i] = 0u;
  }
  // codes: row-major, D/2 bytes per row -> this thread's 8G bytes are contiguous and consecutive threads
  // are consecutive (fully coalesced 16-byte stores)
  uint4* dst = reinterpret_cast<uint4*>(codes_chunk + row * (D / 2) + g * 8 * G);
#pragma unroll
  for (int i = 0; i < G / 2; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  // scales: block columns g*G .. g*G+G-1 of row `row` are consecutive bytes of one 512-byte atom
  const int c0 = g * G;
  const int off = (c0 >> 2) * 512 + (row & 31) * 16 + ((row >> 5) & 3) * 4 + (c0 & 3);
  if constexpr (G == 4)
    *reinterpret_cast<uint32_t*>(sf_stage + off) = scs;
  else
    *reinterpret_cast<uint16_t*>(sf_stage + off) = (uint16_t)scs;
}

// Copy `bytes` (multiple of 16) from smem to global with 16-byte stores by the whole block.
__device__ __forceinline__ void block_copy16(uint8_t* __restrict__ gdst, const uint8_t* sdst, int bytes) {
  for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(gdst + i) = *reinterpret_cast<const uint4*>(sdst + i);
}

// ---------------------------------------------------------------------------------- pass A: Q, V, ΣK
// grid (Np/128, B*H), block 256, one 128-token chunk of one (b,h):
//   φ(Q) rows (along d); φ(Vᵀ) (16-token blocks per channel, via an smem transpose, staged codes and SF
//   atoms written with coalesced 16-byte stores); fp64 per-channel sums of the K chunk (sequential in token
//   order, c10) into ws.  The last chunk CTA of a head (atomic counter) then reduces the chunk sums in
//   ascending chunk order and writes km = fl32(total / N); pass B (φ(K - km)) runs after it in stream order.
template <typename T, int D>
__global__ void __launch_bounds__(256) quant_pass_a_kernel(QKArgs qa, VArgs va, double* __restrict__ ws,
                                                           uint32_t* __restrict__ counters) {
  constexpr int kVec = D / 8;  // 16-byte vectors per token row
  extern __shared__ __align__(16) uint8_t dsm[];
  T* sK = reinterpret_cast<T*>(dsm);                                 // K chunk [128][D]
  T* sV = sK + 128 * D;                                               // V chunk [128][D]
  uint8_t* sVcode = reinterpret_cast<uint8_t*>(sV + 128 * D);         // Vᵀ codes: D channel rows x 64 bytes
  uint8_t(*sSF)[1024] = reinterpret_cast<uint8_t(*)[1024]>(sVcode + D * 64);  // [0] Q SF, [1] Vᵀ SF atoms
  __shared__ uint32_t s_last;
  const int chunk = blockIdx.x, bh = blockIdx.y;
  const int b = bh / qa.H, h = bh % qa.H;
  const int n0 = chunk * 128, N = qa.N, Np = qa.Np;
  const int t = threadIdx.x;
  bool finite = true;
  // ---- stage K and V chunks in smem (16-byte loads, all issued before use)
  {
    const T* kb = reinterpret_cast<const T*>(qa.k) + b * qa.k_sb + h * qa.k_sh;
    const T* vb = reinterpret_cast<const T*>(va.v) + b * va.sb + h * va.sh;
    constexpr int kIters = 128 * kVec / 256;
    uint4 uk[kIters], uv[kIters];
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      const int i = it * 256 + t, r = i / kVec, cv = i % kVec, n = n0 + r;
      uk[it] = n < N ? __ldg(reinterpret_cast<const uint4*>(kb + (int64_t)n * qa.k_sn + cv * 8)) : make_uint4(0, 0, 0, 0);
      uv[it] = n < N ? __ldg(reinterpret_cast<const uint4*>(vb + (int64_t)n * va.sn + cv * 8)) : make_uint4(0, 0, 0, 0);
    }
    // Q rows meanwhile (their loads are in flight with the K/V ones)
    const T* qb = reinterpret_cast<const T*>(qa.q) + b * qa.q_sb + h * qa.q_sh;
    for (int i = t; i < 2 * 1024 / 16; i += 256) reinterpret_cast<uint4*>(sSF)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    quant_rows<T, D, false>(qb, qa.q_sn, N, n0, nullptr, qa.q_data + ((int64_t)bh * Np + n0) * (D / 2), sSF[0],
                            finite);
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      const int i = it * 256 + t;
      reinterpret_cast<uint4*>(sK)[i] = uk[it];
      reinterpret_cast<uint4*>(sV)[i] = uv[it];
      if (qa.nonfinite) {
        float f[8];
        unpack8<T>(uk[it], f);
        finite &= all_finite(f, 8);
        unpack8<T>(uv[it], f);
        finite &= all_finite(f, 8);
      }
    }
  }
  __syncthreads();
  // ---- ΣK over the chunk's real tokens, fp64, ascending token order: threads 0..D/2-1, two channels each
  if (t < D / 2) {
    const int nend = min(128, N - n0);
    double a0 = 0.0, a1 = 0.0;
    const uint32_t* col = reinterpret_cast<const uint32_t*>(sK) + t;
    for (int r = 0; r < nend; ++r) {
      const uint32_t u = col[r * (D / 2)];
      const T* p = reinterpret_cast<const T*>(&u);
      a0 += (double)to_f32<T>(p[0]);
      a1 += (double)to_f32<T>(p[1]);
    }
    double* out = ws + ((int64_t)bh * gridDim.x + chunk) * D + 2 * t;
    out[0] = a0;
    out[1] = a1;
  }
  // ---- φ(Vᵀ): item = (channel pair cp, 16-token block tb); consecutive threads read consecutive 32-bit
  //      words of a token row (conflict-free), 16 token rows per block
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
  // ---- coalesced stores: Vᵀ code rows (64 bytes of channel c per chunk), Q and Vᵀ SF atoms
  for (int i = t; i < D * 4; i += 256) {
    const int c = i >> 2, q = i & 3;
    *reinterpret_cast<uint4*>(va.v_data + ((int64_t)bh * D + c) * (Np >> 1) + chunk * 64 + q * 16) =
        *reinterpret_cast<const uint4*>(sVcode + c * 64 + q * 16);
  }
  block_copy16(qa.q_sf + (int64_t)bh * Np * (D / 16) + (int64_t)chunk * 512 * (D / 64), sSF[0], 512 * (D / 64));
  block_copy16(va.v_sf + (int64_t)bh * 128 * (Np >> 4) + (int64_t)chunk * 1024, sSF[1], 1024);
  // ---- last chunk CTA of this head: km = fl32(Σ_chunks (ascending) / N)
  __threadfence();
  __syncthreads();
  if (t == 0) s_last = atomicAdd(&counters[bh], 1u) == gridDim.x - 1 ? 1u : 0u;
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int nch = gridDim.x;
    for (int c = t; c < D; c += 256) {
      const double* p = ws + (int64_t)bh * nch * D + c;
      double total = 0.0;
      int i = 0;
      for (; i + 8 <= nch; i += 8) {  // loads issued together, added in order
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcg(p + (int64_t)(i + k) * D);
#pragma unroll
        for (int k = 0; k < 8; ++k) total += v[k];
      }
      for (; i < nch; ++i) total += __ldcg(p + (int64_t)i * D);
      qa.k_mean[(int64_t)bh * D + c] = (float)(total / (double)N);
    }
    if (t == 0) counters[bh] = 0u;  // ready for the next call (also zeroed by the host before pass A)
  }
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
constexpr int pass_a_smem() {
  return 2 * 128 * D * 2 + D * 64 + 2 * 1024;
}

template <typename T, int D>
cudaError_t launch_t(const QKArgs& qk, const VArgs& v, double* ws, uint32_t* counters, cudaStream_t stream) {
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(quant_pass_a_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pass_a_smem<D>());
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = qk.B * qk.H;
  dim3 grid(qk.Np / 128, BH);
  quant_pass_a_kernel<T, D><<<grid, 256, pass_a_smem<D>(), stream>>>(qk, v, ws, counters);
  quant_pass_b_kernel<T, D><<<grid, 256, 0, stream>>>(qk);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const QKArgs& qk, const VArgs& v, bool bf16, double* ws, uint32_t* counters,
                            cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(counters, 0, sizeof(uint32_t) * qk.B * qk.H, stream);
  if (e != cudaSuccess) return e;
  if (qk.d == 128)
    return bf16 ? launch_t<__nv_bfloat16, 128>(qk, v, ws, counters, stream)
                : launch_t<__half, 128>(qk, v, ws, counters, stream);
  return bf16 ? launch_t<__nv_bfloat16, 64>(qk, v, ws, counters, stream)
              : launch_t<__half, 64>(qk, v, ws, counters, stream);
}

}  // namespace sage3
