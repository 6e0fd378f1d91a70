// attn_common.cuh — device helpers and host tensor-map setup shared by the two attention kernels
// (attn.cu: the paper's Algorithm 1; attn_lazy.cu: the NEXT #2 lazy-reference variant).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <mutex>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

#ifndef SAGE3_POLY_MASK
#define SAGE3_POLY_MASK 0x1111
#endif
#ifndef SAGE3_POLY_DEGREE
#define SAGE3_POLY_DEGREE 4
#endif
// bit i set: exp2 pair i of each 32-key chunk (16 pairs) runs on the FMA pipe (polynomial), else on MUFU
constexpr uint32_t kPolyMask = SAGE3_POLY_MASK;
constexpr float kOneSixth = 0x1.555556p-3f;  // fl32(1/6)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLog2_2688 = 11.392317422778761f;  // log2(448 * 6)

// TMEM columns of the scale factors (both kernels): s_Q, s_K, s_V, s_P, 8 columns each.
constexpr uint32_t kColSFQ = 384, kColSFK = 392, kColSFV = 400, kColSFP = 408;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x for a pair on the FMA pipe (offloads MUFU): x = j + f with j = rint(x), f in [-0.5, 0.5];
// 2^f by a degree-5 fp32 minimax polynomial (max rel. error 2.3e-7, MUFU grade), 2^j added to the
// exponent field.  x is clamped to >= -126 so the integer add cannot wrap (2^-126 is far below any
// value that survives quantization).
__device__ __forceinline__ f2 ex2_poly2(f2 x) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: x + kMagic rounds x to an integer in the low bits
  x.x = fmaxf(x.x, -126.0f);
  x.y = fmaxf(x.y, -126.0f);
  const f2 t = fadd2(x, make_float2(kMagic, kMagic));
  const f2 jf = fadd2(t, make_float2(-kMagic, -kMagic));  // rint(x), exact
  const f2 f = fadd2(x, make_float2(-jf.x, -jf.y));       // x - rint(x), exact (Sterbenz)
#if SAGE3_POLY_DEGREE == 3
  // degree 3 (max rel. error 7.5e-5)
  f2 p = make_float2(0.055171605199575424f, 0.055171605199575424f);
  p = ffma2(p, f, make_float2(0.2426111400127411f, 0.2426111400127411f));
  p = ffma2(p, f, make_float2(0.6932610273361206f, 0.6932610273361206f));
  p = ffma2(p, f, make_float2(0.9999280571937561f, 0.9999280571937561f));
#elif SAGE3_POLY_DEGREE == 4
  // degree 4 (max rel. error 2.7e-6: below the E2M1 decision noise, reading c14)
  f2 p = make_float2(0.009570094756782055f, 0.009570094756782055f);
  p = ffma2(p, f, make_float2(0.05591786280274391f, 0.05591786280274391f));
  p = ffma2(p, f, make_float2(0.240247443318367f, 0.240247443318367f));
  p = ffma2(p, f, make_float2(0.6931217908859253f, 0.6931217908859253f));
  p = ffma2(p, f, make_float2(0.9999992847442627f, 0.9999992847442627f));
#else
  f2 p = make_float2(0.001327647129073739f, 0.001327647129073739f);
  p = ffma2(p, f, make_float2(0.009675541892647743f, 0.009675541892647743f));
  p = ffma2(p, f, make_float2(0.05550713464617729f, 0.05550713464617729f));
  p = ffma2(p, f, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = ffma2(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = ffma2(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
#endif
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

// tcgen05.wait::ld that also orders the 32 destination registers (they are "+r" operands).
__device__ __forceinline__ void tmem_ld_wait_regs(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_ld_wait_regs(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_ld_wait_regs(uint32_t (&r)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
               :
               : "memory");
}
// 32 lanes x N columns (N = 8, 16, 32) into registers, without the wait
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[16]) { tmem_ld_32x32b_x16(taddr, r); }
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[32]) { tmem_ld_32x32b_x32(taddr, r); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  tmem_ld_32x32b_x16(taddr, v);
  tmem_ld_wait_regs(v);
}

__device__ __forceinline__ uint64_t sf_desc(const void* p) {
  return make_smem_desc(smem_u32(p), 0, 128, kLayoutNone);
}

// max of 16 floats as a 3-input tree (FMNMX3)
__device__ __forceinline__ float max16(const float* v) {
  const float a = fmax3(v[0], v[1], v[2]), b = fmax3(v[3], v[4], v[5]), c = fmax3(v[6], v[7], v[8]);
  const float d = fmax3(v[9], v[10], v[11]), e = fmax3(v[12], v[13], v[14]);
  return fmax3(fmax3(a, b, c), fmax3(d, e, v[15]), -INFINITY);
}

#ifdef SAGE3_TRACE
// Debug-only timeline: clock64 stamps per role r (1,2 softmax WGs, 4 correction, 5 S-MMA, 6 PV-MMA), KV tile
// j < 128 and event k < 8, recorded by one thread per role in the CTAs with blockIdx.y == 0, blockIdx.x < 2.
__device__ unsigned long long g_trace[2][8][128][8];
#define SAGE3_TRACE_EV(role, j, k)                                                              \
  do {                                                                                         \
    if (blockIdx.y == 0 && blockIdx.x < 2 && ((threadIdx.x & 127) == 0 || threadIdx.x == 32 || threadIdx.x == 64) && (j) < 128) \
      g_trace[blockIdx.x][role][j][k] = clock64();                                             \
  } while (0)
// per-warp variant: lane 0 of each warp of the role's warpgroup records event k0 + (warp & 3)
#define SAGE3_TRACE_WARP(role, j, k0)                                                           \
  do {                                                                                         \
    if (blockIdx.y == 0 && blockIdx.x < 2 && (threadIdx.x & 31) == 0 && (j) < 128)               \
      g_trace[blockIdx.x][role][j][(k0) + ((threadIdx.x >> 5) & 3)] = clock64();               \
  } while (0)
#else
#define SAGE3_TRACE_WARP(role, j, k0) \
  do {                                \
  } while (0)
#define SAGE3_TRACE_EV(role, j, k) \
  do {                             \
  } while (0)
#endif

// ---------------------------------------------------------------- coalesced O epilogue (TMA store)
// The epilogue's per-thread row stores (one query row per thread, rows 2·d bytes apart) cost ~32 L1 wavefronts
// per warp instruction; instead each thread writes its row into smem in the SWIZZLE_128B box layout and one
// thread issues TMA tensor stores of [128 rows][128 B] boxes (rows >= N are clipped by the tensor map).
__device__ __forceinline__ void tma_store_4d(const void* tmap, const void* smem_src, int32_t c0, int32_t c1, int32_t c2,
                                             int32_t c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_group_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_group_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// Row r of the O tile (D values o, already divided by l) -> smem staging at `stage` (1024-aligned, D·esize·128
// bytes): box b = 128-byte column slice b, [128 rows][128 B], 16-byte chunk q of row r at (q ^ (r & 7)).
template <int D>
__device__ __forceinline__ void stage_o_row(uint8_t* stage, int r, int dt, const float2* o) {
  const uint32_t base = smem_u32(stage) + r * 128;
  if (dt == 2) {  // fp32: 32 values per box
#pragma unroll
    for (int c = 0; c < D / 4; ++c) {  // chunk c = values 4c..4c+3
      const int bx = c >> 3, q = c & 7;
      sts_v4(base + bx * 16384 + ((q ^ (r & 7)) * 16), __float_as_uint(o[2 * c].x), __float_as_uint(o[2 * c].y),
             __float_as_uint(o[2 * c + 1].x), __float_as_uint(o[2 * c + 1].y));
    }
  } else {  // 16-bit: 64 values per box
#pragma unroll
    for (int c = 0; c < D / 8; ++c) {  // chunk c = values 8c..8c+7
      const int bx = c >> 3, q = c & 7;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 v = o[4 * c + e];
        if (dt == 1) {
          __nv_bfloat162 h2 = __floats2bfloat162_rn(v.x, v.y);
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        } else {
          __half2 h2 = __floats2half2_rn(v.x, v.y);
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
      }
      sts_v4(base + bx * 16384 + ((q ^ (r & 7)) * 16), w[0], w[1], w[2], w[3]);
    }
  }
}
// Columns [32c, 32c + 32) of row r (fp32 values f, already divided by l) -> the same staging layout.
__device__ __forceinline__ void stage_o_cols32(uint8_t* stage, int r, int dt, int c, const float* f) {
  const uint32_t base = smem_u32(stage) + r * 128;
  if (dt == 2) {
#pragma unroll
    for (int k = 0; k < 8; ++k)  // chunk 8c + k: box c, position k
      sts_v4(base + c * 16384 + ((k ^ (r & 7)) * 16), __float_as_uint(f[4 * k]), __float_as_uint(f[4 * k + 1]),
             __float_as_uint(f[4 * k + 2]), __float_as_uint(f[4 * k + 3]));
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // chunk 4c + k
      const int ch = 4 * c + k, bx = ch >> 3, q = ch & 7;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (dt == 1) {
          __nv_bfloat162 h2 = __floats2bfloat162_rn(f[8 * k + 2 * e], f[8 * k + 2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        } else {
          __half2 h2 = __floats2half2_rn(f[8 * k + 2 * e], f[8 * k + 2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&h2);
        }
      }
      sts_v4(base + bx * 16384 + ((q ^ (r & 7)) * 16), w[0], w[1], w[2], w[3]);
    }
  }
}
// The staged tile -> O[b][h][q0 .. q0+128)[0 .. D) (one thread; waits until smem has been read).
template <int D>
__device__ __forceinline__ void store_o_tile(const void* tm_o, const uint8_t* stage, int dt, int q0, int h, int b) {
  const int boxes = D * (dt == 2 ? 4 : 2) / 128, per = dt == 2 ? 32 : 64;
  for (int bx = 0; bx < boxes; ++bx) tma_store_4d(tm_o, stage + bx * 16384, bx * per, q0, h, b);
  bulk_group_commit();
  bulk_group_wait_read0();
}

// ------------------------------------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D uint8 map: rows of `row_bytes`, box = box_bytes x box_rows, swizzle matching the UMMA layout.
bool make_map(CUtensorMap* m, const void* base, uint64_t row_bytes, uint64_t rows, uint32_t box_bytes,
              uint32_t box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle swz = box_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  return encode_tiled_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// O [B][H][N][D] (element strides, d-stride 1) in sage3_dtype dt: 4-D map with 128-byte x 128-row boxes,
// SWIZZLE_128B (the layout stage_o_row writes).
bool make_map_o(CUtensorMap* m, const void* base, int dt, int B, int H, int N, int D, int64_t sb, int64_t sh,
                int64_t sn) {
  auto enc = encode_fn();
  if (!enc) return false;
  const int es = dt == 2 ? 4 : 2;
  if (H == 1) sh = sn * N;
  if (B == 1) sb = sh * H;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)sn * es, (cuuint64_t)sh * es, (cuuint64_t)sb * es};
  cuuint32_t box[4] = {(cuuint32_t)(128 / es), 128, 1, 1};
  cuuint32_t ones[4] = {1, 1, 1, 1};
  return encode_tiled_cached(enc, m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(base),
             dims, strides, box, ones, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace
}  // namespace sage3
