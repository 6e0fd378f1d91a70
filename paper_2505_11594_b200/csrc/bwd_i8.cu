// bwd_i8.cu — SageBwd's 8-bit attention backward (NEXT #3; Algorithm 3) on sm_100a.
//
// Three launches:
//   prep    per 128-row block of dO: ψ(dO_i) (Alg3 L6, per-block INT8, reading b1), D = rowsum(dO∘O) (L2,
//           fp32), L' = lse·log2 e (+inf on padding rows, which makes their P exactly 0).
//   main    one CTA per (b·h, KV tile j), looping over the query tiles i (i >= j under the causal mask).
//           Per (i, j), with S, P and dS held one query row per thread (TMEM lane = query):
//             S    = MM(Q̂_i, K̂_j)                 kind::i8, int32 in TMEM (exact)            (L5)
//             dP   = MM(dO_i, V_jᵀ)               kind::f16 on the 16-bit dO and V    (L8)
//             P    = exp(scale·S·s_Q·s_K − L_i);  ψ(P) with one scale per tile                (L5-L6)
//             dS   = P∘(dP − D_i);                ψ(dS) with one scale per tile              (L9)
//             dV_j += MM(P̂ᵀ, dÔ_i)·s_P·s_dO      kind::i8, A = P̂ᵀ and B = dÔ_i MN-major     (L7)
//             dK_j += MM(dŜᵀ, Q̂_i)·s_dS·s_Q      kind::i8, A = dŜᵀ and B = Q̂_i MN-major     (L11)
//             dQ_i += MM(dŜ, K̂_j)·s_dS·s_K + rowsum(dS)·K_m                              (L10)
//           Every int8 product lands in TMEM as an int32 partial; because s_P and s_dS change per tile, the
//           fp32 accumulation happens outside the tensor core: dV_j in the registers of warpgroup 2, dK_j in
//           warpgroup 3, and the dQ_i partial (one per (i, j) pair, summed over the CTAs of the head) is
//           added into an fp32 workspace with TMA reduce-add (cp.reduce.async.bulk.tensor .add.f32).
//   final   dQ = scale·dQ_acc (the softmax scale multiplies S inside the softmax, reading b7).
//
// Warp roles of the main kernel (16 warps): warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator,
// WG1 element-wise work (P, ψ(P), dS, ψ(dS), rowsum), WG2 dV accumulation + store, WG3 dK accumulation +
// dQ flush + dK store.  TMEM (512 columns): S buffers at 0 and 256 (tile t uses t % 2; its dQ partial is
// written over it); regions Y (128) and W (384) alternate by tile parity between "dP / dS, then the dK partial"
// (R1) and "the dV partial" (R2), so the next tile's dP never waits for the dK read.
// WG2 and WG3 each flush half of every dQ partial.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "attn_common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

#ifndef SAGE3_BWD_I2F
#define SAGE3_BWD_I2F 1  // int32 -> fp32 by cvt (I2F) instead of the magic-number add
#endif
constexpr int kBThreads = 512;
constexpr uint32_t kBRegWG0 = 40, kBRegElem = 136, kBRegDV = 160, kBRegDK = 176;
static_assert(kBRegWG0 + kBRegElem + kBRegDV + kBRegDK <= 512, "register budget");
[[maybe_unused]] constexpr uint32_t kMagicIB = 0x4B400000u;  // float 1.5·2^23 bits: int x + kMagicIB reinterpreted = 12582912 + x
constexpr float kMagicFB = 12582912.0f;
constexpr float kOne127B = 0x1.020408p-7f;  // fl32(1/127)
constexpr int kDQBufs = 3;  // dQ staging buffers per WG3 warp
constexpr uint32_t kColS0 = 0, kColY = 128, kColS1 = 256, kColW = 384;
// Regions Y and W alternate roles by tile parity: tile t holds dP(t) / dS(t) and then its dK partial in
// R1(t), its dV partial in R2(t) = R1(t+1).  dP(t+1) then only waits for WG2 to read dV(t) (early), not for
// WG3 to read dK(t) (late).
__device__ __forceinline__ uint32_t r1col(int t) { return (t & 1) ? kColW : kColY; }
__device__ __forceinline__ uint32_t r2col(int t) { return (t & 1) ? kColY : kColW; }

// kind::i8: D s32, A/B signed; a_mn / b_mn select MN-major operands (bits 15 / 16).
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (a_mn ? 1u << 15 : 0u) | (b_mn ? 1u << 16 : 0u) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}
// kind::f16: D f32, A/B f16 (0) or bf16 (1), K-major.
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N, uint32_t ab) {
  return (1u << 4) | (ab << 7) | (ab << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8b(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_f16b(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ f2 i2f2b(uint32_t a, uint32_t b) {  // exact int32 -> fp32 (|x| < 2^24): I2F
#if SAGE3_BWD_I2F
  return make_float2(__int2float_rn((int)a), __int2float_rn((int)b));
#else
  return fadd2(make_float2(__uint_as_float(a + kMagicIB), __uint_as_float(b + kMagicIB)),
               make_float2(-kMagicFB, -kMagicFB));
#endif
}
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// 4 RNE'd values (already + 1.5·2^23, so the low byte of each is the two's-complement code) -> one word
__device__ __forceinline__ uint32_t pack4(f2 t0, f2 t1) {
  const uint32_t lo = __byte_perm(__float_as_uint(t0.x), __float_as_uint(t0.y), 0x0040);
  const uint32_t hi = __byte_perm(__float_as_uint(t1.x), __float_as_uint(t1.y), 0x0040);
  return __byte_perm(lo, hi, 0x5410);
}

// One row of D fp32 values (x mul) -> a strided [B][H][N][D] tensor in sage3_dtype dt (0 fp16, 1 bf16, 2 fp32).
template <int D>
__device__ __forceinline__ void store_row(void* base, int64_t sb, int64_t sh, int64_t sn, int dt, int b, int h,
                                          int n, const f2* v, float mul) {
  const int64_t off = b * sb + h * sh + (int64_t)n * sn;
  if (dt == 2) {
    float* dst = reinterpret_cast<float*>(base) + off;
#pragma unroll
    for (int c = 0; c < D / 2; c += 2)
      *reinterpret_cast<float4*>(dst + 2 * c) =
          make_float4(v[c].x * mul, v[c].y * mul, v[c + 1].x * mul, v[c + 1].y * mul);
  } else if (dt == 1) {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(base) + off;
#pragma unroll
    for (int c = 0; c < D / 2; c += 4) {
      uint4 u;
      __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) p[e] = __floats2bfloat162_rn(v[c + e].x * mul, v[c + e].y * mul);
      *reinterpret_cast<uint4*>(dst + 2 * c) = u;
    }
  } else {
    __half* dst = reinterpret_cast<__half*>(base) + off;
#pragma unroll
    for (int c = 0; c < D / 2; c += 4) {
      uint4 u;
      __half2* p = reinterpret_cast<__half2*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) p[e] = __floats2half2_rn(v[c + e].x * mul, v[c + e].y * mul);
      *reinterpret_cast<uint4*>(dst + 2 * c) = u;
    }
  }
}

// One warp's share of a dQ partial: columns [c0, c0 + 16·NCH) of its 32 rows (TMEM lanes), scaled
// y = int·w_q + rowsum(dS)·K_m, staged in smem ([32 rows][16 fp32], SWIZZLE_64B, kDQBufs buffers per warp)
// and added into the fp32 dQ accumulator by this warp's own TMA reduce-adds (box 16 x 32).
__device__ __forceinline__ __attribute__((unused)) void red_add_v4(float* gaddr, f2 a, f2 b) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(gaddr), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y)
               : "memory");
}
#ifndef SAGE3_BWD_DQ_TMA
#define SAGE3_BWD_DQ_TMA 1
#endif
template <int NCH>
__device__ __forceinline__ void flush_dq(const CUtensorMap* tm, uint32_t tQ, int c0, uint8_t* stage, int& nflush,
                                         const float* s_km, f2 wq2, f2 rs2, int r, int lane, int row0,
                                         float* dq_row) {
  if constexpr (!SAGE3_BWD_DQ_TMA) {
    // vector reductions straight from registers (red.global.add.v4.f32): no shared-memory traffic, which the
    // MMAs' operand reads already saturate
#pragma unroll
    for (int k = 0; k < NCH; k += 2) {
      uint32_t va[16], vb[16];
      tmem_ld_32x32b_x16(tQ + c0 + 16 * k, va);
      tmem_ld_32x32b_x16(tQ + c0 + 16 * k + 16, vb);
      tmem_ld_wait_regs(va);
      tmem_ld_wait_regs(vb);
      auto put = [&](int kk, const uint32_t(&v)[16]) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col = c0 + 16 * kk + 4 * q;
          float4 km;
          lds_f4(smem_u32(s_km + col), km);
          const f2 y0 = ffma2(i2f2b(v[4 * q], v[4 * q + 1]), wq2, fmul2(rs2, make_float2(km.x, km.y)));
          const f2 y1 = ffma2(i2f2b(v[4 * q + 2], v[4 * q + 3]), wq2, fmul2(rs2, make_float2(km.z, km.w)));
          red_add_v4(dq_row + col, y0, y1);
        }
      };
      put(k, va);
      put(k + 1, vb);
    }
    return;
  }
#pragma unroll 1
  for (int k = 0; k < NCH; ++k, ++nflush) {
    uint8_t* buf = stage + (nflush % kDQBufs) * 2048;
    uint32_t v[16];
    tmem_ld_32x32b_x16(tQ + c0 + 16 * k, v);
    if (lane == 0) bulk_wait_read<kDQBufs - 1>();  // this warp's reduce that last read `buf` is done
    __syncwarp();
    tmem_ld_wait_regs(v);
    const uint32_t row = smem_u32(buf) + (r & 31) * 64;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float4 km;
      lds_f4(smem_u32(s_km + c0 + 16 * k + 4 * q), km);
      const f2 y0 = ffma2(i2f2b(v[4 * q], v[4 * q + 1]), wq2, fmul2(rs2, make_float2(km.x, km.y)));
      const f2 y1 = ffma2(i2f2b(v[4 * q + 2], v[4 * q + 3]), wq2, fmul2(rs2, make_float2(km.z, km.w)));
      sts_v4(row + ((q ^ ((r >> 1) & 3)) * 16), __float_as_uint(y0.x), __float_as_uint(y0.y), __float_as_uint(y1.x),
             __float_as_uint(y1.y));
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_reduce_add_2d(tm, buf, c0 + 16 * k, row0);
      bulk_commit();
    }
  }
}

template <int D>
struct BLayout {
  static constexpr int kI8Tile = 128 * D;         // Q̂ / K̂ / dÔ tile (row-major, D bytes per row)
  static constexpr int k16Tile = 128 * D * 2;     // V / dO tile: D/64 boxes of 128 rows x 128 B
  static constexpr int oK = 0;
  static constexpr int oV = oK + kI8Tile;
  static constexpr int oQ = oV + k16Tile;          // 2 stages
  static constexpr int oDO = oQ + 2 * kI8Tile;
  static constexpr int oDOq = oDO + k16Tile;
  static constexpr int oP = oDOq + kI8Tile;        // P̂: 128 query rows x 128 keys
  static constexpr int oDS = oP + 128 * 128;       // dŜ: same layout
  static constexpr int oDQ = oDS + 128 * 128;      // dQ staging: 8 warps x kDQBufs x [32 rows][16 fp32]
  static constexpr int oLD = oDQ + 8 * kDQBufs * 2048;      // 2 stages x (L' [128], D [128]) fp32
  static constexpr int oKm = oLD + 2 * 1024;       // K_m [D] fp32
  static constexpr int oX = oKm + 512;             // 4 slots x (s_P, s_dS, pad, rowsum(dS)[128] at +512)
  static constexpr int oRed = oX + 4 * 1024;       // 2 x 4 floats (tile amax reductions)
  static constexpr int oScl = oRed + 64;           // s_Q[Np/128], s_dO[Np/128] of the head (<= 1024 each)
  static constexpr int oBar = oScl + 2 * 4096;
  static constexpr int kNumBars = 1 + 2 + 2 + 2 + 2 + 2 + 1 + 1 + 1 + 1 + 1 + 1 + 2 + 1 + 2 + 2 + 4;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kSmemAlloc = oTmem + 16 + 1024;
};

template <int D>
__global__ void __launch_bounds__(kBThreads, 1)
    bwd_i8_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_dq8, const __grid_constant__ CUtensorMap tm_v,
                  const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dqacc,
                  const I8BwdArgs a) {
  using L = BLayout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* kv_full = bars;
  uint64_t* q_full = kv_full + 1;    // [2] Q̂_i + L'/D stage
  uint64_t* q_empty = q_full + 2;    // [2] commit after dK(i) + one arrival per WG1 warp
  uint64_t* do_full = q_empty + 2;   // [2]: [0] full, [1] empty (dO_i, 16-bit)
  uint64_t* dq8_full = do_full + 2;  // [2]: [0] full, [1] empty (dÔ_i)
  uint64_t* s_full = dq8_full + 2;   // [2] S(t) in buffer t % 2
  uint64_t* dp_full = s_full + 2;
  uint64_t* p_full = dp_full + 1;     // WG1 -> MMA: P̂ in smem
  uint64_t* sp_empty = p_full + 1;    // MMA -> WG1: dV MMA done reading P̂
  uint64_t* ds_full = sp_empty + 1;   // WG1 -> MMA: dŜ in smem, S/P and dP/dS columns read
  uint64_t* sds_empty = ds_full + 1;  // MMA -> WG1: dK / dQ MMAs done reading dŜ
  uint64_t* dvp_full = sds_empty + 1;
  uint64_t* dvp_empty = dvp_full + 1;  // [2] WG2 -> MMA: dV partial of tile t read from R2(t)
  uint64_t* kq_full = dvp_empty + 2;
  uint64_t* y_empty = kq_full + 1;    // [2] WG3 -> MMA: dK partial of tile t read from R1(t)
  uint64_t* sb_empty = y_empty + 2;   // [2] WG3 -> MMA: dQ partial read from S buffer t % 2
  uint64_t* x_full = sb_empty + 2;    // [4] WG1 -> WG2 / WG3: s_P, s_dS, rowsum(dS) of tile t in slot t % 4
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);
  float* s_km = reinterpret_cast<float*>(smem + L::oKm);
  float* s_red = reinterpret_cast<float*>(smem + L::oRed);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_t = a.Np >> 7;
  const int bh = blockIdx.x / n_t;
  const int j = (int)(blockIdx.x % n_t);
  const int i0 = a.causal ? j : 0;
  const int nt = n_t - i0;  // query tiles of this KV tile (>= 1)
  const int b = bh / a.H, h = bh % a.H;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 5);
      mbar_init(&s_full[s], 1);
      mbar_init(&sb_empty[s], 8);  // WG2 and WG3 warps (each flushes half of the dQ partial)
    }
    mbar_init(&do_full[0], 1);
    mbar_init(&do_full[1], 1);
    mbar_init(&dq8_full[0], 1);
    mbar_init(&dq8_full[1], 1);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 4);
    mbar_init(sp_empty, 1);
    mbar_init(ds_full, 4);
    mbar_init(sds_empty, 1);
    mbar_init(dvp_full, 1);
    mbar_init(&dvp_empty[0], 4);
    mbar_init(&dvp_empty[1], 4);
    mbar_init(kq_full, 1);
    mbar_init(&y_empty[0], 4);
    mbar_init(&y_empty[1], 4);
    for (int s = 0; s < 4; ++s) mbar_init(&x_full[s], 128);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_dq8);
    prefetch_tmap(&tm_v);
    prefetch_tmap(&tm_do);
    prefetch_tmap(&tm_dqacc);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  float* s_sq = reinterpret_cast<float*>(smem + L::oScl);
  float* s_sdo = s_sq + 1024;
  if (threadIdx.x < D) s_km[threadIdx.x] = a.km[(int64_t)bh * D + threadIdx.x];
  for (int x = threadIdx.x; x < n_t; x += kBThreads) {
    s_sq[x] = a.sq[(int64_t)bh * n_t + x];
    s_sdo[x] = a.sdo[(int64_t)bh * n_t + x];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int wg = warp >> 2;
  const float sk_j = a.sk[(int64_t)bh * n_t + j];

  if (wg == 0) {
    setmaxnreg_dec<kBRegWG0>();
    if (warp == 0) {
      // ------------------------------------------------------------------------ TMA producer
      if (elect_one()) {
        mbar_arrive_expect_tx(kv_full, L::kI8Tile + L::k16Tile);
        tma_load_2d(smem + L::oK, &tm_k, kv_full, 0, bh * a.Np + j * 128);
#pragma unroll
        for (int x = 0; x < D / 64; ++x)
          tma_load_4d(smem + L::oV + x * 16384, &tm_v, kv_full, 64 * x, j * 128, h, b);
        for (int t = 0; t < nt; ++t) {
          const int i = i0 + t, st = t & 1;
          SAGE3_TRACE_EV(3, t, 0);
          mbar_wait(&q_empty[st], ((uint32_t)(t >> 1) & 1u) ^ 1u);
          SAGE3_TRACE_EV(3, t, 1);
          mbar_arrive_expect_tx(&q_full[st], L::kI8Tile + 1024);
          tma_load_2d(smem + L::oQ + st * L::kI8Tile, &tm_q, &q_full[st], 0, bh * a.Np + i * 128);
          bulk_load(smem + L::oLD + st * 1024, a.lp + (int64_t)bh * a.Np + i * 128, 512, &q_full[st]);
          bulk_load(smem + L::oLD + st * 1024 + 512, a.dd + (int64_t)bh * a.Np + i * 128, 512, &q_full[st]);
          mbar_wait(&do_full[1], ((uint32_t)t & 1u) ^ 1u);
          SAGE3_TRACE_EV(3, t, 2);
          mbar_arrive_expect_tx(&do_full[0], L::k16Tile);
#pragma unroll
          for (int x = 0; x < D / 64; ++x)
            tma_load_4d(smem + L::oDO + x * 16384, &tm_do, &do_full[0], 64 * x, i * 128, h, b);
          mbar_wait(&dq8_full[1], ((uint32_t)t & 1u) ^ 1u);
          SAGE3_TRACE_EV(3, t, 3);
          mbar_arrive_expect_tx(&dq8_full[0], L::kI8Tile);
          tma_load_2d(smem + L::oDOq, &tm_dq8, &dq8_full[0], 0, bh * a.Np + i * 128);
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ------------------------------------------------------------------------ MMA issuer
      if (elect_one()) {
        constexpr uint32_t kI8Layout = D == 128 ? kLayoutSw128 : kLayoutSw64;
        constexpr uint32_t kI8Sbo = 8 * D;          // 8 rows of D bytes
        constexpr uint32_t kI8KStep = 32 * D;        // 32 rows (one kind::i8 K-step) of an MN-major operand
        constexpr uint32_t id_s = idesc_i8(128, 128, false, false);
        constexpr uint32_t id_dp = idesc_f16(128, 128, 0);
        constexpr uint32_t id_dvk = idesc_i8(128, D, true, true);
        constexpr uint32_t id_dq = idesc_i8(128, D, false, true);
        const uint32_t id_dp_rt = id_dp | ((uint32_t)a.in_bf16 << 7) | ((uint32_t)a.in_bf16 << 10);
        const uint32_t sK = smem_u32(smem + L::oK), sV = smem_u32(smem + L::oV);
        const uint32_t sDO = smem_u32(smem + L::oDO), sDOq = smem_u32(smem + L::oDOq);
        const uint32_t sP = smem_u32(smem + L::oP), sDS = smem_u32(smem + L::oDS);
        mbar_wait(kv_full, 0);
        auto issue_s = [&](int t) {
          const int st = t & 1;
          const uint32_t sQ = smem_u32(smem + L::oQ + st * L::kI8Tile);
          mbar_wait(&q_full[st], (uint32_t)(t >> 1) & 1u);
          mbar_wait(&sb_empty[st], ((uint32_t)(t >> 1) & 1u) ^ 1u);
          tc_fence_after();
#pragma unroll 1
          for (int ks = 0; ks < D / 32; ++ks)
            mma_i8b(tbase + (st ? kColS1 : kColS0), make_smem_desc(sQ + 32 * ks, 16, kI8Sbo, kI8Layout),
                    make_smem_desc(sK + 32 * ks, 16, kI8Sbo, kI8Layout), id_s, ks > 0);
          mma_commit(&s_full[st]);
        };
        auto issue_dp = [&](int t) {  // into R1(t) = R2(t-1): after WG2 has read the dV partial of t-1
          mbar_wait(&do_full[0], (uint32_t)t & 1u);
          if (t > 0) mbar_wait(&dvp_empty[(t - 1) & 1], (uint32_t)((t - 1) >> 1) & 1u);
          tc_fence_after();
#pragma unroll 1
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
            mma_f16b(tbase + r1col(t), make_smem_desc(sDO + off, 16, 1024, kLayoutSw128),
                     make_smem_desc(sV + off, 16, 1024, kLayoutSw128), id_dp_rt, ks > 0);
          }
          mma_commit(&do_full[1]);
          mma_commit(dp_full);
        };
        auto issue_dv = [&](int t) {  // into R2(t) = R1(t-1): after WG3 has read the dK partial of t-1
          mbar_wait(p_full, (uint32_t)t & 1u);
          if (t > 0) mbar_wait(&y_empty[(t - 1) & 1], (uint32_t)((t - 1) >> 1) & 1u);
          mbar_wait(&dq8_full[0], (uint32_t)t & 1u);
          tc_fence_after();
#pragma unroll 1
          for (int ks = 0; ks < 4; ++ks)
            mma_i8b(tbase + r2col(t), make_smem_desc(sP + 4096 * ks, 8192, 1024, kLayoutSw128),
                    make_smem_desc(sDOq + kI8KStep * ks, 8192, kI8Sbo, kI8Layout), id_dvk, ks > 0);
          mma_commit(&dq8_full[1]);
          mma_commit(sp_empty);
          mma_commit(dvp_full);
        };
        auto issue_dkq = [&](int t) {
          const int st = t & 1;
          const uint32_t sQ = smem_u32(smem + L::oQ + st * L::kI8Tile);
          mbar_wait(ds_full, (uint32_t)t & 1u);
          tc_fence_after();
#pragma unroll 1
          for (int ks = 0; ks < 4; ++ks)  // dK partial: A = dŜᵀ (keys x queries, MN-major), B = Q̂_i (MN-major)
            mma_i8b(tbase + r1col(t), make_smem_desc(sDS + 4096 * ks, 8192, 1024, kLayoutSw128),
                    make_smem_desc(sQ + kI8KStep * ks, 8192, kI8Sbo, kI8Layout), id_dvk, ks > 0);
#pragma unroll 1
          for (int ks = 0; ks < 4; ++ks)  // dQ partial: A = dŜ (queries x keys, K-major), B = K̂_j (MN-major)
            mma_i8b(tbase + (st ? kColS1 : kColS0), make_smem_desc(sDS + 32 * ks, 16, 1024, kLayoutSw128),
                    make_smem_desc(sK + kI8KStep * ks, 8192, kI8Sbo, kI8Layout), id_dq, ks > 0);
          mma_commit(sds_empty);
          mma_commit(&q_empty[st]);
          mma_commit(kq_full);
        };
        issue_s(0);
        issue_dp(0);
        for (int t = 0; t < nt; ++t) {
          SAGE3_TRACE_EV(2, t, 0);
          if (t + 1 < nt) issue_s(t + 1);
          SAGE3_TRACE_EV(2, t, 1);
          issue_dv(t);
          SAGE3_TRACE_EV(2, t, 2);
          issue_dkq(t);
          SAGE3_TRACE_EV(2, t, 3);
          if (t + 1 < nt) issue_dp(t + 1);
          SAGE3_TRACE_EV(2, t, 4);
        }
      }
      __syncwarp();
    }
  } else if (wg == 1) {
    // ---------------------------------------------------------------------------- element-wise (query rows)
    setmaxnreg_inc<kBRegElem>();
    const int r = threadIdx.x - 128;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const float cl2 = a.scale * kLog2e;
    const uint32_t sP_row = smem_u32(smem + L::oP) + r * 128, sDS_row = smem_u32(smem + L::oDS) + r * 128;
    float* red_a = s_red;
    float* red_b = s_red + 4;
    const f2 mg2 = make_float2(kMagicFB, kMagicFB);
    // One (i, j) tile.  Only the causal diagonal and the padded last KV tile need key masking: a separate
    // instantiation keeps the selects out of the common path.
    auto tile = [&](const int t, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const int i = i0 + t, st = t & 1;
      const int q_row = i * 128 + r;
      const uint32_t tS = lane_base + (st ? kColS1 : kColS0), tY = lane_base + r1col(t);
      SAGE3_TRACE_EV(1, t, 0);
      mbar_wait(&q_full[st], (uint32_t)(t >> 1) & 1u);
      const uint32_t ld = smem_u32(smem + L::oLD + st * 1024) + 4 * r;
      const float lp = lds_f32(ld), dr = lds_f32(ld + 512);
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_empty[st]);
      const float c = cl2 * s_sq[i] * sk_j;  // S·scale·log2 e = S_int·c
      const f2 c2 = make_float2(c, c), nl2 = make_float2(-lp, -lp);
      const int lim = a.causal ? min(a.N - 1, q_row) - j * 128 : a.N - 1 - j * 128;  // last visible key
      // ---- phase A: the tile max of P = 2^(S·c − L') is 2^(rowmax(S_int)·c − L') maximised over the rows
      //      (c > 0, exp monotone): an integer row max (3-input VIMNMX) and one exp per row; P itself is
      //      computed once, in phase B, by the same instructions as this row maximum.
      mbar_wait(&s_full[st], (uint32_t)(t >> 1) & 1u);
      SAGE3_TRACE_EV(1, t, 1);
      tc_fence_after();
      int smax = INT_MIN;
      {
        uint32_t va[32], vb[32];
        auto rmax = [&](int ch, const uint32_t(&v)[32]) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            int x0 = (int)v[e], x1 = (int)v[e + 1];
            if constexpr (masked) {
              x0 = (32 * ch + e > lim) ? INT_MIN : x0;
              x1 = (32 * ch + e + 1 > lim) ? INT_MIN : x1;
            }
            smax = __vimax3_s32(smax, x0, x1);
          }
        };
#pragma unroll 1  // rolled loops keep the per-role code small (the four roles share each SM's i-cache)
        for (int ch = 0; ch < 4; ch += 2) {
          tmem_ld_32x32b_x32(tS + 32 * ch, va);
          tmem_ld_32x32b_x32(tS + 32 * ch + 32, vb);
          tmem_ld_wait_regs(va);
          tmem_ld_wait_regs(vb);
          rmax(ch, va);
          rmax(ch + 1, vb);
        }
      }
      float pmax;
      {
        const f2 x = ffma2(i2f2b((uint32_t)smax, (uint32_t)smax), c2, nl2);
        pmax = smax == INT_MIN ? 0.0f : ex2(x.x);
      }
      // tile amax (ψ(P), Alg3 L6): warp shuffle, then across the four warps
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
      if (lane == 0) red_a[warp & 3] = pmax;
      named_bar(1, 128);
      const float amax_p = fmax3(fmaxf(red_a[0], red_a[1]), red_a[2], red_a[3]);
      const float s_p = __fmul_rn(amax_p, kOne127B);
      const float rp = s_p != 0.0f ? __frcp_rn(s_p) : 0.0f;
      SAGE3_TRACE_EV(1, t, 2);
      // ---- phase B: P̂ = RNE(P·(1/s_P)) -> smem; dS = P∘(dP − D) written over dP; rowsum(dS); tile max |dS|
      mbar_wait(dp_full, (uint32_t)t & 1u);
      mbar_wait(sp_empty, ((uint32_t)t & 1u) ^ 1u);
      SAGE3_TRACE_EV(1, t, 3);
      tc_fence_after();
      const f2 rp2 = make_float2(rp, rp), nd2 = make_float2(-dr, -dr);
      float dsmax = 0.0f, rs = 0.0f;
      auto bchunk = [&](int cc, const uint32_t(&vs)[16], uint32_t(&vd)[16]) {  // keys [16cc, 16cc+16)
        uint32_t w[4];
        f2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          f2 pp[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int e = 4 * q + 2 * u;
            f2 x = ffma2(i2f2b(vs[e], vs[e + 1]), c2, nl2);  // Alg3 L5: P = exp(scale·S·s_Q·s_K − L)
            if constexpr (masked) {
              x.x = (16 * cc + e > lim) ? -INFINITY : x.x;
              x.y = (16 * cc + e + 1 > lim) ? -INFINITY : x.y;
            }
            const f2 p = make_float2(ex2(x.x), ex2(x.y));
            pp[u] = fadd2(fmul2(p, rp2), mg2);
            const f2 ds = fmul2(p, fadd2(make_float2(__uint_as_float(vd[e]), __uint_as_float(vd[e + 1])), nd2));
            acc = fadd2(acc, ds);
            dsmax = fmax3(dsmax, fabsf(ds.x), fabsf(ds.y));
            vd[e] = __float_as_uint(ds.x);
            vd[e + 1] = __float_as_uint(ds.y);
          }
          w[q] = pack4(pp[0], pp[1]);
        }
        rs += acc.x + acc.y;
        // 16-byte chunk cc of row r, SWIZZLE_128B (chunk ^= r & 7)
        sts_v4(sP_row + ((cc ^ (r & 7)) * 16), w[0], w[1], w[2], w[3]);
        tmem_st_32x32b_x16(tY + 16 * cc, vd);
      };
      {
        uint32_t pa[16], da[16], pb[16], db[16];
        tmem_ld_32x32b_x16(tS, pa);
        tmem_ld_32x32b_x16(tY, da);
#pragma unroll 1
        for (int cc = 0; cc < 8; cc += 2) {  // the loads of chunk c+1 are in flight while chunk c is computed
          tmem_ld_32x32b_x16(tS + 16 * cc + 16, pb);
          tmem_ld_32x32b_x16(tY + 16 * cc + 16, db);
          tmem_ld_wait_regs(pa);
          tmem_ld_wait_regs(da);
          bchunk(cc, pa, da);
          tmem_ld_wait_regs(pb);  // already complete (waited above); orders the reads of pb, db
          tmem_ld_wait_regs(db);
          if (cc + 2 < 8) {
            tmem_ld_32x32b_x16(tS + 16 * cc + 32, pa);
            tmem_ld_32x32b_x16(tY + 16 * cc + 32, da);
          }
          bchunk(cc + 1, pb, db);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      SAGE3_TRACE_EV(1, t, 4);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dsmax = fmaxf(dsmax, __shfl_xor_sync(0xffffffffu, dsmax, o));
      if (lane == 0) red_b[warp & 3] = dsmax;
      tmem_st_wait();
      named_bar(2, 128);
      const float amax_ds = fmax3(fmaxf(red_b[0], red_b[1]), red_b[2], red_b[3]);
      const float s_ds = __fmul_rn(amax_ds, kOne127B);
      const float rds = s_ds != 0.0f ? __frcp_rn(s_ds) : 0.0f;
      {  // -> WG2 / WG3
        float* x = reinterpret_cast<float*>(smem + L::oX + (t & 3) * 1024);
        if (r == 0) x[0] = s_p, x[1] = s_ds;
        x[128 + r] = rs;
        mbar_arrive(&x_full[t & 3]);
      }
      // ---- phase C: dŜ = RNE(dS·(1/s_dS)) -> smem (two's-complement bytes)
      SAGE3_TRACE_EV(1, t, 5);
      mbar_wait(sds_empty, ((uint32_t)t & 1u) ^ 1u);
      SAGE3_TRACE_EV(1, t, 6);
      const f2 rd2 = make_float2(rds, rds);
      auto dchunk = [&](int ch, const uint32_t(&v)[32]) {
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int e = 4 * q;
          const f2 t0 = fadd2(fmul2(make_float2(__uint_as_float(v[e]), __uint_as_float(v[e + 1])), rd2), mg2);
          const f2 t1 = fadd2(fmul2(make_float2(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3])), rd2), mg2);
          w[q] = pack4(t0, t1);
        }
        sts_v4(sDS_row + (((2 * ch) ^ (r & 7)) * 16), w[0], w[1], w[2], w[3]);
        sts_v4(sDS_row + (((2 * ch + 1) ^ (r & 7)) * 16), w[4], w[5], w[6], w[7]);
      };
      {
        uint32_t va[32], vb[32];
#pragma unroll 1
        for (int ch = 0; ch < 4; ch += 2) {
          tmem_ld_32x32b_x32(tY + 32 * ch, va);
          tmem_ld_32x32b_x32(tY + 32 * ch + 32, vb);
          tmem_ld_wait_regs(va);
          tmem_ld_wait_regs(vb);
          dchunk(ch, va);
          dchunk(ch + 1, vb);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      SAGE3_TRACE_EV(1, t, 7);
    };
    const bool pad_last = j == n_t - 1 && a.N < a.Np;
    for (int t = 0; t < nt; ++t) {
      if ((a.causal && i0 + t == j) || pad_last)
        tile(t, std::true_type{});
      else
        tile(t, std::false_type{});
    }
  } else if (wg == 2) {
    // ---------------------------------------------------------------------------- dV_j accumulation (key rows)
    //                                                                              + dQ partial columns [0, D/2)
    setmaxnreg_inc<kBRegDV>();
    const int r = threadIdx.x - 256;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    uint8_t* stage = smem + L::oDQ + (warp & 3) * (kDQBufs * 2048);
    int nflush = 0;
    f2 acc[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) acc[c] = make_float2(0.f, 0.f);
    for (int t = 0; t < nt; ++t) {
      const int i = i0 + t, st = t & 1;
      mbar_wait(&x_full[t & 3], (uint32_t)(t >> 2) & 1u);
      const uint32_t xs = smem_u32(smem + L::oX + (t & 3) * 1024);
      const float s_p = lds_f32(xs), s_ds = lds_f32(xs + 4), rs = lds_f32(xs + 512 + 4 * r);
      const float w = __fmul_rn(s_p, s_sdo[i]);
      const f2 w2 = make_float2(w, w);
      SAGE3_TRACE_EV(5, t, 0);
      mbar_wait(dvp_full, (uint32_t)t & 1u);
      SAGE3_TRACE_EV(5, t, 1);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < D / 16; ++cc) {
        uint32_t v[16];
        tmem_ld16(lane_base + r2col(t) + 16 * cc, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[8 * cc + e] = ffma2(i2f2b(v[2 * e], v[2 * e + 1]), w2, acc[8 * cc + e]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dvp_empty[t & 1]);
      SAGE3_TRACE_EV(5, t, 2);
      const float wq = __fmul_rn(s_ds, sk_j);
      mbar_wait(kq_full, (uint32_t)t & 1u);
      tc_fence_after();
      flush_dq<D / 32>(&tm_dqacc, lane_base + (st ? kColS1 : kColS0), 0, stage, nflush, s_km, make_float2(wq, wq),
                       make_float2(rs, rs), r, lane, bh * a.Np + i * 128 + (warp & 3) * 32,
                       a.dqacc + ((int64_t)bh * a.Np + i * 128 + r) * D);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sb_empty[st]);
      SAGE3_TRACE_EV(5, t, 3);
    }
    if (lane == 0) bulk_wait<0>();
    const int key = j * 128 + r;
    if (key < a.N) store_row<D>(a.dv, a.dv_sb, a.dv_sh, a.dv_sn, a.g_dtype, b, h, key, acc, 1.0f);
  } else {
    // ---------------------------------------------------------------------------- dK_j accumulation, dQ flush
    setmaxnreg_inc<kBRegDK>();
    const int r = threadIdx.x - 384;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    f2 acc[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) acc[c] = make_float2(0.f, 0.f);
    uint8_t* stage = smem + L::oDQ + (4 + (warp & 3)) * (kDQBufs * 2048);
    int nflush = 0;
    for (int t = 0; t < nt; ++t) {
      const int i = i0 + t, st = t & 1;
      mbar_wait(&x_full[t & 3], (uint32_t)(t >> 2) & 1u);
      const uint32_t xs = smem_u32(smem + L::oX + (t & 3) * 1024);
      const float s_ds = lds_f32(xs + 4), rs = lds_f32(xs + 512 + 4 * r);
      const float wk = __fmul_rn(__fmul_rn(s_ds, s_sq[i]), a.scale);  // dK carries the softmax scale (b7)
      const float wq = __fmul_rn(s_ds, sk_j);
      SAGE3_TRACE_EV(4, t, 0);
      mbar_wait(kq_full, (uint32_t)t & 1u);
      SAGE3_TRACE_EV(4, t, 1);
      tc_fence_after();
      {  // dK partial (TMEM columns kColY..): two 16-column loads in flight
        const f2 w2 = make_float2(wk, wk);
#pragma unroll
        for (int cc = 0; cc < D / 16; cc += 2) {
          uint32_t va[16], vb[16];
          tmem_ld_32x32b_x16(lane_base + r1col(t) + 16 * cc, va);
          tmem_ld_32x32b_x16(lane_base + r1col(t) + 16 * cc + 16, vb);
          tmem_ld_wait_regs(va);
          tmem_ld_wait_regs(vb);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[8 * cc + e] = ffma2(i2f2b(va[2 * e], va[2 * e + 1]), w2, acc[8 * cc + e]);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            acc[8 * cc + 8 + e] = ffma2(i2f2b(vb[2 * e], vb[2 * e + 1]), w2, acc[8 * cc + 8 + e]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&y_empty[t & 1]);
      SAGE3_TRACE_EV(4, t, 2);
      // dQ partial of (i, j): MM(dŜ, K̂_j)·s_dS·s_K + rowsum(dS)·K_m (Alg3 L10), columns [D/2, D)
      flush_dq<D / 32>(&tm_dqacc, lane_base + (st ? kColS1 : kColS0), D / 2, stage, nflush, s_km,
                       make_float2(wq, wq), make_float2(rs, rs), r, lane, bh * a.Np + i * 128 + (warp & 3) * 32,
                       a.dqacc + ((int64_t)bh * a.Np + i * 128 + r) * D);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sb_empty[st]);
      SAGE3_TRACE_EV(4, t, 3);
    }
    if (lane == 0) bulk_wait<0>();
    const int key = j * 128 + r;
    if (key < a.N) store_row<D>(a.dk, a.dk_sb, a.dk_sh, a.dk_sn, a.g_dtype, b, h, key, acc, 1.0f);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ---------------------------------------------------------------------------------------------- prep
// One CTA per (128-row block i, b·h): ψ(dO_i) (codes row-major [BH][Np][D], scale s_dO[BH][Np/128]),
// D = rowsum(dO∘O) (fp32, sequential over each 8-channel group, then a shuffle tree), L' = lse·log2 e.
__device__ __forceinline__ void load8(const void* base, int64_t off, int dt, float (&o)[8]) {
  if (dt == 2) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off);
    const float4 x = p[0], y = p[1];
    o[0] = x.x, o[1] = x.y, o[2] = x.z, o[3] = x.w, o[4] = y.x, o[5] = y.y, o[6] = y.z, o[7] = y.w;
  } else if (dt == 1) {
    const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + off);
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = __bfloat162float(e[k]);
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(base) + off);
    const __half* e = reinterpret_cast<const __half*>(&u);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = __half2float(e[k]);
  }
}

template <int D>
__global__ void __launch_bounds__(256) bwd_prep_kernel(const I8BwdArgs a) {
  constexpr int kVec = D / 8, kIt = 128 * kVec / 256;
  __shared__ float s_red[8];
  const int chunk = blockIdx.x, bh = blockIdx.y, t = threadIdx.x;
  const int b = bh / a.H, h = bh % a.H;
  const int cv = t % kVec;
  const int in_dt = a.in_bf16 ? 1 : 0;
  float x[kIt][8];
  float amax = 0.0f;
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int row = (it * 256 + t) / kVec, n = chunk * 128 + row;
    float dot = 0.0f;
    if (n < a.N) {
      load8(a.dout, b * a.do_sb + h * a.do_sh + (int64_t)n * a.do_sn + cv * 8, in_dt, x[it]);
      float o[8];
      load8(a.o, b * a.o_sb + h * a.o_sh + (int64_t)n * a.o_sn + cv * 8, a.o_dtype, o);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        amax = fmaxf(amax, fabsf(x[it][e]));
        dot = fmaf(x[it][e], o[e], dot);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[it][e] = 0.0f;
    }
#pragma unroll
    for (int o = kVec / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (cv == 0) {
      const int64_t idx = (int64_t)bh * a.Np + n;
      a.dd[idx] = dot;
      a.lp[idx] = n < a.N ? a.lse[(int64_t)bh * a.N + n] * kLog2e : INFINITY;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((t & 31) == 0) s_red[t >> 5] = amax;
  __syncthreads();
  amax = s_red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) amax = fmaxf(amax, s_red[w]);
  const float s = __fmul_rn(amax, kOne127B);
  const float r = s != 0.0f ? __frcp_rn(s) : 0.0f;
  if (t == 0) a.sdo[(int64_t)bh * (a.Np >> 7) + chunk] = s;
  int8_t* dst = a.do8 + ((int64_t)bh * a.Np + chunk * 128) * D;
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int row = (it * 256 + t) / kVec;
    uint32_t w[2];
    int8_t* bytes = reinterpret_cast<int8_t*>(w);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float v = rintf(__fmul_rn(x[it][e], r));
      bytes[e] = (int8_t)(int)fminf(fmaxf(v, -127.0f), 127.0f);
    }
    *reinterpret_cast<uint2*>(dst + row * D + cv * 8) = make_uint2(w[0], w[1]);
  }
}

// dQ = scale · dQ_acc on the real rows, in the gradient dtype (one thread per 4 channels).
template <int D>
__global__ void __launch_bounds__(256) bwd_dq_final_kernel(const I8BwdArgs a) {
  const int64_t total = (int64_t)a.B * a.H * a.N * (D / 4);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int c4 = (int)(g % (D / 4));
    const int64_t rowg = g / (D / 4);
    const int n = (int)(rowg % a.N);
    const int bh = (int)(rowg / a.N), b = bh / a.H, h = bh % a.H;
    const float4 v = *reinterpret_cast<const float4*>(a.dqacc + ((int64_t)bh * a.Np + n) * D + 4 * c4);
    const int64_t off = b * a.dq_sb + h * a.dq_sh + (int64_t)n * a.dq_sn + 4 * c4;
    const float s = a.scale;
    if (a.g_dtype == 2) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.dq) + off) = make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
    } else if (a.g_dtype == 1) {
      __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(a.dq) + off);
      p[0] = __floats2bfloat162_rn(v.x * s, v.y * s);
      p[1] = __floats2bfloat162_rn(v.z * s, v.w * s);
    } else {
      __half2* p = reinterpret_cast<__half2*>(reinterpret_cast<__half*>(a.dq) + off);
      p[0] = __floats2half2_rn(v.x * s, v.y * s);
      p[1] = __floats2half2_rn(v.z * s, v.w * s);
    }
  }
}

// ---------------------------------------------------------------------------------------------- host
bool encode_map(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle swz) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return encode_tiled_cached(enc, m, dt, rank, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// [BH·Np][D] int8 rows, box D x 128, the swizzle of a D-byte row (128 B or 64 B)
bool map_i8(CUtensorMap* m, const void* base, int D, uint64_t rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)D, rows}, strides[1] = {(cuuint64_t)D};
  const cuuint32_t box[2] = {(cuuint32_t)D, 128};
  return encode_map(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box,
                    D == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
}
// [B][H][N][D] 16-bit with element strides, box 64 x 128 x 1 x 1, SWIZZLE_128B (rows >= N read as zeros)
bool map_16(CUtensorMap* m, const void* base, int B, int H, int N, int D, int64_t sb, int64_t sh, int64_t sn) {
  if (H == 1) sh = sn * N;
  if (B == 1) sb = sh * H;
  const cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
  const cuuint64_t strides[3] = {(cuuint64_t)sn * 2, (cuuint64_t)sh * 2, (cuuint64_t)sb * 2};
  const cuuint32_t box[4] = {64, 128, 1, 1};
  return encode_map(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int D>
cudaError_t launch_bwd_d(const I8BwdArgs& a, cudaStream_t stream) {
  using L = BLayout<D>;
  static std::atomic<bool> attr_done[64];  // one-time attribute setup per device (racing callers both set it: idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(bwd_i8_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = a.B * a.H, n_t = a.Np / 128;
  const uint64_t rows = (uint64_t)BH * a.Np;
  CUtensorMap tq, tk, tdq8, tv, tdo, tacc;
  const cuuint64_t adims[2] = {(cuuint64_t)D, rows}, astr[1] = {(cuuint64_t)D * 4};
  const cuuint32_t abox[2] = {16, 32};
  if (!map_i8(&tq, a.q8, D, rows) || !map_i8(&tk, a.k8, D, rows) || !map_i8(&tdq8, a.do8, D, rows) ||
      !map_16(&tv, a.v, a.B, a.H, a.N, D, a.v_sb, a.v_sh, a.v_sn) ||
      !map_16(&tdo, a.dout, a.B, a.H, a.N, D, a.do_sb, a.do_sh, a.do_sn) ||
      !encode_map(&tacc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, a.dqacc, adims, astr, abox, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(a.dqacc, 0, rows * D * sizeof(float), stream);
  if (e != cudaSuccess) return e;
  bwd_prep_kernel<D><<<dim3(n_t, BH), 256, 0, stream>>>(a);
  bwd_i8_kernel<D><<<(unsigned)(BH * n_t), kBThreads, L::kSmemAlloc, stream>>>(tq, tk, tdq8, tv, tdo, tacc, a);
  const int64_t total = (int64_t)BH * a.N * (D / 4);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  bwd_dq_final_kernel<D><<<blocks, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_bwd_i8(const I8BwdArgs& a, cudaStream_t stream) {
  return a.d == 128 ? launch_bwd_d<128>(a, stream) : launch_bwd_d<64>(a, stream);
}

#ifdef SAGE3_TRACE
extern "C" int sage3_debug_trace_copy_bwd(void* host, size_t bytes) {
  if (bytes > sizeof(g_trace)) bytes = sizeof(g_trace);
  return (int)cudaMemcpyFromSymbol(host, g_trace, bytes);
}
#endif

}  // namespace sage3
