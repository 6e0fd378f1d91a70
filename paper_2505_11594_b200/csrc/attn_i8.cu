// attn_i8.cu — SageBwd's 8-bit attention forward (NEXT #3; Algorithm 2) on sm_100a.
//
// Same warp-specialised pipeline as attn.cu (one CTA per 128-query tile, TMA producers, S / PV MMA issuers,
// two softmax warpgroups on alternating KV tiles, a correction warpgroup owning m, l and O in registers),
// with INT8 operands: S = MM(Q̂_i, K̂_j) by tcgen05.mma.kind::i8 (int32 accumulators in TMEM, exact), scaled
// by the per-block s_Q·s_K in the softmax; per-token P (Alg2 L10) in tile-local form
//     P̂_ij = RNE(127 · 2^{sl2 (S − tmax_j)})  (= P̃/s_P with s_P = exp(scale(tmax_j − m_j))/127)
//     O += MM(P̂_ij, V̂_j) · s_P · s_V_j  =  PV_int · 2^{sl2 (tmax_j − m)} / 127 · s_V_j
// l from the unquantized P̃ (reading c9's analog, b5).  int32 -> fp32 conversions are I2F by default
// (SAGE3_I8_I2F=1: exact, |S|, |PV| <= 127·127·128 < 2^24); the magic-number add (exact below 2^22) remains only
// as the SAGE3_I8_I2F=0 alternative.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <type_traits>

#include "attn_common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

#ifndef SAGE3_I8_ROLLED
#define SAGE3_I8_ROLLED 1
#endif
#ifndef SAGE3_POLY_MASK_I8  // exp pairs on the FMA-pipe polynomial in the INT8 softmax; after the I2F change
#define SAGE3_POLY_MASK_I8 0  // all-MUFU is best (A/B at N = 32K: none 1312 TOPS, 1/16 1278, 1/8 1297, 1/4 1268)
#endif
constexpr uint32_t kPolyMaskI8 = SAGE3_POLY_MASK_I8;
#ifndef SAGE3_I8_I2F
#define SAGE3_I8_I2F 1  // int32 -> fp32 by cvt (I2F) instead of the magic-number add
#endif
constexpr int kIKStages = 3, kIVStages = 3, kIPBufs = 3, kIXSlots = 8, kISBufs = 3;
constexpr int kIThreads = 512;
constexpr uint32_t kIRegWG0 = 32, kIRegSoftmax = 144, kIRegCorrection = 192;
constexpr int kIMaxTiles = 1024;  // s_K, s_V of a head staged in smem: N_pad <= 128 K
constexpr float kLog2_127 = 6.988684686772166f;
[[maybe_unused]] constexpr uint32_t kMagicI = 0x4B400000u;  // float 1.5·2^23: int x + kMagicI reinterpreted = 12582912 + x exactly
constexpr float kMagicF = 12582912.0f;

// kind::i8 instruction descriptor: D s32 ([4,6) = 2), A and B signed 8-bit ([7,10) = [10,13) = 1), K-major,
// N >> 3 at [17,23), M >> 4 at [24,29); dense, K = 32 per instruction.
__host__ __device__ constexpr uint32_t make_idesc_i8(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// exact int32 -> fp32 (|x| <= 127·127·128 < 2^24): I2F, which on sm_100 issues outside the MUFU pipe and is
// cheaper than the magic-number form (2 integer adds + FADD2 per pair; measured +7% attention throughput)
__device__ __forceinline__ f2 i2f2(uint32_t a, uint32_t b) {
#if SAGE3_I8_I2F
  return make_float2(__int2float_rn((int)a), __int2float_rn((int)b));
#else
  return fadd2(make_float2(__uint_as_float(a + kMagicI), __uint_as_float(b + kMagicI)), make_float2(-kMagicF, -kMagicF));
#endif
}

template <int D>
struct I8Layout {
  static constexpr int kRow = D;                 // bytes per Q/K row
  static constexpr int kQKBytes = 128 * kRow;    // Q or K tile
  static constexpr int kVBytes = D * 128;        // Vᵀ tile: D channel rows x 128 tokens
  static constexpr int kPBytes = 128 * 128;      // P̂ tile: 128 rows x 128 keys
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + kQKBytes;
  static constexpr int oV = oK + kIKStages * kQKBytes;
  static constexpr int oP = oV + kIVStages * kVBytes;
  static constexpr int oXchg = oP + kIPBufs * kPBytes;              // float [kIXSlots][2][128]
  static constexpr int oScales = oXchg + kIXSlots * 2 * 128 * 4;    // float s_K[kIMaxTiles], s_V[kIMaxTiles]
  static constexpr int oBar = oScales + 2 * kIMaxTiles * 4;
  static constexpr int kNumBars = 1 + 2 * kIKStages + 2 * kIVStages + 3 * kISBufs + 2 * kIPBufs + kIXSlots;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kSmemAlloc = oTmem + 16 + 1024;
};

template <int D>
__global__ void __launch_bounds__(kIThreads, 1)
    attn_i8_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                   const I8AttnArgs a) {
  using L = I8Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  float* s_sk = reinterpret_cast<float*>(smem + L::oScales);
  float* s_sv = s_sk + kIMaxTiles;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + kIKStages;
  uint64_t* v_full = k_empty + kIKStages;
  uint64_t* v_empty = v_full + kIVStages;
  uint64_t* s_full = v_empty + kIVStages;
  uint64_t* pv_full = s_full + kISBufs;
  uint64_t* b_empty = pv_full + kISBufs;
  uint64_t* p_full = b_empty + kISBufs;
  uint64_t* p_empty = p_full + kIPBufs;
  uint64_t* x_full = p_empty + kIPBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = a.Np >> 7;
  const int bh = blockIdx.x / n_qt;
  const int qt = n_qt - 1 - (int)(blockIdx.x % n_qt);
  const int nkv = a.causal ? qt + 1 : n_qt;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kIKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kIVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < kISBufs; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&pv_full[b], 1);
      mbar_init(&b_empty[b], 4);
    }
    for (int b = 0; b < kIPBufs; ++b) {
      mbar_init(&p_full[b], 4);
      mbar_init(&p_empty[b], 1);
    }
    for (int s = 0; s < kIXSlots; ++s) mbar_init(&x_full[s], 128);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  for (int i = threadIdx.x; i < n_qt; i += kIThreads) {  // the head's per-block K and V scales
    s_sk[i] = a.sk[(int64_t)bh * n_qt + i];
    s_sv[i] = a.sv[(int64_t)bh * n_qt + i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int wg = warp >> 2;

  if (wg == 0) {
    setmaxnreg_dec<kIRegWG0>();
    if (warp == 0) {  // ------------------------------------------------------------ TMA: Q, K
      if (elect_one()) {
        const int row_q = bh * a.Np + qt * 128;
        mbar_arrive_expect_tx(q_full, L::kQKBytes);
        tma_load_2d(sQ, &tm_q, q_full, 0, row_q);
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kIKStages;
          mbar_wait(&k_empty[st], ((uint32_t)(j / kIKStages) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&k_full[st], L::kQKBytes);
          tma_load_2d(smem + L::oK + st * L::kQKBytes, &tm_k, &k_full[st], 0, bh * a.Np + j * 128);
        }
      }
      __syncwarp();
    } else if (warp == 3) {  // ----------------------------------------------------- TMA: Vᵀ
      if (elect_one()) {
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kIVStages;
          mbar_wait(&v_empty[st], ((uint32_t)(j / kIVStages) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&v_full[st], L::kVBytes);
          tma_load_2d(smem + L::oV + st * L::kVBytes, &tm_v, &v_full[st], j * 128, bh * D);
        }
      }
      __syncwarp();
    } else {  // -------------------------------------------------------------------- MMA issuers
      if (elect_one()) {
        constexpr uint32_t kQKLayout = D == 128 ? kLayoutSw128 : kLayoutSw64;
        constexpr uint32_t idesc_s = make_idesc_i8(128, 128), idesc_pv = make_idesc_i8(128, D);
        if (warp == 1) {
          mbar_wait(q_full, 0);
          for (int j = 0; j < nkv; ++j) {
            const int b = j % kISBufs, st = j % kIKStages;
            mbar_wait(&b_empty[b], ((uint32_t)(j / kISBufs) & 1u) ^ 1u);
            mbar_wait(&k_full[st], (uint32_t)(j / kIKStages) & 1u);
            tc_fence_after();
            const uint8_t* sK = smem + L::oK + st * L::kQKBytes;
#pragma unroll
            for (int ks = 0; ks < D / 32; ++ks) {
              const uint64_t ad = make_smem_desc(smem_u32(sQ) + 32 * ks, 16, 8 * L::kRow, kQKLayout);
              const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kRow, kQKLayout);
              mma_i8(tbase + 128 * b, ad, bd, idesc_s, ks > 0);
            }
            mma_commit(&k_empty[st]);
            mma_commit(&s_full[b]);
          }
        } else {
          for (int j = 0; j < nkv; ++j) {
            const int b = j % kISBufs, pb = j % kIPBufs, st = j % kIVStages;
            mbar_wait(&p_full[pb], (uint32_t)(j / kIPBufs) & 1u);
            mbar_wait(&v_full[st], (uint32_t)(j / kIVStages) & 1u);
            tc_fence_after();
            const uint8_t* sP = smem + L::oP + pb * L::kPBytes;
            const uint8_t* sV = smem + L::oV + st * L::kVBytes;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 1024, kLayoutSw128);
              const uint64_t bd = make_smem_desc(smem_u32(sV) + 32 * ks, 16, 1024, kLayoutSw128);
              mma_i8(tbase + 128 * b, ad, bd, idesc_pv, ks > 0);
            }
            mma_commit(&v_empty[st]);
            mma_commit(&p_empty[pb]);
            mma_commit(&pv_full[b]);
          }
        }
      }
      __syncwarp();
    }
  } else if (wg >= 2) {
    // ------------------------------------------------------------------ softmax + per-token INT8 P
    setmaxnreg_inc<kIRegSoftmax>();
    const int par = wg - 2;
    const int r = threadIdx.x - 128 * wg;
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const float sq = a.sq[(int64_t)bh * n_qt + qt];
    const float sl2 = a.scale * kLog2e;
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    auto tile = [&](const int j, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const int sb = j % kISBufs, pb = j % kIPBufs;
      const uint32_t s_addr = lane_base + 128 * sb;
      const uint32_t sP = smem_u32(smem + L::oP + pb * L::kPBytes) + r * 128;
      const float cS = sq * s_sk[j];  // S = S_int · s_Q · s_K (Alg2 L8)
      const float c = cS * sl2;
      mbar_wait(&s_full[sb], (uint32_t)(j / kISBufs) & 1u);
      tc_fence_after();
      const int kv0 = j * 128;
      const int lim = a.causal ? min(a.N - 1, q_row) - kv0 : a.N - 1 - kv0;
      // ---- pass 1: the row max of the int32 S (3-input integer max)
      int tm = INT_MIN;
      {
        uint32_t va[32], vb[32], vc[32], vd[32];
        tmem_ld_32x32b_x32(s_addr, va);
        tmem_ld_32x32b_x32(s_addr + 32, vb);
        tmem_ld_32x32b_x32(s_addr + 64, vc);
        tmem_ld_32x32b_x32(s_addr + 96, vd);
        tmem_ld_wait_regs(va);
        tmem_ld_wait_regs(vb);
        tmem_ld_wait_regs(vc);
        tmem_ld_wait_regs(vd);
        auto rmax = [&](int cc, const uint32_t(&v)[32]) {
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            int x0 = (int)v[t], x1 = (int)v[t + 1];
            if constexpr (masked) {
              x0 = (32 * cc + t > lim) ? INT_MIN : x0;
              x1 = (32 * cc + t + 1 > lim) ? INT_MIN : x1;
            }
            tm = __vimax3_s32(tm, x0, x1);
          }
        };
        rmax(0, va);
        rmax(1, vb);
        rmax(2, vc);
        rmax(3, vd);
      }
      const float tmax = (float)tm * cS;          // S units
      const float nb = kLog2_127 - (float)tm * c;  // 127·2^{sl2(S - tmax)} = 2^(S_int·c + nb)
      const f2 c2 = make_float2(c, c), nb2 = make_float2(nb, nb);
      mbar_wait(&p_empty[pb], ((uint32_t)(j / kIPBufs) & 1u) ^ 1u);
      // ---- pass 2: y = 127·2^{sl2(S - tmax)}, P̂ = RNE(y) (magic add), rowsum(y)
      float rowsum = 0.0f;
      auto chunk = [&](int cc, const uint32_t(&v)[32]) {
        f2 y[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          f2 x = ffma2(i2f2(v[2 * i], v[2 * i + 1]), c2, nb2);
          if constexpr (masked) {
            x.x = (32 * cc + 2 * i > lim) ? -INFINITY : x.x;
            x.y = (32 * cc + 2 * i + 1 > lim) ? -INFINITY : x.y;
          }
          y[i] = ((kPolyMaskI8 >> i) & 1u) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        }
        uint32_t w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // 4 keys per word: low bytes of y + 1.5·2^23 are RNE(y)
          const f2 t0 = fadd2(y[2 * q], make_float2(kMagicF, kMagicF));
          const f2 t1 = fadd2(y[2 * q + 1], make_float2(kMagicF, kMagicF));
          const uint32_t lo = __byte_perm(__float_as_uint(t0.x), __float_as_uint(t0.y), 0x0040);
          const uint32_t hi = __byte_perm(__float_as_uint(t1.x), __float_as_uint(t1.y), 0x0040);
          w[q] = __byte_perm(lo, hi, 0x5410);
        }
        const f2 s01 = fadd2(fadd2(fadd2(y[0], y[1]), fadd2(y[2], y[3])), fadd2(fadd2(y[4], y[5]), fadd2(y[6], y[7])));
        const f2 s23 = fadd2(fadd2(fadd2(y[8], y[9]), fadd2(y[10], y[11])), fadd2(fadd2(y[12], y[13]), fadd2(y[14], y[15])));
        const f2 sy = fadd2(s01, s23);
        rowsum += sy.x + sy.y;
        // keys [32cc, 32cc+32) = 16-byte chunks 2cc, 2cc+1 of the row, SWIZZLE_128B (chunk ^= row & 7)
        sts_v4(sP + (((2 * cc) ^ (r & 7)) * 16), w[0], w[1], w[2], w[3]);
        sts_v4(sP + (((2 * cc + 1) ^ (r & 7)) * 16), w[4], w[5], w[6], w[7]);
      };
#if SAGE3_I8_ROLLED
#pragma unroll 1  // rolled: smaller per-role code (the warp roles share each sub-partition's i-cache)
      for (int cc = 0; cc < 4; cc += 2) {
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(s_addr + 32 * cc, va);
        tmem_ld_32x32b_x32(s_addr + 32 * cc + 32, vb);
        tmem_ld_wait_regs(va);
        tmem_ld_wait_regs(vb);
        chunk(cc, va);
        chunk(cc + 1, vb);
      }
#else
      {
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(s_addr, va);
        tmem_ld_32x32b_x32(s_addr + 32, vb);
        tmem_ld_wait_regs(va);
        tmem_ld_wait_regs(vb);
        chunk(0, va);
        tmem_ld_32x32b_x32(s_addr + 64, va);
        chunk(1, vb);
        tmem_ld_32x32b_x32(s_addr + 96, vb);
        tmem_ld_wait_regs(va);
        chunk(2, va);
        tmem_ld_wait_regs(vb);
        chunk(3, vb);
      }
#endif
      const int slot = j % kIXSlots;
      sts_f32(xchg_s + slot * 1024, tmax);
      sts_f32(xchg_s + slot * 1024 + 512, rowsum);
      tc_fence_before();
      fence_proxy_async_smem();
      mbar_arrive(&x_full[slot]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
    };
    const int last = nkv - 1;
    const bool last_masked = last * 128 + 128 > a.N || a.causal;
    for (int j = par; j < last; j += 2) tile(j, std::false_type{});
    if ((last & 1) == par) {
      if (last_masked)
        tile(last, std::true_type{});
      else
        tile(last, std::false_type{});
    }
  } else {
    // ------------------------------------------------------------------ correction + epilogue (as attn.cu)
    // tile j enters with weight w_j = 2^{sl2 (tmax_j − mref)} / 127 · s_V_j (= s_P · s_V relative to mref)
    setmaxnreg_inc<kIRegCorrection>();
    const int r = threadIdx.x - 128;
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    const float sl2 = a.scale * kLog2e;
    float mref = -INFINITY, l = 0.0f;
    f2 o[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = make_float2(0.f, 0.f);
    for (int j = 0; j < nkv; ++j) {
      const int slot = j % kIXSlots, b = j % kISBufs;
      mbar_wait(&x_full[slot], (uint32_t)(j / kIXSlots) & 1u);
      const float tmax = lds_f32(xchg_s + slot * 1024);
      const float rs = lds_f32(xchg_s + slot * 1024 + 512);
      const bool need = (tmax - mref) * sl2 > 8.0f;
      if (__any_sync(0xffffffffu, need)) {
        const float mnew = need ? tmax : mref;
        const float sc = ex2((mref - mnew) * sl2);
        const f2 sc2 = make_float2(sc, sc);
        l *= sc;
#pragma unroll
        for (int c = 0; c < D / 2; ++c) o[c] = fmul2(o[c], sc2);
        mref = mnew;
      }
      const float e = ex2((tmax - mref) * sl2);       // s_P·127 relative to mref
      l = fmaf(e * (1.0f / 127.0f), rs, l);           // l += s_P · Σ y  (= Σ P̃ relative to mref)
      const float w = e * (1.0f / 127.0f) * s_sv[j];  // s_P · s_V
      const f2 ww = make_float2(w, w);
      mbar_wait(&pv_full[b], (uint32_t)(j / kISBufs) & 1u);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 16; ++c) {
        uint32_t v[16];
        tmem_ld16(lane_base + 128 * b + 16 * c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[8 * c + i] = ffma2(i2f2(v[2 * i], v[2 * i + 1]), ww, o[8 * c + i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&b_empty[b]);
    }
    if (a.lse != nullptr && q_row < a.N) a.lse[(int64_t)bh * a.N + q_row] = mref * a.scale + logf(l);
    const float inv_l = 1.0f / l;
    const f2 il{inv_l, inv_l};
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = fmul2(o[c], il);
    uint8_t* stage = smem + L::oK;  // coalesced store through smem + TMA (as attn.cu)
    stage_o_row<D>(stage, r, a.o_dtype, o);
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 128) store_o_tile<D>(&tm_o, stage, a.o_dtype, qt * 128, bh % a.H, bh / a.H);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// 2-D uint8 tensor map with the given swizzle (128 / 64 B rows)
bool make_map_i8(CUtensorMap* m, const void* base, uint64_t row_bytes, uint64_t rows, uint32_t box_bytes,
                 uint32_t box_rows) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle swz = box_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  return encode_tiled_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
cudaError_t launch_i8_d(const I8AttnArgs& a, cudaStream_t stream) {
  using L = I8Layout<D>;
  static std::atomic<bool> attr_done[64];  // one-time attribute setup per device (racing callers both set it: idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_i8_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = a.B * a.H;
  CUtensorMap tq, tk, tv, to;
  if (!make_map_i8(&tq, a.q8, D, (uint64_t)BH * a.Np, D, 128) || !make_map_i8(&tk, a.k8, D, (uint64_t)BH * a.Np, D, 128) ||
      !make_map_i8(&tv, a.vt8, (uint64_t)a.Np, (uint64_t)BH * D, 128, D) ||
      !make_map_o(&to, a.o, a.o_dtype, a.B, a.H, a.N, D, a.o_sb, a.o_sh, a.o_sn))
    return cudaErrorInvalidValue;
  const int64_t units = (int64_t)BH * (a.Np / 128);
  attn_i8_kernel<D><<<(unsigned)units, kIThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_i8(const I8AttnArgs& a, cudaStream_t stream) {
  return a.d == 128 ? launch_i8_d<128>(a, stream) : launch_i8_d<64>(a, stream);
}

}  // namespace sage3
