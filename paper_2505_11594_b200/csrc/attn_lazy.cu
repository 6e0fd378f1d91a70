// attn_lazy.cu — the SURVEY §8(f) NEXT #2 throughput variant of the FP4 attention forward (p_quant =
// SAGE3_P_TWO_LEVEL_LAZY; reading n1; oracle PMODE_LAZY).  NOT the paper's Alg1 L10: the first-level
// P scale is a per-row reference r that moves only when a tile's max exceeds it by more than 2^8 in weight,
//     P̃2_j = 10.5 · 2^{sl2 (S − r_j)}   (≤ 2688 = 448·6 by construction),  (s_P2, P̂2) = φ(P̃2) per 16 keys,
// so every tile of a reference epoch contributes FP4MM(P̂2, s_P2, V̂, s_V) with the SAME weight and the tensor
// core accumulates O across tiles in TMEM.  What that buys over attn.cu (same roles, same operand pipeline):
//   * no per-tile O update: the correction warpgroup only rescales O in TMEM when a row's reference moves
//     (rare after the first tiles) and runs the epilogue — its registers go to the softmax warpgroups;
//   * with 208 registers a softmax thread keeps its whole S row (128 fp32) from pass 1 to pass 2, so the S
//     buffer is released right after the four TMEM loads and S_{j+2} is computed while pass 2 of S_j runs;
//     two S buffers suffice (TMEM: S 2 x 128 columns, O d columns, scale factors 32).
// The price is a chain between the softmax warpgroups (tile j needs r_{j-1}, published right after pass 1)
// and E4M3 range for tiles far below the reference (their weight is < 2^-8 of the row's).
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

constexpr int kLKStages = 5, kLVStages = 4;
constexpr int kLPBufs = 4;   // P̂2 tiles in smem (tile j -> j % 4)
constexpr int kLXSlots = 8;  // softmax -> softmax / correction exchange slots (tile j -> j % 8)
constexpr int kLThreads = 512;
#ifndef SAGE3_LAZY_SPLIT
#define SAGE3_LAZY_SPLIT 1
#endif
// kSplit (NVFP4): the correction warpgroup, idle in this kernel between rescales, also runs pass 2 of the last
// 32-key chunk of every tile (a third warp per sub-partition sharing the MUFU / FMA work); the softmax
// warpgroups do chunks 0-2.  Registers: WG0 32, softmax 192, correction 96 (split) or 208 / 64.
template <bool kMX>
struct LazyCfg {
  static constexpr bool kSplit = SAGE3_LAZY_SPLIT && !kMX;
  static constexpr uint32_t kRegWG0 = 32, kRegSoftmax = kSplit ? 192 : 208, kRegCorrection = kSplit ? 96 : 64;
  static_assert(kRegWG0 + 2 * kRegSoftmax + kRegCorrection <= 512, "register budget");
  static constexpr uint32_t kSArrivals = kSplit ? 8 : 4;  // s_empty / p_full arrivals (warps)
};

// One 32-key chunk of pass 2: y = P̃2/s = 2^(S·sl2 + nb − log2 s) on MUFU or the FMA-pipe polynomial.
__device__ __forceinline__ void chunk_exps(const uint32_t (&vv)[32], f2 sl2x2, float nA, float nB, f2 (&y)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float nbh = i < 8 ? nA : nB;
    const f2 x = ffma2(make_float2(__uint_as_float(vv[2 * i]), __uint_as_float(vv[2 * i + 1])), sl2x2,
                       make_float2(nbh, nbh));
    y[i] = ((kPolyMask >> i) & 1u) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
  }
}
// ... and its E2M1 codes (16 bytes, chunk c of row r in the SWIZZLE_64B P̂2 tile at sP_row) and rowsum share
__device__ __forceinline__ float chunk_finish(const f2 (&y)[16], float sA, float sB, uint32_t sP_row, int c, int r,
                                              float rowsum) {
  uint32_t w[4];
#pragma unroll
  for (int hb = 0; hb < 2; ++hb) {
    const f2* yy = y + 8 * hb;
    const f2 s01 = fadd2(fadd2(yy[0], yy[1]), fadd2(yy[2], yy[3]));
    const f2 s23 = fadd2(fadd2(yy[4], yy[5]), fadd2(yy[6], yy[7]));
    const f2 sy = fadd2(s01, s23);
    rowsum = fmaf(hb ? sB : sA, sy.x + sy.y, rowsum);
    w[2 * hb] = cvt_e2m1x8(yy[0].x, yy[0].y, yy[1].x, yy[1].y, yy[2].x, yy[2].y, yy[3].x, yy[3].y);
    w[2 * hb + 1] = cvt_e2m1x8(yy[4].x, yy[4].y, yy[5].x, yy[5].y, yy[6].x, yy[6].y, yy[7].x, yy[7].y);
  }
  sts_v4(sP_row + ((c ^ ((r >> 1) & 3)) * 16), w[0], w[1], w[2], w[3]);
  return rowsum;
}
constexpr float kLazyTau = 8.0f;                  // reference moves when sl2·(tmax − r) > 8 (reading n1)
constexpr float kLog2Top = 3.3923174227787602f;   // log2(10.5) = log2(2688) − 8
constexpr float kLnTop = 2.3513752571634776f;     // ln(10.5)
// TMEM: S_j in columns [128 (j%2), +128); O in [256, 256 + d); scale factors at kColSF* (384..415).
constexpr uint32_t kColO = 256;
#ifndef SAGE3_LAZY_WARP_ARRIVE
#define SAGE3_LAZY_WARP_ARRIVE 0
#endif
// r_full / x_full arrivals: 128 per-thread (each thread orders its own slot write) or 4 per-warp (after
// __syncwarp, one arrival per warp)
constexpr int kLXArrivals = SAGE3_LAZY_WARP_ARRIVE ? 4 : 128;

template <int D, bool kMX>
struct LazyLayout {
  static constexpr int kQKRow = D / 2;
  static constexpr int kQBytes = 128 * kQKRow;
  static constexpr int kKBytes = 128 * kQKRow;
  static constexpr int kKSlot = ((kKBytes + 1023) / 1024) * 1024;
  static constexpr int kVBytes = D * 64;
  static constexpr int kPBytes = 128 * 64;
  static constexpr int kQKSF = kMX ? 512 : (D / 64) * 512;
  static constexpr int kVSF = kMX ? 512 : 1024, kPSF = kVSF;
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + ((kQBytes + 1023) / 1024) * 1024;
  static constexpr int oV = oK + kLKStages * kKSlot;
  static constexpr int oP = oV + kLVStages * kVBytes;
  static constexpr int oQSF = oP + kLPBufs * kPBytes;
  static constexpr int oKSF = oQSF + kQKSF;
  static constexpr int oVSF = oKSF + kLKStages * kQKSF;
  static constexpr int oPSF = oVSF + kLVStages * kVSF;
  static constexpr int oXchg = oPSF + kLPBufs * kPSF;  // float [kLXSlots][2][128]: r_j, rowsum(P̃2_j)
  static constexpr int oBar = oXchg + kLXSlots * 2 * 128 * 4;
  // q_full, k_full/empty, v_full/empty, s_full/empty[2], pv_full[2], p_full/empty, r_full, x_full, o_ready
  static constexpr int kNumBars = 1 + 2 * kLKStages + 2 * kLVStages + 2 * 2 + 2 + 2 * kLPBufs + 3 * kLXSlots;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kBytes = oTmem + 16;
  static constexpr int kSmemAlloc = kBytes + 1024;
};

template <int D, bool kMX>
__global__ void __launch_bounds__(kLThreads, 1)
    attn_lazy_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                     const AttnArgs a) {
  using L = LazyLayout<D, kMX>;
  using C = LazyCfg<kMX>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(1024) float2 s_lut[128];  // (-log2 s, s) per E4M3 scale code, as in attn.cu
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sQSF = smem + L::oQSF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + kLKStages;
  uint64_t* v_full = k_empty + kLKStages;
  uint64_t* v_empty = v_full + kLVStages;
  uint64_t* s_full = v_empty + kLVStages;  // MMA -> softmax: S_j in buffer j%2
  uint64_t* s_empty = s_full + 2;          // softmax -> MMA: S_j loaded into registers, buffer free
  uint64_t* pv_full = s_empty + 2;         // MMA -> correction: PV_j accumulated into O (tile parity j%2)
  uint64_t* p_full = pv_full + 2;          // softmax -> MMA: P̂2_j / s_P2 in smem buffer j%4
  uint64_t* p_empty = p_full + kLPBufs;    // MMA -> softmax: PV_j done with smem buffer j%4
  uint64_t* r_full = p_empty + kLPBufs;    // softmax -> softmax: r_j in xchg slot j%8 (right after pass 1)
  uint64_t* x_full = r_full + kLXSlots;    // softmax -> correction: rowsum(P̃2_j) in slot j%8
  uint64_t* o_ready = x_full + kLXSlots;   // correction -> MMA: O is relative to r_j (rescaled if it moved)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = a.Np >> 7;
  const int64_t unit = a.unit_begin + (int64_t)blockIdx.x;
  const int bh = (int)(unit / n_qt);
  const int qt = n_qt - 1 - (int)(unit % n_qt);
  const int nkv = a.causal ? qt + 1 : n_qt;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kLKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kLVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], C::kSArrivals);  // one arrival per warp that loads S
      mbar_init(&pv_full[b], 1);
    }
    for (int b = 0; b < kLPBufs; ++b) {
      mbar_init(&p_full[b], C::kSArrivals);
      mbar_init(&p_empty[b], 1);
    }
    for (int s = 0; s < kLXSlots; ++s) {
      mbar_init(&r_full[s], kLXArrivals);
      mbar_init(&x_full[s], kLXArrivals);
      mbar_init(&o_ready[s], 4);   // one arrival per correction warp
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x >= 128 && threadIdx.x < 256) {
    const int c = threadIdx.x - 128;
    const float s = e4m3_to_f32((uint32_t)c);
    const bool zero = (s == 0.0f || c == 0x7F);
    s_lut[c] = make_float2(zero ? 10.0f : -log2f(s), zero ? 0x1p-10f : s);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int wg = warp >> 2;

  if (wg == 0) {
    setmaxnreg_dec<C::kRegWG0>();
    if (warp == 0) {  // ------------------------------------------------------------ TMA producer: Q, K
      if (elect_one()) {
        const int row_q = bh * a.Np + qt * 128;
        mbar_arrive_expect_tx(q_full, L::kQBytes + L::kQKSF);
        tma_load_2d(sQ, &tm_q, q_full, 0, row_q);
        bulk_load(sQSF, a.q_sf + (int64_t)(row_q >> 7) * L::kQKSF, L::kQKSF, q_full);
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kLKStages;
          const int row_k = bh * a.Np + j * 128;
          mbar_wait(&k_empty[st], ((uint32_t)(j / kLKStages) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&k_full[st], L::kKBytes + L::kQKSF);
          tma_load_2d(smem + L::oK + st * L::kKSlot, &tm_k, &k_full[st], 0, row_k);
          bulk_load(smem + L::oKSF + st * L::kQKSF, a.k_sf + (int64_t)(row_k >> 7) * L::kQKSF, L::kQKSF,
                    &k_full[st]);
        }
      }
      __syncwarp();
    } else if (warp == 3) {  // ----------------------------------------------------- TMA producer: V
      if (elect_one()) {
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kLVStages;
          mbar_wait(&v_empty[st], ((uint32_t)(j / kLVStages) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&v_full[st], L::kVBytes + L::kVSF);
          tma_load_2d(smem + L::oV + st * L::kVBytes, &tm_v, &v_full[st], j * 64, bh * D);
          bulk_load(smem + L::oVSF + st * L::kVSF, a.v_sf + ((int64_t)bh * n_qt + j) * L::kVSF, L::kVSF,
                    &v_full[st]);
        }
      }
      __syncwarp();
    } else {  // ------------------------------------------------ MMA issuers: warp 1 S, warp 2 PV
      if (elect_one()) {
        constexpr uint32_t kQKLayout = D == 128 ? kLayoutSw64 : kLayoutSw32;
        constexpr int kQKAtoms = L::kQKSF / 512, kPVAtoms = L::kPSF / 512;
        auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t n, int ks, uint32_t sfa, uint32_t sfb,
                       uint32_t acc) {
          if constexpr (kMX)
            mma_mxf4(d, ad, bd, make_idesc_mxf4(128, n, ks), sfa, sfb, acc);
          else
            mma_nvf4(d, ad, bd, make_idesc_nvf4(128, n), sfa + 4 * ks, sfb + 4 * ks, acc);
        };
        if (warp == 1) {
          mbar_wait(q_full, 0);
          tc_fence_after();
#pragma unroll
          for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kColSFQ + 4 * at, sf_desc(sQSF + 512 * at));
          for (int j = 0; j < nkv; ++j) {
            const int b = j & 1, st = j % kLKStages;
            SAGE3_TRACE_EV(5, j, 0);
            mbar_wait(&s_empty[b], ((uint32_t)(j >> 1) & 1u) ^ 1u);  // softmax loaded S_{j-2}
            SAGE3_TRACE_EV(5, j, 1);
            mbar_wait(&k_full[st], (uint32_t)(j / kLKStages) & 1u);
            SAGE3_TRACE_EV(5, j, 2);
            tc_fence_after();
            const uint8_t* sK = smem + L::oK + st * L::kKSlot;
            const uint8_t* sKSF = smem + L::oKSF + st * L::kQKSF;
#pragma unroll
            for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kColSFK + 4 * at, sf_desc(sKSF + 512 * at));
#pragma unroll
            for (int ks = 0; ks < D / 64; ++ks) {
              const uint64_t ad = make_smem_desc(smem_u32(sQ) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
              const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
              mma(tbase + 128 * b, ad, bd, 128, ks, tbase + kColSFQ, tbase + kColSFK, ks > 0);
            }
            mma_commit(&k_empty[st]);
            mma_commit(&s_full[b]);
            SAGE3_TRACE_EV(5, j, 3);
          }
        } else {
          for (int j = 0; j < nkv; ++j) {
            const int pb = j % kLPBufs, st = j % kLVStages, slot = j % kLXSlots;
            SAGE3_TRACE_EV(6, j, 0);
            mbar_wait(&p_full[pb], (uint32_t)(j / kLPBufs) & 1u);
            SAGE3_TRACE_EV(6, j, 1);
            mbar_wait(&v_full[st], (uint32_t)(j / kLVStages) & 1u);
            SAGE3_TRACE_EV(6, j, 2);
            mbar_wait(&o_ready[slot], (uint32_t)(j / kLXSlots) & 1u);  // O rescaled to r_j if it moved
            SAGE3_TRACE_EV(6, j, 3);
            tc_fence_after();
            const uint8_t* sP = smem + L::oP + pb * L::kPBytes;
            const uint8_t* sV = smem + L::oV + st * L::kVBytes;
            const uint8_t* sPSF = smem + L::oPSF + pb * L::kPSF;
            const uint8_t* sVSF = smem + L::oVSF + st * L::kVSF;
#pragma unroll
            for (int at = 0; at < kPVAtoms; ++at) {
              tmem_cp_32x128b_x4(tbase + kColSFP + 4 * at, sf_desc(sPSF + 512 * at));
              tmem_cp_32x128b_x4(tbase + kColSFV + 4 * at, sf_desc(sVSF + 512 * at));
            }
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
              const uint64_t bd = make_smem_desc(smem_u32(sV) + 32 * ks, 16, 512, kLayoutSw64);
              mma(tbase + kColO, ad, bd, D, ks, tbase + kColSFP, tbase + kColSFV, (j > 0 || ks > 0) ? 1u : 0u);
            }
            mma_commit(&v_empty[st]);
            mma_commit(&p_empty[pb]);
            mma_commit(&pv_full[j & 1]);
            SAGE3_TRACE_EV(6, j, 4);
          }
        }
      }
      __syncwarp();
    }
  } else if (wg >= 2) {
    // ------------------------------------------------------------------ softmax + two-level P (lazy r)
    setmaxnreg_inc<C::kRegSoftmax>();
    const int par = wg - 2;
    const int r = threadIdx.x - 128 * wg;
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    const f2 sl2x2 = make_float2(sl2, sl2);
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    auto tile = [&](const int j, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const int sb = j & 1, pb = j % kLPBufs, slot = j % kLXSlots;
      const uint32_t s_addr = lane_base + 128 * sb;
      const uint32_t sP = smem_u32(smem + L::oP + pb * L::kPBytes) + r * 64;
      const uint32_t sPSF = smem_u32(smem + L::oPSF + pb * L::kPSF) + (r & 31) * 16 + (r >> 5) * 4;
      SAGE3_TRACE_EV(1 + par, j, 0);
      mbar_wait(&s_full[sb], (uint32_t)(j >> 1) & 1u);
      SAGE3_TRACE_EV(1 + par, j, 1);
      tc_fence_after();
      // the whole S row into registers; the buffer is free for S_{j+2} as soon as the loads completed
      uint32_t v[4][32];
      tmem_ld_32x32b_x32(s_addr, v[0]);
      tmem_ld_32x32b_x32(s_addr + 32, v[1]);
      tmem_ld_32x32b_x32(s_addr + 64, v[2]);
      tmem_ld_32x32b_x32(s_addr + 96, v[3]);
      tmem_ld_wait_regs(v[0]);
      tmem_ld_wait_regs(v[1]);
      tmem_ld_wait_regs(v[2]);
      tmem_ld_wait_regs(v[3]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      // ---- pass 1 (registers): masking, 16-key block maxima
      const int kv0 = j * 128;
      const int lim = a.causal ? min(a.N - 1, q_row) - kv0 : a.N - 1 - kv0;
      float bmax[8];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float* f = reinterpret_cast<float*>(v[c]);
        if constexpr (masked) {
#pragma unroll
          for (int t = 0; t < 32; ++t) f[t] = (32 * c + t > lim) ? -INFINITY : f[t];
        }
        bmax[2 * c] = max16(f);
        bmax[2 * c + 1] = max16(f + 16);
      }
      const float tmax = fmax3(fmax3(bmax[0], bmax[1], bmax[2]), fmax3(bmax[3], bmax[4], bmax[5]),
                               fmaxf(bmax[6], bmax[7]));
      SAGE3_TRACE_EV(1 + par, j, 2);
      // ---- the reference chain: r_j = tmax_j if it exceeds r_{j-1} by more than 2^8 in weight, else r_{j-1}
      float rp = -INFINITY;
      if (j > 0) {
        const int ps = (j - 1) % kLXSlots;
        mbar_wait(&r_full[ps], (uint32_t)((j - 1) / kLXSlots) & 1u);
        rp = lds_f32(xchg_s + ps * 1024);
      }
      const float rj = (rp == -INFINITY || (tmax - rp) * sl2 > kLazyTau) ? tmax : rp;
      sts_f32(xchg_s + slot * 1024, rj);
      if constexpr (kLXArrivals == 128) {
        mbar_arrive(&r_full[slot]);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&r_full[slot]);
      }
      SAGE3_TRACE_EV(1 + par, j, 3);
      const float nb = kLog2Top - rj * sl2;  // P̃2 = 2^(S·sl2 + nb) ≤ 2688
      // ---- block scales of φ(P̃2) from the block maxima (as attn.cu)
      float nbb[8], sdec[8];
      uint32_t scw[2] = {0u, 0u};
      if constexpr (kMX) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float bm = fmaxf(bmax[2 * k], bmax[2 * k + 1]);
          const float s32 = __fmul_rn(ex2(fmaf(bm, sl2, nb)), kOneSixth);
          float rs;
          const uint32_t code = e8m0_ceil(s32, rs);
          const bool z = s32 == 0.0f;
          scw[0] |= (z ? 0u : code) << (8 * k);
          nbb[2 * k] = nbb[2 * k + 1] = z ? nb + 10.0f : nb + (127.0f - (float)code);
          sdec[2 * k] = sdec[2 * k + 1] = z ? 0x1p-10f : e8m0_to_f32(code);
        }
      } else {
        constexpr int kPairs = C::kSplit ? 3 : 4;  // split: blocks 6, 7 belong to the correction warpgroup
        uint32_t c2[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < kPairs; ++k) {
          const f2 e = ffma2(make_float2(bmax[2 * k], bmax[2 * k + 1]), sl2x2, make_float2(nb, nb));
          const f2 q = fmul2(make_float2(ex2(e.x), ex2(e.y)), make_float2(kOneSixth, kOneSixth));
          c2[k] = cvt_e4m3x2(q.x, q.y);
        }
        scw[0] = __byte_perm(c2[0], c2[1], 0x5410);
        scw[1] = __byte_perm(c2[2], c2[3], 0x5410);
#pragma unroll
        for (int blk = 0; blk < 2 * kPairs; ++blk) {
          const float2 t = s_lut[(scw[blk >> 2] >> (8 * (blk & 3))) & 0xFFu];
          nbb[blk] = nb + t.x;
          sdec[blk] = t.y;
        }
      }
      mbar_wait(&p_empty[pb], ((uint32_t)(j / kLPBufs) & 1u) ^ 1u);
      SAGE3_TRACE_EV(1 + par, j, 4);
      // ---- pass 2 from registers: y = P̃2/s, E2M1 codes, rowsum(P̃2) = Σ s·Σy (split: chunks 0-2 here)
      float rowsum = 0.0f;
      {
        f2 ya[16], yb[16];
        chunk_exps(v[0], sl2x2, nbb[0], nbb[1], ya);
        chunk_exps(v[1], sl2x2, nbb[2], nbb[3], yb);
        rowsum = chunk_finish(ya, sdec[0], sdec[1], sP, 0, r, rowsum);
        chunk_exps(v[2], sl2x2, nbb[4], nbb[5], ya);
        rowsum = chunk_finish(yb, sdec[2], sdec[3], sP, 1, r, rowsum);
        if constexpr (!C::kSplit) chunk_exps(v[3], sl2x2, nbb[6], nbb[7], yb);
        rowsum = chunk_finish(ya, sdec[4], sdec[5], sP, 2, r, rowsum);
        if constexpr (!C::kSplit) rowsum = chunk_finish(yb, sdec[6], sdec[7], sP, 3, r, rowsum);
      }
      sts_u32(sPSF, scw[0]);
      if constexpr (C::kSplit)
        sts_u16(sPSF + 512, scw[1]);  // blocks 4, 5 (bytes 6, 7 are the correction warpgroup's)
      else if constexpr (!kMX)
        sts_u32(sPSF + 512, scw[1]);
      sts_f32(xchg_s + slot * 1024 + 512, rowsum);
      fence_proxy_async_smem();
      if constexpr (kLXArrivals == 128) mbar_arrive(&x_full[slot]);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&p_full[pb]);
        if constexpr (kLXArrivals == 4) mbar_arrive(&x_full[slot]);
      }
      SAGE3_TRACE_EV(1 + par, j, 5);
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
    // ------------------------------------------------------------------ correction + epilogue
    // l and O are relative to the row's reference r (O in TMEM, accumulated by the PV MMAs).  Tile j: read
    // (r_j, rowsum_j); if r moved for any row of this warp, wait for PV_{j-1} and rescale this warp's 32 O
    // rows in TMEM by 2^{sl2 (r_{j-1} − r_j)} (1 for rows that kept r); then let the PV_j MMA go.
    setmaxnreg_dec<C::kRegCorrection>();
    const int r = threadIdx.x - 128;
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t lane_o = lane_base + kColO;
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    const float sl2 = a.scale * kLog2e;
    const f2 sl2x2 = make_float2(sl2, sl2);
    const int last = nkv - 1;
    const bool last_masked = last * 128 + 128 > a.N || a.causal;
    float rprev = -INFINITY, l = 0.0f;
    for (int j = 0; j < nkv; ++j) {
      const int slot = j % kLXSlots;
      SAGE3_TRACE_EV(4, j, 0);
      float rs3 = 0.0f;
      if constexpr (C::kSplit) {
        // pass 2 of keys [96, 128) of tile j: S chunk, block maxima 6-7, their scales (r_j from the chain),
        // codes into the tile's P̂2 buffer and scale bytes 6-7 of the row's SF word
        const int sb = j & 1, pb = j % kLPBufs;
        const uint32_t sP = smem_u32(smem + L::oP + pb * L::kPBytes) + r * 64;
        const uint32_t sPSF = smem_u32(smem + L::oPSF + pb * L::kPSF) + (r & 31) * 16 + (r >> 5) * 4;
        mbar_wait(&s_full[sb], (uint32_t)(j >> 1) & 1u);
        tc_fence_after();
        uint32_t v[32];
        tmem_ld_32x32b_x32(lane_base + 128 * sb + 96, v);
        tmem_ld_wait_regs(v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        float* f = reinterpret_cast<float*>(v);
        if (j == last && last_masked) {
          const int lim = (a.causal ? min(a.N - 1, q_row) : a.N - 1) - j * 128;
#pragma unroll
          for (int t = 0; t < 32; ++t) f[t] = (96 + t > lim) ? -INFINITY : f[t];
        }
        const float b6 = max16(f), b7 = max16(f + 16);
        mbar_wait(&r_full[slot], (uint32_t)(j / kLXSlots) & 1u);
        const float nb = kLog2Top - lds_f32(xchg_s + slot * 1024) * sl2;
        const f2 e = ffma2(make_float2(b6, b7), sl2x2, make_float2(nb, nb));
        const f2 q = fmul2(make_float2(ex2(e.x), ex2(e.y)), make_float2(kOneSixth, kOneSixth));
        const uint32_t c2 = cvt_e4m3x2(q.x, q.y);
        const float2 t6 = s_lut[c2 & 0xFFu], t7 = s_lut[(c2 >> 8) & 0xFFu];
        mbar_wait(&p_empty[pb], ((uint32_t)(j / kLPBufs) & 1u) ^ 1u);
        f2 y[16];
        chunk_exps(v, sl2x2, nb + t6.x, nb + t7.x, y);
        rs3 = chunk_finish(y, t6.y, t7.y, sP, 3, r, 0.0f);
        sts_u16(sPSF + 512 + 2, c2);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
      }
      mbar_wait(&x_full[slot], (uint32_t)(j / kLXSlots) & 1u);
      SAGE3_TRACE_EV(4, j, 1);
      const float rj = lds_f32(xchg_s + slot * 1024);
      const float rs = lds_f32(xchg_s + slot * 1024 + 512) + rs3;
      const bool moved = rj != rprev;
      const float alpha = (j > 0 && moved) ? ex2((rprev - rj) * sl2) : 1.0f;
      if (j > 0 && __any_sync(0xffffffffu, moved)) {
        mbar_wait(&pv_full[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1u);
        tc_fence_after();
        const f2 a2 = make_float2(alpha, alpha);
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(lane_o + 32 * c, o);
          tmem_ld_wait_regs(o);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const f2 x = fmul2(make_float2(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1])), a2);
            o[2 * i] = __float_as_uint(x.x);
            o[2 * i + 1] = __float_as_uint(x.y);
          }
          tmem_st_32x32b_x32(lane_o + 32 * c, o);
        }
        tmem_st_wait();
        tc_fence_before();
      }
      l = (j > 0) ? fmaf(l, alpha, rs) : rs;
      rprev = rj;
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_ready[slot]);
      SAGE3_TRACE_EV(4, j, 2);
    }
    // Alg1 L13 on the accumulated O: O/l, lse = scale·r + ln(l / 10.5)
    mbar_wait(&pv_full[(nkv - 1) & 1], (uint32_t)((nkv - 1) >> 1) & 1u);
    tc_fence_after();
    if (a.lse != nullptr && q_row < a.N) a.lse[(int64_t)bh * a.N + q_row] = rprev * a.scale + logf(l) - kLnTop;
    const float inv_l = 1.0f / l;
    // coalesced store through smem (the K/V rings are idle after the last PV MMA) and TMA (as attn.cu)
    uint8_t* stage = smem + L::oK;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(lane_o + 32 * c, o);
      tmem_ld_wait_regs(o);
      float* f = reinterpret_cast<float*>(o);
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] *= inv_l;
      stage_o_cols32(stage, r, a.o_dtype, c, f);
    }
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

template <int D, bool kMX>
cudaError_t launch_lazy_d(const AttnArgs& a, cudaStream_t stream) {
  using L = LazyLayout<D, kMX>;
  static std::atomic<bool> attr_done[64];  // one-time attribute setup per device (racing callers both set it: idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_lazy_kernel<D, kMX>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = a.B * a.H;
  CUtensorMap tq, tk, tv;
  CUtensorMap to;
  if (!make_map(&tq, a.q_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tk, a.k_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tv, a.v_data, (uint64_t)a.Np / 2, (uint64_t)BH * D, 64, D) ||
      !make_map_o(&to, a.o, a.o_dtype, a.B, a.H, a.N, D, a.o_sb, a.o_sh, a.o_sn))
    return cudaErrorInvalidValue;
  const int64_t units = a.unit_end - a.unit_begin;
  if (units <= 0) return cudaSuccess;
  attn_lazy_kernel<D, kMX><<<(unsigned)units, kLThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

}  // namespace

#ifdef SAGE3_TRACE
extern "C" int sage3_debug_trace_copy_lazy(void* host, size_t bytes) {
  if (bytes > sizeof(g_trace)) bytes = sizeof(g_trace);
  return (int)cudaMemcpyFromSymbol(host, g_trace, bytes);
}
#endif

cudaError_t launch_attention_lazy(const AttnArgs& a, cudaStream_t stream) {
  if (a.mx) return a.d == 128 ? launch_lazy_d<128, true>(a, stream) : launch_lazy_d<64, true>(a, stream);
  return a.d == 128 ? launch_lazy_d<128, false>(a, stream) : launch_lazy_d<64, false>(a, stream);
}

}  // namespace sage3
