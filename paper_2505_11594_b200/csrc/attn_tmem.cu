// attn_tmem.cu — the paper's Algorithm 1 (two-level P) with O accumulated by the tensor core
// in TMEM.  Same numerics as attn.cu (reading c14's tile-local form: P̃2_j = 2688·2^{sl2(S − tmax_j)}, per-tile
// s_P1, l from the unquantized P̃ — or, with kQSum, the NEXT #2 row-sum variant of reading n2); a different
// division of labour:
//
//   attn.cu keeps O in the correction warpgroup's registers (128 fp32 per row), so PV_j goes to a TMEM buffer the
//   correction must read back before S_{j+3} can reuse it, and the softmax re-reads S from TMEM in pass 2.
//   Here the PV MMA accumulates straight into O in TMEM.  Alg1 L11's per-tile weight s_P1_j is applied by
//   rescaling the accumulator before PV_j lands:  O_acc holds O / c_j with c_j = 2^{e_j}/2688 (log2 units
//   e_j = sl2·tmax_j), so before PV_j the correction multiplies O_acc by ρ_j = 2^{e_{j−1} − e_j} (a TMEM
//   read-modify-write of the row, off the softmax's path: it only has to finish before P̂2_j is ready).
//   The freed registers let each softmax thread keep its whole S row from pass 1 to pass 2 (208 registers), so an
//   S buffer is released right after the four TMEM loads; two S buffers suffice.
//
// Overflow guard: O_acc ≈ O_true / c_j can grow like w_max / w_j when a tile's max is far below an earlier one.
// The accumulator exponent is clamped to e_j = max(sl2·tmax_j, M_j − 64) with M_j the running max (Alg1's m_j in
// log2 units): ρ_j ≤ 2^64 and |O_acc| stays below ~2^90.  A clamped tile (weight < 2^-64 of the row's maximum
// tile) enters the numerator with weight 2^{e_j} instead of 2^{sl2·tmax_j}: an absolute error below
// 2^-46·max|V̂| in O/l, far under fp32 resolution.
//
// Roles (16 warps, 1 CTA per SM): WG0 TMA (Q/K, V) + MMA issuers (S, PV) + TMEM allocator; WG1/WG2 softmax on even /
// odd KV tiles; WG3 correction (accumulator rescale, l, epilogue).  TMEM: S 2 x 128 columns, O at 256 (d columns),
// scale factors 384..415, kQSum row sums at 448 + 16·(j%2), ones-operand scales at 432.
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

constexpr int kTKStages = 5, kTVStages = 4;
constexpr int kTPBufs = 4;   // P̂2 tiles in smem (tile j -> j % 4)
constexpr int kTXSlots = 8;  // softmax -> correction exchange slots (tile j -> j % 8)
constexpr int kTThreads = 512;
constexpr uint32_t kTRegWG0 = 32, kTRegSoftmax = 208, kTRegCorrection = 64;
static_assert(kTRegWG0 + 2 * kTRegSoftmax + kTRegCorrection <= 512, "register budget");
constexpr uint32_t kTColO = 256, kTColSF1 = 432, kTColRS = 448;
constexpr float kTClamp = 64.0f;  // accumulator exponent floor below the running max (log2 units)
#ifndef SAGE3_TM_WARP_ARRIVE
#define SAGE3_TM_WARP_ARRIVE 0  // 1: t_full / x_full get one arrival per warp (after __syncwarp) instead of per thread
#endif
constexpr uint32_t kTXArrivals = SAGE3_TM_WARP_ARRIVE ? 4 : 128;
__device__ __forceinline__ void t_arrive(uint64_t* bar) {
#if SAGE3_TM_WARP_ARRIVE
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
#else
  mbar_arrive(bar);
#endif
}

template <int D>
struct TmemLayout {
  static constexpr int kQKRow = D / 2;
  static constexpr int kQBytes = 128 * kQKRow;
  static constexpr int kKBytes = 128 * kQKRow;
  static constexpr int kKSlot = ((kKBytes + 1023) / 1024) * 1024;
  static constexpr int kVBytes = D * 64;
  static constexpr int kPBytes = 128 * 64;
  static constexpr int kQKSF = (D / 64) * 512;
  static constexpr int kVSF = 1024, kPSF = 1024;
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + ((kQBytes + 1023) / 1024) * 1024;
  static constexpr int oV = oK + kTKStages * kKSlot;
  static constexpr int oP = oV + kTVStages * kVBytes;
  static constexpr int oQSF = oP + kTPBufs * kPBytes;
  static constexpr int oKSF = oQSF + kQKSF;
  static constexpr int oVSF = oKSF + kTKStages * kQKSF;
  static constexpr int oPSF = oVSF + kTVStages * kVSF;
  static constexpr int oOnes = oPSF + kTPBufs * kPSF;  // kQSum: all-ones B operand (1 KB) + its SF atoms (1 KB)
  static constexpr int oXchg = oOnes + 2048;          // float [kTXSlots][2][128]: tmax_j, rowsum(P̃2_j)
  static constexpr int oBar = oXchg + kTXSlots * 2 * 128 * 4;
  // q_full, k_full/empty, v_full/empty, s_full/empty[2], pv_full[2], p_full/empty, t_full, x_full, o_ready
  static constexpr int kNumBars = 1 + 2 * kTKStages + 2 * kTVStages + 2 * 2 + 2 + 2 * kTPBufs + 3 * kTXSlots;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kBytes = oTmem + 16;
  static constexpr int kSmemAlloc = kBytes + 1024;
};

// One 32-key chunk of pass 2: y = P̃2/s = 2^(S·sl2 + nb − log2 s) on MUFU or the FMA-pipe polynomial.
__device__ __forceinline__ void t_chunk_exps(const uint32_t (&vv)[32], f2 sl2x2, float nA, float nB, f2 (&y)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float nbh = i < 8 ? nA : nB;
    const f2 x = ffma2(make_float2(__uint_as_float(vv[2 * i]), __uint_as_float(vv[2 * i + 1])), sl2x2,
                       make_float2(nbh, nbh));
    y[i] = ((kPolyMask >> i) & 1u) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
  }
}
// ... its E2M1 codes (chunk c of row r in the SWIZZLE_64B P̂2 tile) and, unless kQSum, its rowsum share
template <bool kQSum>
__device__ __forceinline__ float t_chunk_finish(const f2 (&y)[16], float sA, float sB, uint32_t sP_row, int c, int r,
                                                float rowsum) {
  uint32_t w[4];
#pragma unroll
  for (int hb = 0; hb < 2; ++hb) {
    const f2* yy = y + 8 * hb;
    if constexpr (!kQSum) {
      const f2 s01 = fadd2(fadd2(yy[0], yy[1]), fadd2(yy[2], yy[3]));
      const f2 s23 = fadd2(fadd2(yy[4], yy[5]), fadd2(yy[6], yy[7]));
      const f2 sy = fadd2(s01, s23);
      rowsum = fmaf(hb ? sB : sA, sy.x + sy.y, rowsum);
    }
    w[2 * hb] = cvt_e2m1x8(yy[0].x, yy[0].y, yy[1].x, yy[1].y, yy[2].x, yy[2].y, yy[3].x, yy[3].y);
    w[2 * hb + 1] = cvt_e2m1x8(yy[4].x, yy[4].y, yy[5].x, yy[5].y, yy[6].x, yy[6].y, yy[7].x, yy[7].y);
  }
  sts_v4(sP_row + ((c ^ ((r >> 1) & 3)) * 16), w[0], w[1], w[2], w[3]);
  return rowsum;
}

template <int D, bool kQSum>
__global__ void __launch_bounds__(kTThreads, 1)
    attn_tmem_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                     const AttnArgs a) {
  using L = TmemLayout<D>;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(1024) float2 s_lut[128];  // (-log2 s, s) per E4M3 scale code, as in attn.cu
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::oQ;
  uint8_t* sQSF = smem + L::oQSF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + kTKStages;
  uint64_t* v_full = k_empty + kTKStages;
  uint64_t* v_empty = v_full + kTVStages;
  uint64_t* s_full = v_empty + kTVStages;  // MMA -> softmax: S_j in buffer j%2
  uint64_t* s_empty = s_full + 2;          // softmax -> MMA: S_j loaded into registers, buffer free
  uint64_t* pv_full = s_empty + 2;         // MMA -> correction: PV_j accumulated into O (tile parity j%2)
  uint64_t* p_full = pv_full + 2;          // softmax -> MMA: P̂2_j / s_P2 in smem buffer j%4
  uint64_t* p_empty = p_full + kTPBufs;    // MMA -> softmax: PV_j done with smem buffer j%4
  uint64_t* t_full = p_empty + kTPBufs;    // softmax -> correction: tmax_j in slot j%8 (right after pass 1)
  uint64_t* x_full = t_full + kTXSlots;    // softmax -> correction: rowsum(P̃2_j) in slot j%8 (end of the tile)
  uint64_t* o_ready = x_full + kTXSlots;   // correction -> MMA: O_acc rescaled to tile j's exponent
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = a.Np >> 7;
  const int64_t unit = a.unit_begin + (int64_t)blockIdx.x;
  const int bh = (int)(unit / n_qt);
  const int qt = n_qt - 1 - (int)(unit % n_qt);
  const int nkv = a.causal ? qt + 1 : n_qt;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kTKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kTVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 4);  // one arrival per softmax warp
      mbar_init(&pv_full[b], 1);
    }
    for (int b = 0; b < kTPBufs; ++b) {
      mbar_init(&p_full[b], 4);
      mbar_init(&p_empty[b], 1);
    }
    for (int s = 0; s < kTXSlots; ++s) {
      mbar_init(&t_full[s], kTXArrivals);  // per thread (each orders its own slot write) or per warp
      mbar_init(&x_full[s], kTXArrivals);
      mbar_init(&o_ready[s], 4);   // one arrival per correction warp
    }
    fence_mbar_init();
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
  if constexpr (kQSum) {  // the constant ones operand (E2M1 1.0 = code 2) and its scales (E4M3 1.0 = 0x38)
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem + L::oOnes);
    for (int i = threadIdx.x; i < 512; i += kTThreads) ones[i] = i < 256 ? 0x22222222u : 0x38383838u;
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int wg = warp >> 2;

  if (wg == 0) {
    setmaxnreg_dec<kTRegWG0>();
    if (warp == 0) {  // ------------------------------------------------------------ TMA producer: Q, K
      if (elect_one()) {
        const int row_q = bh * a.Np + qt * 128;
        mbar_arrive_expect_tx(q_full, L::kQBytes + L::kQKSF);
        tma_load_2d(sQ, &tm_q, q_full, 0, row_q);
        bulk_load(sQSF, a.q_sf + (int64_t)(row_q >> 7) * L::kQKSF, L::kQKSF, q_full);
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kTKStages;
          const int row_k = bh * a.Np + j * 128;
          mbar_wait(&k_empty[st], ((uint32_t)(j / kTKStages) & 1u) ^ 1u);
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
          const int st = j % kTVStages;
          mbar_wait(&v_empty[st], ((uint32_t)(j / kTVStages) & 1u) ^ 1u);
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
        constexpr int kQKAtoms = L::kQKSF / 512;
        if (warp == 1) {
          mbar_wait(q_full, 0);
          tc_fence_after();
#pragma unroll
          for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kColSFQ + 4 * at, sf_desc(sQSF + 512 * at));
          for (int j = 0; j < nkv; ++j) {
            const int b = j & 1, st = j % kTKStages;
            mbar_wait(&s_empty[b], ((uint32_t)(j >> 1) & 1u) ^ 1u);  // softmax loaded S_{j-2}
            mbar_wait(&k_full[st], (uint32_t)(j / kTKStages) & 1u);
            tc_fence_after();
            const uint8_t* sK = smem + L::oK + st * L::kKSlot;
            const uint8_t* sKSF = smem + L::oKSF + st * L::kQKSF;
#pragma unroll
            for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kColSFK + 4 * at, sf_desc(sKSF + 512 * at));
#pragma unroll
            for (int ks = 0; ks < D / 64; ++ks) {
              const uint64_t ad = make_smem_desc(smem_u32(sQ) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
              const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
              mma_nvf4(tbase + 128 * b, ad, bd, make_idesc_nvf4(128, 128), tbase + kColSFQ + 4 * ks,
                       tbase + kColSFK + 4 * ks, ks > 0);
            }
            mma_commit(&k_empty[st]);
            mma_commit(&s_full[b]);
          }
        } else {
          if constexpr (kQSum) {
#pragma unroll
            for (int at = 0; at < 2; ++at)
              tmem_cp_32x128b_x4(tbase + kTColSF1 + 4 * at, sf_desc(smem + L::oOnes + 1024 + 512 * at));
          }
          for (int j = 0; j < nkv; ++j) {
            const int pb = j % kTPBufs, st = j % kTVStages, slot = j % kTXSlots;
            mbar_wait(&p_full[pb], (uint32_t)(j / kTPBufs) & 1u);
            mbar_wait(&v_full[st], (uint32_t)(j / kTVStages) & 1u);
            mbar_wait(&o_ready[slot], (uint32_t)(j / kTXSlots) & 1u);  // O_acc in tile j's exponent
            tc_fence_after();
            const uint8_t* sP = smem + L::oP + pb * L::kPBytes;
            const uint8_t* sV = smem + L::oV + st * L::kVBytes;
            const uint8_t* sPSF = smem + L::oPSF + pb * L::kPSF;
            const uint8_t* sVSF = smem + L::oVSF + st * L::kVSF;
#pragma unroll
            for (int at = 0; at < 2; ++at) {
              tmem_cp_32x128b_x4(tbase + kColSFP + 4 * at, sf_desc(sPSF + 512 * at));
              tmem_cp_32x128b_x4(tbase + kColSFV + 4 * at, sf_desc(sVSF + 512 * at));
            }
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
              const uint64_t bd = make_smem_desc(smem_u32(sV) + 32 * ks, 16, 512, kLayoutSw64);
              mma_nvf4(tbase + kTColO, ad, bd, make_idesc_nvf4(128, D), tbase + kColSFP + 4 * ks,
                       tbase + kColSFV + 4 * ks, (j > 0 || ks > 0) ? 1u : 0u);
            }
            if constexpr (kQSum) {  // row sums of the quantized P̂2: P̂2 x ones (N = 16)
#pragma unroll
              for (int ks = 0; ks < 2; ++ks) {
                const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
                const uint64_t bd = make_smem_desc(smem_u32(smem + L::oOnes) + 32 * ks, 16, 512, kLayoutSw64);
                mma_nvf4(tbase + kTColRS + 16 * (j & 1), ad, bd, make_idesc_nvf4(128, 16), tbase + kColSFP + 4 * ks,
                         tbase + kTColSF1 + 4 * ks, ks > 0);
              }
            }
            mma_commit(&v_empty[st]);
            mma_commit(&p_empty[pb]);
            mma_commit(&pv_full[j & 1]);
          }
        }
      }
      __syncwarp();
    }
  } else if (wg >= 2) {
    // ------------------------------------------------------------------ softmax + two-level P (Alg1 L9-L10)
    setmaxnreg_inc<kTRegSoftmax>();
    const int par = wg - 2;
    const int r = threadIdx.x - 128 * wg;
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    const f2 sl2x2 = make_float2(sl2, sl2);
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    auto tile = [&](const int j, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const int sb = j & 1, pb = j % kTPBufs, slot = j % kTXSlots;
      const uint32_t s_addr = lane_base + 128 * sb;
      const uint32_t sP = smem_u32(smem + L::oP + pb * L::kPBytes) + r * 64;
      const uint32_t sPSF = smem_u32(smem + L::oPSF + pb * L::kPSF) + (r & 31) * 16 + (r >> 5) * 4;
      mbar_wait(&s_full[sb], (uint32_t)(j >> 1) & 1u);
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
      // ---- pass 1 (registers): masking, 16-key block maxima (reused for tmax and s_P2)
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
      sts_f32(xchg_s + slot * 1024, tmax);  // -> correction: the accumulator rescale for this tile
      t_arrive(&t_full[slot]);
      const float nb = kLog2_2688 - tmax * sl2;  // P̃2 = 2^(S·sl2 + nb), max element 2688 (reading c14)
      // ---- block scales of φ(P̃2) (as attn.cu)
      float nbb[8], sdec[8];
      uint32_t scw[2];
      {
        uint32_t c2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const f2 e = ffma2(make_float2(bmax[2 * k], bmax[2 * k + 1]), sl2x2, make_float2(nb, nb));
          const f2 q = fmul2(make_float2(ex2(e.x), ex2(e.y)), make_float2(kOneSixth, kOneSixth));
          c2[k] = cvt_e4m3x2(q.x, q.y);
        }
        scw[0] = __byte_perm(c2[0], c2[1], 0x5410);
        scw[1] = __byte_perm(c2[2], c2[3], 0x5410);
#pragma unroll
        for (int blk = 0; blk < 8; ++blk) {
          const float2 t = s_lut[(scw[blk >> 2] >> (8 * (blk & 3))) & 0xFFu];
          nbb[blk] = nb + t.x;
          sdec[blk] = t.y;
        }
      }
      mbar_wait(&p_empty[pb], ((uint32_t)(j / kTPBufs) & 1u) ^ 1u);
      // ---- pass 2 from registers: y = P̃2/s, E2M1 codes, rowsum(P̃2) = Σ s·Σy (kQSum: from the tensor core)
      float rowsum = 0.0f;
      {
        f2 ya[16], yb[16];
        t_chunk_exps(v[0], sl2x2, nbb[0], nbb[1], ya);
        t_chunk_exps(v[1], sl2x2, nbb[2], nbb[3], yb);
        rowsum = t_chunk_finish<kQSum>(ya, sdec[0], sdec[1], sP, 0, r, rowsum);
        t_chunk_exps(v[2], sl2x2, nbb[4], nbb[5], ya);
        rowsum = t_chunk_finish<kQSum>(yb, sdec[2], sdec[3], sP, 1, r, rowsum);
        t_chunk_exps(v[3], sl2x2, nbb[6], nbb[7], yb);
        rowsum = t_chunk_finish<kQSum>(ya, sdec[4], sdec[5], sP, 2, r, rowsum);
        rowsum = t_chunk_finish<kQSum>(yb, sdec[6], sdec[7], sP, 3, r, rowsum);
      }
      sts_u32(sPSF, scw[0]);
      sts_u32(sPSF + 512, scw[1]);
      if constexpr (!kQSum) {
        sts_f32(xchg_s + slot * 1024 + 512, rowsum);
        t_arrive(&x_full[slot]);
      }
      fence_proxy_async_smem();
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
    // ------------------------------------------------------------------ correction + epilogue
    // O_acc = O / c_j, c_j = 2^{e_j}/2688 relative to exponent 0; e_j = max(sl2·tmax_j, M_j − kTClamp), M_j the
    // running max of sl2·tmax.  l_acc = l / c_j likewise.  Tile j: once tmax_j is known and PV_{j−1} has landed,
    // l_acc += rs_{j−1}·2^{g_{j−1} − e_{j−1}}, then O_acc and l_acc are multiplied by ρ_j = 2^{e_{j−1} − e_j};
    // then PV_j may accumulate (weight 1 in units of c_j).
    setmaxnreg_dec<kTRegCorrection>();
    const int r = threadIdx.x - 128;
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t lane_o = lane_base + kTColO;
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    const float sl2 = a.scale * kLog2e;
    float M = -INFINITY, e_prev = 0.0f, g_prev = 0.0f, l = 0.0f;
    // adds tile jj's row sum to l_acc (units of its own exponent); PV_jj has landed (pv_full waited)
    auto add_rowsum = [&](int jj) {
      float rs;
      if constexpr (kQSum) {
        uint32_t rq;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(rq) : "r"(lane_base + kTColRS + 16 * (jj & 1)));
        tmem_ld_wait();
        asm volatile("" : "+r"(rq));
        rs = __uint_as_float(rq);
      } else {
        const int s = jj % kTXSlots;
        mbar_wait(&x_full[s], (uint32_t)(jj / kTXSlots) & 1u);  // (already complete: it precedes p_full)
        rs = lds_f32(xchg_s + s * 1024 + 512);
      }
      l = fmaf(rs, ex2(g_prev - e_prev), l);
    };
    for (int j = 0; j < nkv; ++j) {
      const int slot = j % kTXSlots;
      mbar_wait(&t_full[slot], (uint32_t)(j / kTXSlots) & 1u);
      const float g = lds_f32(xchg_s + slot * 1024) * sl2;
      M = fmaxf(M, g);
      const float e = fmaxf(g, M - kTClamp);
      if (j > 0) {
        mbar_wait(&pv_full[(j - 1) & 1], (uint32_t)((j - 1) >> 1) & 1u);
        tc_fence_after();
        add_rowsum(j - 1);
        const float rho = ex2(e_prev - e);
        l *= rho;
        if (__any_sync(0xffffffffu, rho != 1.0f)) {
          const f2 r2 = make_float2(rho, rho);
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(lane_o + 32 * c, o);
            tmem_ld_wait_regs(o);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const f2 x = fmul2(make_float2(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1])), r2);
              o[2 * i] = __float_as_uint(x.x);
              o[2 * i + 1] = __float_as_uint(x.y);
            }
            tmem_st_32x32b_x32(lane_o + 32 * c, o);
          }
          tmem_st_wait();
        }
        tc_fence_before();
      }
      e_prev = e, g_prev = g;
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_ready[slot]);
    }
    // Alg1 L13: O/l; lse = ln(l) = ln(l_acc) + e_last·ln 2 − ln 2688 (e in log2 units of scale·S)
    mbar_wait(&pv_full[(nkv - 1) & 1], (uint32_t)((nkv - 1) >> 1) & 1u);
    tc_fence_after();
    add_rowsum(nkv - 1);
    if (a.lse != nullptr && q_row < a.N)
      a.lse[(int64_t)bh * a.N + q_row] = logf(l) + e_prev * 0.69314718055994531f - 7.8966259942968059f;
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

template <int D, bool kQSum>
cudaError_t launch_tmem_d(const AttnArgs& a, cudaStream_t stream) {
  using L = TmemLayout<D>;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_tmem_kernel<D, kQSum>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         L::kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = a.B * a.H;
  CUtensorMap tq, tk, tv, to;
  if (!make_map(&tq, a.q_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tk, a.k_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tv, a.v_data, (uint64_t)a.Np / 2, (uint64_t)BH * D, 64, D) ||
      !make_map_o(&to, a.o, a.o_dtype, a.B, a.H, a.N, D, a.o_sb, a.o_sh, a.o_sn))
    return cudaErrorInvalidValue;
  const int64_t units = a.unit_end - a.unit_begin;
  if (units <= 0) return cudaSuccess;
  attn_tmem_kernel<D, kQSum><<<(unsigned)units, kTThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_tmem(const AttnArgs& a, cudaStream_t stream) {
  if (a.p_qsum) return a.d == 128 ? launch_tmem_d<128, true>(a, stream) : launch_tmem_d<64, true>(a, stream);
  return a.d == 128 ? launch_tmem_d<128, false>(a, stream) : launch_tmem_d<64, false>(a, stream);
}

}  // namespace sage3
