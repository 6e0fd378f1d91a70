// attn.cu — sm_100a SageAttention3 FP4 attention forward: Algorithm 1 L6-L13.
//
// One CTA = one 128-row query tile Q_i of one (b,h); loop over 128-key tiles j (B_q = B_kv = 128).
// Warp roles (12 warps, 3 warpgroups):
//   warp 0      TMA producer: Q̂_i + s_Q once; K̂_j + s_K and V̂ᵀ_j + s_V per stage (kStages ring)
//   warp 1      MMA issuer (one elected lane):
//                 S_j  = FP4MM(Q̂_i, s_Q, K̂_j, s_K)        tcgen05.mma kind::mxf4nvf4, M=128 N=128 K=d
//                 PV_j = FP4MM(P̂2_j, s_P2, V̂_j, s_V)      M=128 N=d K=128, fresh TMEM accumulator
//               scale factors are staged smem -> TMEM with tcgen05.cp.32x128b.warpx4 in issue order
//   warp 2      TMEM allocator (512 columns)
//   warps 4-7   softmax: one query row per thread (TMEM lane = row); online softmax (Alg1 L9) and the
//               two-level P quantization (Alg1 L10, §3.2) entirely in registers; writes P̂2
//               (K-major, SWIZZLE_64B) and s_P2 (SF atoms) to smem for the PV MMA
//   warps 8-11  correction: O kept in registers, O = α·O + s_P1·PV_j (Alg1 L11), O/l (L13), store
//
// Two-level P identity used on the GPU (reading c14): with tmax = rowmax(S_ij) and
// m_ij = max(m_{i,j-1}, tmax),
//     P̃2 = P̃ / s_P1 = 2688 · exp(scale·(S − tmax))          (max element = 2688 -> s_P2 = 448, code 6)
//     s_P1 = rowmax(P̃)/2688 = exp(scale·(tmax − m_ij)) / 2688
//     l_ij = e^{scale(m_{i,j-1} − m_ij)} l_{i,j-1} + s_P1 · rowsum(P̃2)
// and exp(x) = 2^(x·log2 e) on MUFU.EX2.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <mutex>

#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

constexpr int kStages = 3;
constexpr int kThreads = 384;
constexpr float kOneSixth = 0x1.555556p-3f;  // fl32(1/6)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLog2_2688 = 11.392317422778761f;  // log2(448 * 6)

// TMEM column map (512 columns allocated).
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColPV = 256;
constexpr uint32_t kColSFQ = 384, kColSFK = 392, kColSFV = 400, kColSFP = 408;

template <int D>
struct Layout {
  static constexpr int kQKRow = D / 2;         // bytes per Q/K row (64 or 32)
  static constexpr int kQBytes = 128 * kQKRow;  // Q tile codes
  static constexpr int kKBytes = 128 * kQKRow;
  static constexpr int kVBytes = D * 64;     // Vᵀ tile: D channel rows x 128 tokens (64 B)
  static constexpr int kPBytes = 128 * 64;   // P̂2 tile: 128 rows x 128 keys (64 B)
  static constexpr int kQKSF = (D / 64) * 512;  // SF atoms per 128-row tile along d
  static constexpr int kVSF = 1024, kPSF = 1024;  // 8 token-blocks = 2 atoms
  // byte offsets inside the 1024-aligned dynamic smem window
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + ((kQBytes + 1023) / 1024) * 1024;
  static constexpr int oV = oK + kStages * ((kKBytes + 1023) / 1024) * 1024;
  static constexpr int oP = oV + kStages * kVBytes;
  static constexpr int oQSF = oP + 2 * kPBytes;
  static constexpr int oKSF = oQSF + kQKSF;
  static constexpr int oVSF = oKSF + kStages * kQKSF;
  static constexpr int oPSF = oVSF + kStages * kVSF;
  static constexpr int oXchg = oPSF + 2 * kPSF;       // float [4 slots][2][128]
  static constexpr int oLut = oXchg + 4 * 2 * 128 * 4;  // float [128] exact 1/s per E4M3 code
  static constexpr int oFin = oLut + 128 * 4;          // float [2][128] final l, m
  static constexpr int oBar = oFin + 2 * 128 * 4;      // mbarriers (8 B each)
  static constexpr int kNumBars = 1 + 4 * kStages + 2 + 2 + 2 + 2 + 2 + 4;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kBytes = oTmem + 16;
  static constexpr int kSmemAlloc = kBytes + 1024;  // slack for manual 1024-B alignment
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void setmaxnreg_dec40() { asm volatile("setmaxnreg.dec.sync.aligned.u32 40;"); }
__device__ __forceinline__ void setmaxnreg_inc232() { asm volatile("setmaxnreg.inc.sync.aligned.u32 232;"); }
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
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

__device__ __forceinline__ uint64_t sf_desc(const void* p) {
  return make_smem_desc(smem_u32(p), 0, 128, kLayoutNone);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const AttnArgs a) {
  using L = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  uint8_t* sQ = smem + L::oQ;
  uint8_t* sQSF = smem + L::oQSF;
  float* xchg = reinterpret_cast<float*>(smem + L::oXchg);
  float* lut = reinterpret_cast<float*>(smem + L::oLut);
  float* fin = reinterpret_cast<float*>(smem + L::oFin);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + kStages;
  uint64_t* v_full = k_empty + kStages;
  uint64_t* v_empty = v_full + kStages;
  uint64_t* s_full = v_empty + kStages;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 2;
  uint64_t* pv_full = p_empty + 2;
  uint64_t* pv_empty = pv_full + 1;
  uint64_t* x_full = pv_empty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = a.Np >> 7;
  const int bh = blockIdx.x;
  const int qt = n_qt - 1 - (int)blockIdx.y;  // longest-first under causal masking
  const int nkv = a.causal ? qt + 1 : n_qt;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 128);
      mbar_init(&p_full[b], 128);
      mbar_init(&p_empty[b], 1);
    }
    mbar_init(pv_full, 1);
    mbar_init(pv_empty, 128);
    for (int s = 0; s < 4; ++s) mbar_init(&x_full[s], 128);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x >= 128 && threadIdx.x < 256) {  // exact reciprocal of every E4M3 scale; 0 for s = 0
    const int c = threadIdx.x - 128;
    const float s = e4m3_to_f32((uint32_t)c);
    lut[c] = (s == 0.0f || c == 0x7F) ? 0.0f : __frcp_rn(s);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int wg = warp >> 2;

  if (wg == 0) {
    setmaxnreg_dec40();
    if (warp == 0) {
      // ------------------------------------------------------------------ TMA producer
      if (elect_one()) {
        const int row_q = bh * a.Np + qt * 128;
        mbar_arrive_expect_tx(q_full, L::kQBytes + L::kQKSF);
        tma_load_2d(sQ, &tm_q, q_full, 0, row_q);
        bulk_load(sQSF, a.q_sf + (int64_t)row_q * (D / 16), L::kQKSF, q_full);
        for (int j = 0; j < nkv; ++j) {
          const int st = j % kStages;
          const uint32_t ph = (uint32_t)(j / kStages) & 1u;
          const int row_k = bh * a.Np + j * 128;
          mbar_wait(&k_empty[st], ph ^ 1u);
          mbar_arrive_expect_tx(&k_full[st], L::kKBytes + L::kQKSF);
          tma_load_2d(smem + L::oK + st * ((L::kKBytes + 1023) / 1024) * 1024, &tm_k, &k_full[st], 0, row_k);
          bulk_load(smem + L::oKSF + st * L::kQKSF, a.k_sf + (int64_t)row_k * (D / 16), L::kQKSF, &k_full[st]);
          mbar_wait(&v_empty[st], ph ^ 1u);
          mbar_arrive_expect_tx(&v_full[st], L::kVBytes + L::kVSF);
          tma_load_2d(smem + L::oV + st * L::kVBytes, &tm_v, &v_full[st], j * 64, bh * D);
          bulk_load(smem + L::oVSF + st * L::kVSF, a.v_sf + (int64_t)bh * 128 * (a.Np / 16) + j * 1024, L::kVSF,
                    &v_full[st]);
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ------------------------------------------------------------------ MMA issuer
      if (elect_one()) {
        constexpr uint32_t kQKLayout = D == 128 ? kLayoutSw64 : kLayoutSw32;
        constexpr uint32_t idesc_s = make_idesc_nvf4(128, 128);
        constexpr uint32_t idesc_pv = make_idesc_nvf4(128, D);
        mbar_wait(q_full, 0);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < D / 64; ++ks) tmem_cp_32x128b_x4(tbase + kColSFQ + 4 * ks, sf_desc(sQSF + 512 * ks));
        auto issue_s = [&](int j) {
          const int b = j & 1, st = j % kStages;
          mbar_wait(&s_empty[b], ((uint32_t)(j >> 1) & 1u) ^ 1u);
          mbar_wait(&k_full[st], (uint32_t)(j / kStages) & 1u);
          tc_fence_after();
          const uint8_t* sK = smem + L::oK + st * ((L::kKBytes + 1023) / 1024) * 1024;
          const uint8_t* sKSF = smem + L::oKSF + st * L::kQKSF;
#pragma unroll
          for (int ks = 0; ks < D / 64; ++ks) tmem_cp_32x128b_x4(tbase + kColSFK + 4 * ks, sf_desc(sKSF + 512 * ks));
#pragma unroll
          for (int ks = 0; ks < D / 64; ++ks) {
            const uint64_t ad = make_smem_desc(smem_u32(sQ) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
            const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
            mma_nvf4(tbase + (b ? kColS1 : kColS0), ad, bd, idesc_s, tbase + kColSFQ + 4 * ks,
                     tbase + kColSFK + 4 * ks, ks > 0);
          }
          mma_commit(&k_empty[st]);
          mma_commit(&s_full[b]);
        };
        auto issue_pv = [&](int j) {
          const int pb = j & 1, st = j % kStages;
          mbar_wait(&p_full[pb], (uint32_t)(j >> 1) & 1u);
          mbar_wait(&v_full[st], (uint32_t)(j / kStages) & 1u);
          mbar_wait(pv_empty, ((uint32_t)j & 1u) ^ 1u);
          tc_fence_after();
          const uint8_t* sP = smem + L::oP + pb * L::kPBytes;
          const uint8_t* sV = smem + L::oV + st * L::kVBytes;
          const uint8_t* sPSF = smem + L::oPSF + pb * L::kPSF;
          const uint8_t* sVSF = smem + L::oVSF + st * L::kVSF;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            tmem_cp_32x128b_x4(tbase + kColSFP + 4 * ks, sf_desc(sPSF + 512 * ks));
            tmem_cp_32x128b_x4(tbase + kColSFV + 4 * ks, sf_desc(sVSF + 512 * ks));
          }
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
            const uint64_t bd = make_smem_desc(smem_u32(sV) + 32 * ks, 16, 512, kLayoutSw64);
            mma_nvf4(tbase + kColPV, ad, bd, idesc_pv, tbase + kColSFP + 4 * ks, tbase + kColSFV + 4 * ks, ks > 0);
          }
          mma_commit(&v_empty[st]);
          mma_commit(&p_empty[pb]);
          mma_commit(pv_full);
        };
        issue_s(0);
        if (nkv > 1) issue_s(1);
        for (int j = 0; j < nkv; ++j) {
          if (j + 2 < nkv) issue_s(j + 2);
          issue_pv(j);
        }
      }
      __syncwarp();
    }
  } else if (wg == 1) {
    // -------------------------------------------------------------------- softmax + two-level P quant
    setmaxnreg_inc232();
    const int r = threadIdx.x - 128;  // query row in the tile == TMEM lane
    const int q_row = qt * 128 + r;
    const uint32_t lane_addr = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    float m = -INFINITY, l = 0.0f;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (uint32_t)(j >> 1) & 1u);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(lane_addr + (b ? kColS1 : kColS0) + 32 * c, v);
        tmem_ld_wait_regs(v);
#pragma unroll
        for (int i = 0; i < 32; ++i) s[32 * c + i] = __uint_as_float(v[i]);
      }
      tc_fence_before();
      mbar_arrive(&s_empty[b]);
      const int kv0 = j * 128;
      if (kv0 + 128 > a.N || (a.causal && j == qt)) {
        const int lim = a.causal ? min(a.N - 1, q_row) : a.N - 1;
#pragma unroll
        for (int t = 0; t < 128; ++t)
          if (kv0 + t > lim) s[t] = -INFINITY;
      }
      float tmax = s[0];
#pragma unroll
      for (int t = 1; t < 128; ++t) tmax = fmaxf(tmax, s[t]);
      const float m_new = fmaxf(m, tmax);
      const float alpha = ex2((m - m_new) * sl2);
      const float nb = kLog2_2688 - tmax * sl2;  // P̃2 = 2^(S·sl2 + nb) = 2688·e^{scale(S − tmax)}
      float rowsum = 0.0f;
#pragma unroll
      for (int t = 0; t < 128; ++t) {
        s[t] = ex2(fmaf(s[t], sl2, nb));
        rowsum += s[t];
      }
      const float sP1 = ex2((tmax - m_new) * sl2 - kLog2_2688);
      l = alpha * l + sP1 * rowsum;
      // φ(P̃2) over 8 blocks of 16 keys (Eq. 1 with readings c2-c5)
      uint32_t packed[16];
      uint32_t scw0 = 0, scw1 = 0;
#pragma unroll
      for (int blk = 0; blk < 8; ++blk) {
        float amax = s[16 * blk];
#pragma unroll
        for (int i = 1; i < 16; ++i) amax = fmaxf(amax, s[16 * blk + i]);
        const uint32_t sc = cvt_e4m3x2(__fmul_rn(amax, kOneSixth), 0.0f) & 0xFFu;
        const float rcp = lut[sc];
        uint32_t bytes[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          bytes[i] = cvt_e2m1x2(__fmul_rn(s[16 * blk + 2 * i], rcp), __fmul_rn(s[16 * blk + 2 * i + 1], rcp));
        packed[2 * blk] = bytes[0] | (bytes[1] << 8) | (bytes[2] << 16) | (bytes[3] << 24);
        packed[2 * blk + 1] = bytes[4] | (bytes[5] << 8) | (bytes[6] << 16) | (bytes[7] << 24);
        if (blk < 4)
          scw0 |= sc << (8 * blk);
        else
          scw1 |= sc << (8 * (blk - 4));
      }
      const int pb = j & 1;
      mbar_wait(&p_empty[pb], ((uint32_t)(j >> 1) & 1u) ^ 1u);
      uint8_t* sP = smem + L::oP + pb * L::kPBytes;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {  // 16-byte chunk ch = keys [32ch, 32ch+32), SWIZZLE_64B
        const int phys = ch ^ ((r >> 1) & 3);
        *reinterpret_cast<uint4*>(sP + r * 64 + phys * 16) =
            make_uint4(packed[4 * ch], packed[4 * ch + 1], packed[4 * ch + 2], packed[4 * ch + 3]);
      }
      uint8_t* sPSF = smem + L::oPSF + pb * L::kPSF;
      const int sfo = (r & 31) * 16 + (r >> 5) * 4;
      *reinterpret_cast<uint32_t*>(sPSF + sfo) = scw0;
      *reinterpret_cast<uint32_t*>(sPSF + 512 + sfo) = scw1;
      const int slot = j & 3;
      xchg[slot * 256 + r] = alpha;
      xchg[slot * 256 + 128 + r] = sP1;
      fence_proxy_async_smem();
      mbar_arrive(&p_full[pb]);
      mbar_arrive(&x_full[slot]);
      m = m_new;
    }
    fin[r] = l;
    fin[128 + r] = m;
    if (a.lse != nullptr && q_row < a.N) a.lse[(int64_t)bh * a.N + q_row] = m * a.scale + logf(l);
    named_bar_sync(1, 256);
  } else {
    // -------------------------------------------------------------------- correction + epilogue
    setmaxnreg_inc232();
    const int r = threadIdx.x - 256;
    const int q_row = qt * 128 + r;
    const uint32_t lane_addr = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    float o[D];
#pragma unroll
    for (int c = 0; c < D; ++c) o[c] = 0.0f;
    for (int j = 0; j < nkv; ++j) {
      const int slot = j & 3;
      mbar_wait(&x_full[slot], (uint32_t)(j >> 2) & 1u);
      const float alpha = xchg[slot * 256 + r];
      const float sP1 = xchg[slot * 256 + 128 + r];
      mbar_wait(pv_full, (uint32_t)j & 1u);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(lane_addr + kColPV + 32 * c, v);
        tmem_ld_wait_regs(v);
#pragma unroll
        for (int i = 0; i < 32; ++i) o[32 * c + i] = fmaf(alpha, o[32 * c + i], sP1 * __uint_as_float(v[i]));
      }
      tc_fence_before();
      mbar_arrive(pv_empty);
    }
    named_bar_sync(1, 256);
    const float inv_l = 1.0f / fin[r];
    if (q_row < a.N) {
      const int b = bh / a.H, h = bh % a.H;
      if (a.o_dtype == 2) {
        float* dst = reinterpret_cast<float*>(a.o) + b * a.o_sb + h * a.o_sh + (int64_t)q_row * a.o_sn;
#pragma unroll
        for (int c = 0; c < D; c += 4)
          *reinterpret_cast<float4*>(dst + c) =
              make_float4(o[c] * inv_l, o[c + 1] * inv_l, o[c + 2] * inv_l, o[c + 3] * inv_l);
      } else if (a.o_dtype == 1) {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(a.o) + b * a.o_sb + h * a.o_sh + (int64_t)q_row * a.o_sn;
#pragma unroll
        for (int c = 0; c < D; c += 8) {
          uint4 u;
          __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
          for (int i = 0; i < 4; ++i) p[i] = __floats2bfloat162_rn(o[c + 2 * i] * inv_l, o[c + 2 * i + 1] * inv_l);
          *reinterpret_cast<uint4*>(dst + c) = u;
        }
      } else {
        __half* dst = reinterpret_cast<__half*>(a.o) + b * a.o_sb + h * a.o_sh + (int64_t)q_row * a.o_sn;
#pragma unroll
        for (int c = 0; c < D; c += 8) {
          uint4 u;
          __half2* p = reinterpret_cast<__half2*>(&u);
#pragma unroll
          for (int i = 0; i < 4; ++i) p[i] = __floats2half2_rn(o[c + 2 * i] * inv_l, o[c + 2 * i + 1] * inv_l);
          *reinterpret_cast<uint4*>(dst + c) = u;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
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
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t stream) {
  using L = Layout<D>;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = a.B * a.H;
  CUtensorMap tq, tk, tv;
  if (!make_map(&tq, a.q_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tk, a.k_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tv, a.v_data, (uint64_t)a.Np / 2, (uint64_t)BH * D, 64, D))
    return cudaErrorInvalidValue;
  dim3 grid(BH, a.Np / 128);
  attn_fwd_kernel<D><<<grid, kThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t stream) {
  return a.d == 128 ? launch_d<128>(a, stream) : launch_d<64>(a, stream);
}

}  // namespace sage3
