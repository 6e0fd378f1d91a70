// attn5.cu — sm_100a SageAttention3 FP4 attention forward with B_kv = 64 (Algorithm 1 with a 64-key KV block; the
// paper leaves B_q, B_kv free): three softmax warpgroups whose S buffers are independent of the PV path.
//
// attn3.cu (B_kv = 128) writes PV_j over S_j's TMEM columns, so S_{j+3} waits for the correction to read PV_j and the
// softmax warpgroups idle on that chain; a separate PV buffer does not fit next to three 128-column S buffers
// (attn4.cu).  With 64-key tiles it does:
//   TMEM: S buffers b = 0..2 (64 columns each, tile j -> j % 3 = the softmax warpgroup), PV slots p = 0, 1 (d columns,
//   tile j -> j % 2), scale factors s_Q (shared), s_K per S buffer, s_P2 / s_V per PV slot.
// so S_{j+3} is issued as soon as the warpgroup has read S_j, and PV_j / the correction run beside the softmax.
// The tile-local two-level quantization (reading c14) runs over 64 keys; the oracle runs the same Alg1 with
// bkv = 64 (parity tests).  Non-causal only (a causal 64-key tile can hold rows with no visible key).
//
// Hand-offs ("last arriver issues", acq_rel shared-memory counters; no thread waits to issue):
//   S_{j+3}: by the 4th softmax warp of the warpgroup done loading S_j (S_0..S_2: correction warp 1, prologue);
//   PV_j:    by the 4th softmax warp done with tile j, after the correction has read PV_{j-2} (pv_empty); the same
//            thread refills V̂_{j-2}'s ring slot (PV_{j-2} is complete) with V̂_{j-2+kVStages};
//   K ring:  softmax warp 1 of the warpgroup refills K̂_j's slot with K̂_{j+kKStages} once S_j has completed.
// Roles: WG0 = correction rows 32w.. (O in registers, the epilogue); WG1-3 = softmax of tiles j ≡ 0, 1, 2 (mod 3).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "attn_common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

#ifndef SAGE3_A5_POLY_MASK
#define SAGE3_A5_POLY_MASK 0x22  // exp2 pairs of each 16-key block on the FMA-pipe polynomial (1/4 of the exps)
#endif
#ifndef SAGE3_A5_REG_C
#define SAGE3_A5_REG_C 176
#define SAGE3_A5_REG_S 112
#endif
#ifndef SAGE3_A5_REG_C64
#define SAGE3_A5_REG_C64 128
#define SAGE3_A5_REG_S64 128
#endif
static_assert(SAGE3_A5_REG_C + 3 * SAGE3_A5_REG_S <= 512, "register budget");
static_assert(SAGE3_A5_REG_C64 + 3 * SAGE3_A5_REG_S64 <= 512, "register budget (d = 64)");

constexpr int kBkv = 64;
constexpr int kSBufs = 3, kPVBufs = 2;
constexpr int kSlots = 6;  // P̂2 smem buffers, exchange slots, PV hand-off counters (tile j -> j % 6)
constexpr int kKStages = 6, kVStages = 6;
constexpr int kThreads = 512;

template <int D>
struct Layout5 {
  static constexpr int kQKRow = D / 2;
  static constexpr int kQBytes = 128 * kQKRow;
  static constexpr int kKBytes = kBkv * kQKRow;                       // 64 K̂ rows
  static constexpr int kKSlot = ((kKBytes + 1023) / 1024) * 1024;
  static constexpr int kVBytes = D * 32;                              // Vᵀ tile: D channel rows x 64 tokens (32 B)
  static constexpr int kPBytes = 128 * 32;                            // P̂2: 128 rows x 64 keys (32 B)
  static constexpr int kQKSF = (D / 64) * 512;                        // the 128-row SF atoms holding the tile's rows
  static constexpr int kVSF = 512, kPSF = 512;                        // 64 tokens = 4 blocks: one atom
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + ((kQBytes + 1023) / 1024) * 1024;
  static constexpr int oV = oK + kKStages * kKSlot;
  static constexpr int oP = oV + kVStages * kVBytes;
  static constexpr int oQSF = oP + kSlots * kPBytes;
  static constexpr int oKSF = oQSF + kQKSF;
  static constexpr int oVSF = oKSF + kKStages * kQKSF;
  static constexpr int oPSF = oVSF + kVStages * kVSF;
  static constexpr int oXchg = oPSF + kSlots * kPSF;  // float [kSlots][2][128]: tmax_j, rowsum(P̃2_j)
  static constexpr int oBar = oXchg + kSlots * 2 * 128 * 4;
  static constexpr int kNumBars = 1 + kKStages + kVStages + kSBufs + 2 * kPVBufs + 3 * kSlots;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kBytes = oTmem + 16;
  static constexpr int kSmemAlloc = kBytes + 1024;
  // the O epilogue stages [128 rows][D fp32] over the K, V and P̂2 rings (contiguous, idle by then)
  static_assert(oQSF - oK >= D * 4 * 128, "O staging space");
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory");
};

// TMEM columns: S buffers 0..191, PV slots 192.. (D each), then the scale factors
template <int D>
struct Cols5 {
  static constexpr uint32_t kS = 0, kPV = 192;
  static constexpr uint32_t kSFQ = kPV + 2 * D;          // s_Q: D/64 atoms x 4 columns
  static constexpr uint32_t kSFK = kSFQ + 8;             // s_K: 8 columns per S buffer
  static constexpr uint32_t kSFP = kSFK + 8 * kSBufs;    // s_P2: 4 columns per PV slot
  static constexpr uint32_t kSFV = kSFP + 4 * kPVBufs;   // s_V: 4 columns per PV slot
  static_assert(kSFV + 4 * kPVBufs <= 512, "TMEM columns");
};

__device__ __forceinline__ void sts_v2_5(uint32_t saddr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(saddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acqrel_5(uint32_t saddr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(v) : "memory");
  return old;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn5_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                     const AttnArgs a) {
  using L = Layout5<D>;
  using C = Cols5<D>;
  constexpr uint32_t kRegC = D == 64 ? SAGE3_A5_REG_C64 : SAGE3_A5_REG_C;
  constexpr uint32_t kRegS = D == 64 ? SAGE3_A5_REG_S64 : SAGE3_A5_REG_S;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(1024) float2 s_lut[128];  // (-log2 s, s) per E4M3 scale code, as in attn.cu
  // hand-off counters: [0, 3) S issue per softmax warpgroup, [3, 9) PV issue per P̂2 slot
  __shared__ uint32_t cnt[16];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* v_full = k_full + kKStages;
  uint64_t* s_full = v_full + kVStages;   // S MMA -> softmax: S_j in buffer j%3
  uint64_t* pv_full = s_full + kSBufs;    // PV MMA -> correction: PV_j in slot j%2
  uint64_t* x_full = pv_full + kPVBufs;   // softmax -> correction: (tmax_j, rowsum) in slot j%6 (128 arrivals)
  uint64_t* x_empty = x_full + kSlots;    // correction -> softmax: slot j%6 read (4 warp arrivals)
  uint64_t* p_empty = x_empty + kSlots;   // PV MMA -> softmax: P̂2 buffer j%6 read
  uint64_t* pv_empty = p_empty + kSlots;  // correction -> PV issuer: PV slot j%2 read (4 warp arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = a.Np >> 7;
  const int64_t unit = a.unit_begin + (int64_t)blockIdx.x;
  const int bh = (int)(unit / n_qt);
  const int qt = n_qt - 1 - (int)(unit % n_qt);
  const int nkv = (a.N + kBkv - 1) / kBkv;  // non-causal: every 64-key tile up to the last real key

  auto load_k = [&](int j) {  // K̂ rows 64 j .. 64 j + 63 and the SF atoms of their 128-row chunk
    const int st = j % kKStages;
    const int row_k = bh * a.Np + j * kBkv;
    mbar_arrive_expect_tx(&k_full[st], L::kKBytes + L::kQKSF);
    tma_load_2d(smem + L::oK + st * L::kKSlot, &tm_k, &k_full[st], 0, row_k);
    bulk_load(smem + L::oKSF + st * L::kQKSF, a.k_sf + (int64_t)(row_k >> 7) * L::kQKSF, L::kQKSF, &k_full[st]);
  };
  auto load_v = [&](int j) {  // V̂ᵀ tokens 64 j .. 64 j + 63 (32 bytes of every channel row) and their SF atom
    const int st = j % kVStages;
    mbar_arrive_expect_tx(&v_full[st], L::kVBytes + L::kVSF);
    tma_load_2d(smem + L::oV + st * L::kVBytes, &tm_v, &v_full[st], j * 32, bh * D);
    bulk_load(smem + L::oVSF + st * L::kVSF, a.v_sf + ((int64_t)bh * n_qt + (j >> 1)) * 1024 + (j & 1) * 512, L::kVSF,
              &v_full[st]);
  };

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kKStages; ++s) mbar_init(&k_full[s], 1);
    for (int s = 0; s < kVStages; ++s) mbar_init(&v_full[s], 1);
    for (int b = 0; b < kSBufs; ++b) mbar_init(&s_full[b], 1);
    for (int p = 0; p < kPVBufs; ++p) {
      mbar_init(&pv_full[p], 1);
      mbar_init(&pv_empty[p], 4);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&x_full[s], 128);
      mbar_init(&x_empty[s], 4);
      mbar_init(&p_empty[s], 1);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    const int row_q = bh * a.Np + qt * 128;
    mbar_arrive_expect_tx(q_full, L::kQBytes + L::kQKSF);
    tma_load_2d(smem + L::oQ, &tm_q, q_full, 0, row_q);
    bulk_load(smem + L::oQSF, a.q_sf + (int64_t)(row_q >> 7) * L::kQKSF, L::kQKSF, q_full);
    for (int j = 0; j < nkv && j < kKStages; ++j) load_k(j);
    for (int j = 0; j < nkv && j < kVStages; ++j) load_v(j);
  }
  if (threadIdx.x < 16) cnt[threadIdx.x] = 0u;
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
  const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
  const float sl2 = a.scale * kLog2e;
  const uint32_t cnt_s = smem_u32(cnt);
  constexpr uint32_t kQKLayout = D == 128 ? kLayoutSw64 : kLayoutSw32;
  constexpr int kQKAtoms = L::kQKSF / 512;

  // S_j (M = 128, N = 64, K = d) into buffer j%3.  B = the 64 K̂ rows; their scales are columns 2(j%2), 2(j%2)+1 of
  // each 128-row SF atom (column c of an atom holds rows 32c..32c+31).
  auto issue_s = [&](int j) {
    const int b = j % kSBufs, st = j % kKStages;
    mbar_wait(&k_full[st], (uint32_t)(j / kKStages) & 1u);
    tc_fence_after();
    const uint8_t* sK = smem + L::oK + st * L::kKSlot;
    const uint8_t* sKSF = smem + L::oKSF + st * L::kQKSF;
#pragma unroll
    for (int at = 0; at < kQKAtoms; ++at)
      tmem_cp_32x128b_x4(tbase + C::kSFK + 8 * b + 4 * at, sf_desc(sKSF + 512 * at));
#pragma unroll
    for (int ks = 0; ks < D / 64; ++ks) {
      const uint64_t ad = make_smem_desc(smem_u32(smem + L::oQ) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
      const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
      mma_nvf4(tbase + C::kS + 64 * b, ad, bd, make_idesc_nvf4(128, kBkv), tbase + C::kSFQ + 4 * ks,
               tbase + C::kSFK + 8 * b + 4 * ks + 2 * (j & 1), ks > 0);
    }
    mma_commit(&s_full[b]);
  };
  // PV_j (M = 128, N = d, K = 64: one instruction) into slot j%2: A = P̂2_j (128 rows x 32 B), B = V̂ᵀ_j (d rows x
  // 32 B), both 32-byte-swizzled K-major; s_P2 / s_V into the slot's columns (its previous PV has been read).
  auto issue_pv = [&](int j) {
    const int p = j % kPVBufs, st = j % kVStages, ps = j % kSlots;
    mbar_wait(&v_full[st], (uint32_t)(j / kVStages) & 1u);
    tc_fence_after();
    tmem_cp_32x128b_x4(tbase + C::kSFP + 4 * p, sf_desc(smem + L::oPSF + ps * L::kPSF));
    tmem_cp_32x128b_x4(tbase + C::kSFV + 4 * p, sf_desc(smem + L::oVSF + st * L::kVSF));
    const uint64_t ad = make_smem_desc(smem_u32(smem + L::oP + ps * L::kPBytes), 16, 256, kLayoutSw32);
    const uint64_t bd = make_smem_desc(smem_u32(smem + L::oV + st * L::kVBytes), 16, 256, kLayoutSw32);
    mma_nvf4(tbase + C::kPV + D * p, ad, bd, make_idesc_nvf4(128, D), tbase + C::kSFP + 4 * p, tbase + C::kSFV + 4 * p,
             0);
    mma_commit(&p_empty[ps]);
    mma_commit(&pv_full[p]);
  };
  // PV_j is issued by the 4th softmax warp done with tile j, once the correction has read the slot's previous PV
  // (PV_{j-2}; the softmax warpgroups run ahead of the correction, so this wait is off their critical path); the
  // same thread refills V̂_{j-2}'s ring slot (PV_{j-2} is complete) with V̂_{j-2+kVStages}.  (Letting a correction warp
  // issue instead stalls its next TMEM load behind the MMA it issued.)
  auto pv_handoff = [&](int j) {
    uint32_t old = 0;
    if (lane == 0) old = atom_add_acqrel_5(cnt_s + 4 * (3 + j % kSlots), 1u);
    if ((__shfl_sync(0xffffffffu, old, 0) & 3u) == 3u) {
      if (elect_one()) {
        mbar_wait(&pv_empty[j % kPVBufs], ((uint32_t)(j / kPVBufs) & 1u) ^ 1u);
        tc_fence_after();
        issue_pv(j);
        if (j >= 2 && j - 2 + kVStages < nkv) load_v(j - 2 + kVStages);
      }
      __syncwarp();
    }
  };

  if (wg == 0) {
    // ====================================================================== correction
    setmaxnreg_inc<kRegC>();
    if (warp == 1) {  // s_Q once, then S_0..S_2 (the commit of S_0 covers the s_Q copy for every later S issuer)
      if (elect_one()) {
        mbar_wait(q_full, 0);
        tc_fence_after();
#pragma unroll
        for (int at = 0; at < kQKAtoms; ++at)
          tmem_cp_32x128b_x4(tbase + C::kSFQ + 4 * at, sf_desc(smem + L::oQSF + 512 * at));
        for (int j = 0; j < nkv && j < kSBufs; ++j) issue_s(j);
      }
      __syncwarp();
    }
    const int r = threadIdx.x;
    const int q_row = qt * 128 + r;
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    float mref = -INFINITY, l = 0.0f;
    f2 o[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = make_float2(0.f, 0.f);
    for (int j = 0; j < nkv; ++j) {
      const int xs = j % kSlots, p = j % kPVBufs;
      mbar_wait(&x_full[xs], (uint32_t)(j / kSlots) & 1u);
      const float tmax = lds_f32(xchg_s + xs * 1024);
      const float rs2 = lds_f32(xchg_s + xs * 1024 + 512);
      __syncwarp();
      if (lane == 0) mbar_arrive(&x_empty[xs]);
      const bool need = (tmax - mref) * sl2 > 8.0f;  // true on the first tile (mref = -inf)
      if (__any_sync(0xffffffffu, need)) {
        const float mnew = need ? tmax : mref;
        const float sc = ex2((mref - mnew) * sl2);
        const f2 sc2 = make_float2(sc, sc);
        l *= sc;
#pragma unroll
        for (int c = 0; c < D / 2; ++c) o[c] = fmul2(o[c], sc2);
        mref = mnew;
      }
      const float w = ex2((tmax - mref) * sl2 - kLog2_2688);
      l = fmaf(w, rs2, l);
      const f2 ww = make_float2(w, w);
      mbar_wait(&pv_full[p], (uint32_t)(j / kPVBufs) & 1u);
      tc_fence_after();
      const uint32_t pv_base = lane_base + C::kPV + D * p;
      auto acc = [&](int c, const uint32_t(&v)[16]) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          o[8 * c + i] = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), ww, o[8 * c + i]);
      };
      {  // PV_j in 16-column chunks, the next chunk's load in flight; the slot is handed on (PV_{j+2}) as soon as the
         // last chunk is in registers
        uint32_t va[16], vb[16];
        tmem_ld_cols(pv_base, va);
#pragma unroll
        for (int c = 0; c < D / 16; c += 2) {
          tmem_ld_wait_regs(va);
          tmem_ld_cols(pv_base + 16 * (c + 1), vb);
          acc(c, va);
          tmem_ld_wait_regs(vb);
          if (c + 2 < D / 16) {
            tmem_ld_cols(pv_base + 16 * (c + 2), va);
          } else {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&pv_empty[p]);
          }
          acc(c + 1, vb);
        }
      }
    }
    // Alg1 L13: O_i = diag(l)^-1 O_i
    if (a.lse != nullptr && q_row < a.N) a.lse[(int64_t)bh * a.N + q_row] = mref * a.scale + logf(l);
    const float inv_l = 1.0f / l;
    const f2 il{inv_l, inv_l};
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = fmul2(o[c], il);
    uint8_t* stage = smem + L::oK;
    stage_o_row<D>(stage, r, a.o_dtype, o);
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) store_o_tile<D>(&tm_o, stage, a.o_dtype, qt * 128, bh % a.H, bh / a.H);
  } else {
    // ====================================================================== softmax + two-level P quant (64 keys)
    setmaxnreg_dec<kRegS>();
    const int par = wg - 1;  // this warpgroup's tiles: j ≡ par (mod 3), S buffer par
    const int r = threadIdx.x - 128 * wg;
    const f2 sl2x2 = make_float2(sl2, sl2);
    const uint32_t s_addr = lane_base + C::kS + 64 * par;
    const uint32_t swz = (uint32_t)((r >> 2) & 1);  // 32-byte swizzle of P̂2 rows: chunk ^= (row >> 2) & 1
    auto tile = [&](const int j, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const int ps = j % kSlots;
      const uint32_t sP = smem_u32(smem + L::oP + ps * L::kPBytes) + r * 32;
      const uint32_t sPSF = smem_u32(smem + L::oPSF + ps * L::kPSF) + (r & 31) * 16 + (r >> 5) * 4;
      const uint32_t xchg_s = smem_u32(smem + L::oXchg) + ps * 1024 + r * 4;
      mbar_wait(&s_full[par], (uint32_t)(j / kSBufs) & 1u);
      tc_fence_after();
      if ((warp & 3) == 1 && j + kKStages < nkv) {  // S_j complete: K̂_j's slot is free
        if (elect_one()) load_k(j + kKStages);
        __syncwarp();
      }
      const int lim = a.N - 1 - j * kBkv;  // last real key in the tile
      // ---- pass 1: 16-key block maxima; masked keys -> -inf (written back to TMEM)
      float bmax[4];
      {
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(s_addr, va);
        tmem_ld_32x32b_x32(s_addr + 32, vb);
        tmem_ld_wait_regs(va);
        tmem_ld_wait_regs(vb);
        float* fa = reinterpret_cast<float*>(va);
        float* fb = reinterpret_cast<float*>(vb);
        if constexpr (masked) {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            fa[t] = (t > lim) ? -INFINITY : fa[t];
            fb[t] = (32 + t > lim) ? -INFINITY : fb[t];
          }
          tmem_st_32x32b_x32(s_addr, va);
          tmem_st_32x32b_x32(s_addr + 32, vb);
        }
        bmax[0] = max16(fa);
        bmax[1] = max16(fa + 16);
        bmax[2] = max16(fb);
        bmax[3] = max16(fb + 16);
      }
      const float tmax = fmax3(bmax[0], bmax[1], fmaxf(bmax[2], bmax[3]));
      const float nb = kLog2_2688 - tmax * sl2;
      if constexpr (masked) tmem_st_wait();
      uint32_t va[16], vb[16];
      tmem_ld_32x32b_x16(s_addr, va);
      float nbb[4], sdec[4];
      uint32_t scw;
      {
        const f2 e0 = ffma2(make_float2(bmax[0], bmax[1]), sl2x2, make_float2(nb, nb));
        const f2 e1 = ffma2(make_float2(bmax[2], bmax[3]), sl2x2, make_float2(nb, nb));
        const f2 q0 = fmul2(make_float2(ex2(e0.x), ex2(e0.y)), make_float2(kOneSixth, kOneSixth));
        const f2 q1 = fmul2(make_float2(ex2(e1.x), ex2(e1.y)), make_float2(kOneSixth, kOneSixth));
        scw = __byte_perm(cvt_e4m3x2(q0.x, q0.y), cvt_e4m3x2(q1.x, q1.y), 0x5410);
#pragma unroll
        for (int blk = 0; blk < 4; ++blk) {
          const float2 t = s_lut[(scw >> (8 * blk)) & 0xFFu];
          nbb[blk] = nb + t.x;
          sdec[blk] = t.y;
        }
      }
      mbar_wait(&p_empty[ps], ((uint32_t)(j / kSlots) & 1u) ^ 1u);  // PV_{j-6} has read this P̂2 buffer
      float rowsum = 0.0f;
      auto block = [&](int blk, const uint32_t(&v)[16]) {
        f2 y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const f2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2x2,
                             make_float2(nbb[blk], nbb[blk]));
          y[i] = ((SAGE3_A5_POLY_MASK >> i) & 1u) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        }
        const f2 s01 = fadd2(fadd2(y[0], y[1]), fadd2(y[2], y[3]));
        const f2 s23 = fadd2(fadd2(y[4], y[5]), fadd2(y[6], y[7]));
        const f2 sy = fadd2(s01, s23);
        rowsum = fmaf(sdec[blk], sy.x + sy.y, rowsum);
        const uint32_t w0 = cvt_e2m1x8(y[0].x, y[0].y, y[1].x, y[1].y, y[2].x, y[2].y, y[3].x, y[3].y);
        const uint32_t w1 = cvt_e2m1x8(y[4].x, y[4].y, y[5].x, y[5].y, y[6].x, y[6].y, y[7].x, y[7].y);
        // 16-byte chunk blk/2 = keys [32 (blk/2), +32) of row r, 32-byte swizzle
        sts_v2_5(sP + ((((uint32_t)blk >> 1) ^ swz) * 16) + (blk & 1) * 8, w0, w1);
      };
#pragma unroll
      for (int blk = 0; blk < 4; blk += 2) {
        tmem_ld_wait_regs(va);
        tmem_ld_32x32b_x16(s_addr + 16 * (blk + 1), vb);
        block(blk, va);
        tmem_ld_wait_regs(vb);
        if (blk + 2 < 4) {
          tmem_ld_32x32b_x16(s_addr + 16 * (blk + 2), va);
        } else if (j + kSBufs < nkv) {  // S_j is read: the 4th warp issues S_{j+3} into the buffer
          tc_fence_before();
          __syncwarp();
          uint32_t old = 0;
          if (lane == 0) old = atom_add_acqrel_5(cnt_s + 4 * par, 1u);
          if ((__shfl_sync(0xffffffffu, old, 0) & 3u) == 3u) {
            if (elect_one()) {
              tc_fence_after();
              issue_s(j + kSBufs);
            }
            __syncwarp();
          }
        }
        block(blk + 1, vb);
      }
      sts_u32(sPSF, scw);
      mbar_wait(&x_empty[ps], ((uint32_t)(j / kSlots) & 1u) ^ 1u);  // the correction has read tile j-6's slot
      sts_f32(xchg_s, tmax);
      sts_f32(xchg_s + 512, rowsum);
      tc_fence_before();
      fence_proxy_async_smem();
      mbar_arrive(&x_full[ps]);
      __syncwarp();
      pv_handoff(j);
    };
    const int last = nkv - 1;
    const bool last_masked = (last + 1) * kBkv > a.N;
    int j = par;
    for (; j < last; j += kSBufs) tile(j, std::false_type{});
    if (j == last) {
      if (last_masked)
        tile(last, std::true_type{});
      else
        tile(last, std::false_type{});
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// 2D uint8 map with an explicit swizzle (the V̂ᵀ tiles of this kernel are 32-byte boxes)
bool make_map_sw(CUtensorMap* m, const void* base, uint64_t row_bytes, uint64_t rows, uint32_t box_bytes,
                 uint32_t box_rows, CUtensorMapSwizzle swz) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t es[2] = {1, 1};
  return encode_tiled_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
cudaError_t launch5(const AttnArgs& a, cudaStream_t stream) {
  using L = Layout5<D>;
  static std::atomic<bool> attr_done[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn5_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = a.B * a.H;
  CUtensorMap tq, tk, tv, to;
  if (!make_map(&tq, a.q_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tk, a.k_data, D / 2, (uint64_t)BH * a.Np, D / 2, kBkv) ||
      !make_map_sw(&tv, a.v_data, (uint64_t)a.Np / 2, (uint64_t)BH * D, 32, D, CU_TENSOR_MAP_SWIZZLE_32B) ||
      !make_map_o(&to, a.o, a.o_dtype, a.B, a.H, a.N, D, a.o_sb, a.o_sh, a.o_sn))
    return cudaErrorInvalidValue;
  const int64_t units = a.unit_end - a.unit_begin;
  if (units <= 0) return cudaSuccess;
  attn5_fwd_kernel<D><<<(unsigned)units, kThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

}  // namespace

bool attention5_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SAGE3_ATTN_KERNEL");
    return e != nullptr && e[0] == '5';
  }();
  return on;
}

cudaError_t launch_attention5(const AttnArgs& a, cudaStream_t stream) {
  return a.d == 128 ? launch5<128>(a, stream) : launch5<64>(a, stream);
}

}  // namespace sage3
