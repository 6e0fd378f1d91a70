// attn4.cu — sm_100a SageAttention3 FP4 attention forward, three softmax warpgroups and a separate PV accumulator
// buffer: Algorithm 1 L6-L13, the same arithmetic as attn.cu / attn3.cu (tile-local two-level
// P, reading c14).
//
// attn3.cu writes PV_j over S_j's TMEM columns, so S_{j+3} (same buffer) waits until the correction has read PV_j:
// every softmax warpgroup's tile cycle is softmax + PV issue + PV MMA + correction + S issue + S MMA, and the
// softmax warps idle ~25% of the time (ncu).  Here PV_j goes to its own 64-column TMEM buffer, so the S buffer is free
// as soon as the softmax has read S_j, and the PV / correction path runs beside the softmax instead of inside its
// cycle:
//   TMEM: S buffers b = 0..2 at columns 128 b (tile j -> j % 3), the PV buffer at 384..447, scale factors 448..495.
//   d = 128: PV_j is two N = 64 MMAs through the 64-column buffer (O columns 0-63, then 64-127; the second is issued
//   once the correction has read the first).
// Hand-offs (no thread waits to issue; the last warp to complete a hand-off issues, shared-memory acq_rel counters):
//   S_{j+3} (N = 128, into buffer j % 3): by the 4th softmax warp of the warpgroup done loading S_j (S_0..S_2 by
//            correction warp 1 in the prologue);
//   PV_j half 0: by the 8th of {4 softmax warps done with tile j, 4 correction warps done reading PV_{j-1}}; the
//            same thread refills the V ring slot of V̂_{j-1} (PV_{j-1} is complete) with V̂_{j-1+kVStages};
//   PV_j half 1 (d = 128): by the 4th correction warp done reading half 0.
//   K ring: softmax warp 1 of the warpgroup refills K̂_j's slot with K̂_{j+kKStages} once S_j has completed.
// Roles: WG0 (warps 0-3) = correction rows 32w..32w+31 (O in registers, Alg1 L9-L11, L13, the epilogue);
// WG1-3 = softmax + two-level P quantization of tiles j ≡ 0, 1, 2 (mod 3), one query row per thread.
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

#ifndef SAGE3_A4_POLY_MASK
#define SAGE3_A4_POLY_MASK 0x22  // exp2 pairs of each 16-key block on the FMA-pipe polynomial (1/4 of the exps)
#endif
#ifndef SAGE3_A4_REG_C
#define SAGE3_A4_REG_C 176
#define SAGE3_A4_REG_S 112
#endif
#ifndef SAGE3_A4_REG_C64
#define SAGE3_A4_REG_C64 128
#define SAGE3_A4_REG_S64 128
#endif
static_assert(SAGE3_A4_REG_C + 3 * SAGE3_A4_REG_S <= 512, "register budget");
static_assert(SAGE3_A4_REG_C64 + 3 * SAGE3_A4_REG_S64 <= 512, "register budget (d = 64)");

constexpr int kBufs = 3;          // TMEM S buffers = softmax warpgroups
constexpr int kSlots = 6;         // P̂2 smem buffers, exchange slots, PV hand-off counters (tile j -> j % 6)
constexpr int kKStages = 6, kVStages = 5;
constexpr int kThreads = 512;
// TMEM columns
constexpr uint32_t kColPV = 384;                                   // PV buffer, 64 columns
constexpr uint32_t kSFQ = 448, kSFK = 456, kSFP = 480, kSFV = 488;  // s_Q (8), s_K per S buffer (3 x 8), s_P2, s_V

template <int D>
struct Layout4 {
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
  static constexpr int oV = oK + kKStages * kKSlot;
  static constexpr int oP = oV + kVStages * kVBytes;
  static constexpr int oQSF = oP + kSlots * kPBytes;
  static constexpr int oKSF = oQSF + kQKSF;
  static constexpr int oVSF = oKSF + kKStages * kQKSF;
  static constexpr int oPSF = oVSF + kVStages * kVSF;
  static constexpr int oXchg = oPSF + kSlots * kPSF;  // float [kSlots][2][128]: tmax_j, rowsum(P̃2_j)
  static constexpr int oBar = oXchg + kSlots * 2 * 128 * 4;
  static constexpr int kNumBars = 1 + kKStages + kVStages + kBufs + 1 + 3 * kSlots;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kBytes = oTmem + 16;
  static constexpr int kSmemAlloc = kBytes + 1024;
  static_assert(oP - oK >= D * 4 * 128, "O staging space");
  static_assert(kSmemAlloc <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ void sts_v2_(uint32_t saddr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(saddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acqrel_(uint32_t saddr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(v) : "memory");
  return old;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn4_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                     const AttnArgs a) {
  using L = Layout4<D>;
  constexpr uint32_t kRegC = D == 64 ? SAGE3_A4_REG_C64 : SAGE3_A4_REG_C;
  constexpr uint32_t kRegS = D == 64 ? SAGE3_A4_REG_S64 : SAGE3_A4_REG_S;
  constexpr int kHalves = D / 64;  // PV MMAs per tile through the 64-column PV buffer
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(1024) float2 s_lut[128];  // (-log2 s, s) per E4M3 scale code, as in attn.cu
  // hand-off counters: [0, 3) S issue per softmax warpgroup, [3, 9) PV issue per slot, 9: PV half 1 issue
  __shared__ uint32_t cnt[16];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* v_full = k_full + kKStages;
  uint64_t* s_full = v_full + kVStages;  // S MMA -> softmax: S_j in buffer j%3
  uint64_t* pv_full = s_full + kBufs;     // PV MMA -> correction: one phase per PV MMA (kHalves per tile)
  uint64_t* x_full = pv_full + 1;         // softmax -> correction: (tmax_j, rowsum) in slot j%6 (128 arrivals)
  uint64_t* x_empty = x_full + kSlots;    // correction -> softmax: slot j%6 read (4 warp arrivals)
  uint64_t* p_empty = x_empty + kSlots;   // PV MMA -> softmax: P̂2 buffer j%6 read
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_qt = a.Np >> 7;
  const int64_t unit = a.unit_begin + (int64_t)blockIdx.x;
  const int bh = (int)(unit / n_qt);
  const int qt = n_qt - 1 - (int)(unit % n_qt);  // descending within a head (longest first under causal masking)
  const int nkv = a.causal ? qt + 1 : n_qt;

  auto load_k = [&](int j) {
    const int st = j % kKStages;
    const int row_k = bh * a.Np + j * 128;
    mbar_arrive_expect_tx(&k_full[st], L::kKBytes + L::kQKSF);
    tma_load_2d(smem + L::oK + st * L::kKSlot, &tm_k, &k_full[st], 0, row_k);
    bulk_load(smem + L::oKSF + st * L::kQKSF, a.k_sf + (int64_t)(row_k >> 7) * L::kQKSF, L::kQKSF, &k_full[st]);
  };
  auto load_v = [&](int j) {
    const int st = j % kVStages;
    mbar_arrive_expect_tx(&v_full[st], L::kVBytes + L::kVSF);
    tma_load_2d(smem + L::oV + st * L::kVBytes, &tm_v, &v_full[st], j * 64, bh * D);
    bulk_load(smem + L::oVSF + st * L::kVSF, a.v_sf + ((int64_t)bh * n_qt + j) * L::kVSF, L::kVSF, &v_full[st]);
  };

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kKStages; ++s) mbar_init(&k_full[s], 1);
    for (int s = 0; s < kVStages; ++s) mbar_init(&v_full[s], 1);
    for (int b = 0; b < kBufs; ++b) mbar_init(&s_full[b], 1);
    mbar_init(pv_full, 1);
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
  // PV_0 has no PV_{-1} to wait for: its counter starts with the four correction arrivals
  if (threadIdx.x < 16) cnt[threadIdx.x] = threadIdx.x == 3 ? 4u : 0u;
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x >= 128 && threadIdx.x < 256) {  // (-log2 s, s) of every E4M3 scale code; s = 0 -> (10, 2^-10)
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

  // S_j = FP4MM(Q̂_i, s_Q, K̂_j, s_K) into buffer j%3 (the buffer's previous S has been read).  s_K goes to the
  // buffer's own columns (issuers differ); s_Q was copied once, before S_0, by the prologue issuer.
  auto issue_s = [&](int j) {
    const int b = j % kBufs, st = j % kKStages;
    mbar_wait(&k_full[st], (uint32_t)(j / kKStages) & 1u);
    tc_fence_after();
    const uint8_t* sK = smem + L::oK + st * L::kKSlot;
    const uint8_t* sKSF = smem + L::oKSF + st * L::kQKSF;
#pragma unroll
    for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kSFK + 8 * b + 4 * at, sf_desc(sKSF + 512 * at));
#pragma unroll
    for (int ks = 0; ks < D / 64; ++ks) {
      const uint64_t ad = make_smem_desc(smem_u32(smem + L::oQ) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
      const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
      mma_nvf4(tbase + 128 * b, ad, bd, make_idesc_nvf4(128, 128), tbase + kSFQ + 4 * ks, tbase + kSFK + 8 * b + 4 * ks,
               ks > 0);
    }
    mma_commit(&s_full[b]);
  };
  // PV_j half h = FP4MM(P̂2_j, s_P2, V̂_j rows 64h.., s_V) into the PV buffer (O columns 64h..64h+63).  Half 0 copies
  // s_P2 and s_V (the previous PV MMA has completed: the correction has read it); half 1 reuses them (issued after
  // half 0 completed, which orders the copies for its issuer).  B rows 64h.. = V̂ᵀ channel rows; their scales are
  // SF-atom columns 2h, 2h+1 (column c of an atom holds rows 32c..32c+31).
  auto issue_pv = [&](int j, int h) {
    const int st = j % kVStages, ps = j % kSlots;
    if (h == 0) mbar_wait(&v_full[st], (uint32_t)(j / kVStages) & 1u);
    tc_fence_after();
    const uint8_t* sP = smem + L::oP + ps * L::kPBytes;
    const uint8_t* sV = smem + L::oV + st * L::kVBytes;
    if (h == 0) {
      const uint8_t* sPSF = smem + L::oPSF + ps * L::kPSF;
      const uint8_t* sVSF = smem + L::oVSF + st * L::kVSF;
#pragma unroll
      for (int at = 0; at < 2; ++at) {
        tmem_cp_32x128b_x4(tbase + kSFP + 4 * at, sf_desc(sPSF + 512 * at));
        tmem_cp_32x128b_x4(tbase + kSFV + 4 * at, sf_desc(sVSF + 512 * at));
      }
    }
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
      const uint64_t bd = make_smem_desc(smem_u32(sV) + 64 * 64 * h + 32 * ks, 16, 512, kLayoutSw64);
      mma_nvf4(tbase + kColPV, ad, bd, make_idesc_nvf4(128, 64), tbase + kSFP + 4 * ks,
               tbase + kSFV + 4 * ks + 2 * h, ks > 0);
    }
    if (h == kHalves - 1) mma_commit(&p_empty[ps]);
    mma_commit(pv_full);
  };
  // one arrival of this warp on PV_j's hand-off counter; the 8th issues PV_j (half 0) and refills V̂_{j-1}'s slot
  auto pv_handoff = [&](int j) {
    if (j >= nkv) return;
    uint32_t old = 0;
    if (lane == 0) old = atom_add_acqrel_(cnt_s + 4 * (3 + j % kSlots), 1u);
    if ((__shfl_sync(0xffffffffu, old, 0) & 7u) == 7u) {
      if (elect_one()) {
        issue_pv(j, 0);
        if (j >= 1 && j - 1 + kVStages < nkv) load_v(j - 1 + kVStages);
      }
      __syncwarp();
    }
  };

  if (wg == 0) {
    // ====================================================================== correction
    setmaxnreg_inc<kRegC>();
    if (warp == 1) {  // s_Q, then S_0..S_2 (the commit of S_0 covers the s_Q copy for every later S issuer)
      if (elect_one()) {
        mbar_wait(q_full, 0);
        tc_fence_after();
#pragma unroll
        for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kSFQ + 4 * at, sf_desc(smem + L::oQSF + 512 * at));
        for (int j = 0; j < nkv && j < kBufs; ++j) issue_s(j);
      }
      __syncwarp();
    }
    // O and l relative to a lazily moved per-row reference mref (as attn.cu): tile j enters with weight
    // w_j = 2^{sl2 (tmax_j − mref)} / 2688 (= s_P1 · Π α relative to mref).
    const int r = threadIdx.x;
    const int q_row = qt * 128 + r;
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    const uint32_t pv_base = lane_base + kColPV;
    float mref = -INFINITY, l = 0.0f;
    f2 o[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = make_float2(0.f, 0.f);
    uint32_t pv_phase = 0;
    for (int j = 0; j < nkv; ++j) {
      const int xs = j % kSlots;
      mbar_wait(&x_full[xs], (uint32_t)(j / kSlots) & 1u);
      const float tmax = lds_f32(xchg_s + xs * 1024);
      const float rs2 = lds_f32(xchg_s + xs * 1024 + 512);
      __syncwarp();
      if (lane == 0) mbar_arrive(&x_empty[xs]);
      const bool need = (tmax - mref) * sl2 > 8.0f;  // true on the first tile (mref = -inf)
      if (__any_sync(0xffffffffu, need)) {
        const float mnew = need ? tmax : mref;
        const float sc = ex2((mref - mnew) * sl2);  // 0 on the first tile, 1 for rows that keep mref
        const f2 sc2 = make_float2(sc, sc);
        l *= sc;
#pragma unroll
        for (int c = 0; c < D / 2; ++c) o[c] = fmul2(o[c], sc2);
        mref = mnew;
      }
      const float w = ex2((tmax - mref) * sl2 - kLog2_2688);
      l = fmaf(w, rs2, l);
      const f2 ww = make_float2(w, w);
#pragma unroll
      for (int h = 0; h < kHalves; ++h) {
        mbar_wait(pv_full, pv_phase);
        pv_phase ^= 1u;
        tc_fence_after();
        // O columns 64h..64h+63 in 16-column chunks, the next chunk's load in flight during this chunk's FFMA2s
        uint32_t va[16], vb[16];
        tmem_ld_cols(pv_base, va);
#pragma unroll
        for (int c = 0; c < 4; c += 2) {
          tmem_ld_wait_regs(va);
          tmem_ld_cols(pv_base + 16 * (c + 1), vb);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            o[32 * h + 8 * c + i] =
                ffma2(make_float2(__uint_as_float(va[2 * i]), __uint_as_float(va[2 * i + 1])), ww, o[32 * h + 8 * c + i]);
          tmem_ld_wait_regs(vb);
          if (c + 2 < 4) {
            tmem_ld_cols(pv_base + 16 * (c + 2), va);
          } else {  // the PV buffer is read: hand it on (half 1 of this tile, or PV_{j+1})
            tc_fence_before();
            __syncwarp();
            if (h + 1 < kHalves) {
              uint32_t old = 0;
              if (lane == 0) old = atom_add_acqrel_(cnt_s + 4 * 9, 1u);
              if ((__shfl_sync(0xffffffffu, old, 0) & 3u) == 3u) {
                if (elect_one()) issue_pv(j, h + 1);
                __syncwarp();
              }
            } else {
              pv_handoff(j + 1);
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
            o[32 * h + 8 * (c + 1) + i] = ffma2(make_float2(__uint_as_float(vb[2 * i]), __uint_as_float(vb[2 * i + 1])),
                                                ww, o[32 * h + 8 * (c + 1) + i]);
        }
      }
    }
    // Alg1 L13: O_i = diag(l)^-1 O_i
    if (a.lse != nullptr && q_row < a.N) a.lse[(int64_t)bh * a.N + q_row] = mref * a.scale + logf(l);
    const float inv_l = 1.0f / l;
    const f2 il{inv_l, inv_l};
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = fmul2(o[c], il);
    // coalesced store: rows -> smem (the K/V rings, idle once the last PV MMA has completed) -> TMA
    uint8_t* stage = smem + L::oK;
    stage_o_row<D>(stage, r, a.o_dtype, o);
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    if (threadIdx.x == 0) store_o_tile<D>(&tm_o, stage, a.o_dtype, qt * 128, bh % a.H, bh / a.H);
  } else {
    // ====================================================================== softmax + two-level P quant
    setmaxnreg_dec<kRegS>();
    const int par = wg - 1;  // this warpgroup's tiles: j ≡ par (mod 3), S buffer par
    const int r = threadIdx.x - 128 * wg;
    const int q_row = qt * 128 + r;
    const f2 sl2x2 = make_float2(sl2, sl2);
    const uint32_t s_addr = lane_base + 128 * par;
    const uint32_t swz = (uint32_t)((r >> 1) & 3);
    auto tile = [&](const int j, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const int ps = j % kSlots;
      const uint32_t sP = smem_u32(smem + L::oP + ps * L::kPBytes) + r * 64;
      const uint32_t sPSF = smem_u32(smem + L::oPSF + ps * L::kPSF) + (r & 31) * 16 + (r >> 5) * 4;
      const uint32_t xchg_s = smem_u32(smem + L::oXchg) + ps * 1024 + r * 4;
      mbar_wait(&s_full[par], (uint32_t)(j / kBufs) & 1u);
      tc_fence_after();
      // K ring refill, no waiting: S_j has completed, so K̂_j's slot is free for K̂_{j+kKStages}
      if ((warp & 3) == 1 && j + kKStages < nkv) {
        if (elect_one()) load_k(j + kKStages);
        __syncwarp();
      }
      const int kv0 = j * 128;
      const int lim = a.causal ? min(a.N - 1, q_row) - kv0 : a.N - 1 - kv0;  // last visible key in the tile
      // ---- pass 1: 16-key block maxima of S (reused for the row max and for s_P2); masked keys -> -inf,
      //      written back to TMEM so pass 2 needs no masking.  Two 32-column loads in flight at a time.
      float bmax[8];
      auto pass1 = [&](int c, uint32_t(&v)[32]) {
        float* f = reinterpret_cast<float*>(v);
        if constexpr (masked) {
#pragma unroll
          for (int t = 0; t < 32; ++t) f[t] = (32 * c + t > lim) ? -INFINITY : f[t];
          tmem_st_32x32b_x32(s_addr + 32 * c, v);
        }
        bmax[2 * c] = max16(f);
        bmax[2 * c + 1] = max16(f + 16);
      };
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(s_addr + 64 * h, va);
        tmem_ld_32x32b_x32(s_addr + 64 * h + 32, vb);
        tmem_ld_wait_regs(va);
        tmem_ld_wait_regs(vb);
        pass1(2 * h, va);
        pass1(2 * h + 1, vb);
      }
      const float tmax = fmax3(fmax3(bmax[0], bmax[1], bmax[2]), fmax3(bmax[3], bmax[4], bmax[5]),
                               fmaxf(bmax[6], bmax[7]));
      const float nb = kLog2_2688 - tmax * sl2;  // P̃2 = 2^(S·sl2 + nb)
      if constexpr (masked) tmem_st_wait();
      uint32_t va[16], vb[16];
      tmem_ld_32x32b_x16(s_addr, va);  // pass-2 block 0, overlapped with the block-scale math below
      // ---- block scales of φ(P̃2) (as attn.cu): amax_blk = 2^(bmax·sl2 + nb), s = E4M3(amax/6), two blocks per
      //      convert; pass 2 produces y = P̃2/s = 2^(S·sl2 + nb - log2 s) with (-log2 s, s) from the table.
      float nbb[8], sdec[8];
      uint32_t scw[2];
      {
        uint32_t c2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const f2 e = ffma2(make_float2(bmax[2 * k], bmax[2 * k + 1]), sl2x2, make_float2(nb, nb));
          const f2 q = fmul2(make_float2(ex2(e.x), ex2(e.y)), make_float2(kOneSixth, kOneSixth));
          c2[k] = cvt_e4m3x2(q.x, q.y);  // block 2k in the low byte
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
      mbar_wait(&p_empty[ps], ((uint32_t)(j / kSlots) & 1u) ^ 1u);  // PV_{j-6} has read this P̂2 buffer
      // ---- pass 2 per 16-key block: y = P̃2/s, codes E2M1(y), rowsum(P̃2) = Σ_blk s_blk·Σy; the next block's
      //      TMEM load is in flight while this block is computed.
      float rowsum = 0.0f;
      auto block = [&](int blk, const uint32_t(&v)[16]) {
        f2 y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const f2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2x2,
                             make_float2(nbb[blk], nbb[blk]));
          y[i] = ((SAGE3_A4_POLY_MASK >> i) & 1u) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        }
        const f2 s01 = fadd2(fadd2(y[0], y[1]), fadd2(y[2], y[3]));
        const f2 s23 = fadd2(fadd2(y[4], y[5]), fadd2(y[6], y[7]));
        const f2 sy = fadd2(s01, s23);
        rowsum = fmaf(sdec[blk], sy.x + sy.y, rowsum);
        const uint32_t w0 = cvt_e2m1x8(y[0].x, y[0].y, y[1].x, y[1].y, y[2].x, y[2].y, y[3].x, y[3].y);
        const uint32_t w1 = cvt_e2m1x8(y[4].x, y[4].y, y[5].x, y[5].y, y[6].x, y[6].y, y[7].x, y[7].y);
        // 16-byte chunk blk/2 = keys [32 (blk/2), +32) of row r, SWIZZLE_64B (chunk ^= (row>>1)&3)
        sts_v2_(sP + ((((uint32_t)blk >> 1) ^ swz) * 16) + (blk & 1) * 8, w0, w1);
      };
#pragma unroll
      for (int blk = 0; blk < 8; blk += 2) {
        tmem_ld_wait_regs(va);
        tmem_ld_32x32b_x16(s_addr + 16 * (blk + 1), vb);
        block(blk, va);
        tmem_ld_wait_regs(vb);
        if (blk + 2 < 8) {
          tmem_ld_32x32b_x16(s_addr + 16 * (blk + 2), va);
        } else if (j + kBufs < nkv) {  // S_j is read: the 4th warp issues S_{j+3} into the buffer
          tc_fence_before();
          __syncwarp();
          uint32_t old = 0;
          if (lane == 0) old = atom_add_acqrel_(cnt_s + 4 * par, 1u);
          if ((__shfl_sync(0xffffffffu, old, 0) & 3u) == 3u) {
            if (elect_one()) {
              tc_fence_after();
              issue_s(j + kBufs);
            }
            __syncwarp();
          }
        }
        block(blk + 1, vb);
      }
      sts_u32(sPSF, scw[0]);
      sts_u32(sPSF + 512, scw[1]);
      mbar_wait(&x_empty[ps], ((uint32_t)(j / kSlots) & 1u) ^ 1u);  // the correction has read tile j-6's slot
      sts_f32(xchg_s, tmax);
      sts_f32(xchg_s + 512, rowsum);
      tc_fence_before();
      fence_proxy_async_smem();
      mbar_arrive(&x_full[ps]);  // per thread: releases its own exchange-slot writes
      __syncwarp();
      pv_handoff(j);  // P̂2_j / s_P2 written (fenced for the async proxy): one of PV_j's eight arrivals
    };
    const int last = nkv - 1;
    const bool last_masked = last * 128 + 128 > a.N || a.causal;
    int j = par;
    for (; j < last; j += kBufs) tile(j, std::false_type{});
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

template <int D>
cudaError_t launch4(const AttnArgs& a, cudaStream_t stream) {
  using L = Layout4<D>;
  static std::atomic<bool> attr_done[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn4_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
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
  attn4_fwd_kernel<D><<<(unsigned)units, kThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

}  // namespace

bool attention4_enabled(int d) {
  static const bool on = [] {
    const char* e = std::getenv("SAGE3_ATTN_KERNEL");
    return e != nullptr && e[0] == '4';
  }();
  (void)d;
  return on;
}

cudaError_t launch_attention4(const AttnArgs& a, cudaStream_t stream) {
  return a.d == 128 ? launch4<128>(a, stream) : launch4<64>(a, stream);
}

}  // namespace sage3
