// attn3.cu — sm_100a SageAttention3 FP4 attention forward, three softmax warpgroups per CTA:
// Algorithm 1 L6-L13, the same arithmetic as attn.cu (tile-local two-level P, DESIGN.md
// reading c14), with a different warp layout.
//
// Why: attn.cu's softmax is latency-bound — two softmax warps per SM sub-partition cannot keep MUFU and the
// issue port busy through the pass-1 / block-scale chains (ncu: issue 63%, MUFU 56%).  The
// register file decides how many softmax warps fit: attn.cu spends one warpgroup (32 registers) on single-lane TMA
// and MMA issuers and one (192) on the correction.  Here the issue roles are folded into warps that would otherwise
// wait, which frees a warpgroup slot for a third softmax warpgroup (176 + 3 x 112 = 512 registers per lane slot).
//
// One CTA = one 128-row query tile Q_i of one (b,h); loop over 128-key tiles j (B_q = B_kv = 128).
//   WG0 (warps 0-3): correction rows 32w..32w+31 (O in registers, Alg1 L9-L11, L13, the epilogue); thread 0 also
//                    requests Q̂_i + s_Q and the first K̂ / V̂ᵀ tiles in the prologue; warp 2 allocates TMEM
//   WG1-3:           softmax + two-level P quantization of KV tiles j ≡ 0, 1, 2 (mod 3), one row per thread
//                    (TMEM lane = row).  Tile j lives in TMEM buffer j % 3 and P̂2 buffer j % 3, i.e. each
//                    softmax warpgroup always uses the same buffers.
// MMAs are issued on one lane by warps that would otherwise wait, with scale factors in the buffer's own TMEM
// columns (copies by different issuing threads never share columns):
//   S_j  = FP4MM(Q̂_i, s_Q, K̂_j, s_K)    (tcgen05.mma kind::mxf4nvf4, M=128 N=128 K=d): by warp 0 of the softmax
//                                         warpgroup, once the four correction warps have read PV_{j-3} (b_empty);
//   PV_j = FP4MM(P̂2_j, s_P2, V̂_j, s_V)  (M=128 N=d K=128, over S_j's TMEM columns): by the 4th softmax warp done
//                                         with tile j (shared-memory counter, acq_rel atomics).
// Per tile j the correction warps do O += w_j PV_j; warps 1 and 2 of the softmax warpgroup refill the K / V ring
// slots (tiles j + kKStages / j + 2) as soon as S_j is complete — the slot reuse is implied by the S/PV chain, so no
// ring has an "empty" barrier.  Measured alternatives (cycles per tile at N = 16K): refills on
// correction warps (the refilling warp falls ~3000 cycles behind and paces the chain) 2250; all issue roles on fixed
// correction warps (their per-tile loop serialises PV issue, O update and S issue) 2085; PV from warp 0 of each
// softmax warpgroup after waiting for the others (the leader lags its warpgroup) 1680; S by the 4th correction warp
// done with PV_{j-3} (a tcgen05.ld issued after a tcgen05.mma by the same warp waits for the MMA) 1880.
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

// exp2 pairs of each 16-key block on the FMA-pipe polynomial (bit i: pair i of 8); 1/4 of the exps
#ifndef SAGE3_A3_POLY_MASK
#define SAGE3_A3_POLY_MASK 0x22
#endif
#ifndef SAGE3_A3_REG_C  // correction + issuers / softmax registers per thread, d = 128
#define SAGE3_A3_REG_C 176
#define SAGE3_A3_REG_S 112
#endif
#ifndef SAGE3_A3_REG_C64  // d = 64 (O is 64 floats)
#define SAGE3_A3_REG_C64 128
#define SAGE3_A3_REG_S64 128
#endif
static_assert(SAGE3_A3_REG_C + 3 * SAGE3_A3_REG_S <= 512, "register budget");
static_assert(SAGE3_A3_REG_C64 + 3 * SAGE3_A3_REG_S64 <= 512, "register budget (d = 64)");

#ifndef SAGE3_A3_SPREAD
#define SAGE3_A3_SPREAD 0  // 1: the S-issuing warp of softmax warpgroup w sits on SM sub-partition w-1 (else 0)
#endif

constexpr int kBufs = 3;  // TMEM S/PV buffers = P̂2 smem buffers = exchange slots = softmax warpgroups
constexpr int kKStages = 6, kVStages = kBufs + 2;  // (the V refill of tile j + 2 reuses V̂_{j-3}'s slot)
constexpr int kThreads = 512;

template <int D>
struct Layout3 {
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
  static constexpr int oQSF = oP + kBufs * kPBytes;
  static constexpr int oKSF = oQSF + kQKSF;
  static constexpr int oVSF = oKSF + kKStages * kQKSF;
  static constexpr int oPSF = oVSF + kVStages * kVSF;
  static constexpr int oXchg = oPSF + kBufs * kPSF;  // float [kBufs][2][128]: tmax_j, rowsum(P̃2_j)
  static constexpr int oBar = oXchg + kBufs * 2 * 128 * 4;
  static constexpr int kNumBars = 1 + kKStages + kVStages + 4 * kBufs;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kBytes = oTmem + 16;
  static constexpr int kSmemAlloc = kBytes + 1024;
  // the O epilogue stages [128 rows][D fp32] over the K and V rings (idle by then)
  static_assert(oP - oK >= D * 4 * 128, "O staging space");
};

#ifdef SAGE3_TRACE
// Debug-only timeline (tools/trace_a3.py): clock64 stamps of tiles 8..39, [cta < 2][role][tile j][event], kept in
// shared memory during the kernel (a global store before an mbarrier release would delay the release) and copied to
// g_trace3 at the end.
__device__ unsigned long long g_trace3[2][10][128][8];
#define A3_TR(role, j, k)                                                                         \
  do {                                                                                            \
    if (blockIdx.x < 2 && (j) >= 8 && (j) < 40) s_tr[((role) * 32 + (j) - 8) * 8 + (k)] = clock64(); \
  } while (0)
#define A3_EV(tid, role, j, k)                 \
  do {                                         \
    if (threadIdx.x == (tid)) A3_TR(role, j, k); \
  } while (0)
// correction warp w, event e (0 start, 1 x ready, 2 PV ready, 3 done): role 8 + w / 2, slot 4 (w % 2) + e
#define A3_CW(j, e)                                         \
  do {                                                      \
    if (lane == 0) A3_TR(8 + warp / 2, j, 4 * (warp & 1) + (e)); \
  } while (0)
#else
#define A3_CW(j, e) \
  do {              \
  } while (0)
#define A3_EV(tid, role, j, k) \
  do {                         \
  } while (0)
#endif

// Waits on the S/PV chain (s_full, b_empty, x_full, pv_full).  0: try_wait with the library's suspend hint (sm100.cuh
// mbar_wait); 1: spin on test_wait; 2: try_wait without a hint (the hardware's default time limit).
#ifndef SAGE3_A3_WAIT
#define SAGE3_A3_WAIT 0
#endif
__device__ __forceinline__ void chain_wait(uint64_t* bar, uint32_t parity) {
#if SAGE3_A3_WAIT == 1
  while (!ptx::mbar_test_wait(bar, parity)) {
  }
#elif SAGE3_A3_WAIT == 2
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni WAIT_%=;\n\t}\n" ::"r"(ptx::smem_u32(bar)),
      "r"(parity)
      : "memory");
#else
  ptx::mbar_wait(bar, parity);
#endif
}

__device__ __forceinline__ void sts_v2(uint32_t saddr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(saddr), "r"(a), "r"(b) : "memory");
}

// Shared-memory counter add with acquire-release semantics at CTA scope (the "last arriver issues" hand-offs).
__device__ __forceinline__ uint32_t atom_add_acqrel(uint32_t saddr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(v) : "memory");
  return old;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn3_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                     const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                     const AttnArgs a) {
  using L = Layout3<D>;
  constexpr uint32_t kRegC = D == 64 ? SAGE3_A3_REG_C64 : SAGE3_A3_REG_C;
  constexpr uint32_t kRegS = D == 64 ? SAGE3_A3_REG_S64 : SAGE3_A3_REG_S;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(1024) float2 s_lut[128];  // (-log2 s, s) per E4M3 scale code, as in attn.cu
  __shared__ uint32_t cnt[2 * kBufs];
#ifdef SAGE3_TRACE
  __shared__ unsigned long long s_tr[10 * 32 * 8];
#endif  // per buffer: softmax warps done with tile j (0-2), correction warps (3-5)
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* v_full = k_full + kKStages;
  uint64_t* s_full = v_full + kVStages;  // S MMA -> softmax: S_j in buffer j%3
  uint64_t* pv_full = s_full + kBufs;     // PV MMA -> correction: PV_j in buffer j%3
  uint64_t* x_full = pv_full + kBufs;     // softmax -> correction: (tmax_j, rowsum) in slot j%3 (128 arrivals)
  uint64_t* b_empty = x_full + kBufs;     // correction -> S issuer: PV_j read, buffer j%3 free (4 warp arrivals)
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
    for (int b = 0; b < kBufs; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&pv_full[b], 1);
      mbar_init(&x_full[b], 128);
      mbar_init(&b_empty[b], 4);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    // the rings are empty: Q̂, the first K̂ and V̂ tiles are requested before the prologue's __syncthreads
    const int row_q = bh * a.Np + qt * 128;
    mbar_arrive_expect_tx(q_full, L::kQBytes + L::kQKSF);
    tma_load_2d(smem + L::oQ, &tm_q, q_full, 0, row_q);
    bulk_load(smem + L::oQSF, a.q_sf + (int64_t)(row_q >> 7) * L::kQKSF, L::kQKSF, q_full);
    for (int j = 0; j < nkv && j < kKStages; ++j) load_k(j);
    for (int j = 0; j < nkv && j < kVStages; ++j) load_v(j);
  }
  if (threadIdx.x < 2 * kBufs) cnt[threadIdx.x] = 0u;
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

  // MMA issue, by whichever warp completes a buffer's hand-off last ("last arriver issues": no thread waits for
  // the others).  Scale factors sit in per-buffer TMEM columns, so copies by different issuing threads never share
  // columns: s_Q 384 + 8b, s_K 408 + 8b, s_P2 432 + 8b, s_V 456 + 8b.  A buffer's columns are rewritten only after
  // the buffer's previous MMA has completed (its result was consumed).
  constexpr uint32_t kSFQ = 384, kSFK = 408, kSFP = 432, kSFV = 456;
  constexpr uint32_t kQKLayout = D == 128 ? kLayoutSw64 : kLayoutSw32;
  constexpr int kQKAtoms = L::kQKSF / 512;
  auto issue_s = [&](int j) {  // S_j = FP4MM(Q̂_i, s_Q, K̂_j, s_K) into buffer j%3, once PV_{j-3} has been read
    const int b = j % kBufs, st = j % kKStages;
    A3_EV(threadIdx.x, 5, j, 0);
    // s_K first (its columns belong to this buffer, whose previous S MMA has completed), so that only the MMAs
    // wait for the correction's release of the buffer
    mbar_wait(&k_full[st], (uint32_t)(j / kKStages) & 1u);
    A3_EV(threadIdx.x, 5, j, 2);
    tc_fence_after();
    const uint8_t* sK = smem + L::oK + st * L::kKSlot;
    const uint8_t* sKSF = smem + L::oKSF + st * L::kQKSF;
#pragma unroll
    for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kSFK + 8 * b + 4 * at, sf_desc(sKSF + 512 * at));
    chain_wait(&b_empty[b], ((uint32_t)(j / kBufs) & 1u) ^ 1u);
    A3_EV(threadIdx.x, 5, j, 1);
    tc_fence_after();
#pragma unroll
    for (int ks = 0; ks < D / 64; ++ks) {
      const uint64_t ad = make_smem_desc(smem_u32(smem + L::oQ) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
      const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
      mma_nvf4(tbase + 128 * b, ad, bd, make_idesc_nvf4(128, 128), tbase + kSFQ + 8 * b + 4 * ks,
               tbase + kSFK + 8 * b + 4 * ks, ks > 0);
    }
    mma_commit(&s_full[b]);
    A3_EV(threadIdx.x, 5, j, 3);
#if defined(SAGE3_TRACE) && defined(SAGE3_TRACE_MMA)
    chain_wait(&s_full[b], (uint32_t)(j / kBufs) & 1u);  // diagnostics only: MMA completion time
    A3_EV(threadIdx.x, 5, j, 4);
#endif
  };
  auto issue_pv = [&](int j) {  // PV_j = FP4MM(P̂2_j, s_P2, V̂_j, s_V) over S_j's columns (S_j has been read)
    const int b = j % kBufs, st = j % kVStages;
    A3_EV(threadIdx.x, 6, j, 0);
    mbar_wait(&v_full[st], (uint32_t)(j / kVStages) & 1u);
    A3_EV(threadIdx.x, 6, j, 2);
    tc_fence_after();
    const uint8_t* sP = smem + L::oP + b * L::kPBytes;
    const uint8_t* sV = smem + L::oV + st * L::kVBytes;
    const uint8_t* sPSF = smem + L::oPSF + b * L::kPSF;
    const uint8_t* sVSF = smem + L::oVSF + st * L::kVSF;
#pragma unroll
    for (int at = 0; at < 2; ++at) {
      tmem_cp_32x128b_x4(tbase + kSFP + 8 * b + 4 * at, sf_desc(sPSF + 512 * at));
      tmem_cp_32x128b_x4(tbase + kSFV + 8 * b + 4 * at, sf_desc(sVSF + 512 * at));
    }
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
      const uint64_t bd = make_smem_desc(smem_u32(sV) + 32 * ks, 16, 512, kLayoutSw64);
      mma_nvf4(tbase + 128 * b, ad, bd, make_idesc_nvf4(128, D), tbase + kSFP + 8 * b + 4 * ks,
               tbase + kSFV + 8 * b + 4 * ks, ks > 0);
    }
    mma_commit(&pv_full[b]);
    A3_EV(threadIdx.x, 6, j, 3);
#if defined(SAGE3_TRACE) && defined(SAGE3_TRACE_MMA)
    chain_wait(&pv_full[b], (uint32_t)(j / kBufs) & 1u);  // diagnostics only: MMA completion time
    A3_EV(threadIdx.x, 6, j, 1);
#endif
  };
  const uint32_t cnt_s = smem_u32(cnt);

  if (wg == 0) {
    // ====================================================================== correction + TMA producers
    setmaxnreg_inc<kRegC>();
    // O and l relative to a lazily moved per-row reference mref (as attn.cu): tile j enters with weight
    // w_j = 2^{sl2 (tmax_j − mref)} / 2688 (= s_P1 · Π α relative to mref).
    const int r = threadIdx.x;
    const int q_row = qt * 128 + r;
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    float mref = -INFINITY, l = 0.0f;
    f2 o[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = make_float2(0.f, 0.f);
    for (int j = 0; j < nkv; ++j) {
      const int b = j % kBufs;
      A3_EV(0, 4, j, 0);
      A3_CW(j, 0);
      chain_wait(&x_full[b], (uint32_t)(j / kBufs) & 1u);
      A3_EV(0, 4, j, 1);
      A3_CW(j, 1);
      const float tmax = lds_f32(xchg_s + b * 1024);
      const float rs2 = lds_f32(xchg_s + b * 1024 + 512);
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
      chain_wait(&pv_full[b], (uint32_t)(j / kBufs) & 1u);
      A3_EV(0, 4, j, 2);
      A3_CW(j, 2);
      tc_fence_after();
      const uint32_t pv_base = lane_base + 128 * b;
      auto acc = [&](int c, const uint32_t(&v)[16]) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          o[8 * c + i] = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), ww, o[8 * c + i]);
      };
      {  // PV_j in 16-column chunks, the next chunk's load in flight during this chunk's FFMA2s; the buffer is
         // released (b_empty) as soon as the last chunk is in registers, before its FFMA2s
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
            if (lane == 0) mbar_arrive(&b_empty[b]);
          }
          acc(c + 1, vb);
        }
      }
      A3_EV(0, 4, j, 3);
      A3_CW(j, 3);
#ifdef SAGE3_TRACE
      if (lane == 0) A3_TR(0, j, warp);
#endif
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
    const int par = wg - 1;  // this warpgroup's tiles: j ≡ par (mod 3), buffers par
    const int r = threadIdx.x - 128 * wg;
    const int q_row = qt * 128 + r;
    const f2 sl2x2 = make_float2(sl2, sl2);
    const uint32_t s_addr = lane_base + 128 * par;
    const uint32_t sP = smem_u32(smem + L::oP + par * L::kPBytes) + r * 64;
    const uint32_t sPSF = smem_u32(smem + L::oPSF + par * L::kPSF) + (r & 31) * 16 + (r >> 5) * 4;
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + par * 1024 + r * 4;
    const uint32_t swz = (uint32_t)((r >> 1) & 3);
    // warp 0 of the warpgroup issues S_j of its buffer (the warpgroup waits for S_j anyway, and the TMEM loads that
    // follow need S_j complete, so issuing costs this warp nothing): s_Q into the buffer's columns first
    const bool leader = (warp & 3) == (SAGE3_A3_SPREAD ? par : 0);
    if (leader) {
      if (elect_one()) {
        mbar_wait(q_full, 0);
        tc_fence_after();
#pragma unroll
        for (int at = 0; at < kQKAtoms; ++at)
          tmem_cp_32x128b_x4(tbase + kSFQ + 8 * par + 4 * at, sf_desc(smem + L::oQSF + 512 * at));
      }
      __syncwarp();
    }
    auto tile = [&](const int j, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const uint32_t ph = (uint32_t)(j / kBufs) & 1u;
      if (leader) {
        if (elect_one()) issue_s(j);
        __syncwarp();
      }
      A3_EV(128 * wg, wg, j, 0);
      chain_wait(&s_full[par], ph);
      A3_EV(128 * wg, wg, j, 1);
      tc_fence_after();
      // ring refills, no waiting: S_j has completed, so K̂_j's slot is free for K̂_{j+kKStages}; S_j was issued after
      // the correction read PV_{j-3}, so V̂_{j-3}'s slot is free for V̂_{j+2} (kVStages = 5)
      if ((warp & 3) == 1 && j + kKStages < nkv) {
        if (elect_one()) load_k(j + kKStages);
        __syncwarp();
      }
      if ((warp & 3) == 2 && j >= kBufs && j + kVStages - kBufs < nkv) {
        if (elect_one()) load_v(j + kVStages - kBufs);
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
      A3_EV(128 * wg, wg, j, 2);
      // (the P̂2 buffer is free: PV_{j-3} completed before the correction released S_j's buffer)
      // ---- pass 2 per 16-key block: y = P̃2/s, codes E2M1(y), rowsum(P̃2) = Σ_blk s_blk·Σy; the next block's
      //      TMEM load is in flight while this block is computed.
      float rowsum = 0.0f;
      auto block = [&](int blk, const uint32_t(&v)[16]) {
        f2 y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const f2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2x2,
                             make_float2(nbb[blk], nbb[blk]));
          y[i] = ((SAGE3_A3_POLY_MASK >> i) & 1u) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        }
        const f2 s01 = fadd2(fadd2(y[0], y[1]), fadd2(y[2], y[3]));
        const f2 s23 = fadd2(fadd2(y[4], y[5]), fadd2(y[6], y[7]));
        const f2 sy = fadd2(s01, s23);
        rowsum = fmaf(sdec[blk], sy.x + sy.y, rowsum);
        const uint32_t w0 = cvt_e2m1x8(y[0].x, y[0].y, y[1].x, y[1].y, y[2].x, y[2].y, y[3].x, y[3].y);
        const uint32_t w1 = cvt_e2m1x8(y[4].x, y[4].y, y[5].x, y[5].y, y[6].x, y[6].y, y[7].x, y[7].y);
        // 16-byte chunk blk/2 = keys [32 (blk/2), +32) of row r, SWIZZLE_64B (chunk ^= (row>>1)&3)
        sts_v2(sP + ((((uint32_t)blk >> 1) ^ swz) * 16) + (blk & 1) * 8, w0, w1);
      };
#pragma unroll
      for (int blk = 0; blk < 8; blk += 2) {
        tmem_ld_wait_regs(va);
        tmem_ld_32x32b_x16(s_addr + 16 * (blk + 1), vb);
        block(blk, va);
        tmem_ld_wait_regs(vb);
        if (blk + 2 < 8) tmem_ld_32x32b_x16(s_addr + 16 * (blk + 2), va);
        block(blk + 1, vb);
      }
      sts_u32(sPSF, scw[0]);
      sts_u32(sPSF + 512, scw[1]);
      sts_f32(xchg_s, tmax);
      sts_f32(xchg_s + 512, rowsum);
      tc_fence_before();
      fence_proxy_async_smem();
      mbar_arrive(&x_full[par]);  // per thread: releases its own exchange-slot writes
      __syncwarp();
      A3_EV(128 * wg, wg, j, 3);
      {  // the fourth softmax warp done with tile j issues PV_j (its S_j reads and P̂2_j writes are all ordered before
         // this counter update by each warp's fences)
        uint32_t old = 0;
        if (lane == 0) old = atom_add_acqrel(cnt_s + 4 * par, 1u);
        if ((__shfl_sync(0xffffffffu, old, 0) & 3u) == 3u) {
          if (elect_one()) {
            tc_fence_after();
            issue_pv(j);
          }
          __syncwarp();
        }
#ifdef SAGE3_TRACE
        if (lane == 0) A3_TR(7, j, warp & 3);
#endif
      }
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
#ifdef SAGE3_TRACE
  if (blockIdx.x < 2)
    for (int i = threadIdx.x; i < 10 * 32 * 8; i += kThreads)
      g_trace3[blockIdx.x][i / 256][8 + (i / 8) % 32][i % 8] = s_tr[i];
#endif
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int D>
cudaError_t launch3(const AttnArgs& a, cudaStream_t stream) {
  using L = Layout3<D>;
  static std::atomic<bool> attr_done[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn3_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
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
  attn3_fwd_kernel<D><<<(unsigned)units, kThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

}  // namespace

// The north_star path (NVFP4, paper-exact two-level P, no smoothing Q) takes this kernel for d = 64 when it measured
// faster than attn.cu (same-box A/B, B=1, H=32, TOPS attn.cu / attn3.cu: non-causal N = 1K 378 / 349, 2K 508 / 475,
// 4K 652 / 649, 8K 695 / 722, 16K 711 / 763; causal 2K 316 / 332, 8K 550 / 620, 32K 670 / 767; C3-shaped 718 / 768):
// causal, or N >= 8K.  d = 128 stays on attn.cu (1494 vs 1485 at N = 32K).  SAGE3_ATTN_KERNEL=2 / =3 force attn.cu /
// this kernel for every shape (experiments, A/B runs).
bool attention3_enabled(int d, int N, int causal) {
  static const int force = [] {
    const char* e = std::getenv("SAGE3_ATTN_KERNEL");
    return e == nullptr ? 0 : e[0] == '2' ? 2 : e[0] == '3' ? 3 : 0;
  }();
  return force == 3 || (force == 0 && d == 64 && (causal || N >= 8192));
}

cudaError_t launch_attention3(const AttnArgs& a, cudaStream_t stream) {
  return a.d == 128 ? launch3<128>(a, stream) : launch3<64>(a, stream);
}

#ifdef SAGE3_TRACE
extern "C" int sage3_debug_trace_copy3(void* host, size_t bytes) {
  if (bytes > sizeof(g_trace3)) bytes = sizeof(g_trace3);
  return (int)cudaMemcpyFromSymbol(host, g_trace3, bytes);
}
#endif

}  // namespace sage3
