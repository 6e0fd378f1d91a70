// attn.cu — sm_100a SageAttention3 FP4 attention forward: Algorithm 1 L6-L13.
//
// One CTA = one 128-row query tile Q_i of one (b,h); loop over 128-key tiles j (B_q = B_kv = 128).
// Warp roles (16 warps, 4 warpgroups, 1 CTA per SM):
//   WG0 warp 0   TMA producer of Q̂_i + s_Q (once) and K̂_j + s_K (kKStages ring)
//       warp 3   TMA producer of V̂ᵀ_j + s_V (kVStages ring)
//       warp 1   MMA issuer (one elected lane):
//                  S_j  = FP4MM(Q̂_i, s_Q, K̂_j, s_K)      tcgen05.mma kind::mxf4nvf4, M=128 N=128 K=d
//                  PV_j = FP4MM(P̂2_j, s_P2, V̂_j, s_V)    M=128 N=d K=128, written over S_j's TMEM columns
//                scale factors go smem -> TMEM with tcgen05.cp.32x128b.warpx4, in MMA issue order
//       warp 2   TMEM allocator (512 columns)
//   WG2, WG3     softmax + two-level P quantization, one query row per thread (TMEM lane = row);
//                WG2 takes the even KV tiles, WG3 the odd ones.  A tile's P̂2
//                codes and s_P2 depend only on that tile's row max (see below), so the two warpgroups
//                never synchronise with each other.
//   WG1          correction: owns the online-softmax recurrence (m, l; Alg1 L9) and O in registers:
//                O = α·O + s_P1·PV_j (Alg1 L11), then O/l (L13) and the store.
//
// Two-level P in tile-local form (reading c14): with tmax_j = rowmax(S_ij),
// m_j = max(m_{j-1}, tmax_j) and the scale folded into log2 units (sl2 = scale·log2 e):
//     P̃2_j = P̃_j / s_P1 = 2688 · 2^{sl2 (S − tmax_j)}         (max element = 2688 -> s_P2 = 448, code 6)
//     s_P1 = rowmax(P̃_j)/2688 = 2^{sl2 (tmax_j − m_j)} / 2688
//     l_j  = 2^{sl2 (m_{j-1} − m_j)} l_{j-1} + s_P1 · rowsum(P̃2_j)
// The 16-key block maxima of S are taken once (pass 1) and reused twice (the paper's "reuse" of the
// block max): their max is tmax_j, and 2688·2^{sl2 (bmax − tmax)} is the block amax of P̃2
// that sets s_P2 (exp is monotone, and the argmax element is computed by the identical instruction).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "attn_common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

#ifndef SAGE3_EARLY_TMA
#define SAGE3_EARLY_TMA 1  // 0: never launch the kEarly instantiation
#endif
constexpr int kEarlyMinN = 4096;  // sequences at least this long use the kEarly instantiation
#ifndef SAGE3_EARLY_K
#define SAGE3_EARLY_K 1  // K tiles requested in the prologue (<= kKStages)
#endif
#ifndef SAGE3_PV_CHUNK
#define SAGE3_PV_CHUNK 16  // correction: PV_j columns per TMEM load
#endif
#ifndef SAGE3_PV_PIPE
#define SAGE3_PV_PIPE 0  // 1: two PV loads in flight in the correction (chunk c+1 requested before chunk c's FFMA2s)
#endif
#ifndef SAGE3_XCHG_TMEM
#define SAGE3_XCHG_TMEM 0  // 1: (eref, rowsum) softmax -> correction through TMEM columns instead of smem + x_full
#endif
#ifndef SAGE3_PROD_BACKOFF
#define SAGE3_PROD_BACKOFF 0  // 1: TMA producers poll their empty barriers with test_wait + timed sleep
#endif
__device__ __forceinline__ void prod_wait(uint64_t* bar, uint32_t parity) {
#if SAGE3_PROD_BACKOFF
  ptx::mbar_wait_backoff(bar, parity);
#else
  ptx::mbar_wait(bar, parity);
#endif
}
// ---- K/V tile sharing across a 2-CTA cluster (kMC): the two CTAs of a cluster are adjacent query tiles of one head
// and read the same K̂/V̂ tiles, so each CTA TMA-loads half of every tile (K rows / V channels) with .multicast::cluster
// into both CTAs' shared memory (CTA rank 0 also multicasts the tile's scale-factor atoms), and every ring slot is
// released by both CTAs' MMA commits (multicast commit, "empty" barriers count 2).  Halves the L2 -> SM traffic and
// the TMA issue of the K/V rings.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void bulk_load_mc(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}

// Which exp2 pairs of each 32-key chunk run on the FMA-pipe polynomial (bit i: pair i), per instantiation: the
// share is 1/4 (two-level) or 5/16 (row-sum variant, whose softmax has no FADD2 row-sum tree); the positions were
// picked by a same-box sweep of 12 masks (profiles/r2_poly_mask_sweep.txt; the spread is ±5% from ptxas scheduling).
#ifndef SAGE3_POLY_MASK_TL
#define SAGE3_POLY_MASK_TL 0x2222
#endif
#ifndef SAGE3_POLY_MASK_QS
#define SAGE3_POLY_MASK_QS 0x1249
#endif
template <bool kQSum>
constexpr uint32_t poly_mask() { return kQSum ? SAGE3_POLY_MASK_QS : SAGE3_POLY_MASK_TL; }
constexpr int kKStages = 4, kVStages = 4;  // (same-box A/B: 4/4 vs 5/4 +0.3% at N = 32K, causal +0.9%; 6/5, 8/6, 4/3, 3/3 slower)
#ifndef SAGE3_PBUFS
#define SAGE3_PBUFS 4
#endif
constexpr int kPBufs = SAGE3_PBUFS;  // P̂2 tiles in smem (tile j -> j % kPBufs)
#ifndef SAGE3_XSLOTS
#define SAGE3_XSLOTS 4  // (same-box A/B: 4 vs 8 +0.4% at N = 32K; 3, 6 slower)
#endif
constexpr int kXSlots = SAGE3_XSLOTS;  // softmax -> correction exchange slots (tile j -> j % kXSlots)
constexpr int kDsStages = 4;  // smoothing Q: ds (GEMV term) rows in smem (tile j -> j % 4)
constexpr int kDsOps = 3;     // smoothing Q: tf32 B operands of the ds MMA (tile j -> j % 3)
constexpr int kThreads = 512;
// Per-thread register budgets after setmaxnreg (one warp of each warpgroup per SM sub-partition:
// kRegWG0 + 2 kRegSoftmax + kRegCorrection = 512 = 64K registers / 128 lanes).
#ifndef SAGE3_REG_WG0
#define SAGE3_REG_WG0 32
#define SAGE3_REG_SOFTMAX 144
#define SAGE3_REG_CORRECTION 192
#endif
#ifndef SAGE3_REG_SOFTMAX_D64  // d = 64: O is 64 floats, so the correction warpgroup needs fewer registers
#define SAGE3_REG_SOFTMAX_D64 176   // (same-box A/B on C3: 176/128 726 TOPS, 168/144 717, 144/192 722)
#define SAGE3_REG_CORRECTION_D64 128
#endif
constexpr uint32_t kRegWG0 = SAGE3_REG_WG0, kRegSoftmax = SAGE3_REG_SOFTMAX, kRegCorrection = SAGE3_REG_CORRECTION;
static_assert(kRegWG0 + 2 * kRegSoftmax + kRegCorrection <= 512, "register budget");
static_assert(kRegWG0 + 2 * SAGE3_REG_SOFTMAX_D64 + SAGE3_REG_CORRECTION_D64 <= 512, "register budget (d = 64)");
template <int D>
constexpr uint32_t reg_softmax() { return D == 64 ? SAGE3_REG_SOFTMAX_D64 : kRegSoftmax; }
template <int D>
constexpr uint32_t reg_correction() { return D == 64 ? SAGE3_REG_CORRECTION_D64 : kRegCorrection; }

// TMEM column map (512 columns allocated): three 128-column buffers; tile j uses buffer j % 3 first for
// S_j (MMA), then — once the softmax has read S_j — for PV_j (MMA), which the correction warpgroup reads
// before the buffer is reused for S_{j+3}.  Scale factors in 32 more columns.
constexpr int kSBufs = 3;
// Softmax -> correction exchange of (exponent reference, rowsum(P̃2_j)) per row: two TMEM columns per slot in the
// otherwise unused columns 416..431 (tile j -> slot j % 8).  The softmax warp writes its rows' pair with
// tcgen05.st before its p_full arrival; the correction reads it after pv_full (the PV MMA of the same tile was
// issued after p_full), so the hand-off needs no mbarrier of its own.
[[maybe_unused]] constexpr uint32_t kColX = 416;
// Row-sum variant (kQSum, p_quant = SAGE3_P_TWO_LEVEL_QSUM, reading n2): l accumulates the quantized P,
// computed by the tensor core as P̂2 (M=128, K=128) times a 16-column all-ones FP4 matrix (scales 1.0) into 16
// TMEM columns per S/PV buffer (tile j -> kColRS + 16 (j % 3)); the ones operand's scale factors sit at kColSF1.
constexpr uint32_t kColSF1 = 432, kColRS = 448;

template <int D, bool kMX, bool kQSum = false, bool kSQ = false>
struct Layout {
  static constexpr int kQKRow = D / 2;          // bytes per Q/K row (64 or 32)
  static constexpr int kQBytes = 128 * kQKRow;   // Q tile codes
  static constexpr int kKBytes = 128 * kQKRow;
  static constexpr int kKSlot = ((kKBytes + 1023) / 1024) * 1024;
  static constexpr int kVBytes = D * 64;    // Vᵀ tile: D channel rows x 128 tokens (64 B)
  static constexpr int kPBytes = 128 * 64;  // P̂2 tile: 128 rows x 128 keys (64 B)
  // SF atoms per 128-row tile: NVFP4 d/16 blocks along d (1 or 2 atoms), 8 token blocks (2 atoms);
  // MXFP4 d/32 <= 4 blocks along d and 4 token blocks (1 atom each)
  static constexpr int kQKSF = kMX ? 512 : (D / 64) * 512;
  static constexpr int kVSF = kMX ? 512 : 1024, kPSF = kVSF;
  // byte offsets inside the 1024-aligned dynamic smem window
  static constexpr int oQ = 0;
  static constexpr int oK = oQ + ((kQBytes + 1023) / 1024) * 1024;
  static constexpr int oV = oK + kKStages * kKSlot;
  static constexpr int oP = oV + kVStages * kVBytes;
  static constexpr int oQSF = oP + kPBufs * kPBytes;
  static constexpr int oKSF = oQSF + kQKSF;
  static constexpr int oVSF = oKSF + kKStages * kQKSF;
  static constexpr int oPSF = oVSF + kVStages * kVSF;
  static constexpr int oXchg = oPSF + kPBufs * kPSF;            // float [kXSlots][2][128]: tmax_j, rowsum(P̃2_j)
  static constexpr int oDs = oXchg + kXSlots * 2 * 128 * 4;  // smoothing Q: ds rows of 128 keys, kDsStages slots
  // kQSum: the all-ones B operand (16 rows x 128 keys, E2M1 1.0 = code 2 in every nibble) and its SF atoms (E4M3 1.0)
  static constexpr int oOnes = ((oDs + kDsStages * 512 + 1023) / 1024) * 1024;
  static constexpr int oOnesSF = oOnes + 1024;
  // kSQ: the tf32 operands of the ds MMA (S += 1·dsᵀ): A = 128 identical rows [1,1,1,0, 1,1,1,0] (4 KB), and
  // kDsOps B slots of 128 keys x 8 tf32 (32 B per key: [hi, mid, lo, 0] of ds in one 16-byte half, zeros in the other)
  static constexpr int oDsOne = oOnes;
  static constexpr int oDsOp = oDsOne + 4096;
  static constexpr int oBar = kQSum ? oOnesSF + 1024 : kSQ ? oDsOp + kDsOps * 4096 : oDs + kDsStages * 512;
  static constexpr int kNumBars =
      1 + 2 * kKStages + 2 * kVStages + 3 * kSBufs + 2 * kPBufs + 2 * kXSlots + 2 * kDsStages + 2 * kDsOps;
  static constexpr int oTmem = oBar + kNumBars * 8;
  static constexpr int kBytes = oTmem + 16;
  static constexpr int kSmemAlloc = kBytes + 1024;  // slack for manual 1024-B alignment
  // the O epilogue stages [128 rows][D fp32] over the K and V rings (idle once the last PV MMA has completed)
  static_assert(oP - oK >= D * 4 * 128, "O staging space");
};


// kSQ: smoothing Q (S += ds, Alg1 L8's GEMV term).  kMX: MXFP4 operands (Tab1a ablation): scale_vec::2X MMAs
// with UE8M0 scales, P̂2 in 32-key blocks whose scale is the smallest power of two >= amax/6 (reading m1).
// kDirect: the direct-P ablation (Tab1b): P̂ = φ(P̃) with P̃ = exp(scale(S - m_j)) relative to the
// RUNNING max m_j and s_P1 = 1, instead of the two-level form.  m_j is a chain through the tiles: the warpgroup
// of tile j waits for m_{j-1} from the other one (published right after its pass 1), so the two softmax
// warpgroups are no longer independent in this mode.
template <int D, bool kSQ, bool kMX, bool kDirect, bool kEarly, bool kQSum, bool kMC = false>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                    const AttnArgs a) {
  using L = Layout<D, kMX, kQSum, kSQ>;
  extern __shared__ uint8_t smem_raw[];
  // (-log2 s, s) per E4M3 scale code (static shared memory: LDS.64 with an immediate address)
  __shared__ __align__(1024) float2 s_lut[128];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  uint8_t* sQ = smem + L::oQ;
  uint8_t* sQSF = smem + L::oQSF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::oBar);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + kKStages;
  uint64_t* v_full = k_empty + kKStages;
  uint64_t* v_empty = v_full + kVStages;
  uint64_t* s_full = v_empty + kVStages;  // MMA -> softmax: S_j in buffer j%3
  uint64_t* pv_full = s_full + kSBufs;    // MMA -> correction: PV_j in buffer j%3
  uint64_t* b_empty = pv_full + kSBufs;   // correction -> MMA: buffer j%3 free again
  uint64_t* p_full = b_empty + kSBufs;    // softmax -> MMA: P̂2_j / s_P2 in smem buffer j%4, S_j consumed
  uint64_t* p_empty = p_full + kPBufs;    // MMA -> softmax: PV_j done with smem buffer j%4
  uint64_t* x_full = p_empty + kPBufs;    // softmax -> correction: (tmax_j, rowsum P̃2_j) in slot j%8 (smem mode)
  uint64_t* ds_full = x_full + kXSlots;   // smoothing Q: ds row of tile j in slot j%4 (bulk copy)
  uint64_t* ds_empty = ds_full + kDsStages;  // (unused)
  uint64_t* m_full = ds_empty + kDsStages;    // direct P: m_j of tile j in xchg slot j%8 (softmax -> softmax)
  uint64_t* dsop_full = m_full + kXSlots;     // smoothing Q: V-producer warp -> MMA: tf32 ds operand of tile j in slot j%3
  uint64_t* dsop_empty = dsop_full + kDsOps;  // MMA -> V-producer warp: the ds MMA of tile j read slot j%3
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::oTmem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Work unit u = unit_begin + blockIdx.x of the flattened (b·h, q-tile) space, q tiles fastest and in
  // descending order within a head (CTAs of one head run together and share K/V in L2; longest first under
  // causal masking).  sage3_attn_fwd covers every unit; the multi-GPU launcher gives each rank a range.
  const int n_qt = a.Np >> 7;
  const int64_t unit = a.unit_begin + (int64_t)blockIdx.x;
  const int bh = (int)(unit / n_qt);
  const int qt = n_qt - 1 - (int)(unit % n_qt);
  const int nkv = a.causal ? qt + 1 : n_qt;

  SAGE3_TRACE_EV(0, 127, 0);  // CTA start (thread 0)
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], kMC ? 2 : 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], kMC ? 2 : 1);
    }
    for (int b = 0; b < kSBufs; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&pv_full[b], 1);
      mbar_init(&b_empty[b], 4);  // one arrival per correction warp
    }
    for (int b = 0; b < kPBufs; ++b) {
      mbar_init(&p_full[b], 4);  // one arrival per softmax warp
      mbar_init(&p_empty[b], 1);
    }
    for (int s = 0; s < kXSlots; ++s) mbar_init(&x_full[s], 128);
    for (int s = 0; s < kXSlots; ++s) mbar_init(&m_full[s], 128);
    for (int s = 0; s < kDsStages; ++s) {
      mbar_init(&ds_full[s], 1);
      mbar_init(&ds_empty[s], 1);
    }
    for (int s = 0; s < kDsOps; ++s) {
      mbar_init(&dsop_full[s], 1);
      mbar_init(&dsop_empty[s], 1);
    }
    fence_mbar_init();
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_k);
    prefetch_tmap(&tm_v);
    // kEarly: the Q tile and the first K tiles are requested before the prologue's __syncthreads (the rings
    // are empty and the barriers initialised by this thread), overlapping their latency with TMEM allocation
    // and setup.  A separate instantiation, launched for long sequences only (same-box A/B: +0.8% at N = 8K-32K,
    // while the same code path costs 2-4% at N = 1K).
    if constexpr (kEarly) {
    const int row_q = bh * a.Np + qt * 128;
    mbar_arrive_expect_tx(q_full, L::kQBytes + L::kQKSF);
    tma_load_2d(smem + L::oQ, &tm_q, q_full, 0, row_q);
    bulk_load(smem + L::oQSF, a.q_sf + (int64_t)(row_q >> 7) * L::kQKSF, L::kQKSF, q_full);
    for (int j = 0; j < nkv && j < SAGE3_EARLY_K; ++j) {
      const int row_k = bh * a.Np + j * 128;
      mbar_arrive_expect_tx(&k_full[j], L::kKBytes + L::kQKSF);
      tma_load_2d(smem + L::oK + j * L::kKSlot, &tm_k, &k_full[j], 0, row_k);
      bulk_load(smem + L::oKSF + j * L::kQKSF, a.k_sf + (int64_t)(row_k >> 7) * L::kQKSF, L::kQKSF, &k_full[j]);
    }
    }
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  if (threadIdx.x >= 128 && threadIdx.x < 256) {  // exact reciprocal of every E4M3 scale; 0 for s = 0
    const int c = threadIdx.x - 128;
    const float s = e4m3_to_f32((uint32_t)c);
    // -log2(s) per E4M3 scale code (y = P̃2/s = 2^(x - log2 s)); an s = 0 block uses 2^10 (its codes are
    // multiplied by s = 0 in the MMA, reading c5), its row-sum contribution is Σy·2^-10.
    const bool zero = (s == 0.0f || c == 0x7F);
    s_lut[c] = make_float2(zero ? 10.0f : -log2f(s), zero ? 0x1p-10f : s);
  }
  if constexpr (kQSum) {  // the constant ones operand and its scales (generic stores -> async proxy before the sync)
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem + L::oOnes);
    for (int i = threadIdx.x; i < 512; i += kThreads) ones[i] = i < 256 ? 0x22222222u : 0x38383838u;
    fence_proxy_async_smem();
  }
  if constexpr (kSQ) {  // the ds MMA's constant A operand (rows [1,1,1,0, 1,1,1,0]) and zeroed B slots
    uint32_t* one = reinterpret_cast<uint32_t*>(smem + L::oDsOne);
    for (int i = threadIdx.x; i < 1024; i += kThreads) one[i] = (i & 3) == 3 ? 0u : 0x3F800000u;
    uint32_t* op = reinterpret_cast<uint32_t*>(smem + L::oDsOp);
    for (int i = threadIdx.x; i < kDsOps * 1024; i += kThreads) op[i] = 0u;
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kMC) cluster_sync_all();  // both CTAs' barriers initialised before any multicast reaches them
  tc_fence_after();
  SAGE3_TRACE_EV(0, 127, 1);  // prologue done
  const uint32_t tbase = *tmem_slot;
  const int wg = warp >> 2;

  if (wg == 0) {
    setmaxnreg_dec<kRegWG0>();
    if (warp == 0) {
      // ------------------------------------------------------------------ TMA producer: Q, K
      if (elect_one()) {
        constexpr bool early = kEarly;  // Q and K 0.. already requested in the prologue
        if (!early) {
          const int row_q = bh * a.Np + qt * 128;
          mbar_arrive_expect_tx(q_full, L::kQBytes + L::kQKSF);
          tma_load_2d(sQ, &tm_q, q_full, 0, row_q);
          bulk_load(sQSF, a.q_sf + (int64_t)(row_q >> 7) * L::kQKSF, L::kQKSF, q_full);
        }
        for (int j = early ? SAGE3_EARLY_K : 0; j < nkv; ++j) {
          const int st = j % kKStages;
          const int row_k = bh * a.Np + j * 128;
          prod_wait(&k_empty[st], ((uint32_t)(j / kKStages) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&k_full[st], L::kKBytes + L::kQKSF);
          if constexpr (kMC) {  // rows 64 r .. 64 r + 63 of the tile into both CTAs (tm_k has 64-row boxes here)
            const uint32_t cr = cluster_ctarank();
            tma_load_2d_mc(smem + L::oK + st * L::kKSlot + cr * 64 * L::kQKRow, &tm_k, &k_full[st], 0,
                           row_k + 64 * (int)cr, 0x3);
            if (cr == 0)
              bulk_load_mc(smem + L::oKSF + st * L::kQKSF, a.k_sf + (int64_t)(row_k >> 7) * L::kQKSF, L::kQKSF,
                           &k_full[st], 0x3);
          } else {
            tma_load_2d(smem + L::oK + st * L::kKSlot, &tm_k, &k_full[st], 0, row_k);
            bulk_load(smem + L::oKSF + st * L::kQKSF, a.k_sf + (int64_t)(row_k >> 7) * L::kQKSF, L::kQKSF,
                      &k_full[st]);
          }
        }
      }
      __syncwarp();
    } else if (warp == 3) {
      // ------------------------------------------------------------------ TMA producer: V.  Smoothing Q: the
      // whole warp also turns each 512-byte ds row (ds[bh][qt][128 j .. 128 j + 128), the GEMV term of Alg1 L8,
      // fetched kDsStages tiles ahead) into the B operand of the ds MMA: ds = hi + mid + lo, three exact tf32
      // values (hi, mid: the top 11 significant bits of ds and of ds - hi; lo: the rest, <= 2 bits), so the
      // tensor core adds ds to every row of S_j exactly up to its fp32 accumulation.
      const float* ds_row = kSQ ? a.ds + ((int64_t)bh * n_qt + qt) * a.Np : nullptr;
      auto fetch_ds = [&](int j) {
        mbar_arrive_expect_tx(&ds_full[j % kDsStages], 512);
        bulk_load(smem + L::oDs + (j % kDsStages) * 512, ds_row + j * 128, 512, &ds_full[j % kDsStages]);
      };
      if constexpr (kSQ) {
        if (lane == 0)
          for (int j = 0; j < nkv && j < kDsStages; ++j) fetch_ds(j);
        __syncwarp();
      }
      for (int j = 0; j < nkv; ++j) {
        if constexpr (kSQ) {
          const int rs = j % kDsStages, os = j % kDsOps;
          mbar_wait(&ds_full[rs], (uint32_t)(j / kDsStages) & 1u);
          prod_wait(&dsop_empty[os], ((uint32_t)(j / kDsOps) & 1u) ^ 1u);
          float4 g;
          lds_f4(smem_u32(smem + L::oDs + rs * 512) + lane * 16, g);
          const uint32_t dst = smem_u32(smem + L::oDsOp + os * 4096) + lane * 128;  // keys 4 lane .. 4 lane + 3
          const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float hi = __uint_as_float(__float_as_uint(gv[t]) & 0xFFFFE000u);
            const float r1 = gv[t] - hi;  // exact
            const float mid = __uint_as_float(__float_as_uint(r1) & 0xFFFFE000u);
            sts_v4(dst + 32 * t, __float_as_uint(hi), __float_as_uint(mid), __float_as_uint(r1 - mid), 0u);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&dsop_full[os]);
            if (j + kDsStages < nkv) fetch_ds(j + kDsStages);  // raw slot rs read by the whole warp
          }
          __syncwarp();
        }
        if (elect_one()) {
          const int st = j % kVStages;
          prod_wait(&v_empty[st], ((uint32_t)(j / kVStages) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&v_full[st], L::kVBytes + L::kVSF);
          if constexpr (kMC) {  // channels D/2 r .. of the Vᵀ tile into both CTAs (tm_v has D/2-row boxes here)
            const uint32_t cr = cluster_ctarank();
            tma_load_2d_mc(smem + L::oV + st * L::kVBytes + cr * (D / 2) * 64, &tm_v, &v_full[st], j * 64,
                           bh * D + (D / 2) * (int)cr, 0x3);
            if (cr == 0)
              bulk_load_mc(smem + L::oVSF + st * L::kVSF, a.v_sf + ((int64_t)bh * n_qt + j) * L::kVSF, L::kVSF,
                           &v_full[st], 0x3);
          } else {
            tma_load_2d(smem + L::oV + st * L::kVBytes, &tm_v, &v_full[st], j * 64, bh * D);
            bulk_load(smem + L::oVSF + st * L::kVSF, a.v_sf + ((int64_t)bh * n_qt + j) * L::kVSF, L::kVSF,
                      &v_full[st]);
          }
        }
        __syncwarp();
      }
    } else if (warp == 1 || warp == 2) {
      // ------------------------------------------------------------------ MMA issuers: warp 1 issues the S
      // MMAs, warp 2 the PV MMAs (separate sub-partitions; disjoint scale-factor TMEM columns; each commits
      // its own completions)
      if (elect_one()) {
        constexpr uint32_t kQKLayout = D == 128 ? kLayoutSw64 : kLayoutSw32;
        constexpr int kQKAtoms = L::kQKSF / 512, kPVAtoms = L::kPSF / 512;
        // one K-step (64 elements) of a block-scaled FP4 MMA: NVFP4 reads scale columns sf + 4ks; MXFP4 reads
        // bytes 2ks, 2ks+1 of column sf (sf id in the instruction descriptor)
        auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t n, int ks, uint32_t sfa, uint32_t sfb) {
          if constexpr (kMX)
            mma_mxf4(d, ad, bd, make_idesc_mxf4(128, n, ks), sfa, sfb, ks > 0);
          else
            mma_nvf4(d, ad, bd, make_idesc_nvf4(128, n), sfa + 4 * ks, sfb + 4 * ks, ks > 0);
        };
        auto issue_s = [&](int j) {
          const int b = j % kSBufs, st = j % kKStages;
          SAGE3_TRACE_EV(5, j, 0);
          // s_K first (tcgen05.cp executes after the previous S MMA, which read the columns): only the MMAs wait
          // for the correction's release of the buffer
          mbar_wait(&k_full[st], (uint32_t)(j / kKStages) & 1u);
          tc_fence_after();
          const uint8_t* sK = smem + L::oK + st * L::kKSlot;
          const uint8_t* sKSF = smem + L::oKSF + st * L::kQKSF;
#pragma unroll
          for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kColSFK + 4 * at, sf_desc(sKSF + 512 * at));
          mbar_wait(&b_empty[b], ((uint32_t)(j / kSBufs) & 1u) ^ 1u);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < D / 64; ++ks) {
            const uint64_t ad = make_smem_desc(smem_u32(sQ) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
            const uint64_t bd = make_smem_desc(smem_u32(sK) + 32 * ks, 16, 8 * L::kQKRow, kQKLayout);
            mma(tbase + 128 * b, ad, bd, 128, ks, tbase + kColSFQ, tbase + kColSFK);
          }
          if constexpr (kSQ) {  // Alg1 L8: S_j += 1·ds_jᵀ (kind::tf32, K = 8: A rows [1,1,1,0, ..], B rows [hi,mid,lo,0, ..])
            const int os = j % kDsOps;
            mbar_wait(&dsop_full[os], (uint32_t)(j / kDsOps) & 1u);
            tc_fence_after();
            const uint64_t ad = make_smem_desc(smem_u32(smem + L::oDsOne), 16, 256, kLayoutSw32);
            const uint64_t bd = make_smem_desc(smem_u32(smem + L::oDsOp + os * 4096), 16, 256, kLayoutSw32);
            mma_tf32(tbase + 128 * b, ad, bd, make_idesc_tf32(128, 128), 1u);
            mma_commit(&dsop_empty[os]);
          }
          if constexpr (kMC)
            mma_commit_mc(&k_empty[st], 0x3);  // the slot is refilled by both CTAs' producers
          else
            mma_commit(&k_empty[st]);
          mma_commit(&s_full[b]);
          SAGE3_TRACE_EV(5, j, 3);
        };
        auto issue_pv = [&](int j) {
          const int b = j % kSBufs, pb = j % kPBufs, st = j % kVStages;
          SAGE3_TRACE_EV(6, j, 0);
          const uint8_t* sP = smem + L::oP + pb * L::kPBytes;
          const uint8_t* sV = smem + L::oV + st * L::kVBytes;
          const uint8_t* sPSF = smem + L::oPSF + pb * L::kPSF;
          const uint8_t* sVSF = smem + L::oVSF + st * L::kVSF;
          mbar_wait(&p_full[pb], (uint32_t)(j / kPBufs) & 1u);
          SAGE3_TRACE_EV(6, j, 1);
          mbar_wait(&v_full[st], (uint32_t)(j / kVStages) & 1u);
          SAGE3_TRACE_EV(6, j, 2);
          tc_fence_after();
#pragma unroll
          for (int at = 0; at < kPVAtoms; ++at) {
            tmem_cp_32x128b_x4(tbase + kColSFP + 4 * at, sf_desc(sPSF + 512 * at));
            tmem_cp_32x128b_x4(tbase + kColSFV + 4 * at, sf_desc(sVSF + 512 * at));
          }
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
            const uint64_t bd = make_smem_desc(smem_u32(sV) + 32 * ks, 16, 512, kLayoutSw64);
            mma(tbase + 128 * b, ad, bd, D, ks, tbase + kColSFP, tbase + kColSFV);
          }
          if constexpr (kQSum) {  // row sums of the quantized P̂2: P̂2 x ones (N = 16)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t ad = make_smem_desc(smem_u32(sP) + 32 * ks, 16, 512, kLayoutSw64);
              const uint64_t bd = make_smem_desc(smem_u32(smem + L::oOnes) + 32 * ks, 16, 512, kLayoutSw64);
              mma_nvf4(tbase + kColRS + 16 * b, ad, bd, make_idesc_nvf4(128, 16), tbase + kColSFP + 4 * ks,
                       tbase + kColSF1 + 4 * ks, ks > 0);
            }
          }
          if constexpr (kMC)
            mma_commit_mc(&v_empty[st], 0x3);
          else
            mma_commit(&v_empty[st]);
          mma_commit(&p_empty[pb]);
          mma_commit(&pv_full[b]);
          SAGE3_TRACE_EV(6, j, 3);
        };
        if (warp == 1) {
          mbar_wait(q_full, 0);
          tc_fence_after();
#pragma unroll
          for (int at = 0; at < kQKAtoms; ++at) tmem_cp_32x128b_x4(tbase + kColSFQ + 4 * at, sf_desc(sQSF + 512 * at));
          for (int j = 0; j < nkv; ++j) issue_s(j);  // S_j into buffer j%3 once the correction freed it
        } else {
          if constexpr (kQSum) {
#pragma unroll
            for (int at = 0; at < 2; ++at)
              tmem_cp_32x128b_x4(tbase + kColSF1 + 4 * at, sf_desc(smem + L::oOnesSF + 512 * at));
          }
          for (int j = 0; j < nkv; ++j) issue_pv(j);
        }
      }
      __syncwarp();
    }
  } else if (wg >= 2) {
    // -------------------------------------------------------------------- softmax + two-level P quant
    setmaxnreg_inc<reg_softmax<D>()>();
    const int par = wg - 2;                 // this warpgroup's KV-tile parity
    const int r = threadIdx.x - 128 * wg;   // query row in the tile == TMEM lane
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = a.scale * kLog2e;
    const f2 sl2x2 = make_float2(sl2, sl2);
    const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    // One KV tile (Alg1 L8-L10 for this warpgroup's rows).  Only the last tile can need masking (keys >= N,
    // or the causal diagonal), so it is a separate instantiation outside the hot loop: the loop body is
    // straight-line code with no masking branches (instruction-cache friendly).
    auto tile = [&](const int j, auto masked_tag) {
      constexpr bool masked = decltype(masked_tag)::value;
      const int sb = j % kSBufs, pb = j % kPBufs;
      const uint32_t s_addr = lane_base + 128 * sb;
      const uint32_t sP = smem_u32(smem + L::oP + pb * L::kPBytes) + r * 64;
      const uint32_t sPSF = smem_u32(smem + L::oPSF + pb * L::kPSF) + (r & 31) * 16 + (r >> 5) * 4;
      SAGE3_TRACE_EV(1 + par, j, 0);
      mbar_wait(&s_full[sb], (uint32_t)(j / kSBufs) & 1u);
      SAGE3_TRACE_EV(1 + par, j, 1);
      tc_fence_after();
      const int kv0 = j * 128;
      const int lim = a.causal ? min(a.N - 1, q_row) - kv0 : a.N - 1 - kv0;  // last visible key in tile
      // ---- pass 1: 16-key block maxima of S (reused for the row max and for s_P2).  Masked keys are set
      //      to -inf and written back to TMEM so pass 2 needs no masking code.  All four 32-column TMEM
      //      loads are in flight together (one round trip; the pass-2 buffers are not live yet).
      float bmax[8];
      auto pass1 = [&](int c, uint32_t(&v)[32]) {
        float* f = reinterpret_cast<float*>(v);
        if constexpr (masked) {
#pragma unroll
          for (int t = 0; t < 32; ++t) f[t] = (32 * c + t > lim) ? -INFINITY : f[t];
        }
        if constexpr (masked) tmem_st_32x32b_x32(s_addr + 32 * c, v);  // pass 2 reads the final S
        bmax[2 * c] = max16(f);
        bmax[2 * c + 1] = max16(f + 16);
      };
      {  // all four 32-column loads in flight (the pass-2 buffers are not live yet)
        uint32_t va[32], vb[32], vc[32], vd[32];
        tmem_ld_32x32b_x32(s_addr, va);
        tmem_ld_32x32b_x32(s_addr + 32, vb);
        tmem_ld_32x32b_x32(s_addr + 64, vc);
        tmem_ld_32x32b_x32(s_addr + 96, vd);
        tmem_ld_wait_regs(va);
        tmem_ld_wait_regs(vb);
        tmem_ld_wait_regs(vc);
        tmem_ld_wait_regs(vd);
        SAGE3_TRACE_EV(par ? 3 : 0, j, 1);
        pass1(0, va);
        pass1(1, vb);
        pass1(2, vc);
        pass1(3, vd);
      }
      const float tmax = fmax3(fmax3(bmax[0], bmax[1], bmax[2]), fmax3(bmax[3], bmax[4], bmax[5]),
                               fmaxf(bmax[6], bmax[7]));
      SAGE3_TRACE_EV(par ? 3 : 0, j, 2);
      const int slot = j % kXSlots;
      // the exponent reference of this tile's values: tmax_j (two-level: P̃2 = 2688·2^{sl2(S - tmax_j)}) or the
      // running max m_j (direct: P̃ = 2^{sl2(S - m_j)}); the correction warpgroup weights the tile by it
      float eref = tmax;
      if constexpr (kDirect) {
        float mp = -INFINITY;
        if (j > 0) {
          const int ps = (j - 1) % kXSlots;
          mbar_wait(&m_full[ps], (uint32_t)((j - 1) / kXSlots) & 1u);
          mp = lds_f32(xchg_s + ps * 1024);
        }
        eref = fmaxf(mp, tmax);
        sts_f32(xchg_s + slot * 1024, eref);
        mbar_arrive(&m_full[slot]);  // per thread: orders its own slot write
      }
      const float nb = kDirect ? -eref * sl2 : kLog2_2688 - tmax * sl2;  // P̃2 (P̃) = 2^(S·sl2 + nb)
      if constexpr (masked) tmem_st_wait();
      uint32_t va[32], vb[32];
      tmem_ld_32x32b_x32(s_addr, va);  // pass-2 chunk 0, overlapped with the block-scale math below
      // ---- block scales of φ(P̃2): amax_blk = 2^(bmax·sl2 + nb) (the argmax element's own value),
      //      s = E4M3(amax/6), two blocks per convert; pass 2 then produces y = P̃2/s directly as
      //      2^(S·sl2 + nb - log2 s) with (-log2 s, s) from a 128-entry table indexed by the E4M3 code.
      //      A block whose scale underflows to 0 (reading c5) keeps whatever codes pass 2 produces: the
      //      PV MMA multiplies them by s = 0, so they contribute exactly 0, as the oracle's zero codes do;
      //      its table entry (10, 2^-10) keeps its unquantized P̃2 in the row sum (reading c9).
      float nbb[8], sdec[8];
      uint32_t scw[2] = {0u, 0u};
      if constexpr (kMX) {
        // MXFP4: 32-key blocks (block k = keys [32k, 32k+32) = pass-2 chunk k), s = 2^p the smallest power of two
        // >= fl32(amax/6) (UE8M0 code p + 127), so -log2 s = -p exactly.  amax/6 == 0: scale byte 0, and the
        // (10, 2^-10) substitute of the NVFP4 zero scale keeps pass 2 finite (its codes are 0 there anyway).
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
      SAGE3_TRACE_EV(par ? 3 : 0, j, 4);
      SAGE3_TRACE_EV(1 + par, j, 2);
      mbar_wait(&p_empty[pb], ((uint32_t)(j / kPBufs) & 1u) ^ 1u);
      SAGE3_TRACE_EV(1 + par, j, 3);
      // ---- pass 2: y = P̃2/s, codes E2M1(y), rowsum(P̃2) = Σ_blk s_blk·Σy.  Software-pipelined over the four
      //      32-key chunks: the exp2 of chunk c (MUFU / FMA-pipe polynomial) sits in the same straight-line
      //      block as the sums, E2M1 converts and smem store of chunk c-1, so the scheduler can interleave
      //      MUFU with independent FMA/ALU work.
      float rowsum = 0.0f;
      auto exps = [&](int c, const uint32_t(&v)[32], f2(&y)[16]) {
        const float nA = c == 0 ? nbb[0] : c == 1 ? nbb[2] : c == 2 ? nbb[4] : nbb[6];
        const float nB = c == 0 ? nbb[1] : c == 1 ? nbb[3] : c == 2 ? nbb[5] : nbb[7];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float nbh = i < 8 ? nA : nB;
          const f2 x = ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), sl2x2,
                             make_float2(nbh, nbh));
          y[i] = ((poly_mask<kQSum>() >> i) & 1u) ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        }
      };
      auto finish = [&](int c, const f2(&y)[16]) {
        [[maybe_unused]] const float sA = c == 0 ? sdec[0] : c == 1 ? sdec[2] : c == 2 ? sdec[4] : sdec[6];
        [[maybe_unused]] const float sB = c == 0 ? sdec[1] : c == 1 ? sdec[3] : c == 2 ? sdec[5] : sdec[7];
        uint32_t w[4];
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const f2* yy = y + 8 * hb;
          if constexpr (!kQSum) {  // (kQSum: the row sum comes from the tensor core)
            const f2 s01 = fadd2(fadd2(yy[0], yy[1]), fadd2(yy[2], yy[3]));
            const f2 s23 = fadd2(fadd2(yy[4], yy[5]), fadd2(yy[6], yy[7]));
            const f2 sy = fadd2(s01, s23);
            rowsum = fmaf(hb ? sB : sA, sy.x + sy.y, rowsum);
          }
          w[2 * hb] = cvt_e2m1x8(yy[0].x, yy[0].y, yy[1].x, yy[1].y, yy[2].x, yy[2].y, yy[3].x, yy[3].y);
          w[2 * hb + 1] = cvt_e2m1x8(yy[4].x, yy[4].y, yy[5].x, yy[5].y, yy[6].x, yy[6].y, yy[7].x, yy[7].y);
        }
        // 16-byte chunk c = keys [32c, 32c+32) of row r, SWIZZLE_64B (chunk ^= (row>>1)&3)
        sts_v4(sP + ((c ^ ((r >> 1) & 3)) * 16), w[0], w[1], w[2], w[3]);
      };
      {
        f2 ya[16], yb[16];
        tmem_ld_wait_regs(va);
        SAGE3_TRACE_EV(par ? 3 : 0, j, 5);
        tmem_ld_32x32b_x32(s_addr + 32, vb);
        exps(0, va, ya);
        tmem_ld_wait_regs(vb);
        tmem_ld_32x32b_x32(s_addr + 64, va);
        exps(1, vb, yb);
        finish(0, ya);
        tmem_ld_wait_regs(va);
        tmem_ld_32x32b_x32(s_addr + 96, vb);
        exps(2, va, ya);
        finish(1, yb);
        tmem_ld_wait_regs(vb);
        SAGE3_TRACE_EV(par ? 3 : 0, j, 6);
        exps(3, vb, yb);
        finish(2, ya);
        finish(3, yb);
      }
      sts_u32(sPSF, scw[0]);
      if constexpr (!kMX) sts_u32(sPSF + 512, scw[1]);
#if SAGE3_XCHG_TMEM
      {  // (eref, rowsum) -> the correction warpgroup through TMEM (lane = row), ordered by p_full -> PV -> pv_full
        const uint32_t xv[2] = {__float_as_uint(eref), __float_as_uint(rowsum)};
        tmem_st_32x32b_x2(lane_base + kColX + 2 * slot, xv);
      }
      tmem_st_wait();
      tc_fence_before();
      fence_proxy_async_smem();
      // P̂2 / s_P2 (smem) and the TMEM exchange -> MMA: one arrival per warp after the warp's fences
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
#else
      if constexpr (!kDirect) sts_f32(xchg_s + slot * 1024, eref);
      sts_f32(xchg_s + slot * 1024 + 512, rowsum);
      tc_fence_before();
      fence_proxy_async_smem();
      // (tmax, rowsum) -> correction: every thread releases its own slot writes on x_full, so the hand-off is
      // ordered per thread (compute-sanitizer racecheck clean); P̂2 -> MMA: one arrival per warp after the
      // warp's proxy fences
      mbar_arrive(&x_full[slot]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[pb]);
#endif
      SAGE3_TRACE_WARP(1 + par, j, 4);
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
    // -------------------------------------------------------------------- correction + epilogue
    // O and l are kept relative to a per-row reference max mref (lazily moved: only when a tile max
    // exceeds it by more than 2^8 in weight), so tile j enters with weight
    //   w_j = 2^{sl2 (tmax_j − mref)} / 2688  (= s_P1 · Π α relative to mref)
    // which is Alg1 L9-L11 up to fp32 rounding: O/l and lse are independent of the reference.
    setmaxnreg_inc<reg_correction<D>()>();
    const int r = threadIdx.x - 128;
    const int q_row = qt * 128 + r;
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    [[maybe_unused]] const uint32_t xchg_s = smem_u32(smem + L::oXchg) + r * 4;
    const float sl2 = a.scale * kLog2e;
    float mref = -INFINITY, l = 0.0f;
    f2 o[D / 2];
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = make_float2(0.f, 0.f);
    for (int j = 0; j < nkv; ++j) {
      const int slot = j % kXSlots, b = j % kSBufs;
      SAGE3_TRACE_EV(4, j, 0);
#if SAGE3_XCHG_TMEM
      SAGE3_TRACE_EV(4, j, 1);
      mbar_wait(&pv_full[b], (uint32_t)(j / kSBufs) & 1u);
      SAGE3_TRACE_EV(4, j, 2);
      tc_fence_after();
      uint32_t xv[2];
      tmem_ld_32x32b_x2(lane_base + kColX + 2 * slot, xv);
      tmem_ld_wait();
      asm volatile("" : "+r"(xv[0]), "+r"(xv[1]));
      const float tmax = __uint_as_float(xv[0]);
      const float rs2 = __uint_as_float(xv[1]);
#else
      mbar_wait(&x_full[slot], (uint32_t)(j / kXSlots) & 1u);
      SAGE3_TRACE_EV(4, j, 1);
      const float tmax = lds_f32(xchg_s + slot * 1024);
      const float rs2 = lds_f32(xchg_s + slot * 1024 + 512);
#endif
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
      const float w = ex2((tmax - mref) * sl2 - (kDirect ? 0.0f : kLog2_2688));  // tmax = the tile's eref
      if constexpr (!kQSum) l = fmaf(w, rs2, l);
      const f2 ww = make_float2(w, w);
#if !SAGE3_XCHG_TMEM
      mbar_wait(&pv_full[b], (uint32_t)(j / kSBufs) & 1u);
      SAGE3_TRACE_EV(4, j, 2);
      tc_fence_after();
#endif
      if constexpr (kQSum) {  // l += w · Σ deq(P̂2) of this tile, from the tensor core's ones-column product
        uint32_t rq[1];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(rq[0]) : "r"(lane_base + kColRS + 16 * b));
        tmem_ld_wait();
        asm volatile("" : "+r"(rq[0]));
        l = fmaf(w, __uint_as_float(rq[0]), l);
      }
      constexpr int kPVC = SAGE3_PV_CHUNK;
      const uint32_t pv_base = lane_base + 128 * b;
      auto acc = [&](int c, const uint32_t(&v)[kPVC]) {
#pragma unroll
        for (int i = 0; i < kPVC / 2; ++i)
          o[kPVC / 2 * c + i] =
              ffma2(make_float2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), ww, o[kPVC / 2 * c + i]);
      };
#if SAGE3_PV_PIPE
      {  // PV_j in kPVC-column chunks, two in flight: chunk c+1 is requested before the FFMA2s of chunk c
        uint32_t va[kPVC], vb[kPVC];
        tmem_ld_cols(pv_base, va);
        tmem_ld_wait_regs(va);
#pragma unroll
        for (int c = 0; c < D / kPVC; c += 2) {
          tmem_ld_cols(pv_base + kPVC * (c + 1), vb);
          acc(c, va);
          tmem_ld_wait_regs(vb);
          if (c + 2 < D / kPVC) tmem_ld_cols(pv_base + kPVC * (c + 2), va);
          acc(c + 1, vb);
          if (c + 2 < D / kPVC) tmem_ld_wait_regs(va);
        }
      }
#else
#pragma unroll
      for (int c = 0; c < D / kPVC; ++c) {
        uint32_t v[kPVC];
        tmem_ld_cols(pv_base + kPVC * c, v);
        tmem_ld_wait_regs(v);
        acc(c, v);
      }
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&b_empty[b]);
      SAGE3_TRACE_EV(4, j, 3);
    }
    const float m = mref;
    SAGE3_TRACE_EV(4, 126, 0);
    // Alg1 L13: O_i = diag(l)^-1 O_i
    if (a.lse != nullptr && q_row < a.N) a.lse[(int64_t)bh * a.N + q_row] = m * a.scale + logf(l);
    const float inv_l = 1.0f / l;
    const f2 il{inv_l, inv_l};
#pragma unroll
    for (int c = 0; c < D / 2; ++c) o[c] = fmul2(o[c], il);
    SAGE3_TRACE_EV(4, 126, 1);
    // coalesced store: rows -> smem (the K/V rings, idle once the last PV MMA has completed) -> TMA
    uint8_t* stage = smem + L::oK;
    stage_o_row<D>(stage, r, a.o_dtype, o);
    SAGE3_TRACE_EV(4, 126, 2);
    fence_proxy_async_smem();
    named_bar_sync(1, 128);
    SAGE3_TRACE_EV(4, 126, 3);
    if (threadIdx.x == 128) store_o_tile<D>(&tm_o, stage, a.o_dtype, qt * 128, bh % a.H, bh / a.H);
  }
  SAGE3_TRACE_EV(4, 127, 2);  // correction: epilogue stores issued (thread 128)
  tc_fence_before();
  __syncthreads();
  if constexpr (kMC) cluster_sync_all();  // the partner's multicasts and commits into this CTA have all landed
  SAGE3_TRACE_EV(0, 127, 3);  // all roles done
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ------------------------------------------------------------------------------------------- host
template <int D, bool kSQ, bool kMX, bool kDirect, bool kEarly, bool kQSum>
cudaError_t launch_dk(const AttnArgs& a, cudaStream_t stream) {
  using L = Layout<D, kMX, kQSum, kSQ>;
  static std::atomic<bool> attr_done[64];  // one-time attribute setup per device (racing callers both set it: idempotent)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<D, kSQ, kMX, kDirect, kEarly, kQSum>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
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
  attn_fwd_kernel<D, kSQ, kMX, kDirect, kEarly, kQSum><<<(unsigned)units, kThreads, L::kSmemAlloc, stream>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

// K/V tile sharing in 2-CTA clusters (kMC): non-causal north_star path, pairs of adjacent query tiles of one head.
template <int D>
cudaError_t launch_mc(const AttnArgs& a, cudaStream_t stream) {
  using L = Layout<D, false, false, false>;
  auto kern = attn_fwd_kernel<D, false, false, false, false, false, true>;
  static std::atomic<bool> attr_done[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const int BH = a.B * a.H;
  CUtensorMap tq, tk, tv, to;
  if (!make_map(&tq, a.q_data, D / 2, (uint64_t)BH * a.Np, D / 2, 128) ||
      !make_map(&tk, a.k_data, D / 2, (uint64_t)BH * a.Np, D / 2, 64) ||  // half K tiles
      !make_map(&tv, a.v_data, (uint64_t)a.Np / 2, (uint64_t)BH * D, 64, D / 2) ||  // half Vᵀ tiles
      !make_map_o(&to, a.o, a.o_dtype, a.B, a.H, a.N, D, a.o_sb, a.o_sh, a.o_sn))
    return cudaErrorInvalidValue;
  const int64_t units = a.unit_end - a.unit_begin;
  if (units <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)units, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = L::kSmemAlloc;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, to, a);
}
bool kv_multicast_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SAGE3_KV_MULTICAST");
    return e != nullptr && e[0] == '1';
  }();
  return on;
}

template <int D, bool kSQ, bool kMX, bool kDirect, bool kQSum = false>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t stream) {
  if constexpr (!kSQ && !kMX && !kDirect && !kQSum) {
    if (kv_multicast_enabled() && !a.causal && (a.Np / 128) % 2 == 0 && a.unit_begin % 2 == 0 &&
        (a.unit_end - a.unit_begin) % 2 == 0)
      return launch_mc<D>(a, stream);
  }
  if constexpr (!kDirect) {  // the north_star path (and smoothing Q): long sequences take the early-TMA instantiation
    if (SAGE3_EARLY_TMA && a.N >= kEarlyMinN) return launch_dk<D, kSQ, kMX, kDirect, true, kQSum>(a, stream);
  }
  return launch_dk<D, kSQ, kMX, kDirect, false, kQSum>(a, stream);
}

}  // namespace

template <bool kMX>
cudaError_t launch_fmt(const AttnArgs& a, cudaStream_t stream) {
  if (a.p_direct) {  // ablation: no smoothing-Q instantiation (rejected in abi.cu)
    return a.d == 128 ? launch_d<128, false, kMX, true>(a, stream) : launch_d<64, false, kMX, true>(a, stream);
  }
  if constexpr (!kMX) {  // NEXT #2 row-sum variant (NVFP4 only, no smoothing Q: rejected in abi.cu)
    if (a.p_qsum)
      return a.d == 128 ? launch_d<128, false, false, false, true>(a, stream)
                        : launch_d<64, false, false, false, true>(a, stream);
  }
  if (a.ds) return a.d == 128 ? launch_d<128, true, kMX, false>(a, stream) : launch_d<64, true, kMX, false>(a, stream);
  if (!kMX && attention3_enabled(a.d, a.N, a.causal)) return launch_attention3(a, stream);
  return a.d == 128 ? launch_d<128, false, kMX, false>(a, stream) : launch_d<64, false, kMX, false>(a, stream);
}

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t stream) {
  return a.mx ? launch_fmt<true>(a, stream) : launch_fmt<false>(a, stream);
}

#ifdef SAGE3_TRACE
extern "C" int sage3_debug_trace_copy(void* host, size_t bytes) {
  if (bytes > sizeof(g_trace)) bytes = sizeof(g_trace);
  return (int)cudaMemcpyFromSymbol(host, g_trace, bytes);
}
#endif

}  // namespace sage3
