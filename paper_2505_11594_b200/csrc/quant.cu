// quant.cu — sm_100a kernels for sage3_quantize_qkv: smoothing K (Alg1 L2) and NVFP4
// microscaling φ (Eq. 1) of Q, K (1x16 blocks along d) and V (1x16 blocks along tokens, written
// transposed).  HBM-bound: K-mean sums (16-byte coalesced loads, fp64) + their fixed-order reduction,
// then one persistent streaming kernel (TMA tiles -> smem ring -> φ) over all Q, Vᵀ and K chunks.
//
// MXFP4 (Tab1a ablation, template kMX): blocks of 32 with E8M0 scales (e8m0_ceil in sm100.cuh, reading c11).
// Numerics are the DESIGN.md §3 readings, implemented with explicitly rounded intrinsics so that no FMA
// contraction or fast-math can change a bit:
//   km[c] = fl32( (Σ_chunk Σ_token K[n][c]) / N ) in fp64, chunks of 128 tokens, ascending order (c10)
//   x     = fl32(K - km)                                      (K only)
//   s32   = fl32(amax * fl32(1/6))                            (c3)
//   sc    = E4M3 RN satfinite (cvt.rn.satfinite.e4m3x2)       (c2)
//   y     = fl32(x * fl32(1/s)), code = E2M1 RN satfinite    (c1, c4); all codes 0 when s == 0 (c5)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include <cudaTypedefs.h>

#include "internal.h"
#include "sm100.cuh"

namespace sage3 {
namespace {

using namespace ptx;

constexpr float kOneSixth = 0x1.555556p-3f;  // fl32(1/6) = 0x3E2AAAAB

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_q() {
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

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) {
  return __half2float(v);
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

// Unpack 8 16-bit values held in a uint4 to fp32 (exact).
template <typename T>
__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = to_f32<T>(h[i]);
}

// max|x| over 8 / 16 values with NaN propagation (FMNMX3.NAN with |.| source modifiers): an infinite or
// NaN input makes the block amax non-finite, which is how the non-finite flag is detected per block.
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float amax8(const float* x) {
  const float a = fmax3_nan(fabsf(x[0]), fabsf(x[1]), fabsf(x[2]));
  const float b = fmax3_nan(fabsf(x[3]), fabsf(x[4]), fabsf(x[5]));
  return fmax3_nan(a, b, fmax3_nan(fabsf(x[6]), fabsf(x[7]), 0.0f));
}
// E2M1 codes of x·rs for 8 values (element 0 in the low nibble): 4 FMUL2 (RN, exact same rounding as the
// oracle's fl32(x·fl32(1/s))) and 4 converts merged into one word.
__device__ __forceinline__ uint32_t codes8(const float* x, float rs) {
  const f2 r2 = make_float2(rs, rs);
  const f2 y0 = fmul2(make_float2(x[0], x[1]), r2), y1 = fmul2(make_float2(x[2], x[3]), r2);
  const f2 y2 = fmul2(make_float2(x[4], x[5]), r2), y3 = fmul2(make_float2(x[6], x[7]), r2);
  return cvt_e2m1x8(y0.x, y0.y, y1.x, y1.y, y2.x, y2.y, y3.x, y3.y);
}

// ---------------------------------------------------------------------------------- K mean
// grid (ceil(Np/128 / 8), B*H), block 8·d/8 threads: a group of d/8 threads per 128-token chunk (8 chunks per
// block), thread t of a group sums channels 8t .. 8t+7 over the chunk in ascending token order (fp64, sequential,
// reading c10) from one 16-byte load per token row (the group reads a contiguous 2·d-byte row segment), and writes
// ws[bh][channel][chunk]; kmean_final_kernel then reduces the chunk sums in ascending chunk order.
template <typename T>
__global__ void __launch_bounds__(128) kmean_kernel(const T* __restrict__ k, int64_t sb, int64_t sh, int64_t sn,
                                                    int H, int N, int d, int nch, double* __restrict__ ws) {
  const int per = d / 8;  // threads per chunk
  const int chunk = blockIdx.x * (128 / per) + threadIdx.x / per, bh = blockIdx.y;
  if (chunk >= nch) return;
  const int b = bh / H, h = bh % H;
  const int c = (threadIdx.x % per) * 8;
  const T* base = k + b * sb + h * sh + c;
  const int n0 = chunk * 128, n1 = min(n0 + 128, N);
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int n = n0;
  for (; n + 4 <= n1; n += 4) {
    uint4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)(n + i) * sn));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const T* p = reinterpret_cast<const T*>(&v[i]);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += (double)to_f32<T>(p[e]);
    }
  }
  for (; n < n1; ++n) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)n * sn));
    const T* p = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] += (double)to_f32<T>(p[e]);
  }
  double* out = ws + ((int64_t)bh * d + c) * nch + chunk;  // [bh][channel][chunk]
#pragma unroll
  for (int e = 0; e < 8; ++e) out[(int64_t)e * nch] = acc[e];
}

// One warp per (bh, channel): lane l loads chunk sums 8l..8l+7 (the channel's sums are contiguous:
// [bh][channel][chunk]), then every lane adds all of them in ascending chunk order (shuffled out of the
// owning lane) — the sequential fp64 order of reading c10 — and lane 0 writes km = fl32(total / N).
__global__ void __launch_bounds__(256) kmean_final_kernel(const double* __restrict__ ws, int nchunks, int N,
                                                          int total_ch, float* __restrict__ km) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= total_ch) return;
  const double* p = ws + (int64_t)w * nchunks;
  double total = 0.0;
  for (int base = 0; base < nchunks; base += 256) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = base + 8 * lane + k;
      v[k] = i < nchunks ? p[i] : 0.0;
    }
    const int n = min(256, nchunks - base);
    for (int src = 0; src < 32 && 8 * src < n; ++src) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double x = __shfl_sync(0xffffffffu, v[k], src);
        if (8 * src + k < n) total += x;
      }
    }
  }
  if (lane == 0) km[w] = (float)(total / (double)N);
}

// ---------------------------------------------------------------------------------- streaming φ of Q, V, K
// Persistent kernel over work items (tensor, b·h, 128-token chunk): Q items, then Vᵀ items, then K items
// (K needs km, written by the K-mean kernels launched before it).  Warp 8 streams the 128 x d input tiles
// into a kStages-deep smem ring with TMA (4-D tensor maps over the caller's strides; rows >= N arrive as
// zeros, which quantize to the zero codes/scales the padding needs); warps 0-7 quantize from smem:
//   Q, K: φ along d, two threads per 16-element block (shuffle for the amax), coalesced 4-byte code stores;
//   Vᵀ:   φ along tokens through a transposed smem read, codes staged per channel row and stored 64 bytes
//         per channel; scale bytes of every item go to its SF atoms staged in smem, then 16-byte stores.
constexpr int kQStages = 3;

// The fused K-mean path below is selected at run time with the environment variable SAGE3_QUANT_FUSED_K=1 (off by
// default).  Measured on the B200 (B=1, H=32, N=32K): it moves 1.00 GB of DRAM per call instead of
// 1.29 GB (K is read once), but takes 280-336 µs against 269 µs for the three-launch path: the per-head dependency
// (all chunk sums, then km, then φ(K − km)) and the sequential fp64 reductions of reading c10 cost more latency
// than the 0.26 GB of re-read saves.
// Fused K mean (reading c10 unchanged): K is read from HBM once.  Work items are handed out in this global order
// by an atomic counter (an item only depends on items with smaller indices, every claimed item sits on a resident
// CTA that processes its items in increasing order, so waiting cannot deadlock):
//   KS_0, F_0, KS_1, F_1, KS_2, KQ_0, F_2, KS_3, KQ_1, F_3, ..., KQ_{G-2}, KQ_{G-1}   (KQ_g after KS_{g+2})
// KS_g: the fp64 chunk sums of the K tiles of head group g (HBM read, kept in L2: evict_last hint); KQ_g: φ(K − km)
// of the same tiles (L2 hits) once the group's heads have their km; F_g: an equal share of the Q and Vᵀ items
// (evict_first), the distance that lets every KS_g item finish (≈ CTAs x ring depth items are in flight) before
// KQ_g is claimed.  A group holds kKGroupBytes of K, so the groups in flight stay well inside the 126 MB L2.  The
// CTA that adds a head's last chunk sum reduces the head's chunk sums in ascending order (the c10 order), writes
// km and releases a per-head flag the KQ items acquire.
#ifndef SAGE3_KGROUP_MB
#define SAGE3_KGROUP_MB 8
#endif
constexpr int64_t kKGroupBytes = (int64_t)SAGE3_KGROUP_MB << 20;
enum : int { kItemQ = 0, kItemV = 1, kItemKQ = 2, kItemKS = 3 };
struct ItemPlan {
  static constexpr int kLag = 2;  // KQ_g is claimed after KS_{g+kLag}: two groups + fillers of distance
  int BH, nch, GK, G, F;  // heads, chunks per head, heads per K group, groups, filler (Q/Vᵀ) items per group
  __host__ __device__ int group_heads(int g) const { return min(GK, BH - g * GK); }
  __host__ __device__ int total() const { return 4 * BH * nch; }  // KS, KQ, Q, Vᵀ
  __host__ __device__ int filler(int g) const { return max(0, min(F, 2 * BH * nch - g * F)); }
  // item index -> (kind, flattened head, chunk)
  __device__ void decode(int idx, int& kind, int& bh, int& chunk) const {
    auto in_group = [&](int k, int g, int off) { kind = k, bh = g * GK + off / nch, chunk = off % nch; };
    auto in_filler = [&](int g, int off) {
      const int f = g * F + off, per = BH * nch;  // Q items, then Vᵀ items
      kind = f < per ? kItemQ : kItemV;
      const int r = f < per ? f : f - per;
      bh = r / nch, chunk = r % nch;
    };
    for (int g = 0; g < G + kLag; ++g) {
      if (g < G) {
        const int sg = group_heads(g) * nch;
        if (idx < sg) return in_group(kItemKS, g, idx);
        idx -= sg;
      }
      if (g >= kLag) {
        const int sq = group_heads(g - kLag) * nch;
        if (idx < sq) return in_group(kItemKQ, g - kLag, idx);
        idx -= sq;
      }
      if (g < G) {
        const int fg = filler(g);
        if (idx < fg) return in_filler(g, idx);
        idx -= fg;
      }
    }
    kind = -1;  // (unreachable for idx < total())
  }
};
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// per-call control words in the quantize workspace (after the chunk sums), zeroed by the launcher
struct QCtl {
  uint32_t next;    // work counter
  uint32_t pad[3];
  // then BH x {chunk-sum count, km ready}
};

template <int D>
struct QL {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int oVcode = kQStages * kTile;  // Vᵀ codes of one item: D channel rows x 64 bytes
  static constexpr int oSFqk = oVcode + D * 64;     // Q/K SF atoms of one item (512·D/64 bytes)
  static constexpr int oSFv = oSFqk + 1024;         // Vᵀ SF atoms of one item (1024 bytes, rows >= d stay 0)
  static constexpr int oBar = oSFv + 1024;
  static constexpr int kBytes = oBar + 2 * kQStages * 8;
  static constexpr int kAlloc = kBytes + 128;      // slack for the 128-byte alignment of the TMA tiles
};

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <typename T, int D, bool kMX, bool kFusedK>
__global__ void __launch_bounds__(288, 2) quant_stream_kernel(const __grid_constant__ CUtensorMap tm_q,
                                                              const __grid_constant__ CUtensorMap tm_k,
                                                              const __grid_constant__ CUtensorMap tm_v, QKArgs qa,
                                                              VArgs va, ItemPlan ip, double* __restrict__ ws,
                                                              uint32_t* __restrict__ ctl) {
  using L = QL<D>;
  extern __shared__ uint8_t qsm_raw[];
  __shared__ float s_rcp[128];  // fl32(1/s) per E4M3 scale code (c4); 0 for s = 0
  __shared__ __align__(16) float s_qm[D];  // smoothing Q: q̄ of the current Q tile
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(qsm_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::oBar);
  uint64_t* empty = full + kQStages;
  __shared__ int4 s_item[kQStages];  // kFusedK: (kind, head, chunk) of each ring stage (kind -1: no more work)
  __shared__ int s_last;            // kFusedK: this CTA added a head's last chunk sum
  const int t = threadIdx.x, warp = t >> 5;
  const int nch = qa.Np >> 7, BH = qa.B * qa.H;
  const int per_tensor = BH * nch, total = 3 * per_tensor;
  uint32_t* head_cnt = ctl + 4;  // [BH][2]: chunk sums added, km ready
  if (t == 0) {
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);  // one arrival per consumer warp
    }
    fence_mbar_init();
  }
  // SF staging starts zeroed: atom rows (Vᵀ channels >= d) and MXFP4 columns (d/32 < 4) never written stay 0
  for (int i = t; i < 2048 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm + L::oSFqk)[i] = make_uint4(0, 0, 0, 0);
  if (t < 128) {
    const float sd = e4m3_to_f32((uint32_t)t);
    s_rcp[t] = (sd == 0.0f || t == 0x7F) ? 0.0f : __frcp_rn(sd);
  }
  __syncthreads();

  if (warp == 8) {  // ---------------------------------------------------------------- TMA producer
    if constexpr (kFusedK) {
      if (elect_one()) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_v);
        const uint64_t keep = l2_policy_evict_last(), stream_once = l2_policy_evict_first();
        int next = (int)atomicAdd(&ctl[0], 1u);  // the next item is claimed one stage ahead (atomic latency hidden)
        for (int k = 0;; ++k) {
          const int s = k % kQStages;
          mbar_wait(&empty[s], ((uint32_t)(k / kQStages) & 1u) ^ 1u);
          const int idx = next;
          if (idx >= ip.total()) {
            s_item[s] = make_int4(-1, 0, 0, 0);
            mbar_arrive(&full[s]);  // completes the phase without a transfer
            break;
          }
          next = (int)atomicAdd(&ctl[0], 1u);
          int kind, bh, chunk;
          ip.decode(idx, kind, bh, chunk);
          s_item[s] = make_int4(kind, bh, chunk, 0);
          const CUtensorMap* tm = kind == kItemQ ? &tm_q : kind == kItemV ? &tm_v : &tm_k;
          mbar_arrive_expect_tx(&full[s], L::kTile);
          tma_load_4d_hint(sm + s * L::kTile, tm, &full[s], 0, chunk * 128, bh % qa.H, bh / qa.H,
                           kind == kItemKS ? keep : stream_once);
        }
      }
      return;
    }
    if (elect_one()) {
      prefetch_tmap(&tm_q);
      prefetch_tmap(&tm_k);
      prefetch_tmap(&tm_v);
      int k = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x, ++k) {
        const int s = k % kQStages;
        const int tensor = item / per_tensor, rem = item % per_tensor, bh = rem / nch, chunk = rem % nch;
        const CUtensorMap* tm = tensor == 0 ? &tm_q : tensor == 1 ? &tm_v : &tm_k;
        mbar_wait(&empty[s], ((uint32_t)(k / kQStages) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], L::kTile);
        tma_load_4d(sm + s * L::kTile, tm, &full[s], 0, chunk * 128, bh % qa.H, bh / qa.H);
      }
    }
    return;
  }
  // ------------------------------------------------------------------------------------ consumers (256)
  bool finite = true;
  int k = 0;
  for (int item = kFusedK ? 0 : blockIdx.x; kFusedK || item < total; item += gridDim.x, ++k) {
    const int s = k % kQStages;
    int tensor, bh, chunk;
    const T* tile = reinterpret_cast<const T*>(sm + s * L::kTile);
    mbar_wait(&full[s], (uint32_t)(k / kQStages) & 1u);
    if constexpr (kFusedK) {
      const int4 it = s_item[s];
      if (it.x < 0) break;
      const int kind = it.x;
      bh = it.y, chunk = it.z;
      if (kind == kItemKS) {
        // chunk sums of K (reading c10): thread c sums channel c over the chunk's real tokens in ascending order
        // in fp64 (rows >= N arrived as zeros); ws[bh][c][chunk]
        if (t < D) {
          double acc = 0.0;
          const int nr = min(128, qa.N - chunk * 128);
          for (int r = 0; r < nr; ++r) acc += (double)to_f32<T>(tile[r * D + t]);
          ws[((int64_t)bh * nch + chunk) * D + t] = acc;  // [bh][chunk][channel]: the km pass reads rows
        }
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(&empty[s]);
        consumer_bar();  // the CTA's sums are written (CTA scope); thread 0's fence publishes them at gpu scope
        if (t == 0) {
          fence_acq_rel_gpu();
          const bool last = atomicAdd(&head_cnt[2 * bh], 1u) == (uint32_t)nch - 1;
          if (last) fence_acq_rel_gpu();  // acquire the other CTAs' sums of this head
          s_last = last ? 1 : 0;
        }
        consumer_bar();
        if (s_last) {  // this CTA completed the head: km = fl32(Σ_chunks / N), chunks in ascending order
          if (t < D) {  // channel t: its chunk sums are a column of [chunk][channel] (coalesced rows), 16 in flight
            const double* p = ws + (int64_t)bh * nch * D + t;
            double tot = 0.0;
            int c = 0;
            for (; c + 16 <= nch; c += 16) {
              double v[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = __ldcg(p + (int64_t)(c + i) * D);
#pragma unroll
              for (int i = 0; i < 16; ++i) tot += v[i];
            }
            for (; c < nch; ++c) tot += __ldcg(p + (int64_t)c * D);
            qa.k_mean[(int64_t)bh * D + t] = (float)(tot / (double)qa.N);
          }
          consumer_bar();
          if (t == 0) {
            fence_acq_rel_gpu();
            atomicExch(&head_cnt[2 * bh + 1], 1u);
          }
        }
        continue;
      }
      tensor = kind == kItemQ ? 0 : kind == kItemV ? 1 : 2;
      if (tensor == 2) {  // φ(K − km) needs the head's km: wait for its release (all producing CTAs are resident)
        if (t == 0) {
          while (ld_acquire_u32(&head_cnt[2 * bh + 1]) == 0u) __nanosleep(64);
        }
        consumer_bar();
      }
    } else {
      tensor = item / per_tensor;
      const int rem = item % per_tensor;
      bh = rem / nch, chunk = rem % nch;
    }
    if (tensor != 1) {  // Q or K: φ along d
      const bool smooth = tensor == 2;
      const bool sub = smooth || qa.q_mean != nullptr;  // x = fl32(X - mean): K - km, or Q - q̄ (Alg1 L5)
      constexpr int kVec = D / 8, kIt = 128 * kVec / 256;
      const int cv = t % kVec;  // this thread's 8-channel group (fixed: 256 is a multiple of kVec)
      uint8_t* codes = (smooth ? qa.k_data : qa.q_data) + ((int64_t)bh * qa.Np + chunk * 128) * (D / 2);
      if (!smooth && sub) {
        // smoothing Q: q̄ of this 128-row tile, fp64 sequential over its real rows in ascending order,
        // divided by the row count, rounded once (the order of reading c10)
        if (t < D) {
          const int nr = min(128, qa.N - chunk * 128);
          double acc = 0.0;
          for (int r = 0; r < nr; ++r) acc += (double)to_f32<T>(tile[r * D + t]);
          const float qm = (float)(acc / (double)nr);
          s_qm[t] = qm;
          qa.q_mean[((int64_t)bh * nch + chunk) * D + t] = qm;
        }
        consumer_bar();
      }
      float km[8];
      if (sub) {
        const float* msrc = smooth ? qa.k_mean + (int64_t)bh * D + cv * 8 : s_qm + cv * 8;
        const float4 m0 = smooth ? __ldcg(reinterpret_cast<const float4*>(msrc)) : reinterpret_cast<const float4*>(msrc)[0];
        const float4 m1 = smooth ? __ldcg(reinterpret_cast<const float4*>(msrc) + 1) : reinterpret_cast<const float4*>(msrc)[1];
        km[0] = m0.x, km[1] = m0.y, km[2] = m0.z, km[3] = m0.w, km[4] = m1.x, km[5] = m1.y, km[6] = m1.z, km[7] = m1.w;
      }
      uint8_t* sfs = sm + L::oSFqk;
#pragma unroll
      for (int it = 0; it < kIt; ++it) {
        const int i = it * 256 + t, r = i / kVec;
        float x[8];
        unpack8<T>(reinterpret_cast<const uint4*>(tile)[i], x);
        if (sub) {
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const f2 d = fadd2(make_float2(x[e], x[e + 1]), make_float2(-km[e], -km[e + 1]));
            x[e] = d.x, x[e + 1] = d.y;
          }
        }
        float amax = amax8(x);
        amax = fmax3_nan(amax, __shfl_xor_sync(0xffffffffu, amax, 1), 0.0f);
        if constexpr (kMX) amax = fmax3_nan(amax, __shfl_xor_sync(0xffffffffu, amax, 2), 0.0f);  // 32-blocks
        finite &= isfinite(amax);
        // padding rows (n >= N) arrive as zeros from TMA; they must stay zero codes / zero scales even
        // after smoothing (reading c13)
        const bool real = chunk * 128 + r < qa.N;
        uint32_t sc, w;
        if constexpr (kMX) {
          const float s32 = __fmul_rn(amax, kOneSixth);
          float rs;
          sc = e8m0_ceil(s32, rs);
          const bool nz = real && s32 != 0.0f;  // amax = 0: scale byte 0 with zero codes (reading m1)
          sc = nz ? sc : 0u;
          w = nz ? codes8(x, rs) : 0u;
        } else {
          sc = real ? cvt_e4m3x2(__fmul_rn(amax, kOneSixth), 0.0f) & 0xFFu : 0u;
          // a zero scale gives all-zero codes (c5; x·0 would keep the sign of x: E2M1 -0 = 0x8)
          w = sc ? codes8(x, s_rcp[sc]) : 0u;
        }
        *reinterpret_cast<uint32_t*>(codes + r * (D / 2) + cv * 4) = w;
        constexpr int kPer = kMX ? 4 : 2;  // threads per scale block
        if ((cv & (kPer - 1)) == 0) {
          const int c = cv / kPer;
          sfs[(c >> 2) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (c & 3)] = (uint8_t)sc;
        }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[s]);  // tile consumed
      consumer_bar();                             // SF staging complete
      constexpr int kSFqk = kMX ? 512 : 512 * (D / 64);  // SF bytes of one 128-row tile
      uint8_t* sf_dst = (smooth ? qa.k_sf : qa.q_sf) + ((int64_t)bh * nch + chunk) * kSFqk;
      for (int i = t * 16; i < kSFqk; i += 256 * 16)
        *reinterpret_cast<uint4*>(sf_dst + i) = *reinterpret_cast<const uint4*>(sfs + i);
      consumer_bar();  // staging free for the next item
    } else {  // Vᵀ: φ along tokens
      uint8_t* vcode = sm + L::oVcode;
      uint8_t* sfs = sm + L::oSFv;
      if constexpr (kMX) {  // blocks of 32 tokens: (channel pair, 32-token block) per item
        for (int it = t; it < (D / 2) * 4; it += 256) {
          const int cp = it % (D / 2), tb = it / (D / 2);
          float x0[32], x1[32];
          const uint32_t* col = reinterpret_cast<const uint32_t*>(tile) + tb * 32 * (D / 2) + cp;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const uint32_t u = col[e * (D / 2)];
            const T* p = reinterpret_cast<const T*>(&u);
            x0[e] = to_f32<T>(p[0]);
            x1[e] = to_f32<T>(p[1]);
          }
          const int c = 2 * cp;
          const float a0 = fmax3_nan(fmax3_nan(amax8(x0), amax8(x0 + 8), amax8(x0 + 16)), amax8(x0 + 24), 0.0f);
          const float a1 = fmax3_nan(fmax3_nan(amax8(x1), amax8(x1 + 8), amax8(x1 + 16)), amax8(x1 + 24), 0.0f);
          finite &= isfinite(a0) & isfinite(a1);
          const float s0 = __fmul_rn(a0, kOneSixth), s1 = __fmul_rn(a1, kOneSixth);
          float r0, r1;
          uint32_t sc0 = e8m0_ceil(s0, r0), sc1 = e8m0_ceil(s1, r1);
          sc0 = s0 != 0.0f ? sc0 : 0u;
          sc1 = s1 != 0.0f ? sc1 : 0u;
          *reinterpret_cast<uint4*>(vcode + c * 64 + tb * 16) =
              s0 != 0.0f ? make_uint4(codes8(x0, r0), codes8(x0 + 8, r0), codes8(x0 + 16, r0), codes8(x0 + 24, r0))
                         : make_uint4(0u, 0u, 0u, 0u);
          *reinterpret_cast<uint4*>(vcode + (c + 1) * 64 + tb * 16) =
              s1 != 0.0f ? make_uint4(codes8(x1, r1), codes8(x1 + 8, r1), codes8(x1 + 16, r1), codes8(x1 + 24, r1))
                         : make_uint4(0u, 0u, 0u, 0u);
          const int base = ((c >> 5) & 3) * 4 + tb;  // one atom per chunk: 4 token blocks
          sfs[base + (c & 31) * 16] = (uint8_t)sc0;
          sfs[base + ((c + 1) & 31) * 16] = (uint8_t)sc1;
        }
      } else {
      for (int it = t; it < (D / 2) * 8; it += 256) {
        const int cp = it % (D / 2), tb = it / (D / 2);
        float x0[16], x1[16];
        const uint32_t* col = reinterpret_cast<const uint32_t*>(tile) + tb * 16 * (D / 2) + cp;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint32_t u = col[e * (D / 2)];
          const T* p = reinterpret_cast<const T*>(&u);
          x0[e] = to_f32<T>(p[0]);
          x1[e] = to_f32<T>(p[1]);
        }
        const int c = 2 * cp;
        const float a0 = fmax3_nan(amax8(x0), amax8(x0 + 8), 0.0f), a1 = fmax3_nan(amax8(x1), amax8(x1 + 8), 0.0f);
        finite &= isfinite(a0) & isfinite(a1);
        const uint32_t sc2 = cvt_e4m3x2(__fmul_rn(a0, kOneSixth), __fmul_rn(a1, kOneSixth));
        const uint32_t sc0 = sc2 & 0xFFu, sc1 = (sc2 >> 8) & 0xFFu;
        const float r0 = s_rcp[sc0], r1 = s_rcp[sc1];
        // 8-byte group tb of channel rows c, c+1 at position tb ^ ((c >> 1) & 7): the 32 threads of a warp
        // (consecutive channel pairs, same tb) spread over 8 positions instead of one bank (was 32-way)
        const int pos = (tb ^ ((c >> 1) & 7)) * 8;
        *reinterpret_cast<uint2*>(vcode + c * 64 + pos) =
            sc0 ? make_uint2(codes8(x0, r0), codes8(x0 + 8, r0)) : make_uint2(0u, 0u);
        *reinterpret_cast<uint2*>(vcode + (c + 1) * 64 + pos) =
            sc1 ? make_uint2(codes8(x1, r1), codes8(x1 + 8, r1)) : make_uint2(0u, 0u);
        const int base = (tb >> 2) * 512 + ((c >> 5) & 3) * 4 + (tb & 3);
        sfs[base + (c & 31) * 16] = (uint8_t)sc0;
        sfs[base + ((c + 1) & 31) * 16] = (uint8_t)sc1;
      }
      }
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[s]);
      consumer_bar();
      if constexpr (kMX) {
        for (int i = t; i < D * 4; i += 256) {
          const int c = i >> 2, q = i & 3;
          *reinterpret_cast<uint4*>(va.v_data + ((int64_t)bh * D + c) * (qa.Np >> 1) + chunk * 64 + q * 16) =
              *reinterpret_cast<const uint4*>(vcode + c * 64 + q * 16);
        }
      } else {  // un-swizzle: 8 threads per channel row, 8 bytes each (coalesced 64-byte rows)
        for (int i = t; i < D * 8; i += 256) {
          const int c = i >> 3, g = i & 7;
          *reinterpret_cast<uint2*>(va.v_data + ((int64_t)bh * D + c) * (qa.Np >> 1) + chunk * 64 + g * 8) =
              *reinterpret_cast<const uint2*>(vcode + c * 64 + ((g ^ ((c >> 1) & 7)) * 8));
        }
      }
      constexpr int kSFv = kMX ? 512 : 1024;  // SF bytes of one 128-token chunk (128 channel rows)
      uint8_t* sf_dst = va.v_sf + ((int64_t)bh * nch + chunk) * kSFv;
      for (int i = t * 16; i < kSFv; i += 256 * 16)
        *reinterpret_cast<uint4*>(sf_dst + i) = *reinterpret_cast<const uint4*>(sfs + i);
      consumer_bar();
    }
  }
  if (qa.nonfinite && !finite) atomicOr(qa.nonfinite, 1u);
}

// ---------------------------------------------------------------------------------- smoothing Q: ds
// ds[bh][i][key] = Σ_c q̄_i[c]·Ks[key][c], Ks = fl32(K - km) (Alg1 L8's GEMV(q̄_i, K_j^T) with the
// full-precision smoothed K), fp32 FFMA2 on the CUDA cores.  grid (Np/128 key chunks, B·H), 256 threads;
// thread (ig, kg) owns 8 query tiles x 4 keys of each 64-tile block.  Keys >= N get Ks = 0 (they are masked).
template <typename T, int D>
__global__ void __launch_bounds__(256) smooth_q_ds_kernel(QKArgs qa) {
  extern __shared__ __align__(16) float dsm_f[];
  float* kst = dsm_f;            // [D][128] smoothed K of this key chunk, transposed
  constexpr int kQS = 68;        // row stride of the transposed q̄ block (16-byte rows, 4-way store conflicts)
  float* qmt = dsm_f + D * 128;  // [D][kQS] q̄ of 64 query tiles, transposed
  const int chunk = blockIdx.x, bh = blockIdx.y;
  const int b = bh / qa.H, h = bh % qa.H;
  const int t = threadIdx.x, nt = qa.Np >> 7;
  const T* kb = reinterpret_cast<const T*>(qa.k) + b * qa.k_sb + h * qa.k_sh;
  // keys fastest across threads: each thread reads 8 channels of one key (16 bytes) and writes them down
  // the transposed tile, consecutive threads hitting consecutive banks
  for (int i = t; i < 128 * (D / 8); i += 256) {
    const int key = i % 128, c8 = i / 128, n = chunk * 128 + key;
    float x[8];
    if (n < qa.N) {
      unpack8<T>(*reinterpret_cast<const uint4*>(kb + (int64_t)n * qa.k_sn + c8 * 8), x);
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = __fsub_rn(x[e], qa.k_mean[(int64_t)bh * D + c8 * 8 + e]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = 0.0f;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) kst[(c8 * 8 + e) * 128 + key] = x[e];
  }
  const int kg = t & 31, ig = t >> 5;
  // q̄ blocks of 64 tiles: coalesced global reads (channels fastest across threads) into registers one block ahead,
  // stored transposed once the previous block has been consumed
  constexpr int kPre = 64 * D / 256;
  float pre[kPre];
  auto fetch = [&](int i0) {
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
      const int i = t + 256 * k, ti = i / D, c = i % D;
      pre[k] = i0 + ti < nt ? qa.q_mean[((int64_t)bh * nt + i0 + ti) * D + c] : 0.0f;
    }
  };
  fetch(0);
  for (int i0 = 0; i0 < nt; i0 += 64) {
    __syncthreads();  // kst written / previous block's qmt consumed
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
      const int i = t + 256 * k, ti = i / D, c = i % D;
      qmt[c * kQS + ti] = pre[k];
    }
    if (i0 + 64 < nt) fetch(i0 + 64);
    __syncthreads();
    f2 acc[8][2];
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) acc[ii][0] = acc[ii][1] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int c = 0; c < D; ++c) {
      const float4 a0 = reinterpret_cast<const float4*>(qmt + c * kQS + ig * 8)[0];
      const float4 a1 = reinterpret_cast<const float4*>(qmt + c * kQS + ig * 8)[1];
      const float4 bb = reinterpret_cast<const float4*>(kst + c * 128)[kg];
      const f2 b01 = make_float2(bb.x, bb.y), b23 = make_float2(bb.z, bb.w);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) {
        acc[ii][0] = ffma2(make_float2(av[ii], av[ii]), b01, acc[ii][0]);
        acc[ii][1] = ffma2(make_float2(av[ii], av[ii]), b23, acc[ii][1]);
      }
    }
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) {
      const int ti = i0 + ig * 8 + ii;
      if (ti < nt)
        *reinterpret_cast<float4*>(qa.ds + ((int64_t)bh * nt + ti) * qa.Np + chunk * 128 + kg * 4) =
            make_float4(acc[ii][0].x, acc[ii][0].y, acc[ii][1].x, acc[ii][1].y);
    }
  }
}

// 4-D tensor map over a [B][H][N][d] 16-bit operand with element strides (sb, sh, sn): box d x 128 x 1 x 1.
bool make_input_map(CUtensorMap* m, const void* base, int B, int H, int N, int d, int64_t sb, int64_t sh,
                    int64_t sn) {
  auto enc = encode_fn_q();
  if (!enc) return false;
  // strides of extent-1 dimensions are irrelevant; give them a valid value
  if (H == 1) sh = sn * N;
  if (B == 1) sb = sh * H;
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)sn * 2, (cuuint64_t)sh * 2, (cuuint64_t)sb * 2};
  cuuint32_t box[4] = {(cuuint32_t)d, 128, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_tiled_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int D, bool kMX>
cudaError_t launch_t(const QKArgs& qk, const VArgs& v, double* ws, cudaStream_t stream) {
  using L = QL<D>;
  static std::atomic<bool> attr_done[64];  // one-time attribute setup per device (racing callers both set it: idempotent)  // per instantiation
  static int n_sm[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(quant_stream_kernel<T, D, kMX, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, L::kAlloc);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(quant_stream_kernel<T, D, kMX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               L::kAlloc);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&n_sm[dev], cudaDevAttrMultiProcessorCount, dev);
    attr_done[dev] = true;
  }
  CUtensorMap tq, tk, tv;
  if (!make_input_map(&tq, qk.q, qk.B, qk.H, qk.N, D, qk.q_sb, qk.q_sh, qk.q_sn) ||
      !make_input_map(&tk, qk.k, qk.B, qk.H, qk.N, D, qk.k_sb, qk.k_sh, qk.k_sn) ||
      !make_input_map(&tv, v.v, qk.B, qk.H, qk.N, D, v.sb, v.sh, v.sn))
    return cudaErrorInvalidValue;
  const int BH = qk.B * qk.H, nch = qk.Np / 128;
  dim3 grid(nch, BH);
  ItemPlan ip{};
  ip.BH = BH, ip.nch = nch;
  {
    const int64_t gk = kKGroupBytes / ((int64_t)qk.Np * D * 2);
    ip.GK = (int)(gk < 1 ? 1 : gk > BH ? BH : gk);
  }
  ip.G = (BH + ip.GK - 1) / ip.GK;
  ip.F = (2 * BH * nch + ip.G - 1) / ip.G;
  uint32_t* ctl = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ws) + quant_sums_bytes(BH, nch, D));
  const int items = 3 * BH * nch;
  const int ctas = min(items, 2 * (dev < 64 && n_sm[dev] ? n_sm[dev] : 148));
  static const bool fused_k = [] {
    const char* e = std::getenv("SAGE3_QUANT_FUSED_K");
    return e != nullptr && e[0] == '1';
  }();
  if (fused_k) {
    cudaError_t e = cudaMemsetAsync(ctl, 0, quant_ctl_bytes(BH), stream);
    if (e != cudaSuccess) return e;
    quant_stream_kernel<T, D, kMX, true><<<ctas, 288, L::kAlloc, stream>>>(tq, tk, tv, qk, v, ip, ws, ctl);
  } else {
    kmean_kernel<T><<<dim3((nch * (D / 8) + 127) / 128, BH), 128, 0, stream>>>(
        reinterpret_cast<const T*>(qk.k), qk.k_sb, qk.k_sh, qk.k_sn, qk.H, qk.N, D, nch, ws);
    kmean_final_kernel<<<(BH * D * 32 + 255) / 256, 256, 0, stream>>>(ws, nch, qk.N, BH * D, qk.k_mean);
    quant_stream_kernel<T, D, kMX, false><<<ctas, 288, L::kAlloc, stream>>>(tq, tk, tv, qk, v, ip, ws, ctl);
  }
  if (qk.q_mean) {  // smoothing Q: the GEMV term, after every q̄ of the head is written
    static bool ds_attr[64] = {};
    constexpr int kDsSmem = (D * 128 + D * 68) * 4;
    if (dev < 64 && !ds_attr[dev]) {
      cudaError_t e = cudaFuncSetAttribute(smooth_q_ds_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDsSmem);
      if (e != cudaSuccess) return e;
      ds_attr[dev] = true;
    }
    smooth_q_ds_kernel<T, D><<<grid, 256, kDsSmem, stream>>>(qk);
  }
  return cudaGetLastError();
}

}  // namespace

template <bool kMX>
cudaError_t launch_fmt(const QKArgs& qk, const VArgs& v, bool bf16, double* ws, cudaStream_t stream) {
  if (qk.d == 128)
    return bf16 ? launch_t<__nv_bfloat16, 128, kMX>(qk, v, ws, stream)
                : launch_t<__half, 128, kMX>(qk, v, ws, stream);
  return bf16 ? launch_t<__nv_bfloat16, 64, kMX>(qk, v, ws, stream)
              : launch_t<__half, 64, kMX>(qk, v, ws, stream);
}

// The smoothing-K mean alone (Alg1 L2 / Alg2 L2, reading c10), for the INT8 (SageBwd) quantizer.
cudaError_t launch_kmean(const QKArgs& qk, bool bf16, double* ws, cudaStream_t stream) {
  const int BH = qk.B * qk.H;
  dim3 grid(qk.Np / 128, BH);
  const int nch = qk.Np / 128;
  const dim3 kgrid((nch * (qk.d / 8) + 127) / 128, BH);
  if (bf16)
    kmean_kernel<__nv_bfloat16><<<kgrid, 128, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(qk.k), qk.k_sb,
                                                           qk.k_sh, qk.k_sn, qk.H, qk.N, qk.d, nch, ws);
  else
    kmean_kernel<__half><<<kgrid, 128, 0, stream>>>(reinterpret_cast<const __half*>(qk.k), qk.k_sb, qk.k_sh, qk.k_sn,
                                                    qk.H, qk.N, qk.d, nch, ws);
  kmean_final_kernel<<<(BH * qk.d * 32 + 255) / 256, 256, 0, stream>>>(ws, qk.Np / 128, qk.N, BH * qk.d, qk.k_mean);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const QKArgs& qk, const VArgs& v, bool bf16, double* ws, cudaStream_t stream) {
  return qk.mx ? launch_fmt<true>(qk, v, bf16, ws, stream) : launch_fmt<false>(qk, v, bf16, ws, stream);
}

}  // namespace sage3
