// probe_mx.cu — on-box probe of the MXFP4 form of the block-scaled FP4 MMA: E2M1
// operands with UE8M0 scales per 32 elements, tcgen05.mma kind::mxf4nvf4.block_scale.scale_vec::2X, scale
// factors staged with tcgen05.cp.32x128b.warpx4 from the same 128x4 SF atom (4 scales = 128 K per row).
// Hypotheses for which scale bytes the two K=64 steps read: sf_id (instruction descriptor) = 0 / 2 with the
// same TMEM column, or consecutive column pairs.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2505_11594_b200/csrc tools/probe_mx.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "sm100.cuh"

using namespace sage3::ptx;

__device__ __forceinline__ void mma_mx2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                        uint32_t sfa_tmem, uint32_t sfb_tmem, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(sfa_tmem), "r"(sfb_tmem)
      : "memory");
}

static double e2m1_val(int c) {
  static const double t[8] = {0, 0.5, 1, 1.5, 2, 3, 4, 6};
  return (c & 8) ? -t[c & 7] : t[c & 7];
}
__device__ inline uint32_t swz64(uint32_t r, uint32_t byte) { return r * 64 + (((byte >> 4) ^ ((r >> 1) & 3)) << 4) + (byte & 15); }

__global__ void probe(const uint8_t* A, const uint8_t* B, const uint8_t* SFA, const uint8_t* SFB, float* D, int hyp) {
  __shared__ __align__(1024) uint8_t sA[128 * 64];
  __shared__ __align__(1024) uint8_t sB[128 * 64];
  __shared__ __align__(128) uint8_t sSFA[512];
  __shared__ __align__(128) uint8_t sSFB[512];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    sA[swz64(i / 64, i % 64)] = A[i];
    sB[swz64(i / 64, i % 64)] = B[i];
  }
  for (int i = tid; i < 512; i += blockDim.x) {
    sSFA[i] = SFA[i];
    sSFB[i] = SFB[i];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp_id() == 0) tmem_alloc<512>(&tbase);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t0 = tbase;
  if (warp_id() == 1) {
    if (elect_one()) {
      tmem_cp_32x128b_x4(t0 + 256, make_smem_desc(smem_u32(sSFA), 0, 128, kLayoutNone));
      tmem_cp_32x128b_x4(t0 + 256 + 16, make_smem_desc(smem_u32(sSFB), 0, 128, kLayoutNone));
      // also a copy at +32/+48 for the "column pair" hypothesis
      tmem_cp_32x128b_x4(t0 + 288, make_smem_desc(smem_u32(sSFA), 0, 128, kLayoutNone));
      tmem_cp_32x128b_x4(t0 + 288 + 16, make_smem_desc(smem_u32(sSFB), 0, 128, kLayoutNone));
      for (int ks = 0; ks < 2; ++ks) {
        uint64_t ad = make_smem_desc(smem_u32(sA) + ks * 32, 16, 512, kLayoutSw64);
        uint64_t bd = make_smem_desc(smem_u32(sB) + ks * 32, 16, 512, kLayoutSw64);
        uint32_t idesc = make_idesc_nvf4(128, 128) | (1u << 23);  // UE8M0 scales
        uint32_t ca = t0 + 256, cb = t0 + 272;
        if (hyp == 0) idesc |= ((2u * ks) << 29) | ((2u * ks) << 4);          // sf_id = 2*ks
        else if (hyp == 1) { ca += 2 * ks; cb += 2 * ks; }                      // column + 2*ks
        else { ca += ks; cb += ks; }                                            // column + ks
        mma_mx2(t0, ad, bd, idesc, ca, cb, ks > 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  if (warp_id() < 4) {
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int row = warp_id() * 32 + lane_id();
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(t0 + ((warp_id() * 32) << 16) + c0, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) D[row * 128 + c0 + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(t0);
}

int main() {
  std::mt19937 rng(7);
  std::vector<uint8_t> A(128 * 64), B(128 * 64), SFA(512), SFB(512);
  for (auto& x : A) x = rng() & 0xFF;
  for (auto& x : B) x = rng() & 0xFF;
  std::vector<int> ea(128 * 4), eb(128 * 4);  // E8M0 exponents (biased 127) in [124, 130]
  for (auto& x : ea) x = 124 + rng() % 7;
  for (auto& x : eb) x = 124 + rng() % 7;
  auto atom_off = [](int r, int c) { return (r % 32) * 16 + ((r / 32) % 4) * 4 + (c % 4); };
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 4; ++c) {
      SFA[atom_off(r, c)] = (uint8_t)ea[r * 4 + c];
      SFB[atom_off(r, c)] = (uint8_t)eb[r * 4 + c];
    }
  uint8_t *dA, *dB, *dSA, *dSB;
  float* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dSA, 512);
  cudaMalloc(&dSB, 512);
  cudaMalloc(&dD, 128 * 128 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dSA, SFA.data(), 512, cudaMemcpyHostToDevice);
  cudaMemcpy(dSB, SFB.data(), 512, cudaMemcpyHostToDevice);
  for (int hyp = 0; hyp < 3; ++hyp) {
    cudaMemset(dD, 0, 128 * 128 * 4);
    probe<<<1, 256>>>(dA, dB, dSA, dSB, dD, hyp);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(128 * 128);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double acc = 0;
        for (int k = 0; k < 128; ++k) {
          int ca = (A[m * 64 + k / 2] >> ((k & 1) * 4)) & 15, cb = (B[n * 64 + k / 2] >> ((k & 1) * 4)) & 15;
          acc += e2m1_val(ca) * std::ldexp(1.0, ea[m * 4 + k / 32] - 127) * e2m1_val(cb) * std::ldexp(1.0, eb[n * 4 + k / 32] - 127);
        }
        maxerr = std::fmax(maxerr, std::fabs(acc - D[m * 128 + n]));
        maxref = std::fmax(maxref, std::fabs(acc));
      }
    printf("hyp %d (%s): %s max|err|=%.6g max|ref|=%.6g\n", hyp,
           hyp == 0 ? "sf_id=2ks" : hyp == 1 ? "col+2ks" : "col+ks", cudaGetErrorString(e), maxerr, maxref);
  }
  printf("PROBE DONE\n");
  return 0;
}
