// probe_mma.cu — standalone on-box probe of the sm_100a building blocks the attention kernel relies on:
//  (1) tcgen05.mma kind::mxf4nvf4 block_scale (scale_vec::4X) with K-major SWIZZLE_64B / SWIZZLE_32B operands,
//      scale factors staged smem -> TMEM with tcgen05.cp.32x128b.warpx4 from the 128x4 SF-atom layout;
//  (2) nibble order of packed E2M1 operands.
// Not product code: a diagnostic that prints max |err| per hypothesis.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2505_11594_b200/csrc tools/probe_mma.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "sm100.cuh"

using namespace sage3::ptx;

static double e2m1_val(int c) {
  static const double t[8] = {0, 0.5, 1, 1.5, 2, 3, 4, 6};
  return (c & 8) ? -t[c & 7] : t[c & 7];
}
static double e4m3_val(int c) {
  int e = (c >> 3) & 15, m = c & 7;
  double v = e == 0 ? m * std::ldexp(1.0, -9) : (1 + m / 8.0) * std::ldexp(1.0, e - 7);
  return (c & 0x80) ? -v : v;
}

// K-major FP4 tile of R rows x KB bytes per row, in smem with 'swz' swizzle (KB == 64 -> sw64, 32 -> sw32).
__device__ inline uint32_t swz_off(uint32_t r, uint32_t byte, uint32_t KB) {
  uint32_t chunk = byte >> 4, within = byte & 15;
  if (KB == 64) chunk ^= (r >> 1) & 3;
  else if (KB == 32) chunk ^= (r >> 2) & 1;
  return r * KB + chunk * 16 + within;
}

template <int N, int K>
__global__ void probe_kernel(const uint8_t* A, const uint8_t* B, const uint8_t* SFA, const uint8_t* SFB, float* D) {
  constexpr int KB = K / 2;  // bytes per row
  constexpr int KSTEPS = K / 64;
  __shared__ __align__(1024) uint8_t sA[128 * KB];
  __shared__ __align__(1024) uint8_t sB[128 * KB];
  __shared__ __align__(128) uint8_t sSFA[KSTEPS * 512];
  __shared__ __align__(128) uint8_t sSFB[KSTEPS * 512];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * KB; i += blockDim.x) {
    int r = i / KB, b = i % KB;
    sA[swz_off(r, b, KB)] = A[i];
  }
  for (int i = tid; i < N * KB; i += blockDim.x) {
    int r = i / KB, b = i % KB;
    sB[swz_off(r, b, KB)] = B[i];
  }
  for (int i = tid; i < KSTEPS * 512; i += blockDim.x) {
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
      const uint32_t idesc = make_idesc_nvf4(128, N);
      for (int ks = 0; ks < KSTEPS; ++ks) {
        tmem_cp_32x128b_x4(t0 + 256 + ks * 4, make_smem_desc(smem_u32(sSFA + ks * 512), 0, 128, kLayoutNone));
        tmem_cp_32x128b_x4(t0 + 256 + 16 + ks * 4, make_smem_desc(smem_u32(sSFB + ks * 512), 0, 128, kLayoutNone));
      }
      const uint32_t lay = KB == 64 ? kLayoutSw64 : kLayoutSw32;
      for (int ks = 0; ks < KSTEPS; ++ks) {
        uint64_t ad = make_smem_desc(smem_u32(sA) + ks * 32, 16, 8 * KB, lay);
        uint64_t bd = make_smem_desc(smem_u32(sB) + ks * 32, 16, 8 * KB, lay);
        mma_nvf4(t0, ad, bd, idesc, t0 + 256 + ks * 4, t0 + 256 + 16 + ks * 4, ks > 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  if (warp_id() < 4) {
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int row = warp_id() * 32 + lane_id();
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(t0 + ((warp_id() * 32) << 16) + c0, v);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(t0);
}

__global__ void cvt_probe(float* in, uint32_t* out4, uint32_t* out8, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    out4[i] = cvt_e2m1x2(in[i], 0.0f);
    out8[i] = cvt_e4m3x2(in[i], 0.0f);
  }
}

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

template <int N, int K>
static void run_case(std::mt19937& rng) {
  constexpr int KB = K / 2, KSTEPS = K / 64;
  std::vector<uint8_t> A(128 * KB), B(N * KB), SFA(KSTEPS * 512, 0), SFB(KSTEPS * 512, 0);
  for (auto& x : A) x = rng() & 0xFF;
  for (auto& x : B) x = rng() & 0xFF;
  // scale codes for values in [2^-3, 2^3): e in [4, 10)
  auto rnd_sf = [&]() { return (uint8_t)(((4 + rng() % 6) << 3) | (rng() & 7)); };
  std::vector<uint8_t> sfa_log(128 * (K / 16)), sfb_log(128 * (K / 16), 0);
  for (auto& x : sfa_log) x = rnd_sf();
  for (int r = 0; r < N; ++r)
    for (int c = 0; c < K / 16; ++c) sfb_log[r * (K / 16) + c] = rnd_sf();
  auto atom_off = [&](int r, int c) { return (c / 4) * 512 + (r % 32) * 16 + ((r / 32) % 4) * 4 + (c % 4); };
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < K / 16; ++c) {
      SFA[atom_off(r, c)] = sfa_log[r * (K / 16) + c];
      SFB[atom_off(r, c)] = sfb_log[r * (K / 16) + c];
    }
  uint8_t *dA, *dB, *dSFA, *dSFB;
  float* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dSFA, SFA.size()));
  CK(cudaMalloc(&dSFB, SFB.size()));
  CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dSFA, SFA.data(), SFA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dSFB, SFB.data(), SFB.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, 128 * N * 4));
  probe_kernel<N, K><<<1, 256>>>(dA, dB, dSFA, dSFB, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> D(128 * N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  for (int hyp = 0; hyp < 2; ++hyp) {
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double acc = 0;
        for (int k = 0; k < K; ++k) {
          int ba = A[m * KB + k / 2], bb = B[n * KB + k / 2];
          int sh = ((k & 1) ^ hyp) ? 4 : 0;
          double a = e2m1_val((ba >> sh) & 15) * e4m3_val(sfa_log[m * (K / 16) + k / 16]);
          double b = e2m1_val((bb >> sh) & 15) * e4m3_val(sfb_log[n * (K / 16) + k / 16]);
          acc += a * b;
        }
        maxerr = std::fmax(maxerr, std::fabs(acc - D[m * N + n]));
        maxref = std::fmax(maxref, std::fabs(acc));
      }
    printf("case N=%d K=%d hyp(nibble %s first): max|err|=%.6g max|ref|=%.6g  D[0]=%g D[1]=%g\n", N, K,
           hyp ? "high" : "low", maxerr, maxref, D[0], D[1]);
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dSFA);
  cudaFree(dSFB);
  cudaFree(dD);
}

int main() {
  std::mt19937 rng(1234);
  run_case<128, 128>(rng);
  run_case<64, 128>(rng);
  run_case<128, 64>(rng);
  run_case<64, 64>(rng);
  // quick converts
  const int n = 12;
  float h[n] = {-0.2f, 0.25f, 0.75f, 2.5f, 5.0f, 7.0f, -0.0f, 448.0f, 460.0f, 500.0f, 0.0009765625f, 0.001f};
  float* din;
  uint32_t *d4, *d8;
  CK(cudaMalloc(&din, n * 4));
  CK(cudaMalloc(&d4, n * 4));
  CK(cudaMalloc(&d8, n * 4));
  CK(cudaMemcpy(din, h, n * 4, cudaMemcpyHostToDevice));
  cvt_probe<<<1, 32>>>(din, d4, d8, n);
  CK(cudaDeviceSynchronize());
  uint32_t o4[n], o8[n];
  CK(cudaMemcpy(o4, d4, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(o8, d8, n * 4, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) printf("cvt %g -> e2m1x2 0x%02x  e4m3x2 0x%04x\n", h[i], o4[i], o8[i]);
  printf("PROBE DONE\n");
  return 0;
}
