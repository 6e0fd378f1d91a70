// ubench_tmem.cu — tcgen05.ld throughput / latency on sm_100a (cycles per warp-instruction per sub-partition).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_11594_b200/csrc -o build/ubench_tmem tools/ubench_tmem.cu
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace sage3::ptx;

constexpr int kIters = 512;

template <int MODE>
__global__ void bench(float* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t v[32], u[32];
  float acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    const uint32_t col = ((it + warp) & 3) * 128;
    if (MODE == 0) {  // one x32 load, wait (latency)
      tmem_ld_32x32b_x32(base + col, v);
      tmem_ld_wait();
      acc += __uint_as_float(v[0]) + __uint_as_float(v[31]);
    } else if (MODE == 1) {  // two x32 loads in flight (throughput)
      tmem_ld_32x32b_x32(base + col, v);
      tmem_ld_32x32b_x32(base + col + 32, u);
      tmem_ld_wait();
      acc += __uint_as_float(v[0]) + __uint_as_float(u[31]);
    } else if (MODE == 2) {  // x16 loads, 2 in flight
      uint32_t (&a)[16] = *reinterpret_cast<uint32_t(*)[16]>(v);
      uint32_t (&b)[16] = *reinterpret_cast<uint32_t(*)[16]>(u);
      tmem_ld_32x32b_x16(base + col, a);
      tmem_ld_32x32b_x16(base + col + 16, b);
      tmem_ld_wait();
      acc += __uint_as_float(v[0]) + __uint_as_float(u[15]);
    } else if (MODE == 3) {  // x32 store + load
      tmem_st_32x32b_x32(base + col, v);
      tmem_st_wait();
      acc += 1.0f;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(slot);
  }
}

template <int MODE>
void run(const char* name, int loads_per_iter, int bytes_per_load) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  printf("%-28s", name);
  for (int w = 1; w <= 4; w *= 2) {
    bench<MODE><<<148, 128 * w>>>(out, cyc);
    bench<MODE><<<148, 128 * w>>>(out, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += h[i];
    c /= 148;
    const double per = c / ((double)kIters * loads_per_iter);  // cycles per load per warp
    // per SM: 4*w warps each doing loads; bytes per SM per cycle
    printf("  w=%d: %6.1f cyc/ld/warp  %6.0f B/clk/SM", w, per, 4.0 * w * kIters * loads_per_iter * bytes_per_load / c);
  }
  printf("   %s\n", cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("ld x32, wait each", 1, 4096);
  run<1>("2x ld x32, wait", 2, 4096);
  run<2>("2x ld x16, wait", 2, 2048);
  run<3>("st x32, wait each", 1, 4096);
  return 0;
}
