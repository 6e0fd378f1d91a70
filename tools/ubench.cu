// ubench.cu — sm_100a pipe microbenchmarks for the softmax design (cycles per warp-instruction per SM
// sub-partition, by warps per sub-partition).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench tools/ubench.cu && build/ubench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 256;

template <int OP>
__global__ void bench(float* out, long long* cyc, float seed) {
  float r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = seed * (threadIdx.x + i);
  float2 p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = make_float2(r[2 * i], r[2 * i + 1]);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if (OP == 0) {  // MUFU.EX2, 16 independent chains
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[i]));
    } else if (OP == 1) {  // FFMA2, 8 independent chains
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = __ffma2_rn(p[i], p[i], make_float2(0.5f, 0.5f));
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = __ffma2_rn(p[i], p[i], make_float2(0.5f, 0.5f));
    } else if (OP == 2) {  // FFMA scalar, 16 chains
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = __fmaf_rn(r[i], r[i], 0.5f);
    } else if (OP == 3) {  // F2FP e2m1x2, 16 independent
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint32_t o;
        asm volatile("{\n\t.reg .b8 t;\n\tcvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n\tcvt.u32.u8 %0, t;\n\t}"
                     : "=r"(o) : "f"(r[i]), "f"(r[(i + 1) & 15]));
        acc += o;
      }
    } else if (OP == 4) {  // FMNMX3, 16 chains
#pragma unroll
      for (int i = 0; i < 16; ++i)
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(r[i]) : "f"(r[(i + 3) & 15]), "f"(r[(i + 7) & 15]));
    } else if (OP == 5) {  // mix: 4 MUFU + 16 FFMA2 per step (the pass-2 ratio)
#pragma unroll
      for (int i = 0; i < 4; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[i]));
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = __ffma2_rn(p[i], p[i], make_float2(0.5f, 0.5f));
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = __ffma2_rn(p[i], p[i], make_float2(0.5f, 0.5f));
    } else if (OP == 6) {  // FADD2
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = __fadd2_rn(p[i], make_float2(0.5f, 0.25f));
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = __fadd2_rn(p[i], make_float2(0.5f, 0.25f));
    } else if (OP == 7) {  // MUFU dependent chain (latency): 1 chain
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[0]));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[0]));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[0]));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[0]));
    } else if (OP == 8) {  // FFMA2 dependent chain (latency)
      p[0] = __ffma2_rn(p[0], p[0], make_float2(0.5f, 0.5f));
      p[0] = __ffma2_rn(p[0], p[0], make_float2(0.5f, 0.5f));
      p[0] = __ffma2_rn(p[0], p[0], make_float2(0.5f, 0.5f));
      p[0] = __ffma2_rn(p[0], p[0], make_float2(0.5f, 0.5f));
    } else if (OP == 9) {  // IMAD (shift-add form used by the polynomial exp2)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        int v = __float_as_int(r[i]);
        asm volatile("mad.lo.s32 %0, %0, 8388608, %1;" : "+r"(v) : "r"(i));
        r[i] = __int_as_float(v);
      }
    } else if (OP == 10) {  // mix: 2 MUFU + 16 F2FP-free FADD2 + 8 FMNMX3
#pragma unroll
      for (int i = 0; i < 4; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(r[i]));
#pragma unroll
      for (int i = 4; i < 16; ++i)
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(r[i]) : "f"(r[(i + 3) & 15]), "f"(r[(i + 7) & 15]));
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += p[i].x + p[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int per_step_instr) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  printf("%-34s", name);
  for (int w = 1; w <= 8; w *= 2) {
    int threads = 128 * w;  // w warps per sub-partition
    bench<OP><<<148, threads>>>(out, cyc, 1e-3f);
    bench<OP><<<148, threads>>>(out, cyc, 1e-3f);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += h[i];
    c /= 148;
    // warp-instructions issued per sub-partition = w warps * kIters * per_step
    printf("  w=%d: %6.2f cyc/instr", w, c / ((double)w * kIters * per_step_instr));
  }
  printf("\n");
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("MUFU.EX2 (16 indep)", 16);
  run<7>("MUFU.EX2 (dependent chain)", 4);
  run<1>("FFMA2 (8 indep)", 16);
  run<8>("FFMA2 (dependent chain)", 4);
  run<2>("FFMA (16 indep)", 16);
  run<6>("FADD2 (8 indep)", 16);
  run<3>("F2FP e2m1x2 (+IADD)", 32);
  run<4>("FMNMX3 (16)", 16);
  run<9>("IMAD (16)", 16);
  run<5>("mix 4 MUFU + 16 FFMA2", 20);
  run<10>("mix 4 MUFU + 12 FMNMX3", 16);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
