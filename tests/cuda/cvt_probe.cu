// cvt_probe.cu — TEST HELPER (not part of the product library): the raw hardware converts the kernels use,
// exposed for the exhaustive 2^32 comparison against the oracle encoders (SURVEY §4 layer 2).
//   out_e2m1[i] = cvt.rn.satfinite.e2m1x2.f32(x[i]) (low nibble), out_e4m3[i] = cvt.rn.satfinite.e4m3x2.f32(x[i])
#include <cstdint>
#include <cuda_runtime.h>

__global__ void cvt_kernel(const float* __restrict__ x, uint8_t* __restrict__ e2m1, uint8_t* __restrict__ e4m3,
                           int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    uint32_t a;
    uint16_t b;
    asm("{\n\t.reg .b8 t;\n\tcvt.rn.satfinite.e2m1x2.f32 t, %1, %1;\n\tcvt.u32.u8 %0, t;\n\t}" : "=r"(a) : "f"(v));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %1;" : "=h"(b) : "f"(v));
    e2m1[i] = (uint8_t)(a & 0xF);
    e4m3[i] = (uint8_t)(b & 0xFF);
  }
}

extern "C" int probe_cvt(const float* x, uint8_t* e2m1, uint8_t* e4m3, int64_t n, void* stream) {
  cvt_kernel<<<1184, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, e2m1, e4m3, n);
  return (int)cudaGetLastError();
}
