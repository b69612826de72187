// FP32 FFMA vs FFMA2 (packed f32x2) issue throughput on this B200: many independent
// chains per thread, all SMs busy; reports FMA/s (an FFMA2 counts 2 FMA).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NCH = 8, IT = 4096;
__global__ void k_ffma(float* out, float a, float b) {
  float c[NCH];
  for (int i = 0; i < NCH; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = fmaf(c[i], a, b);
  float s = 0; for (int i = 0; i < NCH; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 c[NCH];
  for (int i = 0; i < NCH; ++i) c[i] = make_float2(threadIdx.x + i, i);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = __ffma2_rn(c[i], a2, b2);
  float s = 0; for (int i = 0; i < NCH; ++i) s += c[i].x + c[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4 * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nb = 148 * 8, nt = 256;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma<<<nb, nt>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double f = (double)nb * nt * IT * NCH;
    printf("FFMA : %.1f T FMA/s (%.1f TFLOP/s)\n", f / ms / 1e9, 2 * f / ms / 1e9);
    cudaEventRecord(e0); k_ffma2<<<nb, nt>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    f *= 2;
    printf("FFMA2: %.1f T FMA/s (%.1f TFLOP/s)\n", f / ms / 1e9, 2 * f / ms / 1e9);
  }
  return 0;
}
