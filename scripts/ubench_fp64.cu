// Microbenchmark: FP64 DFMA vs DMMA (mma.sync.m8n8k4.f64) throughput on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp64 ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a[8], b = 1.0000001 + threadIdx.x * 1e-9, c = 0.9999999;
  for (int i = 0; i < 8; ++i) a[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int warps : {4, 8, 16, 32}) {
      int threads = 32 * warps;
      cudaEventRecord(e0);
      k_dfma<<<sms * 2, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 8 * iters * (double)threads * sms * 2;
      printf("DFMA  warps/CTA %2d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
      cudaEventRecord(e0);
      k_dmma<<<sms * 2, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 4 * iters * (double)warps * sms * 2;
      printf("DMMA  warps/CTA %2d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    }
  }
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  return 0;
}
