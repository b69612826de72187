// umma_probe.cu -- checks this repo's hand-written tcgen05 (UMMA) kind::tf32 path on one
// CTA: shared-memory descriptors for K-major operands without swizzle, the instruction
// descriptor, TMEM allocation, MMA issue by one thread, commit to an mbarrier and the
// 32x32b TMEM loads -- D[M=128][N] = sum_k A[m][k] B[n][k] against a host fp64 GEMM,
// once with exact small integers (layout) and once with random fp32 data split 3xTF32
// (accuracy).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2308_00292_b200/csrc/umma.cuh"

constexpr int M = 128, N = 32, K = 32;   // K = 4 MMA k-steps of 8

// smem operand layout (K-major, no swizzle): [row/8][k/4][row%8][k%4] fp32 words
__device__ __host__ inline int koff(int row, int k) { return (row >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (row & 7) * 4 + (k & 3); }

__global__ void probe(const float* A, const float* B, float* D, int split) {
  __shared__ __align__(128) float sAh[M * K], sAl[M * K], sBh[N * K], sBl[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const float a = A[i];
    const float h = split ? dmk::umma::tf32_rna(a) : a;
    sAh[koff(m, k)] = h;
    sAl[koff(m, k)] = dmk::umma::tf32_rna(a - h);
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const float b = B[i];
    const float h = split ? dmk::umma::tf32_rna(b) : b;
    sBh[koff(n, k)] = h;
    sBl[koff(n, k)] = dmk::umma::tf32_rna(b - h);
  }
  if (warp == 0) dmk::umma::tmem_alloc<64>(&tbase);
  if (tid == 0) dmk::umma::mbar_init(&mbar, 1);
  dmk::umma::fence_smem_to_async();
  dmk::umma::fence_before_sync();
  __syncthreads();
  dmk::umma::fence_after_sync();
  const uint32_t td = tbase;
  if (tid == 0) {
    const uint32_t idesc = dmk::umma::idesc_tf32(M, N);
    const int nprod = split ? 3 : 1;
    int first = 1;
    for (int pr = 0; pr < nprod; ++pr) {
      const float* a = pr == 1 ? sAl : sAh;
      const float* b = pr == 2 ? sBl : sBh;
      for (int s = 0; s < K / 8; ++s) {
        const uint64_t da = dmk::umma::sdesc_kmajor(a + s * 64, 128, (K / 4) * 128);
        const uint64_t db = dmk::umma::sdesc_kmajor(b + s * 64, 128, (K / 4) * 128);
        dmk::umma::mma_tf32(td, da, db, idesc, !first);
        first = 0;
      }
    }
    dmk::umma::commit(&mbar);
  }
  dmk::umma::mbar_wait(&mbar, 0);
  dmk::umma::fence_after_sync();
  // warp w reads TMEM lanes 32w..32w+31 = rows m; 32 columns
  float v[32];
  dmk::umma::ld32x32b_x32(td + ((uint32_t)(32 * warp) << 16), v);
  for (int n = 0; n < N; ++n) D[(32 * warp + (tid & 31)) * N + n] = v[n];
  dmk::umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) dmk::umma::tmem_free<64>(td);
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  int bad = 0;
  for (int trial = 0; trial < 2; ++trial) {
    srand(7 + trial);
    for (int i = 0; i < M * K; ++i) A[i] = trial == 0 ? (float)((i * 7) % 13 - 6) : (float)rand() / RAND_MAX * 2 - 1;
    for (int i = 0; i < N * K; ++i) B[i] = trial == 0 ? (float)((i * 5) % 11 - 5) : (float)rand() / RAND_MAX * 2 - 1;
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dA, dB, dD, trial);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * B[n * K + k];
        maxerr = fmax(maxerr, fabs(r - D[m * N + n]));
        maxref = fmax(maxref, fabs(r));
      }
    printf("trial %d (%s): max |D - ref| = %.3e, max |ref| = %.3e, rel %.3e\n", trial,
           trial == 0 ? "integers, 1xTF32" : "random, 3xTF32", maxerr, maxref, maxerr / maxref);
    if (trial == 0 && maxerr != 0) bad = 1;
    if (trial == 1 && maxerr / maxref > 1e-6) bad = 1;
  }
  printf(bad ? "FAIL\n" : "OK\n");
  return bad;
}
