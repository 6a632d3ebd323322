// umma_off_test.cu -- K-major no-swizzle A operand whose descriptor start address is only
// 16-byte aligned (row shift inside a core-matrix group): does tcgen05.mma read the rows
// starting exactly there?  M=128, N=16, K=8 tf32; A rows are "pixels" at a 16 B pitch.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1912_12675_b200/csrc/ptx.cuh"
using namespace pst::ptx;
constexpr int M = 128, N = 16, K = 8, ROWS = 160;
// A: plane p (4 channels) at stride PLANE bytes; row r at 16 B pitch inside the plane
constexpr int PLANE = ROWS * 16;
__global__ void kern(const float* A, const float* B, float* D, int shift) {
  __shared__ __align__(1024) uint8_t sa[2 * PLANE];
  __shared__ __align__(1024) uint8_t sb[4096];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < ROWS * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sa + (k / 4) * PLANE + r * 16 + (k % 4) * 4) = A[r * K + k];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<float*>(sb + (n / 8) * 128 + (k / 4) * 256 + (n % 8) * 16 + (k % 4) * 4) = B[n * K + k];
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 32);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_mma(M, N, 0, 0, 2);
    const uint64_t ad = smem_desc(smem_u32(sa) + shift * 16, PLANE, 128);
    const uint64_t bd = smem_desc(smem_u32(sb), 256, 128);
    if (elect_one()) { umma_tf32(tm, ad, bd, idesc, 0); umma_commit(&bar); }
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  float v[16];
  tmem_ld16(tm + ((uint32_t)(threadIdx.x & ~31) << 16), v);
  for (int j = 0; j < 16; ++j) D[threadIdx.x * N + j] = v[j];
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 32);
}
int main() {
  static float hA[ROWS * K], hB[N * K], hD[M * N];
  srand(1);
  for (auto& x : hA) x = (float)(rand() % 17 - 8);
  for (auto& x : hB) x = (float)(rand() % 13 - 6);
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int shift : {0, 1, 3, 8, 13, 31}) {
    kern<<<1, 128>>>(A, B, D, shift);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)hA[(m + shift) * K + k] * hB[n * K + k];
        err = fmax(err, fabs(r - hD[m * N + n]));
      }
    printf("shift %2d rows (%4d B): max|err| = %g\n", shift, shift * 16, err);
  }
  return 0;
}
