// umma_mn_test.cu -- does tcgen05.mma kind::tf32 accept an MN-major A operand (no swizzle)?
// One CTA, M=128, N=16, K=8 (one MMA), A MN-major, B K-major; compares with a CPU product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/umma_mn_test tools/umma_mn_test.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1912_12675_b200/csrc/ptx.cuh"

using namespace pst::ptx;

constexpr int M = 128, N = 16, K = 8;

// A MN-major canonical (no swizzle): ((T,1,m),(8,k)) : ((1,T,SBO),(1T,LBO)), T = 4 tf32 per 16 B
__host__ __device__ inline int a_off(int m, int k, int sbo, int lbo) {
  return (m / 4) * sbo + (k / 8) * lbo + (k % 8) * 16 + (m % 4) * 4;
}
// B K-major: ((8,n),(T,2k)) : ((1T,SBO),(1,LBO))
__host__ __device__ inline int b_off(int n, int k, int sbo, int lbo) {
  return (n / 8) * sbo + (k / 4) * lbo + (n % 8) * 16 + (k % 4) * 4;
}

__global__ void kern(const float* A, const float* B, float* D, int a_sbo, int a_lbo, int swap) {
  __shared__ __align__(1024) uint8_t sa[32768];
  __shared__ __align__(1024) uint8_t sb[4096];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *reinterpret_cast<float*>(sa + a_off(m, k, a_sbo, a_lbo)) = A[m * K + k];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<float*>(sb + b_off(n, k, 128, 256)) = B[n * K + k];
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 32);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_mma(M, N, 1, 0, 2);
    // descriptor: LBO field / SBO field; `swap` exchanges which stride goes where
    const uint64_t ad = swap ? smem_desc(smem_u32(sa), a_sbo, a_lbo) : smem_desc(smem_u32(sa), a_lbo, a_sbo);
    const uint64_t bd = smem_desc(smem_u32(sb), 256, 128);
    if (elect_one()) {
      umma_tf32(tm, ad, bd, idesc, 0);
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 128) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(threadIdx.x & ~31) << 16), v);
    for (int j = 0; j < 16; ++j) D[threadIdx.x * N + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 32);
}

int main() {
  float hA[M * K], hB[N * K], hD[M * N];
  srand(1);
  for (auto& x : hA) x = (float)(rand() % 17 - 8);
  for (auto& x : hB) x = (float)(rand() % 13 - 6);
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  struct { int sbo, lbo; } cfgs[] = {{128, 4096}, {256, 128}, {128, 128 * 32}};
  for (auto c : cfgs)
    for (int swap = 0; swap < 2; ++swap) {
      cudaMemset(D, 0, sizeof hD);
      kern<<<1, 128>>>(A, B, D, c.sbo, c.lbo, swap);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
      double err = 0, ref_max = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double r = 0;
          for (int k = 0; k < K; ++k) r += (double)hA[m * K + k] * hB[n * K + k];
          err = fmax(err, fabs(r - hD[m * N + n]));
          ref_max = fmax(ref_max, fabs(r));
        }
      printf("A MN-major sbo=%d lbo=%d swap=%d: max|err| = %g (max|ref| %g)  D[0..3] = %g %g %g %g\n", c.sbo, c.lbo,
             swap, err, ref_max, hD[0], hD[1], hD[2], hD[3]);
    }
  return 0;
}
