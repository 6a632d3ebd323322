// mma_bench2.cu -- issue-structure microbenchmark: cycles per TS-mode kind::tf32 MMA (M=128, N=16)
// when issued in groups of G MMAs per elected region, with/without a tcgen05.commit per group,
// with/without an mbarrier wait per group (the conv_ts MMA-warp pattern).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1912_12675_b200/csrc/ptx.cuh"
using namespace pst::ptx;

template <int G, bool COMMIT, bool WAIT>
__global__ void __launch_bounds__(128, 1) bench(int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); mbar_init(&bar3, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_mma(128, N, 0, 0, 2);
    const uint64_t bd0 = smem_desc(smem_u32(smem), 128, 1024);
    if (WAIT && elect_one()) mbar_arrive(&bar3);   // bar3 phase 0 completes: waits below pass
    __syncwarp();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (WAIT) mbar_wait(&bar3, 0);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < G; ++kk)
          umma_tf32_ts(tm + (kk & 1) * 16, tm + 256 + (kk & 3) * 8, desc_add(bd0, (kk & 3) * 256), idesc, 1);
        if (COMMIT) umma_commit(&bar2);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

template <int G, bool COMMIT, bool WAIT>
void run(unsigned long long* d) {
  const int iters = 2048 / G;
  cudaFuncSetAttribute(bench<G, COMMIT, WAIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  bench<G, COMMIT, WAIT><<<148, 128, 32768>>>(16, iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("G=%2d commit=%d wait=%d: %7.2f cyc/mma\n", G, (int)COMMIT, (int)WAIT, (double)mx / (iters * G));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  run<1, false, false>(d); run<6, false, false>(d); run<12, false, false>(d); run<24, false, false>(d);
  run<1, true, false>(d); run<6, true, false>(d); run<12, true, false>(d); run<24, true, false>(d);
  run<6, false, true>(d); run<6, true, true>(d); run<12, true, true>(d); run<24, true, true>(d);
  return 0;
}
