// mma_bench3.cu -- conv_ts issue pattern: M=128 kind::tf32 TS MMAs at N=16/32/64, accumulating
// into NACC independent accumulators, optionally with 8 warps streaming tcgen05.st into other
// TMEM columns at the same time (the converters).  Prints cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1912_12675_b200/csrc/ptx.cuh"
using namespace pst::ptx;

template <int NACC, int STORES>
__global__ void __launch_bounds__(320, 1) bench(int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const uint32_t idesc = idesc_mma(128, N, 0, 0, 2);
    const uint64_t bd0 = smem_desc(smem_u32(smem), N * 16, 128);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 18; ++kk)
          umma_tf32_ts(tm + (kk % NACC) * N, tm + 256 + (kk % 6) * 8, desc_add(bd0, (kk % 6) * 256), idesc, 1);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = (unsigned long long)(t1 - t0); stop = 1; }
  } else if (warp >= 2 && STORES) {
    const int q = warp & 3;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = (float)i;
    int n = 0;
    while (!stop && n < 100000) {
      if (STORES == 1) {
        tmem_st16(tm + lane_addr + 320 + ((warp >> 2) & 1) * 64 + (n & 1) * 16, v);
        tmem_st16(tm + lane_addr + 352 + ((warp >> 2) & 1) * 64 + (n & 1) * 16, v);
      } else {
#pragma unroll
        for (int j = 0; j < 6; ++j) tmem_st16(tm + lane_addr + 320 + ((warp >> 2) & 1) * 96 + j * 16, v);
      }
      tmem_st_wait();
      ++n;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

template <int NACC, int STORES>
void run(int N, unsigned long long* d) {
  const int iters = 256;
  cudaFuncSetAttribute(bench<NACC, STORES>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  bench<NACC, STORES><<<148, 320, 32768>>>(N, iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("N=%3d nacc=%d stores=%d: %7.2f cyc/mma\n", N, NACC, (int)STORES, (double)mx / (iters * 18));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  for (int N : {16, 32, 64}) {
    run<1, 0>(N, d); run<3, 0>(N, d);
    run<1, 1>(N, d); run<3, 1>(N, d); run<1, 2>(N, d); run<3, 2>(N, d);
  }
  return 0;
}
