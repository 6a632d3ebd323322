// mma_bench4.cu -- the conv_ts MMA issue loop in isolation (KC=16, BN=16, tps=3, weights of 9
// taps hi|lo resident in smem, A slots in TMEM), no waits: cycles per MMA.  MODE 0: as conv_ts
// (3 MMAs per K step: hi*hi, hi*lo, lo*hi, N=16); MODE 1: hi*[hi|lo] as one N=32 MMA + lo*hi.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1912_12675_b200/csrc/ptx.cuh"
using namespace pst::ptx;

template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  if (threadIdx.x < 32) {
    const int BN = 16, KC = 16, taps = 9;
    const uint32_t w_bytes = taps * 16 * BN * 4;           // hi plane: [tap][Cin/4][BN][4]
    const uint32_t idesc = idesc_mma(128, BN, 0, 0, 2);
    const uint32_t idesc32 = idesc_mma(128, 2 * BN, 0, 0, 2);
    const uint32_t wtap = 4 * BN * 16;
    const uint64_t wdesc = smem_desc(smem_u32(smem), BN * 16, 128);
    const uint64_t wdesc32 = smem_desc(smem_u32(smem), 2 * BN * 16, 128);   // interleaved [hi|lo] rows
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int g = 0; g < 3; ++g) {
        const int slot = (it * 3 + g) % 5;
        if (elect_one()) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            const int t = g * 3 + i;
            const uint32_t ahi = tm + 32 + (slot * 3 + i) * 2 * KC;
            if (MODE == 0) {
              const uint64_t bt = desc_add(wdesc, t * wtap);
#pragma unroll
              for (int kk = 0; kk < KC / 8; ++kk) {
                const uint64_t bd = desc_add(bt, 2 * kk * (BN * 16));
                const uint64_t bdl = desc_add(bd, w_bytes);
                umma_tf32_ts(tm, ahi + kk * 8, bd, idesc, 1u);
                umma_tf32_ts(tm, ahi + kk * 8, bdl, idesc, 1u);
                umma_tf32_ts(tm, ahi + KC + kk * 8, bd, idesc, 1u);
              }
            } else {
              const uint64_t bt = desc_add(wdesc32, t * 2 * wtap);
#pragma unroll
              for (int kk = 0; kk < KC / 8; ++kk) {
                const uint64_t bd = desc_add(bt, 2 * kk * (2 * BN * 16));
                umma_tf32_ts(tm, ahi + kk * 8, bd, idesc32, 1u);
                umma_tf32_ts(tm + 16, ahi + KC + kk * 8, bd, idesc, 1u);
              }
            }
          }
        }
        __syncwarp();
      }
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

template <int MODE>
void run(unsigned long long* d) {
  const int iters = 200;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  bench<MODE><<<148, 128, 65536>>>(iters, d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ksteps = (double)iters * 3 * 3 * 2;   // (tap, kk) steps
  printf("mode %d: %7.2f cyc per (tap,kk) step, %7.2f cyc per tile (18 steps)\n", MODE, mx / ksteps, 18 * mx / ksteps);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  run<0>(d); run<1>(d);
  return 0;
}
