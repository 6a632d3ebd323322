// ss_conv_bench.cu -- cycles per 128-pixel conv tile of the shifted-window SS form (kind::tf32, 3xTF32:
// per tap and K step of 8 channels, A_raw x [W_hi|W_lo] (N = 2*Cout) and A_lo x W_hi (N = Cout);
// A read from the shared-memory band at a 16*shift byte offset, no im2col).  One CTA per SM, the MMA
// warp issues TILES tiles into two alternating TMEM accumulators, committing each tile to an mbarrier
// and waiting for tile t-1 before issuing tile t+1 (the real kernel's double-buffered accumulator).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1912_12675_b200/csrc -o build/ss_conv_bench tools/ss_conv_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace pst::ptx;

constexpr int TILES = 64;

template <int CIN, int COUT, int WP>   // WP = padded row width (W + 2)
__global__ void __launch_bounds__(128, 1) kern(long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int BAND = 128 + 2 * WP + 2 + 8;      // band pixels
  constexpr int PB = BAND * 16;                   // plane bytes
  constexpr int PLANES = CIN / 4;
  uint8_t* sraw = sm;
  uint8_t* slo = sm + PLANES * PB;
  uint8_t* sw = slo + PLANES * PB;                // weights: 9 taps x (hi|lo stacked N) ; K-major
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < (2 * PLANES * PB + 9 * 2 * COUT * CIN * 4) / 4; i += blockDim.x)
    reinterpret_cast<float*>(sm)[i] = 0.001f * (i % 97);
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint32_t id2 = idesc_mma(128, 2 * COUT, 0, 0, 2);
    const uint32_t id1 = idesc_mma(128, COUT, 0, 0, 2);
    // weights per tap: [hi rows (COUT) | lo rows (COUT)] stacked along N, K-major cores (8 rows x 16 B):
    // SBO = 128 (next 8 N rows), LBO = (2*COUT/8)*128 (next 4 input channels)
    constexpr uint32_t WLBO = (2 * COUT / 8) * 128;
    constexpr uint32_t WTAP = WLBO * (CIN / 4);
    const uint64_t a_raw = smem_desc(smem_u32(sraw), PB, 128);
    const uint64_t a_lo = smem_desc(smem_u32(slo), PB, 128);
    const uint64_t w0 = smem_desc(smem_u32(sw), WLBO, 128);
    for (int t = 0; t < TILES; ++t) {
      const uint32_t acc = tm + (uint32_t)(t & 1) * 128;
      if (t >= 2) mbar_wait(&bar[t & 1], ((t >> 1) - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const uint32_t sh = (uint32_t)((tap / 3) * WP + tap % 3) * 16;
#pragma unroll
        for (int ks = 0; ks < CIN / 8; ++ks) {
          const uint32_t ko = (uint32_t)(2 * ks) * PB + sh;
          const uint64_t wd = desc_add(w0, tap * WTAP + 2 * ks * WLBO);
          if (elect_one()) {
            umma_tf32(acc, desc_add(a_raw, ko), wd, id2, (tap | ks) != 0);
            umma_tf32(acc, desc_add(a_lo, ko), wd, id1, 1);
          }
          __syncwarp();
        }
      }
      if (elect_one()) umma_commit(&bar[t & 1]);
      __syncwarp();
    }
    mbar_wait(&bar[(TILES - 1) & 1], ((TILES - 1) >> 1) & 1);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 256);
}

template <int CIN, int COUT, int WP>
void run(const char* name) {
  constexpr int BAND = 128 + 2 * WP + 2 + 8;
  const int smem = 2 * (CIN / 4) * BAND * 16 + 9 * 2 * COUT * CIN * 4 + 1024;
  cudaFuncSetAttribute(kern<CIN, COUT, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<CIN, COUT, WP><<<148, 128, smem>>>(d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: error %s\n", name, cudaGetErrorString(e)); exit(1); }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (long long v : h) mx = v > mx ? v : mx;
    const double macs = 128.0 * 9 * CIN * 3 * COUT;   // useful 3xTF32 MACs per tile
    printf("%s Cin=%d Cout=%d W+2=%d: %.0f cyc/tile (%.1f cyc/MMA), %.1f TF32-MAC/cyc/SM, kernel %.1f us for %d tiles/SM\n",
           name, CIN, COUT, WP, (double)mx / TILES, (double)mx / TILES / (9 * CIN / 8 * 2), macs * TILES / mx, ms * 1e3, TILES);
  }
  cudaFree(d);
}

int main() {
  run<16, 16, 34>("g1");
  run<32, 32, 18>("g2");
  run<64, 32, 10>("g3 (N half)");
  return 0;
}
