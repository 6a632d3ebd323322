// mma_bench.cu -- microbenchmark: cycles per tcgen05.mma (M=128, cta_group::1) on resident
// operands, by kind (f16 / tf32), operand mode (SS no-swizzle, SS 128B-swizzle, A in TMEM)
// and N.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1912_12675_b200/csrc/ptx.cuh"

using namespace pst::ptx;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_ts(int kind, uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc) {
  if (kind == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b),
                 "r"(idesc) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a_tmem), "l"(b),
                 "r"(idesc) : "memory");
}

// mode 0: SS no swizzle; 1: SS 128B swizzle; 2: A in TMEM (B no swizzle)
__global__ void __launch_bounds__(128, 1) bench(int kind, int mode, int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* A = smem;                 // 128 rows x 128 B = 16 KB
  uint8_t* B = smem + 16384;         // 256 rows x 128 B = 32 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_mma(128, N, 0, 0, kind == 1 ? 2 : 1);
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad, bd;
        if (mode == 1) { ad = desc_sw128(a0 + kk * 32); bd = desc_sw128(b0 + kk * 32); }
        else { ad = smem_desc(a0 + kk * 256, 128, 1024); bd = smem_desc(b0 + kk * 256, 128, 1024); }
        if (mode == 2) umma_ts(kind, tm, tm + 256 + kk * 8, bd, idesc);
        else if (kind == 1) umma_tf32(tm, ad, bd, idesc, 1);
        else umma_f16(tm, ad, bd, idesc, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024);
  const char* kn[2] = {"f16 ", "tf32"};
  const char* mn[3] = {"SS-noswz", "SS-sw128", "TS(A tmem)"};
  const int iters = 512;
  for (int kind = 0; kind < 2; ++kind)
    for (int mode = 0; mode < 3; ++mode)
      for (int N : {8, 16, 32, 64, 128, 256}) {
        for (int grid : {1, 148}) {
          bench<<<grid, 128, 49152 + 1024>>>(kind, mode, N, iters, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          unsigned long long h[148];
          cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
          unsigned long long mx = 0;
          for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
          const double cyc = (double)mx / (iters * 4);
          const double macs = 128.0 * N * (kind == 1 ? 8 : 16);
          printf("%s %-10s N=%3d grid=%3d  %7.2f cyc/mma  %7.1f MAC/cyc/SM\n", kn[kind], mn[mode], N, grid, cyc,
                 macs / cyc);
        }
      }
  return 0;
}
