// mma_bench.cu -- microbenchmark: cycles per tcgen05.mma (M=128, cta_group::1) on resident
// operands, by kind (f16 / tf32), operand mode (SS no-swizzle, SS 128B-swizzle, A in TMEM)
// and N.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdlib>
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

// mode 0: SS no swizzle; 1: SS 128B swizzle; 2: A in TMEM (B no swizzle).  The issue loop is
// kept lean (descriptors = base + constant offsets, warp-uniform, elect.sync) so the number
// measures the tensor core, not the issuing thread.
template <int KIND, int MODE, int NACC>
__global__ void __launch_bounds__(128, 1) bench(int N, int iters, unsigned long long* out, int commit_every) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* A = smem;                 // 128 rows x 128 B = 16 KB
  uint8_t* B = smem + 16384;         // 256 rows x 128 B = 32 KB
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  if (threadIdx.x < 32) {
    const uint32_t idesc = idesc_mma(128, N, 0, 0, KIND == 1 ? 2 : 1);
    const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
    const uint64_t ad0 = MODE == 1 ? desc_sw128(a0) : smem_desc(a0, 128, 1024);
    const uint64_t bd0 = MODE == 1 ? desc_sw128(b0) : smem_desc(b0, 128, 1024);
    const uint32_t kstep = MODE == 1 ? 2 : 16;   // descriptor units (16 B) per K step
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const uint64_t ad = ad0 + (uint64_t)((kk & 3) * kstep), bd = bd0 + (uint64_t)((kk & 3) * kstep);
        const uint32_t dt = tm + (uint32_t)((kk % NACC) * N);
        if (elect_one()) {
          if (MODE == 2) umma_ts(KIND, dt, tm + 256 + (kk & 3) * 8, bd, idesc);
          else if (KIND == 1) umma_tf32(dt, ad, bd, idesc, 1);
          else umma_f16(dt, ad, bd, idesc, 1);
          if (commit_every && ((kk + 1) % commit_every) == 0) umma_commit(&bar2);
        }
      }
    }
    __syncwarp();
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

template <int KIND, int MODE, int NACC>
void run(int N, unsigned long long* d, int commit_every = 0) {
  const int iters = 128;
  if (N * NACC > (MODE == 2 ? 256 : 512)) return;
  cudaFuncSetAttribute(bench<KIND, MODE, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 1024);
  bench<KIND, MODE, NACC><<<148, 128, 49152 + 1024>>>(N, iters, d, commit_every);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cyc = (double)mx / (iters * 16);
  const double macs = 128.0 * N * (KIND == 1 ? 8 : 16);
  const char* kn[2] = {"f16 ", "tf32"};
  const char* mn[3] = {"SS-noswz", "SS-sw128", "TS(A tmem)"};
  printf("%s %-10s N=%3d nacc=%2d commit/%d  %7.2f cyc/mma  %7.1f MAC/cyc/SM\n", kn[KIND], mn[MODE], N, NACC, commit_every, cyc, macs / cyc);
}

template <int KIND, int MODE>
void sweep(unsigned long long* d) {
  for (int N : {16, 32, 64, 128, 256}) {
    run<KIND, MODE, 1>(N, d);
    run<KIND, MODE, 2>(N, d);
    run<KIND, MODE, 4>(N, d);
    run<KIND, MODE, 8>(N, d);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  for (int ce : {0, 2}) { run<1, 2, 1>(16, d, ce); run<1, 2, 2>(16, d, ce); run<1, 2, 4>(16, d, ce); run<1, 0, 1>(16, d, ce); run<1, 2, 1>(64, d, ce); run<1,2,4>(64,d,ce);}
  return 0;
}
