// umma_shift_probe.cu -- can shifted-window SS-form tcgen05.mma kind::tf32 replace the im2col converters?
// One CTA per case.  Activations sit in shared memory in the channel-planar band layout the TMA
// produces ([plane][pixel][4 floats], 16 B per pixel per plane); a conv tap is a shift of the band
// by s pixels, i.e. a UMMA descriptor whose start address moves by 16*s bytes.
//   case K: A K-major   A[q][ci] = band[q+s][ci]          (forward / dgrad: M = pixels, K = channels)
//   case W: A MN-major  A[co][q] = dY[q][co], B MN-major B[q][ci] = band[q+s][ci]  (wgrad: K = pixels)
// Also checks what the tensor core does with the low 13 mantissa bits of an fp32 container
// (truncation is what the 3xTF32 split a_lo = a - (a & ~0x1fff) assumes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1912_12675_b200/csrc -o build/umma_shift_probe tools/umma_shift_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace pst::ptx;

constexpr int PIX = 256;                 // band pixels per plane
constexpr int PB = PIX * 16;             // plane bytes
constexpr int MAXP = 16;                 // planes (64 channels)

struct Case {
  int mode;      // 0: K-major A (fwd), 1: MN-major A and B (wgrad)
  int M, N, K;   // MMA shape (K = 8 * ksteps)
  int shift;     // pixel shift of the band operand
  int lbo_sbo_swap;
};

// fwd: D[q][co] = sum_ci band[q+s][ci] * W[co][ci]; W K-major core matrices (8 rows x 16 B), SBO 128, LBO = N*16
// wgrad: D[co][ci] = sum_q dY[q][co] * band[q+s][ci]
__global__ void kern(const float* band, const float* other, float* D, Case c) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sband = sm;                       // MAXP planes of PB bytes
  uint8_t* soth = sm + MAXP * PB;            // weights (fwd) or dY planes (wgrad), up to 2*MAXP planes
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < MAXP * PIX * 4; i += blockDim.x)
    reinterpret_cast<float*>(sband)[i] = band[i];
  if (c.mode == 0) {
    // W[co][ci] (N = co, K = ci) K-major: core (8 co x 4 ci); SBO = 128 (next 8 co), LBO = (N/8)*128 (next 4 ci)
    for (int i = threadIdx.x; i < c.N * c.K; i += blockDim.x) {
      const int n = i / c.K, k = i % c.K;
      const int off = (n / 8) * 128 + (k / 4) * ((c.N / 8) * 128) + (n % 8) * 16 + (k % 4) * 4;
      *reinterpret_cast<float*>(soth + off) = other[n * c.K + k];
    }
  } else if (c.mode == 4) {
    // W[co][ci] as MN-major B (N = co, K = ci): [co/4][ci][4], SBO = K*16 (next 4 co), LBO = 128 (next 8 ci)
    for (int i = threadIdx.x; i < c.N * c.K; i += blockDim.x) {
      const int n = i / c.K, k = i % c.K;
      *reinterpret_cast<float*>(soth + (n / 4) * (c.K * 16) + k * 16 + (n % 4) * 4) = other[n * c.K + k];
    }
  } else {
    for (int i = threadIdx.x; i < 2 * MAXP * PIX * 4; i += blockDim.x)
      reinterpret_cast<float*>(soth)[i] = other[i];
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tptr, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tptr;
  if (threadIdx.x < 32) {
    if (c.mode == 0 || c.mode == 3 || c.mode == 4) {
      const uint32_t idesc = idesc_mma(c.M, c.N, 0, c.mode == 4, 2);
      for (int ks = 0; ks < c.K / 8; ++ks) {
        // A: rows q (8-row groups 128 B apart), K chunks = planes (PB apart); two planes per K=8 step
        const uint32_t a0 = smem_u32(sband) + (uint32_t)(2 * ks) * PB + (uint32_t)c.shift * 16;
        const uint64_t ad = (c.lbo_sbo_swap && c.mode == 0) ? smem_desc(a0, 128, PB) : smem_desc(a0, PB, 128);
        const uint32_t b0 = smem_u32(soth) + (uint32_t)(2 * ks) * ((c.N / 8) * 128);
        uint64_t bd = smem_desc(b0, (c.N / 8) * 128, 128);
        if (c.mode == 4) {
          const uint32_t b4 = smem_u32(soth) + (uint32_t)ks * 128;
          bd = c.lbo_sbo_swap ? smem_desc(b4, c.K * 16, 128) : smem_desc(b4, 128, c.K * 16);
        }
        if (elect_one()) umma_tf32(tm, ad, bd, idesc, ks > 0);
        __syncwarp();
      }
    } else {
      const uint32_t idesc = idesc_mma(c.M, c.N, 1, c.mode == 1, 2);
      for (int ks = 0; ks < c.K / 8; ++ks) {
        // MN-major: core = 16 B along M/N (4 channels) x 8 K rows (pixels, 16 B apart);
        // M/N chunks = planes (PB apart), K groups = next 8 pixels (128 B)
        const uint32_t a0 = smem_u32(soth) + (uint32_t)ks * 128;
        const uint32_t b0 = smem_u32(sband) + (uint32_t)ks * 128 + (uint32_t)c.shift * 16;
        const uint64_t ad = c.lbo_sbo_swap ? smem_desc(a0, PB, 128) : smem_desc(a0, 128, PB);
        uint64_t bd = c.lbo_sbo_swap ? smem_desc(b0, PB, 128) : smem_desc(b0, 128, PB);
        if (c.mode == 2) {   // B = weights K-major (N = ci, K = pixel): [n/8][k/4] core matrices
          const uint32_t w0 = smem_u32(sband) + (uint32_t)(2 * ks) * ((c.N / 8) * 128);
          bd = smem_desc(w0, (c.N / 8) * 128, 128);
        }
        if (elect_one()) umma_tf32(tm, ad, bd, idesc, ks > 0);
        __syncwarp();
      }
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  // dump all 128 lanes x N columns
  for (int c0 = 0; c0 < c.N; c0 += 16) {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(threadIdx.x & ~31) << 16) + (uint32_t)c0, v);
    for (int j = 0; j < 16; ++j) D[threadIdx.x * 256 + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tm, 256);
}

static float trunc_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= ~0x1fffu;
  memcpy(&x, &u, 4);
  return x;
}
static float rn_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x1000u;
  u &= ~0x1fffu;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  std::vector<float> band(MAXP * PIX * 4), oth(2 * MAXP * PIX * 4), wt(256 * 64), D(128 * 256);
  srand(3);
  auto rnd = [] { return (float)((rand() % 2001) - 1000) / 997.0f; };
  for (auto& x : band) x = rnd();
  for (auto& x : oth) x = rnd();
  for (auto& x : wt) x = rnd();
  float *dband, *doth, *dwt, *dD;
  cudaMalloc(&dband, band.size() * 4); cudaMalloc(&doth, oth.size() * 4); cudaMalloc(&dwt, wt.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dband, band.data(), band.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(doth, oth.data(), oth.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dwt, wt.data(), wt.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 3 * MAXP * PB + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  auto B = [&](int q, int ch) { return band[(ch / 4) * PIX * 4 + q * 4 + ch % 4]; };
  auto Y = [&](int q, int ch) { return oth[(ch / 4) * PIX * 4 + q * 4 + ch % 4]; };
  std::vector<Case> cases;
  for (int sw = 0; sw < 2; ++sw) {
    cases.push_back({2, 128, 16, 16, 0, sw});
    cases.push_back({2, 128, 32, 32, 0, sw});
    cases.push_back({3, 64, 16, 16, 0, sw});
    cases.push_back({3, 64, 32, 32, 5, sw});
    cases.push_back({4, 128, 16, 16, 0, sw});
    cases.push_back({4, 128, 32, 32, 3, sw});
  }
  for (int sw = 0; sw < 2; ++sw)
    for (int s : {0, 17}) {
      cases.push_back({0, 128, 16, 16, s, sw});
      cases.push_back({0, 128, 32, 64, s, sw});
      cases.push_back({0, 128, 64, 32, s, sw});
      cases.push_back({1, 64, 16, 64, s, sw});
      cases.push_back({1, 64, 32, 32, s, sw});
      cases.push_back({1, 64, 64, 16, s, sw});
    }
  for (const Case& c : cases) {
    cudaMemset(dD, 0, D.size() * 4);
    kern<<<1, 128, smem>>>(c.mode == 2 ? dwt : dband, (c.mode == 0 || c.mode >= 3) ? dwt : doth, dD, c);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("case mode=%d M=%d N=%d K=%d s=%d swap=%d: error %s\n", c.mode, c.M, c.N, c.K, c.shift, c.lbo_sbo_swap, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    // reference with truncated and round-to-nearest tf32 operands; search each row's TMEM lane
    double et = 0, er = 0, ref_max = 0;
    int lane_pattern_ok = 1, nrow = c.M;
    std::vector<int> lane_of(nrow, -1);
    for (int m = 0; m < nrow; ++m) {
      std::vector<double> rt(c.N), rr(c.N);
      for (int n = 0; n < c.N; ++n) {
        double st = 0, sr = 0;
        for (int k = 0; k < c.K; ++k) {
          float a, b;
          if (c.mode == 0 || c.mode == 3 || c.mode == 4) { a = B(m + c.shift, k); b = wt[n * c.K + k]; }
          else if (c.mode == 2) {
            a = Y(k, m);
            b = wt[((n / 8) * 128 + (k / 4) * ((c.N / 8) * 128) + (n % 8) * 16 + (k % 4) * 4) / 4];
          }
          else { a = Y(k, m); b = B(k + c.shift, n); }
          st += (double)trunc_tf32(a) * trunc_tf32(b);
          sr += (double)rn_tf32(a) * rn_tf32(b);
        }
        rt[n] = st; rr[n] = sr;
        ref_max = fmax(ref_max, fabs(st));
      }
      // expected lane: M=128 -> m; M=64 -> (m/16)*32 + m%16
      int lane = c.M == 128 ? m : (m / 16) * 32 + m % 16;
      double dt = 0, dr = 0;
      for (int n = 0; n < c.N; ++n) {
        dt = fmax(dt, fabs(rt[n] - D[lane * 256 + n]));
        dr = fmax(dr, fabs(rr[n] - D[lane * 256 + n]));
      }
      if (dt > 1e-3 * (1 + ref_max) && dr > 1e-3 * (1 + ref_max)) {
        lane_pattern_ok = 0;
        for (int l = 0; l < 128; ++l) {
          double d2 = 0;
          for (int n = 0; n < c.N; ++n) d2 = fmax(d2, fabs(rt[n] - D[l * 256 + n]));
          if (d2 < 1e-3 * (1 + ref_max)) { lane_of[m] = l; break; }
        }
      }
      et = fmax(et, dt); er = fmax(er, dr);
    }
    int nz = 0;
    for (float v : D) nz += v != 0.f;
    static const char* names[] = {"fwd  K-major A ", "wgrad MN-major A,B", "MN-major A, K-major B", "K-major A M=64", "K-major A, MN-major B"};
    printf("nonzero %5d D0[0..3] %.3f %.3f %.3f %.3f | ", nz, D[0], D[1], D[2], D[3]);
    printf("%s M=%3d N=%2d K=%2d shift=%2d lbo/sbo swap=%d: max|D-ref_trunc| %.3g  max|D-ref_rn| %.3g  (|ref| %.3g) lanes %s",
           names[c.mode], c.M, c.N, c.K, c.shift, c.lbo_sbo_swap, et, er,
           ref_max, lane_pattern_ok ? "ok" : "MISMATCH");
    if (!lane_pattern_ok) {
      printf(" [");
      for (int m = 0; m < 20 && m < nrow; ++m) printf("%d ", lane_of[m]);
      printf("]");
    }
    printf("\n");
  }
  return 0;
}
