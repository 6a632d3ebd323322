// ffma_wgrad_bench.cu -- experiment: the 3x3 weight gradient of the ResNet-CIFAR layer shapes on the
// FP32 pipe (FFMA, exact float32 products) instead of 3xTF32 tcgen05 tiles.
//   dW[tap][ci][co] = sum_p X[p shifted by tap][ci] * dY[p][co]      (k = 3, pad = 1, stride S)
// Layout: channel-planar float32 [C/4][N][H][W][4] (libpst act_t).  One thread owns a 4-ci x 4-co
// plane pair and a run of output rows; it slides a 3x3 window of float4 input columns along x and
// does 144 FFMAs per output pixel from 4 (S=1) or 7 (S=2) float4 loads.  Partials per block are
// written as [ks][tap*Cin + ci][Cout] and summed by a second kernel (deterministic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_wgrad_bench tools/ffma_wgrad_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ float4 ld4(const float* base, bool ok) {
  return ok ? __ldg(reinterpret_cast<const float4*>(base)) : make_float4(0.f, 0.f, 0.f, 0.f);
}

#define FMA16(ACC, XV, DV)                                                          \
  do {                                                                              \
    ACC[0] += XV.x * DV.x; ACC[1] += XV.x * DV.y; ACC[2] += XV.x * DV.z; ACC[3] += XV.x * DV.w; \
    ACC[4] += XV.y * DV.x; ACC[5] += XV.y * DV.y; ACC[6] += XV.y * DV.z; ACC[7] += XV.y * DV.w; \
    ACC[8] += XV.z * DV.x; ACC[9] += XV.z * DV.y; ACC[10] += XV.z * DV.z; ACC[11] += XV.z * DV.w; \
    ACC[12] += XV.w * DV.x; ACC[13] += XV.w * DV.y; ACC[14] += XV.w * DV.z; ACC[15] += XV.w * DV.w; \
  } while (0)

// grid: (ksplit, (Cin/4)*(Cout/4)); block: T threads; task = one output row (n, yo)
template <int S, int WO, int T>
__global__ void __launch_bounds__(T) wgrad_ffma_kernel(const float* __restrict__ X, const float* __restrict__ DY,
                                                       float* __restrict__ part, int N, int H, int W, int Cin,
                                                       int Ho, int Cout) {
  const int a = blockIdx.y % (Cin / 4), b = blockIdx.y / (Cin / 4);
  const int64_t xpl = (int64_t)N * H * W, dpl = (int64_t)N * Ho * WO;
  const float* Xa = X + (int64_t)a * xpl * 4;
  const float* Db = DY + (int64_t)b * dpl * 4;
  float acc[9][16];
#pragma unroll
  for (int t = 0; t < 9; ++t)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[t][i] = 0.f;
  const int ntask = N * Ho;
  for (int task = blockIdx.x * T + threadIdx.x; task < ntask; task += gridDim.x * T) {
    const int n = task / Ho, yo = task - n * Ho;
    const float* rows[3];
    bool rok[3];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      const int yi = S * yo - 1 + dy;
      rok[dy] = yi >= 0 && yi < H;
      rows[dy] = Xa + ((int64_t)(n * H + (rok[dy] ? yi : 0)) * W) * 4;
    }
    const float* drow = Db + ((int64_t)(n * Ho + yo) * WO) * 4;
    float4 win[3][3];
    // column xi = -1 (zero padding) and 0
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      win[dy][0] = make_float4(0.f, 0.f, 0.f, 0.f);
      win[dy][1] = ld4(rows[dy], rok[dy]);
    }
#pragma unroll
    for (int xo = 0; xo < WO; ++xo) {
      const float4 d = __ldg(reinterpret_cast<const float4*>(drow + xo * 4));
      if (S == 1) {
        const int xi = xo + 1;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) win[dy][2] = ld4(rows[dy] + xi * 4, rok[dy] && xi < W);
      } else {
        const int x0 = 2 * xo - 1;
        if (xo > 0) {
#pragma unroll
          for (int dy = 0; dy < 3; ++dy) win[dy][0] = win[dy][2];
        }
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          win[dy][1] = ld4(rows[dy] + (x0 + 1) * 4, rok[dy]);
          win[dy][2] = ld4(rows[dy] + (x0 + 2) * 4, rok[dy] && x0 + 2 < W);
        }
      }
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) FMA16(acc[dy * 3 + dx], win[dy][dx], d);
      if (S == 1) {
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) { win[dy][0] = win[dy][1]; win[dy][1] = win[dy][2]; }
      }
    }
  }
  // block reduction: warp shuffles, then the warps through shared memory
  __shared__ float red[T / 32][144];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < 9; ++t)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float v = acc[t][i];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp][t * 16 + i] = v;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < 144; e += T) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < T / 32; ++w) v += red[w][e];
    const int t = e / 16, i = (e % 16) / 4, j = e % 4;
    const int row = t * Cin + 4 * a + i, col = 4 * b + j;
    part[((int64_t)blockIdx.x * 9 * Cin + row) * Cout + col] = v;
  }
}

__global__ void sum_parts(const float* part, int ks, int n, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int k = 0; k < ks; ++k) s += part[(int64_t)k * n + i];
  out[i] = s;
}

// reference: one thread per dW element, fp64 accumulation
__global__ void wgrad_ref(const float* X, const float* DY, double* out, int N, int H, int W, int Cin, int Ho, int Wo,
                          int Cout, int S) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 9 * Cin * Cout) return;
  const int co = idx % Cout, row = idx / Cout, t = row / Cin, ci = row % Cin;
  const int dy = t / 3, dx = t % 3;
  const int64_t xpl = (int64_t)N * H * W, dpl = (int64_t)N * Ho * Wo;
  double s = 0.0;
  for (int n = 0; n < N; ++n)
    for (int yo = 0; yo < Ho; ++yo)
      for (int xo = 0; xo < Wo; ++xo) {
        const int yi = S * yo - 1 + dy, xi = S * xo - 1 + dx;
        if (yi < 0 || yi >= H || xi < 0 || xi >= W) continue;
        const double xv = X[((ci / 4) * xpl + (n * H + yi) * W + xi) * 4 + ci % 4];
        const double dv = DY[((co / 4) * dpl + (n * Ho + yo) * Wo + xo) * 4 + co % 4];
        s += xv * dv;
      }
  out[idx] = s;
}

template <int S, int WO, int T>
float run(int N, int H, int W, int Cin, int Cout, int ks, float* dX, float* dD, float* part, float* out, int reps) {
  const int Ho = (H - 1) / S + 1;
  dim3 grid(ks, (Cin / 4) * (Cout / 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int n = 9 * Cin * Cout;
  for (int r = 0; r < 3; ++r) {
    wgrad_ffma_kernel<S, WO, T><<<grid, T>>>(dX, dD, part, N, H, W, Cin, Ho, Cout);
    sum_parts<<<(n + 255) / 256, 256>>>(part, ks, n, out);
  }
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) wgrad_ffma_kernel<S, WO, T><<<grid, T>>>(dX, dD, part, N, H, W, Cin, Ho, Cout);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  sum_parts<<<(n + 255) / 256, 256>>>(part, ks, n, out);
  CK(cudaDeviceSynchronize());
  return 1e3f * ms / reps;
}

template <int S, int WO, int T>
void shape(const char* name, int N, int H, int W, int Cin, int Cout) {
  const int Ho = (H - 1) / S + 1, Wo = (W - 1) / S + 1;
  if (Wo != WO) { printf("bad WO\n"); return; }
  const size_t nx = (size_t)N * H * W * Cin, nd = (size_t)N * Ho * Wo * Cout;
  std::vector<float> hx(nx), hd(nd);
  srand(1);
  for (auto& v : hx) v = (float)rand() / RAND_MAX - 0.5f;
  for (auto& v : hd) v = (float)rand() / RAND_MAX - 0.5f;
  float *dX, *dD, *part, *out;
  double* ref;
  const int n = 9 * Cin * Cout;
  CK(cudaMalloc(&dX, nx * 4));
  CK(cudaMalloc(&dD, nd * 4));
  CK(cudaMalloc(&part, (size_t)512 * n * 4));
  CK(cudaMalloc(&out, n * 4));
  CK(cudaMalloc(&ref, n * 8));
  CK(cudaMemcpy(dX, hx.data(), nx * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dD, hd.data(), nd * 4, cudaMemcpyHostToDevice));
  wgrad_ref<<<(n + 127) / 128, 128>>>(dX, dD, ref, N, H, W, Cin, Ho, Wo, Cout, S);
  CK(cudaDeviceSynchronize());
  std::vector<double> hr(n);
  CK(cudaMemcpy(hr.data(), ref, n * 8, cudaMemcpyDeviceToHost));
  const double flops = 2.0 * n * (double)N * Ho * Wo;
  for (int ks : {8, 16, 32, 64, 128}) {
    if ((size_t)ks * n > (size_t)512 * n) continue;
    const float us = run<S, WO, T>(N, H, W, Cin, Cout, ks, dX, dD, part, out, 50);
    std::vector<float> ho(n);
    CK(cudaMemcpy(ho.data(), out, n * 4, cudaMemcpyDeviceToHost));
    double err = 0, mx = 0;
    for (int i = 0; i < n; ++i) { err = fmax(err, fabs(ho[i] - hr[i])); mx = fmax(mx, fabs(hr[i])); }
    printf("%-24s T=%d ks=%3d blocks=%5d  %8.2f us  %6.1f TFLOP/s  rel err %.2e\n", name, T, ks,
           ks * (Cin / 4) * (Cout / 4), us, flops / us * 1e-6, err / mx);
  }
  cudaFree(dX); cudaFree(dD); cudaFree(part); cudaFree(out); cudaFree(ref);
}

int main() {
  shape<1, 32, 128>("g1 16->16 32x32", 128, 32, 32, 16, 16);
  shape<1, 32, 64>("g1 16->16 32x32", 128, 32, 32, 16, 16);
  shape<1, 16, 128>("g2 32->32 16x16", 128, 16, 16, 32, 32);
  shape<1, 16, 64>("g2 32->32 16x16", 128, 16, 16, 32, 32);
  shape<1, 8, 128>("g3 64->64 8x8", 128, 8, 8, 64, 64);
  shape<1, 8, 64>("g3 64->64 8x8", 128, 8, 8, 64, 64);
  shape<2, 16, 128>("s2 16->32 32x32", 128, 32, 32, 16, 32);
  shape<2, 8, 128>("s2 32->64 16x16", 128, 16, 16, 32, 64);
  return 0;
}
