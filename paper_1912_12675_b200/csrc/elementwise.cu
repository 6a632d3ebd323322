// elementwise.cu -- HBM-bound kernels of the hot path: layout conversion, BatchNorm
// (train mode) forward apply and backward, ReLU/pool backward, max/avg pooling,
// gradient dilation, softmax cross-entropy, fused SGD-momentum update.
//
// Activation layout ("channel-planar", see kernels.h): element (n, c, y, x) of a
// tensor with Cp channels lives at ((c/EPC)*NPIX + (n*H + y)*W + x)*EPC + c%EPC,
// EPC = 16 bytes / sizeof(act_t).  A tensor is therefore a flat array of 16-byte
// vectors v = plane*NPIX + pixel; every kernel moves one vector per thread per
// iteration (coalesced), and per-channel reductions run over one plane per block.
#include "kernels.h"

#include <algorithm>

namespace pst {

namespace {

constexpr int kBlock = 256;
constexpr int E = kEPC;   // channels per 16-byte vector

__device__ __forceinline__ void ldv(const act_t* p, float* f) {
  alignas(16) act_t h[E];
  *reinterpret_cast<uint4*>(h) = *reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < E; ++i) f[i] = act2f(h[i]);
}
__device__ __forceinline__ void stv(act_t* p, const float* f) {
  alignas(16) act_t h[E];
#pragma unroll
  for (int i = 0; i < E; ++i) h[i] = f2act(f[i]);
  *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(h);
}

int grid_for(int64_t work, int per_block = kBlock) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = num_sms(dev);
  int64_t g = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 8));
}

// ------------------------------------------------------------------ layout conversion
__global__ void nchw_to_act_kernel(const float* __restrict__ x, act_t* __restrict__ out, int N, int C, int H,
                                   int W, int Cp) {
  pdl_wait();
  pdl_trigger();
  const int64_t npix = (int64_t)N * H * W;
  const int64_t nvec = npix * (Cp / E);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int plane = (int)(v / npix);
    const int64_t p = v % npix;
    const int n = (int)(p / ((int64_t)H * W));
    const int hw = (int)(p % ((int64_t)H * W));
    float f[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int c = plane * E + i;
      f[i] = c < C ? __ldg(&x[((int64_t)n * C + c) * H * W + hw]) : 0.f;
    }
    stv(out + v * E, f);
  }
}

__global__ void act_to_nchw_kernel(const void* in, int in_f32, float* out, int N, int C, int H, int W) {
  pdl_wait();
  pdl_trigger();
  const int64_t n_el = (int64_t)N * C * H * W;
  const int64_t npix = (int64_t)N * H * W;
  const int e = in_f32 ? 4 : E;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_el; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % W);
    const int y = (int)((i / W) % H);
    const int c = (int)((i / ((int64_t)W * H)) % C);
    const int n = (int)(i / ((int64_t)W * H * C));
    const int64_t p = ((int64_t)n * H + y) * W + x;
    const int64_t src = ((int64_t)(c / e) * npix + p) * e + c % e;
    out[i] = in_f32 ? reinterpret_cast<const float*>(in)[src] : act2f(reinterpret_cast<const act_t*>(in)[src]);
  }
}

// ------------------------------------------------------------------ BN forward apply
// grid (x = pixel chunks of kU*kBlock vectors, y = channel plane): 32-bit pixel indices, the
// plane's 4 scale/shift pairs in registers, kU independent 16-byte loads in flight per thread.
#ifndef PST_KU
#define PST_KU 4
#endif
constexpr int kU = PST_KU;   // 16-byte vectors per thread per pass (plane-blocked kernels)
__global__ void bn_apply_kernel(const BnApplySpec s) {
  pdl_wait();
  pdl_trigger();
  // per-warp coefficients (lanes 0..E-1 compute, shuffles broadcast): no block-wide barrier
  const int plane = blockIdx.y;
  const int c0 = plane * E;
  const int npix = s.N * s.H * s.W;
  const double M = (double)npix;
  const int lane = threadIdx.x & 31;
  float my_scale = 0.f, my_shift = 0.f;
  if (lane < E && c0 + lane < s.C) {
    const int c = c0 + lane;
    const double mean = s.stats[2 * c] / M;
    double var = s.stats[2 * c + 1] / M - mean * mean;
    var = var < 0.0 ? 0.0 : var;
    const float invstd = (float)(1.0 / sqrt(var + (double)s.eps));
    const float g = s.gamma[c], b = s.beta[c];
    my_scale = g * invstd;
    my_shift = b - (float)mean * g * invstd;
    if (blockIdx.x == 0 && threadIdx.x < 32) {
      s.saved[2 * c] = (float)mean;
      s.saved[2 * c + 1] = invstd;
      s.run_mean[c] = (1.f - s.momentum) * s.run_mean[c] + s.momentum * (float)mean;
      s.run_var[c] = (1.f - s.momentum) * s.run_var[c] + s.momentum * (float)(var * M / (M - 1.0));
    }
  }
  float scale[E], shift[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    scale[j] = __shfl_sync(0xffffffffu, my_scale, j);
    shift[j] = __shfl_sync(0xffffffffu, my_shift, j);
  }
  const act_t* yp = s.y + (size_t)plane * npix * E;
  act_t* zp = s.z + (size_t)plane * npix * E;
  const int rnpix = s.N * s.res_H * s.res_W;
  const int HW = s.H * s.W;
  for (int base = blockIdx.x * (kU * kBlock); base < npix; base += gridDim.x * (kU * kBlock)) {
    float f[kU][E];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = base + u * kBlock + threadIdx.x;
      if (p < npix) ldv(yp + (size_t)p * E, f[u]);
    }
    if (s.res_mode == 1) {
      const act_t* rp = s.res + (size_t)plane * npix * E;
      float r[kU][E];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int p = base + u * kBlock + threadIdx.x;
        if (p < npix) ldv(rp + (size_t)p * E, r[u]);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int j = 0; j < E; ++j) f[u][j] = f[u][j] * scale[j] + shift[j] + ((c0 + j < s.C) ? r[u][j] : 0.f);
    } else {
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int j = 0; j < E; ++j) f[u][j] = f[u][j] * scale[j] + shift[j];
      if (s.res_mode == 2) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int p = base + u * kBlock + threadIdx.x;
          if (p >= npix) continue;
          const int n = p / HW, hw = p - n * HW;
          const int y = hw / s.W, x = hw - y * s.W;
          const int rp = (n * s.res_H + 2 * y) * s.res_W + 2 * x;
#pragma unroll
          for (int j = 0; j < E; ++j) {
            const int cr = c0 + j - s.res_pad;
            if (cr >= 0 && cr < s.res_Creal) f[u][j] += act2f(s.res[((size_t)(cr / E) * rnpix + rp) * E + cr % E]);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = base + u * kBlock + threadIdx.x;
      if (p >= npix) continue;
      if (s.relu) {
#pragma unroll
        for (int j = 0; j < E; ++j) f[u][j] = fmaxf(f[u][j], 0.f);
      }
      stv(zp + (size_t)p * E, f[u]);
    }
  }
}

// ------------------------------------------------------------------ pooling
__global__ void maxpool2_kernel(const act_t* __restrict__ in, act_t* __restrict__ out, uint8_t* __restrict__ arg,
                                int N, int H, int W, int Cp) {
  pdl_wait();
  pdl_trigger();
  const int Ho = H / 2, Wo = W / 2;
  const int64_t npo = (int64_t)N * Ho * Wo, npi = (int64_t)N * H * W;
  const int64_t nvec = npo * (Cp / E);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int plane = (int)(v / npo);
    const int64_t po = v % npo;
    const int n = (int)(po / ((int64_t)Ho * Wo));
    const int hw = (int)(po % ((int64_t)Ho * Wo));
    const int yo = hw / Wo, xo = hw % Wo;
    float best[E];
    uint8_t a[E];
    for (int q = 0; q < 4; ++q) {
      const int y = 2 * yo + (q >> 1), x = 2 * xo + (q & 1);
      float f[E];
      ldv(in + ((int64_t)plane * npi + ((int64_t)n * H + y) * W + x) * E, f);
#pragma unroll
      for (int j = 0; j < E; ++j) {
        if (q == 0 || f[j] > best[j]) {
          best[j] = f[j];
          a[j] = (uint8_t)q;
        }
      }
    }
    stv(out + v * E, best);
#pragma unroll
    for (int j = 0; j < E; ++j) arg[v * E + j] = a[j];
  }
}

__global__ void gap_kernel(const act_t* __restrict__ in, act_t* __restrict__ out, int N, int H, int W, int Cp) {
  pdl_wait();
  pdl_trigger();
  const int64_t nvec = (int64_t)N * (Cp / E);
  const int HW = H * W;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int plane = (int)(v / N), n = (int)(v % N);
    float acc[E];
#pragma unroll
    for (int j = 0; j < E; ++j) acc[j] = 0.f;
    for (int p = 0; p < HW; ++p) {
      float f[E];
      ldv(in + (((int64_t)plane * N + n) * HW + p) * E, f);
#pragma unroll
      for (int j = 0; j < E; ++j) acc[j] += f[j];
    }
#pragma unroll
    for (int j = 0; j < E; ++j) acc[j] /= (float)HW;
    stv(out + v * E, acc);
  }
}

// ------------------------------------------------------------------ backward pre (pool^T, relu^T, sums)
// grid: (x = pixel chunks, y = channel plane).  All threads of a block share one plane.
__global__ void bwd_pre_kernel(const BwdPreSpec s) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[kBlock / 32][2 * E];
  const int plane = blockIdx.y;
  const int c0 = plane * E;
  const int npix = s.N * s.H * s.W;
  const int HW = s.H * s.W;
  float mean[E], inv[E], a1[E], a2[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    mean[j] = s.bn ? s.saved[2 * (c0 + j)] : 0.f;
    inv[j] = s.bn ? s.saved[2 * (c0 + j) + 1] : 0.f;
    a1[j] = a2[j] = 0.f;
  }
  const size_t pb = (size_t)plane * npix;
  const int Ho2 = s.H / 2, Wo2 = s.W / 2;
  const int npo = s.N * Ho2 * Wo2;
  for (int base = blockIdx.x * (kU * kBlock); base < npix; base += gridDim.x * (kU * kBlock)) {
    float g[kU][E];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = base + u * kBlock + threadIdx.x;
#pragma unroll
      for (int j = 0; j < E; ++j) g[u][j] = 0.f;
      if (p >= npix) continue;
      if (s.pool == 0) {
        if (s.gout_f32) {   // float tensors use 4-channel planes: [Cp/4][npix][4]
          const float* gp = reinterpret_cast<const float*>(s.gout);
#pragma unroll
          for (int j = 0; j < E; ++j) {
            const int c = c0 + j;
            g[u][j] = gp[((size_t)(c >> 2) * npix + p) * 4 + (c & 3)];
          }
        } else {
          ldv(s.gout + (pb + p) * E, g[u]);
        }
      } else if (s.pool == 1) {
        const int n = p / HW, hw = p - n * HW;
        const int y = hw / s.W, x = hw - y * s.W;
        const size_t vo = (size_t)plane * npo + (n * Ho2 + (y >> 1)) * Wo2 + (x >> 1);
        float gg[E];
        ldv(s.gout + vo * E, gg);
        const uint8_t q = (uint8_t)(((y & 1) << 1) | (x & 1));
#pragma unroll
        for (int j = 0; j < E; ++j) g[u][j] = (s.arg[vo * E + j] == q) ? gg[j] : 0.f;
      } else {
        const int n = p / HW;
        float gg[E];
        ldv(s.gout + ((size_t)plane * s.N + n) * E, gg);
#pragma unroll
        for (int j = 0; j < E; ++j) g[u][j] = gg[j] / (float)HW;
      }
    }
    if (s.relu) {
      float z[kU][E];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int p = base + u * kBlock + threadIdx.x;
        if (p < npix) ldv(s.z + (pb + p) * E, z[u]);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int p = base + u * kBlock + threadIdx.x;
        if (p >= npix) continue;
#pragma unroll
        for (int j = 0; j < E; ++j) g[u][j] = z[u][j] > 0.f ? g[u][j] * s.rscale : 0.f;   // dropout scale (or 1)
      }
    }
    float y[kU][E];
    if (s.bn) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int p = base + u * kBlock + threadIdx.x;
        if (p < npix) ldv(s.y + (pb + p) * E, y[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = base + u * kBlock + threadIdx.x;
      if (p >= npix) continue;
#pragma unroll
      for (int j = 0; j < E; ++j) g[u][j] = act2f(f2act(g[u][j]));  // sums use exactly what is stored
      stv(s.gpre + (pb + p) * E, g[u]);
      if (s.bn) {
#pragma unroll
        for (int j = 0; j < E; ++j) {
          a1[j] += g[u][j];
          a2[j] += g[u][j] * (y[u][j] - mean[j]) * inv[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < E; ++j) a1[j] += g[u][j];
      }
    }
  }
  // block reduction (one plane per block)
#pragma unroll
  for (int j = 0; j < E; ++j) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      a1[j] += __shfl_xor_sync(0xffffffffu, a1[j], o);
      a2[j] += __shfl_xor_sync(0xffffffffu, a2[j], o);
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      red[w][2 * j] = a1[j];
      red[w][2 * j + 1] = a2[j];
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * E) {
    float t = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i][threadIdx.x];
    const int c = c0 + (threadIdx.x >> 1);
    if (c < s.C) atomicAdd(&s.sums[2 * c + (threadIdx.x & 1)], (double)t);
  }
}

__global__ void bn_bwd_apply_kernel(const BnBwdSpec s) {
  pdl_wait();
  pdl_trigger();
  // per-warp coefficients (k1, m1, m2, mean, invstd of the plane's channels; lanes 0..E-1, shuffles)
  const int plane = blockIdx.y;
  const int c0 = plane * E;
  const int npix = s.N * s.H * s.W;
  const double M = (double)npix;
  const int lane = threadIdx.x & 31;
  float mk1 = 0.f, mm1 = 0.f, mm2 = 0.f, mmu = 0.f, miv = 0.f;
  if (lane < E && c0 + lane < s.C) {
    const int c = c0 + lane;
    mmu = s.saved[2 * c];
    miv = s.saved[2 * c + 1];
    mk1 = s.gamma[c] * miv;
    mm1 = (float)(s.sums[2 * c] / M);
    mm2 = (float)(s.sums[2 * c + 1] / M);
  }
  float k1[E], m1[E], m2[E], mu[E], iv[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    k1[j] = __shfl_sync(0xffffffffu, mk1, j); m1[j] = __shfl_sync(0xffffffffu, mm1, j);
    m2[j] = __shfl_sync(0xffffffffu, mm2, j); mu[j] = __shfl_sync(0xffffffffu, mmu, j);
    iv[j] = __shfl_sync(0xffffffffu, miv, j);
  }
  const act_t* gp = s.gpre + (size_t)plane * npix * E;
  const act_t* yp = s.y + (size_t)plane * npix * E;
  act_t* op = s.gy + (size_t)plane * npix * E;
  for (int base = blockIdx.x * (kU * kBlock); base < npix; base += gridDim.x * (kU * kBlock)) {
    float g[kU][E], y[kU][E];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = base + u * kBlock + threadIdx.x;
      if (p < npix) { ldv(gp + (size_t)p * E, g[u]); ldv(yp + (size_t)p * E, y[u]); }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int p = base + u * kBlock + threadIdx.x;
      if (p >= npix) continue;
      float o[E];
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const float xh = (y[u][j] - mu[j]) * iv[j];
        o[j] = k1[j] * (g[u][j] - m1[j] - xh * m2[j]);
      }
      stv(op + (size_t)p * E, o);
    }
  }
}

__global__ void dilate2_kernel(const act_t* __restrict__ dy, act_t* __restrict__ out, int N, int Ho, int Wo,
                               int H, int W, int Cp) {
  pdl_wait();
  pdl_trigger();
  const int64_t npo = (int64_t)N * Ho * Wo, npi = (int64_t)N * H * W;
  const int64_t nvec = npi * (Cp / E);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int plane = (int)(v / npi);
    const int64_t p = v % npi;
    const int n = (int)(p / ((int64_t)H * W));
    const int hw = (int)(p % ((int64_t)H * W));
    const int y = hw / W, x = hw % W;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (((y | x) & 1) == 0 && (y >> 1) < Ho && (x >> 1) < Wo)
      val = *reinterpret_cast<const uint4*>(dy + ((int64_t)plane * npo + ((int64_t)n * Ho + (y >> 1)) * Wo + (x >> 1)) * E);
    *reinterpret_cast<uint4*>(out + v * E) = val;
  }
}

// ------------------------------------------------------------------ softmax cross-entropy
// logits / dz: float, 4-channel planes [Cp/4][B][4].
__global__ void softmax_ce_kernel(const float* __restrict__ logits, const int32_t* __restrict__ label_ring, int ring,
                                  float* __restrict__ loss_ring, int64_t* fwd_counter, float* __restrict__ dz, int B,
                                  int C, int Cp) {
  pdl_wait();
  pdl_trigger();
  __shared__ float wsum[32];
  const int64_t f = *fwd_counter;
  const int32_t* labels = label_ring + (f % ring) * B;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  auto at = [&](int b, int c) { return ((int64_t)(c >> 2) * B + b) * 4 + (c & 3); };
  float lsum = 0.f;
  for (int b = warp; b < B; b += nw) {
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = fmaxf(m, logits[at(b, c)]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float se = 0.f;
    for (int c = lane; c < C; c += 32) se += expf(logits[at(b, c)] - m);
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int yb = labels[b];
    const float lse = m + logf(se);
    if (lane == 0) lsum += lse - logits[at(b, yb)];
    for (int c = lane; c < Cp; c += 32) {
      float v = 0.f;
      if (c < C) v = (expf(logits[at(b, c)] - m) / se - (c == yb ? 1.f : 0.f)) / (float)B;
      dz[at(b, c)] = v;
    }
  }
  if (lane == 0) wsum[warp] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < nw; ++w) t += wsum[w];
    loss_ring[f % 1024] = t / (float)B;
    *fwd_counter = f + 1;
  }
}

// ------------------------------------------------------------------ SGD
// shadow index helpers (kernels.h): fwd [tap][Cinp/E][Coutp][E], dgrad [tap][Coutp/E][Cinp][E]
__device__ __forceinline__ int64_t shf_idx(int tap, int co, int ci, int Coutp, int Cinp) {
  return (((int64_t)tap * (Cinp / E) + ci / E) * Coutp + co) * E + ci % E;
}
__device__ __forceinline__ int64_t shb_idx(int tap, int co, int ci, int Coutp, int Cinp) {
  return (((int64_t)tap * (Coutp / E) + co / E) * Cinp + ci) * E + co % E;
}

template <bool kUpdate>
__global__ void sgd_kernel(const SgdSpec s) {
  pdl_wait();      // no early pdl_trigger: the next kernels may read the weights before their pdl_wait

  __shared__ float lr_sh;
  __shared__ int seg_sh;
  __shared__ int last_sh;
  if (threadIdx.x == 0) {
    int lo = 0, hi = s.n_segs - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s.seg_block_start[mid] <= blockIdx.x) lo = mid; else hi = mid - 1;
    }
    seg_sh = lo;
    if (kUpdate) {
      const int64_t vc = *s.v_count;
      const float base = (vc < *s.n_p) ? *s.lr_pipe : s.lr_np;
      if (s.lr_policy == 1) {   // Caffe "inv": base (1 + gamma i)^(-power)
        lr_sh = (float)((double)base * pow(1.0 + (double)s.inv_gamma * (double)vc, -(double)s.inv_power));
      } else {
        const int64_t epoch = vc / s.spe;
        float f = 1.f;
        for (int m = 0; m < s.n_ms; ++m)
          if (epoch >= s.milestones[m]) f *= s.gamma;
        lr_sh = base * f;
      }
    }
  }
  __syncthreads();
  const SgdSeg& g = s.segs[seg_sh];
  const int64_t e = (int64_t)(blockIdx.x - s.seg_block_start[seg_sh]) * blockDim.x + threadIdx.x;
  if (e < g.n) {
    float w = s.w[g.off + e];
    int tap = 0, ci = 0, co = 0;
    if (g.kind == SEG_CONVW) {  // canonical OIHW [co][ci][r][s]
      const int kk = g.k * g.k;
      co = (int)(e / ((int64_t)g.cin * kk));
      ci = (int)((e / kk) % g.cin);
      tap = (int)(e % kk);
    }
    if (kUpdate) {
      float grad = 0.f;
      if (g.kind == SEG_VEC) {
        grad = (float)g.src_d[2 * e + g.comp];
      } else {
        const int64_t row = (int64_t)tap * g.Cinp + ci;
        grad = g.gsum[row * g.Coutp + co];
      }
      float v = s.v[g.off + e];
      const float d = grad + s.wd * w;
      if (s.solver == 0) {                 // PyTorch form (AMB-7)
        v = s.momentum * v + d;
        w = s.nesterov ? w - lr_sh * (d + s.momentum * v) : w - lr_sh * v;
      } else {                             // Caffe form
        const float vo = v;
        v = s.momentum * v + lr_sh * d;
        w = s.nesterov ? w - ((1.f + s.momentum) * v - s.momentum * vo) : w - v;
      }
      s.v[g.off + e] = v;
      s.w[g.off + e] = w;
    }
    if (g.kind == SEG_CONVW) {
      const act_t h = f2act(w);
      const int64_t i_f = shf_idx(tap, co, ci, g.Coutp, g.Cinp);
      const int64_t i_b = shb_idx(tap, co, ci, g.Coutp, g.Cinp);
      g.sh_fwd[i_f] = h;
      g.sh_bwd[i_b] = h;
#if PST_SPLIT
      const int64_t nsh = (int64_t)g.k * g.k * g.Coutp * g.Cinp;   // lo plane follows the raw plane
      g.sh_fwd[nsh + i_f] = tf32_lo(w);
      g.sh_bwd[nsh + i_b] = tf32_lo(w);
#endif
    }
  }
  if (kUpdate) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const int t = atomicAdd(s.ticket, 1);
      last_sh = (t == (int)s.total_blocks - 1);
    }
    __syncthreads();
    if (last_sh && threadIdx.x == 0) {
      *s.v_count += 1;
      *s.ticket = 0;
      __threadfence();
    }
  }
}

// Split-K reduction of every conv segment's wgrad partials: gsum[i] = sum_ks part[ks][i], one
// float4 per thread, coalesced in the partials' own [rows][Coutp] order.
__global__ void wgrad_sum_kernel(const SgdSpec s) {
  pdl_wait();
  pdl_trigger();
  __shared__ int seg_sh;
  if (threadIdx.x == 0) {
    int lo = 0, hi = s.n_segs - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s.red_block_start[mid] <= blockIdx.x) lo = mid; else hi = mid - 1;
    }
    seg_sh = lo;
  }
  __syncthreads();
  const SgdSeg& g = s.segs[seg_sh];
  const int64_t nv = (int64_t)g.k * g.k * g.Cinp * g.Coutp / 4;
  const int64_t i = (int64_t)(blockIdx.x - s.red_block_start[seg_sh]) * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const float4* p = reinterpret_cast<const float4*>(g.part) + i;
  float4 a = __ldg(p);
  for (int ks = 1; ks < g.ksplit; ++ks) {
    const float4 b = __ldg(p + (int64_t)ks * nv);
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
  }
  reinterpret_cast<float4*>(g.gsum)[i] = a;
}

__global__ void conv_w_shadow_kernel(const float* w, int cout, int cin, int k, int Coutp, int Cinp, act_t* sf,
                                     act_t* sb) {
  pdl_wait();      // writes weight shadows: no early pdl_trigger (sgd_kernel)

  const int64_t n = (int64_t)cout * cin * k * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int kk = k * k;
    const int co = (int)(e / ((int64_t)cin * kk));
    const int ci = (int)((e / kk) % cin);
    const int tap = (int)(e % kk);
    const act_t h = f2act(w[e]);
    const int64_t i_f = shf_idx(tap, co, ci, Coutp, Cinp);
    const int64_t i_b = shb_idx(tap, co, ci, Coutp, Cinp);
    sf[i_f] = h;
    sb[i_b] = h;
#if PST_SPLIT
    const int64_t nsh = (int64_t)kk * Coutp * Cinp;
    sf[nsh + i_f] = tf32_lo(w[e]);
    sb[nsh + i_b] = tf32_lo(w[e]);
#endif
  }
}

__global__ void wgrad_reduce_kernel(const float* part, int ksplit, int Coutp, int Cinp, int cout, int cin, int k,
                                    float* out) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = (int64_t)cout * cin * k * k;
  const int64_t rows = (int64_t)k * k * Cinp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int kk = k * k;
    const int co = (int)(e / ((int64_t)cin * kk));
    const int ci = (int)((e / kk) % cin);
    const int tap = (int)(e % kk);
    float g = 0.f;
    for (int ks = 0; ks < ksplit; ++ks) g += part[((int64_t)ks * rows + (int64_t)tap * Cinp + ci) * Coutp + co];
    out[e] = g;
  }
}

}  // namespace

// ------------------------------------------------------------------ launchers
// pixel-chunk grid for the plane-blocked kernels: about 4 resident blocks per SM in total
// ------------------------------------------------------------------ dropout (SURVEY f-3)
// Counter-based inverted dropout, the definition DESIGN.md gives (reading AMB-16b):
//   key = fmix32(seed ^ fmix32(mb * 0x9E3779B9 + (layer + 1) * 0x632BE5AB))
//   keep element e (logical NCHW index) iff fmix32(e ^ key) >= thresh; kept values *= scale.
// Applied in place to the post-ReLU tensor z; mb is the stage's forward counter (device memory, so
// the captured step graphs stay valid).  The backward needs no generator: z > 0 <=> kept and
// ReLU-active, and bwd_pre / the fused dgrad epilogue multiply the gradient by `scale` there.
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
  return h;
}

__global__ void dropout_fwd_kernel(act_t* __restrict__ z, int N, int HW, int Cp, int C, uint32_t seed, int layer,
                                   uint32_t thresh, float scale, const int64_t* __restrict__ fmb) {
  pdl_wait();
  pdl_trigger();
  const uint32_t mb = (uint32_t)(*fmb);
  const uint32_t key = fmix32(seed ^ fmix32(mb * 0x9E3779B9u + (uint32_t)(layer + 1) * 0x632BE5ABu));
  const int64_t npix = (int64_t)N * HW;
  const int64_t nvec = npix * (Cp / E);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
    const int plane = (int)(v / npix);
    const int64_t p = v - (int64_t)plane * npix;
    const int n = (int)(p / HW), hw = (int)(p - (int64_t)n * HW);
    float f[E];
    ldv(z + v * E, f);
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int c = plane * E + i;
      const uint32_t e = (uint32_t)(((int64_t)n * C + c) * HW + hw);
      f[i] = (c < C && fmix32(e ^ key) >= thresh) ? f[i] * scale : 0.f;
    }
    stv(z + v * E, f);
  }
}

__global__ void counter_inc_kernel(int64_t* c) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && blockIdx.x == 0) *c += 1;
}

static dim3 plane_grid(int npix, int planes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int want = std::max(1, num_sms(dev) * 4 / planes);
  const int chunks = (npix + kU * kBlock - 1) / (kU * kBlock);
  return dim3((unsigned)std::max(1, std::min(chunks, want)), (unsigned)planes);
}

void input_to_act(const float* x, act_t* out, int N, int C, int H, int W, int Cp, cudaStream_t st) {
  const int64_t nvec = (int64_t)N * H * W * (Cp / E);
  prof::begin(st);
  PST_CUDA(launch_k(nchw_to_act_kernel, dim3(grid_for(nvec)), dim3(kBlock), 0, st, x, out, N, C, H, W, Cp));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::MISC, (double)N * H * W * (C * 4.0 + Cp * sizeof(act_t)), 0);
}

void act_to_nchw(const void* in, int in_f32, float* out, int N, int C, int H, int W, cudaStream_t st) {
  PST_CUDA(launch_k(act_to_nchw_kernel, dim3(grid_for((int64_t)N * C * H * W)), dim3(kBlock), 0, st, in, in_f32, out, N, C, H, W));
  PST_CUDA(cudaGetLastError());
}

void bn_apply(const BnApplySpec& s, cudaStream_t st) {
  const int64_t nvec = (int64_t)s.N * s.H * s.W * (s.Cp / E);
  prof::begin(st);
  PST_CUDA(launch_k(bn_apply_kernel, plane_grid(s.N * s.H * s.W, s.Cp / E), dim3(kBlock), 0, st, s));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::BN_APPLY, (double)nvec * 16 * (s.res_mode ? 3 : 2), 0);
}

void maxpool2_fwd(const act_t* in, act_t* out, uint8_t* arg, int N, int H, int W, int Cp, cudaStream_t st) {
  PST_CHECK_ARG(H % 2 == 0 && W % 2 == 0, "maxpool2 needs even H, W");
  const int64_t nvec = (int64_t)N * (H / 2) * (W / 2) * (Cp / E);
  prof::begin(st);
  PST_CUDA(launch_k(maxpool2_kernel, dim3(grid_for(nvec)), dim3(kBlock), 0, st, in, out, arg, N, H, W, Cp));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::POOL, (double)nvec * (16 * 5 + E), 0);
}

void gap_fwd(const act_t* in, act_t* out, int N, int H, int W, int Cp, cudaStream_t st) {
  const int64_t nvec = (int64_t)N * (Cp / E);
  prof::begin(st);
  PST_CUDA(launch_k(gap_kernel, dim3(grid_for(nvec)), dim3(kBlock), 0, st, in, out, N, H, W, Cp));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::POOL, (double)nvec * 16 * (H * W + 1), 0);
}

void dropout_fwd(act_t* z, int N, int H, int W, int Cp, int C, uint32_t seed, int layer, uint32_t thresh, float scale,
                 const int64_t* fmb, cudaStream_t st) {
  const int64_t nvec = (int64_t)N * H * W * (Cp / E);
  prof::begin(st);
  PST_CUDA(launch_k(dropout_fwd_kernel, dim3(grid_for(nvec)), dim3(kBlock), 0, st, z, N, H * W, Cp, C, seed, layer,
                    thresh, scale, fmb));
  prof::end(st, prof::MISC, 2.0 * nvec * 16, 0.0);
}

void counter_inc(int64_t* c, cudaStream_t st) {
  prof::begin(st);
  PST_CUDA(launch_k(counter_inc_kernel, dim3(1), dim3(32), 0, st, c));
  prof::end(st, prof::MISC, 16.0, 0.0);
}

void bwd_pre(const BwdPreSpec& s, cudaStream_t st) {
  const int64_t npix = (int64_t)s.N * s.H * s.W;
  const int planes = s.Cp / E;
  int dev = 0;
  cudaGetDevice(&dev);
  (void)dev;
  prof::begin(st);
  PST_CUDA(launch_k(bwd_pre_kernel, plane_grid((int)npix, planes), dim3(kBlock), 0, st, s));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::BWD_PRE, (double)npix * planes * 16 * (2 + (s.relu ? 1 : 0) + (s.bn ? 1 : 0)), 0);
}

void bn_bwd_apply(const BnBwdSpec& s, cudaStream_t st) {
  const int64_t nvec = (int64_t)s.N * s.H * s.W * (s.Cp / E);
  prof::begin(st);
  PST_CUDA(launch_k(bn_bwd_apply_kernel, plane_grid(s.N * s.H * s.W, s.Cp / E), dim3(kBlock), 0, st, s));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::BN_BWD, (double)nvec * 16 * 3, 0);
}

void dilate2(const act_t* dy, act_t* dyd, int N, int Ho, int Wo, int H, int W, int Cp, cudaStream_t st) {
  const int64_t nvec = (int64_t)N * H * W * (Cp / E);
  prof::begin(st);
  PST_CUDA(launch_k(dilate2_kernel, dim3(grid_for(nvec)), dim3(kBlock), 0, st, dy, dyd, N, Ho, Wo, H, W, Cp));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::MISC, (double)nvec * 16 * 1.25, 0);
}

void softmax_ce(const float* logits, const int32_t* label_ring, int ring, float* loss_ring, int64_t* fwd_counter,
                float* dz, int B, int C, int Cp, cudaStream_t st) {
  prof::begin(st);
  PST_CUDA(launch_k(softmax_ce_kernel, dim3(1), dim3(512), 0, st, logits, label_ring, ring, loss_ring, fwd_counter, dz, B, C, Cp));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::LOSS, (double)B * Cp * 8.0, 0);
}

void sgd_update(const SgdSpec& s, cudaStream_t st) {
  prof::begin(st);
  PST_CUDA(launch_k(wgrad_sum_kernel, dim3((unsigned)s.red_total_blocks), dim3(kBlock), 0, st, s));
  PST_CUDA(cudaGetLastError());
  PST_CUDA(launch_k(sgd_kernel<true>, dim3((unsigned)s.total_blocks), dim3(kBlock), 0, st, s));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::SGD, (double)s.total_blocks * kBlock * 4.0 * 5, 0);
}

void build_shadows(const SgdSpec& s, cudaStream_t st) {
  PST_CUDA(launch_k(sgd_kernel<false>, dim3((unsigned)s.total_blocks), dim3(kBlock), 0, st, s));
  PST_CUDA(cudaGetLastError());
}

void conv_weights_to_shadows(const float* w, int cout, int cin, int k, int Coutp, int Cinp, act_t* sf, act_t* sb,
                             cudaStream_t st) {
  PST_CUDA(launch_k(conv_w_shadow_kernel, dim3(grid_for((int64_t)cout * cin * k * k)), dim3(kBlock), 0, st, w, cout, cin, k, Coutp, Cinp, sf, sb));
  PST_CUDA(cudaGetLastError());
}

void wgrad_reduce(const float* part, int ksplit, int Coutp, int Cinp, int cout, int cin, int k, float* out,
                  cudaStream_t st) {
  PST_CUDA(launch_k(wgrad_reduce_kernel, dim3(grid_for((int64_t)cout * cin * k * k)), dim3(kBlock), 0, st, part, ksplit, Coutp, Cinp, cout, cin,
                                                                               k, out));
  PST_CUDA(cudaGetLastError());
}

}  // namespace pst
