// elementwise.cu -- HBM-bound kernels of the hot path: layout conversion, BatchNorm
// (train-mode) forward apply and backward, ReLU/pool backward, max/avg pooling,
// gradient dilation, softmax cross-entropy, fused SGD-momentum update.
//
// All tensors are NHWC act_t with channels padded to Cp (multiple of 16); each
// thread moves 8 channels (16 bytes) per access.  Per-channel reductions use
// shared-memory partials and one float64 atomicAdd per channel per CTA.
#include "kernels.h"

#include <algorithm>

namespace pst {

namespace {

constexpr int kBlock = 256;

// 8 consecutive channels = 8*sizeof(act_t) bytes (16 or 32), vectorised
constexpr int kVec = (int)(8 * sizeof(act_t) / 16);   // uint4 per 8 elements

__device__ __forceinline__ void load8(const act_t* p, float* f) {
  alignas(16) act_t h[8];
#pragma unroll
  for (int i = 0; i < kVec; ++i) reinterpret_cast<uint4*>(h)[i] = reinterpret_cast<const uint4*>(p)[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = act2f(h[i]);
}
__device__ __forceinline__ void store8(act_t* p, const float* f) {
  alignas(16) act_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = f2act(f[i]);
#pragma unroll
  for (int i = 0; i < kVec; ++i) reinterpret_cast<uint4*>(p)[i] = reinterpret_cast<const uint4*>(h)[i];
}
__device__ __forceinline__ void copy8(act_t* d, const act_t* s) {
#pragma unroll
  for (int i = 0; i < kVec; ++i) reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
}
__device__ __forceinline__ void zero8(act_t* d) {
#pragma unroll
  for (int i = 0; i < kVec; ++i) reinterpret_cast<uint4*>(d)[i] = make_uint4(0, 0, 0, 0);
}

int grid_for(int64_t work, int per_block = kBlock) {
  int dev = 0;
  cudaGetDevice(&dev);
  const int sms = num_sms(dev);
  int64_t g = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * 8));
}

// ------------------------------------------------------------------ input conversion
__global__ void input_to_nhwc_kernel(const float* __restrict__ x, act_t* __restrict__ out, int N,
                                     int C, int H, int W, int Cp) {
  const int64_t npx = (int64_t)N * H * W;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npx;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(p / (H * W));
    const int hw = (int)(p % (H * W));
    for (int c0 = 0; c0 < Cp; c0 += 8) {
      float f[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = c0 + i;
        f[i] = c < C ? __ldg(&x[((int64_t)n * C + c) * H * W + hw]) : 0.f;
      }
      store8(out + p * Cp + c0, f);
    }
  }
}

// ------------------------------------------------------------------ BN forward apply
__global__ void bn_apply_kernel(const BnApplySpec s) {
  extern __shared__ float sh[];  // scale[Cp], shift[Cp]
  float* scale = sh;
  float* shift = sh + s.Cp;
  const double M = (double)s.N * s.H * s.W;
  for (int c = threadIdx.x; c < s.Cp; c += blockDim.x) {
    if (c < s.C) {
      const double mean = s.stats[2 * c] / M;
      double var = s.stats[2 * c + 1] / M - mean * mean;
      var = var < 0.0 ? 0.0 : var;
      const float invstd = (float)(1.0 / sqrt(var + (double)s.eps));
      const float g = s.gamma[c], b = s.beta[c];
      scale[c] = g * invstd;
      shift[c] = b - (float)mean * g * invstd;
      if (blockIdx.x == 0) {
        s.saved[2 * c] = (float)mean;
        s.saved[2 * c + 1] = invstd;
        s.run_mean[c] = (1.f - s.momentum) * s.run_mean[c] + s.momentum * (float)mean;
        s.run_var[c] = (1.f - s.momentum) * s.run_var[c] + s.momentum * (float)(var * M / (M - 1.0));
      }
    } else {
      scale[c] = 0.f;
      shift[c] = 0.f;
    }
  }
  __syncthreads();
  const int cv = s.Cp / 8;
  const int64_t nvec = (int64_t)s.N * s.H * s.W * cv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / cv;
    const int c0 = (int)(i % cv) * 8;
    float f[8];
    load8(s.y + p * s.Cp + c0, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * scale[c0 + j] + shift[c0 + j];
    if (s.res_mode == 1) {
      float r[8];
      load8(s.res + p * s.Cp + c0, r);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += (c0 + j < s.C) ? r[j] : 0.f;
    } else if (s.res_mode == 2) {
      const int n = (int)(p / ((int64_t)s.H * s.W));
      const int hw = (int)(p % ((int64_t)s.H * s.W));
      const int y = hw / s.W, x = hw % s.W;
      const act_t* rp = s.res + (((int64_t)n * s.res_H + 2 * y) * s.res_W + 2 * x) * s.res_C;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int cr = c0 + j - s.res_pad;
        if (cr >= 0 && cr < s.res_Creal) f[j] += act2f(rp[cr]);
      }
    }
    if (s.relu) {
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = fmaxf(f[j], 0.f);
    }
    store8(s.z + p * s.Cp + c0, f);
  }
}

// ------------------------------------------------------------------ pooling
__global__ void maxpool2_kernel(const act_t* __restrict__ in, act_t* __restrict__ out,
                                uint8_t* __restrict__ arg, int N, int H, int W, int Cp) {
  const int Ho = H / 2, Wo = W / 2, cv = Cp / 8;
  const int64_t nvec = (int64_t)N * Ho * Wo * cv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t po = i / cv;
    const int c0 = (int)(i % cv) * 8;
    const int n = (int)(po / ((int64_t)Ho * Wo));
    const int hw = (int)(po % ((int64_t)Ho * Wo));
    const int yo = hw / Wo, xo = hw % Wo;
    float best[8];
    uint8_t a[8];
    for (int q = 0; q < 4; ++q) {
      const int y = 2 * yo + (q >> 1), x = 2 * xo + (q & 1);
      float f[8];
      load8(in + (((int64_t)n * H + y) * W + x) * Cp + c0, f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (q == 0 || f[j] > best[j]) {
          best[j] = f[j];
          a[j] = (uint8_t)q;
        }
      }
    }
    store8(out + po * Cp + c0, best);
    *reinterpret_cast<uint2*>(arg + po * Cp + c0) = *reinterpret_cast<const uint2*>(a);
  }
}

__global__ void gap_kernel(const act_t* __restrict__ in, act_t* __restrict__ out, int N, int H, int W,
                           int Cp) {
  const int64_t nout = (int64_t)N * Cp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nout;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i / Cp), c = (int)(i % Cp);
    float acc = 0.f;
    for (int p = 0; p < H * W; ++p) acc += act2f(in[((int64_t)n * H * W + p) * Cp + c]);
    out[i] = f2act(acc / (float)(H * W));
  }
}

// ------------------------------------------------------------------ backward pre (pool^T, relu^T, sums)
__global__ void bwd_pre_kernel(const BwdPreSpec s) {
  extern __shared__ float red[];  // [Cp][2]
  for (int i = threadIdx.x; i < 2 * s.Cp; i += blockDim.x) red[i] = 0.f;
  __syncthreads();
  const int cv = s.Cp / 8;
  const int64_t nvec = (int64_t)s.N * s.H * s.W * cv;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // multiple of cv (host guarantees)
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c0 = (int)(i0 % cv) * 8;
  float mean[8], inv[8];
  if (s.bn) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      mean[j] = s.saved[2 * (c0 + j)];
      inv[j] = s.saved[2 * (c0 + j) + 1];
    }
  }
  float a1[8], a2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a1[j] = a2[j] = 0.f;
  const int HW = s.H * s.W;
  for (int64_t i = i0; i < nvec; i += stride) {
    const int64_t p = i / cv;
    float g[8];
    if (s.pool == 0) {
      if (s.gout_f32) {
        const float* gp = reinterpret_cast<const float*>(s.gout) + p * s.Cp + c0;
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = gp[j];
      } else {
        load8(s.gout + p * s.Cp + c0, g);
      }
    } else if (s.pool == 1) {
      const int n = (int)(p / HW), hw = (int)(p % HW);
      const int y = hw / s.W, x = hw % s.W;
      const int64_t po = ((int64_t)n * (s.H / 2) + y / 2) * (s.W / 2) + x / 2;
      float gg[8];
      load8(s.gout + po * s.Cp + c0, gg);
      const uint2 au = *reinterpret_cast<const uint2*>(s.arg + po * s.Cp + c0);
      const uint8_t* a = reinterpret_cast<const uint8_t*>(&au);
      const uint8_t q = (uint8_t)(((y & 1) << 1) | (x & 1));
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = (a[j] == q) ? gg[j] : 0.f;
    } else {
      const int n = (int)(p / HW);
      float gg[8];
      load8(s.gout + (int64_t)n * s.Cp + c0, gg);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = gg[j] / (float)HW;
    }
    if (s.relu) {
      float z[8];
      load8(s.z + p * s.Cp + c0, z);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = z[j] > 0.f ? g[j] : 0.f;
    }
    // round to the stored precision; sums use exactly what later kernels read
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] = act2f(f2act(g[j]));
    store8(s.gpre + p * s.Cp + c0, g);
    if (s.bn) {
      float y[8];
      load8(s.y + p * s.Cp + c0, y);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a1[j] += g[j];
        a2[j] += g[j] * (y[j] - mean[j]) * inv[j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) a1[j] += g[j];
    }
  }
  // lanes sharing a channel group (lane = c mod cv) pre-reduce with shuffles
  if (cv < 32 && (32 % cv) == 0) {
    for (int o = 16; o >= cv; o >>= 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a1[j] += __shfl_xor_sync(0xffffffffu, a1[j], o);
        a2[j] += __shfl_xor_sync(0xffffffffu, a2[j], o);
      }
    }
  }
  if (cv >= 32 || (32 % cv) != 0 || (threadIdx.x & 31) < cv) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      atomicAdd(&red[2 * (c0 + j)], a1[j]);
      atomicAdd(&red[2 * (c0 + j) + 1], a2[j]);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * s.C; i += blockDim.x) {
    const int c = i >> 1;
    if (c < s.C) atomicAdd(&s.sums[i], (double)red[i]);
  }
}

__global__ void bn_bwd_apply_kernel(const BnBwdSpec s) {
  extern __shared__ float sh[];  // k1, m1, m2, mean, inv  [5][Cp]
  float* k1 = sh;
  float* m1 = sh + s.Cp;
  float* m2 = sh + 2 * s.Cp;
  float* mu = sh + 3 * s.Cp;
  float* iv = sh + 4 * s.Cp;
  const double M = (double)s.N * s.H * s.W;
  for (int c = threadIdx.x; c < s.Cp; c += blockDim.x) {
    if (c < s.C) {
      mu[c] = s.saved[2 * c];
      iv[c] = s.saved[2 * c + 1];
      k1[c] = s.gamma[c] * iv[c];
      m1[c] = (float)(s.sums[2 * c] / M);
      m2[c] = (float)(s.sums[2 * c + 1] / M);
    } else {
      mu[c] = iv[c] = k1[c] = m1[c] = m2[c] = 0.f;
    }
  }
  __syncthreads();
  const int cv = s.Cp / 8;
  const int64_t nvec = (int64_t)s.N * s.H * s.W * cv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / cv;
    const int c0 = (int)(i % cv) * 8;
    float g[8], y[8], o[8];
    load8(s.gpre + p * s.Cp + c0, g);
    load8(s.y + p * s.Cp + c0, y);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      const float xh = (y[j] - mu[c]) * iv[c];
      o[j] = k1[c] * (g[j] - m1[c] - xh * m2[c]);
    }
    store8(s.gy + p * s.Cp + c0, o);
  }
}

__global__ void dilate2_kernel(const act_t* __restrict__ dy, act_t* __restrict__ out, int N, int Ho,
                               int Wo, int H, int W, int Cp) {
  const int cv = Cp / 8;
  const int64_t nvec = (int64_t)N * H * W * cv;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / cv;
    const int c0 = (int)(i % cv) * 8;
    const int n = (int)(p / ((int64_t)H * W));
    const int hw = (int)(p % ((int64_t)H * W));
    const int y = hw / W, x = hw % W;
    if (((y | x) & 1) == 0 && (y >> 1) < Ho && (x >> 1) < Wo)
      copy8(out + p * Cp + c0, dy + (((int64_t)n * Ho + (y >> 1)) * Wo + (x >> 1)) * Cp + c0);
    else
      zero8(out + p * Cp + c0);
  }
}

// ------------------------------------------------------------------ softmax cross-entropy
__global__ void softmax_ce_kernel(const float* __restrict__ logits, const int32_t* __restrict__ label_ring,
                                  int ring, float* __restrict__ loss_ring, int64_t* fwd_counter,
                                  float* __restrict__ dz, int B, int C, int Cp) {
  __shared__ float wsum[32];
  const int64_t f = *fwd_counter;
  const int32_t* labels = label_ring + (f % ring) * B;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float lsum = 0.f;
  for (int b = warp; b < B; b += nw) {
    const float* z = logits + (int64_t)b * Cp;
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = fmaxf(m, z[c]);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float se = 0.f;
    for (int c = lane; c < C; c += 32) se += expf(z[c] - m);
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int yb = labels[b];
    const float lse = m + logf(se);
    if (lane == 0) lsum += lse - z[yb];
    for (int c = lane; c < Cp; c += 32) {
      float v = 0.f;
      if (c < C) v = (expf(z[c] - m) / se - (c == yb ? 1.f : 0.f)) / (float)B;
      dz[(int64_t)b * Cp + c] = v;
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
template <bool kUpdate>
__global__ void sgd_kernel(const SgdSpec s) {
  __shared__ float lr_sh;
  __shared__ int seg_sh;
  __shared__ int last_sh;
  if (threadIdx.x == 0) {
    // segment of this block (binary search over the prefix)
    int lo = 0, hi = s.n_segs - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s.seg_block_start[mid] <= blockIdx.x) lo = mid; else hi = mid - 1;
    }
    seg_sh = lo;
    if (kUpdate) {
      const int64_t vc = *s.v_count;
      const float base = (vc < *s.n_p) ? *s.lr_pipe : s.lr_np;
      const int64_t epoch = vc / s.spe;
      float f = 1.f;
      for (int m = 0; m < s.n_ms; ++m)
        if (epoch >= s.milestones[m]) f *= s.gamma;
      lr_sh = base * f;
    }
  }
  __syncthreads();
  const SgdSeg& g = s.segs[seg_sh];
  const int64_t e = (int64_t)(blockIdx.x - s.seg_block_start[seg_sh]) * blockDim.x + threadIdx.x;
  if (e < g.n) {
    float w = s.w[g.off + e];
    float grad = 0.f;
    int tap = 0, ci = 0, co = 0;
    int64_t row = 0;
    if (g.kind == SEG_CONVW) {
      const int kk = g.k * g.k;
      co = (int)(e / ((int64_t)g.cin * kk));
      ci = (int)((e / kk) % g.cin);
      tap = (int)(e % kk);
      row = (int64_t)tap * g.Cinp + ci;
    } else if (g.kind == SEG_FCW) {
      co = (int)(e / g.cin);
      const int i = (int)(e % g.cin);  // NCHW flatten index of the input tensor
      const int c = i / (g.fc_H * g.fc_W);
      const int yx = i % (g.fc_H * g.fc_W);
      ci = yx * g.fc_Cp + c;           // NHWC GEMM row
      row = ci;
    }
    if (kUpdate) {
      if (g.kind == SEG_VEC) {
        grad = (float)g.src_d[2 * e + g.comp];
      } else {
        const int64_t rows = (int64_t)g.k * g.k * g.Cinp;
        for (int ks = 0; ks < g.ksplit; ++ks) grad += g.part[((int64_t)ks * rows + row) * g.Coutp + co];
      }
      float v = s.v[g.off + e];
      v = s.momentum * v + (grad + s.wd * w);
      w = w - lr_sh * v;
      s.v[g.off + e] = v;
      s.w[g.off + e] = w;
    }
    if (g.kind != SEG_VEC) {
      const act_t h = f2act(w);
      const int64_t i_f = ((int64_t)tap * g.Coutp + co) * g.Cinp + ci;
      const int64_t i_b = ((int64_t)tap * g.Cinp + ci) * g.Coutp + co;
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

}  // namespace

void input_to_nhwc(const float* x, act_t* out, int N, int C, int H, int W, int Cp, cudaStream_t st) {
  prof::begin(st);
  input_to_nhwc_kernel<<<grid_for((int64_t)N * H * W), kBlock, 0, st>>>(x, out, N, C, H, W, Cp);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::MISC, (double)N * H * W * (C * 4.0 + Cp * sizeof(act_t)), 0);
}

void bn_apply(const BnApplySpec& s, cudaStream_t st) {
  const int64_t nvec = (int64_t)s.N * s.H * s.W * (s.Cp / 8);
  prof::begin(st);
  bn_apply_kernel<<<grid_for(nvec), kBlock, 2 * s.Cp * sizeof(float), st>>>(s);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::BN_APPLY, (double)nvec * 8 * sizeof(act_t) * (s.res_mode ? 3 : 2), 0);
}

void maxpool2_fwd(const act_t* in, act_t* out, uint8_t* arg, int N, int H, int W, int Cp, cudaStream_t st) {
  PST_CHECK_ARG(H % 2 == 0 && W % 2 == 0, "maxpool2 needs even H, W");
  const int64_t nvec = (int64_t)N * (H / 2) * (W / 2) * (Cp / 8);
  prof::begin(st);
  maxpool2_kernel<<<grid_for(nvec), kBlock, 0, st>>>(in, out, arg, N, H, W, Cp);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::POOL, (double)nvec * 8 * (5 * sizeof(act_t) + 1), 0);
}

void gap_fwd(const act_t* in, act_t* out, int N, int H, int W, int Cp, cudaStream_t st) {
  prof::begin(st);
  gap_kernel<<<grid_for((int64_t)N * Cp), kBlock, 0, st>>>(in, out, N, H, W, Cp);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::POOL, (double)N * Cp * (H * W + 1) * sizeof(act_t), 0);
}

void bwd_pre(const BwdPreSpec& s, cudaStream_t st) {
  const int cv = s.Cp / 8;
  // block size a multiple of cv so every thread keeps one channel group across the grid stride
  int block = cv <= kBlock ? (kBlock / cv) * cv : 0;
  PST_CHECK_ARG(block > 0 || cv % kBlock == 0, "bwd_pre: unsupported channel count");
  if (block == 0) block = kBlock;
  const int64_t nvec = (int64_t)s.N * s.H * s.W * cv;
  const int g = grid_for(nvec, block);
  prof::begin(st);
  bwd_pre_kernel<<<g, block, 2 * s.Cp * sizeof(float), st>>>(s);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::BWD_PRE, (double)nvec * 8 * sizeof(act_t) * (2 + (s.relu ? 1 : 0) + (s.bn ? 1 : 0)), 0);
}

void bn_bwd_apply(const BnBwdSpec& s, cudaStream_t st) {
  const int64_t nvec = (int64_t)s.N * s.H * s.W * (s.Cp / 8);
  prof::begin(st);
  bn_bwd_apply_kernel<<<grid_for(nvec), kBlock, 5 * s.Cp * sizeof(float), st>>>(s);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::BN_BWD, (double)nvec * 8 * sizeof(act_t) * 3, 0);
}

void dilate2(const act_t* dy, act_t* dyd, int N, int Ho, int Wo, int H, int W, int Cp, cudaStream_t st) {
  const int64_t nvec = (int64_t)N * H * W * (Cp / 8);
  prof::begin(st);
  dilate2_kernel<<<grid_for(nvec), kBlock, 0, st>>>(dy, dyd, N, Ho, Wo, H, W, Cp);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::MISC, (double)nvec * 8 * sizeof(act_t) * 1.25, 0);
}

void softmax_ce(const float* logits, const int32_t* label_ring, int ring, float* loss_ring,
                int64_t* fwd_counter, float* dz, int B, int C, int Cp, cudaStream_t st) {
  prof::begin(st);
  softmax_ce_kernel<<<1, 512, 0, st>>>(logits, label_ring, ring, loss_ring, fwd_counter, dz, B, C, Cp);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::LOSS, (double)B * Cp * 8.0, 0);
}

void sgd_update(const SgdSpec& s, cudaStream_t st) {
  prof::begin(st);
  sgd_kernel<true><<<(unsigned)s.total_blocks, kBlock, 0, st>>>(s);
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::SGD, (double)s.total_blocks * kBlock * 4.0 * 5, 0);
}

void build_shadows(const SgdSpec& s, cudaStream_t st) {
  sgd_kernel<false><<<(unsigned)s.total_blocks, kBlock, 0, st>>>(s);
  PST_CUDA(cudaGetLastError());
}

}  // namespace pst

namespace pst {
namespace {
__global__ void nhwc_to_nchw_kernel(const void* in, int in_f32, float* out, int N, int C, int H, int W, int Cp) {
  const int64_t n_el = (int64_t)N * C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_el; i += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % W);
    const int y = (int)((i / W) % H);
    const int c = (int)((i / ((int64_t)W * H)) % C);
    const int n = (int)(i / ((int64_t)W * H * C));
    const int64_t src = (((int64_t)n * H + y) * W + x) * Cp + c;
    out[i] = in_f32 ? reinterpret_cast<const float*>(in)[src] : act2f(reinterpret_cast<const act_t*>(in)[src]);
  }
}
__global__ void conv_w_shadow_kernel(const float* w, int cout, int cin, int k, int Coutp, int Cinp, act_t* sf,
                                     act_t* sb) {
  const int64_t n = (int64_t)cout * cin * k * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int kk = k * k;
    const int co = (int)(e / ((int64_t)cin * kk));
    const int ci = (int)((e / kk) % cin);
    const int tap = (int)(e % kk);
    const act_t h = f2act(w[e]);
    const int64_t i_f = ((int64_t)tap * Coutp + co) * Cinp + ci;
    const int64_t i_b = ((int64_t)tap * Cinp + ci) * Coutp + co;
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

void nhwc_to_nchw(const void* in, int in_f32, float* out, int N, int C, int H, int W, int Cp, cudaStream_t st) {
  nhwc_to_nchw_kernel<<<grid_for((int64_t)N * C * H * W), kBlock, 0, st>>>(in, in_f32, out, N, C, H, W, Cp);
  PST_CUDA(cudaGetLastError());
}
void conv_weights_to_shadows(const float* w, int cout, int cin, int k, int Coutp, int Cinp, act_t* sf, act_t* sb,
                             cudaStream_t st) {
  conv_w_shadow_kernel<<<grid_for((int64_t)cout * cin * k * k), kBlock, 0, st>>>(w, cout, cin, k, Coutp, Cinp, sf, sb);
  PST_CUDA(cudaGetLastError());
}
void wgrad_reduce(const float* part, int ksplit, int Coutp, int Cinp, int cout, int cin, int k, float* out,
                  cudaStream_t st) {
  wgrad_reduce_kernel<<<grid_for((int64_t)cout * cin * k * k), kBlock, 0, st>>>(part, ksplit, Coutp, Cinp, cout,
                                                                               cin, k, out);
  PST_CUDA(cudaGetLastError());
}
}  // namespace pst
