// conv_tc.cu -- implicit-GEMM convolution on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Forward (x^(l) from x^(l-1) and W^(l)) and dgrad (L47: delta^(l-1)
// from delta^(l) with the CURRENT weights, reading AMB-2) are one kernel:
//   D[p, co] = sum_tap sum_ci  X[n, y*S + off + sgn*r, x*S + off + sgn*s, ci] * Wt[tap][co][ci]
// M = 128 output pixels (an (img, y, x) box), N = output channels, K = taps x
// input channels.  Each K step loads, with one TMA per 16-byte channel chunk, the
// shifted 128-pixel box of the input (zero fill outside the image = the
// convolution's zero padding) and the tap's weight slice.
//
// Weight gradient (L47: de/dW^(l) from x^(l-1) and delta^(l)):
//   D[tap*Cinp + ci, co] = sum_p X_shift(tap)[p, ci] * dY[p, co]
// M = (tap, ci) rows from shifted input boxes (MN-major operand), N = co
// (MN-major), K = output pixels split over CTAs; partial sums are reduced by the
// SGD kernel.
//
// Precision (common.h): in the default build operands are float32 in smem and
// every product is 3xTF32 -- D += Ahi*Bhi + Ahi*Blo + Alo*Bhi, where the tensor
// core truncates float32 to tf32 (= hi) and lo = v - trunc(v) comes from a
// converter warpgroup (activations) or from a precomputed shadow (weights).
//
// Structure: persistent CTAs, warp-specialised: warp 0 TMA producer, warp 1 MMA
// issuer (+TMEM allocator), warps 2..5 epilogue, warps 6..9 split converter
// (3xTF32 build only).  smem ring of `stages` slots (full / ready / empty
// mbarriers), double-buffered TMEM accumulators (tmem_full / tmem_empty).
#include "kernels.h"
#include "ptx.cuh"

#include <algorithm>
#include <cstdlib>

namespace pst {

namespace {

constexpr int kBaseThreads = 192;
constexpr int kThreads = kBaseThreads + (PST_SPLIT ? 128 : 0);
constexpr int kEpiThreads = 128;
constexpr int kMaxStages = 8;
constexpr int kMmaK = 32 / (int)sizeof(act_t);   // K elements per MMA instruction (2 chunks)

struct FwdArgs {
  int N, Ho, Wo;
  int bimg, bh, bw, tn, ty, tx;
  int n_mtiles, n_ntiles, n_tiles;
  int Cinp, kc, n_kc, k, taps, S, off, sgn;
  int Coutp, BN, Cout;
  int stages;
  uint32_t a_bytes, b_bytes, stage_bytes, tx_bytes;
  uint32_t tmem_cols;
  int epi, relu;
  void* out;
  const float* bias;
  double* stats;
  const act_t* res;
  int res_mode, res_H, res_W, res_C, res_pad;
  int a4, b3;   // tensor-map forms (act_tmap / w_tmap)
  // HALO mode: virtual-grid pitch, lowest tap offset, tiles per image, band plane bytes,
  // resident weight bytes (0: per stage), stage B bytes, per-tap start offsets (positions)
  int Wv, lo, tpi, MT, Pimg;   // Pimg = Ho*Wv positions per image; MT M-tiles per super tile
  uint32_t plane_bytes, wres_bytes, sb_bytes;
  int tapoff[49];
  unsigned long long* dbg;   // optional timeline (CTA 0), see PST_DBG_TL
};

__device__ __forceinline__ void decode_tile_px(const FwdArgs& a, int mt, int row, int& n, int& y,
                                               int& x) {
  const int ix = mt % a.tx;
  const int iy = (mt / a.tx) % a.ty;
  const int it = mt / (a.tx * a.ty);
  const int xb = row % a.bw;
  const int yb = (row / a.bw) % a.bh;
  const int nb = row / (a.bw * a.bh);
  n = it * a.bimg + nb;
  y = iy * a.bh + yb;
  x = ix * a.bw + xb;
}

// 3xTF32 split: lo[i] = raw[i] - trunc_tf32(raw[i]) over `nbytes` of smem, by 128 threads.
__device__ __forceinline__ void split_lo(const uint8_t* raw, uint8_t* lo, uint32_t nbytes, int t) {
  const float4* r = reinterpret_cast<const float4*>(raw);
  float4* l = reinterpret_cast<float4*>(lo);
  for (uint32_t i = t; i < nbytes / 16; i += 128) {
    float4 v = r[i];
    l[i] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
  }
}

// 16 consecutive channels c0..c0+15 of one pixel into a channel-planar tensor:
// plane (c/EPC) at stride npix*16 bytes.
__device__ __forceinline__ void store16_planar(act_t* base, int64_t npix, int64_t pix, int c0, const float* v) {
  alignas(16) act_t h[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) h[i] = f2act(v[i]);
#pragma unroll
  for (int j = 0; j < 16 / kEPC; ++j)
    *reinterpret_cast<uint4*>(base + ((int64_t)(c0 / kEPC + j) * npix + pix) * kEPC) =
        reinterpret_cast<const uint4*>(h)[j];
}
__device__ __forceinline__ void store16_f32(float* base, int64_t npix, int64_t pix, int c0, const float* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<float4*>(base + ((int64_t)(c0 / 4 + j) * npix + pix) * 4) =
        make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
__device__ __forceinline__ float ld_planar(const act_t* base, int64_t npix, int64_t pix, int c) {
  return act2f(base[((int64_t)(c / kEPC) * npix + pix) * kEPC + c % kEPC]);
}

// load one activation box (act_tmap): x/y in pixels (may be negative: zero fill), image n0, plane cc
__device__ __forceinline__ void tma_act(void* dst, const CUtensorMap* tm, uint64_t* bar, bool is4d, int x, int y,
                                        int n0, int cc) {
  if (is4d) ptx::tma_load_4d(dst, tm, bar, x * kEPC, y, n0, cc);
  else ptx::tma_load_5d(dst, tm, bar, 0, x, y, n0, cc);
}
// load one weight box (w_tmap): rows co0.., planes cc.., tap
__device__ __forceinline__ void tma_w(void* dst, const CUtensorMap* tm, uint64_t* bar, bool is3d, int co0, int cc,
                                      int tap) {
  if (is3d) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(ptx::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(ptx::smem_u32(bar)), "r"(co0 * kEPC), "r"(cc), "r"(tap)
        : "memory");
  } else {
    ptx::tma_load_4d(dst, tm, bar, 0, co0, cc, tap);
  }
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// timeline probe (debug only): event ev, occurrence i, CTA 0
#define TL(ev, i)                                                                  \
  do {                                                                             \
    if (a.dbg != nullptr && blockIdx.x == 0) {                                     \
      const int i_ = (i);                                                          \
      if (i_ < 256) a.dbg[(ev) * 256 + i_] = gtime();                              \
    }                                                                              \
  } while (0)

// HALO (stride-1 layers, Wo >= 16): the M tile is 128 consecutive positions of a
// "virtual" output grid of row pitch Wv = Wo + k - 1 inside one image (positions with
// x >= Wo are computed and discarded).  One TMA box loads the input band those
// positions read for EVERY tap; tap (oy, ox) is then just the band shifted by
// (oy-lo)*Wv + (ox-lo) positions -- a descriptor start offset, no re-load.  Weights of
// all taps stay resident in smem when they fit.
// DG distinguishes the dgrad instantiation (same code, separate name in profiles).
template <bool HALO, bool DG>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fwd_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmBlo, const FwdArgs a) {
  int dbg_i[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (threadIdx.x == 0) TL(7, 0);
  extern __shared__ __align__(1024) uint8_t smem[];
  // [stages x stage_bytes] [resident weights (HALO && wres)] [sbuf 16x129 f32] [acc doubles 2*Coutp]
  // [barriers] [tmem ptr];  stage: [A raw][B raw]([A lo][B lo] in the split build)
  uint8_t* ring = smem;
  uint8_t* wres = smem + a.stages * a.stage_bytes;
  float* sbuf = reinterpret_cast<float*>(wres + a.wres_bytes);
  double* cacc = reinterpret_cast<double*>(sbuf + 16 * 129 + 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(cacc + 2 * a.Coutp);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* ready = bars + 2 * kMaxStages;
  uint64_t* tfull = bars + 3 * kMaxStages;
  uint64_t* tempty = bars + 3 * kMaxStages + 2;
  uint64_t* wbar = bars + 3 * kMaxStages + 4;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 3 * kMaxStages + 5);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
      ptx::mbar_init(&ready[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 4);
    }
    ptx::mbar_init(wbar, 1);
    ptx::fence_mbar_init();
  }
  if (a.epi == EPI_BN_STATS)
    for (int i = threadIdx.x; i < 2 * a.Coutp; i += blockDim.x) cacc[i] = 0.0;
  if (warp == 1) ptx::tmem_alloc(tmem_ptr, a.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  pdl_wait();      // no global memory access above this line
  pdl_trigger();
  const int nch = a.kc / kEPC;   // 16-byte channel chunks per stage

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmB);
      if (PST_SPLIT) ptx::prefetch_tmap(&tmBlo);
      int st = 0;
      uint32_t ph = 0;
      if (HALO && a.wres_bytes) {   // resident weights: every chunk, every tap (+lo), once per CTA
        ptx::mbar_expect_tx(wbar, a.wres_bytes);
        for (int kcc = 0; kcc < a.n_kc; ++kcc) {
          tma_w(wres + kcc * a.b_bytes, &tmB, wbar, a.b3, 0, kcc * nch, 0);
#if PST_SPLIT
          tma_w(wres + (a.n_kc + kcc) * a.b_bytes, &tmBlo, wbar, a.b3, 0, kcc * nch, 0);
#endif
        }
      }
      for (int t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
        const int mt = t / a.n_ntiles, nt = t % a.n_ntiles;
        if (HALO) {
          const int n = mt / a.tpi, g0 = (mt % a.tpi) * 128 * a.MT;
          const int yf = g0 / a.Wv;
          for (int kcc = 0; kcc < a.n_kc; ++kcc) {
            ptx::mbar_wait(&empty[st], ph ^ 1);
            TL(0, dbg_i[0]++);
            ptx::mbar_expect_tx(&full[st], a.tx_bytes);
            uint8_t* sa = ring + st * a.stage_bytes;
            // one band box: rows [yf+lo, yf+lo+band_r) x columns [lo, lo+Wv), zero outside the image
            tma_act(sa, &tmA, &full[st], true, a.lo, yf + a.lo, n, kcc * nch);
            if (!a.wres_bytes) {
              uint8_t* sb = sa + a.a_bytes;
              tma_w(sb, &tmB, &full[st], a.b3, nt * a.BN, kcc * nch, 0);
#if PST_SPLIT
              tma_w(sb + a.a_bytes + a.sb_bytes, &tmBlo, &full[st], a.b3, nt * a.BN, kcc * nch, 0);
#endif
            }
            if (++st == a.stages) { st = 0; ph ^= 1; }
          }
          continue;
        }
        const int ix = mt % a.tx, iy = (mt / a.tx) % a.ty, it = mt / (a.tx * a.ty);
        const int x0 = ix * a.bw * a.S + a.off, y0 = iy * a.bh * a.S + a.off, n0 = it * a.bimg;
        for (int tap = 0; tap < a.taps; ++tap) {
          const int r = tap / a.k, s = tap % a.k;
          for (int kcc = 0; kcc < a.n_kc; ++kcc) {
            ptx::mbar_wait(&empty[st], ph ^ 1);
            TL(0, dbg_i[0]++);
            ptx::mbar_expect_tx(&full[st], a.tx_bytes);
            uint8_t* sa = ring + st * a.stage_bytes;
            uint8_t* sb = sa + a.a_bytes;
            const int cc = kcc * nch;
            // one box each: A = nch planes x 128 pixels (rows of contiguous pixels), B = nch x BN rows
            tma_act(sa, &tmA, &full[st], a.a4, x0 + a.sgn * s, y0 + a.sgn * r, n0, cc);
            tma_w(sb, &tmB, &full[st], a.b3, nt * a.BN, cc, tap);
#if PST_SPLIT
            tma_w(sb + a.a_bytes + a.sb_bytes, &tmBlo, &full[st], a.b3, nt * a.BN, cc, tap);
#endif
            if (++st == a.stages) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (warp-uniform, elected lane)
    const uint32_t idesc = ptx::idesc_mma(128, a.BN, 0, 0, PST_AB_FORMAT);
    int st = 0;
    uint32_t ph = 0;
    int local = 0;
    if (HALO && a.wres_bytes) ptx::mbar_wait(wbar, 0);
    for (int t = blockIdx.x; t < a.n_tiles; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t dtm = tmem_base + acc * a.BN * (HALO ? a.MT : 1);
      if (HALO) {
        const int mt = t / a.n_ntiles;
        const int g0 = (mt % a.tpi) * 128 * a.MT;
        const int mtv = min(a.MT, (a.Pimg - g0 + 127) / 128);         // M tiles with valid rows
        const uint32_t base_pos = (uint32_t)(g0 - (g0 / a.Wv) * a.Wv);   // g0 relative to its band row
        for (int kcc = 0; kcc < a.n_kc; ++kcc) {
          ptx::mbar_wait(PST_SPLIT ? &ready[st] : &full[st], ph);
          if (lane == 0) TL(3, dbg_i[3]++);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(ring + st * a.stage_bytes);
          const uint32_t off_lo = a.a_bytes + a.sb_bytes;
          const uint32_t wb = a.wres_bytes ? ptx::smem_u32(wres) + kcc * a.b_bytes : sa + a.a_bytes;
          const uint32_t wb_lo = a.wres_bytes ? wb + a.n_kc * a.b_bytes : wb + off_lo;
          const uint32_t tapb = (uint32_t)nch * a.BN * 16;   // bytes of one tap's weights in the box
          const uint64_t bd0 = ptx::smem_desc(wb, a.BN * 16, 128);
          const uint64_t bdl0 = ptx::smem_desc(wb_lo, a.BN * 16, 128);
          const uint64_t ad0 = ptx::smem_desc(sa + base_pos * 16, a.plane_bytes, 128);
          if (ptx::elect_one()) {
            // consecutive MMAs go to the mtv independent accumulators of the super tile
            for (int tap = 0; tap < a.taps; ++tap) {
              const uint64_t adt = ptx::desc_add(ad0, (uint32_t)a.tapoff[tap]);
              for (int kk = 0; kk < nch / 2; ++kk) {
                const uint64_t bd = ptx::desc_add(bd0, tap * tapb + kk * 2 * (a.BN * 16));
                const uint64_t adk = ptx::desc_add(adt, kk * 2 * a.plane_bytes);
                const uint32_t acc0 = (kcc > 0 || tap > 0 || kk > 0) ? 1u : 0u;
                for (int j = 0; j < mtv; ++j) ptx::umma(dtm + j * a.BN, ptx::desc_add(adk, j * 2048), bd, idesc, acc0);
#if PST_SPLIT
                const uint64_t bdl = ptx::desc_add(bdl0, tap * tapb + kk * 2 * (a.BN * 16));
                for (int j = 0; j < mtv; ++j) ptx::umma(dtm + j * a.BN, ptx::desc_add(adk, j * 2048), bdl, idesc, 1u);
                for (int j = 0; j < mtv; ++j)
                  ptx::umma(dtm + j * a.BN, ptx::desc_add(adk, off_lo + j * 2048), bd, idesc, 1u);
#endif
              }
            }
            ptx::umma_commit(&empty[st]);
          }
          __syncwarp();
          if (lane == 0) TL(4, dbg_i[4]++);
          if (++st == a.stages) { st = 0; ph ^= 1; }
        }
        if (ptx::elect_one()) ptx::umma_commit(&tfull[acc]);
        __syncwarp();
        continue;
      }
      const uint32_t off_lo = a.a_bytes + a.sb_bytes;
      int kiter = 0;
      for (int tap = 0; tap < a.taps; ++tap) {
        for (int kcc = 0; kcc < a.n_kc; ++kcc, ++kiter) {
          ptx::mbar_wait(PST_SPLIT ? &ready[st] : &full[st], ph);
          if (lane == 0) TL(3, dbg_i[3]++);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(ring + st * a.stage_bytes);
          const uint64_t ad0 = ptx::smem_desc(sa, 2048, 128);
          const uint64_t bd0 = ptx::smem_desc(sa + a.a_bytes, a.BN * 16, 128);
          if (ptx::elect_one()) {
            for (int kk = 0; kk < nch / 2; ++kk) {
              const uint64_t ad = ptx::desc_add(ad0, kk * 2 * 2048);
              const uint64_t bd = ptx::desc_add(bd0, kk * 2 * (a.BN * 16));
              ptx::umma(dtm, ad, bd, idesc, (kiter > 0 || kk > 0) ? 1u : 0u);
#if PST_SPLIT
              ptx::umma(dtm, ad, ptx::desc_add(bd, off_lo), idesc, 1u);
              ptx::umma(dtm, ptx::desc_add(ad, off_lo), bd, idesc, 1u);
#endif
            }
            ptx::umma_commit(&empty[st]);
          }
          __syncwarp();
          if (lane == 0) TL(4, dbg_i[4]++);
          if (++st == a.stages) { st = 0; ph ^= 1; }
        }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;            // TMEM lane quarter accessible by this warp
    const int row = q * 32 + lane;     // pixel row within the tile
    const int et = threadIdx.x - 64;   // 0..127
    int local = 0;
    for (int t = blockIdx.x; t < a.n_tiles; t += gridDim.x, ++local) {
      const int mt = t / a.n_ntiles, nt = t % a.n_ntiles;
      const int acc = local & 1;
      const uint32_t use = (uint32_t)(local >> 1);
      ptx::mbar_wait(&tfull[acc], use & 1);
      if (threadIdx.x == 64) TL(5, dbg_i[5]++);
      ptx::tc_fence_after();
      const int g0s = HALO ? (mt % a.tpi) * 128 * a.MT : 0;
      const int mts = HALO ? min(a.MT, (a.Pimg - g0s + 127) / 128) : 1;
      for (int j = 0; j < mts; ++j) {
      int n, y, x;
      if (HALO) {
        n = mt / a.tpi;
        const int g = g0s + j * 128 + row;
        y = g / a.Wv;
        x = g % a.Wv;
      } else {
        decode_tile_px(a, mt, row, n, y, x);
      }
      const bool valid = (n < a.N) && (y < a.Ho) && (x < a.Wo);
      const int64_t pix = ((int64_t)n * a.Ho + y) * a.Wo + x;
      const int64_t npix = (int64_t)a.N * a.Ho * a.Wo;
      for (int ch = 0; ch < a.BN / 16; ++ch) {
        float v[16];
        const uint32_t col = HALO ? (uint32_t)((acc * a.MT + j) * a.BN) : (uint32_t)(acc * a.BN);
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + col + ch * 16;
        ptx::tmem_ld16(taddr, v);
        if (ch == a.BN / 16 - 1 && j == mts - 1) {
          ptx::tc_fence_before();
          if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        }
        const int c0 = nt * a.BN + ch * 16;
        if (a.epi == EPI_BN_STATS) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = valid ? act2f(f2act(v[i])) : 0.f;
        } else if (a.epi == EPI_BIAS_ACT || a.epi == EPI_BIAS_F32) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = c0 + i;
            const float b = (a.bias != nullptr && c < a.Cout) ? __ldg(&a.bias[c]) : 0.f;
            float o = v[i] + b;
            if (a.relu) o = fmaxf(o, 0.f);
            v[i] = (c < a.Cout) ? o : 0.f;
          }
        } else {  // EPI_DGRAD: + shortcut^T of the residual layer's gradient
          if (valid && a.res_mode == 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += ld_planar(a.res, npix, pix, c0 + i);
          } else if (valid && a.res_mode == 2 && ((y | x) & 1) == 0) {
            const int64_t rpix = ((int64_t)n * a.res_H + (y >> 1)) * a.res_W + (x >> 1);
            const int64_t rnpix = (int64_t)a.N * a.res_H * a.res_W;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int c = c0 + i;
              if (c < a.Cout) v[i] += ld_planar(a.res, rnpix, rpix, c + a.res_pad);
            }
          }
        }
        if (valid) {
          if (a.epi == EPI_BIAS_F32) store16_f32(reinterpret_cast<float*>(a.out), npix, pix, c0, v);
          else store16_planar(reinterpret_cast<act_t*>(a.out), npix, pix, c0, v);
        }
        if (a.epi == EPI_BN_STATS) {
          // per-channel sums over the 128 pixel rows via an smem transpose
#pragma unroll
          for (int i = 0; i < 16; ++i) sbuf[i * 129 + row] = v[i];
          ptx::named_bar_sync(1, kEpiThreads);
          const int c = et >> 3, part = et & 7;
          float s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float u = sbuf[c * 129 + part * 16 + j];
            s1 += u;
            s2 += u * u;
          }
#pragma unroll
          for (int o = 1; o < 8; o <<= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          }
          if (part == 0) {
            cacc[2 * (c0 + c)] += (double)s1;
            cacc[2 * (c0 + c) + 1] += (double)s2;
          }
          ptx::named_bar_sync(1, kEpiThreads);
        }
      }
      }  // sub-tiles j
      if (threadIdx.x == 64) TL(6, dbg_i[6]++);
    }
    if (a.epi == EPI_BN_STATS) {
      ptx::named_bar_sync(1, kEpiThreads);
      for (int i = et; i < 2 * a.Coutp; i += kEpiThreads)
        if (cacc[i] != 0.0) atomicAdd(&a.stats[i], cacc[i]);
    }
  } else {
#if PST_SPLIT
    // ------------------------------------------------------------ 3xTF32 split converter (warps 6..9)
    const int ct = threadIdx.x - kBaseThreads;   // 0..127
    int st = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < a.n_tiles; t += gridDim.x) {
      for (int kit = 0; kit < (HALO ? 1 : a.taps) * a.n_kc; ++kit) {
        ptx::mbar_wait(&full[st], ph);
        if (ct == 0) TL(1, dbg_i[1]++);
        uint8_t* sa = ring + st * a.stage_bytes;
        split_lo(sa, sa + a.a_bytes + a.sb_bytes, a.a_bytes, ct);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ready[st]);
        if (ct == 0) TL(2, dbg_i[2]++);
        if (++st == a.stages) { st = 0; ph ^= 1; }
      }
    }
#endif
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// ---------------------------------------------------------------- weight gradient
// pixels per K stage.  The 3xTF32 build stages 32 pixels: kind::tf32 needs
// K-major operands, so the converter transposes each [pixel][4 ch] chunk into
// K-major core matrices (8 rows x 4 pixels) in place while it splits hi/lo.
constexpr int kWgPix = PST_SPLIT ? 32 : 64;
constexpr int kWgSbo = (kWgPix / 4) * 128;   // split build: byte stride between 8-row groups
constexpr int kWgUnitsPerThread = 6;         // split build: 4x4 transpose blocks per converter thread

// split build: raw MN-major [chunk][px][4 ch] -> K-major hi (in place) and lo planes
__device__ __forceinline__ void split_transpose(uint8_t* base, uint8_t* lo_base, int nchunks, int ct) {
  const int units = nchunks * (kWgPix / 4);
  float4 v[kWgUnitsPerThread][4];
#pragma unroll
  for (int i = 0; i < kWgUnitsPerThread; ++i) {
    const int u = ct + i * 128;
    if (u < units) {
      const int q = u / (kWgPix / 4), pq = u % (kWgPix / 4);
      const float4* src = reinterpret_cast<const float4*>(base + (q * kWgPix + 4 * pq) * 16);
#pragma unroll
      for (int k = 0; k < 4; ++k) v[i][k] = src[k];
    }
  }
  ptx::named_bar_sync(2, 128);
#pragma unroll
  for (int i = 0; i < kWgUnitsPerThread; ++i) {
    const int u = ct + i * 128;
    if (u < units) {
      const int q = u / (kWgPix / 4), pq = u % (kWgPix / 4);
      const float* f = reinterpret_cast<const float*>(v[i]);   // f[px*4 + ch]
#pragma unroll
      for (int cl = 0; cl < 4; ++cl) {
        const int r = 4 * q + cl;
        const uint32_t off = (uint32_t)((r >> 3) * kWgSbo + pq * 128 + (r & 7) * 16);
        const float4 hi = make_float4(f[cl], f[4 + cl], f[8 + cl], f[12 + cl]);
        *reinterpret_cast<float4*>(base + off) = hi;
        *reinterpret_cast<float4*>(lo_base + off) =
            make_float4(tf32_lo(hi.x), tf32_lo(hi.y), tf32_lo(hi.z), tf32_lo(hi.w));
      }
    }
  }
}

struct WgArgs {
  int N, Ho, Wo;
  int bimg, bh, bw, tn, ty, tx, n_ptiles;
  int Cinp, Coutp, BNw, n_ntiles, k, taps, S, pad;
  int rows, n_mt, G, n_mgroups, ksplit;
  int stages;
  uint32_t x_bytes, d_bytes, stage_bytes;
  uint32_t tmem_cols;
  float* part;
  int x4, d4;   // act_tmap forms
};

__global__ void __launch_bounds__(kThreads, 1)
    conv_wgrad_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD,
                      const WgArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // stage: [X raw (x_bytes)][dY raw (d_bytes)]([X lo][dY lo] in the split build)
  uint8_t* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.stages * a.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* ready = bars + 2 * kMaxStages;
  uint64_t* tfull = bars + 3 * kMaxStages;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 3 * kMaxStages + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int b = blockIdx.x;
  const int mg = b % a.n_mgroups;
  const int nt = (b / a.n_mgroups) % a.n_ntiles;
  const int ks = b / (a.n_mgroups * a.n_ntiles);
  const int p_lo = (int)((int64_t)ks * a.n_ptiles / a.ksplit);
  const int p_hi = (int)((int64_t)(ks + 1) * a.n_ptiles / a.ksplit);
  const int mt0 = mg * a.G;
  const int g_cnt = min(a.G, a.n_mt - mt0);
  const int r0 = mt0 * 128;
  const int r_end = min(r0 + g_cnt * 128, a.rows);
  const int q0 = r0 / kEPC, q1 = (r_end + kEPC - 1) / kEPC;   // global row chunks loaded: [q0, q1)
  const int cin_c = a.Cinp / kEPC, bn_c = a.BNw / kEPC;
  const uint32_t used_x = (uint32_t)(q1 - q0) * (kWgPix * 16);
  const uint32_t used_d = (uint32_t)bn_c * (kWgPix * 16);

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
      ptx::mbar_init(&ready[i], 4);
    }
    ptx::mbar_init(&tfull[0], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_ptr, a.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  pdl_wait();      // no global memory access above this line
  pdl_trigger();
  const int n_iter = p_hi - p_lo;

  if (warp == 0) {
    if (lane == 0 && n_iter > 0) {
      ptx::prefetch_tmap(&tmX);
      ptx::prefetch_tmap(&tmD);
      int st = 0;
      uint32_t ph = 0;
      for (int pt = p_lo; pt < p_hi; ++pt) {
        const int ix = pt % a.tx, iy = (pt / a.tx) % a.ty, it = pt / (a.tx * a.ty);
        const int xo = ix * a.bw, yo = iy * a.bh, n0 = it * a.bimg;
        ptx::mbar_wait(&empty[st], ph ^ 1);
        ptx::mbar_expect_tx(&full[st], used_x + used_d);
        uint8_t* sx = ring + st * a.stage_bytes;
        uint8_t* sd = sx + a.x_bytes;
        tma_act(sd, &tmD, &full[st], a.d4, xo, yo, n0, nt * bn_c);   // all bn_c planes, one box
        for (int qq = q0; qq < q1; ++qq) {
          const int tap = qq / cin_c, cc = qq % cin_c;
          const int r = tap / a.k, s = tap % a.k;
          tma_act(sx + (qq - q0) * (kWgPix * 16), &tmX, &full[st], a.x4, xo * a.S - a.pad + s,
                  yo * a.S - a.pad + r, n0, cc);
        }
        if (++st == a.stages) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && n_iter > 0) {
#if PST_SPLIT
      const uint32_t idesc = ptx::idesc_mma(128, a.BNw, 0, 0, PST_AB_FORMAT);   // K-major (converted)
#else
      const uint32_t idesc = ptx::idesc_mma(128, a.BNw, 1, 1, PST_AB_FORMAT);   // MN-major (as loaded)
#endif
      const uint32_t mtile_bytes = 128 * kWgPix * (uint32_t)sizeof(act_t);   // one 128-row M tile
      int st = 0;
      uint32_t ph = 0;
      for (int it = 0; it < n_iter; ++it) {
        ptx::mbar_wait(PST_SPLIT ? &ready[st] : &full[st], ph);
        ptx::tc_fence_after();
        const uint32_t sx = ptx::smem_u32(ring + st * a.stage_bytes);
        const uint32_t sd = sx + a.x_bytes;
        for (int j = 0; j < g_cnt; ++j) {
          const uint32_t abase = sx + (uint32_t)j * mtile_bytes;
          const uint32_t dt = tmem_base + j * a.BNw;
          for (int kk = 0; kk < kWgPix / kMmaK; ++kk) {
#if PST_SPLIT
            // K-major: core matrix = 8 rows x 4 pixels (128 B); LBO 128 (next 4 px), SBO = 8-row group
            const uint32_t lo = a.x_bytes + a.d_bytes;
            const uint64_t ad = ptx::smem_desc(abase + kk * 256, 128, kWgSbo);
            const uint64_t bd = ptx::smem_desc(sd + kk * 256, 128, kWgSbo);
            const uint64_t adl = ptx::smem_desc(abase + lo + kk * 256, 128, kWgSbo);
            const uint64_t bdl = ptx::smem_desc(sd + lo + kk * 256, 128, kWgSbo);
            ptx::umma(dt, ad, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
            ptx::umma(dt, ad, bdl, idesc, 1u);
            ptx::umma(dt, adl, bd, idesc, 1u);
#else
            const uint64_t ad = ptx::smem_desc(abase + kk * kMmaK * 16, 128, kWgPix * 16);
            const uint64_t bd = ptx::smem_desc(sd + kk * kMmaK * 16, 128, kWgPix * 16);
            ptx::umma(dt, ad, bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
#endif
          }
        }
        ptx::umma_commit(&empty[st]);
        if (++st == a.stages) { st = 0; ph ^= 1; }
      }
      ptx::umma_commit(&tfull[0]);
    }
  } else if (warp < 6) {
    const int q = warp & 3;
    const int rowl = q * 32 + lane;
    if (n_iter > 0) {
      ptx::mbar_wait(&tfull[0], 0);
      ptx::tc_fence_after();
    }
    for (int j = 0; j < g_cnt; ++j) {
      const int rg = r0 + j * 128 + rowl;
      for (int ch = 0; ch < a.BNw / 16; ++ch) {
        float v[16];
        if (n_iter > 0) {
          ptx::tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + j * a.BNw + ch * 16, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (rg < a.rows) {
          float4* op = reinterpret_cast<float4*>(a.part + ((int64_t)ks * a.rows + rg) * a.Coutp +
                                                 nt * a.BNw + ch * 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) op[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
    }
  } else {
#if PST_SPLIT
    const int ct = threadIdx.x - kBaseThreads;
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < n_iter; ++it) {
      ptx::mbar_wait(&full[st], ph);
      uint8_t* sx = ring + st * a.stage_bytes;
      const uint32_t lo = a.x_bytes + a.d_bytes;
      split_transpose(sx, sx + lo, q1 - q0, ct);
      split_transpose(sx + a.x_bytes, sx + a.x_bytes + lo, bn_c, ct);
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ready[st]);
      if (++st == a.stages) { st = 0; ph ^= 1; }
    }
#endif
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// ---------------------------------------------------------------- weight gradient, 3xTF32 build
// One K stage = P output pixels (nb images x bh rows x Wo cols).  Two TMA boxes per
// stage: the dY tile (all bn_c planes) and the input band that every tap of those
// pixels reads (band_r x band_c pixels per image, the group's channel planes).  The
// converter warpgroup then builds, in shared memory, the K-major hi/lo operand rows
// (tap, ci) x P -- the 9-fold tap replication happens in smem, not through TMA.
struct WbArgs {
  int N, H, W, Cinp, Ho, Wo, Coutp;
  int k, S, pad;
  int nb, bh, P, P8, band_r, band_c, ny, n_units;
  int rows, n_mt, G, n_mgroups, BNw, n_ntiles, ksplit;
  int pl_grp, pl_all;   // X planes per box; whether every group loads all planes
  int stages;
  uint32_t rawx_bytes, rawx_tx, rawd_bytes, a_bytes, d_bytes, stage_bytes, sbo;
  uint32_t tmem_cols;
  float* part;
  unsigned long long* dbg;
};

__global__ void __launch_bounds__(kThreads, 1)
    conv_wgrad_band_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD,
                           const WbArgs a) {
  int dbg_i[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (threadIdx.x == 0) TL(7, 0);
  extern __shared__ __align__(1024) uint8_t smem[];
  // stage: [raw X][raw dY][A hi][A lo][D hi][D lo]
  uint8_t* ring = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.stages * a.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* ready = bars + 2 * kMaxStages;
  uint64_t* tfull = bars + 3 * kMaxStages;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 3 * kMaxStages + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int b = blockIdx.x;
  const int mg = b % a.n_mgroups;
  const int nt = (b / a.n_mgroups) % a.n_ntiles;
  const int ks = b / (a.n_mgroups * a.n_ntiles);
  const int u_lo = (int)((int64_t)ks * a.n_units / a.ksplit);
  const int u_hi = (int)((int64_t)(ks + 1) * a.n_units / a.ksplit);
  const int mt0 = mg * a.G;
  const int g_cnt = min(a.G, a.n_mt - mt0);
  const int r0 = mt0 * 128;
  const int r_end = min(r0 + g_cnt * 128, a.rows);
  const int pl0 = a.pl_all ? 0 : (r0 % a.Cinp) / kEPC;
  const int bn_c = a.BNw / kEPC;
  const int n_iter = u_hi - u_lo;
  const uint32_t off_rawd = a.rawx_bytes;
  const uint32_t off_a = off_rawd + a.rawd_bytes;
  const uint32_t off_d = off_a + 2 * a.a_bytes;

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
      ptx::mbar_init(&ready[i], 8);
    }
    ptx::mbar_init(&tfull[0], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_ptr, a.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  pdl_wait();      // no global memory access above this line
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0 && n_iter > 0) {
      ptx::prefetch_tmap(&tmX);
      ptx::prefetch_tmap(&tmD);
      int st = 0;
      uint32_t ph = 0;
      for (int u = u_lo; u < u_hi; ++u) {
        const int n0 = (u / a.ny) * a.nb, y0 = (u % a.ny) * a.bh;
        ptx::mbar_wait(&empty[st], ph ^ 1);
        TL(0, dbg_i[0]++);
        ptx::mbar_expect_tx(&full[st], a.rawx_tx + a.rawd_bytes);
        uint8_t* s0 = ring + st * a.stage_bytes;
        ptx::tma_load_4d(s0, &tmX, &full[st], -a.pad * kEPC, y0 * a.S - a.pad, n0, pl0);
        ptx::tma_load_4d(s0 + off_rawd, &tmD, &full[st], 0, y0, n0, nt * bn_c);
        if (++st == a.stages) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (n_iter > 0) {
      const uint32_t idesc = ptx::idesc_mma(128, a.BNw, 0, 0, PST_AB_FORMAT);
      const uint32_t mtile = 16 * a.sbo;   // 128 rows
      int st = 0;
      uint32_t ph = 0;
      for (int it = 0; it < n_iter; ++it) {
        ptx::mbar_wait(&ready[st], ph);
        if (lane == 0) TL(3, dbg_i[3]++);
        ptx::tc_fence_after();
        const uint32_t s0 = ptx::smem_u32(ring + st * a.stage_bytes);
        const uint64_t ad0 = ptx::smem_desc(s0 + off_a, 128, a.sbo);
        const uint64_t bd0 = ptx::smem_desc(s0 + off_d, 128, a.sbo);
        if (ptx::elect_one()) {
          // consecutive MMAs target different accumulators (M tiles)
          for (int kk = 0; kk < a.P8 / 8; ++kk) {
            const uint64_t bd = ptx::desc_add(bd0, kk * 256);
            const uint64_t bdl = ptx::desc_add(bd, a.d_bytes);
            const uint64_t ak = ptx::desc_add(ad0, kk * 256);
            for (int j = 0; j < g_cnt; ++j)
              ptx::umma(tmem_base + j * a.BNw, ptx::desc_add(ak, j * mtile), bd, idesc, (it > 0 || kk > 0) ? 1u : 0u);
            for (int j = 0; j < g_cnt; ++j)
              ptx::umma(tmem_base + j * a.BNw, ptx::desc_add(ak, j * mtile), bdl, idesc, 1u);
            for (int j = 0; j < g_cnt; ++j)
              ptx::umma(tmem_base + j * a.BNw, ptx::desc_add(ak, a.a_bytes + j * mtile), bd, idesc, 1u);
          }
          ptx::umma_commit(&empty[st]);
        }
        __syncwarp();
        if (lane == 0) TL(4, dbg_i[4]++);
        if (++st == a.stages) { st = 0; ph ^= 1; }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[0]);
      __syncwarp();
    }
  } else {
    // Warps 2..9 convert every stage (raw band / raw dY -> K-major hi/lo operands); warps
    // 2..5 then drain the accumulators.  One task = 4 operand rows (one 16-byte channel
    // quad of one tap) x 4 pixels: four 16-byte loads (one per pixel) transposed into four
    // 16-byte K-major row segments.  Lane bits: 0 = row-quad parity, 1-2 = pixel quad (low),
    // which also rotates the store order -> the 8 lanes of each 16-byte store phase hit 8
    // distinct bank quads.
    const int ct = threadIdx.x - 64;            // 0..255
    const int hw = a.bh * a.Wo;
    const int nq = a.P8 / 4;
    const int nqh = (nq + 3) / 4;
    const int arows = g_cnt * 128;
    const int mqA = arows / 4, mqD = a.BNw / 4;
    int* rowbase = reinterpret_cast<int*>(smem + a.stages * a.stage_bytes + (3 * kMaxStages + 2) * 8 + 16);
    int* pixb = rowbase + g_cnt * 128;
    for (int mq = ct; mq < mqA; mq += 256) {
      const int R = r0 + 4 * mq;
      if (R >= r_end) { rowbase[mq] = -1; continue; }
      const int tap = R / a.Cinp, ci = R % a.Cinp;
      const int r = tap / a.k, s2 = tap % a.k;
      const int plane = ci / kEPC - pl0;
      rowbase[mq] = ((plane * a.nb * a.band_r + r) * a.band_c + s2) * 4;
    }
    for (int p = ct; p < a.P8; p += 256) {
      if (p >= a.P) { pixb[p] = -1; continue; }
      const int jj = p / hw, py = (p / a.Wo) % a.bh, px = p % a.Wo;
      pixb[p] = ((jj * a.band_r + py * a.S) * a.band_c + px * a.S) * 4;
    }
    ptx::named_bar_sync(2, 256);
    const int par = ct & 1, kql = (ct >> 1) & 3;
    const int rot = kql;                        // store / load rotation
    const int tasksA = (mqA / 2) * nqh, tasksD = ((mqD + 1) / 2) * nqh;
    int st = 0;
    uint32_t ph = 0;
    for (int it = 0; it < n_iter; ++it) {
      ptx::mbar_wait(&full[st], ph);
      if (ct == 0) TL(1, dbg_i[1]++);
      uint8_t* s0 = ring + st * a.stage_bytes;
      const float* rawxf = reinterpret_cast<const float*>(s0);
      const float* rawdf = reinterpret_cast<const float*>(s0 + off_rawd);
      uint8_t* ahi = s0 + off_a;
      uint8_t* alo = ahi + a.a_bytes;
      uint8_t* dhi = s0 + off_d;
      uint8_t* dlo = dhi + a.d_bytes;
      for (int rest = ct >> 3; rest < tasksA + tasksD; rest += 32) {
        const bool isA = rest < tasksA;
        const int rr = isA ? rest : rest - tasksA;
        const int kq = (rr % nqh) * 4 + kql;
        const int mq = (rr / nqh) * 2 + par;
        if (kq >= nq || (!isA && mq >= mqD)) continue;
        float4 v[4];
        if (isA) {
          const int rb = rowbase[mq];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int pb = pixb[4 * kq + i];
            v[i] = (rb >= 0 && pb >= 0) ? *reinterpret_cast<const float4*>(rawxf + rb + pb)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int p = 4 * kq + i;
            v[i] = p < a.P ? *reinterpret_cast<const float4*>(rawdf + ((int64_t)mq * a.P + p) * 4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        uint8_t* hi = isA ? ahi : dhi;
        uint8_t* lo = isA ? alo : dlo;
        const uint32_t base = (uint32_t)((mq >> 1) * a.sbo + kq * 128 + (mq & 1) * 64);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = (j + rot) & 3;          // row c of the quad = channel c over the 4 pixels
          float4 h;
          if (c == 0) h = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
          else if (c == 1) h = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
          else if (c == 2) h = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
          else h = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
          const uint32_t off = base + c * 16;
          *reinterpret_cast<float4*>(hi + off) = h;
          *reinterpret_cast<float4*>(lo + off) = make_float4(tf32_lo(h.x), tf32_lo(h.y), tf32_lo(h.z), tf32_lo(h.w));
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ready[st]);
      if (ct == 0) TL(2, dbg_i[2]++);
      if (++st == a.stages) { st = 0; ph ^= 1; }
    }
    if (warp < 6) {
      // epilogue: accumulators -> split-K partials
      const int q = warp & 3;
      const int rowl = q * 32 + lane;
      if (n_iter > 0) {
        ptx::mbar_wait(&tfull[0], 0);
        ptx::tc_fence_after();
      }
      if (threadIdx.x == 64) TL(5, 0);
      for (int j = 0; j < g_cnt; ++j) {
        const int rg = r0 + j * 128 + rowl;
        for (int ch = 0; ch < a.BNw / 16; ++ch) {
          float v[16];
          if (n_iter > 0) {
            ptx::tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + j * a.BNw + ch * 16, v);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          }
          if (rg < a.rows) {
            float4* op = reinterpret_cast<float4*>(a.part + ((int64_t)ks * a.rows + rg) * a.Coutp + nt * a.BNw + ch * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) op[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, a.tmem_cols);
  }
}

// largest multiple of 16 that divides C and is <= cap (C a multiple of 16)
int tile_n(int C, int cap) {
  int best = 16;
  for (int b = 16; b <= cap && b <= C; b += 16)
    if (C % b == 0) best = b;
  return best;
}

int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

void pixel_tile(int N, int Ho, int Wo, int npx, int& bimg, int& bh, int& bw) {
  (void)N;
  bw = std::min(pow2_at_least(Wo), npx);
  bh = std::min(pow2_at_least(Ho), npx / bw);
  bimg = npx / (bw * bh);
}

// channel-planar activation map.  smem receives [plane][img][y][x][16 B]: nch K-major
// core-matrix columns of 128 pixel rows.
//  stride 1: dims (W*EPC, H, N, Cp/EPC), box (bw*EPC, bh, bimg, nch) -- the innermost box
//            extent is a whole run of bw pixels (bw*16 bytes), so TMA moves long rows;
//            x coordinates are in elements (x*EPC).
//  stride 2: dims (EPC, W, H, N, Cp/EPC) with element strides (1, 2, 2, 1, 1).
CUtensorMap act_tmap(const act_t* p, int N, int H, int W, int Cp, int bimg, int bh, int bw, int S, int nch) {
  if (S == 1 && bw * kEPC <= 256) {
    uint64_t dims[4] = {(uint64_t)W * kEPC, (uint64_t)H, (uint64_t)N, (uint64_t)Cp / kEPC};
    uint64_t str[3] = {(uint64_t)W * 16, (uint64_t)H * W * 16, (uint64_t)N * H * W * 16};
    uint32_t box[4] = {(uint32_t)(bw * kEPC), (uint32_t)bh, (uint32_t)bimg, (uint32_t)nch};
    return make_tmap(act_tmap_dtype(), 4, p, dims, str, box, nullptr);
  }
  uint64_t dims[5] = {(uint64_t)kEPC, (uint64_t)W, (uint64_t)H, (uint64_t)N, (uint64_t)Cp / kEPC};
  uint64_t str[4] = {16, (uint64_t)W * 16, (uint64_t)H * W * 16, (uint64_t)N * H * W * 16};
  uint32_t box[5] = {(uint32_t)kEPC, (uint32_t)(bw * S), (uint32_t)(bh * S), (uint32_t)bimg, (uint32_t)nch};
  uint32_t est[5] = {1, (uint32_t)S, (uint32_t)S, 1, 1};
  return make_tmap(act_tmap_dtype(), 5, p, dims, str, box, est);
}
inline bool act_tmap_is4d(int S, int bw) { return S == 1 && bw * kEPC <= 256; }

// weight shadow map over [taps][Cinp/EPC][Coutp][EPC]; smem receives [plane][BN rows][16 B].
//  BN*EPC <= 256: dims (Coutp*EPC, Cinp/EPC, taps), box (BN*EPC, nch, 1) -- long rows;
//  else         : dims (EPC, Coutp, Cinp/EPC, taps), box (EPC, BN, nch, 1).
inline bool w_tmap_is3d(int BN) { return BN * kEPC <= 256; }
CUtensorMap w_tmap(const act_t* p, int taps, int Coutp, int Cinp, int BN, int nch, int box_taps = 1) {
  if (w_tmap_is3d(BN)) {
    uint64_t wd[3] = {(uint64_t)Coutp * kEPC, (uint64_t)Cinp / kEPC, (uint64_t)taps};
    uint64_t ws[2] = {(uint64_t)Coutp * 16, (uint64_t)Coutp * Cinp * sizeof(act_t)};
    uint32_t wb[3] = {(uint32_t)(BN * kEPC), (uint32_t)nch, (uint32_t)box_taps};
    return make_tmap(act_tmap_dtype(), 3, p, wd, ws, wb, nullptr);
  }
  uint64_t wd[4] = {(uint64_t)kEPC, (uint64_t)Coutp, (uint64_t)Cinp / kEPC, (uint64_t)taps};
  uint64_t ws[3] = {16, (uint64_t)Coutp * 16, (uint64_t)Coutp * Cinp * sizeof(act_t)};
  uint32_t wb[4] = {(uint32_t)kEPC, (uint32_t)BN, (uint32_t)nch, (uint32_t)box_taps};
  return make_tmap(act_tmap_dtype(), 4, p, wd, ws, wb, nullptr);
}

int choose_wg_G(int n_mt, int BNw) {
  int G = std::max(1, std::min(n_mt, 512 / BNw));
  const int lo = PST_SPLIT ? 2 : 1;
  while (G > 1 && lo * (G * (128 / kEPC) + BNw / kEPC) * (kWgPix * 16) > 96 * 1024) --G;
  // split build: each converter thread transposes at most kWgUnitsPerThread 4x4 blocks
  while (PST_SPLIT && G > 1 && (G * (128 / kEPC) + BNw / kEPC) * (kWgPix / 4) > 128 * kWgUnitsPerThread) --G;
  return G;
}

}  // namespace

void conv_tc(const ConvSpec& c, cudaStream_t st) {
  PST_CHECK_ARG(c.Cinp % 16 == 0 && c.Coutp % 16 == 0, "conv channels must be padded to 16");
  PST_CHECK_ARG(c.S == 1 || c.S == 2, "conv stride must be 1 or 2");
  PST_CHECK_ARG((reinterpret_cast<uintptr_t>(c.in) & 15) == 0, "conv input must be 16B aligned");
  if (conv_ts(c, st)) return;
  PST_CHECK_ARG(!c.pre, "the band pre-pass needs the TS conv kernel");
  PST_CHECK_ARG(!c.bfuse,"fused bwd_pre needs the TS conv kernel");   // activation operand in TMEM (conv_ts.cu) where the tiling fits
  FwdArgs a{};
  a.N = c.N; a.Ho = c.Ho; a.Wo = c.Wo;
  pixel_tile(c.N, c.Ho, c.Wo, 128, a.bimg, a.bh, a.bw);
  a.tn = ceil_div(c.N, a.bimg); a.ty = ceil_div(c.Ho, a.bh); a.tx = ceil_div(c.Wo, a.bw);
  a.n_mtiles = a.tn * a.ty * a.tx;
  a.BN = tile_n(c.Coutp, 256);
  a.n_ntiles = c.Coutp / a.BN;
  a.n_tiles = a.n_mtiles * a.n_ntiles;
  a.Cinp = c.Cinp;
  // channels per K stage: <= 128 bytes per pixel, a multiple of one MMA's K (2 chunks)
  const int kc_max = 128 / (int)sizeof(act_t);
  a.kc = 2 * kEPC;
  for (int kc = 2 * kEPC; kc <= kc_max; kc += 2 * kEPC)
    if (c.Cinp % kc == 0) a.kc = kc;
  a.n_kc = c.Cinp / a.kc;
  a.k = c.k; a.taps = c.k * c.k; a.S = c.S; a.off = c.off; a.sgn = c.sgn;
  a.Coutp = c.Coutp; a.Cout = c.Cout;
  const int nch = a.kc / kEPC;
  const int budget = 190 * 1024;
  const int xsplit = PST_SPLIT ? 2 : 1;
  // ---- HALO plan (stride 1, wide images): virtual grid of pitch Wv, one band per tile
  bool halo = false;
  int nch_h = nch;
  // HALO by default where it applies (PST_NOHALO=1: per-tap loads everywhere, for comparison)
  static const bool halo_on = pst_knob("PST_NOHALO", 0) == 0;
  const int o1 = c.off, o2 = c.off + c.sgn * (c.k - 1);
  const int lo = std::min(o1, o2), hi = std::max(o1, o2);
  const int Wv = c.Wo + (hi - lo);   // virtual-grid row pitch = band row = output row + halo columns
  if (halo_on && c.S == 1 && c.k > 1 && c.Wo >= 16 && Wv * kEPC <= 256) {
    // candidates: M tiles per super tile (independent accumulators) x channels per stage
    for (int MT : {2, 1}) {
      if (halo) break;
      if (2 * MT * a.BN > 512) continue;
      for (int kc = a.kc; kc >= 2 * kEPC && !halo; kc -= 2 * kEPC) {
        if (c.Cinp % kc) continue;
        const int nc = kc / kEPC, nkc = c.Cinp / kc;
        // rows spanned by 128*MT consecutive positions starting anywhere in a row, + halo rows
        const int band_r = (128 * MT + Wv - 2) / Wv + 1 + (hi - lo);
        const uint32_t plane = (uint32_t)band_r * Wv * 16;
        if (band_r > 256 || plane >= (1u << 18)) continue;
        const uint32_t ab_tx = plane * nc;                           // band box bytes
        const uint32_t ab = (uint32_t)round_up((int)ab_tx, 128);     // smem footprint (128-B aligned)
        const uint32_t bb = (uint32_t)a.taps * nc * a.BN * 16;      // one chunk, all taps
        const uint32_t wres_all = bb * nkc * xsplit;
        const bool wres = (a.n_ntiles == 1) && wres_all <= 96 * 1024;
        const uint32_t sb = wres ? 0 : bb;
        const uint32_t stage = round_up((int)((ab + sb) * xsplit), 128);
        const int stages = std::min(kMaxStages, (int)((budget - (wres ? wres_all : 0)) / stage));
        if (stages < 2) continue;
        halo = true;
        nch_h = nc;
        a.kc = kc; a.n_kc = nkc;
        a.Wv = Wv; a.lo = lo; a.MT = MT;
        a.Pimg = c.Ho * Wv;
        a.tpi = ceil_div(a.Pimg, 128 * MT);
        a.n_mtiles = c.N * a.tpi;
        a.n_tiles = a.n_mtiles * a.n_ntiles;
        a.plane_bytes = plane;
        a.a_bytes = ab; a.b_bytes = bb; a.sb_bytes = sb;
        a.wres_bytes = wres ? wres_all : 0;
        a.tx_bytes = ab_tx + sb * xsplit;
        a.stage_bytes = stage;
        a.stages = stages;
        for (int t = 0; t < a.taps; ++t) {
          const int oy = c.off + c.sgn * (t / c.k), ox = c.off + c.sgn * (t % c.k);
          a.tapoff[t] = ((oy - lo) * Wv + (ox - lo)) * 16;   // bytes: a 16-B aligned row shift
        }
      }
    }
  }
  int nch_nh = nch;
  if (!halo) {
    // the fixed smem (epilogue scratch, per-channel stat slots of all Coutp channels, barriers)
    // grows with Coutp (e.g. AlexNet's FC 4096->2048 as a valid conv): shrink the channel chunk
    // until two stages fit beside it
    const int fixed = (16 * 129 + 4) * 4 + 2 * c.Coutp * 8 + (3 * kMaxStages + 5) * 8 + 16;
    const int room = std::min(budget, 227 * 1024 - fixed);
    for (int n = nch; n >= 2; n -= 2) {
      if ((c.Cinp / kEPC) % n != 0) continue;
      nch_nh = n;
      if (2 * (n * 2048 + n * a.BN * 16) * xsplit <= room) break;
    }
    if (nch_nh != nch) { a.kc = nch_nh * kEPC; a.n_kc = c.Cinp / a.kc; }
    a.a_bytes = (uint32_t)nch_nh * 2048;
    a.b_bytes = (uint32_t)nch_nh * a.BN * 16;
    a.sb_bytes = a.b_bytes;
    a.wres_bytes = 0;
    a.tx_bytes = a.a_bytes + a.b_bytes * xsplit;
    a.stage_bytes = (a.a_bytes + a.b_bytes) * xsplit;
    a.stages = std::max(2, std::min(kMaxStages, room / (int)a.stage_bytes));
  }
  a.tmem_cols = (uint32_t)std::max(32, pow2_at_least(2 * a.BN * (halo ? a.MT : 1)));
  a.epi = c.epi; a.relu = c.relu; a.out = c.out; a.bias = c.bias; a.stats = c.stats;
  a.res = c.res; a.res_mode = c.res_mode; a.res_H = c.res_H; a.res_W = c.res_W; a.res_C = c.res_C;
  a.res_pad = c.res_pad;
  a.dbg = c.dbg;

  a.a4 = halo ? 1 : (act_tmap_is4d(c.S, a.bw) ? 1 : 0);
  a.b3 = w_tmap_is3d(a.BN) ? 1 : 0;
  CUtensorMap tA;
  if (halo) {  // band box: (Wv*EPC, band_r, 1 image, nch planes)
    const int band_r = (int)(a.plane_bytes / (a.Wv * 16));
    uint64_t dims[4] = {(uint64_t)c.W * kEPC, (uint64_t)c.H, (uint64_t)c.N, (uint64_t)c.Cinp / kEPC};
    uint64_t str[3] = {(uint64_t)c.W * 16, (uint64_t)c.H * c.W * 16, (uint64_t)c.N * c.H * c.W * 16};
    uint32_t box[4] = {(uint32_t)(a.Wv * kEPC), (uint32_t)band_r, 1, (uint32_t)nch_h};
    tA = make_tmap(act_tmap_dtype(), 4, c.in, dims, str, box, nullptr);
  } else {
    tA = act_tmap(c.in, c.N, c.H, c.W, c.Cinp, a.bimg, a.bh, a.bw, c.S, nch_nh);
  }
  const int btaps = halo ? a.taps : 1;
  const int nch_b = halo ? nch_h : nch_nh;
  CUtensorMap tB = w_tmap(c.wshadow, a.taps, c.Coutp, c.Cinp, a.BN, nch_b, btaps);
  CUtensorMap tBlo = PST_SPLIT ? w_tmap(c.wshadow + (size_t)a.taps * c.Coutp * c.Cinp, a.taps, c.Coutp, c.Cinp, a.BN,
                                        nch_b, btaps)
                               : tB;
  const size_t smem = (size_t)a.stages * a.stage_bytes + a.wres_bytes + (16 * 129 + 4) * 4 + 2 * c.Coutp * 8 +
                      (3 * kMaxStages + 5) * 8 + 16;
  PST_CHECK_ARG(smem <= 227 * 1024, "conv smem budget");
  const bool dg = c.epi == EPI_DGRAD;
  auto kern = halo ? (dg ? conv_fwd_kernel<true, true> : conv_fwd_kernel<true, false>)
                   : (dg ? conv_fwd_kernel<false, true> : conv_fwd_kernel<false, false>);
  PST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev;
  PST_CUDA(cudaGetDevice(&dev));
  const int grid = std::min(a.n_tiles, num_sms(dev));
  const double es = sizeof(act_t);
  const double bytes = (double)c.N * c.H * c.W * c.Cinp * es +
                       (double)c.N * c.Ho * c.Wo * c.Coutp * (c.epi == EPI_BIAS_F32 ? 4.0 : es) +
                       (double)a.taps * c.Coutp * c.Cinp * es * (PST_SPLIT ? 2 : 1) +
                       (c.res ? (double)c.N * c.res_H * c.res_W * c.res_C * es : 0.0);
  const double flops = 2.0 * c.N * c.Ho * c.Wo * c.Coutp * (double)c.Cinp * a.taps;
  prof::begin(st);
  PST_CUDA(launch_k(kern, dim3(grid), dim3(kThreads), smem, st, tA, tB, tBlo, a));
  PST_CUDA(cudaGetLastError());
  prof::end(st, c.epi == EPI_DGRAD ? prof::CONV_DGRAD : prof::CONV_FWD, bytes, flops);
}

// Stage geometry, M grouping, smem layout and split-K factor of conv_wgrad_band_kernel.
WbArgs plan_band(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad, int num_sm) {
  WbArgs a{};
  a.N = N; a.H = H; a.W = W; a.Cinp = Cinp; a.Ho = Ho; a.Wo = Wo; a.Coutp = Coutp;
  a.k = k; a.S = S; a.pad = pad;
  a.rows = k * k * Cinp;
  a.n_mt = ceil_div(a.rows, 128);
  a.BNw = tile_n(Coutp, 128);
  a.n_ntiles = Coutp / a.BNw;
  const int budget = 200 * 1024;
  for (int ptarget : {32, 16, 8}) {
    if (Ho * Wo >= ptarget) { a.nb = 1; a.bh = std::max(1, std::min(Ho, ptarget / Wo)); }
    else { a.nb = std::max(1, std::min(N, ptarget / (Ho * Wo))); a.bh = Ho; }
    a.P = a.nb * a.bh * Wo;
    a.P8 = round_up(a.P, 8);
    a.band_r = (a.bh - 1) * S + k;
    a.band_c = (Wo - 1) * S + k;
    bool ok = false;
    for (int G = std::min(a.n_mt, std::max(1, 512 / a.BNw)); G >= 1; --G) {
      const bool all = (G * 128 >= Cinp) || (Cinp % (G * 128) != 0);
      const int pl = all ? Cinp / kEPC : G * 128 / kEPC;
      const uint32_t rawx = (uint32_t)pl * a.nb * a.band_r * a.band_c * 16;
      const uint32_t rawd = (uint32_t)(a.BNw / kEPC) * a.P * 16;
      const uint32_t ab = (uint32_t)G * 128 * a.P8 * 4, db = (uint32_t)a.BNw * a.P8 * 4;
      const uint32_t stage = round_up((int)(rawx + rawd), 128) + 2 * ab + 2 * db;
      const bool units_ok = (G * 128 / 4 + a.BNw / 4) * (a.P8 / 4) <= 128 * 64;
      if (a.band_c * kEPC <= 256 && units_ok && 2 * stage <= (uint32_t)budget) {
        a.G = G; a.pl_all = all ? 1 : 0; a.pl_grp = pl;
        a.rawx_bytes = round_up((int)rawx, 128); a.rawx_tx = rawx; a.rawd_bytes = rawd;
        a.a_bytes = ab; a.d_bytes = db; a.stage_bytes = a.rawx_bytes + rawd + 2 * ab + 2 * db;
        ok = true;
        break;
      }
    }
    if (ok) break;
  }
  if (a.G < 1) return a;   // infeasible (huge input bands): caller falls back to per-tap loads
  a.stage_bytes = round_up((int)a.stage_bytes, 1024);
  a.stages = std::max(1, std::min(4, budget / (int)a.stage_bytes));
  a.sbo = (uint32_t)(a.P8 / 4) * 128;
  a.n_mgroups = ceil_div(a.n_mt, a.G);
  a.ny = ceil_div(Ho, a.bh);
  a.n_units = ceil_div(N, a.nb) * a.ny;
  const int base = a.n_mgroups * a.n_ntiles;
  a.ksplit = std::max(1, std::min(std::max(1, a.n_units / 2), num_sm / base));
  a.tmem_cols = (uint32_t)std::max(32, pow2_at_least(a.G * a.BNw));
  return a;
}

WgradPlan wgrad_plan(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad, int num_sm) {
#if PST_SPLIT
  if (const int ks = wgrad_ts_ksplit(N, H, W, Cinp, Ho, Wo, Coutp, k, S, pad, num_sm)) {
    WgradPlan p;
    p.ksplit = ks;
    p.part_floats = (int64_t)ks * k * k * Cinp * Coutp;
    return p;
  }
  {
    const WbArgs b = plan_band(N, H, W, Cinp, Ho, Wo, Coutp, k, S, pad, num_sm);
    if (b.G >= 1) {
      WgradPlan p;
      p.ksplit = b.ksplit;
      p.part_floats = (int64_t)b.ksplit * b.rows * Coutp;
      return p;
    }
  }
#endif
  (void)H; (void)W; (void)S; (void)pad;
  int bimg, bh, bw;
  pixel_tile(N, Ho, Wo, kWgPix, bimg, bh, bw);
  const int n_ptiles = ceil_div(N, bimg) * ceil_div(Ho, bh) * ceil_div(Wo, bw);
  const int rows = k * k * Cinp;
  const int n_mt = ceil_div(rows, 128);
  const int BNw = tile_n(Coutp, 256);
  const int n_nt = Coutp / BNw;
  const int G = choose_wg_G(n_mt, BNw);
  const int n_mg = ceil_div(n_mt, G);
  const int base = n_mg * n_nt;
  int ksplit = std::max(1, std::min(n_ptiles, (2 * num_sm) / base));
  ksplit = std::min(ksplit, std::max(1, n_ptiles / 2));
  WgradPlan p;
  p.ksplit = ksplit;
  p.part_floats = (int64_t)ksplit * rows * Coutp;
  return p;
}

void conv_wgrad_tc(const WgradSpec& w, cudaStream_t st) {
  PST_CHECK_ARG(w.Cinp % 16 == 0 && w.Coutp % 16 == 0, "wgrad channels must be padded to 16");
  if (conv_wgrad_ts(w, st)) return;   // expanded input operand in TMEM (conv_wgrad_ts.cu)
#if PST_SPLIT
  int dev_b;
  PST_CUDA(cudaGetDevice(&dev_b));
  WbArgs b = plan_band(w.N, w.H, w.W, w.Cinp, w.Ho, w.Wo, w.Coutp, w.k, w.S, w.pad, wgrad_sms(dev_b));
  if (b.G >= 1) {
    PST_CHECK_ARG(b.ksplit == w.ksplit, "wgrad: workspace planned for a different split");
    b.part = w.part;
    b.dbg = w.dbg;
    // X: dims (W*EPC, H, N, Cinp/EPC), box (band_c*EPC, band_r, nb, pl_grp)
    uint64_t xd[4] = {(uint64_t)w.W * kEPC, (uint64_t)w.H, (uint64_t)w.N, (uint64_t)w.Cinp / kEPC};
    uint64_t xs[3] = {(uint64_t)w.W * 16, (uint64_t)w.H * w.W * 16, (uint64_t)w.N * w.H * w.W * 16};
    uint32_t xb[4] = {(uint32_t)(b.band_c * kEPC), (uint32_t)b.band_r, (uint32_t)b.nb, (uint32_t)b.pl_grp};
    CUtensorMap tX = make_tmap(act_tmap_dtype(), 4, w.x, xd, xs, xb, nullptr);
    // dY: dims (Wo*EPC, Ho, N, Coutp/EPC), box (Wo*EPC, bh, nb, BNw/EPC)
    uint64_t dd[4] = {(uint64_t)w.Wo * kEPC, (uint64_t)w.Ho, (uint64_t)w.N, (uint64_t)w.Coutp / kEPC};
    uint64_t ds[3] = {(uint64_t)w.Wo * 16, (uint64_t)w.Ho * w.Wo * 16, (uint64_t)w.N * w.Ho * w.Wo * 16};
    uint32_t db[4] = {(uint32_t)(w.Wo * kEPC), (uint32_t)b.bh, (uint32_t)b.nb, (uint32_t)(b.BNw / kEPC)};
    CUtensorMap tD = make_tmap(act_tmap_dtype(), 4, w.dy, dd, ds, db, nullptr);
    const size_t smem = (size_t)b.stages * b.stage_bytes + (3 * kMaxStages + 2) * 8 + 16 + (size_t)(b.G * 128 + b.P8) * 4;
    PST_CHECK_ARG(smem <= 227 * 1024, "wgrad smem budget");
    PST_CUDA(cudaFuncSetAttribute(conv_wgrad_band_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = b.n_mgroups * b.n_ntiles * b.ksplit;
    const double es = sizeof(act_t);
    const double bytes = (double)w.N * w.H * w.W * w.Cinp * es + (double)w.N * w.Ho * w.Wo * w.Coutp * es +
                         (double)b.rows * w.Coutp * 4.0;   // algorithmic: X + dY read, dW written once
    const double flops = 2.0 * b.rows * (double)w.Coutp * w.N * w.Ho * w.Wo;
    prof::begin(st);
    PST_CUDA(launch_k(conv_wgrad_band_kernel, dim3(grid), dim3(kThreads), smem, st, tX, tD, b));
    PST_CUDA(cudaGetLastError());
    prof::end(st, prof::CONV_WGRAD, bytes, flops);
    return;
  }
#endif
  WgArgs a{};
  a.N = w.N; a.Ho = w.Ho; a.Wo = w.Wo;
  pixel_tile(w.N, w.Ho, w.Wo, kWgPix, a.bimg, a.bh, a.bw);
  a.tn = ceil_div(w.N, a.bimg); a.ty = ceil_div(w.Ho, a.bh); a.tx = ceil_div(w.Wo, a.bw);
  a.n_ptiles = a.tn * a.ty * a.tx;
  a.Cinp = w.Cinp; a.Coutp = w.Coutp;
  a.BNw = tile_n(w.Coutp, 256);
  a.n_ntiles = w.Coutp / a.BNw;
  a.k = w.k; a.taps = w.k * w.k; a.S = w.S; a.pad = w.pad;
  a.rows = a.taps * w.Cinp;
  a.n_mt = ceil_div(a.rows, 128);
  a.G = choose_wg_G(a.n_mt, a.BNw);
  a.n_mgroups = ceil_div(a.n_mt, a.G);
  a.ksplit = w.ksplit;
  a.x_bytes = (uint32_t)a.G * (128 / kEPC) * (kWgPix * 16);
  a.d_bytes = (uint32_t)(a.BNw / kEPC) * (kWgPix * 16);
  a.stage_bytes = (a.x_bytes + a.d_bytes) * (PST_SPLIT ? 2 : 1);
  a.stages = std::max(1, std::min(4, (200 * 1024) / (int)a.stage_bytes));
  const size_t smem = (size_t)a.stages * a.stage_bytes + (3 * kMaxStages + 2) * 8 + 16;
  PST_CHECK_ARG(smem <= 227 * 1024, "wgrad smem budget");
  a.tmem_cols = (uint32_t)std::max(32, pow2_at_least(a.G * a.BNw));
  a.part = w.part;

  a.x4 = act_tmap_is4d(w.S, a.bw) ? 1 : 0;
  a.d4 = act_tmap_is4d(1, a.bw) ? 1 : 0;
  CUtensorMap tX = act_tmap(w.x, w.N, w.H, w.W, w.Cinp, a.bimg, a.bh, a.bw, w.S, 1);
  CUtensorMap tD = act_tmap(w.dy, w.N, w.Ho, w.Wo, w.Coutp, a.bimg, a.bh, a.bw, 1, a.BNw / kEPC);
  PST_CUDA(cudaFuncSetAttribute(conv_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = a.n_mgroups * a.n_ntiles * a.ksplit;
  const double es = sizeof(act_t);
  const double bytes = (double)w.N * w.H * w.W * w.Cinp * es + (double)w.N * w.Ho * w.Wo * w.Coutp * es +
                       (double)a.rows * w.Coutp * 4.0;   // algorithmic: X + dY read, dW written once
  const double flops = 2.0 * a.rows * (double)w.Coutp * w.N * w.Ho * w.Wo;
  prof::begin(st);
  PST_CUDA(launch_k(conv_wgrad_kernel, dim3(grid), dim3(kThreads), smem, st, tX, tD, a));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::CONV_WGRAD, bytes, flops);
}

}  // namespace pst
