// conv_ts.cu -- implicit-GEMM convolution (forward, and dgrad as a stride-1 correlation) with
// the activation operand in TENSOR MEMORY ("TS" tcgen05.mma), 3xTF32 build.
//
// Why (tools/mma_bench.cu, B200): a kind::tf32 M=128 MMA with A read from shared memory costs
// ~39 cycles at N=16/32 regardless of N (the 4 KB A read), ~88 when A starts off a 128-B line;
// with A in TMEM it costs ~14-18 cycles.  ResNet-CIFAR convolutions have N = Cout = 16..64, so
// the contraction is A-bandwidth bound; TS mode removes that bound.
//
// Tile = 128 consecutive output pixels (whole output rows of one image, or whole images).
//   warp 0     TMA producer: the input "band" of a tile (all rows/columns the tile's taps read,
//              one box per channel chunk, zero-filled outside the image) into a smem ring;
//              the layer's weights (all taps, hi and lo planes) once per CTA.
//   warps 6-9  converters: thread = one output pixel = one TMEM lane; per tap it reads the
//              pixel's shifted input channels from the band (16-B loads), splits
//              v = hi + lo (hi = tf32(v) by the tensor core's truncation, lo = v - trunc(v)) and
//              tcgen05.st's both into an A slot (KC + KC columns) of a TMEM ring.
//   warp 1     MMA issuer: per (tap, 8 channels): D += A_hi*W_hi + A_hi*W_lo + A_lo*W_hi.
//   warps 2-5  epilogue (BN statistics / bias+ReLU / dgrad residual), double-buffered D.
//
// Two experiment forms of the same kernel (template flags, built only with -DPST_EXPERIMENTS;
// both parity-green on the GPU and measured slower):
//   SS   A straight from shared memory: three dense column-shifted band copies (dx = -1, 0, +1, zero
//        fill from the TMA at the image edges) make every tap a row shift of one of them, i.e. a UMMA
//        descriptor start offset; 4 warps write the lo planes once per band (no per-tap conversion).
//        The MMAs then read 4 KB of A per instruction from shared memory (~40 cycles each at N <= 64).
//   PRE  the BatchNorm step producing this conv's input (forward BN apply, or this layer's BN backward
//        in the dgrad) done on the band in shared memory by 4 extra warps, replacing the bn_apply /
//        bn_bwd_apply kernels.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.h"
#include "kernels.h"
#include "ptx.cuh"

namespace pst {

// Experiment switches inside the kernels (PST_TS_KNOB) and timeline probes exist only in
// -DPST_EXPERIMENTS builds; in the production library they are compile-time zero.
#ifdef PST_EXPERIMENTS
#define KNOB(x) (a.knob & (x))
#else
#define KNOB(x) 0
#endif

#if PST_SPLIT
namespace {

#ifndef PST_TS_SETS
#define PST_TS_SETS 2
#endif
constexpr int kTsSets = PST_TS_SETS;               // converter sets (4 warps each) taking groups in turn
constexpr int kTsThreads = (6 + 4 * kTsSets) * 32;  // warps: 0 TMA, 1 MMA, 2-5 epilogue, 6.. converters
constexpr int kMaxBand = 4;
constexpr int kMaxSlots = 16;
constexpr int kMaxAcc = 4;      // accumulator buffers (MMA runs up to kMaxAcc-1 tiles ahead of the epilogue)
constexpr int kCoefBytes = 5 * 256 * 4;   // band pre-pass coefficients (Cinp <= 256)

struct TsArgs {
  int N, Ho, Wo, Cinp, Coutp, Cout, BN, n_ntiles, n_mtiles, tpi;
  int k, taps, S;
  int n_kc;                  // channel chunks of KC
  int rows_t, nb, Hb, Wb;    // output rows per tile (per image), images per tile, band rows/cols
  int lo;                    // lowest tap offset (both dims)
  int band_stages, n_slots;
  int tps;                   // taps per TMEM A slot (one handshake)
  int n_acc;                 // accumulator buffers in TMEM (2..kMaxAcc)
  int w3d;                   // weight tensor map form (3D long rows when BN*EPC <= 256)
  int stack;                 // N-stacked weights: per plane [hi rows | lo rows], one N = 2 BN MMA
                             // computes A_hi*W_hi and A_hi*W_lo, a second (N = BN) A_lo*W_hi
  int accw;                  // TMEM columns per accumulator buffer (2 BN stacked, else BN)
  uint32_t band_bytes, band_tx, plane_bytes, w_bytes;
  int tapshift[49];          // band rows (16 B) between the tile origin and tap t's input
  int epi, relu;
  void* out;
  const float* bias;
  double* stats;
  const act_t* res;
  int res_mode, res_H, res_W, res_C, res_pad;
  unsigned long long* dbg;   // optional timeline (CTA 0), PST_DBG_TL
  int knob;                  // experiment switches (PST_TS_KNOB), 0 in production
  const act_t* bz; const act_t* by; const float* bsaved; double* bsums;   // fused bwd_pre (EPI_DGRAD)
  int bfuse, brelu, bbn;
  float bscale;
  // band pre-pass (ConvSpec.pre): the BatchNorm step producing this conv's input, done on the band
  int pre, pre_relu, pre_C, pre2;   // pre2: a second tensor (shortcut / BN input y) rides in the band
  int Hin, Win;                     // input tensor rows / columns (zero padding outside)
  uint32_t band2_off;               // byte offset of the second tensor inside a band stage
  int ss;                           // SS form: three dense dx-bands (raw + lo each) per stage, A read from smem
  uint32_t ss_band;                 // SS: bytes of one dx-band (raw or lo), 1024-aligned
  const double* pre_stats; const float* pre_gamma; const float* pre_beta; float* pre_saved;
  float* pre_run_mean; float* pre_run_var; float pre_momentum, pre_eps;
  act_t* pre_out;
};

__device__ __forceinline__ unsigned long long ts_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));   // SM cycles (globaltimer reads are slow)
  return t;
}
#ifdef PST_EXPERIMENTS
#define TSL(ev, i)                                                   \
  do {                                                               \
    if (a.dbg != nullptr && blockIdx.x == 0) { const int i_ = (i); if (i_ < 256) a.dbg[(ev) * 256 + i_] = ts_gtime(); } \
  } while (0)
#else
#define TSL(ev, i) do { } while (0)
#endif

__device__ __forceinline__ float ld_planar_f(const act_t* base, int64_t npix, int64_t pix, int c) {
  return act2f(base[((int64_t)(c / kEPC) * npix + pix) * kEPC + c % kEPC]);
}

// Per-channel sums over a warp's 32 pixels of 16 channels (u, v per lane): reduce-scatter leaves
// channel (lane >> 1) in lanes 2c, 2c+1; the even lane adds both sums into its fp64 slots w2.
__device__ __forceinline__ void warp_chan_sums(float* s1, float* s2, int lane, double* w2) {
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {       // 16 -> 8 -> 4 -> 2 -> 1 values per lane
    const bool up = (lane & (2 * w)) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float t1 = up ? s1[i] : s1[i + w], k1 = up ? s1[i + w] : s1[i];
      const float t2 = up ? s2[i] : s2[i + w], k2 = up ? s2[i + w] : s2[i];
      s1[i] = k1 + __shfl_xor_sync(0xffffffffu, t1, 2 * w);
      s2[i] = k2 + __shfl_xor_sync(0xffffffffu, t2, 2 * w);
    }
  }
  s1[0] += __shfl_xor_sync(0xffffffffu, s1[0], 1);
  s2[0] += __shfl_xor_sync(0xffffffffu, s2[0], 1);
  if ((lane & 1) == 0) {
    w2[0] += (double)s1[0];
    w2[1] += (double)s2[0];
  }
}

// Per-channel coefficients of the band pre-pass (5 arrays of Cinp floats in shared memory):
//   pre 1: [0] scale = gamma*invstd, [1] shift = beta - mean*gamma*invstd (as bn_apply_kernel);
//          CTA 0 writes (mean, invstd) to pre_saved and updates the running statistics
//   pre 2: [0] k1 = gamma*invstd, [1] m1 = S1/M, [2] m2 = S2/M, [3] mean, [4] invstd (as bn_bwd_apply_kernel)
__device__ __forceinline__ void pre_coefficients(const TsArgs& a, float* coef, int tid, int nthr) {
  const double M = (double)a.N * a.Hin * a.Win;
  for (int c = tid; c < a.Cinp; c += nthr) {
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f, v4 = 0.f;
    if (c < a.pre_C) {
      if (a.pre == 1) {
        const double mean = a.pre_stats[2 * c] / M;
        double var = a.pre_stats[2 * c + 1] / M - mean * mean;
        var = var < 0.0 ? 0.0 : var;
        const float invstd = (float)(1.0 / sqrt(var + (double)a.pre_eps));
        const float g = a.pre_gamma[c], b = a.pre_beta[c];
        v0 = g * invstd;
        v1 = b - (float)mean * g * invstd;
        if (blockIdx.x == 0) {
          a.pre_saved[2 * c] = (float)mean;
          a.pre_saved[2 * c + 1] = invstd;
          a.pre_run_mean[c] = (1.f - a.pre_momentum) * a.pre_run_mean[c] + a.pre_momentum * (float)mean;
          a.pre_run_var[c] = (1.f - a.pre_momentum) * a.pre_run_var[c] + a.pre_momentum * (float)(var * M / (M - 1.0));
        }
      } else {
        v3 = a.pre_saved[2 * c];
        v4 = a.pre_saved[2 * c + 1];
        v0 = a.pre_gamma[c] * v4;
        v1 = (float)(a.pre_stats[2 * c] / M);
        v2 = (float)(a.pre_stats[2 * c + 1] / M);
      }
    }
    coef[c] = v0; coef[a.Cinp + c] = v1; coef[2 * a.Cinp + c] = v2; coef[3 * a.Cinp + c] = v3; coef[4 * a.Cinp + c] = v4;
  }
}

// The pre-pass over one band stage (KC channels from channel kc0) by the 128 pre-pass threads:
// transform in place, zero outside the image, write the tile's own input rows to pre_out.
// Thread layout: planes split the threads evenly (np = KC/4 planes, 128/np threads each), a thread
// walks the band positions q, q + tpp, ... of its plane with the plane's 4 channel coefficients in
// registers and its (image, row, column) advanced incrementally; 4 positions per round (loads first).
template <int KC>
__device__ __forceinline__ void pre_pass(const TsArgs& a, const float* coef, uint8_t* band, int kc0, int n0, int y0,
                                         int nt, int tid) {
  constexpr int NP = KC / kEPC, TPP = 128 / NP;
  const int pl = tid / TPP, q = tid - pl * TPP;
  const int ppl = a.nb * a.Hb * a.Wb;
  const bool last = a.nb > 1 || y0 + a.rows_t >= a.Ho;
  const int own_lo = a.nb > 1 ? 0 : y0 * a.S, own_hi = last ? a.Hin : (y0 + a.rows_t) * a.S;
  const int64_t npix_in = (int64_t)a.N * a.Hin * a.Win;
  const int ybase = y0 * a.S + a.lo;
  const int c = kc0 + 4 * pl;
  float k0[4], k1[4], k2[4], k3[4], k4[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    k0[e] = coef[c + e]; k1[e] = coef[a.Cinp + c + e];
    k2[e] = coef[2 * a.Cinp + c + e]; k3[e] = coef[3 * a.Cinp + c + e]; k4[e] = coef[4 * a.Cinp + c + e];
    if (a.pre == 1) k2[e] = (c + e < a.pre_C) ? 1.f : 0.f;   // shortcut mask of padded channels
  }
  uint8_t* pb = band + (size_t)pl * a.plane_bytes;
  float* dst = reinterpret_cast<float*>(a.pre_out) + (int64_t)(c / 4) * npix_in * 4;   // act_t == float here
  int col = q % a.Wb, rr = q / a.Wb;
  int j = rr / a.Hb, row = rr - j * a.Hb;
  for (int p0 = q; p0 < ppl; p0 += 4 * TPP) {
    int off[4], gidx[4];
    bool val[4], own[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * TPP;
      const int xin = a.lo + col, yin = ybase + row, n = n0 + j;
      val[u] = p < ppl && xin >= 0 && xin < a.Win && yin >= 0 && yin < a.Hin && n < a.N;
      own[u] = val[u] && nt == 0 && yin >= own_lo && yin < own_hi;
      off[u] = p < ppl ? p * 16 : 0;
      gidx[u] = ((n * a.Hin + yin) * a.Win + xin) * 4;
      col += TPP;
      while (col >= a.Wb) { col -= a.Wb; if (++row == a.Hb) { row = 0; ++j; } }
    }
    float4 v[4], r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = *reinterpret_cast<const float4*>(pb + off[u]);
      r[u] = a.pre2 ? *reinterpret_cast<const float4*>(pb + a.band2_off + off[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float o[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
      const float rr4[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (a.pre == 1) {   // as bn_apply_kernel: y*scale + shift + shortcut, then ReLU
          o[e] = o[e] * k0[e] + k1[e] + rr4[e] * k2[e];
          if (a.pre_relu) o[e] = fmaxf(o[e], 0.f);
        } else {            // as bn_bwd_apply_kernel
          const float xh = (rr4[e] - k3[e]) * k4[e];
          o[e] = k0[e] * (o[e] - k1[e] - xh * k2[e]);
        }
      }
      const float4 w = val[u] ? make_float4(o[0], o[1], o[2], o[3]) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (p0 + u * TPP < ppl) *reinterpret_cast<float4*>(pb + off[u]) = w;
      if (own[u]) *reinterpret_cast<float4*>(dst + gidx[u]) = w;
    }
  }
}

template <int KC, int EPI, int TPS, int PRE, int SS>
__global__ void __launch_bounds__(kTsThreads + PRE * 128, 1)
    conv_ts_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ TsArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // [weights hi | weights lo] [band ring] [stats scratch 4 x 32 x 17 f32] [barriers] [tmem ptr]
  uint8_t* wsm = smem;
  uint8_t* bands = smem + 2 * a.w_bytes;
  float* sst = reinterpret_cast<float*>(bands + a.band_stages * a.band_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sst + 4 * 32 * 17 + 512);   // + cacc (<= 256 doubles = 512 floats)
  uint64_t* full = bars;
  uint64_t* bempty = full + kMaxBand;
  uint64_t* afull = bempty + kMaxBand;
  uint64_t* aempty = afull + kMaxSlots;
  uint64_t* tfull = aempty + kMaxSlots;
  uint64_t* tempty = tfull + kMaxAcc;
  uint64_t* wbar = tempty + kMaxAcc;
  uint64_t* ready = wbar + 1;                        // band pre-pass done (PRE)
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(ready + kMaxBand);
  int* tsh = reinterpret_cast<int*>(tmem_ptr + 4);   // tap shifts (a.tapshift indexed dynamically
                                                     // from the param space would be copied to local memory)
  float* coef = reinterpret_cast<float*>(tsh + 64);  // band pre-pass coefficients, 5 x Cinp

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TSL(7, 0);
  int dbg_i[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int nt = blockIdx.x % a.n_ntiles;            // a CTA keeps one N tile (resident weights)
  const int m0 = blockIdx.x / a.n_ntiles, mstep = gridDim.x / a.n_ntiles;
  const int planes_w = a.Cinp / kEPC;                // weight planes per tap

  if (warp == 0) {   // lane i initialises the i-th barrier of each ring (the rings have <= 16 entries)
    bool any = false;
    if (lane < a.band_stages) {
      ptx::mbar_init(&full[lane], 1);
      ptx::mbar_init(&bempty[lane], SS ? 1 : 4 * kTsSets);   // SS: released by the MMA commit
      ptx::mbar_init(&ready[lane], 4);
      any = true;
    }
    if (lane < a.n_slots) { ptx::mbar_init(&afull[lane], 4); ptx::mbar_init(&aempty[lane], 1); any = true; }
    if (lane < a.n_acc) { ptx::mbar_init(&tfull[lane], 1); ptx::mbar_init(&tempty[lane], 4); any = true; }
    if (lane == 0) { ptx::mbar_init(wbar, 1); any = true; }
    if (any) ptx::fence_mbar_init();
  }
  if (threadIdx.x == 0) TSL(7, 1);   // barriers initialised
  if (warp == 1) ptx::tmem_alloc(tmem_ptr, 512);
  if (threadIdx.x == 32) TSL(7, 2);  // TMEM allocated
  if (threadIdx.x < 49) tsh[threadIdx.x] = a.tapshift[threadIdx.x];   // __grid_constant__: read in place
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  if (threadIdx.x == 0) TSL(7, 3);   // past the prologue barrier
  // The weight shadows are written only by the update kernels (sgd_kernel, build_shadows), which do
  // not release their dependents early (common.h pdl_trigger), and at least one kernel separates
  // them from any conv; so the layer's weights load before pdl_wait, overlapping the previous
  // kernel's tail.  Everything else this kernel reads comes after pdl_wait.
  if (warp == 0 && ptx::elect_one() && !KNOB(16)) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmW);
    if (a.pre2) ptx::prefetch_tmap(&tmB);
    ptx::mbar_expect_tx(wbar, 2 * a.w_bytes);
    if (a.stack) {  // (BN*EPC, hi/lo, planes, taps) -> smem [tap][plane][hi BN rows | lo BN rows]
      ptx::tma_load_4d(wsm, &tmW, wbar, nt * a.BN * kEPC, 0, 0, 0);
    } else if (a.w3d) {   // long rows: (BN*EPC, planes, taps)
      ptx::tma_load_3d(wsm, &tmW, wbar, nt * a.BN * kEPC, 0, 0);                 // hi: taps [0, taps)
      ptx::tma_load_3d(wsm + a.w_bytes, &tmW, wbar, nt * a.BN * kEPC, 0, a.taps);  // lo: taps [taps, 2 taps)
    } else {
      ptx::tma_load_4d(wsm, &tmW, wbar, 0, nt * a.BN, 0, 0);
      ptx::tma_load_4d(wsm + a.w_bytes, &tmW, wbar, 0, nt * a.BN, 0, a.taps);
    }
  }
  __syncwarp();
  pdl_wait();      // no activation / statistics access above this line
  pdl_trigger();
  if (threadIdx.x == 0) TSL(7, 4);   // past griddepcontrol.wait
  const uint32_t a_col0 = a.n_acc * a.accw;          // accumulators: columns [0, n_acc accw)
  // band stage bs <- tile m, channel chunk kcc (elected producer lane)
  auto issue_band = [&](int bs, int m, int kcc) {
    const int n0 = a.nb > 1 ? m * a.nb : m / a.tpi;
    const int y0 = a.nb > 1 ? 0 : (m % a.tpi) * a.rows_t;
    if (KNOB(32)) { ptx::mbar_arrive(&full[bs]); return; }
    if (SS) {   // three dense column-shifted bands (dx = lo .. lo+2), zero-filled outside the image
      ptx::mbar_expect_tx(&full[bs], 3 * a.band_tx);
#pragma unroll
      for (int bx = 0; bx < 3; ++bx)
        ptx::tma_load_4d(bands + bs * a.band_bytes + bx * 2 * a.ss_band, &tmA, &full[bs], (a.lo + bx) * kEPC,
                         y0 + a.lo, n0, kcc * (KC / kEPC));
      return;
    }
    ptx::mbar_expect_tx(&full[bs], a.pre2 ? 2 * a.band_tx : a.band_tx);
    ptx::tma_load_4d(bands + bs * a.band_bytes, &tmA, &full[bs], a.lo * kEPC, y0 * a.S + a.lo, n0, kcc * (KC / kEPC));
    if (a.pre2)
      ptx::tma_load_4d(bands + bs * a.band_bytes + a.band2_off, &tmB, &full[bs], a.lo * kEPC, y0 * a.S + a.lo, n0,
                       kcc * (KC / kEPC));
  };
  // the first band right after the dependency wait, before the role dispatch (the producer loop's
  // code is cold at this point: issuing from here saves ~1 kcycle of the first tile's latency)
#ifndef PST_NO_EARLY_BAND
  if (warp == 0 && m0 < a.n_mtiles && !KNOB(16) && ptx::elect_one()) issue_band(0, m0, 0);
#endif
  __syncwarp();

  if (KNOB(16)) {
    // experiment: prologue and teardown only
  } else if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    __syncwarp();
    int bs = 0;
    uint32_t bph = 0;
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        ptx::mbar_wait(&bempty[bs], bph ^ 1);
        if (lane == 0) TSL(0, dbg_i[0]++);
#ifndef PST_NO_EARLY_BAND
        if (!(m == m0 && kcc == 0) && ptx::elect_one()) issue_band(bs, m, kcc);   // the first: in the prologue
#else
        if (ptx::elect_one()) issue_band(bs, m, kcc);
#endif
        __syncwarp();
        if (++bs == a.band_stages) { bs = 0; bph ^= 1; }
      }
    }
  } else if (SS && warp == 1) {
    // ---------------------------------------------------------------- MMA issuer, SS form
    // per (tap, 8 channels): D += A_raw*[W_hi|W_lo] (N = 2 BN; the tensor core reads the raw fp32
    // band as tf32 by truncation) and A_lo*W_hi (N = BN); A = the tap's band rows straight from
    // shared memory: the dx-band of the tap's column offset, started (oy - lo) image rows in.
    const uint32_t idesc = ptx::idesc_mma(128, a.BN, 0, 0, 2);
    const uint32_t idesc2 = ptx::idesc_mma(128, 2 * a.BN, 0, 0, 2);
    const uint32_t pl2 = 2u * a.BN * 16;                      // stacked weights: bytes per plane (hi + lo rows)
    const uint64_t wdesc2 = ptx::smem_desc(ptx::smem_u32(wsm), pl2, 128);
    const uint64_t adesc = ptx::smem_desc(ptx::smem_u32(bands), a.plane_bytes, 128);   // K-major, rows 16 B apart
    ptx::mbar_wait(wbar, 0);
    int bs = 0;
    uint32_t bph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      ptx::mbar_wait(&tempty[acc], aph ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem + acc * a.accw;
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        ptx::mbar_wait(&ready[bs], bph);   // band landed and its lo planes written
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint64_t ab = ptx::desc_add(adesc, bs * a.band_bytes);
#pragma unroll
          for (int t = 0; t < 9; ++t) {
            const uint64_t at = ptx::desc_add(ab, (uint32_t)a.tapshift[t]);
            const uint64_t bt = ptx::desc_add(wdesc2, t * planes_w * pl2 + kcc * (KC / kEPC) * pl2);
#pragma unroll
            for (int kk = 0; kk < KC / 8; ++kk) {
              const uint64_t ad = ptx::desc_add(at, 2 * kk * a.plane_bytes);
              const uint64_t bd = ptx::desc_add(bt, 2 * kk * pl2);
              ptx::umma_tf32(d, ad, bd, idesc2, (kcc | t | kk) ? 1u : 0u);          // raw*[hi | lo]
              ptx::umma_tf32(d, ptx::desc_add(ad, a.ss_band), bd, idesc, 1u);      // lo*hi
            }
          }
          ptx::umma_commit(&bempty[bs]);   // band stage free once these MMAs have read it
        }
        __syncwarp();
        if (++bs == a.band_stages) { bs = 0; bph ^= 1; }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == a.n_acc) { acc = 0; aph ^= 1; }
    }
  } else if (SS && warp >= 6) {
    // ---------------------------------------------------------------- lo planes (SS; warps 6-9)
    // lo = v - trunc_tf32(v) of the three raw bands, written beside them; one pass per band stage
    if (warp < 10) {
      const int tid = threadIdx.x - 6 * 32;
      const int nvec = (int)(a.band_tx / 16);
      int bs = 0;
      uint32_t bph = 0;
      for (int m = m0; m < a.n_mtiles; m += mstep) {
        for (int kcc = 0; kcc < a.n_kc; ++kcc) {
          ptx::mbar_wait(&full[bs], bph);
          uint8_t* band = bands + bs * a.band_bytes;
#pragma unroll 1
          for (int bx = 0; bx < 3 && !KNOB(8192); ++bx) {
            const float4* src = reinterpret_cast<const float4*>(band + bx * 2 * a.ss_band);
            float4* dst = reinterpret_cast<float4*>(band + bx * 2 * a.ss_band + a.ss_band);
#pragma unroll 4
            for (int i = tid; i < nvec; i += 128) {
              const float4 v = src[i];
              dst[i] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
            }
          }
          ptx::fence_proxy_async_smem();   // generic writes read by tcgen05.mma (async proxy)
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&ready[bs]);
          if (++bs == a.band_stages) { bs = 0; bph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = ptx::idesc_mma(128, a.BN, 0, 0, 2);
    const uint32_t idesc2 = ptx::idesc_mma(128, 2 * a.BN, 0, 0, 2);
    const uint32_t wtap = (uint32_t)planes_w * a.BN * 16;     // weight bytes per tap (hi)
    const uint64_t wdesc = ptx::smem_desc(ptx::smem_u32(wsm), a.BN * 16, 128);
    const uint32_t pl2 = 2u * a.BN * 16;                      // stacked: bytes per plane (hi + lo rows)
    const uint64_t wdesc2 = ptx::smem_desc(ptx::smem_u32(wsm), pl2, 128);
    ptx::mbar_wait(wbar, 0);
    int slot = 0;
    uint32_t sph = 0;
    int acc = 0;
    uint32_t aph = 0;
    const int ngrp = a.taps / TPS;
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      ptx::mbar_wait(&tempty[acc], aph ^ 1);
      if (!KNOB(256)) ptx::tc_fence_after();
      const uint32_t d = tmem + acc * a.accw;
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        for (int gi = 0; gi < ngrp; ++gi) {
          ptx::mbar_wait(&afull[slot], sph);
          if (!KNOB(256)) ptx::tc_fence_after();
          if (lane == 0) TSL(4, dbg_i[4]++);
          if (ptx::elect_one()) {
            if (!KNOB(2) && a.stack) {
#pragma unroll
            for (int i = 0; i < TPS; ++i) {
              const int t = gi * TPS + i;
              const uint32_t ahi = tmem + a_col0 + (slot * TPS + i) * 2 * KC;
              const uint64_t bt = ptx::desc_add(wdesc2, t * planes_w * pl2 + kcc * (KC / kEPC) * pl2);
#pragma unroll
              for (int kk = 0; kk < KC / 8; ++kk) {
                const uint64_t bd = ptx::desc_add(bt, 2 * kk * pl2);
                ptx::umma_tf32_ts(d, ahi + kk * 8, bd, idesc2, (kcc | t | kk) ? 1u : 0u);   // [hi*hi | hi*lo]
                ptx::umma_tf32_ts(d, ahi + KC + kk * 8, bd, idesc, 1u);                    // lo*hi
              }
            }
            } else if (!KNOB(2)) {
            // one slot = tps taps x (KC hi + KC lo columns): 3 x KC/8 x tps MMAs per handshake
            // compile-time trip counts: the elected lane's block is straight-line code (a runtime
            // loop here costs an R2UR round trip per tcgen05.mma, ~4x the small-N MMA time)
#pragma unroll
            for (int i = 0; i < TPS; ++i) {
              const int t = gi * TPS + i;
              const uint32_t ahi = tmem + a_col0 + (slot * TPS + i) * 2 * KC;
              const uint64_t bt = ptx::desc_add(wdesc, t * wtap + kcc * (KC / kEPC) * (a.BN * 16));
#pragma unroll
              for (int kk = 0; kk < KC / 8; ++kk) {
                const uint64_t bd = ptx::desc_add(bt, 2 * kk * (a.BN * 16));
                const uint64_t bdl = ptx::desc_add(bd, a.w_bytes);
                ptx::umma_tf32_ts(d, ahi + kk * 8, bd, idesc, (kcc | t | kk) ? 1u : 0u);
                ptx::umma_tf32_ts(d, ahi + kk * 8, bdl, idesc, 1u);
                ptx::umma_tf32_ts(d, ahi + KC + kk * 8, bd, idesc, 1u);
              }
            }
            }
            ptx::umma_commit(&aempty[slot]);
          }
          __syncwarp();
          if (lane == 0) TSL(2, dbg_i[2]++);
          if (++slot == a.n_slots) { slot = 0; sph ^= 1; }
        }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == a.n_acc) { acc = 0; aph ^= 1; }
    }
  } else if (PRE && warp >= 6 + 4 * kTsSets) {
    // ---------------------------------------------------------------- band pre-pass (4 warps)
    // BN apply / BN backward on each band stage after its TMA load, one stage ahead of the converters
    pre_coefficients(a, coef, threadIdx.x - (6 + 4 * kTsSets) * 32, 128);
    ptx::named_bar_sync(2, 128);
    int bs = 0;
    uint32_t bph = 0;
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      const int n0 = a.nb > 1 ? m * a.nb : m / a.tpi;
      const int y0 = a.nb > 1 ? 0 : (m % a.tpi) * a.rows_t;
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        ptx::mbar_wait(&full[bs], bph);
        if (!KNOB(8192))
          pre_pass<KC>(a, coef, bands + bs * a.band_bytes, kcc * KC, n0, y0, KNOB(4096) ? 1 : nt,
                       threadIdx.x - (6 + 4 * kTsSets) * 32);
        if (!KNOB(2048)) ptx::fence_proxy_async_smem();   // generic writes to a buffer the TMA refills later
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ready[bs]);
        if (++bs == a.band_stages) { bs = 0; bph ^= 1; }
      }
    }
  } else if (warp >= 6) {
    // ---------------------------------------------------------------- converters (warps 6..)
    // kTsSets sets of 4 warps (one warp per TMEM lane quarter each) take the tap groups of the
    // global sequence in turn (several groups in flight hide the tcgen05.st -> wait::st latency).  Per group: for each of its tps taps, load the pixel's shifted input
    // channels from the band, split hi/lo, tcgen05.st both (no wait); one wait + one arrive
    // per group, so loads and stores of consecutive taps overlap.
    const int q = warp & 3;                  // TMEM lane quarter of this warp
    const int set = (warp - 6) >> 2;
    const int r = q * 32 + lane;             // tile pixel = TMEM lane
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int per_img = a.rows_t * a.Wo;
    const int j = r / per_img, yy = (r / a.Wo) % a.rows_t, xx = r % a.Wo;
    const int pixoff = (j * a.Hb + yy * a.S) * a.Wb + xx * a.S;
    const int ngrp = a.taps / TPS;
    int bs = 0;
    uint32_t bph = 0;
    int turn = 0;                            // set owning the next group (same order as the MMA issuer)
    int slot = 0;                            // slot / phase of group cnt (advanced for every group)
    uint32_t sph = 0;
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        ptx::mbar_wait(PRE ? &ready[bs] : &full[bs], bph);
        const uint8_t* band = bands + bs * a.band_bytes;
        for (int gi = 0; gi < ngrp; ++gi) {
          const int my_slot = slot;
          const uint32_t my_ph = sph;
          if (++slot == a.n_slots) { slot = 0; sph ^= 1; }
          const bool mine = turn == set;
          if (++turn == kTsSets) turn = 0;
          if (!mine) continue;                               // another set's group
          ptx::mbar_wait(&aempty[my_slot], my_ph ^ 1);
          if (!KNOB(256)) ptx::tc_fence_after();
          if (threadIdx.x == 192) TSL(1, dbg_i[1]++);
#pragma unroll 1
          for (int i = 0; i < TPS && !KNOB(1); ++i) {
            const int t = gi * TPS + i;
            const uint8_t* src = band + (uint32_t)(pixoff + tsh[t]) * 16;
            float hi[KC], lo[KC];
#pragma unroll
            for (int p4 = 0; p4 < KC / 4; ++p4) {
              const float4 v = *reinterpret_cast<const float4*>(src + p4 * a.plane_bytes);
              hi[4 * p4 + 0] = v.x; hi[4 * p4 + 1] = v.y; hi[4 * p4 + 2] = v.z; hi[4 * p4 + 3] = v.w;
            }
#pragma unroll
            for (int e = 0; e < KC; ++e) lo[e] = tf32_lo(hi[e]);
            const uint32_t ta = tmem + lane_addr + a_col0 + (my_slot * TPS + i) * 2 * KC;
#pragma unroll
            for (int h = 0; h < KC / 16; ++h) {
              ptx::tmem_st16(ta + h * 16, hi + 16 * h);
              ptx::tmem_st16(ta + KC + h * 16, lo + 16 * h);
            }
          }
          if (KNOB(1024) && threadIdx.x == 192) TSL(5, dbg_i[5]++);   // timeline: stores issued
          if (!KNOB(512)) ptx::tmem_st_wait();
          if (KNOB(1024) && threadIdx.x == 192) TSL(6, dbg_i[6]++);   // timeline: stores complete
          if (!KNOB(256)) ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&afull[my_slot]);
          if (threadIdx.x == 192) TSL(3, dbg_i[3]++);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&bempty[bs]);
        if (++bs == a.band_stages) { bs = 0; bph ^= 1; }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    // BN statistics: per 16-channel group a warp reduce-scatter leaves the sum over the warp's
    // 32 pixels of channel (lane >> 1) in lanes lane, lane^1; the even lane accumulates it into
    // the warp's fp64 slot in shared memory; the four warps' slots are combined at the end and
    // written with one global atomic per channel.
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const int et = threadIdx.x - 64;         // 0..127
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    double* wacc = reinterpret_cast<double*>(sst);   // [4 warps][BN][2]  (<= 8 KB)
    const bool sums = EPI == EPI_BN_STATS || (EPI == EPI_DGRAD && a.bfuse);
    if (sums) {
      for (int i = lane; i < 2 * a.BN; i += 32) wacc[q * 2 * a.BN + i] = 0.0;
      __syncwarp();
    }
    const int per_img = a.rows_t * a.Wo;
    const int64_t npix = (int64_t)a.N * a.Ho * a.Wo;
    const int ng = a.BN / 16;
    // this thread's pixel inside a tile (fixed), and the tile origin advanced incrementally
    const int jt = r / per_img, yt = (r / a.Wo) % a.rows_t, x = r % a.Wo;
    int mq = a.nb > 1 ? m0 : m0 / a.tpi, mr = a.nb > 1 ? 0 : m0 % a.tpi;
    const int sq = a.nb > 1 ? mstep : mstep / a.tpi, sr = a.nb > 1 ? 0 : mstep % a.tpi;
    int acc = 0;
    uint32_t aph = 0;
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      const int n = (a.nb > 1 ? mq * a.nb : mq) + jt;
      const int y = mr * a.rows_t + yt;
      mq += sq; mr += sr;
      if (mr >= a.tpi && a.nb == 1) { mr -= a.tpi; ++mq; }
      const bool valid = n < a.N;
      const int64_t pix = ((int64_t)n * a.Ho + y) * a.Wo + x;
      for (int g = 0; g < ng; ++g) {
        // dgrad: the group's global operands (residual gradient, the lower layer's z and y) are
        // loaded first -- for g == 0 before waiting for the accumulator -- so their latency
        // overlaps the MMAs instead of stalling the epilogue three times per group
        float4 rv[4], zv[4], yv[4];
        if (EPI == EPI_DGRAD) {
          const int cq0 = (nt * a.BN + g * 16) / 4;
          const bool r1 = valid && a.res_mode == 1;
          const bool zr = valid && a.bfuse && a.brelu;
          const bool yb = valid && a.bfuse && a.bbn;
          const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int64_t off = ((int64_t)(cq0 + jj) * npix + pix) * 4;
            rv[jj] = r1 ? __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.res) + off)) : z4;
            zv[jj] = zr ? __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.bz) + off)) : z4;
            yv[jj] = yb ? __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(a.by) + off)) : z4;
          }
        }
        if (g == 0) {
          ptx::mbar_wait(&tfull[acc], aph);
          if (!KNOB(256)) ptx::tc_fence_after();
          if (threadIdx.x == 64 && !KNOB(1024)) TSL(5, dbg_i[5]++);
        }
        float u[16];
        if (KNOB(64)) {
#pragma unroll
          for (int i = 0; i < 16; ++i) u[i] = 0.f;
        } else {
          ptx::tmem_ld16(tmem + lane_addr + acc * a.accw + g * 16, u);
          if (a.stack) {                   // + the A_hi*W_lo half
            float u2[16];
            ptx::tmem_ld16(tmem + lane_addr + acc * a.accw + a.BN + g * 16, u2);
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] += u2[i];
          }
        }
        if (g == ng - 1) {
          if (!KNOB(256)) ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
          if (++acc == a.n_acc) { acc = 0; aph ^= 1; }
        }
        const int c0 = nt * a.BN + g * 16;
        if (EPI == EPI_BN_STATS) {
          if (!valid) {
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] = 0.f;
          }
        } else if (EPI == EPI_DGRAD) {   // + shortcut^T of the residual layer's gradient
          if (valid && a.res_mode == 1) {   // act_t == float in this build
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const float4 v = rv[jj];
              u[4 * jj] += v.x; u[4 * jj + 1] += v.y; u[4 * jj + 2] += v.z; u[4 * jj + 3] += v.w;
            }
          } else if (valid && a.res_mode == 2 && ((y | x) & 1) == 0) {
            const int64_t rpix = ((int64_t)n * a.res_H + (y >> 1)) * a.res_W + (x >> 1);
            const int64_t rnpix = (int64_t)a.N * a.res_H * a.res_W;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int c = c0 + i;
              if (c < a.Cout) u[i] += ld_planar_f(a.res, rnpix, rpix, c + a.res_pad);
            }
          }
          if (a.bfuse) {                   // fused bwd_pre: relu'(z) of the lower layer; zero padding pixels
            if (!valid) {
#pragma unroll
              for (int i = 0; i < 16; ++i) u[i] = 0.f;
            } else if (a.brelu) {
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                u[4 * jj] = zv[jj].x > 0.f ? u[4 * jj] * a.bscale : 0.f;
                u[4 * jj + 1] = zv[jj].y > 0.f ? u[4 * jj + 1] * a.bscale : 0.f;
                u[4 * jj + 2] = zv[jj].z > 0.f ? u[4 * jj + 2] * a.bscale : 0.f;
                u[4 * jj + 3] = zv[jj].w > 0.f ? u[4 * jj + 3] * a.bscale : 0.f;
              }
            }
          }
        } else {                           // EPI_BIAS_ACT / EPI_BIAS_F32
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = c0 + i;
            const float b = (a.bias != nullptr && c < a.Cout) ? __ldg(&a.bias[c]) : 0.f;
            float o = u[i] + b;
            if (a.relu) o = fmaxf(o, 0.f);
            u[i] = (c < a.Cout) ? o : 0.f;
          }
        }
        if (valid && !KNOB(8)) {
          float* o = reinterpret_cast<float*>(a.out);   // act_t == float in this build
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            *reinterpret_cast<float4*>(o + ((int64_t)(c0 / 4 + jj) * npix + pix) * 4) =
                make_float4(u[4 * jj], u[4 * jj + 1], u[4 * jj + 2], u[4 * jj + 3]);
        }
        if (EPI == EPI_BN_STATS && !KNOB(4)) {
          float s1[16], s2[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) { s1[i] = u[i]; s2[i] = u[i] * u[i]; }
          warp_chan_sums(s1, s2, lane, wacc + q * 2 * a.BN + 2 * (g * 16 + (lane >> 1)));
        }
        if (EPI == EPI_DGRAD && a.bfuse) {   // sums of the fused bwd_pre (u is the stored gpre)
          float s1[16], s2[16];
          if (a.bbn && valid) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const float yy[4] = {yv[jj].x, yv[jj].y, yv[jj].z, yv[jj].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = c0 + 4 * jj + e;
                const float xh = (yy[e] - __ldg(&a.bsaved[2 * c])) * __ldg(&a.bsaved[2 * c + 1]);
                s1[4 * jj + e] = u[4 * jj + e];
                s2[4 * jj + e] = u[4 * jj + e] * xh;
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) { s1[i] = u[i]; s2[i] = 0.f; }
          }
          warp_chan_sums(s1, s2, lane, wacc + q * 2 * a.BN + 2 * (g * 16 + (lane >> 1)));
        }
      }
      if (threadIdx.x == 64 && !KNOB(1024)) TSL(6, dbg_i[6]++);
    }
    if (sums) {
      double* dst = EPI == EPI_BN_STATS ? a.stats : a.bsums;
      const int nreal = EPI == EPI_BN_STATS ? 2 * a.BN : 2 * min(a.BN, a.Cout - nt * a.BN);
      ptx::named_bar_sync(1, 128);
      for (int i = et; i < nreal; i += 128) {
        const double v = wacc[i] + wacc[2 * a.BN + i] + wacc[4 * a.BN + i] + wacc[6 * a.BN + i];
        if (v != 0.0) atomicAdd(&dst[2 * nt * a.BN + i], v);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

// Plans the TS kernel for this convolution; false if the shape does not fit its tiling.
static bool ts_plan_kc(const ConvSpec& c, TsArgs& a, int kc, bool ss);
// SS form (A read from shared memory; kernel comment): stride-1 3x3 convolutions whose tile is whole
// rows of one image, no band pre-pass
static bool ss_eligible(const ConvSpec& c) {
#ifndef PST_EXPERIMENTS
  (void)c;
  return false;   // measured slower than the TS form; experiment builds only
#endif
  static const bool on = pst_knob("PST_SS", 0) != 0;
  const int per_img = c.Ho * c.Wo;
  return on && c.S == 1 && c.k == 3 && c.pre == 0 && c.H == c.Ho && c.W == c.Wo && per_img >= 128 &&
         c.Wo * kEPC <= 256;
}
static bool ts_plan(const ConvSpec& c, TsArgs& a, int& kc) {
  // 32-channel band chunks where they divide Cinp; 16 if the stage would not fit twice at 32
  for (bool ss : {true, false}) {
    if (ss && !ss_eligible(c)) continue;
    static const bool kc8 = pst_knob("PST_SS_KC8", 0) != 0;
    if (ss && kc8 && ts_plan_kc(c, a, 8, ss)) { kc = 8; return true; }
    if (c.Cinp % 32 == 0 && ts_plan_kc(c, a, 32, ss)) { kc = 32; return true; }
    if (ts_plan_kc(c, a, 16, ss)) { kc = 16; return true; }
  }
  return false;
}
static bool ts_plan_kc(const ConvSpec& c, TsArgs& a, int kc, bool ss) {
  if (pst_knob("PST_NOTS", 0)) return false;
  if (c.k > 7 || (c.S != 1 && c.S != 2) || c.Coutp > 256) return false;
  if (c.Wo > 128 || 128 % c.Wo != 0) return false;
  const int per_img = c.Ho * c.Wo;
  if (!(per_img % 128 == 0 || 128 % per_img == 0)) return false;
  a = TsArgs{};
  a.N = c.N; a.Ho = c.Ho; a.Wo = c.Wo; a.Cinp = c.Cinp; a.Coutp = c.Coutp; a.Cout = c.Cout;
  a.k = c.k; a.taps = c.k * c.k; a.S = c.S;
  a.n_kc = c.Cinp / kc;
  if (per_img >= 128) { a.nb = 1; a.rows_t = 128 / c.Wo; a.tpi = c.Ho / a.rows_t; a.n_mtiles = c.N * a.tpi; }
  else { a.nb = 128 / per_img; a.rows_t = c.Ho; a.tpi = 1; a.n_mtiles = ceil_div(c.N, a.nb); }
  a.Hb = (a.rows_t - 1) * c.S + c.k;
  a.Wb = (c.Wo - 1) * c.S + c.k;
  if (a.Wb * kEPC > 256 || a.Hb > 256 || a.nb > 256) return false;
  const int o1 = c.off, o2 = c.off + c.sgn * (c.k - 1);
  a.lo = std::min(o1, o2);
  for (int t = 0; t < a.taps; ++t) {
    const int oy = c.off + c.sgn * (t / c.k), ox = c.off + c.sgn * (t % c.k);
    a.tapshift[t] = (oy - a.lo) * a.Wb + (ox - a.lo);
  }
  a.ss = ss ? 1 : 0;
  a.plane_bytes = (uint32_t)a.nb * a.Hb * (ss ? c.Wo : a.Wb) * 16;
  a.band_tx = a.plane_bytes * (kc / kEPC);
  a.ss_band = (uint32_t)round_up((int)a.band_tx, 1024);
  if (ss)   // tap t: the dx-band of its column offset (raw at bx * 2 ss_band), (oy - lo) rows in
    for (int t = 0; t < a.taps; ++t) {
      const int oy = c.off + c.sgn * (t / c.k), ox = c.off + c.sgn * (t % c.k);
      a.tapshift[t] = (ox - a.lo) * 2 * (int)a.ss_band + (oy - a.lo) * c.Wo * 16;
    }
  a.pre = c.pre;
  a.pre2 = (c.pre == 1 && c.pre_res != nullptr) || c.pre == 2;
  if (c.pre && c.Cinp > 256) return false;
  a.band2_off = (uint32_t)round_up((int)a.band_tx, 1024);
  a.band_bytes = a.pre2 ? (uint32_t)round_up((int)(a.band2_off + a.band_tx), 1024) : a.band2_off;
  if (ss) a.band_bytes = 6 * a.ss_band;   // three dx-bands, raw + lo each
  // N tile: resident hi+lo weights of all taps <= wmax KB (PST_TS_WMAX: planning experiments;
  // 150 lets the 64-channel convs take BN = 32: half the N tiles, each MMA twice as wide)
  static const int wmax = pst_knob("PST_TS_WMAX", 150);
  static const int force_tps = pst_knob("PST_TS_TPS", 0);
  static const int force_nacc = pst_knob("PST_TS_NACC", 0);
  a.BN = 0;
  for (int bn = std::min(c.Coutp, 128); bn >= 16; bn -= 16)
    if (c.Coutp % bn == 0 && 2ll * a.taps * c.Cinp * bn * 4 <= (int64_t)wmax * 1024) { a.BN = bn; break; }
  if (a.BN == 0) return false;
  a.n_ntiles = c.Coutp / a.BN;
  a.w_bytes = (uint32_t)a.taps * c.Cinp * a.BN * 4;
  static const bool stack_on = pst_knob("PST_TS_STACK", 1) != 0;
  a.stack = (stack_on && a.BN * kEPC <= 256) ? 1 : 0;
  a.accw = a.stack ? 2 * a.BN : a.BN;
  const int fixed = 2 * (int)a.w_bytes + 4 * 32 * 17 * 4 + 2048 + (3 * kMaxBand + 2 * kMaxSlots + 2 * kMaxAcc + 1) * 8 + 16 + 256 + kCoefBytes;
  a.band_stages = std::min(kMaxBand, (227 * 1024 - 1024 - fixed) / (int)a.band_bytes);
  if (a.band_stages < 2) return false;
  if (ss) {   // TMEM holds only the accumulators
    if (!a.stack) return false;
    a.tps = 3;
    a.n_acc = std::min(kMaxAcc, 512 / a.accw);
    a.n_slots = 0;
    return a.n_acc >= 2;
  }
  // accumulator buffers: as many as leave >= 3 A slots of the largest group (fall back to 2)
  a.tps = 0;
  a.n_acc = 0;
  // (largest tap group first: every group costs one converter->MMA handshake)
  for (int tps : {3, 2, 1}) {
    if (a.taps % tps != 0 || (force_tps && tps != force_tps)) continue;
    for (int nacc : {4, 3, 2}) {
      if (force_nacc && nacc != force_nacc) continue;
      // a set may reuse a slot only after the group kTsSets earlier completed its own wait on it
      // (mbarrier parity aliasing): n_slots >= kTsSets
      if ((512 - nacc * a.accw) / (2 * kc * tps) >= std::max(nacc > 2 ? 3 : 2, kTsSets)) { a.n_acc = nacc; break; }
    }
    if (a.n_acc) { a.tps = tps; break; }
  }
  if (a.tps == 0) return false;
  a.n_slots = std::min(kMaxSlots, (512 - a.n_acc * a.accw) / (2 * kc * a.tps));
  if (a.n_slots < std::max(2, kTsSets)) return false;
  return true;
}

bool conv_ts_fits(const ConvSpec& c) {
  TsArgs a;
  int kc;
  return ts_plan(c, a, kc);
}

bool conv_ts(const ConvSpec& c, cudaStream_t st) {
  TsArgs a;
  int kc;
  if (!ts_plan(c, a, kc)) return false;
  a.epi = c.epi; a.relu = c.relu; a.out = c.out; a.bias = c.bias; a.stats = c.stats;
  a.res = c.res; a.res_mode = c.res_mode; a.res_H = c.res_H; a.res_W = c.res_W; a.res_C = c.res_C;
  a.res_pad = c.res_pad;
  a.dbg = c.dbg;
  a.bz = c.bz; a.by = c.by; a.bsaved = c.bsaved; a.bsums = c.bsums;
  a.bfuse = c.bfuse; a.brelu = c.brelu; a.bbn = c.bbn;
  a.bscale = c.bscale == 0.f ? 1.f : c.bscale;
  a.pre_relu = c.pre_relu; a.pre_C = c.pre_C; a.Hin = c.H; a.Win = c.W;
  a.pre_stats = c.pre_stats; a.pre_gamma = c.pre_gamma; a.pre_beta = c.pre_beta; a.pre_saved = c.pre_saved;
  a.pre_run_mean = c.pre_run_mean; a.pre_run_var = c.pre_run_var;
  a.pre_momentum = c.pre_momentum; a.pre_eps = c.pre_eps; a.pre_out = c.pre_out;
  PST_CHECK_ARG(!c.pre || c.pre_out != nullptr, "band pre-pass without an output tensor");
  { static const int kn = pst_knob("PST_TS_KNOB", 0); a.knob = kn; }
  // band box: (Wb*EPC, Hb, nb images, KC/EPC planes) of the planar input, zero outside
  uint64_t dims[4] = {(uint64_t)c.W * kEPC, (uint64_t)c.H, (uint64_t)c.N, (uint64_t)c.Cinp / kEPC};
  uint64_t str[3] = {(uint64_t)c.W * 16, (uint64_t)c.H * c.W * 16, (uint64_t)c.N * c.H * c.W * 16};
  uint32_t box[4] = {(uint32_t)((a.ss ? c.Wo : a.Wb) * kEPC), (uint32_t)a.Hb, (uint32_t)a.nb, (uint32_t)(kc / kEPC)};
  CUtensorMap tA = make_tmap(act_tmap_dtype(), 4, c.in, dims, str, box, nullptr);
  // the band's second tensor (pre-pass shortcut / BN input), same geometry
  const act_t* second = c.pre == 2 ? c.pre_y : c.pre_res;
  CUtensorMap tB = a.pre2 ? make_tmap(act_tmap_dtype(), 4, second, dims, str, box, nullptr) : tA;
  // weights: shadow [2 (hi, lo)][taps][Cinp/EPC][Coutp][EPC] viewed as (EPC, Coutp, Cinp/EPC, 2 taps)
  CUtensorMap tW;
  a.w3d = a.BN * kEPC <= 256 ? 1 : 0;
  if (a.stack) {
    // the shadow is [2 (hi, lo)][taps][Cinp/EPC][Coutp][EPC]; view it as (Coutp*EPC, hi/lo,
    // planes, taps) so one box lands as [tap][plane][hi rows | lo rows] in shared memory
    const uint64_t plane_b = (uint64_t)c.Coutp * 16, tap_b = (uint64_t)(c.Cinp / kEPC) * plane_b;
    uint64_t wd[4] = {(uint64_t)c.Coutp * kEPC, 2, (uint64_t)c.Cinp / kEPC, (uint64_t)a.taps};
    uint64_t ws[3] = {tap_b * a.taps, plane_b, tap_b};
    uint32_t wb[4] = {(uint32_t)(a.BN * kEPC), 2, (uint32_t)(c.Cinp / kEPC), (uint32_t)a.taps};
    tW = make_tmap(act_tmap_dtype(), 4, c.wshadow, wd, ws, wb, nullptr);
  } else if (a.w3d) {
    uint64_t wd[3] = {(uint64_t)c.Coutp * kEPC, (uint64_t)c.Cinp / kEPC, (uint64_t)(2 * a.taps)};
    uint64_t ws[2] = {(uint64_t)c.Coutp * 16, (uint64_t)(c.Cinp / kEPC) * c.Coutp * 16};
    uint32_t wb[3] = {(uint32_t)(a.BN * kEPC), (uint32_t)(c.Cinp / kEPC), (uint32_t)a.taps};
    tW = make_tmap(act_tmap_dtype(), 3, c.wshadow, wd, ws, wb, nullptr);
  } else {
    uint64_t wd[4] = {(uint64_t)kEPC, (uint64_t)c.Coutp, (uint64_t)c.Cinp / kEPC, (uint64_t)(2 * a.taps)};
    uint64_t ws[3] = {16, (uint64_t)c.Coutp * 16, (uint64_t)(c.Cinp / kEPC) * c.Coutp * 16};
    uint32_t wb[4] = {(uint32_t)kEPC, (uint32_t)a.BN, (uint32_t)(c.Cinp / kEPC), (uint32_t)a.taps};
    tW = make_tmap(act_tmap_dtype(), 4, c.wshadow, wd, ws, wb, nullptr);
  }
  const size_t smem = 2 * (size_t)a.w_bytes + (size_t)a.band_stages * a.band_bytes + 4 * 32 * 17 * 4 + 2048 +
                      (3 * kMaxBand + 2 * kMaxSlots + 2 * kMaxAcc + 1) * 8 + 16 + 256 + kCoefBytes;
  auto pick3 = [&](auto kcc, auto tpc) {
    constexpr int K = decltype(kcc)::value, T = decltype(tpc)::value;
#ifdef PST_EXPERIMENTS
    if (a.ss)
      return c.epi == EPI_BN_STATS ? conv_ts_kernel<K, EPI_BN_STATS, 3, 0, 1>
           : c.epi == EPI_DGRAD    ? conv_ts_kernel<K, EPI_DGRAD, 3, 0, 1>
                                   : conv_ts_kernel<K, EPI_BIAS_ACT, 3, 0, 1>;
    if (c.pre)   // the band pre-pass exists for the forward (BN apply) and the dgrad (BN backward)
      return c.epi == EPI_DGRAD ? conv_ts_kernel<K, EPI_DGRAD, T, 1, 0> : conv_ts_kernel<K, EPI_BN_STATS, T, 1, 0>;
#endif
    return c.epi == EPI_BN_STATS ? conv_ts_kernel<K, EPI_BN_STATS, T, 0, 0>
         : c.epi == EPI_DGRAD    ? conv_ts_kernel<K, EPI_DGRAD, T, 0, 0>
                                 : conv_ts_kernel<K, EPI_BIAS_ACT, T, 0, 0>;
  };
  PST_CHECK_ARG(!c.pre || c.epi == EPI_DGRAD || c.epi == EPI_BN_STATS, "band pre-pass needs a BN-stats or dgrad epilogue");
#ifndef PST_EXPERIMENTS
  PST_CHECK_ARG(!c.pre, "the band pre-pass is built only into experiment builds (DESIGN.md section 9)");
#endif
  auto pick = [&](auto kcc) {
    return a.tps == 3 ? pick3(kcc, std::integral_constant<int, 3>{})
         : a.tps == 2 ? pick3(kcc, std::integral_constant<int, 2>{})
                      : pick3(kcc, std::integral_constant<int, 1>{});
  };
  auto kern = kc == 32 ? pick(std::integral_constant<int, 32>{}) : pick(std::integral_constant<int, 16>{});
#ifdef PST_EXPERIMENTS
  if (kc == 8)
    kern = c.epi == EPI_BN_STATS ? conv_ts_kernel<8, EPI_BN_STATS, 3, 0, 1>
         : c.epi == EPI_DGRAD    ? conv_ts_kernel<8, EPI_DGRAD, 3, 0, 1>
                                 : conv_ts_kernel<8, EPI_BIAS_ACT, 3, 0, 1>;
#endif
  PST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev;
  PST_CUDA(cudaGetDevice(&dev));
  const int sms = num_sms(dev);
  const int total = a.n_mtiles * a.n_ntiles;
  const int cap = c.max_ctas > 0 ? std::min(c.max_ctas, sms) : sms;
  const int grid = std::min(total, std::max(a.n_ntiles, (cap / a.n_ntiles) * a.n_ntiles));
  const double es = sizeof(act_t);
  const double bytes = (double)c.N * c.H * c.W * c.Cinp * es +
                       (double)c.N * c.Ho * c.Wo * c.Coutp * (c.epi == EPI_BIAS_F32 ? 4.0 : es) +
                       (double)a.taps * c.Coutp * c.Cinp * es * 2 +
                       (c.res ? (double)c.N * c.res_H * c.res_W * c.res_C * es : 0.0) +
                       (double)c.N * c.H * c.W * c.Cinp * es * ((a.pre2 ? 1.0 : 0.0) + (c.pre ? 1.0 : 0.0));
  const double flops = 2.0 * c.N * c.Ho * c.Wo * c.Coutp * (double)c.Cinp * a.taps;
  prof::begin(st);
  PST_CUDA(launch_k(kern, dim3(grid), dim3(kTsThreads + (c.pre ? 128 : 0)), smem, st, tA, tW, tB, a));
  PST_CUDA(cudaGetLastError());
  prof::end(st, c.epi == EPI_DGRAD ? prof::CONV_DGRAD : prof::CONV_FWD, bytes, flops);
  return true;
}
#else
bool conv_ts(const ConvSpec&, cudaStream_t) { return false; }
bool conv_ts_fits(const ConvSpec&) { return false; }
#endif

}  // namespace pst
