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
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.h"
#include "kernels.h"
#include "ptx.cuh"

namespace pst {

#if PST_SPLIT
namespace {

constexpr int kTsThreads = 448;   // warps: 0 TMA, 1 MMA, 2-5 epilogue, 6-13 converters
constexpr int kMaxBand = 4;
constexpr int kMaxSlots = 16;

struct TsArgs {
  int N, Ho, Wo, Cinp, Coutp, Cout, BN, n_ntiles, n_mtiles, tpi;
  int k, taps, S;
  int n_kc;                  // channel chunks of KC
  int rows_t, nb, Hb, Wb;    // output rows per tile (per image), images per tile, band rows/cols
  int lo;                    // lowest tap offset (both dims)
  int band_stages, n_slots;
  int tps;                   // taps per TMEM A slot (one handshake)
  int w3d;                   // weight tensor map form (3D long rows when BN*EPC <= 256)
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
};

__device__ __forceinline__ unsigned long long ts_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));   // SM cycles (globaltimer reads are slow)
  return t;
}
#define TSL(ev, i)                                                   \
  do {                                                               \
    if (a.dbg != nullptr && blockIdx.x == 0) { const int i_ = (i); if (i_ < 256) a.dbg[(ev) * 256 + i_] = ts_gtime(); } \
  } while (0)

__device__ __forceinline__ float ld_planar_f(const act_t* base, int64_t npix, int64_t pix, int c) {
  return act2f(base[((int64_t)(c / kEPC) * npix + pix) * kEPC + c % kEPC]);
}

template <int KC, int EPI>
__global__ void __launch_bounds__(kTsThreads, 1)
    conv_ts_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, const TsArgs a) {
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
  uint64_t* tempty = tfull + 2;
  uint64_t* wbar = tempty + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(wbar + 1);
  int* tsh = reinterpret_cast<int*>(tmem_ptr + 4);   // tap shifts (a.tapshift indexed dynamically
                                                     // from the param space would be copied to local memory)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TSL(7, 0);
  int dbg_i[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int nt = blockIdx.x % a.n_ntiles;            // a CTA keeps one N tile (resident weights)
  const int m0 = blockIdx.x / a.n_ntiles, mstep = gridDim.x / a.n_ntiles;
  const int planes_w = a.Cinp / kEPC;                // weight planes per tap

  if (threadIdx.x == 0) {
    for (int i = 0; i < a.band_stages; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&bempty[i], 8); }
    for (int i = 0; i < a.n_slots; ++i) { ptx::mbar_init(&afull[i], 4); ptx::mbar_init(&aempty[i], 1); }
    for (int i = 0; i < 2; ++i) { ptx::mbar_init(&tfull[i], 1); ptx::mbar_init(&tempty[i], 4); }
    ptx::mbar_init(wbar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_ptr, 512);
#pragma unroll 1
  for (int t = threadIdx.x; t < 49; t += blockDim.x) {
    int v = 0;
#pragma unroll
    for (int j = 0; j < 49; ++j) v = (j == t) ? a.tapshift[j] : v;
    tsh[t] = v;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  pdl_wait();      // no global memory access above this line
  pdl_trigger();
  const uint32_t a_col0 = 2 * a.BN;                  // accumulators: columns [0, 2 BN)

  if (a.knob & 16) {
    // experiment: prologue and teardown only
  } else if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&tmA);
      ptx::prefetch_tmap(&tmW);
      ptx::mbar_expect_tx(wbar, 2 * a.w_bytes);
      if (a.w3d) {   // long rows: (BN*EPC, planes, taps)
        ptx::tma_load_3d(wsm, &tmW, wbar, nt * a.BN * kEPC, 0, 0);                 // hi: taps [0, taps)
        ptx::tma_load_3d(wsm + a.w_bytes, &tmW, wbar, nt * a.BN * kEPC, 0, a.taps);  // lo: taps [taps, 2 taps)
      } else {
        ptx::tma_load_4d(wsm, &tmW, wbar, 0, nt * a.BN, 0, 0);
        ptx::tma_load_4d(wsm + a.w_bytes, &tmW, wbar, 0, nt * a.BN, 0, a.taps);
      }
    }
    __syncwarp();
    int bs = 0;
    uint32_t bph = 0;
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      const int n0 = a.nb > 1 ? m * a.nb : m / a.tpi;
      const int y0 = a.nb > 1 ? 0 : (m % a.tpi) * a.rows_t;
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        ptx::mbar_wait(&bempty[bs], bph ^ 1);
        if (lane == 0) TSL(0, dbg_i[0]++);
        if (ptx::elect_one()) {
          if (a.knob & 32) { ptx::mbar_arrive(&full[bs]); } else {
          ptx::mbar_expect_tx(&full[bs], a.band_tx);
          ptx::tma_load_4d(bands + bs * a.band_bytes, &tmA, &full[bs], a.lo * kEPC, y0 * a.S + a.lo, n0,
                           kcc * (KC / kEPC));
          }
        }
        __syncwarp();
        if (++bs == a.band_stages) { bs = 0; bph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = ptx::idesc_mma(128, a.BN, 0, 0, 2);
    const uint32_t wtap = (uint32_t)planes_w * a.BN * 16;     // weight bytes per tap (hi)
    const uint64_t wdesc = ptx::smem_desc(ptx::smem_u32(wsm), a.BN * 16, 128);
    ptx::mbar_wait(wbar, 0);
    int slot = 0;
    uint32_t sph = 0;
    int local = 0;
    const int ngrp = a.taps / a.tps;
    for (int m = m0; m < a.n_mtiles; m += mstep, ++local) {
      const int acc = local & 1;
      ptx::mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d = tmem + acc * a.BN;
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        for (int gi = 0; gi < ngrp; ++gi) {
          ptx::mbar_wait(&afull[slot], sph);
          ptx::tc_fence_after();
          if (lane == 0) TSL(4, dbg_i[4]++);
          if (ptx::elect_one()) {
            // one slot = tps taps x (KC hi + KC lo columns): 3 x KC/8 x tps MMAs per handshake
            for (int i = 0; i < a.tps && !(a.knob & 2); ++i) {
              const int t = gi * a.tps + i;
              const uint32_t ahi = tmem + a_col0 + (slot * a.tps + i) * 2 * KC;
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
            ptx::umma_commit(&aempty[slot]);
          }
          __syncwarp();
          if (lane == 0) TSL(2, dbg_i[2]++);
          if (++slot == a.n_slots) { slot = 0; sph ^= 1; }
        }
      }
      if (ptx::elect_one()) ptx::umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= 6) {
    // ---------------------------------------------------------------- converters (warps 6..13)
    // Two sets of 4 warps (one warp per TMEM lane quarter each) take alternate tap groups of
    // the global sequence.  Per group: for each of its tps taps, load the pixel's shifted input
    // channels from the band, split hi/lo, tcgen05.st both (no wait); one wait + one arrive
    // per group, so loads and stores of consecutive taps overlap.
    const int q = warp & 3;                  // TMEM lane quarter of this warp
    const int set = (warp - 6) >> 2;
    const int r = q * 32 + lane;             // tile pixel = TMEM lane
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    const int per_img = a.rows_t * a.Wo;
    const int j = r / per_img, yy = (r / a.Wo) % a.rows_t, xx = r % a.Wo;
    const int pixoff = (j * a.Hb + yy * a.S) * a.Wb + xx * a.S;
    const int ngrp = a.taps / a.tps;
    int bs = 0;
    uint32_t bph = 0;
    uint32_t cnt = 0;                        // global group counter (same order as the MMA issuer)
    for (int m = m0; m < a.n_mtiles; m += mstep) {
      for (int kcc = 0; kcc < a.n_kc; ++kcc) {
        if (a.knob & 128) ptx::mbar_wait_sleep(&full[bs], bph, 100); else ptx::mbar_wait(&full[bs], bph);
        const uint8_t* band = bands + bs * a.band_bytes;
        for (int gi = (int)((cnt + set) & 1); gi < ngrp; gi += 2) {
          const uint32_t c = cnt + gi;
          const int slot = (int)(c % a.n_slots);
          if (a.knob & 128) ptx::mbar_wait_sleep(&aempty[slot], ((c / a.n_slots) & 1) ^ 1, 100);
          else ptx::mbar_wait(&aempty[slot], ((c / a.n_slots) & 1) ^ 1);
          ptx::tc_fence_after();
          if (threadIdx.x == 192) TSL(1, dbg_i[1]++);
          for (int i = 0; i < a.tps && !(a.knob & 1); ++i) {
            const int t = gi * a.tps + i;
            const uint8_t* src = band + (uint32_t)(pixoff + tsh[t]) * 16;
            float hi[KC], lo[KC];
#pragma unroll
            for (int p4 = 0; p4 < KC / 4; ++p4) {
              const float4 v = *reinterpret_cast<const float4*>(src + p4 * a.plane_bytes);
              hi[4 * p4 + 0] = v.x; hi[4 * p4 + 1] = v.y; hi[4 * p4 + 2] = v.z; hi[4 * p4 + 3] = v.w;
            }
#pragma unroll
            for (int e = 0; e < KC; ++e) lo[e] = tf32_lo(hi[e]);
            const uint32_t ta = tmem + lane_addr + a_col0 + (slot * a.tps + i) * 2 * KC;
#pragma unroll
            for (int h = 0; h < KC / 16; ++h) {
              ptx::tmem_st16(ta + h * 16, hi + 16 * h);
              ptx::tmem_st16(ta + KC + h * 16, lo + 16 * h);
            }
          }
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&afull[slot]);
          if (threadIdx.x == 192) TSL(3, dbg_i[3]++);
        }
        cnt += ngrp;
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
    if (EPI == EPI_BN_STATS) {
      for (int i = lane; i < 2 * a.BN; i += 32) wacc[q * 2 * a.BN + i] = 0.0;
      __syncwarp();
    }
    const int per_img = a.rows_t * a.Wo;
    const int64_t npix = (int64_t)a.N * a.Ho * a.Wo;
    const int ng = a.BN / 16;
    int local = 0;
    for (int m = m0; m < a.n_mtiles; m += mstep, ++local) {
      const int acc = local & 1;
      ptx::mbar_wait(&tfull[acc], (local >> 1) & 1);
      ptx::tc_fence_after();
      if (threadIdx.x == 64) TSL(5, dbg_i[5]++);
      const int n = (a.nb > 1 ? m * a.nb : m / a.tpi) + r / per_img;
      const int y = (a.nb > 1 ? 0 : (m % a.tpi) * a.rows_t) + (r / a.Wo) % a.rows_t;
      const int x = r % a.Wo;
      const bool valid = n < a.N;
      const int64_t pix = ((int64_t)n * a.Ho + y) * a.Wo + x;
      for (int g = 0; g < ng; ++g) {
        float u[16];
        if (a.knob & 64) {
#pragma unroll
          for (int i = 0; i < 16; ++i) u[i] = 0.f;
        } else ptx::tmem_ld16(tmem + lane_addr + acc * a.BN + g * 16, u);
        if (g == ng - 1) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        }
        const int c0 = nt * a.BN + g * 16;
        if (EPI == EPI_BN_STATS) {
          if (!valid) {
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] = 0.f;
          }
        } else if (EPI == EPI_DGRAD) {   // + shortcut^T of the residual layer's gradient
          if (valid && a.res_mode == 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) u[i] += ld_planar_f(a.res, npix, pix, c0 + i);
          } else if (valid && a.res_mode == 2 && ((y | x) & 1) == 0) {
            const int64_t rpix = ((int64_t)n * a.res_H + (y >> 1)) * a.res_W + (x >> 1);
            const int64_t rnpix = (int64_t)a.N * a.res_H * a.res_W;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int c = c0 + i;
              if (c < a.Cout) u[i] += ld_planar_f(a.res, rnpix, rpix, c + a.res_pad);
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
        if (valid && !(a.knob & 8)) {
          float* o = reinterpret_cast<float*>(a.out);   // act_t == float in this build
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            *reinterpret_cast<float4*>(o + ((int64_t)(c0 / 4 + jj) * npix + pix) * 4) =
                make_float4(u[4 * jj], u[4 * jj + 1], u[4 * jj + 2], u[4 * jj + 3]);
        }
        if (EPI == EPI_BN_STATS && !(a.knob & 4)) {
          float s1[16], s2[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) { s1[i] = u[i]; s2[i] = u[i] * u[i]; }
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
          s1[0] += __shfl_xor_sync(0xffffffffu, s1[0], 1);   // lanes 2c, 2c+1 hold channel c
          s2[0] += __shfl_xor_sync(0xffffffffu, s2[0], 1);
          if ((lane & 1) == 0) {
            double* w2 = wacc + q * 2 * a.BN + 2 * (g * 16 + (lane >> 1));
            w2[0] += (double)s1[0];
            w2[1] += (double)s2[0];
          }
        }
      }
      if (threadIdx.x == 64) TSL(6, dbg_i[6]++);
    }
    if (EPI == EPI_BN_STATS) {
      ptx::named_bar_sync(1, 128);
      for (int i = et; i < 2 * a.BN; i += 128) {
        const double v = wacc[i] + wacc[2 * a.BN + i] + wacc[4 * a.BN + i] + wacc[6 * a.BN + i];
        if (v != 0.0) atomicAdd(&a.stats[2 * nt * a.BN + i], v);
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
static bool ts_plan(const ConvSpec& c, TsArgs& a, int& kc) {
  if (std::getenv("PST_NOTS") != nullptr) return false;
  if (c.k > 7 || (c.S != 1 && c.S != 2) || c.Coutp > 256) return false;
  if (c.Wo > 128 || 128 % c.Wo != 0) return false;
  const int per_img = c.Ho * c.Wo;
  if (!(per_img % 128 == 0 || 128 % per_img == 0)) return false;
  kc = (c.Cinp % 32 == 0) ? 32 : 16;
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
  a.plane_bytes = (uint32_t)a.nb * a.Hb * a.Wb * 16;
  a.band_tx = a.plane_bytes * (kc / kEPC);
  a.band_bytes = (uint32_t)round_up((int)a.band_tx, 1024);
  // N tile: resident hi+lo weights of all taps <= 112 KB
  a.BN = 0;
  for (int bn = std::min(c.Coutp, 128); bn >= 16; bn -= 16)
    if (c.Coutp % bn == 0 && 2ll * a.taps * c.Cinp * bn * 4 <= 112 * 1024) { a.BN = bn; break; }
  if (a.BN == 0) return false;
  a.n_ntiles = c.Coutp / a.BN;
  a.w_bytes = (uint32_t)a.taps * c.Cinp * a.BN * 4;
  const int fixed = 2 * (int)a.w_bytes + 4 * 32 * 17 * 4 + 2048 + (2 * kMaxBand + 2 * kMaxSlots + 5) * 8 + 16 + 256;
  a.band_stages = std::min(kMaxBand, (227 * 1024 - 1024 - fixed) / (int)a.band_bytes);
  if (a.band_stages < 2) return false;
  a.tps = 1;
  for (int tps : {3, 2, 1})
    if (a.taps % tps == 0 && (512 - 2 * a.BN) / (2 * kc * tps) >= 2) { a.tps = tps; break; }
  a.n_slots = std::min(kMaxSlots, (512 - 2 * a.BN) / (2 * kc * a.tps));
  if (a.n_slots < 2) return false;
  return true;
}

bool conv_ts(const ConvSpec& c, cudaStream_t st) {
  TsArgs a;
  int kc;
  if (!ts_plan(c, a, kc)) return false;
  a.epi = c.epi; a.relu = c.relu; a.out = c.out; a.bias = c.bias; a.stats = c.stats;
  a.res = c.res; a.res_mode = c.res_mode; a.res_H = c.res_H; a.res_W = c.res_W; a.res_C = c.res_C;
  a.res_pad = c.res_pad;
  a.dbg = c.dbg;
  { static const char* kn = std::getenv("PST_TS_KNOB"); a.knob = kn ? std::atoi(kn) : 0; }
  // band box: (Wb*EPC, Hb, nb images, KC/EPC planes) of the planar input, zero outside
  uint64_t dims[4] = {(uint64_t)c.W * kEPC, (uint64_t)c.H, (uint64_t)c.N, (uint64_t)c.Cinp / kEPC};
  uint64_t str[3] = {(uint64_t)c.W * 16, (uint64_t)c.H * c.W * 16, (uint64_t)c.N * c.H * c.W * 16};
  uint32_t box[4] = {(uint32_t)(a.Wb * kEPC), (uint32_t)a.Hb, (uint32_t)a.nb, (uint32_t)(kc / kEPC)};
  CUtensorMap tA = make_tmap(act_tmap_dtype(), 4, c.in, dims, str, box, nullptr);
  // weights: shadow [2 (hi, lo)][taps][Cinp/EPC][Coutp][EPC] viewed as (EPC, Coutp, Cinp/EPC, 2 taps)
  CUtensorMap tW;
  a.w3d = a.BN * kEPC <= 256 ? 1 : 0;
  if (a.w3d) {
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
                      (2 * kMaxBand + 2 * kMaxSlots + 5) * 8 + 16 + 256;
  auto pick = [&](auto kcc) {
    constexpr int K = decltype(kcc)::value;
    return c.epi == EPI_BN_STATS ? conv_ts_kernel<K, EPI_BN_STATS>
         : c.epi == EPI_DGRAD    ? conv_ts_kernel<K, EPI_DGRAD>
                                 : conv_ts_kernel<K, EPI_BIAS_ACT>;
  };
  auto kern = kc == 32 ? pick(std::integral_constant<int, 32>{}) : pick(std::integral_constant<int, 16>{});
  PST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev;
  PST_CUDA(cudaGetDevice(&dev));
  const int sms = num_sms(dev);
  const int total = a.n_mtiles * a.n_ntiles;
  const int grid = std::min(total, std::max(a.n_ntiles, (sms / a.n_ntiles) * a.n_ntiles));
  const double es = sizeof(act_t);
  const double bytes = (double)c.N * c.H * c.W * c.Cinp * es +
                       (double)c.N * c.Ho * c.Wo * c.Coutp * (c.epi == EPI_BIAS_F32 ? 4.0 : es) +
                       (double)a.taps * c.Coutp * c.Cinp * es * 2 +
                       (c.res ? (double)c.N * c.res_H * c.res_W * c.res_C * es : 0.0);
  const double flops = 2.0 * c.N * c.Ho * c.Wo * c.Coutp * (double)c.Cinp * a.taps;
  prof::begin(st);
  PST_CUDA(launch_k(kern, dim3(grid), dim3(kTsThreads), smem, st, tA, tW, a));
  PST_CUDA(cudaGetLastError());
  prof::end(st, c.epi == EPI_DGRAD ? prof::CONV_DGRAD : prof::CONV_FWD, bytes, flops);
  return true;
}
#else
bool conv_ts(const ConvSpec&, cudaStream_t) { return false; }
#endif

}  // namespace pst
