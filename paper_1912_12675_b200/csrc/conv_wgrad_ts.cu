// conv_wgrad_ts.cu -- weight gradient dW = X_shifted^T dY on tcgen05 with the expanded input
// operand in TENSOR MEMORY (3xTF32 build).
//
//   dW[tap*Cinp + ci][co] = sum_p X[p shifted by tap][ci] * dY[p][co]
//   M = rows (tap, ci), N = co, K = output pixels p.
//
// A (M x K) is the im2col expansion of the input.  The smem-operand design materialised it
// (hi and lo planes, M padded to 128) in shared memory and re-read it three times per K step;
// here each converter thread owns one row (= one TMEM lane) and writes that row's K values
// straight into a TMEM slot with tcgen05.st (hi and lo), so the expansion costs one 4-byte
// shared load per element and the MMAs read A from TMEM ("TS" form, tools/mma_bench.cu).
//   warp 0     TMA: per stage one input band box (all taps' rows/cols of the stage's pixels)
//              and one dY box
//   warps 2-9  converters (two per TMEM lane quarter): A rows -> TMEM slot; dY -> K-major
//              hi/lo B rows in smem
//   warp 1     MMA: D_j += A_hi B_hi + A_hi B_lo + A_lo B_hi for the CTA's M tiles j
//   warps 2-5  finally drain D into split-K partials part[ks][rows][Coutp]
#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "kernels.h"
#include "ptx.cuh"

namespace pst {

#if PST_SPLIT
namespace {

// warps: 0 TMA, 1 MMA, 2.. converters in SETS sets of 4 taking units in turn (2-5 also epilogue)
constexpr int wt_threads(int sets) { return (2 + 4 * sets) * 32; }
constexpr int kWtMaxSB = 8;
constexpr int kWtMaxSlots = 8;

struct WtArgs {
  int N, H, W, Cinp, Ho, Wo, Coutp;
  int k, S, pad;
  int nb, bh, P, P16, band_r, band_c, ny, n_units;
  int rows, n_mt, G, n_mgroups, BNw, n_ntiles, ksplit;
  int pl_grp, pl_all;
  int SB, St;                          // smem stages, TMEM A slots
  int sets;                            // converter sets (2 or 3; compile-time in the kernel)
  uint32_t rawx_bytes, rawx_tx, rawd_bytes, b_bytes, stage_bytes, sboB;
  float* part;
  unsigned long long* dbg;   // optional timeline (CTA 0, clock64), PST_DBG_TL
};
#ifdef PST_EXPERIMENTS
#define WTL(ev, i)                                                                        \
  do {                                                                                   \
    if (a.dbg != nullptr && blockIdx.x == 0) {                                           \
      const int i_ = (i);                                                                \
      unsigned long long t_;                                                             \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));                                 \
      if (i_ < 256) a.dbg[(ev) * 256 + i_] = t_;                                         \
    }                                                                                    \
  } while (0)
#else
#define WTL(ev, i) do { } while (0)
#endif

template <int G, int P16, int SETS>
__global__ void __launch_bounds__(wt_threads(SETS), 1)
    conv_wgrad_ts_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD,
                         const WtArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // [SB stages: raw X | raw dY | B hi | B lo] [pixel table P16 ints] [barriers] [tmem ptr]
  uint8_t* ring = smem;
  int* pixb = reinterpret_cast<int*>(smem + a.SB * a.stage_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(pixb + 128);
  uint64_t* full = bars;
  uint64_t* empty = full + kWtMaxSB;
  uint64_t* ready = empty + kWtMaxSB;
  uint64_t* afree = ready + kWtMaxSlots;
  uint64_t* tfull = afree + kWtMaxSlots;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) WTL(7, 0);

  const int b = blockIdx.x;
  const int mg = b % a.n_mgroups;
  const int nt = (b / a.n_mgroups) % a.n_ntiles;
  const int ks = b / (a.n_mgroups * a.n_ntiles);
  const int u_lo = (int)((int64_t)ks * a.n_units / a.ksplit);
  const int u_hi = (int)((int64_t)(ks + 1) * a.n_units / a.ksplit);
  const int n_iter = u_hi - u_lo;
  const int mt0 = mg * a.G;
  const int g_cnt = min(a.G, a.n_mt - mt0);
  const int r0 = mt0 * 128;
  const int r_end = min(r0 + g_cnt * 128, a.rows);
  const int pl0 = a.pl_all ? 0 : (r0 % a.Cinp) / kEPC;
  const uint32_t off_rawd = a.rawx_bytes;
  const uint32_t off_b = off_rawd + ((a.rawd_bytes + 127u) & ~127u);
  const uint32_t acc_cols = (uint32_t)a.G * a.BNw;       // accumulators: [0, G*BNw)
  const uint32_t slot_cols = (uint32_t)a.G * 2 * a.P16;  // per slot: G tiles x (P16 hi + P16 lo)

  if (warp == 0) {   // lane i initialises the i-th barrier of each ring (<= 8 entries each)
    bool any = false;
    if (lane < a.SB) { ptx::mbar_init(&full[lane], 1); ptx::mbar_init(&empty[lane], 1); any = true; }
    if (lane < a.St) { ptx::mbar_init(&ready[lane], 4); ptx::mbar_init(&afree[lane], 1); any = true; }
    if (lane == 0) { ptx::mbar_init(tfull, 1); any = true; }
    if (any) ptx::fence_mbar_init();
  }
  if (threadIdx.x < a.P16) {   // pixel table: float offset of pixel p in the band (-1: padding)
    const int p = threadIdx.x;
    const int hw = a.bh * a.Wo;
    if (p >= a.P) pixb[p] = -1;
    else {
      const int jj = p / hw, py = (p / a.Wo) % a.bh, px = p % a.Wo;
      pixb[p] = ((jj * a.band_r + py * a.S) * a.band_c + px * a.S) * 4;
    }
  }
  if (warp == 1) ptx::tmem_alloc(tmem_ptr, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  pdl_wait();      // no global memory access above this line
  pdl_trigger();
  // stage sb <- unit (image group n0, row block y0): input band + dY box (elected producer lane)
  auto issue_unit = [&](int sb, int n0, int y0) {
    uint8_t* s0 = ring + sb * a.stage_bytes;
    ptx::mbar_expect_tx(&full[sb], a.rawx_tx + a.rawd_bytes);
    ptx::tma_load_4d(s0, &tmX, &full[sb], -a.pad * kEPC, y0 * a.S - a.pad, n0, pl0);
    ptx::tma_load_4d(s0 + off_rawd, &tmD, &full[sb], 0, y0, n0, nt * (a.BNw / kEPC));
  };
  // the first unit right after the dependency wait, before the role dispatch (cold producer code)
#ifndef PST_NO_EARLY_BAND
  if (warp == 0 && n_iter > 0 && ptx::elect_one())
    issue_unit(0, (u_lo / a.ny) * a.nb, (u_lo % a.ny) * a.bh);
#endif
  __syncwarp();

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    int sb = 0;
    uint32_t sbph = 0;
    int uq = u_lo / a.ny, ur = u_lo % a.ny;   // unit -> (image group, row block), advanced incrementally
    for (int it = 0; it < n_iter; ++it) {
      const int n0 = uq * a.nb, y0 = ur * a.bh;
      if (++ur == a.ny) { ur = 0; ++uq; }
      ptx::mbar_wait(&empty[sb], sbph ^ 1);
      if (lane == 0) WTL(0, it);
#ifndef PST_NO_EARLY_BAND
      if (it > 0 && ptx::elect_one()) issue_unit(sb, n0, y0);
#else
      if (ptx::elect_one()) issue_unit(sb, n0, y0);
#endif
      __syncwarp();
      if (++sb == a.SB) { sb = 0; sbph ^= 1; }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = ptx::idesc_mma(128, a.BNw, 0, 0, 2);
    int sb = 0, slot = 0;
    uint32_t slph = 0;
    for (int it = 0; it < n_iter; ++it) {
      ptx::mbar_wait(&ready[slot], slph);
      ptx::tc_fence_after();
      if (lane == 0) WTL(4, it);
      const uint64_t bd0 = ptx::smem_desc(ptx::smem_u32(ring + sb * a.stage_bytes + off_b), 128, a.sboB);
      if (ptx::elect_one()) {
        // straight-line block (compile-time G, P16): all G tiles are issued, a missing last
        // tile only accumulates into an unused accumulator
        const uint32_t abase = tmem + acc_cols + slot * slot_cols;
#pragma unroll
        for (int kk = 0; kk < P16 / 8; ++kk) {
          const uint64_t bd = ptx::desc_add(bd0, kk * 256);
          const uint64_t bdl = ptx::desc_add(bd, a.b_bytes);
          const uint32_t acc0 = (it > 0 || kk > 0) ? 1u : 0u;
#pragma unroll
          for (int j = 0; j < G; ++j) {
            const uint32_t ahi = abase + j * 2 * P16 + kk * 8;
            const uint32_t d = tmem + j * a.BNw;
            ptx::umma_tf32_ts(d, ahi, bd, idesc, acc0);
            ptx::umma_tf32_ts(d, ahi, bdl, idesc, 1u);
            ptx::umma_tf32_ts(d, ahi + P16, bd, idesc, 1u);
          }
        }
        ptx::umma_commit(&empty[sb]);
        ptx::umma_commit(&afree[slot]);
      }
      __syncwarp();
      if (lane == 0) WTL(2, it);
      if (++sb == a.SB) sb = 0;
      if (++slot == a.St) { slot = 0; slph ^= 1; }
    }
    if (n_iter > 0 && ptx::elect_one()) ptx::umma_commit(tfull);
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- converters (warps 2..9)
    // Two sets of 4 warps (one warp per TMEM lane quarter each) take alternate iterations, so two
    // units are converted concurrently (the per-unit chain -- shared loads, hi/lo split,
    // tcgen05.st, wait::st -- is latency-bound).  A set converts all P16 pixels of its unit for
    // every M tile the CTA owns, and the unit's dY block into the K-major hi/lo B rows.
    const int q = warp & 3;
    const int set = (warp - 2) >> 2;            // 0 .. SETS-1
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    int rb[4] = {-1, -1, -1, -1};               // this thread's A row (one per owned M tile)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int R = r0 + j * 128 + q * 32 + lane;
      if (j < g_cnt && R < r_end) {
        const int tap = R / a.Cinp, ci = R % a.Cinp;
        const int rr = tap / a.k, ss = tap % a.k;
        const int plane = ci / kEPC - pl0;
        rb[j] = ((plane * a.nb * a.band_r + rr) * a.band_c + ss) * 4 + ci % kEPC;
      }
    }
    const int nq = a.P16 / 4;
    const int unitsB = (a.BNw / 4) * nq;

    int sb = 0, slot = 0;
    uint32_t sbph = 0, slph = 0;
    int turn = 0;                               // set owning unit `it`
    for (int it = 0; it < n_iter; ++it) {
      const int my_sb = sb, my_slot = slot;
      const uint32_t my_sbph = sbph, my_slph = slph;
      if (++sb == a.SB) { sb = 0; sbph ^= 1; }
      if (++slot == a.St) { slot = 0; slph ^= 1; }
      const bool mine = turn == set;
      if (++turn == SETS) turn = 0;
      if (!mine) continue;                       // another set's unit
      ptx::mbar_wait(&full[my_sb], my_sbph);
      ptx::mbar_wait(&afree[my_slot], my_slph ^ 1);
      ptx::tc_fence_after();
      if (threadIdx.x == 64) WTL(1, it);
      uint8_t* s0 = ring + my_sb * a.stage_bytes;
      const float* rawxf = reinterpret_cast<const float*>(s0);
      const float* rawdf = reinterpret_cast<const float*>(s0 + off_rawd);
      uint8_t* bhi = s0 + off_b;
      uint8_t* blo = bhi + a.b_bytes;
      // B: dY [co/4][P][4] -> K-major hi/lo rows (co) x pixels, 4 co x 4 px per task
      // (the set's even lanes: task u runs on warp quarter u % 4, lane 2 * ((u / 4) % 16))
      for (int u = (lane % 2 == 0) ? (lane / 2) * 4 + q : unitsB; u < unitsB; u += 64) {
        const int kq = u % nq, cq = u / nq;
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int p = 4 * kq + i;
          v[i] = p < a.P ? *reinterpret_cast<const float4*>(rawdf + ((int64_t)cq * a.P + p) * 4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int co = 4 * cq + c;
          float4 h;
          if (c == 0) h = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
          else if (c == 1) h = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
          else if (c == 2) h = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
          else h = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
          const uint32_t off = (uint32_t)((co >> 3) * a.sboB + kq * 128 + (co & 7) * 16);
          *reinterpret_cast<float4*>(bhi + off) = h;
          *reinterpret_cast<float4*>(blo + off) = make_float4(tf32_lo(h.x), tf32_lo(h.y), tf32_lo(h.z), tf32_lo(h.w));
        }
      }
      // A: rows -> TMEM slot (hi columns [0,P16), lo columns [P16, 2 P16) per tile), all pixels
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= g_cnt) break;
        // a warp whose 32 rows all lie past the last real row (the padded tail of the last M tile:
        // 112 of the 256 rows of a 16-channel layer) leaves its TMEM lanes stale: they only feed
        // accumulator rows the epilogue never writes
        if (r0 + j * 128 + q * 32 >= r_end) continue;
        const uint32_t ta = tmem + lane_addr + acc_cols + my_slot * slot_cols + j * 2 * a.P16;
#pragma unroll
        for (int h = 0; h < P16 / 16; ++h) {
          float hv[16], lv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int pbv = pixb[h * 16 + i];       // broadcast shared load
            hv[i] = (rb[j] >= 0 && pbv >= 0) ? rawxf[rb[j] + pbv] : 0.f;
            lv[i] = tf32_lo(hv[i]);
          }
          ptx::tmem_st16(ta + h * 16, hv);
          ptx::tmem_st16(ta + a.P16 + h * 16, lv);
        }
      }
      ptx::tmem_st_wait();
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ready[my_slot]);
      if (threadIdx.x == 64) WTL(3, it);
    }
    if (warp < 6) {
      // ---------------------------------------------------------------- epilogue (warps 2..5)
      if (n_iter > 0) {
        ptx::mbar_wait(tfull, 0);
        ptx::tc_fence_after();
      }
      if (threadIdx.x == 64) WTL(5, 0);
      for (int j = 0; j < g_cnt; ++j) {
        const int R = r0 + j * 128 + q * 32 + lane;
        for (int ch = 0; ch < a.BNw / 16; ++ch) {
          float v[16];
          if (n_iter > 0) {
            ptx::tmem_ld16(tmem + lane_addr + j * a.BNw + ch * 16, v);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          }
          if (R < a.rows) {
            float4* op = reinterpret_cast<float4*>(a.part + ((int64_t)ks * a.rows + R) * a.Coutp + nt * a.BNw + ch * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) op[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        }
      }
    }
  }
  if (threadIdx.x == 64) WTL(6, 0);
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

int tile_n16(int C, int cap) {
  int best = 16;
  for (int b = 16; b <= cap && b <= C; b += 16)
    if (C % b == 0) best = b;
  return best;
}

}  // namespace

static bool wgrad_ts_plan_p(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad,
                            int num_sm, int ptarget, WtArgs& a);

// Pixels per unit: 32 by default; 16 when 32-pixel units leave fewer than 3 TMEM A slots and 16-pixel
// units do not (the 32-channel ResNet-CIFAR layers: 3 M tiles at N = 32 fit 2 slots of 32 pixels but
// 4 of 16; measured g2 wgrad 19.9 -> 13.7 us, profiles/r2_wgrad_knobs.txt).
bool wgrad_ts_plan(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad, int num_sm,
                   void* out) {
  if (pst_knob("PST_NOTS", 0)) return false;
  static const int forced = pst_knob("PST_WT_PTARGET", 0);   // experiment: fixed pixels per unit
  WtArgs a{}, b{};
  bool ok = wgrad_ts_plan_p(N, H, W, Cinp, Ho, Wo, Coutp, k, S, pad, num_sm, forced ? forced : 32, a);
  if (!forced && ok && a.St < 3 && wgrad_ts_plan_p(N, H, W, Cinp, Ho, Wo, Coutp, k, S, pad, num_sm, 16, b) &&
      b.St >= 3 && b.G == a.G)
    a = b;
  if (ok && out) *reinterpret_cast<WtArgs*>(out) = a;
  return ok;
}

static bool wgrad_ts_plan_p(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad,
                            int num_sm, int ptarget, WtArgs& a) {
  a = WtArgs{};
  a.N = N; a.H = H; a.W = W; a.Cinp = Cinp; a.Ho = Ho; a.Wo = Wo; a.Coutp = Coutp;
  a.k = k; a.S = S; a.pad = pad;
  a.rows = k * k * Cinp;
  a.n_mt = ceil_div(a.rows, 128);
  a.BNw = tile_n16(Coutp, 128);
  a.n_ntiles = Coutp / a.BNw;
  if (Ho * Wo >= ptarget) { a.nb = 1; a.bh = std::max(1, std::min(Ho, ptarget / Wo)); }
  else { a.nb = std::max(1, std::min(N, ptarget / (Ho * Wo))); a.bh = Ho; }
  a.P = a.nb * a.bh * Wo;
  a.P16 = round_up(a.P, 16);
  if (a.P16 != 16 && a.P16 != 32 && a.P16 != 64) return false;
  a.band_r = (a.bh - 1) * S + k;
  a.band_c = (Wo - 1) * S + k;
  if (a.band_c * kEPC > 256 || a.band_r > 256) return false;
  // M tiles per CTA: largest G with >= 2 TMEM slots
  a.G = 0;
  static const int gmax = pst_knob("PST_WT_GMAX", 4);   // experiment: cap on M tiles per CTA
  for (int G = std::min(std::min(a.n_mt, 4), std::max(1, gmax)); G >= 1; --G) {
    const int slots = (512 - G * a.BNw) / (G * 2 * a.P16);
    if (slots >= 2) { a.G = G; a.St = std::min(kWtMaxSlots, slots); break; }
  }
  if (a.G == 0) return false;
  const bool all = (a.G * 128 >= Cinp) || (Cinp % (a.G * 128) != 0);
  a.pl_all = all ? 1 : 0;
  a.pl_grp = all ? Cinp / kEPC : a.G * 128 / kEPC;
  if (a.pl_grp > 256) return false;
  a.rawx_tx = (uint32_t)a.pl_grp * a.nb * a.band_r * a.band_c * 16;
  a.rawx_bytes = (uint32_t)round_up((int)a.rawx_tx, 128);
  a.rawd_bytes = (uint32_t)(a.BNw / kEPC) * a.P * 16;
  a.b_bytes = (uint32_t)a.BNw * a.P16 * 4;
  a.sboB = (uint32_t)(a.P16 / 4) * 128;
  a.stage_bytes = (uint32_t)round_up((int)(a.rawx_bytes + round_up((int)a.rawd_bytes, 128) + 2 * a.b_bytes), 1024);
  const int budget = 200 * 1024;
  a.SB = std::min(kWtMaxSB, budget / (int)a.stage_bytes);
  if (a.SB < 2) return false;
  // a third converter set (three units in flight) where the slots allow it without shrinking G:
  // a set reuses a slot / band stage only after the unit SETS earlier waited on it (mbarrier
  // parity aliasing), so St >= SETS and SB >= SETS
  static const int max_sets = pst_knob("PST_WT_SETS", 3);
  // (measured: g1 wgrad 24.2 -> 21.3 us with 3 sets; the 576-row g3 gets slower, so only the
  // small-row layers take it)
  static const int sets3_rows = pst_knob("PST_WT_SETS3_ROWS", 256);   // experiment: row limit for 3 sets
  a.sets = (max_sets >= 3 && a.St >= 3 && a.SB >= 3 && a.rows <= sets3_rows) ? 3 : 2;
  a.n_mgroups = ceil_div(a.n_mt, a.G);
  a.ny = ceil_div(Ho, a.bh);
  a.n_units = ceil_div(N, a.nb) * a.ny;
  const int base = a.n_mgroups * a.n_ntiles;
  a.ksplit = std::max(1, std::min(std::max(1, a.n_units / 2), num_sm / base));
  // cap on the split (PST_WT_KSPLIT_MAX experiments): fewer fp32 partials to write and reduce
  static const int ks_max = pst_knob("PST_WT_KSPLIT_MAX", 0);
  if (ks_max > 0) a.ksplit = std::min(a.ksplit, ks_max);
  static const int ks_big = pst_knob("PST_WT_KSPLIT_MAX_BIG", 0);
  if (ks_big > 0 && a.rows > 256) a.ksplit = std::min(a.ksplit, ks_big);   // the many-row (64-channel) layers only
  return true;
}

int wgrad_ts_ksplit(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad, int num_sm) {
  WtArgs a;
  if (!wgrad_ts_plan(N, H, W, Cinp, Ho, Wo, Coutp, k, S, pad, num_sm, &a)) return 0;
  return a.ksplit;
}

bool conv_wgrad_ts(const WgradSpec& w, cudaStream_t st) {
  int dev;
  PST_CUDA(cudaGetDevice(&dev));
  WtArgs a;
  if (!wgrad_ts_plan(w.N, w.H, w.W, w.Cinp, w.Ho, w.Wo, w.Coutp, w.k, w.S, w.pad, wgrad_sms(dev), &a)) return false;
  PST_CHECK_ARG(a.ksplit == w.ksplit, "wgrad: workspace planned for a different split");
  a.part = w.part;
  a.dbg = w.dbg;
  uint64_t xd[4] = {(uint64_t)w.W * kEPC, (uint64_t)w.H, (uint64_t)w.N, (uint64_t)w.Cinp / kEPC};
  uint64_t xs[3] = {(uint64_t)w.W * 16, (uint64_t)w.H * w.W * 16, (uint64_t)w.N * w.H * w.W * 16};
  uint32_t xb[4] = {(uint32_t)(a.band_c * kEPC), (uint32_t)a.band_r, (uint32_t)a.nb, (uint32_t)a.pl_grp};
  CUtensorMap tX = make_tmap(act_tmap_dtype(), 4, w.x, xd, xs, xb, nullptr);
  uint64_t dd[4] = {(uint64_t)w.Wo * kEPC, (uint64_t)w.Ho, (uint64_t)w.N, (uint64_t)w.Coutp / kEPC};
  uint64_t ds[3] = {(uint64_t)w.Wo * 16, (uint64_t)w.Ho * w.Wo * 16, (uint64_t)w.N * w.Ho * w.Wo * 16};
  uint32_t db[4] = {(uint32_t)(w.Wo * kEPC), (uint32_t)a.bh, (uint32_t)a.nb, (uint32_t)(a.BNw / kEPC)};
  CUtensorMap tD = make_tmap(act_tmap_dtype(), 4, w.dy, dd, ds, db, nullptr);
  const size_t smem = (size_t)a.SB * a.stage_bytes + 128 * 4 + (2 * kWtMaxSB + 2 * kWtMaxSlots + 1) * 8 + 16;
  PST_CHECK_ARG(smem <= 227 * 1024, "wgrad smem budget");
  using KernT = void (*)(const CUtensorMap, const CUtensorMap, const WtArgs);
  KernT kern = nullptr;
  {
    const KernT tab[2][2][4] = {
        {{conv_wgrad_ts_kernel<1, 16, 2>, conv_wgrad_ts_kernel<2, 16, 2>, conv_wgrad_ts_kernel<3, 16, 2>,
          conv_wgrad_ts_kernel<4, 16, 2>},
         {conv_wgrad_ts_kernel<1, 32, 2>, conv_wgrad_ts_kernel<2, 32, 2>, conv_wgrad_ts_kernel<3, 32, 2>,
          conv_wgrad_ts_kernel<4, 32, 2>}},
        {{conv_wgrad_ts_kernel<1, 16, 3>, conv_wgrad_ts_kernel<2, 16, 3>, conv_wgrad_ts_kernel<3, 16, 3>,
          conv_wgrad_ts_kernel<4, 16, 3>},
         {conv_wgrad_ts_kernel<1, 32, 3>, conv_wgrad_ts_kernel<2, 32, 3>, conv_wgrad_ts_kernel<3, 32, 3>,
          conv_wgrad_ts_kernel<4, 32, 3>}}};
    PST_CHECK_ARG((a.P16 == 16 || a.P16 == 32 || a.P16 == 64) && a.G >= 1 && a.G <= 4, "wgrad tiling");
    if (a.P16 == 64) {
      PST_CHECK_ARG(a.G <= 2, "wgrad tiling (64-pixel units)");
      const KernT t64[2][2] = {{conv_wgrad_ts_kernel<1, 64, 2>, conv_wgrad_ts_kernel<2, 64, 2>},
                               {conv_wgrad_ts_kernel<1, 64, 3>, conv_wgrad_ts_kernel<2, 64, 3>}};
      kern = t64[a.sets == 3 ? 1 : 0][a.G - 1];
    } else {
      kern = tab[a.sets == 3 ? 1 : 0][a.P16 == 32 ? 1 : 0][a.G - 1];
    }
  }
  PST_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = a.n_mgroups * a.n_ntiles * a.ksplit;
  const double es = sizeof(act_t);
  const double bytes = (double)w.N * w.H * w.W * w.Cinp * es + (double)w.N * w.Ho * w.Wo * w.Coutp * es +
                       (double)a.rows * w.Coutp * 4.0;   // algorithmic: X + dY read, dW written once
  const double flops = 2.0 * a.rows * (double)w.Coutp * w.N * w.Ho * w.Wo;
  prof::begin(st);
  PST_CUDA(launch_k(kern, dim3(grid), dim3(wt_threads(a.sets)), smem, st, tX, tD, a));
  PST_CUDA(cudaGetLastError());
  prof::end(st, prof::CONV_WGRAD, bytes, flops);
  return true;
}
#else
int wgrad_ts_ksplit(int, int, int, int, int, int, int, int, int, int, int) { return 0; }
bool conv_wgrad_ts(const WgradSpec&, cudaStream_t) { return false; }
#endif

}  // namespace pst
