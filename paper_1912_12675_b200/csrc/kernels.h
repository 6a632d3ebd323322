// kernels.h -- launch interfaces of the hand-written sm_100a kernels of libpst.
//
// Layouts:
//   activations / gradients : channel-planar act_t [Cp/EPC][N][H][W][EPC], channels padded
//                             to Cp = round_up(C, 16), EPC = 16 B / sizeof(act_t); a TMA box
//                             row is then a contiguous run of pixels of one 16-byte plane.
//   float tensors (logits, loss gradient): [Cp/4][N][H][W][4]
//   conv weight shadows     : fwd   [k*k][Cinp/EPC][Coutp][EPC]  (K-major B operand rows)
//                             dgrad [k*k][Coutp/EPC][Cinp][EPC]
//                             3xTF32 build: a lo plane (w - trunc_tf32(w)) follows each.
//   master weights          : canonical float32 (OIHW; an FC layer over a CxHxW tensor is
//                             the valid convolution with k = H = W) per stage
#pragma once
#include "common.h"

namespace pst {

enum EpiMode { EPI_BN_STATS = 0, EPI_BIAS_ACT = 1, EPI_BIAS_F32 = 2, EPI_DGRAD = 3 };

// One implicit-GEMM convolution on tcgen05 (forward, or dgrad expressed as a
// stride-1 correlation of dY with the flipped, transposed weights).
struct ConvSpec {
  // input tensor (NHWC act_t, channels Cinp), output grid and tensor
  const act_t* in; int N, H, W, Cinp;
  int Ho, Wo, Coutp, Cout;
  int k, S;                 // kernel size, input element stride
  int off, sgn;             // input coord = out*S + off + sgn*tap  (fwd: -pad,+1; dgrad: +pad,-1)
  int max_ctas;             // grid cap (0: all SMs) -- the dgrad shares the GPU with the forked wgrad
  const act_t* wshadow;     // [k*k][Coutp][Cinp]
  int epi;                  // EpiMode
  int relu;
  void* out;                // act_t or float NHWC [N][Ho][Wo][Coutp]
  const float* bias;        // [Cout] or null
  double* stats;            // [Coutp][2] (EPI_BN_STATS), accumulated with atomics
  const act_t* res;         // EPI_DGRAD residual gradient (identity or option A) or null
  int res_mode;             // 0 none, 1 identity, 2 option A
  int res_H, res_W, res_C, res_pad;
  // EPI_DGRAD with bfuse: the output is the NEXT-lower layer's pre-activation gradient (the work
  // of bwd_pre fused into the epilogue): gpre = relu'(bz) * (dgrad + res) is written to `out`,
  // and sums[c] += (sum gpre, sum gpre * (by - mean) * invstd) with bsaved = (mean, invstd)
  const act_t* bz; const act_t* by; const float* bsaved; double* bsums;
  int bfuse, brelu, bbn;
  float bscale;             // fused bwd_pre: dropout scale of the lower layer where z > 0 (0 = 1)
  unsigned long long* dbg;  // optional device timeline buffer [8][256] (CTA 0), debug only
  // Band pre-pass (TS kernel only): the per-element BatchNorm step that produces this conv's
  // input is done on the input band in shared memory after its TMA load, before the taps read it,
  // instead of by a separate kernel; the transformed tensor is also written to `pre_out` for the
  // tile's own input rows (every element exactly once), for the consumers that need it later.
  //   pre 1 (forward, BN apply of the producing layer): `in` is that layer's conv output y;
  //         x = relu?( gamma*(y-mean)*invstd + beta [+ pre_res] ), mean/invstd from pre_stats
  //         (sum, sumsq over M values); CTA 0 writes pre_saved = (mean, invstd) and the running stats.
  //   pre 2 (dgrad, BN backward of this layer): `in` is the pre-activation gradient gpre;
  //         gy = gamma*invstd*(gpre - S1/M - xhat*S2/M), xhat = (pre_y - mean)*invstd,
  //         (mean, invstd) = pre_saved, (S1, S2) = pre_stats.
  // Positions outside the image are zero after the transform (the conv's zero padding).
  int pre, pre_relu, pre_C;
  const act_t* pre_res;     // pre 1: identity shortcut of the producer's block (shape of `in`) or null
  const act_t* pre_y;       // pre 2: this layer's BN input y
  const double* pre_stats;
  const float* pre_gamma; const float* pre_beta;
  float* pre_saved;
  float* pre_run_mean; float* pre_run_var;
  float pre_momentum, pre_eps;
  act_t* pre_out;
};
void conv_tc(const ConvSpec& c, cudaStream_t st);
// TS-mode variant (A operand in tensor memory, 3xTF32 build); returns false if the shape
// does not fit its tiling (conv_tc then runs the smem-operand kernel).
bool conv_ts(const ConvSpec& c, cudaStream_t st);
bool conv_ts_fits(const ConvSpec& c);   // conv_ts would take this shape

// Weight gradient dW[tap*Cinp+ci][co] = sum_pixels X(shifted by tap)[p][ci] * dY[p][co],
// split over pixel ranges: part[ks][rows][Coutp] float32 (reduced by sgd_update).
struct WgradSpec {
  const act_t* x; int N, H, W, Cinp;
  const act_t* dy; int Ho, Wo, Coutp;
  int k, S, pad;
  float* part;              // workspace, ksplit * rows * Coutp floats
  int ksplit;               // chosen by wgrad_plan
  unsigned long long* dbg;  // optional device timeline buffer [8][256] (CTA 0), debug only
};
struct WgradPlan { int ksplit; int64_t part_floats; };
WgradPlan wgrad_plan(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad, int num_sm);
void conv_wgrad_tc(const WgradSpec& w, cudaStream_t st);
// TS-mode wgrad (expanded input operand in TMEM, 3xTF32 build): false if the shape does not fit;
// wgrad_ts_ksplit() is its split-K factor (0 if it does not apply).
bool conv_wgrad_ts(const WgradSpec& w, cudaStream_t st);
int wgrad_ts_ksplit(int N, int H, int W, int Cinp, int Ho, int Wo, int Coutp, int k, int S, int pad, int num_sm);

// ---------------------------------------------------------------- elementwise / reductions
// NCHW float32 -> channel-planar act_t, channels zero-padded to Cp.
void input_to_act(const float* x, act_t* out, int N, int C, int H, int W, int Cp, cudaStream_t st);

// BN forward apply (train mode): batch stats from `stats` (sum, sumsq over M values),
// z = relu?( gamma*(y-mean)*invstd + beta + shortcut(block) ).  Block 0 also writes
// saved[c] = (mean, invstd) and updates running statistics.
struct BnApplySpec {
  const act_t* y; act_t* z; int N, H, W, Cp, C;
  const double* stats; const float* gamma; const float* beta;
  float* saved;             // [Cp][2] mean, invstd
  float* run_mean; float* run_var;
  float momentum, eps;
  int relu;
  // forward shortcut: res [N][res_H][res_W][res_C] (res_C = padded channels, res_Creal real);
  // identity (mode 1) or option A (mode 2): out channel c reads res channel c - res_pad at (2y, 2x)
  const act_t* res; int res_mode; int res_H, res_W, res_C, res_Creal, res_pad;
};
void bn_apply(const BnApplySpec& s, cudaStream_t st);

// Bias + ReLU forward for convs/FCs without BN is fused in the conv epilogue.

// 2x2/2 max-pool: out [N][H/2][W/2][Cp], arg uint8 (window index 0..3, first max).
void maxpool2_fwd(const act_t* in, act_t* out, uint8_t* arg, int N, int H, int W, int Cp, cudaStream_t st);
// Global average pool: [N][H][W][Cp] -> [N][Cp]
void gap_fwd(const act_t* in, act_t* out, int N, int H, int W, int Cp, cudaStream_t st);

// Backward "pre" kernel for one layer's non-weighted tail, reading the gradient
// w.r.t. the layer's (pooled) output:
//   g_z  = pool^T(g_out)           (none / max2 via arg / gap broadcast / H*W)
//   gpre = g_z * (z > 0)           if relu
//   if bn: accumulate sums[c] += (sum gpre, sum gpre*xhat), xhat = (y-mean)*invstd
//   else : accumulate sums[c] += (sum gpre, 0)   (bias gradient)
// gpre written as act_t [N][H][W][Cp].
struct BwdPreSpec {
  const act_t* gout; int pool; const uint8_t* arg;  // pool: 0 none, 1 max2, 2 gap
  const act_t* z; int relu;
  float rscale;             // where z > 0: the layer's dropout scale 1/(1-p), else 1
  const act_t* y; const float* saved; int bn;
  act_t* gpre; int N, H, W, Cp, C;
  double* sums;             // [Cp][2]
  int gout_f32;             // gout is float (loss gradient) instead of act_t
};
void bwd_pre(const BwdPreSpec& s, cudaStream_t st);

// Counter-based inverted dropout in place on z (reading AMB-16b); fmb: device counter
// holding the mini-batch index of the running forward.
void dropout_fwd(act_t* z, int N, int H, int W, int Cp, int C, uint32_t seed, int layer, uint32_t thresh, float scale,
                 const int64_t* fmb, cudaStream_t st);
void counter_inc(int64_t* c, cudaStream_t st);

// BN backward apply: gy = gamma_cur*invstd/M * (M*gpre - S1 - xhat*S2)
struct BnBwdSpec {
  const act_t* gpre; const act_t* y; const float* saved; const double* sums;
  const float* gamma; act_t* gy; int N, H, W, Cp, C;
};
void bn_bwd_apply(const BnBwdSpec& s, cudaStream_t st);

// Zero-insertion of a stride-2 gradient: dyd[n][2y][2x][c] = dy[n][y][x][c], else 0.
void dilate2(const act_t* dy, act_t* dyd, int N, int Ho, int Wo, int H, int W, int Cp, cudaStream_t st);

// Softmax cross-entropy over logits [B][Cp] (first C columns): loss (mean) into
// loss_ring[(*fwd_counter) % ring], dz = (softmax - onehot)/B as float [B][Cp]
// (padded columns 0).  Labels come from label_ring[(*fwd_counter) % ring][B].
// Increments *fwd_counter.
void softmax_ce(const float* logits, const int32_t* label_ring, int ring, float* loss_ring,
                int64_t* fwd_counter, float* dz, int B, int C, int Cp, cudaStream_t st);

// ---------------------------------------------------------------- optimiser
// One SGD-momentum update of a whole stage (PyTorch form): for every canonical
// parameter, g = (wgrad partial sum | BN/bias double sums | grad buffer),
// v = mu v + (g + lambda w), w -= lr v, plus the act_t weight shadows.
// lr = (v_count < n_p ? lr_pipe : lr_np) * gamma^(#milestones <= v_count/spe);
// the kernel reads and then increments *v_count.
enum SegKind { SEG_CONVW = 0, SEG_VEC = 2 };
struct SgdSeg {
  int kind;
  int64_t off;              // canonical offset in the stage's flat parameter vector
  int64_t n;                // elements
  // SEG_CONVW (an FC layer over a CxHxW input is the valid conv with k = H)
  int cout, cin, k;         // canonical dims
  int Coutp, Cinp;          // padded GEMM dims
  const float* part; int ksplit;  // wgrad partials [ksplit][k*k*Cinp][Coutp]
  float* gsum;              // reduced gradient [k*k*Cinp][Coutp] (written by the reduce pass)
  act_t* sh_fwd;            // [k*k][Coutp][Cinp]
  act_t* sh_bwd;            // [k*k][Cinp][Coutp]
  // SEG_VEC: gradient = src_d[c*2 + comp] (double sums) for c < n
  const double* src_d; int comp;
};
struct SgdSpec {
  float* w; float* v;       // stage flat fp32
  const SgdSeg* segs;       // device array
  int n_segs;
  const int64_t* seg_block_start;  // device: first block of each segment (prefix), n_segs+1
  int64_t total_blocks;
  int64_t* v_count;         // device version counter of the stage
  int* ticket;              // device, for last-block increment
  const float* lr_pipe;     // device scalar: this stage's pipelined lr
  float lr_np, momentum, wd, gamma;
  const int64_t* milestones; int n_ms; int64_t spe;
  const int64_t* n_p;       // device scalar: hybrid switch mini-batch (huge if none)
  int solver, nesterov, lr_policy;   // pst_hparams solver variants (0: PyTorch form, 1: Caffe)
  float inv_gamma, inv_power;
  // split-K reduction pass (one launch for all conv segments, coalesced float4 over [rows][Coutp])
  const int64_t* red_block_start;  // device: first reduce block of each segment (0 blocks for non-conv)
  int64_t red_total_blocks;
};
void sgd_update(const SgdSpec& s, cudaStream_t st);
// Writes the shadows from the master weights only (used at create / import).
void build_shadows(const SgdSpec& s, cudaStream_t st);

}  // namespace pst

namespace pst {
// ---------------------------------------------------------------- test/debug helpers (ops ABI)
void act_to_nchw(const void* in, int in_f32, float* out, int N, int C, int H, int W, cudaStream_t st);
void conv_weights_to_shadows(const float* w, int cout, int cin, int k, int Coutp, int Cinp, act_t* sh_fwd,
                             act_t* sh_bwd, cudaStream_t st);
void wgrad_reduce(const float* part, int ksplit, int Coutp, int Cinp, int cout, int cin, int k, float* out,
                  cudaStream_t st);
}  // namespace pst
