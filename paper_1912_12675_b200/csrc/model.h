// model.h -- network description, derived shapes, canonical parameter offsets,
// PPV partition (reading AMB-13/14) and the step schedule
// (PAPER.md L61/L63/L75, reading AMB-1).  Host only; no CUDA calls.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/pst.h"

namespace pst {

struct LayerInfo {
  pst_layer spec;
  int idx = 0;
  // input tensor (NCHW geometry of what arrives; for FC the pre-flatten tensor)
  int in_C = 0, in_H = 0, in_W = 0, in_Cp = 0;
  // GEMM view: every weighted layer is a convolution over the input tensor; an FC
  // layer over a CxHxW tensor is the valid convolution with kk = H = W (its
  // canonical [out][c*H*W + y*W + x] weights are exactly OIHW).
  int kk = 1, S = 1, pad = 0;
  int Cinp = 0;             // K channels per tap = in_Cp
  int Ho = 0, Wo = 0;       // conv output spatial (FC: 1x1)
  int Coutp = 0;            // padded output channels
  // the layer's output tensor (after pool): next layer's input
  int out_C = 0, out_H = 0, out_W = 0;
  // canonical parameter offsets (global, in floats); -1 if absent
  int64_t off_W = -1, off_b = -1, off_g = -1, off_be = -1;
  int64_t n_W = 0;
  int64_t p_begin = 0, p_end = 0;  // canonical range of this layer
  int block_src = -1;       // layer whose input is the residual block input (for residual layers)
  int block_end = -1;       // for block_begin layers: the residual layer closing the block
  int res_mode = 0;         // residual layers: 1 identity, 2 option A
  int res_pad = 0;          // option A channel pad
  int bn_index = -1;        // order among BN layers (for running-stat export)
};

struct NetInfo {
  std::vector<LayerInfo> layers;
  int in_C = 0, in_H = 0, in_W = 0, in_Cp = 0;
  int n_classes = 0;
  int64_t n_params = 0;
  int n_bn = 0;
};

// Throws InvalidArg / Unsupported on a bad description.
NetInfo derive_net(const pst_net& net);

// Validated stage ranges [start, end) (0-based layer indices).
std::vector<std::pair<int, int>> partition(const NetInfo& net, int K, const int32_t* ppv);

// Schedule of global step t (pipelined mode), relative to a fill that started at
// step t0 with mini-batch m0, with n_fed mini-batches fed so far:
//   backward mini-batch b = m0 + (t-t0) - 2K + 1 + s   (runs first, AMB-1)
//   forward  mini-batch f = m0 + (t-t0) - s
// each valid only in [m0, n_fed); -1 otherwise.
struct StepPlan { int64_t bwd_mb = -1, fwd_mb = -1; };
StepPlan plan_step(int K, int s, int64_t t, int64_t t0, int64_t m0, int64_t n_fed);

// Saved-activation / input ring slots per stage.  Stage s keeps the saved forward state of the
// mini-batches between its forward (step f+s) and its backward (step f+2K-1-s): 2(K-s)-1 of them
// right after a forward (the paper's activation storage), plus 2 so a forward never
// overwrites an input slot the neighbour's copy of the same step is writing or an in-flight read
// still needs: need_s = 2(K-s)+1.  Every R_s is a divisor of one common period P = 2K+2 (the
// smallest divisor >= need_s), so all ring indices and the gradient-buffer parity cycle with
// period P and a stage needs at most P distinct step graphs (arbitrary per-stage sizes 2(K-s)+1
// would make the graph key cycle with lcm(2, R_s, R_{s+1}): 6630 step graphs for the second stage
// of an 8-stage pipeline).  K=8: 18,18,18,18,9,9,6,3 slots instead of 18 on every stage.
inline int ring_need(int K, int s) { return 2 * (K - s) + 1; }
inline int ring_period(int K) { return 2 * K + 2; }
inline int ring_slots(int K, int s) {
  const int P = ring_period(K), need = ring_need(K, s);
  for (int d = need; d < P; ++d)
    if (P % d == 0) return d;
  return P;
}

}  // namespace pst
