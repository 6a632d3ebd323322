// model.cpp -- network derivation, partition, schedule (host only).
#include "model.h"

#include <algorithm>

#include "common.h"

namespace pst {

static int rup16(int c) { return (c + 15) / 16 * 16; }

NetInfo derive_net(const pst_net& net) {
  PST_CHECK_ARG(net.n_layers >= 1 && net.layers != nullptr, "net has no layers");
  PST_CHECK_ARG(net.in_c >= 1 && net.in_h >= 1 && net.in_w >= 1, "bad input shape");
  NetInfo ni;
  ni.in_C = net.in_c; ni.in_H = net.in_h; ni.in_W = net.in_w; ni.in_Cp = rup16(net.in_c);
  ni.n_classes = net.n_classes;
  int C = net.in_c, H = net.in_h, W = net.in_w;
  int64_t off = 0;
  int open_block = -1;
  bool spatial = true;  // tensor still 4-D (no GAP / FC yet)
  for (int i = 0; i < net.n_layers; ++i) {
    const pst_layer& L = net.layers[i];
    LayerInfo li;
    li.spec = L;
    li.idx = i;
    li.in_C = C; li.in_H = H; li.in_W = W; li.in_Cp = rup16(C);
    const std::string at = "layer " + std::to_string(i + 1) + ": ";
    PST_CHECK_ARG(L.cout >= 1, at + "cout");
    PST_CHECK_ARG(L.pool >= 0 && L.pool <= 2, at + "pool");
    if (L.kind == PST_LAYER_CONV) {
      PST_CHECK_ARG(spatial, at + "conv after GAP/FC");
      PST_CHECK_ARG(L.cin == C, at + "conv cin does not match the incoming tensor");
      PST_CHECK_ARG(L.k >= 1 && L.k <= 7 && L.pad >= 0 && L.pad < L.k, at + "conv k/pad");
      PST_CHECK_ARG(L.stride == 1 || L.stride == 2, at + "stride must be 1 or 2");
      li.Cinp = li.in_Cp;
      li.kk = L.k; li.S = L.stride; li.pad = L.pad;
      li.Ho = (H + 2 * L.pad - L.k) / L.stride + 1;
      li.Wo = (W + 2 * L.pad - L.k) / L.stride + 1;
      PST_CHECK_ARG(li.Ho >= 1 && li.Wo >= 1, at + "empty conv output");
      if (L.stride == 2)
        PST_CHECK_ARG(L.k == 3 && L.pad == 1, at + "stride-2 conv supported for k=3, pad=1");
    } else if (L.kind == PST_LAYER_FC) {
      PST_CHECK_ARG(L.cin == C * H * W, at + "FC cin must equal C*H*W of the incoming tensor");
      PST_CHECK_ARG(H == W && H <= 7, at + "FC input must be square with H <= 7 (valid-conv view)");
      li.Cinp = li.in_Cp;
      li.kk = H; li.S = 1; li.pad = 0;
      li.Ho = li.Wo = 1;
    } else {
      throw InvalidArg(at + "unknown layer kind");
    }
    li.Coutp = rup16(L.cout);
    if (L.bias && L.bn) throw Unsupported(at + "bias followed by BatchNorm");
    PST_CHECK_ARG(L.dropout >= 0.f && L.dropout < 1.f, at + "dropout must be in [0, 1)");
    if (L.dropout > 0.f) PST_CHECK_ARG(L.relu, at + "dropout needs a ReLU before it (build restriction)");
    if (L.residual) {
      PST_CHECK_ARG(open_block >= 0, at + "residual without an open block");
      PST_CHECK_ARG(L.bn, at + "residual layers must have BN (build restriction)");
      PST_CHECK_ARG(L.kind == PST_LAYER_CONV, at + "residual on FC");
      const LayerInfo& src = ni.layers[open_block];
      li.block_src = open_block;
      if (src.in_C == L.cout && src.in_H == li.Ho && src.in_W == li.Wo) {
        li.res_mode = 1;
      } else {
        PST_CHECK_ARG(src.in_H == 2 * li.Ho && src.in_W == 2 * li.Wo && L.cout > src.in_C &&
                          (L.cout - src.in_C) % 2 == 0,
                      at + "residual shapes incompatible with identity or option-A shortcut");
        li.res_mode = 2;
        li.res_pad = (L.cout - src.in_C) / 2;
      }
      ni.layers[open_block].block_end = i;
      open_block = -1;
    }
    if (L.block_begin) {
      PST_CHECK_ARG(open_block < 0, at + "nested residual block");
      open_block = i;
    }
    // parameters
    li.p_begin = off;
    li.off_W = off;
    li.n_W = (int64_t)L.cout * L.cin * (L.kind == PST_LAYER_CONV ? L.k * L.k : 1);
    off += li.n_W;
    if (L.bias) { li.off_b = off; off += L.cout; }
    if (L.bn) {
      li.off_g = off; off += L.cout;
      li.off_be = off; off += L.cout;
      li.bn_index = ni.n_bn++;
    }
    li.p_end = off;
    // output tensor
    C = L.cout;
    H = li.Ho; W = li.Wo;
    if (L.pool == PST_POOL_MAX2) {
      PST_CHECK_ARG(L.kind == PST_LAYER_CONV && H % 2 == 0 && W % 2 == 0, at + "max-pool needs even H, W");
      H /= 2; W /= 2;
    } else if (L.pool == PST_POOL_GAP) {
      PST_CHECK_ARG(L.kind == PST_LAYER_CONV, at + "GAP after FC");
      H = 1; W = 1;
      spatial = false;
    }
    if (L.kind == PST_LAYER_FC) spatial = false;
    li.out_C = C; li.out_H = H; li.out_W = W;
    ni.layers.push_back(li);
  }
  PST_CHECK_ARG(open_block < 0, "unterminated residual block");
  const LayerInfo& last = ni.layers.back();
  PST_CHECK_ARG(last.spec.kind == PST_LAYER_FC && !last.spec.relu && !last.spec.bn && last.spec.pool == 0,
                "the last layer must be a plain FC producing the logits");
  PST_CHECK_ARG(last.spec.cout == net.n_classes, "last layer cout must equal n_classes");
  PST_CHECK_ARG(net.n_classes >= 2, "n_classes");
  ni.n_params = off;
  return ni;
}

std::vector<std::pair<int, int>> partition(const NetInfo& net, int K, const int32_t* ppv) {
  const int L = (int)net.layers.size();
  PST_CHECK_ARG(K >= 1 && K <= L, "n_stages must be in [1, n_layers]");
  std::vector<int> b = {0};
  for (int i = 0; i < K - 1; ++i) {
    PST_CHECK_ARG(ppv != nullptr, "ppv missing");
    const int p = ppv[i];
    PST_CHECK_ARG(p >= 1 && p <= L - 1, "PPV entries must be in [1, n_layers-1]");
    PST_CHECK_ARG(p > b.back(), "PPV must be strictly increasing");
    b.push_back(p);
  }
  b.push_back(L);
  // A boundary may fall inside a residual block (mid-block register pair, reading
  // AMB-14): the register then carries the block input beside the activation (forward) and the
  // shortcut gradient beside the input gradient (backward).  Build restriction: at most one
  // boundary inside any block (every block of the supported nets has two weighted layers).
  for (int j = 0; j < L; ++j) {
    const LayerInfo& li = net.layers[j];
    if (!li.spec.block_begin || li.block_end < 0) continue;
    int inside = 0;
    for (size_t i = 1; i + 1 < b.size(); ++i)
      if (b[i] > j && b[i] <= li.block_end) ++inside;
    if (inside > 1)
      throw Unsupported("more than one PPV boundary inside the residual block of layers " + std::to_string(j + 1) +
                        ".." + std::to_string(li.block_end + 1));
  }
  std::vector<std::pair<int, int>> r;
  for (int s = 0; s < K; ++s) r.push_back({b[s], b[s + 1]});
  return r;
}

StepPlan plan_step(int K, int s, int64_t t, int64_t t0, int64_t m0, int64_t n_fed) {
  StepPlan p;
  const int64_t rel = t - t0;
  const int64_t b = m0 + rel - 2 * K + 1 + s;
  const int64_t f = m0 + rel - s;
  p.bwd_mb = (b >= m0 && b < n_fed) ? b : -1;
  p.fwd_mb = (f >= m0 && f < n_fed) ? f : -1;
  return p;
}

}  // namespace pst
