// stage.cu -- buffers and launch program of one pipeline stage.
#include "stage.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace pst {

// Timing experiments only (PST_SKIP=fwd,bnapply,bwdpre,bnbwd,wgrad,dgrad,sgd): leave a kernel class
// out of the step to measure its in-graph cost.  Results are wrong when set.
static bool side_wgrad() {
  static const bool on = pst_knob("PST_WSTREAM", 1) != 0;
  // the per-kernel event profile (pst_profile) times launches one at a time: a wgrad running
  // beside the dgrad would be charged the time it waits for SMs
  return on && !prof::enabled;
}
static bool skip(const char* cls) {
#ifdef PST_EXPERIMENTS
  static const char* env = std::getenv("PST_SKIP");
  return env != nullptr && std::strstr(env, cls) != nullptr;
#else
  (void)cls;
  return false;
#endif
}

// Dropout threshold and scale from the float32 probability (pst.h pst_layer.dropout).
static uint32_t drop_thresh(float p) {
  const double t = std::floor((double)p * 4294967296.0);
  return t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
}
static float drop_scale(float p) { return (float)(1.0 / (1.0 - (double)p)); }

template <typename T>
T* Stage::alloc(size_t n, bool zero) {
  void* p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) throw CudaError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
  allocs_.push_back(p);
  bytes_total += n * sizeof(T);
  if (zero) PST_CUDA(cudaMemset(p, 0, n * sizeof(T)));
  return static_cast<T*>(p);
}

Stage::Stage(const NetInfo& net, int s_, int K_, int l0_, int l1_, int device, const pst_hparams& hp,
             const float* init_params, int batch)
    : s(s_), K(K_), l0(l0_), l1(l1_), dev(device), R(ring_saved(K_, s_)), Rin(ring_input(K_, s_)), batch_(batch),
      net_(net) {
  PST_CUDA(cudaSetDevice(dev));
  PST_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  PST_CUDA(cudaStreamCreateWithFlags(&wstream, cudaStreamNonBlocking));
  PST_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  PST_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  PST_CUDA(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
  PST_CUDA(cudaEventCreateWithFlags(&ev_cb, cudaEventDisableTiming));
  PST_CUDA(cudaEventCreateWithFlags(&ev_cf, cudaEventDisableTiming));
  PST_CUDA(cudaEventCreateWithFlags(&ev_cj, cudaEventDisableTiming));
  const int B = batch;
  const int nsm = num_sms(dev);
  p_base = net.layers[l0].p_begin;
  n_params = net.layers[l1 - 1].p_end - p_base;
  w_ = alloc<float>(n_params);
  v_ = alloc<float>(n_params);
  PST_CUDA(cudaMemcpy(w_, init_params + p_base, n_params * sizeof(float), cudaMemcpyHostToDevice));
  dseed_ = hp.dropout_seed;
  for (int l = l0; l < l1; ++l) has_drop_ = has_drop_ || net.layers[l].spec.dropout > 0.f;
  if (has_drop_) d_fmb_ = alloc<int64_t>(1);   // mini-batch index of the running forward (dropout masks)

  // mid-block registers: the block open across each end of the stage
  for (int l = 0; l < l0; ++l)
    if (net.layers[l].spec.block_begin && net.layers[l].block_end >= l0) start_res_ = net.layers[l].block_end;
  for (int l = l0; l < l1; ++l)
    if (net.layers[l].spec.block_begin && net.layers[l].block_end >= l1) end_block_ = l;
  // input ring of the stage
  const LayerInfo& f0 = net.layers[l0];
  for (int r = 0; r < Rin; ++r) xin_.push_back(alloc<act_t>((size_t)B * f0.in_H * f0.in_W * f0.in_Cp));
  bytes_slot += (size_t)B * f0.in_H * f0.in_W * f0.in_Cp * sizeof(act_t);
  if (starts_mid()) {
    const LayerInfo& src = net.layers[net.layers[start_res_].block_src];
    for (int r = 0; r < Rin; ++r) xin2_.push_back(alloc<act_t>((size_t)B * src.in_H * src.in_W * src.in_Cp));
    bytes_slot += (size_t)B * src.in_H * src.in_W * src.in_Cp * sizeof(act_t);
  }
  if (is_first()) xstage_ = alloc<float>((size_t)B * net.in_C * net.in_H * net.in_W);

  // per-layer buffers
  size_t nrun = 0;
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& li = net.layers[l];
    if (li.spec.bn) { run_off_.push_back((int64_t)nrun); nrun += 2 * li.Coutp; }
    fwd_arena_n_ += li.spec.bn ? 2 * li.Coutp : 0;
    bwd_arena_n_ += 2 * li.Coutp;
  }
  run_ = alloc<float>(std::max<size_t>(nrun, 1));
  {
    std::vector<float> init(std::max<size_t>(nrun, 1), 0.f);
    for (int l = l0, b = 0; l < l1; ++l) {
      const LayerInfo& li = net.layers[l];
      if (!li.spec.bn) continue;
      for (int c = 0; c < li.Coutp; ++c) init[run_off_[b] + li.Coutp + c] = 1.f;  // running var = 1
      ++b;
    }
    PST_CUDA(cudaMemcpy(run_, init.data(), init.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  fwd_arena_ = alloc<double>(fwd_arena_n_);
  bwd_arena_ = alloc<double>(bwd_arena_n_);
  size_t fo = 0, bo = 0;
  L_.resize(l1 - l0);
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& li = net.layers[l];
    LayerBufs& b = L_[l - l0];
    const size_t out_el = (size_t)B * li.Ho * li.Wo * li.Coutp;
    const bool last_net = (l == (int)net.layers.size() - 1);
    const size_t before_ring = bytes_total;
    b.y_bytes = li.spec.bn ? out_el * sizeof(act_t) : 0;
    b.z_bytes = last_net ? out_el * sizeof(float) : out_el * sizeof(act_t);
    b.p_bytes = li.spec.pool == PST_POOL_MAX2 ? out_el / 4 * sizeof(act_t)
              : li.spec.pool == PST_POOL_GAP ? (size_t)B * li.Coutp * sizeof(act_t) : 0;
    b.arg_bytes = li.spec.pool == PST_POOL_MAX2 ? out_el / 4 : 0;
    b.saved_bytes = li.spec.bn ? 2 * li.Coutp * sizeof(float) : 0;
    for (int r = 0; r < R; ++r) {
      if (li.spec.bn) b.y.push_back(alloc<act_t>(out_el, false));
      if (last_net) b.zf.push_back(alloc<float>(out_el));
      else b.z.push_back(alloc<act_t>(out_el, false));
      if (li.spec.pool == PST_POOL_MAX2) {
        b.p.push_back(alloc<act_t>(out_el / 4, false));
        b.arg.push_back(alloc<uint8_t>(out_el / 4, false));
      } else if (li.spec.pool == PST_POOL_GAP) {
        b.p.push_back(alloc<act_t>((size_t)B * li.Coutp, false));
      }
      if (li.spec.bn) b.saved.push_back(alloc<float>(2 * li.Coutp));
    }
    bytes_slot += (bytes_total - before_ring) / R;
    b.gpre = alloc<act_t>(out_el, false);
    if (li.spec.bn) b.gy = alloc<act_t>(out_el, false);
    const bool need_gin = !(is_first() && l == l0);
    if (need_gin) b.gin = alloc<act_t>((size_t)B * li.in_H * li.in_W * li.in_Cp, false);
    if (li.S == 2 && need_gin)
      b.dil = alloc<act_t>((size_t)B * li.in_H * li.in_W * li.Coutp, false);
    const int kk = li.kk;
    WgradPlan wp = wgrad_plan(B, li.in_H, li.in_W, li.Cinp, li.Ho, li.Wo, li.Coutp, kk, li.S, li.pad, wgrad_sms(dev));
    b.ksplit = wp.ksplit;
    b.wpart = alloc<float>((size_t)wp.part_floats, false);
    // weight shadows (+ the 3xTF32 lo plane right after the raw plane in the split build)
    b.sh_fwd = alloc<act_t>((size_t)kk * kk * li.Coutp * li.Cinp * (PST_SPLIT ? 2 : 1));
    b.sh_bwd = alloc<act_t>((size_t)kk * kk * li.Coutp * li.Cinp * (PST_SPLIT ? 2 : 1));
    if (li.spec.bn) { b.stats = fwd_arena_ + fo; fo += 2 * li.Coutp; }
    b.sums = bwd_arena_ + bo; bo += 2 * li.Coutp;
  }
  const LayerInfo& lastl = net.layers[l1 - 1];
  if (!is_last()) {
    const size_t ob = (size_t)B * lastl.out_H * lastl.out_W * ((lastl.out_C + 15) / 16 * 16);
    dbuf_[0] = alloc<act_t>(ob);
    dbuf_[1] = alloc<act_t>(ob);
    if (ends_mid()) {
      dbuf2_[0] = alloc<act_t>(dbuf2_bytes() / sizeof(act_t));
      dbuf2_[1] = alloc<act_t>(dbuf2_bytes() / sizeof(act_t));
    }
  } else {
    label_ring_n_ = 2 * K + 2;
    label_ring_ = alloc<int32_t>((size_t)label_ring_n_ * B);
    loss_ring_ = alloc<float>(1024);
    fwd_counter_ = alloc<int64_t>(1);
    dz_ = alloc<float>((size_t)B * lastl.Coutp);
  }

  // ---- optimiser segments
  std::vector<SgdSeg> segs;
  std::vector<int64_t> starts, rstarts;
  int64_t blocks = 0, rblocks = 0;
  auto add = [&](SgdSeg g) {
    starts.push_back(blocks);
    rstarts.push_back(rblocks);
    blocks += (g.n + 255) / 256;
    if (g.kind == SEG_CONVW) rblocks += ((int64_t)g.k * g.k * g.Cinp * g.Coutp / 4 + 255) / 256;
    segs.push_back(g);
  };
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& li = net.layers[l];
    LayerBufs& b = L_[l - l0];
    SgdSeg g{};
    g.off = li.off_W - p_base;
    g.n = li.n_W;
    g.cout = li.spec.cout;
    g.cin = li.spec.cin;
    g.Coutp = li.Coutp;
    g.Cinp = li.Cinp;
    g.part = b.wpart;
    g.ksplit = b.ksplit;
    g.gsum = alloc<float>((size_t)li.kk * li.kk * li.Cinp * li.Coutp);
    g.sh_fwd = b.sh_fwd;
    g.sh_bwd = b.sh_bwd;
    g.kind = SEG_CONVW;   // FC over CxHxW = valid conv with k = H (canonical [o][c*H*W+y*W+x] == OIHW)
    g.k = li.kk;
    g.cin = li.in_C;
    add(g);
    if (li.spec.bias) {
      SgdSeg v{}; v.kind = SEG_VEC; v.off = li.off_b - p_base; v.n = li.spec.cout; v.src_d = b.sums; v.comp = 0;
      add(v);
    }
    if (li.spec.bn) {
      SgdSeg gg{}; gg.kind = SEG_VEC; gg.off = li.off_g - p_base; gg.n = li.spec.cout; gg.src_d = b.sums; gg.comp = 1;
      add(gg);
      SgdSeg bb{}; bb.kind = SEG_VEC; bb.off = li.off_be - p_base; bb.n = li.spec.cout; bb.src_d = b.sums; bb.comp = 0;
      add(bb);
    }
  }
  starts.push_back(blocks);
  rstarts.push_back(rblocks);
  d_red_start_ = alloc<int64_t>(rstarts.size());
  PST_CUDA(cudaMemcpy(d_red_start_, rstarts.data(), rstarts.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  d_segs_ = alloc<SgdSeg>(segs.size());
  PST_CUDA(cudaMemcpy(d_segs_, segs.data(), segs.size() * sizeof(SgdSeg), cudaMemcpyHostToDevice));
  d_seg_start_ = alloc<int64_t>(starts.size());
  PST_CUDA(cudaMemcpy(d_seg_start_, starts.data(), starts.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  d_vcount_ = alloc<int64_t>(1);
  d_ticket_ = alloc<int>(1);
  d_lr_ = alloc<float>(1);
  PST_CUDA(cudaMemcpy(d_lr_, &hp.lr_pipelined[s], sizeof(float), cudaMemcpyHostToDevice));
  d_np_ = alloc<int64_t>(1);
  set_n_p(INT64_MAX);
  d_ms_ = alloc<int64_t>(std::max(1, hp.n_milestones));
  if (hp.n_milestones > 0)
    PST_CUDA(cudaMemcpy(d_ms_, hp.milestone_epochs, hp.n_milestones * sizeof(int64_t), cudaMemcpyHostToDevice));
  sgd_.w = w_;
  sgd_.v = v_;
  sgd_.segs = d_segs_;
  sgd_.n_segs = (int)segs.size();
  sgd_.seg_block_start = d_seg_start_;
  sgd_.total_blocks = blocks;
  sgd_.red_block_start = d_red_start_;
  sgd_.red_total_blocks = rblocks;
  sgd_.v_count = d_vcount_;
  sgd_.ticket = d_ticket_;
  sgd_.lr_pipe = d_lr_;
  sgd_.lr_np = hp.lr_nonpipelined;
  sgd_.momentum = hp.momentum;
  sgd_.wd = hp.weight_decay;
  sgd_.gamma = hp.gamma;
  sgd_.milestones = d_ms_;
  sgd_.n_ms = hp.n_milestones;
  sgd_.spe = hp.steps_per_epoch > 0 ? hp.steps_per_epoch : INT64_MAX;
  sgd_.n_p = d_np_;
  sgd_.solver = hp.solver;
  sgd_.nesterov = hp.nesterov;
  sgd_.lr_policy = hp.lr_policy;
  sgd_.inv_gamma = hp.inv_gamma;
  sgd_.inv_power = hp.inv_power;
  build_shadows(sgd_, stream);
  PST_CUDA(cudaStreamSynchronize(stream));
  for (int l = l0, b = 0; l < l1; ++l) bn_idx_.push_back(net.layers[l].spec.bn ? b++ : -1);
  plan_fusion();
}

Stage::~Stage() {
  cudaSetDevice(dev);
  if (stream) cudaStreamSynchronize(stream);
  if (wstream) cudaStreamSynchronize(wstream);
  for (void* p : allocs_) cudaFree(p);
  if (stream) cudaStreamDestroy(stream);
  if (wstream) cudaStreamDestroy(wstream);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (cstream) { cudaStreamSynchronize(cstream); cudaStreamDestroy(cstream); }
  for (cudaEvent_t e : {ev_cb, ev_cf, ev_cj})
    if (e) cudaEventDestroy(e);
}

void Stage::set_n_p(int64_t n_p) {
  PST_CUDA(cudaSetDevice(dev));
  PST_CUDA(cudaMemcpy(d_np_, &n_p, sizeof(int64_t), cudaMemcpyHostToDevice));
}

act_t* Stage::in_tensor(int l, int64_t mb) const {
  return l == l0 ? xin_[mb % Rin] : out_tensor(l - 1, (int)(mb % R));
}
act_t* Stage::out_tensor(int l, int slot) const {
  const LayerBufs& b = L_[l - l0];
  if (!b.p.empty()) return b.p[slot];
  return b.z.empty() ? nullptr : b.z[slot];
}
act_t* Stage::output_slot(int64_t mb) const { return out_tensor(l1 - 1, (int)(mb % R)); }
act_t* Stage::dgrad_out() const { return L_[0].gin; }
size_t Stage::input_bytes() const {
  const LayerInfo& f0 = net_.layers[l0];
  return (size_t)batch_ * f0.in_H * f0.in_W * f0.in_Cp * sizeof(act_t);
}
size_t Stage::output_bytes() const {
  const LayerInfo& li = net_.layers[l1 - 1];
  return (size_t)batch_ * li.out_H * li.out_W * ((li.out_C + 15) / 16 * 16) * sizeof(act_t);
}
// Mid-block register sizes.  A stage may both start and end inside (different) blocks, so the
// sent and the received tensors of each direction are sized from their own block.
static size_t block_input_bytes(const NetInfo& net, int block_begin, int B) {   // the block's input
  const LayerInfo& src = net.layers[block_begin];
  return (size_t)B * src.in_H * src.in_W * src.in_Cp * sizeof(act_t);
}
static size_t residual_grad_bytes(const NetInfo& net, int residual, int B) {   // its pre-activation gradient
  const LayerInfo& e = net.layers[residual];
  return (size_t)B * e.Ho * e.Wo * e.Coutp * sizeof(act_t);
}
size_t Stage::block_out_bytes() const { return block_input_bytes(net_, end_block_, batch_); }
size_t Stage::dbuf2_bytes() const { return residual_grad_bytes(net_, net_.layers[end_block_].block_end, batch_); }
size_t Stage::input2_bytes() const { return block_input_bytes(net_, net_.layers[start_res_].block_src, batch_); }
size_t Stage::sgrad_bytes() const { return residual_grad_bytes(net_, start_res_, batch_); }
size_t Stage::stage_x_bytes() const {
  return (size_t)batch_ * net_.in_C * net_.in_H * net_.in_W * sizeof(float);
}

// ------------------------------------------------------------------ forward
ConvSpec Stage::fwd_spec(int l, int64_t mb) const {
  const int slot = (int)(mb % R);
  const LayerInfo& li = net_.layers[l];
  const LayerBufs& b = L_[l - l0];
  const bool last_net = (l == (int)net_.layers.size() - 1);
  ConvSpec c{};
  c.in = in_tensor(l, mb);
  c.N = batch_;
  c.H = li.in_H;
  c.W = li.in_W;
  c.Cinp = li.Cinp;
  c.Ho = li.Ho; c.Wo = li.Wo; c.Coutp = li.Coutp; c.Cout = li.spec.cout;
  c.k = li.kk;
  c.S = li.S;
  c.off = -li.pad;
  c.sgn = 1;
  c.wshadow = b.sh_fwd;
  c.relu = li.spec.relu;
  c.bias = li.spec.bias ? w_ + (li.off_b - p_base) : nullptr;
  if (li.spec.bn) {
    c.epi = EPI_BN_STATS;
    c.out = b.y[slot];
    c.stats = b.stats;
    c.relu = 0;
  } else if (last_net) {
    c.epi = EPI_BIAS_F32;
    c.out = b.zf[slot];
  } else {
    c.epi = EPI_BIAS_ACT;
    c.out = b.z[slot];
  }
  return c;
}

BnApplySpec Stage::bn_spec(int l, int64_t mb) const {
  const int slot = (int)(mb % R);
  const LayerInfo& li = net_.layers[l];
  const LayerBufs& b = L_[l - l0];
  const int bl = bn_idx_[l - l0];
  BnApplySpec a{};
  a.y = b.y[slot]; a.z = b.z[slot];
  a.N = batch_; a.H = li.Ho; a.W = li.Wo; a.Cp = li.Coutp; a.C = li.spec.cout;
  a.stats = b.stats;
  a.gamma = w_ + (li.off_g - p_base);
  a.beta = w_ + (li.off_be - p_base);
  a.saved = b.saved[slot];
  a.run_mean = run_ + run_off_[bl];
  a.run_var = run_ + run_off_[bl] + li.Coutp;
  a.momentum = 0.1f; a.eps = 1e-5f;
  a.relu = li.spec.relu;
  if (li.spec.residual) {
    const LayerInfo& src = net_.layers[li.block_src];
    a.res = li.block_src < l0 ? xin2_[mb % Rin] : in_tensor(li.block_src, mb);   // mid-block: received
    a.res_mode = li.res_mode;
    a.res_H = src.in_H; a.res_W = src.in_W; a.res_C = src.in_Cp; a.res_Creal = src.in_C;
    a.res_pad = li.res_pad;
  }
  return a;
}

// The forward conv c of layer l+1 takes the BN apply of layer l: it reads l's conv output y and
// writes l's z (kernels.h ConvSpec.pre 1).
void Stage::set_pre_bn_apply(ConvSpec& c, int l, int64_t mb) const {
  const BnApplySpec a = bn_spec(l, mb);
  c.in = a.y;
  c.pre = 1;
  c.pre_relu = a.relu;
  c.pre_C = a.C;
  c.pre_res = a.res_mode == 1 ? a.res : nullptr;
  c.pre_stats = a.stats;
  c.pre_gamma = a.gamma; c.pre_beta = a.beta;
  c.pre_saved = a.saved;
  c.pre_run_mean = a.run_mean; c.pre_run_var = a.run_var;
  c.pre_momentum = a.momentum; c.pre_eps = a.eps;
  c.pre_out = a.z;
}

void Stage::plan_fusion() {
  static const bool on = pst_knob("PST_FUSE_BN", 0) != 0;
  fuse_fwd_.assign(l1 - l0, 0);
  fuse_bwd_.assign(l1 - l0, 0);
  if (!on) return;
  for (int l = l0 + 1; l < l1; ++l) {
    const LayerInfo& p = net_.layers[l - 1];
    if (!p.spec.bn || p.spec.pool != 0 || p.spec.dropout > 0.f) continue;
    if (p.spec.residual && p.res_mode != 1) continue;
    ConvSpec c = fwd_spec(l, 0);
    set_pre_bn_apply(c, l - 1, 0);
    if (c.Cinp != p.Coutp || c.H != p.Ho || c.W != p.Wo) continue;
    fuse_fwd_[l - l0] = conv_ts_fits(c) ? 1 : 0;
  }
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& li = net_.layers[l];
    const LayerBufs& b = L_[l - l0];
    if (!li.spec.bn || li.S != 1 || b.gin == nullptr) continue;
    ConvSpec c{};
    c.in = b.gpre; c.N = batch_; c.H = li.Ho; c.W = li.Wo; c.Cinp = li.Coutp;
    c.Ho = li.in_H; c.Wo = li.in_W; c.Coutp = li.Cinp; c.Cout = li.in_C;
    c.k = li.kk; c.S = 1; c.off = li.pad; c.sgn = -1; c.wshadow = b.sh_bwd; c.epi = EPI_DGRAD; c.out = b.gin;
    c.pre = 2; c.pre_y = b.y[0]; c.pre_out = b.gy;
    fuse_bwd_[l - l0] = conv_ts_fits(c) ? 1 : 0;
  }
}

void Stage::enqueue_forward(int64_t mb, cudaStream_t st) {
  const int B = batch_;
  const int slot = (int)(mb % R);
  if (fwd_arena_n_) PST_CUDA(cudaMemsetAsync(fwd_arena_, 0, fwd_arena_n_ * sizeof(double), st));
  if (is_first())
    input_to_act(xstage_, xin_[mb % Rin], B, net_.in_C, net_.in_H, net_.in_W, net_.in_Cp, st);
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& li = net_.layers[l];
    LayerBufs& b = L_[l - l0];
    const bool last_net = (l == (int)net_.layers.size() - 1);
    ConvSpec c = fwd_spec(l, mb);
    if (fuse_fwd_[l - l0]) set_pre_bn_apply(c, l - 1, mb);   // BN apply of layer l-1 on the band
    if (!skip("fwd")) conv_tc(c, st);
    const bool next_takes_bn = l + 1 < l1 && fuse_fwd_[l + 1 - l0];
    if (li.spec.bn && !next_takes_bn && !skip("bnapply")) bn_apply(bn_spec(l, mb), st);
    if (li.spec.dropout > 0.f)   // after the ReLU, before the pool (pst.h pst_layer.dropout)
      dropout_fwd(b.z[slot], B, li.Ho, li.Wo, li.Coutp, li.spec.cout, dseed_, l, drop_thresh(li.spec.dropout),
                  drop_scale(li.spec.dropout), d_fmb_, st);
    if (li.spec.pool == PST_POOL_MAX2)
      maxpool2_fwd(b.z[slot], b.p[slot], b.arg[slot], B, li.Ho, li.Wo, li.Coutp, st);
    else if (li.spec.pool == PST_POOL_GAP)
      gap_fwd(b.z[slot], b.p[slot], B, li.Ho, li.Wo, li.Coutp, st);
    if (last_net)
      softmax_ce(b.zf[slot], label_ring_, label_ring_n_, loss_ring_, fwd_counter_, dz_, B,
                 li.spec.cout, li.Coutp, st);
  }
  if (has_drop_) counter_inc(d_fmb_, st);
}

// ------------------------------------------------------------------ backward + update
void Stage::enqueue_backward(int64_t mb, int dpar, cudaStream_t st) {
  const int B = batch_;
  const int slot = (int)(mb % R);
  static const bool fuse_on = pst_knob("PST_FUSE_PRE", 1) != 0;
  std::vector<char> pre_done(l1 - l0, 0);   // bwd_pre(l) already done by dgrad(l+1)'s epilogue
  PST_CUDA(cudaMemsetAsync(bwd_arena_, 0, bwd_arena_n_ * sizeof(double), st));
  for (int l = l1 - 1; l >= l0; --l) {
    const LayerInfo& li = net_.layers[l];
    LayerBufs& b = L_[l - l0];
    const bool last_net = (l == (int)net_.layers.size() - 1);
    BwdPreSpec pr{};
    if (last_net) {
      pr.gout = reinterpret_cast<const act_t*>(dz_);
      pr.gout_f32 = 1;
    } else if (l == l1 - 1) {
      pr.gout = dbuf_[dpar];
    } else {
      pr.gout = L_[l + 1 - l0].gin;
    }
    pr.pool = li.spec.pool;
    pr.arg = li.spec.pool == PST_POOL_MAX2 ? b.arg[slot] : nullptr;
    pr.z = b.z.empty() ? nullptr : b.z[slot];
    pr.relu = li.spec.relu;
    pr.rscale = li.spec.dropout > 0.f ? drop_scale(li.spec.dropout) : 1.f;
    pr.bn = li.spec.bn;
    pr.y = li.spec.bn ? b.y[slot] : nullptr;
    pr.saved = li.spec.bn ? b.saved[slot] : nullptr;
    pr.gpre = b.gpre;
    pr.N = B; pr.H = li.Ho; pr.W = li.Wo; pr.Cp = li.Coutp; pr.C = li.spec.cout;
    pr.sums = b.sums;
    if (!skip("bwdpre") && !pre_done[l - l0]) bwd_pre(pr, st);
    const bool fb = fuse_bwd_[l - l0] != 0;   // the dgrad does this layer's BN backward on its band
    const act_t* dY = b.gpre;
    if (li.spec.bn) {
      if (!fb) {
        BnBwdSpec bb{};
        bb.gpre = b.gpre; bb.y = b.y[slot]; bb.saved = b.saved[slot]; bb.sums = b.sums;
        bb.gamma = w_ + (li.off_g - p_base);  // current gamma (no stash)
        bb.gy = b.gy;
        bb.N = B; bb.H = li.Ho; bb.W = li.Wo; bb.Cp = li.Coutp; bb.C = li.spec.cout;
        if (!skip("bnbwd")) bn_bwd_apply(bb, st);
      }
      dY = b.gy;
    }
    // weight gradient from the saved input of this mini-batch
    auto wgrad = [&]() {
      WgradSpec wg{};
      wg.x = in_tensor(l, mb);
      wg.N = B;
      wg.H = li.in_H;
      wg.W = li.in_W;
      wg.Cinp = li.Cinp;
      wg.dy = dY; wg.Ho = li.Ho; wg.Wo = li.Wo; wg.Coutp = li.Coutp;
      wg.k = li.kk;
      wg.S = li.S;
      wg.pad = li.pad;
      wg.part = b.wpart;
      wg.ksplit = b.ksplit;
      if (skip("wgrad")) return;
      if (side_wgrad()) {
        PST_CUDA(cudaEventRecord(ev_fork, st));
        PST_CUDA(cudaStreamWaitEvent(wstream, ev_fork, 0));
        static const bool wg_pdl = pst_knob("PST_WG_PDL", 1) != 0;
        pdl_suppressed = !wg_pdl;
        conv_wgrad_tc(wg, wstream);
        pdl_suppressed = false;
      } else {
        conv_wgrad_tc(wg, st);
      }
    };
    // input gradient with the CURRENT weights
    auto dgrad = [&]() {
      ConvSpec c{};
      const act_t* src = dY;
      int sH = li.Ho, sW = li.Wo;
      if (li.S == 2) {
        dilate2(dY, b.dil, B, li.Ho, li.Wo, li.in_H, li.in_W, li.Coutp, st);
        src = b.dil; sH = li.in_H; sW = li.in_W;
      }
      c.in = src; c.N = B;
      c.H = sH; c.W = sW;
      c.Cinp = li.Coutp;
      c.Ho = li.in_H; c.Wo = li.in_W;
      c.Coutp = li.Cinp;
      c.Cout = li.in_C;
      c.k = li.kk;
      c.S = 1;
      c.off = li.pad;
      c.sgn = -1;
      c.wshadow = b.sh_bwd;
      c.epi = EPI_DGRAD;
      c.out = b.gin;
      if (fb) {   // BN backward of this layer on the band: gpre (+ y) in, gy written for the wgrad
        c.in = b.gpre;
        c.pre = 2;
        c.pre_C = li.spec.cout;
        c.pre_y = b.y[slot];
        c.pre_saved = b.saved[slot];
        c.pre_stats = b.sums;
        c.pre_gamma = w_ + (li.off_g - p_base);   // current gamma (no stash)
        c.pre_out = b.gy;
      }
      // fuse bwd_pre of layer l-1 (ReLU mask + BN backward sums) into this epilogue when layer
      // l-1 has no pooling and the TS kernel takes the shape
      if (fuse_on && l - 1 >= l0 && net_.layers[l - 1].spec.pool == 0 && conv_ts_fits(c)) {
        const LayerInfo& lo = net_.layers[l - 1];
        LayerBufs& bl = L_[l - 1 - l0];
        c.out = bl.gpre;
        c.bfuse = 1;
        c.brelu = lo.spec.relu;
        c.bscale = lo.spec.dropout > 0.f ? drop_scale(lo.spec.dropout) : 1.f;
        c.bbn = lo.spec.bn;
        c.bz = bl.z.empty() ? nullptr : bl.z[slot];
        c.by = lo.spec.bn ? bl.y[slot] : nullptr;
        c.bsaved = lo.spec.bn ? bl.saved[slot] : nullptr;
        c.bsums = bl.sums;
        pre_done[l - 1 - l0] = 1;
      }
      if (li.spec.block_begin && li.block_end >= 0) {
        const LayerInfo& e = net_.layers[li.block_end];
        c.res = li.block_end >= l1 ? dbuf2_[dpar] : L_[li.block_end - l0].gpre;   // mid-block: received
        c.res_mode = e.res_mode;
        c.res_H = e.Ho; c.res_W = e.Wo; c.res_C = e.Coutp; c.res_pad = e.res_pad;
      }
      static const int dg_ctas = pst_knob("PST_DG_CTAS", 0);
      c.max_ctas = side_wgrad() ? dg_ctas : 0;
      if (!skip("dgrad")) conv_tc(c, st);
    };
    if (fb) {
      dgrad();
      wgrad();
    } else {
      wgrad();
      if (b.gin != nullptr) dgrad();
    }
  }
  if (side_wgrad()) {
    PST_CUDA(cudaEventRecord(ev_join, wstream));
    PST_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  }
  if (!skip("sgd")) sgd_update(sgd_, st);
}

// ------------------------------------------------------------------ FS/BKS mapping
void Stage::copy_saved_to(const Stage& d, int64_t mb, cudaStream_t st) const {
  const int ss = (int)(mb % R), ds = (int)(mb % d.R);
  PST_CUDA(cudaMemcpyAsync(d.xin_[mb % d.Rin], xin_[mb % Rin], input_bytes(), cudaMemcpyDefault, st));
  if (starts_mid())
    PST_CUDA(cudaMemcpyAsync(d.xin2_[mb % d.Rin], xin2_[mb % Rin], input2_bytes(), cudaMemcpyDefault, st));
  for (int l = l0; l < l1; ++l) {
    const LayerBufs& a = L_[l - l0];
    const LayerBufs& b = d.L_[l - l0];
    if (a.y_bytes) PST_CUDA(cudaMemcpyAsync(b.y[ds], a.y[ss], a.y_bytes, cudaMemcpyDefault, st));
    if (!a.z.empty()) PST_CUDA(cudaMemcpyAsync(b.z[ds], a.z[ss], a.z_bytes, cudaMemcpyDefault, st));
    if (!a.zf.empty()) PST_CUDA(cudaMemcpyAsync(b.zf[ds], a.zf[ss], a.z_bytes, cudaMemcpyDefault, st));
    if (a.p_bytes) PST_CUDA(cudaMemcpyAsync(b.p[ds], a.p[ss], a.p_bytes, cudaMemcpyDefault, st));
    if (a.arg_bytes) PST_CUDA(cudaMemcpyAsync(b.arg[ds], a.arg[ss], a.arg_bytes, cudaMemcpyDefault, st));
    if (a.saved_bytes) PST_CUDA(cudaMemcpyAsync(b.saved[ds], a.saved[ss], a.saved_bytes, cudaMemcpyDefault, st));
  }
}

void Stage::copy_weights_from(const Stage& src, cudaStream_t st) {
  PST_CUDA(cudaMemcpyAsync(w_, src.w_, n_params * sizeof(float), cudaMemcpyDefault, st));
  build_shadows(sgd_, st);   // the forward copy's weight shadows (hi/lo planes) from the new weights
}

// ------------------------------------------------------------------ host readback
void Stage::read_params(float* out_params, float* out_mom) const {
  PST_CUDA(cudaSetDevice(dev));
  if (out_params) PST_CUDA(cudaMemcpy(out_params, w_, n_params * sizeof(float), cudaMemcpyDeviceToHost));
  if (out_mom) PST_CUDA(cudaMemcpy(out_mom, v_, n_params * sizeof(float), cudaMemcpyDeviceToHost));
}

void Stage::read_bnstats(std::vector<float>& mv) const {
  PST_CUDA(cudaSetDevice(dev));
  int b = 0;
  for (int l = l0; l < l1; ++l) {
    const LayerInfo& li = net_.layers[l];
    if (!li.spec.bn) continue;
    std::vector<float> tmp(2 * li.Coutp);
    PST_CUDA(cudaMemcpy(tmp.data(), run_ + run_off_[b], tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
    mv.insert(mv.end(), tmp.begin(), tmp.begin() + li.spec.cout);
    mv.insert(mv.end(), tmp.begin() + li.Coutp, tmp.begin() + li.Coutp + li.spec.cout);
    ++b;
  }
}

int64_t Stage::read_version() const {
  PST_CUDA(cudaSetDevice(dev));
  int64_t v = 0;
  PST_CUDA(cudaMemcpy(&v, d_vcount_, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return v;
}

void Stage::read_losses(int64_t first_mb, int64_t n, float* out) const {
  PST_CUDA(cudaSetDevice(dev));
  std::vector<float> ring(1024);
  PST_CUDA(cudaMemcpy(ring.data(), loss_ring_, 1024 * sizeof(float), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) out[i] = ring[(first_mb + i) % 1024];
}

}  // namespace pst
