// stage.h -- one pipeline stage: the contiguous weighted layers p_{s}+1..p_{s+1}
// with their weights (one copy, no stash: P:L35/L236), momentum,
// the saved-activation ring (activations kept until the stage's backward),
// and the launch program for its forward and backward(+update) passes.
#pragma once
#include <vector>

#include "common.h"
#include "kernels.h"
#include "model.h"

namespace pst {

struct LayerBufs {
  std::vector<act_t*> y, z, p;   // per ring slot: conv out (BN input), post-op, pooled
  std::vector<float*> zf;        // per slot: float logits (last FC)
  std::vector<uint8_t*> arg;     // per slot: max-pool argmax
  std::vector<float*> saved;     // per slot: BN (mean, invstd) [Coutp][2]
  act_t* gpre = nullptr;         // gradient w.r.t. pre-activation (after pool^T, relu^T)
  act_t* gy = nullptr;           // gradient w.r.t. conv output (after BN^T)
  act_t* gin = nullptr;          // gradient w.r.t. the layer input
  act_t* dil = nullptr;          // zero-inserted gradient for stride-2 dgrad
  float* wpart = nullptr;        // wgrad split-K partials
  int ksplit = 1;
  double* stats = nullptr;       // forward BN sums [Coutp][2]
  double* sums = nullptr;        // backward sums [Coutp][2]
  size_t y_bytes = 0, z_bytes = 0, p_bytes = 0, arg_bytes = 0, saved_bytes = 0;   // per ring slot
  act_t* sh_fwd = nullptr;       // [k*k][Coutp][Cinp]
  act_t* sh_bwd = nullptr;       // [k*k][Cinp][Coutp]
};

class Stage {
 public:
  Stage(const NetInfo& net, int s, int K, int l0, int l1, int device, const pst_hparams& hp,
        const float* init_params, int batch);
  ~Stage();
  Stage(const Stage&) = delete;
  Stage& operator=(const Stage&) = delete;

  // Enqueue work (capturable): forward of mini-batch mb (its saved state goes to ring slot mb % R,
  // its input is read from input-ring slot mb % Rin).
  void enqueue_forward(int64_t mb, cudaStream_t st);
  // Backward + SGD update of mini-batch mb, reading the output gradient from dbuf[dpar] (non-last
  // stages) or the stored dz (last stage).
  void enqueue_backward(int64_t mb, int dpar, cudaStream_t st);

  act_t* input_slot(int64_t mb) const { return xin_[mb % Rin]; }
  act_t* output_slot(int64_t mb) const;          // stage output tensor (non-last stages)
  act_t* dgrad_out() const;                      // gradient w.r.t. the stage input
  act_t* dbuf(int par) const { return dbuf_[par]; }
  size_t input_bytes() const;
  size_t output_bytes() const;
  // Mid-block register pair (reading AMB-14).  A stage that ENDS inside a residual
  // block also sends the block input forward and receives the shortcut gradient (the residual
  // layer's pre-activation gradient) back; a stage that STARTS inside a block receives the block
  // input and sends its residual layer's pre-activation gradient back.
  bool ends_mid() const { return end_block_ >= 0; }
  bool starts_mid() const { return start_res_ >= 0; }
  act_t* block_out(int64_t mb) const { return in_tensor(end_block_, mb); }  // ends_mid: sent forward
  size_t block_out_bytes() const;
  act_t* dbuf2(int par) const { return dbuf2_[par]; }                         // ends_mid: received
  size_t dbuf2_bytes() const;
  act_t* input2_slot(int64_t mb) const { return xin2_[mb % Rin]; }          // starts_mid: received
  size_t input2_bytes() const;
  act_t* sgrad_out() const { return L_[start_res_ - l0].gpre; }               // starts_mid: sent back
  size_t sgrad_bytes() const;
  float* stage_x() const { return xstage_; }     // stage 0: float NCHW staging of the batch
  size_t stage_x_bytes() const;
  int32_t* label_slot(int64_t mb) const { return label_ring_ + (mb % label_ring_n_) * batch_; }

  void set_n_p(int64_t n_p);
  // The paper's FS/BKS mapping (pst.h PST_MAP_FS_BKS): the forward copy of a stage hands the saved
  // forward state of mini-batch mb to the backward copy, and the backward copy forwards
  // its new weights to the forward copy.  Both enqueue on `st` (the caller orders them).
  void copy_saved_to(const Stage& dst, int64_t mb, cudaStream_t st) const;
  void copy_weights_from(const Stage& src, cudaStream_t st);
  // Synchronous host copies (call only when the stream is idle).
  void read_params(float* out_params, float* out_mom) const;   // canonical stage block
  void read_bnstats(std::vector<float>& mean_var) const;       // per BN layer: mean[C], var[C]
  int64_t read_version() const;
  void read_losses(int64_t first_mb, int64_t n, float* out) const;

  const int s, K, l0, l1, dev;
  const int R;     // saved-state ring slots (ring_saved)
  const int Rin;   // input ring slots (ring_input)
  const int batch_;
  int64_t p_base = 0, n_params = 0;
  size_t bytes_total = 0;   // device bytes this stage allocated
  size_t bytes_slot = 0;    // saved forward state of ONE mini-batch (input + per-layer y/z/pool/argmax/stats)
  cudaStream_t stream = nullptr;
  // weight-gradient side stream: wgrad(l) depends only on dY(l) and the saved input, so it runs
  // concurrently with the dgrad chain of the layers below and joins before the update
  cudaStream_t wstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // distributed mode: boundary exchanges on their own stream, overlapping the forward pass
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_cb = nullptr, ev_cf = nullptr, ev_cj = nullptr;
  bool is_first() const { return s == 0; }
  bool is_last() const { return l1 == (int)net_.layers.size(); }

 private:
  const NetInfo& net_;
  std::vector<void*> allocs_;
  template <typename T> T* alloc(size_t n, bool zero = true);
  act_t* in_tensor(int l, int64_t mb) const;     // input of layer l for mini-batch mb
  act_t* out_tensor(int l, int slot) const;      // saved output of layer l in ring slot `slot`

  ConvSpec fwd_spec(int l, int64_t mb) const;                 // forward conv of layer l (no pre-pass)
  BnApplySpec bn_spec(int l, int64_t mb) const;               // BN apply of layer l (bn layers)
  void set_pre_bn_apply(ConvSpec& c, int l, int64_t mb) const;   // c (layer l+1) takes l's BN apply
  void plan_fusion();
  // Band pre-pass fusion (kernels.h ConvSpec.pre): fuse_fwd_[i] -- the forward conv of layer l0+i
  // does the BN apply of layer l0+i-1; fuse_bwd_[i] -- the dgrad of layer l0+i does its own BN
  // backward (its wgrad then forks after the dgrad, which writes gy).
  std::vector<char> fuse_fwd_, fuse_bwd_;
  std::vector<int> bn_idx_;                      // local BN index of each layer (run_off_), -1 if none

  std::vector<LayerBufs> L_;
  std::vector<act_t*> xin_;
  act_t* dbuf_[2] = {nullptr, nullptr};
  int end_block_ = -1;     // block_begin layer of the block open at the stage's end (-1: none)
  int start_res_ = -1;     // residual layer closing the block open at the stage's start (-1: none)
  std::vector<act_t*> xin2_;                     // block input ring (starts_mid)
  act_t* dbuf2_[2] = {nullptr, nullptr};          // shortcut gradient double buffer (ends_mid)
  float* xstage_ = nullptr;
  float* w_ = nullptr;
  float* v_ = nullptr;
  float* run_ = nullptr;          // per local BN layer: mean[Coutp], var[Coutp]
  std::vector<int64_t> run_off_;
  double* fwd_arena_ = nullptr; size_t fwd_arena_n_ = 0;
  double* bwd_arena_ = nullptr; size_t bwd_arena_n_ = 0;
  // last stage
  int32_t* label_ring_ = nullptr; int label_ring_n_ = 0;
  float* loss_ring_ = nullptr;
  int64_t* fwd_counter_ = nullptr;
  // dropout
  bool has_drop_ = false;
  uint32_t dseed_ = 0;
  int64_t* d_fmb_ = nullptr;
  float* dz_ = nullptr;
  // optimiser
  SgdSpec sgd_{};
  SgdSeg* d_segs_ = nullptr;
  int64_t* d_red_start_ = nullptr;
  int64_t* d_seg_start_ = nullptr;
  int64_t* d_vcount_ = nullptr;
  int* d_ticket_ = nullptr;
  float* d_lr_ = nullptr;
  int64_t* d_np_ = nullptr;
  int64_t* d_ms_ = nullptr;
};

}  // namespace pst
