/*
 * pst.h -- C ABI of libpst.so: pipelined backpropagation with stale weights
 * (Zhang & Abdelrahman, arXiv 1912.12675) on NVIDIA B200 (sm_100a).
 *
 * Citations "P:Lnn" are lines of the paper text, with the section.
 *
 * What one call does (the paper's problem statement, section 3
 * section 4, section 6.5):
 *   pst_create      a network + a Pipeline Placement Vector -> K stages,
 *                   one per device (the per-GPU mapping FS_i + BKS_{K_p-i+2},
 *                   P:L183; K = K_p + 1).
 *   pst_step        one global pipeline step t (one "execution cycle"):
 *                   stage s runs the backward pass + SGD update of mini-batch
 *                   b = t-2K+1+s, then the forward pass of mini-batch f = t-s,
 *                   reading weights 2(K-1-s) updates old; no
 *                   micro-batching, no weight stashing.
 *   pst_set_hybrid  switch to non-pipelined training after n_p mini-batches
 *                   (section 4): drain, then forward/backward one
 *                   mini-batch at a time through the same stages.
 *   pst_weights     the current weights (and optionally momentum, BN running
 *                   statistics) in the canonical layout below.
 *
 * Notation: K stages s = 0..K-1 (stage 0 holds the input layers); d_s =
 * 2(K-1-s) is the degree of staleness (the paper's 2(K_p-i+1)).
 *
 * Canonical parameter layout ("canonical order"): for each weighted layer in
 * network order: conv W as OIHW float32 [cout][cin][k][k] (FC: [cout][cin],
 * cin in the NCHW-flatten order of the incoming tensor); then bias [cout] if
 * layer.bias; then BatchNorm gamma [cout], beta [cout] if layer.bn.
 *
 * Errors: every int-returning call returns a pst_status.  No C++ exception
 * crosses the ABI.  After PST_E_CUDA or PST_E_NCCL the context is poisoned:
 * every later call returns the same code; pst_last_error() gives the message.
 *
 * Ownership: the library copies every input structure and array at create
 * time; the caller keeps ownership of all buffers it passes.  pst_step has
 * finished reading a host batch when it returns (device batches: see pst_batch).  Output buffers are
 * caller-allocated; pass out == NULL to query the required size in *n.
 *
 * Threading: one host thread of control per context.
 */
#ifndef PST_H_
#define PST_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pst_ctx pst_ctx;

typedef enum {
  PST_OK = 0,
  PST_E_INVALID = -1,      /* bad argument (shape, PPV, size, pointer) */
  PST_E_OOM = -2,          /* device or host allocation failed */
  PST_E_CUDA = -3,         /* CUDA runtime/driver error (context poisoned) */
  PST_E_NCCL = -4,         /* NCCL error (context poisoned) */
  PST_E_STATE = -5,        /* call not valid in the current state */
  PST_E_UNSUPPORTED = -6   /* valid request this build does not implement */
} pst_status;

/* Kinds of weighted layer (the paper numbers weighted layers for the PPV, Table 1). */
typedef enum { PST_LAYER_CONV = 0, PST_LAYER_FC = 1 } pst_layer_kind;
/* Pooling attached after a layer's ReLU. */
typedef enum { PST_POOL_NONE = 0, PST_POOL_MAX2 = 1, PST_POOL_GAP = 2 } pst_pool;

/* One weighted layer with the non-weighted ops that follow it, applied in this
 * order: y = conv/fc(x) (+bias); BN_train(y) if bn; + shortcut(block input) if
 * residual (identity, or option A: stride-2 subsample + equal zero channel pad,
 * when shapes differ); ReLU if relu; dropout if dropout > 0; pool.  block_begin marks a layer whose
 * INPUT is the residual block input of the next residual layer. */
typedef struct {
  int32_t kind;        /* pst_layer_kind */
  int32_t cin, cout;   /* conv: channels; FC: features (cin = C*H*W of the input tensor) */
  int32_t k, stride, pad; /* conv only: square kernel, stride (1 or 2), zero padding */
  int32_t bias;        /* 0/1 */
  int32_t bn;          /* 0/1: training-mode BatchNorm, momentum 0.1, eps 1e-5 */
  int32_t block_begin; /* 0/1 */
  int32_t residual;    /* 0/1 */
  int32_t relu;        /* 0/1 */
  int32_t pool;        /* pst_pool */
  float dropout;       /* drop probability p in [0, 1) applied after the ReLU, before the pool
                          (VGG-16 "batch normalization and dropout"; needs relu).  Inverted
                          dropout with the counter-based masks of DESIGN.md (reading AMB-16b):
                          key = fmix32(seed ^ fmix32(mb*0x9E3779B9 + (layer+1)*0x632BE5AB)), element
                          e (logical NCHW index) kept iff fmix32(e ^ key) >= floor(p * 2^32), kept
                          values scaled by 1/(1-p); mb = the mini-batch index, layer = 0-based. */
} pst_layer;

typedef struct {
  int32_t n_layers;
  const pst_layer* layers;       /* n_layers entries, network order */
  int32_t in_c, in_h, in_w;      /* input image shape (NCHW without N) */
  int32_t n_classes;             /* softmax cross-entropy over the last layer's cout */
  const float* init_params;      /* host, canonical order, n_params floats */
  int64_t n_params;
} pst_net;

/* Pipeline Placement Vector: ppv[i] is the 1-indexed weighted layer
 * after which register pair i sits; stage s holds layers ppv[s-1]+1..ppv[s]
 * (reading AMB-13).  Strictly increasing, in [1, n_layers-1].  A point inside a
 * residual block is a two-tensor register (reading AMB-14; at most
 * one point per block, else PST_E_UNSUPPORTED).
 *
 * mapping (section 3, section 6.5):
 *   PST_MAP_PER_GPU (0)  one accelerator per stage runs FS_i and BKS_{K_p-i+2}
 *                        (the paper's 2-GPU implementation); `devices` has
 *                        K entries.
 *   PST_MAP_FS_BKS  (1)  the paper's 2K_p+1-accelerator mapping: the
 *                        forward stage and the backward stage of every stage but
 *                        the last run on separate accelerators; the last stage's FS
 *                        and BKS share one (forward, then backward of the same
 *                        mini-batch).  Each cycle the BKS forwards its new weights
 *                        to its FS and the FS sends the saved activations
 *                        to its BKS.  Same weight versions as mapping 0.
 *                        `devices` has 2K-1 entries: FS of stages 0..K-1, then BKS
 *                        of stages 0..K-2.  Local mode only; no hybrid switch
 *                        (PST_E_UNSUPPORTED). */
#define PST_MAP_PER_GPU 0
#define PST_MAP_FS_BKS 1
typedef struct {
  int32_t n_stages;          /* K >= 1 */
  const int32_t* ppv;        /* K-1 entries (may be NULL when K == 1) */
  const int32_t* devices;    /* CUDA device ordinals, see mapping (NULL: all on device 0) */
  int32_t mapping;           /* PST_MAP_PER_GPU or PST_MAP_FS_BKS */
} pst_partition;

typedef struct {
  int32_t batch;             /* mini-batch size B (fixed per context) */
  float momentum;            /* mu */
  float weight_decay;        /* lambda, applied to every parameter */
  const float* lr_pipelined; /* K per-stage rates used while pipelined (Table 7) */
  float lr_nonpipelined;     /* rate of every stage after the hybrid switch */
  int32_t n_milestones;
  const int64_t* milestone_epochs; /* lr *= gamma at each epoch >= milestone */
  float gamma;
  int64_t steps_per_epoch;   /* mini-batches per epoch (epoch of mb i = i / steps_per_epoch) */
  /* Solver variants of the paper's Caffe-simulated runs (SURVEY f-3).
   * Zero-initialised fields give the PyTorch form the real 2-GPU runs used (AMB-7). */
  int32_t solver;            /* 0: PyTorch  v <- mu v + (g + lambda w);  w <- w - lr v
                                1: Caffe    v <- mu v + lr (g + lambda w);  w <- w - v      */
  int32_t nesterov;          /* Nesterov momentum (AlexNet, VGG-16):
                                PyTorch  w <- w - lr (g + lambda w + mu v_new)
                                Caffe    w <- w - ((1 + mu) v_new - mu v_old)               */
  int32_t lr_policy;         /* 0: milestones x gamma (above);  1: Caffe "inv" (LeNet-5):
                                lr(i) = base (1 + inv_gamma i)^(-inv_power), i = the gradient's
                                mini-batch index (reading AMB-8)                          */
  float inv_gamma, inv_power;
  uint32_t dropout_seed;     /* seed of the dropout masks (pst_layer.dropout) */
} pst_hparams;

/* Distributed mode: one process per stage (rank == stage), NCCL send/recv
 * between neighbouring stages.  Pass NULL to pst_create for local mode (every
 * stage driven by this process, stages may share a device). */
typedef struct {
  int32_t rank;              /* this process's stage */
  int32_t world;             /* == n_stages */
  const void* nccl_id;       /* PST_NCCL_ID_BYTES bytes from pst_nccl_unique_id() on rank 0 */
} pst_dist;

#define PST_NCCL_ID_BYTES 128

/* One mini-batch.  x: NCHW float32 [batch][in_c][in_h][in_w]; y: int32 [batch]
 * labels in [0, n_classes).  on_device != 0: both are device pointers on stage
 * 0's / stage K-1's device, produced by work on `stream` (a cudaStream_t; NULL =
 * the legacy default stream): pst_step orders its copies after everything
 * enqueued on that stream so far.  In distributed mode only rank 0 reads x and
 * only rank K-1 reads y (others may pass NULL).
 * Lifetime: a host batch may be reused as soon as pst_step returns; a device
 * batch must stay valid (unmodified) until the NEXT pst_step, pst_flush or
 * pst_sync call on this context returns. */
typedef struct {
  const float* x;
  const int32_t* y;
  int32_t on_device;
  void* stream;
} pst_batch;

/* what-flags for pst_weights; blocks are concatenated in this order. */
#define PST_W_PARAMS   1u  /* canonical parameters */
#define PST_W_MOMENTUM 2u  /* SGD momentum buffers, canonical order */
#define PST_W_BNSTATS  4u  /* per BN layer in order: running_mean[cout], running_var[cout] */

int pst_create(const pst_net* net, const pst_partition* part, const pst_hparams* hp,
               const pst_dist* dist, pst_ctx** out);

/* One global step t: feeds mini-batch t (or, after the hybrid switch, trains
 * mini-batch t non-pipelined).  Asynchronous w.r.t. the host. */
int pst_step(pst_ctx* ctx, const pst_batch* batch);

/* Switch to non-pipelined training once switch_epoch*steps_per_epoch
 * mini-batches have been fed (reading AMB-10: drain, keep momentum).  < 0 disables. */
int pst_set_hybrid(pst_ctx* ctx, int64_t switch_epoch);

/* Drain: run the 2K-1 backward-only steps that complete every fed mini-batch. */
int pst_flush(pst_ctx* ctx);

/* Synchronises, then copies the requested blocks (float32) into out[cap].
 * Local mode: the whole network.  Distributed mode: this rank's stage only
 * (canonical order restricted to its layers).  *n = floats written/needed. */
int pst_weights(pst_ctx* ctx, uint32_t what, float* out, int64_t cap, int64_t* n);

/* Losses of mini-batches first_mb .. first_mb+n-1 (computed by their forward
 * pass); waits for the queued work that computes them.  Only the context
 * owning the last stage has losses (else PST_E_STATE).  At most the last 1024
 * are kept; asking for a mini-batch whose forward has not been enqueued yet, or
 * one older than that window, returns PST_E_STATE. */
int pst_losses(pst_ctx* ctx, int64_t first_mb, int64_t n, float* out);

/* v_s = number of SGD updates applied by each owned stage (local: K values;
 * distributed: 1).  cap = entries available in v. */
int pst_versions(pst_ctx* ctx, int64_t* v, int32_t cap);

/* Host counters: steps executed and mini-batches fed so far. */
int pst_progress(pst_ctx* ctx, int64_t* steps, int64_t* fed);

/* cudaStream_t (as void*) on which stage `stage` (an owned stage) launches its work. */
int pst_stream(pst_ctx* ctx, int32_t stage, void** stream);

/* Blocks until all queued work of this context has finished. */
int pst_sync(pst_ctx* ctx);

/* Kernels launched by the library so far in this process (graph replays counted
 * by the kernels captured in each graph). */
int pst_launches(pst_ctx* ctx, int64_t* n);

/* Kernel classes for pst_profile_read. */
typedef enum { PST_K_CONV_FWD = 0, PST_K_CONV_DGRAD, PST_K_CONV_WGRAD, PST_K_BN_APPLY, PST_K_BWD_PRE,
               PST_K_BN_BWD, PST_K_POOL, PST_K_SGD, PST_K_LOSS, PST_K_MISC, PST_K_NCLASSES } pst_kernel_class;

/* enable != 0: later steps run eagerly (no CUDA graphs) with a CUDA-event pair
 * around every kernel launch; counters are reset.  enable == 0: back to graphs. */
int pst_profile(pst_ctx* ctx, int32_t enable);
/* Totals since pst_profile(ctx, 1) for one kernel class: event-timed milliseconds,
 * launches, and the algorithmic bytes / FLOPs of those launches (DESIGN.md
 * "Roofline accounting").  Synchronises. */
int pst_profile_read(pst_ctx* ctx, int32_t cls, double* ms, int64_t* launches, double* bytes,
                     double* flops);

/* Per-stage timing (balance diagnostics for the partition, SURVEY f-1).  enable != 0: from the
 * next pst_step on, the owned stages of each step run one after another (stage s waits for
 * stage s-1's work of the same step; the schedule's results are unchanged) with a CUDA-event
 * pair around each stage's step program, so each stage's device time is measured alone.
 * Counters are reset.  enable == 0: back to concurrent stages. */
int pst_stage_timing(pst_ctx* ctx, int32_t enable);
/* Accumulated milliseconds per owned stage since pst_stage_timing(ctx, 1) (cap entries) and
 * the number of timed steps.  Synchronises. */
int pst_stage_times(pst_ctx* ctx, double* ms, int32_t cap, int64_t* steps);

/* Device memory of an owned stage (the paper's memory analysis, section 3 and Table 6
 * P:L198-212 section 6.6: a stage keeps the activations of 2(K-s)-1 mini-batches).  out[cap >= 5]:
 *   out[0] device bytes the stage allocated (all buffers);
 *   out[1] saved-activation ring slots R_s this build keeps (2(K-s)-1 rounded up to a divisor of
 *          2K+2, model.h ring_saved);
 *   out[2] the paper's count 2(K-s)-1;
 *   out[3] bytes of the saved forward state of one mini-batch (one slot);
 *   out[4] bytes of the stage's parameters (one float32 copy);
 *   out[5] (cap >= 6) input-ring slots (2(K-s)+1 for s > 0 rounded likewise, model.h ring_input). */
int pst_memory(pst_ctx* ctx, int32_t stage, int64_t* out, int32_t cap);

void pst_destroy(pst_ctx* ctx);
const char* pst_last_error(const pst_ctx* ctx);

/* ---- host-only helpers (no GPU needed) ---------------------------------- */

/* Fills PST_NCCL_ID_BYTES bytes with a fresh NCCL unique id (rank 0). */
int pst_nccl_unique_id(void* out);

/* Validates a PPV for a network; writes the 0-based [start, end) layer range
 * of each stage into ranges[2*K].  Same rules as pst_create. */
int pst_partition_ranges(const pst_net* net, const pst_partition* part, int32_t* ranges);

/* Number of canonical parameters of the network (net->init_params unused). */
int64_t pst_param_count(const pst_net* net);

/* Schedule of step t for stage s of a K-stage pipeline fed n_fed mini-batches
 * so far, n_total to be fed before a drain (-1: unbounded):
 *   *bwd_mb = t-2K+1+s if that mini-batch exists else -1   (runs first, P:L61/AMB-1)
 *   *fwd_mb = t-s       if that mini-batch exists else -1
 *   *fwd_version = version of W_s read by that forward = #updates done = max(0, fwd_mb - 2(K-1-s)).
 * Returns PST_E_INVALID for bad arguments. */
int pst_schedule(int32_t K, int32_t s, int64_t t, int64_t n_total,
                 int64_t* bwd_mb, int64_t* fwd_mb, int64_t* fwd_version);

/* Ring sizes libpst uses for stage s of a K-stage pipeline (host only): *saved = slots of saved
 * forward state (>= the paper's 2(K-s)-1), *input = slots of the received-activation ring
 * (>= 2(K-s)+1 for s > 0), both divisors of the graph-key period *period = 2K+2. */
int pst_ring_slots(int32_t K, int32_t s, int32_t* saved, int32_t* input, int32_t* period);

/* Library build string (arch, compute dtype). */
const char* pst_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* PST_H_ */
