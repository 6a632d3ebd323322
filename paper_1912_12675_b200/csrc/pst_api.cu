// pst_api.cu -- the C ABI (include/pst.h): context, step scheduler, hybrid switch,
// CUDA-graph cache, inter-stage transport (local copies or NCCL send/recv).
//
// Schedule (PAPER.md L61/L63/L75, reading AMB-1): at global step t, stage s runs
// the backward + SGD update of mini-batch b = t-2K+1+s, then the forward of
// mini-batch f = t-s.  Messages produced at step t are consumed at step t+1:
// the forward activation of f goes into stage s+1's input ring slot, the input
// gradient of b into stage s-1's gradient buffer dbuf[b % 2].
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pst.h"
#include "common.h"
#include "model.h"
#include "stage.h"

using namespace pst;

#define PST_NCCL(expr)                                                                       \
  do {                                                                                       \
    ncclResult_t r_ = (expr);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      throw ::pst::NcclError(std::string(#expr) + ": " + ncclGetErrorString(r_) + " at " +   \
                             __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)

namespace {

enum Mode { MODE_PIPE = 0, MODE_NP = 1 };

struct GraphKey {
  std::vector<int64_t> k;
  bool operator<(const GraphKey& o) const { return k < o.k; }
};
struct GraphEntry {
  cudaGraphExec_t exec;
  int64_t kernels;  // kernel launches captured in the graph
};

}  // namespace

struct pst_ctx {
  std::string err;
  int sticky = 0;
  NetInfo net;
  std::vector<std::pair<int, int>> ranges;
  int K = 1;
  bool dist = false;
  int rank = 0;
  ncclComm_t comm = nullptr;
  std::vector<std::unique_ptr<Stage>> stages;   // local: K stages; dist: 1 (stage == rank)
  // PST_MAP_FS_BKS: stages[s] is FS_s (the last stage does both), bks[s] is BKS_s, s < K-1
  int mapping = PST_MAP_PER_GPU;
  std::vector<std::unique_ptr<Stage>> bks;
  std::vector<cudaEvent_t> bdone, wev;          // per BKS: last step's work / new weights ready
  std::vector<int> devices;
  pst_hparams hp{};
  std::vector<float> lr_pipe;
  std::vector<int64_t> milestones;
  int batch = 0;
  // schedule state
  int64_t t = 0, t0 = 0, m0 = 0, n_fed = 0, n_p = INT64_MAX;
  int64_t n_loss = 0;   // mini-batches whose loss (last stage's forward) has been enqueued
  // per-stage timing (pst_stage_timing): stages serialised within a step, events around each
  bool stage_timing = false;
  std::vector<cudaEvent_t> st_beg, st_end;      // per owned stage
  std::vector<double> st_ms;
  int64_t st_steps = 0;
  bool st_pending = false;
  int mode = MODE_PIPE;
  bool use_graphs = true;
  std::vector<std::map<GraphKey, GraphEntry>> graphs;        // per owned stage
  std::vector<std::map<GraphKey, GraphEntry>> graphs_b;      // per BKS object (PST_MAP_FS_BKS)
  std::vector<cudaEvent_t> done;                              // per owned stage: last step's work
  // host staging (pinned) for the batch
  float* pin_x[2] = {nullptr, nullptr};
  int32_t* pin_y[2] = {nullptr, nullptr};
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
  cudaEvent_t pin_ev2[2] = {nullptr, nullptr};
  cudaEvent_t prod_ev = nullptr;   // recorded on a device batch's producer stream
  int pin_i = 0;

  Stage* stage(int s) {
    if (!dist) return stages[s].get();
    return s == rank ? stages[0].get() : nullptr;
  }
  int local_index(int s) const { return dist ? 0 : s; }
  bool owns(int s) const { return !dist || s == rank; }
};

static thread_local std::string g_last_global_error;

template <typename F>
static int guard(pst_ctx* ctx, F&& f) {
  if (ctx && ctx->sticky) return ctx->sticky;
  try {
    f();
    return PST_OK;
  } catch (const InvalidArg& e) {
    if (ctx) ctx->err = e.what(); else g_last_global_error = e.what();
    return PST_E_INVALID;
  } catch (const Unsupported& e) {
    if (ctx) ctx->err = e.what(); else g_last_global_error = e.what();
    return PST_E_UNSUPPORTED;
  } catch (const StateError& e) {
    if (ctx) ctx->err = e.what(); else g_last_global_error = e.what();
    return PST_E_STATE;
  } catch (const NcclError& e) {
    if (ctx) { ctx->err = e.what(); ctx->sticky = PST_E_NCCL; } else g_last_global_error = e.what();
    return PST_E_NCCL;
  } catch (const CudaError& e) {
    std::string m = e.what();
    bool oom = m.find("out of memory") != std::string::npos;
    if (ctx) { ctx->err = m; if (!oom) ctx->sticky = PST_E_CUDA; } else g_last_global_error = m;
    return oom ? PST_E_OOM : PST_E_CUDA;
  } catch (const std::bad_alloc& e) {
    if (ctx) ctx->err = "host allocation failed"; else g_last_global_error = "host allocation failed";
    return PST_E_OOM;
  } catch (const std::exception& e) {
    if (ctx) { ctx->err = e.what(); ctx->sticky = PST_E_CUDA; } else g_last_global_error = e.what();
    return PST_E_CUDA;
  }
}

// ------------------------------------------------------------------ step programs
// Enqueue stage s's share of pipelined step t (plan computed by the caller).
static void enqueue_pipe(pst_ctx* c, int s, const StepPlan& p, const StepPlan& prev_stage,
                         const StepPlan& next_stage, cudaStream_t st) {
  Stage* S = c->stage(s);
  const int K = c->K;
  // distributed mode: which messages this step exchanges with each neighbour (both ends of a pair
  // derive the same answer from the same plans)
  const bool send_f = c->dist && p.fwd_mb >= 0 && s < K - 1;
  const bool recv_f = c->dist && s > 0 && prev_stage.fwd_mb >= 0;
  const bool send_b = c->dist && p.bwd_mb >= 0 && s > 0;
  const bool recv_b = c->dist && s < K - 1 && next_stage.bwd_mb >= 0;
  auto exchange_b = [&](cudaStream_t cs) {   // error of b to s-1, error of the next stage's b from s+1
    PST_NCCL(ncclGroupStart());
    if (send_b) {
      PST_NCCL(ncclSend(S->dgrad_out(), S->input_bytes(), ncclUint8, s - 1, c->comm, cs));
      if (S->starts_mid()) PST_NCCL(ncclSend(S->sgrad_out(), S->sgrad_bytes(), ncclUint8, s - 1, c->comm, cs));
    }
    if (recv_b) {
      const int par = (int)(next_stage.bwd_mb & 1);
      PST_NCCL(ncclRecv(S->dbuf(par), S->output_bytes(), ncclUint8, s + 1, c->comm, cs));
      if (S->ends_mid()) PST_NCCL(ncclRecv(S->dbuf2(par), S->dbuf2_bytes(), ncclUint8, s + 1, c->comm, cs));
    }
    PST_NCCL(ncclGroupEnd());
  };
  auto exchange_f = [&](cudaStream_t cs) {   // activation of f to s+1, the previous stage's f from s-1
    PST_NCCL(ncclGroupStart());
    if (send_f) {
      const int64_t f = p.fwd_mb;
      PST_NCCL(ncclSend(S->output_slot(f), S->output_bytes(), ncclUint8, s + 1, c->comm, cs));
      if (S->ends_mid()) PST_NCCL(ncclSend(S->block_out(f), S->block_out_bytes(), ncclUint8, s + 1, c->comm, cs));
    }
    if (recv_f) {
      const int64_t f = prev_stage.fwd_mb;
      PST_NCCL(ncclRecv(S->input_slot(f), S->input_bytes(), ncclUint8, s - 1, c->comm, cs));
      if (S->starts_mid())
        PST_NCCL(ncclRecv(S->input2_slot(f), S->input2_bytes(), ncclUint8, s - 1, c->comm, cs));
    }
    PST_NCCL(ncclGroupEnd());
  };
  // With comm overlap (default) the error exchange runs on the stage's communication stream while
  // the forward pass computes, the activation exchange after it; the step joins that stream at its
  // end, so the next step sees every received buffer.  The buffers the exchanges touch are disjoint
  // from what the forward reads and writes (input ring slots f+1 vs f, dbuf parity of b+1 vs b).
  static const bool overlap = pst_knob("PST_COMM_OVERLAP", 1) != 0;
  const bool ov = c->dist && overlap;
  bool forked = false;
  if (p.bwd_mb >= 0) {
    S->enqueue_backward(p.bwd_mb, (int)(p.bwd_mb & 1), st);
    if (s > 0 && !c->dist) {
      Stage* D = c->stage(s - 1);
      const int par = (int)(p.bwd_mb & 1);
      PST_CUDA(cudaMemcpyAsync(D->dbuf(par), S->dgrad_out(), D->output_bytes(), cudaMemcpyDefault, st));
      if (S->starts_mid())   // mid-block register: the shortcut gradient goes back too
        PST_CUDA(cudaMemcpyAsync(D->dbuf2(par), S->sgrad_out(), S->sgrad_bytes(), cudaMemcpyDefault, st));
    }
  }
  if (ov && (send_b || recv_b)) {
    PST_CUDA(cudaEventRecord(S->ev_cb, st));
    PST_CUDA(cudaStreamWaitEvent(S->cstream, S->ev_cb, 0));
    exchange_b(S->cstream);
    forked = true;
  }
  if (p.fwd_mb >= 0) {
    S->enqueue_forward(p.fwd_mb, st);
    if (s < K - 1 && !c->dist) {
      Stage* D = c->stage(s + 1);
      const int64_t f = p.fwd_mb;
      PST_CUDA(cudaMemcpyAsync(D->input_slot(f), S->output_slot(f), S->output_bytes(), cudaMemcpyDefault, st));
      if (S->ends_mid())     // mid-block register: the block input goes forward too
        PST_CUDA(cudaMemcpyAsync(D->input2_slot(f), S->block_out(f), S->block_out_bytes(), cudaMemcpyDefault, st));
    }
  }
  if (ov) {
    if (send_f || recv_f) {
      PST_CUDA(cudaEventRecord(S->ev_cf, st));
      PST_CUDA(cudaStreamWaitEvent(S->cstream, S->ev_cf, 0));
      exchange_f(S->cstream);
      forked = true;
    }
    if (forked) {   // join: the step ends when its exchanges have completed
      PST_CUDA(cudaEventRecord(S->ev_cj, S->cstream));
      PST_CUDA(cudaStreamWaitEvent(st, S->ev_cj, 0));
    }
  } else if (c->dist && (send_f || recv_f || send_b || recv_b)) {
    // one grouped exchange at the end of the step (PST_COMM_OVERLAP=0 experiment builds)
    PST_NCCL(ncclGroupStart());
    exchange_f(st);
    exchange_b(st);
    PST_NCCL(ncclGroupEnd());
  }
}

// Non-pipelined (hybrid phase 2) forward or backward part of mini-batch i on stage s.
static void enqueue_np(pst_ctx* c, int s, int64_t i, bool fwd, cudaStream_t st) {
  Stage* S = c->stage(s);
  const int K = c->K;
  const int par = (int)(i & 1);
  if (fwd) {
    if (c->dist && s > 0) {
      PST_NCCL(ncclGroupStart());
      PST_NCCL(ncclRecv(S->input_slot(i), S->input_bytes(), ncclUint8, s - 1, c->comm, st));
      if (S->starts_mid()) PST_NCCL(ncclRecv(S->input2_slot(i), S->input2_bytes(), ncclUint8, s - 1, c->comm, st));
      PST_NCCL(ncclGroupEnd());
    }
    S->enqueue_forward(i, st);
    if (s < K - 1) {
      if (c->dist) {
        PST_NCCL(ncclGroupStart());
        PST_NCCL(ncclSend(S->output_slot(i), S->output_bytes(), ncclUint8, s + 1, c->comm, st));
        if (S->ends_mid()) PST_NCCL(ncclSend(S->block_out(i), S->block_out_bytes(), ncclUint8, s + 1, c->comm, st));
        PST_NCCL(ncclGroupEnd());
      } else {
        Stage* D = c->stage(s + 1);
        PST_CUDA(cudaMemcpyAsync(D->input_slot(i), S->output_slot(i), S->output_bytes(), cudaMemcpyDefault, st));
        if (S->ends_mid())
          PST_CUDA(cudaMemcpyAsync(D->input2_slot(i), S->block_out(i), S->block_out_bytes(), cudaMemcpyDefault, st));
      }
    }
  } else {
    if (c->dist && s < K - 1) {
      PST_NCCL(ncclGroupStart());
      PST_NCCL(ncclRecv(S->dbuf(par), S->output_bytes(), ncclUint8, s + 1, c->comm, st));
      if (S->ends_mid()) PST_NCCL(ncclRecv(S->dbuf2(par), S->dbuf2_bytes(), ncclUint8, s + 1, c->comm, st));
      PST_NCCL(ncclGroupEnd());
    }
    S->enqueue_backward(i, par, st);
    if (s > 0) {
      if (c->dist) {
        PST_NCCL(ncclGroupStart());
        PST_NCCL(ncclSend(S->dgrad_out(), S->input_bytes(), ncclUint8, s - 1, c->comm, st));
        if (S->starts_mid()) PST_NCCL(ncclSend(S->sgrad_out(), S->sgrad_bytes(), ncclUint8, s - 1, c->comm, st));
        PST_NCCL(ncclGroupEnd());
      } else {
        Stage* D = c->stage(s - 1);
        PST_CUDA(cudaMemcpyAsync(D->dbuf(par), S->dgrad_out(), D->output_bytes(), cudaMemcpyDefault, st));
        if (S->starts_mid())
          PST_CUDA(cudaMemcpyAsync(D->dbuf2(par), S->sgrad_out(), S->sgrad_bytes(), cudaMemcpyDefault, st));
      }
    }
  }
}

template <typename F>
static void run_program(pst_ctx* c, Stage* S, std::map<GraphKey, GraphEntry>& cache, const GraphKey& key,
                        F&& enqueue) {
  PST_CUDA(cudaSetDevice(S->dev));
  if (!c->use_graphs || prof::enabled) {   // profiling runs eagerly: events bracket each kernel
    enqueue(S->stream);
    return;
  }
  auto it = cache.find(key);
  if (it == cache.end()) {
    cudaGraph_t g;
    const int64_t before = prof::launches;
    PST_CUDA(cudaStreamBeginCapture(S->stream, cudaStreamCaptureModeRelaxed));
    try {
      enqueue(S->stream);
    } catch (...) {
      cudaStreamEndCapture(S->stream, &g);
      throw;
    }
    PST_CUDA(cudaStreamEndCapture(S->stream, &g));
    const int64_t nk = prof::launches - before;
    prof::launches = before;  // counted per replay below
    cudaGraphExec_t ge;
    PST_CUDA(cudaGraphInstantiate(&ge, g, 0));
    PST_CUDA(cudaGraphDestroy(g));
    it = cache.emplace(key, GraphEntry{ge, nk}).first;
  }
  PST_CUDA(cudaGraphLaunch(it->second.exec, S->stream));
  prof::launches += it->second.kernels;
}

template <typename F>
static void run_program(pst_ctx* c, int s, const GraphKey& key, F&& enqueue) {
  run_program(c, c->stage(s), c->graphs[c->local_index(s)], key, std::forward<F>(enqueue));
}

// In local mode stage s's step depends on its neighbours' previous step.
static void wait_neighbours(pst_ctx* c, int s) {
  if (c->dist) return;
  Stage* S = c->stage(s);
  for (int n : {s - 1, s + 1}) {
    if (n < 0 || n >= c->K) continue;
    PST_CUDA(cudaStreamWaitEvent(S->stream, c->done[n], 0));
  }
}

static void pipe_step(pst_ctx* c) {
  const int K = c->K;
  std::vector<StepPlan> plans(K);
  for (int s = 0; s < K; ++s) plans[s] = plan_step(K, s, c->t, c->t0, c->m0, c->n_fed);
  if (plans[K - 1].fwd_mb >= 0) c->n_loss = std::max(c->n_loss, plans[K - 1].fwd_mb + 1);
  // all waits first (events of the previous step), then launches, then records
  std::vector<int> active;
  for (int s = 0; s < K; ++s) {
    if (!c->owns(s)) continue;
    wait_neighbours(c, s);
  }
  for (int s = 0; s < K; ++s) {
    if (!c->owns(s)) continue;
    const StepPlan& p = plans[s];
    const StepPlan prev = s > 0 ? plans[s - 1] : StepPlan{};
    const StepPlan next = s < K - 1 ? plans[s + 1] : StepPlan{};
    Stage* S = c->stage(s);
    GraphKey key;
    // every ring size divides P (model.h), so the buffers a step program touches are functions of
    // its mini-batch indices mod P (P even: parities too)
    const int64_t P = ring_period(K);
    auto m = [P](int64_t mb) { return mb >= 0 ? mb % P : -1; };
    key.k = {0, m(p.bwd_mb), m(p.fwd_mb), s > 0 ? m(prev.fwd_mb) : -1,
             s < K - 1 && next.bwd_mb >= 0 ? (next.bwd_mb & 1) : -1};
    if (p.bwd_mb < 0 && p.fwd_mb < 0 && key.k[3] < 0 && key.k[4] < 0) continue;
    const int li = c->local_index(s);
    if (c->stage_timing) {
      if (!c->dist && s > 0) PST_CUDA(cudaStreamWaitEvent(S->stream, c->st_end[s - 1], 0));
      PST_CUDA(cudaEventRecord(c->st_beg[li], S->stream));
    }
    run_program(c, s, key, [&](cudaStream_t st) { enqueue_pipe(c, s, p, prev, next, st); });
    if (c->stage_timing) PST_CUDA(cudaEventRecord(c->st_end[li], S->stream));
  }
  if (c->stage_timing) {   // accumulate this step's per-stage times (diagnostic: synchronises)
    for (int s = 0; s < K; ++s) {
      if (!c->owns(s)) continue;
      const int li = c->local_index(s);
      PST_CUDA(cudaEventSynchronize(c->st_end[li]));
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, c->st_beg[li], c->st_end[li]) == cudaSuccess) c->st_ms[li] += ms;
      cudaGetLastError();
      // a stage with no work this step leaves its events at the previous step: re-record both
      PST_CUDA(cudaEventRecord(c->st_beg[li], c->stage(s)->stream));
      PST_CUDA(cudaEventRecord(c->st_end[li], c->stage(s)->stream));
    }
    c->st_steps += 1;
  }
  for (int s = 0; s < K; ++s) {
    if (!c->owns(s)) continue;
    Stage* S = c->stage(s);
    PST_CUDA(cudaSetDevice(S->dev));
    PST_CUDA(cudaEventRecord(c->done[c->local_index(s)], S->stream));
  }
  c->t += 1;
}

// One cycle of the paper's 2K_p+1-accelerator mapping (PST_MAP_FS_BKS; Oracle C in
// oracle/pipeline.py run_fs_bks).  Cycle t: FS_s forwards f = t-s with the weights its BKS forwarded
// at the end of cycle t-1 and hands the saved activations of f to BKS_s; the last stage forwards f
// and then runs the backward + update of the same f; BKS_s (s < K-1) runs the backward + update of
// b = t-2K+2+s and forwards its new weights to FS_s, which installs them after its own forward of
// this cycle.  All messages of cycle t are consumed in cycle t+1 (events between the objects).
static void fsbks_step(pst_ctx* c) {
  const int K = c->K;
  const int64_t rel = c->t - c->t0, P = ring_period(K);
  auto valid = [&](int64_t mb) { return mb >= c->m0 && mb < c->n_fed ? mb : (int64_t)-1; };
  auto m = [P](int64_t mb) { return mb >= 0 ? mb % P : -1; };
  std::vector<int64_t> f(K), b(K);
  for (int s = 0; s < K; ++s) {
    f[s] = valid(c->m0 + rel - s);
    b[s] = s == K - 1 ? f[s] : valid(c->m0 + rel - 2 * K + 2 + s);
  }
  if (f[K - 1] >= 0) c->n_loss = std::max(c->n_loss, f[K - 1] + 1);
  // waits on the previous cycle (all before any launch)
  for (int s = 0; s < K; ++s) {
    Stage* F = c->stages[s].get();
    if (s > 0) PST_CUDA(cudaStreamWaitEvent(F->stream, c->done[s - 1], 0));    // activation of f
    if (s < K - 1) {
      Stage* Bk = c->bks[s].get();
      PST_CUDA(cudaStreamWaitEvent(Bk->stream, c->done[s], 0));                 // saved state of b
      PST_CUDA(cudaStreamWaitEvent(Bk->stream, s + 1 < K - 1 ? c->bdone[s + 1] : c->done[K - 1], 0));   // error of b
    }
  }
  // BKS_s: backward + update of b, error to BKS_{s-1}, new weights ready
  for (int s = 0; s + 1 < K; ++s) {
    if (b[s] < 0) continue;
    Stage* Bk = c->bks[s].get();
    GraphKey key;
    key.k = {4, m(b[s])};
    PST_CUDA(cudaSetDevice(Bk->dev));
    const int64_t bb = b[s];
    run_program(c, Bk, c->graphs_b[s], key, [&](cudaStream_t st) {
      Bk->enqueue_backward(bb, (int)(bb & 1), st);
      if (s > 0) {
        Stage* D = c->bks[s - 1].get();
        PST_CUDA(cudaMemcpyAsync(D->dbuf((int)(bb & 1)), Bk->dgrad_out(), D->output_bytes(), cudaMemcpyDefault, st));
        if (Bk->starts_mid())
          PST_CUDA(cudaMemcpyAsync(D->dbuf2((int)(bb & 1)), Bk->sgrad_out(), Bk->sgrad_bytes(), cudaMemcpyDefault, st));
      }
    });
    PST_CUDA(cudaEventRecord(c->wev[s], Bk->stream));
  }
  // FS_s: forward of f (+ the last stage's backward of the same f), activation to FS_{s+1}, saved
  // state to BKS_s; then the weights BKS_s produced in this cycle
  for (int s = 0; s < K; ++s) {
    Stage* F = c->stages[s].get();
    PST_CUDA(cudaSetDevice(F->dev));
    if (f[s] >= 0) {
      GraphKey key;
      key.k = {3, m(f[s])};
      const int64_t ff = f[s];
      run_program(c, F, c->graphs[s], key, [&](cudaStream_t st) {
        F->enqueue_forward(ff, st);
        if (s < K - 1) {
          Stage* D = c->stages[s + 1].get();
          PST_CUDA(cudaMemcpyAsync(D->input_slot(ff), F->output_slot(ff), F->output_bytes(), cudaMemcpyDefault, st));
          if (F->ends_mid())
            PST_CUDA(cudaMemcpyAsync(D->input2_slot(ff), F->block_out(ff), F->block_out_bytes(), cudaMemcpyDefault, st));
          F->copy_saved_to(*c->bks[s], ff, st);
        } else {
          F->enqueue_backward(ff, 0, st);   // the last stage: FS_{K_p+1} and BKS_1 on one accelerator
          if (s > 0) {
            Stage* D = c->bks[s - 1].get();
            PST_CUDA(cudaMemcpyAsync(D->dbuf((int)(ff & 1)), F->dgrad_out(), D->output_bytes(), cudaMemcpyDefault, st));
            if (F->starts_mid())
              PST_CUDA(cudaMemcpyAsync(D->dbuf2((int)(ff & 1)), F->sgrad_out(), F->sgrad_bytes(), cudaMemcpyDefault, st));
          }
        }
      });
    }
    if (s < K - 1 && b[s] >= 0) {      // weight forwarding BKS_s -> FS_s (after this cycle's forward)
      PST_CUDA(cudaStreamWaitEvent(F->stream, c->wev[s], 0));
      F->copy_weights_from(*c->bks[s], F->stream);
    }
  }
  for (int s = 0; s < K; ++s) {
    PST_CUDA(cudaSetDevice(c->stages[s]->dev));
    PST_CUDA(cudaEventRecord(c->done[s], c->stages[s]->stream));
    if (s < K - 1) {
      PST_CUDA(cudaSetDevice(c->bks[s]->dev));
      PST_CUDA(cudaEventRecord(c->bdone[s], c->bks[s]->stream));
    }
  }
  c->t += 1;
}

static void drain(pst_ctx* c) {
  if (c->mode != MODE_PIPE) return;
  // the last backward is stage 0's of mini-batch n_fed-1 at relative step n_fed-1-m0 + 2K-1
  // (FS/BKS mapping: one cycle earlier, BKS_0 at n_fed-1-m0 + 2K-2)
  const int64_t last = c->t0 + (c->n_fed - 1 - c->m0) + 2 * c->K - 1 - (c->mapping == PST_MAP_FS_BKS ? 1 : 0);
  while (c->n_fed > c->m0 && c->t <= last) {
    if (c->mapping == PST_MAP_FS_BKS) fsbks_step(c);
    else pipe_step(c);
  }
  c->t0 = c->t;
  c->m0 = c->n_fed;
}

static void np_step(pst_ctx* c) {
  const int K = c->K;
  const int64_t i = c->n_fed - 1;
  c->n_loss = std::max(c->n_loss, i + 1);
  for (int s = 0; s < K; ++s) {
    if (!c->owns(s)) continue;
    Stage* S = c->stage(s);
    if (!c->dist && s > 0) {
      PST_CUDA(cudaSetDevice(S->dev));
      PST_CUDA(cudaStreamWaitEvent(S->stream, c->done[s - 1], 0));
    }
    GraphKey key;
    key.k = {1, i % ring_period(K)};
    run_program(c, s, key, [&](cudaStream_t st) { enqueue_np(c, s, i, true, st); });
    PST_CUDA(cudaEventRecord(c->done[c->local_index(s)], S->stream));
  }
  for (int s = K - 1; s >= 0; --s) {
    if (!c->owns(s)) continue;
    Stage* S = c->stage(s);
    if (!c->dist && s < K - 1) {
      PST_CUDA(cudaSetDevice(S->dev));
      PST_CUDA(cudaStreamWaitEvent(S->stream, c->done[s + 1], 0));
    }
    GraphKey key;
    key.k = {2, i % ring_period(K)};
    run_program(c, s, key, [&](cudaStream_t st) { enqueue_np(c, s, i, false, st); });
    PST_CUDA(cudaEventRecord(c->done[c->local_index(s)], S->stream));
  }
  c->t += 1;
}

static void sync_all(pst_ctx* c) {
  for (auto* v : {&c->stages, &c->bks})
    for (auto& S : *v) {
      PST_CUDA(cudaSetDevice(S->dev));
      PST_CUDA(cudaStreamSynchronize(S->stream));
    }
}

// ------------------------------------------------------------------ ABI
extern "C" {

int pst_create(const pst_net* net, const pst_partition* part, const pst_hparams* hp, const pst_dist* dist,
               pst_ctx** out) {
  if (!out) return PST_E_INVALID;
  *out = nullptr;
  auto* c = new pst_ctx();
  int rc = guard(nullptr, [&] {
    PST_CHECK_ARG(net && part && hp, "null argument");
    PST_CHECK_ARG(net->init_params != nullptr, "init_params is null");
    c->net = derive_net(*net);
    PST_CHECK_ARG(net->n_params == c->net.n_params, "n_params does not match the network");
    c->K = part->n_stages;
    c->ranges = partition(c->net, c->K, part->ppv);
    PST_CHECK_ARG(hp->batch >= 1 && hp->batch <= 4096, "batch");
    PST_CHECK_ARG(hp->lr_pipelined != nullptr, "lr_pipelined");
    PST_CHECK_ARG((hp->solver == 0 || hp->solver == 1) && (hp->nesterov == 0 || hp->nesterov == 1) &&
                      (hp->lr_policy == 0 || hp->lr_policy == 1),
                  "solver / nesterov / lr_policy");
    c->batch = hp->batch;
    c->hp = *hp;
    c->lr_pipe.assign(hp->lr_pipelined, hp->lr_pipelined + c->K);
    c->hp.lr_pipelined = c->lr_pipe.data();
    if (hp->n_milestones > 0) {
      PST_CHECK_ARG(hp->milestone_epochs != nullptr, "milestones");
      c->milestones.assign(hp->milestone_epochs, hp->milestone_epochs + hp->n_milestones);
    }
    c->hp.milestone_epochs = c->milestones.data();
    int ndev = 0;
    PST_CUDA(cudaGetDeviceCount(&ndev));
    PST_CHECK_ARG(ndev >= 1, "no CUDA device");
    PST_CHECK_ARG(part->mapping == PST_MAP_PER_GPU || part->mapping == PST_MAP_FS_BKS, "mapping");
    c->mapping = part->mapping;
    if (c->mapping == PST_MAP_FS_BKS && dist)
      throw Unsupported("the FS/BKS mapping runs in local mode only (one process drives all 2K-1 accelerators)");
    const int ndevs = c->mapping == PST_MAP_FS_BKS ? 2 * c->K - 1 : c->K;
    c->devices.resize(ndevs);
    for (int s = 0; s < ndevs; ++s) {
      c->devices[s] = part->devices ? part->devices[s] : 0;
      PST_CHECK_ARG(c->devices[s] >= 0 && c->devices[s] < ndev, "device ordinal");
    }
    const char* g = std::getenv("PST_GRAPHS");
    c->use_graphs = !(g && std::string(g) == "0");
    if (dist) {
      PST_CHECK_ARG(dist->world == c->K && dist->rank >= 0 && dist->rank < c->K && dist->nccl_id,
                    "distributed: world must equal n_stages");
      c->dist = true;
      c->rank = dist->rank;
    }
    for (int s = 0; s < c->K; ++s) {
      if (!c->owns(s)) continue;
      c->stages.emplace_back(new Stage(c->net, s, c->K, c->ranges[s].first, c->ranges[s].second, c->devices[s],
                                       c->hp, net->init_params, c->batch));
      cudaEvent_t e;
      PST_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      PST_CUDA(cudaEventRecord(e, c->stages.back()->stream));
      c->done.push_back(e);
    }
    c->graphs.resize(c->stages.size());
    if (c->mapping == PST_MAP_FS_BKS) {   // BKS_s objects on their own accelerators
      for (int s = 0; s + 1 < c->K; ++s) {
        c->bks.emplace_back(new Stage(c->net, s, c->K, c->ranges[s].first, c->ranges[s].second, c->devices[c->K + s],
                                      c->hp, net->init_params, c->batch));
        cudaEvent_t e1, e2;
        PST_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        PST_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
        PST_CUDA(cudaEventRecord(e1, c->bks.back()->stream));
        c->bdone.push_back(e1);
        c->wev.push_back(e2);
      }
      c->graphs_b.resize(c->bks.size());
    }
    if (!c->dist) {  // peer access between distinct stage devices (best effort)
      for (int a = 0; a < (int)c->devices.size(); ++a)
        for (int b = 0; b < (int)c->devices.size(); ++b) {
          if (c->devices[a] == c->devices[b]) continue;
          int ok = 0;
          cudaDeviceCanAccessPeer(&ok, c->devices[a], c->devices[b]);
          if (ok) {
            cudaSetDevice(c->devices[a]);
            cudaDeviceEnablePeerAccess(c->devices[b], 0);
            cudaGetLastError();
          }
        }
    } else {
      ncclUniqueId id;
      std::memcpy(&id, dist->nccl_id, sizeof(id));
      PST_CUDA(cudaSetDevice(c->devices[c->rank]));
      PST_NCCL(ncclCommInitRank(&c->comm, c->K, id, c->rank));
      // Establish the P2P connections to both neighbours eagerly (one small exchange outside any
      // stream capture): NCCL connects lazily on first use, and the step graphs capture the
      // exchange, so the first captured send/recv must find the connection already set up.
      Stage* S = c->stages[0].get();
      void* wbuf = nullptr;
      PST_CUDA(cudaMalloc(&wbuf, 2 * 256));
      PST_CUDA(cudaMemset(wbuf, 0, 2 * 256));
      const int s = c->rank;
      for (int pass = 0; pass < 2; ++pass) {   // fwd direction, then bwd direction
        PST_NCCL(ncclGroupStart());
        if (pass == 0 && s < c->K - 1) PST_NCCL(ncclSend(wbuf, 256, ncclUint8, s + 1, c->comm, S->stream));
        if (pass == 0 && s > 0) PST_NCCL(ncclRecv((char*)wbuf + 256, 256, ncclUint8, s - 1, c->comm, S->stream));
        if (pass == 1 && s > 0) PST_NCCL(ncclSend(wbuf, 256, ncclUint8, s - 1, c->comm, S->stream));
        if (pass == 1 && s < c->K - 1) PST_NCCL(ncclRecv((char*)wbuf + 256, 256, ncclUint8, s + 1, c->comm, S->stream));
        PST_NCCL(ncclGroupEnd());
      }
      PST_CUDA(cudaStreamSynchronize(S->stream));
      PST_CUDA(cudaFree(wbuf));
    }
    const size_t xb = (size_t)c->batch * c->net.in_C * c->net.in_H * c->net.in_W;
    for (int i = 0; i < 2; ++i) {
      PST_CUDA(cudaMallocHost(&c->pin_x[i], xb * sizeof(float)));
      PST_CUDA(cudaMallocHost(&c->pin_y[i], c->batch * sizeof(int32_t)));
      PST_CUDA(cudaEventCreateWithFlags(&c->pin_ev[i], cudaEventDisableTiming));
      PST_CUDA(cudaEventCreateWithFlags(&c->pin_ev2[i], cudaEventDisableTiming));
    }
    PST_CUDA(cudaSetDevice(c->stages[0]->dev));
    PST_CUDA(cudaEventCreateWithFlags(&c->prod_ev, cudaEventDisableTiming));
  });
  if (rc != PST_OK) {
    g_last_global_error = c->err.empty() ? g_last_global_error : c->err;
    pst_destroy(c);
    return rc;
  }
  *out = c;
  return PST_OK;
}

int pst_step(pst_ctx* c, const pst_batch* batch) {
  if (!c) return PST_E_INVALID;
  return guard(c, [&] {
    PST_CHECK_ARG(batch != nullptr, "batch is null");
    if (c->mode == MODE_PIPE && c->n_fed >= c->n_p) {
      drain(c);
      c->mode = MODE_NP;
    }
    const int64_t mb = c->n_fed;
    // stage the batch: x into stage 0, labels into the last stage's ring
    const size_t xb = (size_t)c->batch * c->net.in_C * c->net.in_H * c->net.in_W;
    const int pi = c->pin_i;
    c->pin_i ^= 1;
    Stage* S0 = c->stage(0);
    Stage* SL = c->stage(c->K - 1);
    // The previous step's batch copies must have executed before this call returns (pst_batch
    // lifetime: a device batch stays valid until the next pst_step/pst_flush/pst_sync) and before
    // the pinned slot of two steps ago is reused.  The copy of step t-1 sits on the stage stream
    // behind step t-2's work, so the host runs at most one step ahead of the device.
    PST_CUDA(cudaEventSynchronize(c->pin_ev[pi ^ 1]));
    PST_CUDA(cudaEventSynchronize(c->pin_ev2[pi ^ 1]));
    if (batch->on_device) {   // order the copies after the producer's work (pst_batch.stream)
      cudaStream_t prod = batch->stream ? (cudaStream_t)batch->stream : cudaStreamLegacy;
      PST_CUDA(cudaSetDevice(c->stages[0]->dev));   // prod_ev lives on the first owned stage's device
      PST_CUDA(cudaEventRecord(c->prod_ev, prod));
      for (Stage* S : {S0, SL})
        if (S) PST_CUDA(cudaStreamWaitEvent(S->stream, c->prod_ev, 0));
    }
    if (S0) {
      PST_CHECK_ARG(batch->x != nullptr, "batch x is null");
      PST_CUDA(cudaSetDevice(S0->dev));
      if (batch->on_device) {
        PST_CUDA(cudaMemcpyAsync(S0->stage_x(), batch->x, xb * sizeof(float), cudaMemcpyDeviceToDevice, S0->stream));
      } else {
        std::memcpy(c->pin_x[pi], batch->x, xb * sizeof(float));
        PST_CUDA(cudaMemcpyAsync(S0->stage_x(), c->pin_x[pi], xb * sizeof(float), cudaMemcpyHostToDevice, S0->stream));
      }
      PST_CUDA(cudaEventRecord(c->pin_ev[pi], S0->stream));
    }
    if (SL) {
      PST_CHECK_ARG(batch->y != nullptr, "batch y is null");
      PST_CUDA(cudaSetDevice(SL->dev));
      if (batch->on_device) {
        PST_CUDA(cudaMemcpyAsync(SL->label_slot(mb), batch->y, c->batch * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                 SL->stream));
      } else {
        std::memcpy(c->pin_y[pi], batch->y, c->batch * sizeof(int32_t));
        PST_CUDA(cudaMemcpyAsync(SL->label_slot(mb), c->pin_y[pi], c->batch * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, SL->stream));
      }
      PST_CUDA(cudaEventRecord(c->pin_ev2[pi], SL->stream));
    }
    c->n_fed += 1;
    if (c->mode == MODE_PIPE) {
      if (c->mapping == PST_MAP_FS_BKS) fsbks_step(c);
      else pipe_step(c);
    } else {
      np_step(c);
    }
  });
}

int pst_set_hybrid(pst_ctx* c, int64_t switch_epoch) {
  if (!c) return PST_E_INVALID;
  return guard(c, [&] {
    if (c->mode == MODE_NP) throw StateError("already switched to non-pipelined training");
    if (c->mapping == PST_MAP_FS_BKS) throw Unsupported("hybrid training with the FS/BKS mapping");
    const int64_t spe = c->hp.steps_per_epoch > 0 ? c->hp.steps_per_epoch : 1;
    c->n_p = switch_epoch < 0 ? INT64_MAX : switch_epoch * spe;
    if (c->n_p < c->n_fed) c->n_p = c->n_fed;  // switch at the next step
    for (auto& S : c->stages) S->set_n_p(c->n_p);
  });
}

int pst_flush(pst_ctx* c) {
  if (!c) return PST_E_INVALID;
  return guard(c, [&] { drain(c); });
}

int pst_weights(pst_ctx* c, uint32_t what, float* out, int64_t cap, int64_t* n) {
  if (!c || !n) return PST_E_INVALID;
  return guard(c, [&] {
    int64_t np = 0, nbn = 0;
    for (auto& S : c->stages) {
      np += S->n_params;
      for (int l = S->l0; l < S->l1; ++l)
        if (c->net.layers[l].spec.bn) nbn += 2 * c->net.layers[l].spec.cout;
    }
    int64_t need = 0;
    if (what & PST_W_PARAMS) need += np;
    if (what & PST_W_MOMENTUM) need += np;
    if (what & PST_W_BNSTATS) need += nbn;
    *n = need;
    if (!out) return;
    PST_CHECK_ARG(cap >= need, "output buffer too small");
    sync_all(c);
    int64_t o = 0;
    // the master weights and momentum live with the backward stage (FS/BKS mapping: BKS_s)
    auto master = [&](size_t i) -> Stage* { return i < c->bks.size() ? c->bks[i].get() : c->stages[i].get(); };
    if (what & PST_W_PARAMS)
      for (size_t i = 0; i < c->stages.size(); ++i) { master(i)->read_params(out + o, nullptr); o += master(i)->n_params; }
    if (what & PST_W_MOMENTUM)
      for (size_t i = 0; i < c->stages.size(); ++i) { master(i)->read_params(nullptr, out + o); o += master(i)->n_params; }
    if (what & PST_W_BNSTATS) {
      std::vector<float> mv;
      for (auto& S : c->stages) S->read_bnstats(mv);
      std::memcpy(out + o, mv.data(), mv.size() * sizeof(float));
    }
  });
}

int pst_losses(pst_ctx* c, int64_t first_mb, int64_t n, float* out) {
  if (!c || (n > 0 && !out) || first_mb < 0 || n < 0) return PST_E_INVALID;
  return guard(c, [&] {
    Stage* SL = c->stage(c->K - 1);
    if (!SL) throw StateError("losses live on the last stage's rank");
    PST_CHECK_ARG(n <= 1024, "at most 1024 losses are kept");
    if (first_mb + n > c->n_loss || first_mb < c->n_loss - 1024)
      throw StateError("losses of mini-batches [" + std::to_string(first_mb) + ", " + std::to_string(first_mb + n) +
                       ") are not available (computed: [" + std::to_string(std::max<int64_t>(0, c->n_loss - 1024)) +
                       ", " + std::to_string(c->n_loss) + "))");
    PST_CUDA(cudaSetDevice(SL->dev));
    PST_CUDA(cudaStreamSynchronize(SL->stream));
    SL->read_losses(first_mb, n, out);
  });
}

int pst_versions(pst_ctx* c, int64_t* v, int32_t cap) {
  if (!c || !v) return PST_E_INVALID;
  return guard(c, [&] {
    PST_CHECK_ARG(cap >= (int32_t)c->stages.size(), "cap");
    sync_all(c);
    for (size_t i = 0; i < c->stages.size(); ++i)
      v[i] = (i < c->bks.size() ? c->bks[i] : c->stages[i])->read_version();
  });
}

int pst_progress(pst_ctx* c, int64_t* steps, int64_t* fed) {
  if (!c) return PST_E_INVALID;
  if (steps) *steps = c->t;
  if (fed) *fed = c->n_fed;
  return c->sticky ? c->sticky : PST_OK;
}

int pst_stream(pst_ctx* c, int32_t stage, void** stream) {
  if (!c || !stream) return PST_E_INVALID;
  return guard(c, [&] {
    PST_CHECK_ARG(stage >= 0 && stage < c->K && c->owns(stage), "stage not owned by this context");
    *stream = (void*)c->stage(stage)->stream;
  });
}

int pst_sync(pst_ctx* c) {
  if (!c) return PST_E_INVALID;
  return guard(c, [&] { sync_all(c); });
}

void pst_destroy(pst_ctx* c) {
  if (!c) return;
  for (auto* v : {&c->stages, &c->bks})
    for (auto& S : *v) {
      cudaSetDevice(S->dev);
      cudaStreamSynchronize(S->stream);
    }
  for (auto* gv : {&c->graphs, &c->graphs_b})
    for (auto& m : *gv)
      for (auto& kv : m) cudaGraphExecDestroy(kv.second.exec);
  for (auto e : c->bdone) cudaEventDestroy(e);
  for (auto e : c->wev) cudaEventDestroy(e);
  c->bks.clear();
  for (auto e : c->done) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (c->pin_x[i]) cudaFreeHost(c->pin_x[i]);
    if (c->pin_y[i]) cudaFreeHost(c->pin_y[i]);
    if (c->pin_ev[i]) cudaEventDestroy(c->pin_ev[i]);
    if (c->pin_ev2[i]) cudaEventDestroy(c->pin_ev2[i]);
  }
  if (c->prod_ev) cudaEventDestroy(c->prod_ev);
  for (auto e : c->st_beg) cudaEventDestroy(e);
  for (auto e : c->st_end) cudaEventDestroy(e);
  if (c->comm) ncclCommDestroy(c->comm);
  c->stages.clear();
  delete c;
}

const char* pst_last_error(const pst_ctx* c) {
  if (!c) return g_last_global_error.c_str();
  return c->err.c_str();
}

int pst_nccl_unique_id(void* out) {
  if (!out) return PST_E_INVALID;
  return guard(nullptr, [&] {
    static_assert(sizeof(ncclUniqueId) == PST_NCCL_ID_BYTES, "nccl id size");
    ncclUniqueId id;
    PST_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

int pst_partition_ranges(const pst_net* net, const pst_partition* part, int32_t* ranges) {
  if (!net || !part || !ranges) return PST_E_INVALID;
  return guard(nullptr, [&] {
    NetInfo ni = derive_net(*net);
    auto r = partition(ni, part->n_stages, part->ppv);
    for (size_t s = 0; s < r.size(); ++s) {
      ranges[2 * s] = r[s].first;
      ranges[2 * s + 1] = r[s].second;
    }
  });
}

int64_t pst_param_count(const pst_net* net) {
  if (!net) return PST_E_INVALID;
  int64_t n = -1;
  int rc = guard(nullptr, [&] { n = derive_net(*net).n_params; });
  return rc == PST_OK ? n : rc;
}

int pst_schedule(int32_t K, int32_t s, int64_t t, int64_t n_total, int64_t* bwd_mb, int64_t* fwd_mb,
                 int64_t* fwd_version) {
  if (K < 1 || s < 0 || s >= K || t < 0 || !bwd_mb || !fwd_mb || !fwd_version) return PST_E_INVALID;
  const int64_t nf = n_total < 0 ? INT64_MAX : n_total;
  StepPlan p = plan_step(K, s, t, 0, 0, std::min<int64_t>(nf, t + 1));
  *bwd_mb = p.bwd_mb;
  *fwd_mb = p.fwd_mb;
  // updates applied by stage s before its forward at step t = backwards at steps <= t
  // (backward runs first within a step): mini-batches 0 .. t-2K+1+s
  int64_t done = t - 2 * K + 2 + s;
  if (done < 0) done = 0;
  if (done > nf) done = nf;
  *fwd_version = p.fwd_mb >= 0 ? done : -1;
  return PST_OK;
}

int pst_launches(pst_ctx* c, int64_t* n) {
  if (!c || !n) return PST_E_INVALID;
  *n = prof::launches;
  return PST_OK;
}

int pst_profile(pst_ctx* c, int32_t enable) {
  if (!c) return PST_E_INVALID;
  return guard(c, [&] {
    sync_all(c);
    prof::read(-1, nullptr, nullptr, nullptr, nullptr);
    prof::enabled = enable != 0;
  });
}

int pst_stage_timing(pst_ctx* c, int32_t enable) {
  if (!c) return PST_E_INVALID;
  return guard(c, [&] {
    if (c->mapping == PST_MAP_FS_BKS) throw Unsupported("per-stage timing with the FS/BKS mapping");
    sync_all(c);
    if (c->st_beg.empty()) {
      for (size_t i = 0; i < c->stages.size(); ++i) {
        PST_CUDA(cudaSetDevice(c->stages[i]->dev));
        cudaEvent_t a, b;
        PST_CUDA(cudaEventCreate(&a));
        PST_CUDA(cudaEventCreate(&b));
        PST_CUDA(cudaEventRecord(a, c->stages[i]->stream));
        PST_CUDA(cudaEventRecord(b, c->stages[i]->stream));
        c->st_beg.push_back(a);
        c->st_end.push_back(b);
      }
    }
    c->st_ms.assign(c->stages.size(), 0.0);
    c->st_steps = 0;
    c->stage_timing = enable != 0;
  });
}

int pst_stage_times(pst_ctx* c, double* ms, int32_t cap, int64_t* steps) {
  if (!c || !ms) return PST_E_INVALID;
  return guard(c, [&] {
    PST_CHECK_ARG(cap >= (int32_t)c->stages.size(), "cap");
    sync_all(c);
    for (size_t i = 0; i < c->stages.size(); ++i) ms[i] = i < c->st_ms.size() ? c->st_ms[i] : 0.0;
    if (steps) *steps = c->st_steps;
  });
}

int pst_profile_read(pst_ctx* c, int32_t cls, double* ms, int64_t* launches, double* bytes, double* flops) {
  if (!c) return PST_E_INVALID;
  return guard(c, [&] {
    PST_CHECK_ARG(cls >= 0 && cls < prof::NCLS, "kernel class");
    sync_all(c);
    prof::read(cls, ms, launches, bytes, flops);
  });
}

int pst_memory(pst_ctx* c, int32_t stage, int64_t* out, int32_t cap) {
  if (!c || !out) return PST_E_INVALID;
  return guard(c, [&] {
    PST_CHECK_ARG(stage >= 0 && stage < c->K && c->owns(stage), "stage not owned by this context");
    PST_CHECK_ARG(cap >= 5, "cap");
    Stage* S = c->stage(stage);
    out[0] = (int64_t)S->bytes_total;
    out[1] = S->R;
    out[2] = 2 * (c->K - stage) - 1;
    if (cap >= 6) out[5] = S->Rin;
    out[3] = (int64_t)S->bytes_slot;
    out[4] = S->n_params * (int64_t)sizeof(float);
  });
}

int pst_ring_slots(int32_t K, int32_t s, int32_t* saved, int32_t* input, int32_t* period) {
  if (K < 1 || s < 0 || s >= K || !saved || !input || !period) return PST_E_INVALID;
  *saved = ring_saved(K, s);
  *input = ring_input(K, s);
  *period = ring_period(K);
  return PST_OK;
}

const char* pst_build_info(void) {
  return "libpst sm_100a act=" PST_ACT_NAME " tcgen05+TMA implicit-GEMM conv, NCCL " ;
}

}  // extern "C"
