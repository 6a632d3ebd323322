// ops_api.cu -- include/pst_ops.h: single convolution passes on the tcgen05 path.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/pst.h"
#include "../../include/pst_ops.h"
#include "common.h"
#include "kernels.h"

using namespace pst;

namespace {

struct Scratch {
  std::vector<void*> p;
  template <typename T> T* get(size_t n) {
    void* q = nullptr;
    PST_CUDA(cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)));
    PST_CUDA(cudaMemset(q, 0, std::max<size_t>(n, 1) * sizeof(T)));
    p.push_back(q);
    return static_cast<T*>(q);
  }
  ~Scratch() { for (void* q : p) cudaFree(q); }
};

thread_local std::string g_err;

template <typename F>
int run(F&& f) {
  try {
    f();
    return PST_OK;
  } catch (const InvalidArg& e) { g_err = e.what(); return PST_E_INVALID; }
  catch (const Unsupported& e) { g_err = e.what(); return PST_E_UNSUPPORTED; }
  catch (const std::exception& e) { g_err = e.what(); return PST_E_CUDA; }
}

struct Geo {
  int N, Cin, H, W, Cout, k, S, pad, Ho, Wo, Cinp, Coutp;
};
Geo geo(int N, int Cin, int H, int W, int Cout, int k, int S, int pad) {
  PST_CHECK_ARG(N > 0 && Cin > 0 && H > 0 && W > 0 && Cout > 0 && k > 0 && pad >= 0, "shape");
  PST_CHECK_ARG(S == 1 || S == 2, "stride");
  Geo g{N, Cin, H, W, Cout, k, S, pad, (H + 2 * pad - k) / S + 1, (W + 2 * pad - k) / S + 1,
        round_up(Cin, 16), round_up(Cout, 16)};
  PST_CHECK_ARG(g.Ho > 0 && g.Wo > 0, "empty output");
  return g;
}

}  // namespace

extern "C" {

int pst_op_conv2d_fwd(const float* x, const float* w, float* y, int N, int Cin, int H, int W, int Cout, int k,
                      int stride, int pad) {
  return run([&] {
    Geo g = geo(N, Cin, H, W, Cout, k, stride, pad);
    Scratch s;
    act_t* xa = s.get<act_t>((size_t)N * H * W * g.Cinp);
    act_t* sf = s.get<act_t>((size_t)k * k * g.Coutp * g.Cinp * (PST_SPLIT ? 2 : 1));
    act_t* sb = s.get<act_t>((size_t)k * k * g.Coutp * g.Cinp * (PST_SPLIT ? 2 : 1));
    float* yo = s.get<float>((size_t)N * g.Ho * g.Wo * g.Coutp);
    input_to_act(x, xa, N, Cin, H, W, g.Cinp, 0);
    conv_weights_to_shadows(w, Cout, Cin, k, g.Coutp, g.Cinp, sf, sb, 0);
    ConvSpec c{};
    c.in = xa; c.N = N; c.H = H; c.W = W; c.Cinp = g.Cinp;
    c.Ho = g.Ho; c.Wo = g.Wo; c.Coutp = g.Coutp; c.Cout = Cout;
    c.k = k; c.S = stride; c.off = -pad; c.sgn = 1;
    c.wshadow = sf; c.epi = EPI_BIAS_F32; c.out = yo;
    const bool tl = pst_knob("PST_DBG_TL", 0) != 0;
    if (tl) c.dbg = s.get<unsigned long long>(8 * 256);
    conv_tc(c, 0);
    if (tl) {  // debug: print CTA 0's timeline (us since kernel start)
      std::vector<unsigned long long> h(8 * 256);
      PST_CUDA(cudaMemcpy(h.data(), c.dbg, h.size() * 8, cudaMemcpyDeviceToHost));
      const char* names[8] = {"prod_issue", "ev1", "ev2", "ev3", "ev4", "epi_start", "epi_done", "start"};
      std::printf("TL prologue  barriers %.2f  tmem %.2f  sync %.2f  pdl_wait %.2f\n",
                  (double)(long long)(h[7 * 256 + 1] - h[7 * 256]) / 1e3, (double)(long long)(h[7 * 256 + 2] - h[7 * 256]) / 1e3,
                  (double)(long long)(h[7 * 256 + 3] - h[7 * 256]) / 1e3, (double)(long long)(h[7 * 256 + 4] - h[7 * 256]) / 1e3);
      for (int e = 0; e < 7; ++e) {
        std::printf("TL %-10s", names[e]);
        for (int i = 0; i < 40 && h[e * 256 + i]; ++i) std::printf(" %7.2f", (double)(long long)(h[e * 256 + i] - h[7 * 256]) / 1e3);
        std::printf("\n");
      }
    }
    act_to_nchw(yo, 1, y, N, Cout, g.Ho, g.Wo, 0);
    PST_CUDA(cudaDeviceSynchronize());
  });
}

int pst_op_conv2d_dgrad(const float* gy, const float* w, float* gx, int N, int Cin, int H, int W, int Cout, int k,
                        int stride, int pad) {
  return run([&] {
    Geo g = geo(N, Cin, H, W, Cout, k, stride, pad);
    if (stride == 2) PST_CHECK_ARG(k == 3 && pad == 1, "stride-2 dgrad needs k=3, pad=1");
    Scratch s;
    act_t* ga = s.get<act_t>((size_t)N * g.Ho * g.Wo * g.Coutp);
    act_t* sf = s.get<act_t>((size_t)k * k * g.Coutp * g.Cinp * (PST_SPLIT ? 2 : 1));
    act_t* sb = s.get<act_t>((size_t)k * k * g.Coutp * g.Cinp * (PST_SPLIT ? 2 : 1));
    act_t* gxa = s.get<act_t>((size_t)N * H * W * g.Cinp);
    input_to_act(gy, ga, N, Cout, g.Ho, g.Wo, g.Coutp, 0);
    conv_weights_to_shadows(w, Cout, Cin, k, g.Coutp, g.Cinp, sf, sb, 0);
    const act_t* src = ga;
    int sH = g.Ho, sW = g.Wo;
    if (stride == 2) {
      act_t* dil = s.get<act_t>((size_t)N * H * W * g.Coutp);
      dilate2(ga, dil, N, g.Ho, g.Wo, H, W, g.Coutp, 0);
      src = dil; sH = H; sW = W;
    }
    ConvSpec c{};
    c.in = src; c.N = N; c.H = sH; c.W = sW; c.Cinp = g.Coutp;
    c.Ho = H; c.Wo = W; c.Coutp = g.Cinp; c.Cout = Cin;
    c.k = k; c.S = 1; c.off = pad; c.sgn = -1;
    c.wshadow = sb; c.epi = EPI_DGRAD; c.out = gxa;
    conv_tc(c, 0);
    act_to_nchw(gxa, 0, gx, N, Cin, H, W, 0);
    PST_CUDA(cudaDeviceSynchronize());
  });
}

int pst_op_conv2d_wgrad(const float* x, const float* gy, float* gw, int N, int Cin, int H, int W, int Cout, int k,
                        int stride, int pad) {
  return run([&] {
    Geo g = geo(N, Cin, H, W, Cout, k, stride, pad);
    Scratch s;
    act_t* xa = s.get<act_t>((size_t)N * H * W * g.Cinp);
    act_t* ga = s.get<act_t>((size_t)N * g.Ho * g.Wo * g.Coutp);
    input_to_act(x, xa, N, Cin, H, W, g.Cinp, 0);
    input_to_act(gy, ga, N, Cout, g.Ho, g.Wo, g.Coutp, 0);
    int dev;
    PST_CUDA(cudaGetDevice(&dev));
    WgradPlan p = wgrad_plan(N, H, W, g.Cinp, g.Ho, g.Wo, g.Coutp, k, stride, pad, wgrad_sms(dev));
    float* part = s.get<float>((size_t)p.part_floats);
    WgradSpec wg{};
    wg.x = xa; wg.N = N; wg.H = H; wg.W = W; wg.Cinp = g.Cinp;
    wg.dy = ga; wg.Ho = g.Ho; wg.Wo = g.Wo; wg.Coutp = g.Coutp;
    wg.k = k; wg.S = stride; wg.pad = pad; wg.part = part; wg.ksplit = p.ksplit;
    const bool tl = pst_knob("PST_DBG_TL", 0) != 0;
    if (tl) wg.dbg = s.get<unsigned long long>(8 * 256);
    conv_wgrad_tc(wg, 0);
    if (tl) {
      std::vector<unsigned long long> h(8 * 256);
      PST_CUDA(cudaMemcpy(h.data(), wg.dbg, h.size() * 8, cudaMemcpyDeviceToHost));
      const char* names[8] = {"prod_issue", "conv_full", "conv_ready", "mma_start", "mma_commit", "epi_start",
                              "epi_done", "start"};
      for (int e = 0; e < 6; ++e) {
        std::printf("TLW %-10s", names[e]);
        for (int i = 0; i < 40 && h[e * 256 + i]; ++i) std::printf(" %7.2f", (double)(long long)(h[e * 256 + i] - h[7 * 256]) / 1e3);
        std::printf("\n");
      }
    }
    wgrad_reduce(part, p.ksplit, g.Coutp, g.Cinp, Cout, Cin, k, gw, 0);
    PST_CUDA(cudaDeviceSynchronize());
  });
}

}  // extern "C"

// error text for ops calls: pst_last_error(NULL) returns the global message of pst_api.cu;
// ops keep their own, exported for the binding.
extern "C" const char* pst_op_last_error(void) { return g_err.c_str(); }

// Kernel timing for tuning (tools/conv_lab.py): `which` 0 fwd, 1 dgrad, 2 wgrad of one
// convolution shape on resident device buffers; warm-up, then `iters` launches timed with CUDA
// events on one stream; *us = mean microseconds per launch.  Inputs are zero (MMA and TMA time
// do not depend on values).
extern "C" int pst_op_time_conv(int which, int N, int Cin, int H, int W, int Cout, int k, int stride, int pad,
                                int iters, float* us) {
  return run([&] {
    Geo g = geo(N, Cin, H, W, Cout, k, stride, pad);
    Scratch s;
    cudaStream_t st;
    PST_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    act_t* xa = s.get<act_t>((size_t)N * H * W * g.Cinp);
    act_t* ya = s.get<act_t>((size_t)N * g.Ho * g.Wo * g.Coutp);
    act_t* sf = s.get<act_t>((size_t)k * k * g.Coutp * g.Cinp * (PST_SPLIT ? 2 : 1));
    double* stats = s.get<double>((size_t)2 * g.Coutp);
    int dev;
    PST_CUDA(cudaGetDevice(&dev));
    WgradPlan p = wgrad_plan(N, H, W, g.Cinp, g.Ho, g.Wo, g.Coutp, k, stride, pad, wgrad_sms(dev));
    float* part = which == 2 ? s.get<float>((size_t)p.part_floats) : nullptr;
    auto launch = [&] {
      if (which == 0) {
        ConvSpec c{};
        c.in = xa; c.N = N; c.H = H; c.W = W; c.Cinp = g.Cinp;
        c.Ho = g.Ho; c.Wo = g.Wo; c.Coutp = g.Coutp; c.Cout = Cout;
        c.k = k; c.S = stride; c.off = -pad; c.sgn = 1;
        c.wshadow = sf; c.epi = EPI_BN_STATS; c.out = ya; c.stats = stats;
        conv_tc(c, st);
      } else if (which == 1) {
        PST_CHECK_ARG(stride == 1, "time dgrad: stride 1 only");
        ConvSpec c{};
        c.in = ya; c.N = N; c.H = g.Ho; c.W = g.Wo; c.Cinp = g.Coutp;
        c.Ho = H; c.Wo = W; c.Coutp = g.Cinp; c.Cout = Cin;
        c.k = k; c.S = 1; c.off = pad; c.sgn = -1;
        c.wshadow = sf; c.epi = EPI_DGRAD; c.out = xa;
        conv_tc(c, st);
      } else {
        WgradSpec wg{};
        wg.x = xa; wg.N = N; wg.H = H; wg.W = W; wg.Cinp = g.Cinp;
        wg.dy = ya; wg.Ho = g.Ho; wg.Wo = g.Wo; wg.Coutp = g.Coutp;
        wg.k = k; wg.S = stride; wg.pad = pad; wg.part = part; wg.ksplit = p.ksplit;
        conv_wgrad_tc(wg, st);
      }
    };
    // the timed launches are one CUDA graph (as in the pipeline), so host launch cost is excluded
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    PST_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) launch();
    PST_CUDA(cudaStreamEndCapture(st, &graph));
    PST_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    PST_CUDA(cudaGraphLaunch(exec, st));
    cudaEvent_t e0, e1;
    PST_CUDA(cudaEventCreate(&e0));
    PST_CUDA(cudaEventCreate(&e1));
    PST_CUDA(cudaEventRecord(e0, st));
    PST_CUDA(cudaGraphLaunch(exec, st));
    PST_CUDA(cudaEventRecord(e1, st));
    PST_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PST_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *us = ms * 1e3f / (float)iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    PST_CUDA(cudaStreamSynchronize(st));
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(st);
  });
}
