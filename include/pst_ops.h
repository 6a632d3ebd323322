/*
 * pst_ops.h -- single-operation entry points of libpst.so, for kernel-level
 * parity tests against the CPU oracle.  Each call runs the SAME sm_100a kernels
 * the pipeline uses (tcgen05 implicit-GEMM convolution; layout conversion) on
 * device buffers and blocks until done.  Not needed to train.
 *
 * All pointers are DEVICE pointers to float32 tensors in NCHW (activations),
 * OIHW (weights) layout.  Inputs are rounded to the library's compute dtype
 * (pst_build_info) on entry; accumulation is float32.  Shapes: x [N][Cin][H][W],
 * w [Cout][Cin][k][k], y / gy [N][Cout][Ho][Wo] with Ho = (H+2pad-k)/stride+1.
 * stride 1 or 2 (stride 2 requires k=3, pad=1 for dgrad).  An FC layer is the
 * case H = W = k = 1.  Returns pst_status; message via pst_last_error(NULL).
 *
 *   fwd:   y[n,o,i,j]  = sum_{c,r,s} w[o,c,r,s] x[n,c,i*S+r-pad,j*S+s-pad]
 *   dgrad: gx[n,c,h,w] = sum_{o,r,s} w[o,c,r,s] gy[n,o,(h+pad-r)/S,(w+pad-s)/S]  (L47, current W)
 *   wgrad: gw[o,c,r,s] = sum_{n,i,j} gy[n,o,i,j] x[n,c,i*S+r-pad,j*S+s-pad]     (L47, saved x)
 */
#ifndef PST_OPS_H_
#define PST_OPS_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

int pst_op_conv2d_fwd(const float* x, const float* w, float* y, int N, int Cin, int H, int W, int Cout,
                      int k, int stride, int pad);
int pst_op_conv2d_dgrad(const float* gy, const float* w, float* gx, int N, int Cin, int H, int W, int Cout,
                        int k, int stride, int pad);
int pst_op_conv2d_wgrad(const float* x, const float* gy, float* gw, int N, int Cin, int H, int W, int Cout,
                        int k, int stride, int pad);
/* Tuning aid: mean device time (microseconds, *us) of one fwd (which=0, BN-statistics
 * epilogue), dgrad (1, stride 1) or wgrad (2) launch of this shape on resident zero buffers,
 * `iters` launches replayed as one CUDA graph after a warm-up replay. */
int pst_op_time_conv(int which, int N, int Cin, int H, int W, int Cout, int k, int stride, int pad,
                     int iters, float* us);
/* Message of the last failing pst_op_* call on this thread. */
const char* pst_op_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
