// common.h -- shared host/device utilities for libpst (B200, sm_100a).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace pst {

// Compute precision of the tensor-core path (one per library build):
//   default        PST_PREC_TF32X3: activations/gradients/weight shadows stored as
//                  float32; every tensor-core product is split 3xTF32
//                  (a*b ~= ahi*bhi + ahi*blo + alo*bhi, hi = tf32 truncation) so the
//                  convolutions are float32-accurate.
//   PST_PREC_BF16  bf16 storage, one bf16 MMA per product (fast; does not meet the
//                  north-star weight tolerance).
//   PST_ACT_FP16   fp16 storage, one fp16 MMA (diagnostics only).
// Accumulation, master weights, BN statistics and softmax are always float32.
#if defined(PST_ACT_FP16)
typedef __half act_t;
#define PST_ACT_NAME "f16"
#define PST_KIND_TF32 0
#define PST_SPLIT 0
#define PST_AB_FORMAT 0
#elif defined(PST_PREC_BF16)
typedef __nv_bfloat16 act_t;
#define PST_ACT_NAME "bf16"
#define PST_KIND_TF32 0
#define PST_SPLIT 0
#define PST_AB_FORMAT 1
#else
typedef float act_t;
#define PST_ACT_NAME "f32-tf32x3"
#define PST_KIND_TF32 1
#define PST_SPLIT 1
#define PST_AB_FORMAT 2
#endif
// elements of act_t per 16-byte chunk (the unit of TMA boxes and UMMA core matrices)
constexpr int kEPC = 16 / (int)sizeof(act_t);

__host__ __device__ inline float act2f(act_t v) {
#if defined(PST_ACT_FP16)
  return __half2float(v);
#elif defined(PST_PREC_BF16)
  return __bfloat162float(v);
#else
  return v;
#endif
}
__host__ __device__ inline act_t f2act(float v) {
#if defined(PST_ACT_FP16)
  return __float2half_rn(v);
#elif defined(PST_PREC_BF16)
  return __float2bfloat16_rn(v);
#else
  return v;
#endif
}
// low part of the 3xTF32 split: v - trunc_tf32(v) (exact in float32)
__host__ __device__ inline float tf32_lo(float v) {
  union { float f; uint32_t u; } a;
  a.f = v;
  a.u &= 0xFFFFE000u;
  return v - a.f;
}

inline CUtensorMapDataType act_tmap_dtype() {
#if defined(PST_ACT_FP16)
  return CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
#elif defined(PST_PREC_BF16)
  return CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
#else
  return CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
#endif
}

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};
struct InvalidArg : std::runtime_error {
  explicit InvalidArg(const std::string& s) : std::runtime_error(s) {}
};
struct Unsupported : std::runtime_error {
  explicit Unsupported(const std::string& s) : std::runtime_error(s) {}
};
struct StateError : std::runtime_error {
  explicit StateError(const std::string& s) : std::runtime_error(s) {}
};
struct NcclError : std::runtime_error {
  explicit NcclError(const std::string& s) : std::runtime_error(s) {}
};

#define PST_CUDA(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::pst::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                  \
  } while (0)

#define PST_CHECK_ARG(cond, msg)                                         \
  do {                                                                   \
    if (!(cond)) throw ::pst::InvalidArg(std::string("invalid: ") + msg); \
  } while (0)

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
inline int64_t round_up64(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// CUtensorMap encoding through the runtime's driver entry point (no -lcuda).
CUtensorMap make_tmap(CUtensorMapDataType dt, int rank, const void* gaddr, const uint64_t* dims,
                      const uint64_t* strides_bytes /* rank-1 */, const uint32_t* box,
                      const uint32_t* estrides);

int num_sms(int device);
// SMs the weight-gradient kernels plan their split-K grid for (PST_WG_SMS; default all): the
// wgrad runs on a forked stream beside the dgrad, so it can be given part of the GPU.
int wgrad_sms(int device);

// Experiment switches (environment variables) exist only in builds with -DPST_EXPERIMENTS
// (tools/, A/B runs); the production library always takes the default.
int pst_knob(const char* name, int dflt);

// Launch accounting and optional per-kernel CUDA-event timing (bench.py's roofline).
// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the step is launched with the PDL attribute: its CTAs may become resident and
// run their prologue (barrier init, TMEM alloc, descriptor prefetch) while the previous kernel
// drains.  Kernels call pdl_wait() before their first global-memory access (read or write) and
// pdl_trigger() right after it, so kernel N starts only once kernel N-1 has passed its own wait,
// i.e. every kernel before N-1 is complete.  PST_PDL=0 disables the attribute (A/B timing).
// Exception: the kernels that write weight shadows (sgd_kernel, conv_w_shadow_kernel) never call
// pdl_trigger, so their dependents start only once they are complete; conv_ts_kernel relies on it
// to load a layer's weights before its pdl_wait.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
// Launches of this thread skip the programmatic-dependent-launch attribute while set (the forked
// wgrad stream: its next kernel's CTAs must not sit on SMs waiting while the dgrad needs them).
extern thread_local bool pdl_suppressed;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl_enabled() && !pdl_suppressed) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

namespace prof {
enum Cls { CONV_FWD = 0, CONV_DGRAD, CONV_WGRAD, BN_APPLY, BWD_PRE, BN_BWD, POOL, SGD, LOSS, MISC, NCLS };
extern thread_local int64_t launches;  // kernels enqueued by this thread (graph capture included)
extern bool enabled;                   // when true, launchers bracket kernels with events
void begin(cudaStream_t st);
void end(cudaStream_t st, int cls, double alg_bytes, double alg_flops);
// Resolves pending events (caller synchronised).  cls < 0 resets everything.
void read(int cls, double* ms, int64_t* n, double* bytes, double* flops);
}  // namespace prof

}  // namespace pst
