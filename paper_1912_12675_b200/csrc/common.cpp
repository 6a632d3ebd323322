#include <algorithm>
#include <cstdlib>
// common.cpp -- tensor-map encoding and device queries.
#include "common.h"

#include <cudaTypedefs.h>
#include <mutex>
#include <vector>

namespace pst {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static void load_encode() {
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PST_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn)
      throw CudaError("cuTensorMapEncodeTiled entry point not found");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
}

CUtensorMap make_tmap(CUtensorMapDataType dt, int rank, const void* gaddr, const uint64_t* dims,
                      const uint64_t* strides_bytes, const uint32_t* box, const uint32_t* estrides) {
  load_encode();
  CUtensorMap m;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = estrides ? estrides[i] : 1;
  }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  CUresult r = g_encode(&m, dt, (cuuint32_t)rank, const_cast<void*>(gaddr), d, s, b, e,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::string msg = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rank=" +
                      std::to_string(rank) + " dims=";
    for (int i = 0; i < rank; ++i) msg += std::to_string(dims[i]) + ",";
    msg += " box=";
    for (int i = 0; i < rank; ++i) msg += std::to_string(box[i]) + ",";
    throw CudaError(msg);
  }
  return m;
}

int pst_knob(const char* name, int dflt) {
#ifdef PST_EXPERIMENTS
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

int wgrad_sms(int device) {
  static const int over = pst_knob("PST_WG_SMS", 0);
  const int n = num_sms(device);
  return over > 0 ? std::min(over, n) : n;
}

int num_sms(int device) {
  static int cache[64] = {0};
  if (device >= 0 && device < 64 && cache[device]) return cache[device];
  int n = 0;
  PST_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
  if (device >= 0 && device < 64) cache[device] = n;
  return n;
}

namespace prof {
thread_local int64_t launches = 0;
bool enabled = false;
namespace {
struct Rec { cudaEvent_t a, b; int cls; double bytes, flops; };
std::vector<Rec> pending;
cudaEvent_t open_ev = nullptr;
double tot_ms[NCLS], tot_bytes[NCLS], tot_flops[NCLS];
int64_t tot_n[NCLS];
}  // namespace

void begin(cudaStream_t st) {
  ++launches;
  if (!enabled) return;
  PST_CUDA(cudaEventCreate(&open_ev));
  PST_CUDA(cudaEventRecord(open_ev, st));
}

void end(cudaStream_t st, int cls, double b, double f) {
  if (!enabled || !open_ev) return;
  cudaEvent_t e;
  PST_CUDA(cudaEventCreate(&e));
  PST_CUDA(cudaEventRecord(e, st));
  pending.push_back({open_ev, e, cls, b, f});
  open_ev = nullptr;
}

void read(int cls, double* ms, int64_t* n, double* bytes, double* flops) {
  for (Rec& r : pending) {
    float t = 0.f;
    PST_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    tot_ms[r.cls] += t;
    tot_bytes[r.cls] += r.bytes;
    tot_flops[r.cls] += r.flops;
    tot_n[r.cls] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  pending.clear();
  if (cls < 0 || cls >= NCLS) {
    for (int i = 0; i < NCLS; ++i) tot_ms[i] = tot_bytes[i] = tot_flops[i] = 0, tot_n[i] = 0;
    return;
  }
  if (ms) *ms = tot_ms[cls];
  if (n) *n = tot_n[cls];
  if (bytes) *bytes = tot_bytes[cls];
  if (flops) *flops = tot_flops[cls];
}
}  // namespace prof

}  // namespace pst

namespace pst {
thread_local bool pdl_suppressed = false;
bool pdl_enabled() {
  static const bool on = pst_knob("PST_PDL", 1) != 0;
  return on;
}
}  // namespace pst
