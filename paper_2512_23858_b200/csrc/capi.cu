// Library-level C ABI: version, thread-local error text, device check.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"
#include "host_util.h"

namespace ygg {
static thread_local char g_err[512] = "";

int ygg_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// Kernel-timeline tracing (profiling only) is armed per host thread: the state is thread_local, so
// one thread's armed buffer never receives another thread's launches and the library keeps no
// process-wide mutable state.
namespace {
thread_local unsigned long long* g_trace = nullptr;
thread_local int g_trace_cap = 0, g_trace_used = 0;
thread_local int g_trace_ids[4096];
}  // namespace

unsigned long long* trace_next(int kernel_id) {
  if (!g_trace || g_trace_used >= g_trace_cap) return nullptr;
  g_trace_ids[g_trace_used] = kernel_id;  // kept host-side: kernels only fill the timer fields
  return g_trace + 8 * g_trace_used++;
}
}  // namespace ygg

extern "C" {
int ygg_prepare_tree(void);
int ygg_prepare_gemm(void);
int ygg_prepare_layers(void);
int ygg_prepare_attn_tc(void);
int ygg_prepare_gemv(void);
int ygg_prepare_attn_dec(void);
int ygg_prepare_attn_tree(void);

int ygg_version(void) { return 100; }

const char* ygg_last_error(void) { return ygg::g_err; }

int ygg_trace_arm(unsigned long long* buf, int slots) {
  ygg::g_trace = slots > 0 ? buf : nullptr;
  ygg::g_trace_cap = slots < 0 ? 0 : (slots > 4096 ? 4096 : slots);
  ygg::g_trace_used = 0;
  return YGG_OK;
}

int ygg_trace_used(int* kernel_ids, int cap) {
  const int n = ygg::g_trace_used;
  for (int i = 0; i < n && i < cap; ++i) kernel_ids[i] = ygg::g_trace_ids[i];
  return n;
}

int ygg_device_check(int* num_sms, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return ygg::ygg_fail(YGG_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return ygg::ygg_fail(YGG_ERR_CUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
  if (num_sms) *num_sms = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (prop.major != 10 || prop.minor != 0)
    return ygg::ygg_fail(YGG_ERR_UNSUPPORTED, "libygg is built for sm_100a; found sm_%d%d", prop.major, prop.minor);
  // One-time kernel attributes (dynamic shared memory opt-in) — set here, outside any graph capture.
  if (int rc = ygg_prepare_tree()) return rc;
  if (int rc = ygg_prepare_gemm()) return rc;
  if (int rc = ygg_prepare_layers()) return rc;
  if (int rc = ygg_prepare_attn_tc()) return rc;
  if (int rc = ygg_prepare_gemv()) return rc;
  if (int rc = ygg_prepare_attn_dec()) return rc;
  if (int rc = ygg_prepare_attn_tree()) return rc;
  return YGG_OK;
}

}  // extern "C"
