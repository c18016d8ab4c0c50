// abi.cu — error plumbing of the C ABI (include/nmk_b200.h).
//
// Every entry point returns 0 or a negative NMK_ERR_* code and leaves a
// thread-local message readable through nmk_last_error(); the Python mirror
// maps the codes onto the reference's exception types (ValueError,
// PipelineError(phase, ...), CodecError — pipeline.py:28-33, codec.py:24-25).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "nmk_common.cuh"

namespace nmk {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(NMK_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return NMK_OK;
}

void ensure_dyn_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{func, dev}];
  if (bytes > cur) {
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cur = bytes;
  }
}

int sm_count() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

unsigned pdl_mask() {
  static const unsigned mask = [] {
    const char* e = getenv("NMK_PDL");
    if (!e || !e[0]) return 0u;
    if (e[0] == '0' && (e[1] == 'x' || e[1] == 'X')) return (unsigned)strtoul(e, nullptr, 16);
    return e[0] == '1' ? 0xffffffffu : 0u;
  }();
  return mask;
}

}  // namespace nmk

extern "C" const char* nmk_last_error(void) { return nmk::g_err; }
extern "C" int nmk_version(void) { return 1; }
