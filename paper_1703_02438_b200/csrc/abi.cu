// abi.cu — error plumbing of the C ABI (include/nmk_b200.h).
//
// Every entry point returns 0 or a negative NMK_ERR_* code and leaves a
// thread-local message readable through nmk_last_error(); the Python mirror
// maps the codes onto the reference's exception types (ValueError,
// PipelineError(phase, ...), CodecError — pipeline.py:28-33, codec.py:24-25).
#include <cstdarg>
#include <cstdio>

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

}  // namespace nmk

extern "C" const char* nmk_last_error(void) { return nmk::g_err; }
extern "C" int nmk_version(void) { return 1; }
