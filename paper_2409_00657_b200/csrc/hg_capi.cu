// Error plumbing of the C ABI (include/hopgnn.h).  No C++ exception or CUDA
// error crosses the boundary: everything becomes an hg_status plus a
// thread-local message the Python wrapper turns into the reference's
// exception types (errors.py:4-12).
#include <cstdarg>
#include <cstdio>

#include "hg_common.cuh"

static thread_local char g_err[512] = "";

int hg_fail_cuda(cudaError_t e, const char* what, const char* file, int line) {
  snprintf(g_err, sizeof(g_err), "CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e),
           cudaGetErrorString(e), file, line, what);
  return HG_ECUDA;
}

int hg_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

extern "C" const char* hg_last_error(void) { return g_err; }

extern "C" int hg_version(void) { return 1; }

extern "C" int hg_device_sync(void* stream) {
  HG_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  HG_CUDA_TRY(cudaGetLastError());
  return HG_OK;
}
