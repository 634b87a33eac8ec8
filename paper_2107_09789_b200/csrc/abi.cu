// Error plumbing and small utilities of the C ABI (include/tobf.h).
#include <cstdarg>
#include <cstdio>
#include "tobf_internal.h"

static thread_local char g_last_error[512] = "";

int tobf_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

int tobf_cuda_check(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return tobf_fail(TOBF_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
  return TOBF_OK;
}

extern "C" const char* tobf_last_error(void) { return g_last_error; }

extern "C" int tobf_version(void) { return 1; }

extern "C" int tobf_device_sync(void) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return tobf_fail(TOBF_E_CUDA, "cudaDeviceSynchronize: %s", cudaGetErrorString(e));
  return TOBF_OK;
}
