// Host-side helpers shared by the libtobf translation units.
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include "../../include/tobf.h"

// Records a printf-style message as the thread's last error and returns code.
int tobf_fail(int code, const char* fmt, ...);
// Returns TOBF_OK, or TOBF_E_CUDA with the pending launch error recorded.
int tobf_cuda_check(const char* where);
