// host_common.h -- host-side error plumbing shared by the C-ABI entry points.
#pragma once
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/taper.h"

namespace taper {
int fail(int code, const char *msg);
int fail_cuda(cudaError_t e, const char *what);
void set_launches(int n);
void add_launches(int n);
}  // namespace taper
