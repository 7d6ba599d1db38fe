// spmm_tc.cu -- K2, the tcgen05 tensor-core path (work in progress).
#include <cuda_runtime.h>

#include "si_internal.h"

bool k2_supported(const SiImage *, int64_t, int32_t, int64_t, int64_t) { return false; }
uint64_t k2_workspace(const SiImage *, int64_t, int32_t) { return 0; }
int k2_launch_count(const SiImage *, int32_t) { return 1; }
int k2_launch(const SpmmArgs &) { return (int)cudaErrorNotSupported; }
