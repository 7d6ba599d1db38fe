// si_internal.h -- declarations shared by the native translation units.
#pragma once
#include <stdint.h>
#include <string>

#include "../../include/sparseinfer_b200.h"
#include "image.h"

void si_set_error(const std::string &msg);

#ifdef __CUDACC__
#include <cuda_runtime.h>
#include <utility>
// Launch with programmatic stream serialization (PDL): the kernel's prologue
// (barrier init, TMEM allocation, descriptor prefetch) overlaps the tail of
// the previous kernel on the stream; every kernel launched this way calls
// tc::pdl_wait() before its first access to data another kernel produced.
// kernel entry of a PDL-launched kernel with no prologue worth overlapping
#define SI_PDL_ENTRY()                                                      \
    do {                                                                    \
        asm volatile("griddepcontrol.wait;" ::: "memory");                 \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");    \
    } while (0)

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#endif

struct SpmmArgs {
    const SiImage *h;       // host copy of the header
    const void *img;        // device image
    const uint8_t *x;       // device activation
    int32_t layout;         // si_act_layout
    int64_t ldx;            // leading dimension (elements)
    int64_t n;              // tokens
    const float *sides;     // device f32 [n_sides, N, M] or null
    void *out;              // device output [N, ldo]
    int64_t ldo;
    void *ws;               // workspace
    uint64_t ws_bytes;
    void *stream;           // cudaStream_t
};

// K1: CUDA-core gather (spmm_gather.cu).  Returns a cudaError_t value.
int k1_launch(const SpmmArgs &a);
// AUTO: the staged gather kernel (K1s) is the faster one for this call (one
// wave of CTAs, few blocks per group; measured crossover)
bool k1s_preferred(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx);
uint64_t k1_workspace(const SiImage *h, int64_t n, int32_t layout);
int k1_launch_count(const SiImage *h, int32_t layout);

// naive per-element reference kernel (spmm_gather.cu)
int kref_launch(const SpmmArgs &a);

// K2: tcgen05 tensor-core tiles (spmm_tc.cu)
int k2_launch(const SpmmArgs &a);
bool k2_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx, int64_t ldo);
uint64_t k2_workspace(const SiImage *h, int64_t n, int32_t layout);
int k2_launch_count(const SiImage *h, int32_t layout);

// K3: X-stationary 2:4-sparse tensor-core kernel (spmm_xs.cu): token-major X, K <= 1024
int k3_launch(const SpmmArgs &a);
bool k3_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx);

// K4: W-stationary 2:4-sparse tensor-core kernel (spmm_ws.cu): token-major X, K <= 1024
int k4_launch(const SpmmArgs &a);
bool k4_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx);
