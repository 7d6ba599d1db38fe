// si_internal.h -- declarations shared by the native translation units.
#pragma once
#include <stdint.h>
#include <string>

#include "../../include/sparseinfer_b200.h"
#include "image.h"

void si_set_error(const std::string &msg);

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
