// abi.cu -- si_spmm dispatch (include/sparseinfer_b200.h).
//
// Replaces spmm_exec (spmm.py:283-333): the reference validates the plan
// against the activation and picks a task kernel by the program's output
// dtype, then fans tasks out on its thread pool; here the plan image picks
// the epilogue form and the shape picks K1 (gather, CUDA cores) or K2
// (tcgen05 tensor-core tiles).  All launches are on the caller's stream.
#include <cuda_runtime.h>
#include <string>

#include "../../include/sparseinfer_b200.h"
#include "si_internal.h"

namespace {

const SiImage *check_image(const void *host_image)
{
    const SiImage *h = (const SiImage *)host_image;
    if (!h || h->magic != SI_IMG_MAGIC || h->version != SI_IMG_VERSION) {
        si_set_error("not a plan image (magic/version mismatch)");
        return nullptr;
    }
    return h;
}

int32_t pick_kernel(const SiImage *h, int64_t n, int32_t layout, int32_t kernel, const void *x, int64_t ldx,
                    int64_t ldo)
{
    if (kernel != SI_KERNEL_AUTO) return kernel;
    // tensor cores once the token tile is worth a 128-row MMA tile; the
    // crossover is measured
    if (n >= 1024 && k2_supported(h, n, layout, x, ldx, ldo)) return SI_KERNEL_TC;
    return SI_KERNEL_GATHER;
}

}  // namespace

extern "C" int32_t si_spmm_workspace_size(const void *host_image, int64_t n, int32_t x_layout, int32_t kernel,
                                          uint64_t *bytes)
{
    const SiImage *h = check_image(host_image);
    if (!h) return SI_EINVAL;
    int32_t k = pick_kernel(h, n, x_layout, kernel, nullptr, x_layout == SI_ACT_KN ? n : h->K, h->M);
    *bytes = k == SI_KERNEL_GATHER ? k1_workspace(h, n, x_layout)
           : k == SI_KERNEL_TC     ? k2_workspace(h, n, x_layout)
                                   : 0;
    return SI_OK;
}

extern "C" int32_t si_spmm_launch_count(const void *host_image, int64_t n, int32_t x_layout, int32_t kernel)
{
    const SiImage *h = check_image(host_image);
    if (!h) return -1;
    int32_t k = pick_kernel(h, n, x_layout, kernel, nullptr, x_layout == SI_ACT_KN ? n : h->K, h->M);
    return k == SI_KERNEL_GATHER ? k1_launch_count(h, x_layout)
         : k == SI_KERNEL_TC     ? k2_launch_count(h, x_layout)
                                 : 1;
}

extern "C" int32_t si_spmm(const void *host_image, const void *dev_image, const void *x, int32_t x_layout,
                           int64_t ldx, int64_t n, const float *sides, void *out, int64_t ldo, void *workspace,
                           uint64_t workspace_bytes, int32_t kernel, void *stream)
{
    const SiImage *h = check_image(host_image);
    if (!h) return SI_EINVAL;
    if (!dev_image || !x || !out || n <= 0) {
        si_set_error("null pointer or N <= 0");
        return SI_EINVAL;
    }
    if (((uintptr_t)dev_image) % 16) {
        si_set_error("device image must be 16-byte aligned");
        return SI_EINVAL;
    }
    if (x_layout != SI_ACT_KN && x_layout != SI_ACT_NK) {
        si_set_error("bad activation layout");
        return SI_EINVAL;
    }
    if ((x_layout == SI_ACT_KN && ldx < n) || (x_layout == SI_ACT_NK && ldx < h->K) || ldo < h->M) {
        si_set_error("leading dimension smaller than the row");
        return SI_EINVAL;
    }
    if (h->n_sides > 0 && !sides) {
        si_set_error("program needs side inputs");
        return SI_EINVAL;
    }
    int32_t k = pick_kernel(h, n, x_layout, kernel, x, ldx, ldo);
    uint64_t need = k == SI_KERNEL_GATHER ? k1_workspace(h, n, x_layout)
                  : k == SI_KERNEL_TC     ? k2_workspace(h, n, x_layout)
                                          : 0;
    if (workspace_bytes < need || (need && !workspace)) {
        si_set_error("workspace too small: need " + std::to_string(need) + " bytes");
        return SI_ENOSPACE;
    }
    if (k == SI_KERNEL_TC && !k2_supported(h, n, x_layout, x, ldx, ldo)) {
        si_set_error("tensor-core kernel does not support this shape/layout");
        return SI_EUNSUPPORTED;
    }
    SpmmArgs a{h, dev_image, (const uint8_t *)x, x_layout, ldx, n, sides, out, ldo, workspace, workspace_bytes,
               stream};
    int err = k == SI_KERNEL_GATHER ? k1_launch(a) : k == SI_KERNEL_TC ? k2_launch(a) : kref_launch(a);
    if (err != cudaSuccess) {
        si_set_error(std::string("CUDA launch failed: ") + cudaGetErrorString((cudaError_t)err));
        return SI_ECUDA;
    }
    return SI_OK;
}
