/*
 * sparseinfer_b200.h -- C ABI of the B200 4x1-block INT8 SpMM.
 *
 * The reference (sparseinfer 0.1.0, /root/reference/pkg) is pure Python +
 * numba and has no FFI; its operator API is the set of Python functions in
 * sparseinfer.kernels (kernels/__init__.py:1-40).  Each entry point below is
 * what that API binds to when it crosses into native code -- the mapping is
 * given per function as "replaces <file>:<line>".  Plain C types only: host
 * arrays are the numpy buffers of Sparse4x1Weight / EpilogueProgram, device
 * pointers are raw CUDA addresses (torch.Tensor.data_ptr()), the stream is a
 * cudaStream_t passed as void*.  The library never allocates device memory;
 * the caller owns every buffer (plan image, activations, outputs, workspace).
 *
 * Errors: every function returns an si_status (0 = SI_OK).  The text of the
 * last error on the calling thread is available from si_last_error().  The
 * Python layer validates shapes and raises the reference's exception types
 * (ValueError / SparseFormatError) before calling in; a nonzero status
 * surfaces as RuntimeError.
 */
#ifndef SPARSEINFER_B200_H
#define SPARSEINFER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SI_ABI_VERSION 2  /* 2: side inputs on the host-buffer entry points */

typedef enum {
    SI_OK = 0,
    SI_EINVAL = 1,       /* bad argument / shape mismatch (reference: ValueError) */
    SI_EFORMAT = 2,      /* malformed 4x1 encoding (reference: SparseFormatError) */
    SI_ECUDA = 3,        /* CUDA launch / runtime error */
    SI_EUNSUPPORTED = 4, /* legal input outside what this build implements */
    SI_ENOSPACE = 5      /* caller buffer too small */
} si_status;

/* element types, order of tensor.py:27-31 (DType F32, S8, U8, S32) */
typedef enum { SI_F32 = 0, SI_S8 = 1, SI_U8 = 2, SI_S32 = 3 } si_dtype;

/* epilogue opcodes, epilogue.py:22-29, plus SI_OP_GELU_ERF (extension) */
typedef enum {
    SI_OP_REQUANT = 0, SI_OP_LUT = 1, SI_OP_DEQ = 2, SI_OP_GELU = 3,
    SI_OP_ADD_SIDE = 4, SI_OP_ADD_CHAN = 5, SI_OP_QUANT = 6, SI_OP_DEQ_ACC = 7,
    SI_OP_GELU_ERF = 8
} si_op;

/* activation orientation: logical [K, N] (relayout_activation, spmm.py:82)
 * or token-major [N, K] (relayout_tokens, spmm.py:96).  Neither is relaid
 * out: the kernels read both directly. */
typedef enum { SI_ACT_KN = 0, SI_ACT_NK = 1 } si_act_layout;

/* kernel selection; SI_KERNEL_AUTO picks by shape */
typedef enum {
    SI_KERNEL_AUTO = 0,
    SI_KERNEL_GATHER = 1,  /* K1: CUDA-core dp4a gather over 4x1 micro-tiles */
    SI_KERNEL_TC = 2,      /* K2: tcgen05 kind::i8 tensor-core tiles, dense-expanded W */
    SI_KERNEL_REF = 3,     /* naive per-element kernel (spmm_ref, spmm.py:401) */
    SI_KERNEL_SP = 4,      /* K3: tcgen05.mma.sp 2:4 W images, X-stationary (token-major X, K <= 1024) */
    SI_KERNEL_WS = 5       /* K4: tcgen05.mma.sp 2:4 W images resident per CTA pair, X streamed (token-major X, K <= 1024) */
} si_kernel;

/* Host view of a Sparse4x1Weight (sparse.py:23-41). */
typedef struct {
    int32_t rows;          /* padded to 4 */
    int32_t cols;          /* K */
    int32_t logical_rows;  /* M */
    const int32_t *group_ptr; /* [rows/4 + 1] padded block offsets */
    const int32_t *idx;       /* [group_ptr[rows/4]] column per block */
    const int8_t *vals;       /* [4 * group_ptr[rows/4]] micro-tiles */
} si_weight;

/* Host view of an EpilogueProgram (epilogue.py:34-50). */
typedef struct {
    int32_t m;                /* channels == logical_rows */
    const float *scale_in;    /* [m] */
    int32_t a_zp;
    int32_t n_ops;
    const int32_t *ops;       /* [n_ops] */
    const float *fparams;     /* [n_ops] */
    const int32_t *iparams;   /* [n_ops * 3] */
    int32_t n_luts;
    const uint8_t *luts;      /* [n_luts * 256] */
    int32_t n_chans;
    const float *chans;       /* [n_chans * m] */
    int32_t out_dtype;        /* si_dtype */
    int32_t n_sides;
} si_program;

/* ABI version of the loaded library (SI_ABI_VERSION). */
int32_t si_abi_version(void);

/* Thread-local text of the last failure ("" if none). */
const char *si_last_error(void);

/* Size in bytes of the plan image for (weight, program, bias).
 * replaces plan_spmm, spmm.py:160-189 (tiling, compensation, program). */
int32_t si_plan_image_size(const si_weight *w, const si_program *p, uint64_t *bytes);

/* Build the plan image into host memory (caller copies it to the device
 * unchanged; it is position independent).  Validates the encoding
 * (SI_EFORMAT on idx outside [0, K), as decode_sparse, sparse.py:119-120),
 * packs the GPU tile formats, computes comp[m] (Sparse4x1Weight.row_sums,
 * sparse.py:51-62) and adj[m] = bias[m] - a_zp*comp[m] (spmm.py:231), and
 * compiles the epilogue program (LUT / breakpoint-table forms).
 * bias may be NULL (zeros, spmm.py:179-180). */
int32_t si_plan_image_build(const si_weight *w, const si_program *p, const int32_t *bias,
                            void *host_image, uint64_t bytes);

/* Query facts of a built image: the kernel AUTO would choose for n tokens,
 * whether the compiled epilogue is bit-exact (0 only for GELU feeding an
 * f32 output or a residual add, where the device tanh/erf is used), etc. */
typedef struct {
    int32_t m, k, groups, out_dtype, epi_mode, exact;
    int64_t nnz_blocks, padded_blocks;
    uint64_t image_bytes;
} si_plan_info;
int32_t si_plan_info_get(const void *host_image, si_plan_info *info);

/* Structural validation of `bytes` bytes claiming to be a plan image (e.g.
 * read from a plan file): header size, magic/version, header consistency and
 * every section's extent inside the image.  SI_EFORMAT names the defect.
 * Images from si_plan_image_build always pass. */
int32_t si_plan_image_validate(const void *image, uint64_t bytes);

/* Device workspace the run needs (0 when none).  For SI_KERNEL_AUTO this is
 * enough for either kernel AUTO may pick (the pick also depends on the
 * alignment of x and ldx, which this query does not see). */
int32_t si_spmm_workspace_size(const void *host_image, int64_t n, int32_t x_layout,
                               int32_t kernel, uint64_t *bytes);

/* Run the SpMM: out[n, m] = epilogue(sum_k W[m,k] x[k,n] + adj[m]) for
 * n < N, m < M, stream-ordered on `stream`.
 * replaces spmm_exec, spmm.py:283-333 (and its kernels _spmm_task_*, :215-280).
 *   host_image  the host copy of the image (kernel selection reads it)
 *   dev_image   the same bytes in device memory (16-byte aligned)
 *   x           device u8 activation, layout x_layout, leading dim ldx (elements)
 *   sides       device f32 [n_sides, N, M] or NULL when the program has none
 *   out         device output [N, ldo] of the program's dtype (ldo >= M)
 *   workspace   device scratch of si_spmm_workspace_size bytes (may be NULL if 0) */
int32_t si_spmm(const void *host_image, const void *dev_image, const void *x, int32_t x_layout,
                int64_t ldx, int64_t n, const float *sides, void *out, int64_t ldo,
                void *workspace, uint64_t workspace_bytes, int32_t kernel, void *stream);

/* Host-buffer run (the reference's spmm_exec takes host arrays,
 * spmm.py:283-333): x_host [K, ldx] (SI_ACT_KN) or [N, ldx] (SI_ACT_NK),
 * sides_host f32 [n_sides, N, M] (the pack_sides form, epilogue.py:256-263;
 * NULL when the program has none) and out_host [N, ldo], all in host memory
 * (pinned for full overlap).  Token chunks of chunk_n are pipelined: H2D of
 * chunk i+1 and D2H of chunk i-1 overlap the kernel on chunk i (launched on
 * `stream`), in a 4-deep device buffer ring inside `workspace` (device,
 * si_spmm_host_workspace_size bytes).  Each call takes its own pair of copy
 * streams, so concurrent calls with separate workspaces are independent.
 * Returns when out_host is complete (on error paths too, every copy the call
 * queued has finished).
 * replaces spmm_exec, spmm.py:283-333, for callers holding host arrays. */
int32_t si_spmm_host_workspace_size(const void *host_image, int64_t chunk_n, int32_t x_layout, int32_t kernel,
                                    uint64_t *bytes);
int32_t si_spmm_host(const void *host_image, const void *dev_image, const void *x_host, int32_t x_layout,
                     int64_t ldx, int64_t n, const float *sides_host, void *out_host, int64_t ldo, void *workspace,
                     uint64_t workspace_bytes, int64_t chunk_n, int32_t kernel, void *stream);

/* Several independent host-buffer SpMMs (e.g. Q/K/V projections) as one
 * pipelined chunk sequence, so the copy-in of one job overlaps the copy-out
 * of the previous one.  Same rules as si_spmm_host per job. */
typedef struct {
    const void *host_image, *dev_image;
    const void *x_host;
    int32_t x_layout;
    int64_t ldx, n;
    void *out_host;
    int64_t ldo;
    const float *sides_host;  /* f32 [n_sides, n, M] or NULL (ABI 2) */
} si_host_job;
int32_t si_spmm_host_batch_workspace_size(const si_host_job *jobs, int32_t count, int64_t chunk_n,
                                          uint64_t *bytes);
int32_t si_spmm_host_batch(const si_host_job *jobs, int32_t count, void *workspace, uint64_t workspace_bytes,
                           int64_t chunk_n, int32_t kernel, void *stream);

/* Number of kernels si_spmm launches for these arguments (for launch
 * accounting in bench.py). */
int32_t si_spmm_launch_count(const void *host_image, int64_t n, int32_t x_layout, int32_t kernel);

/* ---- dense f32 auxiliary operators (encoder composition, BASELINE config 4).
 * Same fixed summation orders and expression trees as the reference's numba
 * kernels, so results match element for element.  All pointers are device
 * pointers; launches go to `stream`. */

/* softmax over the last axis of a row-major [rows, n] tensor; replaces
 * softmax_f32 (eltwise.py:34-59).  out may alias x. */
int32_t si_softmax_rows_f32(const float *x, float *out, int64_t rows, int64_t n, void *stream);

/* layer norm over the last axis of [rows, n] with affine gamma/beta [n];
 * replaces layer_norm_f32 (eltwise.py:62-99). */
int32_t si_layer_norm_f32(const float *x, const float *gamma, const float *beta, double eps, float *out,
                          int64_t rows, int64_t n, void *stream);

/* batched f32 matmul over a two-level batch (b0 < nb0, b1 < nb1): operand
 * a at a + b0*sa0 + b1*sa1 is [m, k] with row stride lda; b likewise ([k, n],
 * or [n, k] when transpose_b); out [m, n] with row stride ldo.  out = (a @ b)
 * * alpha; replaces batch_matmul_f32 (eltwise.py:102-160) and covers the
 * per-(sequence, head) attention products on token-major [N, H] tensors
 * without copies. */
int32_t si_bmm_f32(const float *a, const float *b, float *out, int64_t nb0, int64_t nb1, int64_t m, int64_t k,
                   int64_t n, int64_t sa0, int64_t sa1, int64_t lda, int64_t sb0, int64_t sb1, int64_t ldb,
                   int64_t so0, int64_t so1, int64_t ldo, int32_t transpose_b, float alpha, void *stream);

/* per-tensor affine quantization of n floats: clamp(rint(f64 x / f64 scale) +
 * zp, lo, hi) stored as u8 (lo >= 0) or s8 (lo < 0); replaces quantize
 * (tensor.py:140-151) for per-tensor params. */
int32_t si_quantize_f32(const float *x, int64_t n, float scale, int32_t zp, int32_t lo, int32_t hi, void *out,
                        void *stream);

/* the encoder's attention block for one (sequence, head) per CTA, all in
 * shared memory: scores = q k^T * alpha (bmm_nt), softmax_rows, context =
 * p v (bmm_nn) -- eltwise.py:34-160 in those orders, so bit-equal to the three
 * ops run separately.  qkv is token-major [batch*seq, ld_qkv] with q, k, v at
 * columns 0, H, 2H (H = heads*head_dim); ctx is [batch*seq, ld_ctx].
 * SI_EUNSUPPORTED for seq > 128 or head_dim > 64 (use the separate ops). */
int32_t si_attention_f32(const float *qkv, float *ctx, int64_t batch, int64_t seq, int64_t heads,
                         int64_t head_dim, int64_t ld_qkv, int64_t ld_ctx, float alpha, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEINFER_B200_H */
