// eltwise.cu -- the dense f32 auxiliary operators of the encoder composition
// (BASELINE config 4): softmax, layer norm, batched matmul and per-tensor
// quantization, with the reference's fixed summation orders and expression
// trees (eltwise.py:34-160, tensor.py:140-151) so the results match its
// numba kernels element for element.
//
// The orders are sequential per row (the reference's only implementation),
// so each row is owned by one thread; warps stage their 32 rows through
// shared memory in column chunks so the global traffic stays coalesced while
// every lane walks its own row in order.  Compiled with -ffp-contract=off and
// explicit __fmul_rn / __fadd_rn: no FMA contraction anywhere.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sparseinfer_b200.h"
#include "si_internal.h"

namespace {

constexpr int ROWS = 32;   // rows per warp (one per lane)

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
constexpr int CH = 64;     // columns per staged chunk

// Stage rows [r0, r0+32) x columns [c0, c0+cw) of x (row stride ld) into
// tile[32][CH+1] (padded: lane r reads column c conflict-free).
__device__ __forceinline__ void stage(const float *x, int64_t ld, int64_t rows, int64_t r0, int64_t c0, int cw,
                                      float (*tile)[CH + 1])
{
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < ROWS; ++r) {
        const int64_t row = r0 + r;
        for (int c = lane; c < cw; c += 32) tile[r][c] = row < rows ? x[row * ld + c0 + c] : 0.0f;
    }
    __syncwarp();
}

// softmax_rows (eltwise.py:34-50): m = max, e = f32(exp(f64 x - f64 m)),
// s = sequential f64 sum, out = e * f32(1/s)
__global__ void k_softmax_rows(const float *x, float *out, int64_t rows, int64_t n, int64_t ld)
{
    __shared__ float tile[4][ROWS][CH + 1];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = ((int64_t)blockIdx.x * 4 + w) * ROWS;
    if (r0 >= rows) return;
    const int64_t row = r0 + lane;
    float (*t)[CH + 1] = tile[w];
    float m = -INFINITY;
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int cw = (int)imin64(CH, n - c0);
        stage(x, ld, rows, r0, c0, cw, t);
        for (int c = 0; c < cw; ++c) {
            const float v = t[lane][c];
            if (c0 + c == 0 || v > m) m = v;
        }
        __syncwarp();
    }
    double s = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int cw = (int)imin64(CH, n - c0);
        stage(x, ld, rows, r0, c0, cw, t);
        for (int c = 0; c < cw; ++c) {
            const float e = (float)exp((double)t[lane][c] - (double)m);
            t[lane][c] = e;
            s = __dadd_rn(s, (double)e);
        }
        __syncwarp();
        for (int r = 0; r < ROWS; ++r)   // unnormalised e back out, coalesced
            if (r0 + r < rows)
                for (int c = lane; c < cw; c += 32) out[(r0 + r) * ld + c0 + c] = t[r][c];
        __syncwarp();
    }
    const float inv = (float)(1.0 / s);
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int cw = (int)imin64(CH, n - c0);
        stage(out, ld, rows, r0, c0, cw, t);
        for (int c = 0; c < cw; ++c) t[lane][c] = __fmul_rn(t[lane][c], inv);
        __syncwarp();
        for (int r = 0; r < ROWS; ++r)
            if (r0 + r < rows)
                for (int c = lane; c < cw; c += 32) out[(r0 + r) * ld + c0 + c] = t[r][c];
        __syncwarp();
    }
    (void)row;
}

// layer_norm_rows (eltwise.py:62-76): f64 sequential mean and variance,
// inv = f32(1/sqrt(v/n + eps)), y = (x - f32(mean)) * inv, out = y*gamma + beta
__global__ void k_layer_norm_rows(const float *x, const float *gamma, const float *beta, double eps, float *out,
                                  int64_t rows, int64_t n)
{
    __shared__ float tile[4][ROWS][CH + 1];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = ((int64_t)blockIdx.x * 4 + w) * ROWS;
    if (r0 >= rows) return;
    float (*t)[CH + 1] = tile[w];
    double s = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int cw = (int)imin64(CH, n - c0);
        stage(x, n, rows, r0, c0, cw, t);
        for (int c = 0; c < cw; ++c) s = __dadd_rn(s, (double)t[lane][c]);
        __syncwarp();
    }
    const double mean = __ddiv_rn(s, (double)n);
    double v = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int cw = (int)imin64(CH, n - c0);
        stage(x, n, rows, r0, c0, cw, t);
        for (int c = 0; c < cw; ++c) {
            const double d = __dsub_rn((double)t[lane][c], mean);
            v = __dadd_rn(v, __dmul_rn(d, d));
        }
        __syncwarp();
    }
    const float inv = (float)__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(v, (double)n), eps)));
    const float mean32 = (float)mean;
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int cw = (int)imin64(CH, n - c0);
        stage(x, n, rows, r0, c0, cw, t);
        for (int c = 0; c < cw; ++c) {
            const float y = __fmul_rn(__fsub_rn(t[lane][c], mean32), inv);
            t[lane][c] = __fadd_rn(__fmul_rn(y, gamma[c0 + c]), beta[c0 + c]);
        }
        __syncwarp();
        for (int r = 0; r < ROWS; ++r)
            if (r0 + r < rows)
                for (int c = lane; c < cw; c += 32) out[(r0 + r) * n + c0 + c] = t[r][c];
        __syncwarp();
    }
}

// batch_matmul_f32 (eltwise.py:102-127) on strided operands: one thread per
// output element, the k-sum in order p = 0..k-1 in f32 from 0 (each product
// and each sum one rounding), then * alpha.  32x32 output tiles; A rows and
// the B panel staged in shared memory k-chunk by k-chunk.
constexpr int BT = 32, BK = 32;
__global__ void k_bmm(const float *a, const float *b, float *out, int64_t nb1, int64_t m, int64_t k, int64_t n,
                      int64_t sa0, int64_t sa1, int64_t lda, int64_t sb0, int64_t sb1, int64_t ldb, int64_t so0,
                      int64_t so1, int64_t ldo, int transpose_b, float alpha)
{
    __shared__ float As[BT][BK + 1];
    __shared__ float Bs[BK][BT + 1];
    const int64_t bz = blockIdx.z, b0 = bz / nb1, b1 = bz % nb1;
    const float *A = a + b0 * sa0 + b1 * sa1;
    const float *B = b + b0 * sb0 + b1 * sb1;
    float *O = out + b0 * so0 + b1 * so1;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8 threads, 4 rows each
    const int64_t i0 = (int64_t)blockIdx.y * BT, j0 = (int64_t)blockIdx.x * BT;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int64_t p0 = 0; p0 < k; p0 += BK) {
        for (int r = ty; r < BT; r += 8) {
            const int64_t i = i0 + r, p = p0 + tx;
            As[r][tx] = (i < m && p < k) ? A[i * lda + p] : 0.0f;
        }
        for (int r = ty; r < BK; r += 8) {
            const int64_t p = p0 + r, j = j0 + tx;
            float v = 0.0f;
            if (p < k && j < n) v = transpose_b ? B[j * ldb + p] : B[p * ldb + j];
            Bs[r][tx] = v;
        }
        __syncthreads();
        const int pk = (int)imin64(BK, k - p0);
        for (int p = 0; p < pk; ++p) {
            const float bv = Bs[p][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(As[ty + 8 * q][p], bv));
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t i = i0 + ty + 8 * q, j = j0 + tx;
        if (i < m && j < n) O[i * ldo + j] = __fmul_rn(acc[q], alpha);
    }
}

// quantize (tensor.py:140-151): clamp(rint(f64 x / f64 scale) + zp, lo, hi)
__global__ void k_quantize(const float *x, int64_t n, double scale, int32_t zp, int32_t lo, int32_t hi, void *out,
                           int out_s8)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double q = rint(__ddiv_rn((double)x[i], scale)) + (double)zp;
        q = fmin(fmax(q, (double)lo), (double)hi);
        if (out_s8) static_cast<int8_t *>(out)[i] = (int8_t)q;
        else static_cast<uint8_t *>(out)[i] = (uint8_t)q;
    }
}

int grid_rows(int64_t rows) { return (int)((rows + 4 * ROWS - 1) / (4 * ROWS)); }

}  // namespace

extern "C" int32_t si_softmax_rows_f32(const float *x, float *out, int64_t rows, int64_t n, void *stream)
{
    if (!x || !out || rows < 0 || n <= 0) {
        si_set_error("softmax: bad arguments");
        return SI_EINVAL;
    }
    if (rows == 0) return SI_OK;
    k_softmax_rows<<<grid_rows(rows), 128, 0, (cudaStream_t)stream>>>(x, out, rows, n, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { si_set_error(cudaGetErrorString(e)); return SI_ECUDA; }
    return SI_OK;
}

extern "C" int32_t si_layer_norm_f32(const float *x, const float *gamma, const float *beta, double eps, float *out,
                                     int64_t rows, int64_t n, void *stream)
{
    if (!x || !gamma || !beta || !out || rows < 0 || n <= 0) {
        si_set_error("layer_norm: bad arguments");
        return SI_EINVAL;
    }
    if (rows == 0) return SI_OK;
    k_layer_norm_rows<<<grid_rows(rows), 128, 0, (cudaStream_t)stream>>>(x, gamma, beta, eps, out, rows, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { si_set_error(cudaGetErrorString(e)); return SI_ECUDA; }
    return SI_OK;
}

extern "C" int32_t si_bmm_f32(const float *a, const float *b, float *out, int64_t nb0, int64_t nb1, int64_t m,
                              int64_t k, int64_t n, int64_t sa0, int64_t sa1, int64_t lda, int64_t sb0, int64_t sb1,
                              int64_t ldb, int64_t so0, int64_t so1, int64_t ldo, int32_t transpose_b, float alpha,
                              void *stream)
{
    if (!a || !b || !out || nb0 < 0 || nb1 <= 0 || m < 0 || k <= 0 || n < 0 || nb0 * nb1 > 65535 * 64) {
        si_set_error("bmm: bad arguments");
        return SI_EINVAL;
    }
    if (nb0 == 0 || m == 0 || n == 0) return SI_OK;
    dim3 grid((unsigned)((n + BT - 1) / BT), (unsigned)((m + BT - 1) / BT), (unsigned)(nb0 * nb1));
    k_bmm<<<grid, 256, 0, (cudaStream_t)stream>>>(a, b, out, nb1, m, k, n, sa0, sa1, lda, sb0, sb1, ldb, so0, so1, ldo,
                                                  transpose_b, alpha);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { si_set_error(cudaGetErrorString(e)); return SI_ECUDA; }
    return SI_OK;
}

extern "C" int32_t si_quantize_f32(const float *x, int64_t n, float scale, int32_t zp, int32_t lo, int32_t hi,
                                   void *out, void *stream)
{
    if (!x || !out || n < 0 || !(scale > 0.0f) || lo > hi) {
        si_set_error("quantize: bad arguments");
        return SI_EINVAL;
    }
    if (n == 0) return SI_OK;
    const int threads = 256;
    const int64_t blocks = imin64((n + threads - 1) / threads, 148 * 16);
    k_quantize<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(x, n, (double)scale, zp, lo, hi, out, lo < 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { si_set_error(cudaGetErrorString(e)); return SI_ECUDA; }
    return SI_OK;
}
