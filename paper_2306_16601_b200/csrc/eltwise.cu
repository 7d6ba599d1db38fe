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
#include "tc_ptx.cuh"

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
    SI_PDL_ENTRY();
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
    SI_PDL_ENTRY();
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

// Whole-row variants: the warp's 32 rows are loaded into shared memory once
// (row stride n+1: lane r walks row r conflict-free), so the three sequential
// passes read smem and the global traffic is one coalesced read and write.
// One warp per block; dynamic smem 32*(n+1)*4 bytes.
__device__ __forceinline__ void load_rows(const float *x, int64_t ld, int64_t rows, int64_t r0, int n, float *t)
{
    const int lane = threadIdx.x & 31;
    if ((n & 3) == 0 && (ld & 3) == 0 && (((uintptr_t)x) & 15) == 0) {
        // 16-byte loads, 8 rows in flight per lane (the load phase is latency-bound)
        const int n4 = n >> 2;
        for (int r0i = 0; r0i < ROWS; r0i += 8) {
#pragma unroll
            for (int rr = 0; rr < 8; ++rr) {
                const int r = r0i + rr;
                const int64_t row = r0 + r;
                for (int c4 = lane; c4 < n4; c4 += 32) {
                    const float4 v = row < rows ? __ldg(reinterpret_cast<const float4 *>(x + row * ld) + c4)
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
                    float *d = t + r * (n + 1) + 4 * c4;
                    d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
                }
            }
        }
    } else {
        for (int r = 0; r < ROWS; ++r) {
            const int64_t row = r0 + r;
#pragma unroll 4
            for (int c = lane; c < n; c += 32) t[r * (n + 1) + c] = row < rows ? x[row * ld + c] : 0.0f;
        }
    }
    __syncwarp();
}
__device__ __forceinline__ void store_rows(float *out, int64_t ld, int64_t rows, int64_t r0, int n, const float *t)
{
    const int lane = threadIdx.x & 31;
    __syncwarp();
    if ((n & 3) == 0 && (ld & 3) == 0 && (((uintptr_t)out) & 15) == 0) {
        const int n4 = n >> 2;
        for (int r = 0; r < ROWS; ++r) {
            const int64_t row = r0 + r;
            if (row >= rows) break;
            for (int c4 = lane; c4 < n4; c4 += 32) {
                const float *sv = t + r * (n + 1) + 4 * c4;
                reinterpret_cast<float4 *>(out + row * ld)[c4] = make_float4(sv[0], sv[1], sv[2], sv[3]);
            }
        }
        return;
    }
    for (int r = 0; r < ROWS; ++r) {
        const int64_t row = r0 + r;
        if (row >= rows) break;
#pragma unroll 4
        for (int c = lane; c < n; c += 32) out[row * ld + c] = t[r * (n + 1) + c];
    }
}

__global__ void k_softmax_rows_smem(const float *x, float *out, int64_t rows, int n)
{
    SI_PDL_ENTRY();
    extern __shared__ float t_sm[];
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * ROWS;
    load_rows(x, n, rows, r0, n, t_sm);
    float *t = t_sm + lane * (n + 1);
    float m = t[0];
    for (int c = 1; c < n; ++c)
        if (t[c] > m) m = t[c];
    double s = 0.0;
    for (int c = 0; c < n; ++c) {
        const float e = (float)exp((double)t[c] - (double)m);
        t[c] = e;
        s = __dadd_rn(s, (double)e);
    }
    const float inv = (float)(1.0 / s);
    for (int c = 0; c < n; ++c) t[c] = __fmul_rn(t[c], inv);
    store_rows(out, n, rows, r0, n, t_sm);
}

__global__ void k_layer_norm_rows_smem(const float *x, const float *gamma, const float *beta, double eps, float *out,
                                       int64_t rows, int n)
{
    SI_PDL_ENTRY();
    extern __shared__ float t_sm[];
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * ROWS;
    load_rows(x, n, rows, r0, n, t_sm);
    float *t = t_sm + lane * (n + 1);
    double s = 0.0;
    for (int c = 0; c < n; ++c) s = __dadd_rn(s, (double)t[c]);
    const double mean = __ddiv_rn(s, (double)n);
    double v = 0.0;
    for (int c = 0; c < n; ++c) {
        const double d = __dsub_rn((double)t[c], mean);
        v = __dadd_rn(v, __dmul_rn(d, d));
    }
    const float inv = (float)__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(v, (double)n), eps)));
    const float mean32 = (float)mean;
    for (int c = 0; c < n; ++c) {
        const float y = __fmul_rn(__fsub_rn(t[c], mean32), inv);
        t[c] = __fadd_rn(__fmul_rn(y, __ldg(gamma + c)), __ldg(beta + c));
    }
    store_rows(out, n, rows, r0, n, t_sm);
}

// The same computation for n % 4 == 0 with the 32 rows moved by the bulk-copy
// engine: each lane issues the 1-D copy of its own row into a 16-byte-aligned
// smem row (stride n + 4, so the lanes' float4 reads of a quarter warp hit
// distinct banks), then streams its row back out the same way.  All of an
// SM's rows are in flight at once instead of one warp's loads at a time.
__global__ void k_layer_norm_rows_bulk(const float *x, const float *gamma, const float *beta, double eps, float *out,
                                       int64_t rows, int n)
{
    SI_PDL_ENTRY();
    extern __shared__ __align__(16) float b_sm[];
    __shared__ __align__(8) uint64_t bar;
    const int lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * ROWS;
    const int nr = (int)imin64(ROWS, rows - r0);
    const int ldr = n + 4;
    const uint32_t row_bytes = (uint32_t)n * 4;
    if (lane == 0) {
        tc::mbar_init(&bar, 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc::mbar_expect_tx(&bar, row_bytes * (uint32_t)nr);
    }
    __syncwarp();
    float *t = b_sm + lane * ldr;
    if (lane < nr) tc::bulk_load(t, x + (r0 + lane) * n, row_bytes, &bar);
    tc::mbar_wait(&bar, 0);
    if (lane < nr) {
        const float4 *t4 = reinterpret_cast<const float4 *>(t);
        double s = 0.0;
        for (int c = 0; c < n / 4; ++c) {
            const float4 v = t4[c];
            s = __dadd_rn(s, (double)v.x); s = __dadd_rn(s, (double)v.y);
            s = __dadd_rn(s, (double)v.z); s = __dadd_rn(s, (double)v.w);
        }
        const double mean = __ddiv_rn(s, (double)n);
        double v2 = 0.0;
        for (int c = 0; c < n / 4; ++c) {
            const float4 v = t4[c];
            double d;
            d = __dsub_rn((double)v.x, mean); v2 = __dadd_rn(v2, __dmul_rn(d, d));
            d = __dsub_rn((double)v.y, mean); v2 = __dadd_rn(v2, __dmul_rn(d, d));
            d = __dsub_rn((double)v.z, mean); v2 = __dadd_rn(v2, __dmul_rn(d, d));
            d = __dsub_rn((double)v.w, mean); v2 = __dadd_rn(v2, __dmul_rn(d, d));
        }
        const float inv = (float)__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__ddiv_rn(v2, (double)n), eps)));
        const float mean32 = (float)mean;
        float4 *w4 = reinterpret_cast<float4 *>(t);
        const float4 *g4 = reinterpret_cast<const float4 *>(gamma), *b4 = reinterpret_cast<const float4 *>(beta);
        for (int c = 0; c < n / 4; ++c) {
            float4 v = w4[c];
            const float4 g = __ldg(g4 + c), b = __ldg(b4 + c);
            v.x = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v.x, mean32), inv), g.x), b.x);
            v.y = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v.y, mean32), inv), g.y), b.y);
            v.z = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v.z, mean32), inv), g.z), b.z);
            v.w = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v.w, mean32), inv), g.w), b.w);
            w4[c] = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (r0 + lane) * n),
                     "r"(tc::smem_u32(t)), "r"(row_bytes)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

constexpr int SMEM_ROWS_MAX = 200 * 1024;
inline bool rows_fit(int64_t n) { return n <= 4096 && (int64_t)ROWS * (n + 1) * 4 <= SMEM_ROWS_MAX; }

// batch_matmul_f32 (eltwise.py:102-127) on strided operands.  Each output's
// k-sum runs in order p = 0..k-1 in f32 from 0 (each product and each sum
// one rounding), then * alpha -- exactly the reference's sequence.  64x64
// output tiles, 256 threads with 4x4 register blocks; A and B panels staged
// in shared memory 16 k at a time, coalesced along each operand's contiguous
// dimension.
constexpr int BT = 64, BK = 32;
__global__ void __launch_bounds__(256) k_bmm(const float *a, const float *b, float *out, int64_t nb1, int64_t m,
                                             int64_t k, int64_t n, int64_t sa0, int64_t sa1, int64_t lda, int64_t sb0,
                                             int64_t sb1, int64_t ldb, int64_t so0, int64_t so1, int64_t ldo,
                                             int transpose_b, float alpha)
{
    SI_PDL_ENTRY();
    __shared__ float As[BK][BT + 4];   // [p][i]
    __shared__ float Bs[BK][BT + 4];   // [p][j]
    const int64_t bz = blockIdx.z, b0 = bz / nb1, b1 = bz % nb1;
    const float *A = a + b0 * sa0 + b1 * sa1;
    const float *B = b + b0 * sb0 + b1 * sb1;
    float *O = out + b0 * so0 + b1 * so1;
    const int t = threadIdx.x;
    const int tx = t & 15, ty = t >> 4;             // 16 x 16 threads, rows ty*4.., cols tx*4..
    const int64_t i0 = (int64_t)blockIdx.y * BT, j0 = (int64_t)blockIdx.x * BT;
    float acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0f;
    for (int64_t p0 = 0; p0 < k; p0 += BK) {
        // A [m][k] rows: lanes along p
        for (int e = t; e < BT * BK; e += 256) {
            const int r = e / BK, p = e % BK;
            const int64_t i = i0 + r, pp = p0 + p;
            As[p][r] = (i < m && pp < k) ? A[i * lda + pp] : 0.0f;
        }
        if (transpose_b) {   // B [n][k]: lanes along p
            for (int e = t; e < BT * BK; e += 256) {
                const int r = e / BK, p = e % BK;
                const int64_t j = j0 + r, pp = p0 + p;
                Bs[p][r] = (j < n && pp < k) ? B[j * ldb + pp] : 0.0f;
            }
        } else {             // B [k][n]: lanes along j
            for (int e = t; e < BT * BK; e += 256) {
                const int p = e / BT, r = e % BT;
                const int64_t j = j0 + r, pp = p0 + p;
                Bs[p][r] = (j < n && pp < k) ? B[pp * ldb + j] : 0.0f;
            }
        }
        __syncthreads();
        const int pk = (int)imin64(BK, k - p0);
        for (int p = 0; p < pk; ++p) {
            const float4 av = *reinterpret_cast<const float4 *>(&As[p][ty * 4]);
            const float4 bv = *reinterpret_cast<const float4 *>(&Bs[p][tx * 4]);
            const float ar[4] = {av.x, av.y, av.z, av.w}, br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = __fadd_rn(acc[u][v], __fmul_rn(ar[u], br[v]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t i = i0 + ty * 4 + u, j = j0 + tx * 4 + v;
            if (i < m && j < n) O[i * ldo + j] = __fmul_rn(acc[u][v], alpha);
        }
}

// quantize (tensor.py:140-151): clamp(rint(f64 x / f64 scale) + zp, lo, hi)
__device__ __forceinline__ uint32_t quant1(float x, double scale, int32_t zp, int32_t lo, int32_t hi)
{
    double q = rint(__ddiv_rn((double)x, scale)) + (double)zp;
    q = fmin(fmax(q, (double)lo), (double)hi);
    return (uint32_t)(uint8_t)(int32_t)q;   // the s8 / u8 byte
}
// four elements per thread: 16-byte loads, one 4-byte store
__global__ void k_quantize4(const float4 *x, int64_t n4, double scale, int32_t zp, int32_t lo, int32_t hi,
                            uint32_t *out)
{
    SI_PDL_ENTRY();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(x + i);
        out[i] = quant1(v.x, scale, zp, lo, hi) | quant1(v.y, scale, zp, lo, hi) << 8 |
                 quant1(v.z, scale, zp, lo, hi) << 16 | quant1(v.w, scale, zp, lo, hi) << 24;
    }
}

__global__ void k_quantize(const float *x, int64_t n, double scale, int32_t zp, int32_t lo, int32_t hi, void *out,
                           int out_s8)
{
    SI_PDL_ENTRY();
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
    if (rows_fit(n)) {
        const int smem = ROWS * (int)(n + 1) * 4;
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_softmax_rows_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        launch_pdl(k_softmax_rows_smem, dim3((unsigned)((rows + ROWS - 1) / ROWS)), dim3(32), smem, (cudaStream_t)stream, x, out, rows,
                                                                                                       (int)n);
    } else {
        launch_pdl(k_softmax_rows, dim3(grid_rows(rows)), dim3(128), 0, (cudaStream_t)stream, x, out, rows, n, n);
    }
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
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out) |
                           reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(beta)) & 15) == 0;
    if (n % 4 == 0 && aligned && (int64_t)ROWS * (n + 4) * 4 <= SMEM_ROWS_MAX) {   // 84 -> 46 us on config 4
        const int smem = ROWS * (int)(n + 4) * 4;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_layer_norm_rows_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        launch_pdl(k_layer_norm_rows_bulk, dim3((unsigned)((rows + ROWS - 1) / ROWS)), dim3(32), smem, (cudaStream_t)stream, 
            x, gamma, beta, eps, out, rows, (int)n);
    } else if (rows_fit(n)) {
        const int smem = ROWS * (int)(n + 1) * 4;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_layer_norm_rows_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        launch_pdl(k_layer_norm_rows_smem, dim3((unsigned)((rows + ROWS - 1) / ROWS)), dim3(32), smem, (cudaStream_t)stream, 
            x, gamma, beta, eps, out, rows, (int)n);
    } else {
        launch_pdl(k_layer_norm_rows, dim3(grid_rows(rows)), dim3(128), 0, (cudaStream_t)stream, x, gamma, beta, eps, out, rows, n);
    }
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
    launch_pdl(k_bmm, dim3(grid), dim3(256), 0, (cudaStream_t)stream, a, b, out, nb1, m, k, n, sa0, sa1, lda, sb0, sb1, ldb, so0, so1, ldo,
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
    if (n % 4 == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
        const int64_t b4 = imin64((n / 4 + threads - 1) / threads, 148 * 16);
        launch_pdl(k_quantize4, dim3((unsigned)b4), dim3(threads), 0, (cudaStream_t)stream, reinterpret_cast<const float4 *>(x), n / 4,
                                                                       (double)scale, zp, lo, hi,
                                                                       static_cast<uint32_t *>(out));
    } else {
        launch_pdl(k_quantize, dim3((unsigned)blocks), dim3(threads), 0, (cudaStream_t)stream, x, n, (double)scale, zp, lo, hi, out,
                                                                           lo < 0);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { si_set_error(cudaGetErrorString(e)); return SI_ECUDA; }
    return SI_OK;
}

// ---- fused attention block of the encoder: per (sequence, head), scores,
// softmax and context in one CTA with everything in shared memory.  The same
// three reference operators in the same orders (bmm_nt * alpha, softmax_rows,
// bmm_nn; eltwise.py:34-160), so the result equals the unfused ops bit for
// bit, without the scores' round trip through HBM.
namespace {
constexpr int AT_S = 128, AT_D = 64;   // supported maximum seq, head dim
constexpr int AT_LQ = AT_D + 4;        // q / k row stride: 16-byte rows, rows 4 banks apart
constexpr int AT_LP = AT_S + 1;        // row stride of the probabilities
// smem: [ Q | K ] ([S][D+4] each) aliased by P [S][S+1] once the scores are
// in registers, then V [S][D]: ~100 KB, two CTAs per SM.
constexpr int AT_QK = 2 * AT_S * AT_LQ > AT_S * AT_LP ? 2 * AT_S * AT_LQ : AT_S * AT_LP;
constexpr int AT_SMEM = (AT_QK + AT_S * AT_D) * 4;

// two CTAs per SM (128 registers, a few spills) measured 248 us on config 4
// against 268 us for one CTA per SM at 138 registers
__global__ void __launch_bounds__(256, 2) k_attention(const float *qkv, float *ctx, int64_t seq, int64_t heads,
                                                      int64_t d, int64_t ld, int64_t ldo, float alpha)
{
    SI_PDL_ENTRY();
    extern __shared__ __align__(16) float sm[];
    float *Qs = sm;                    // [S][D+4]
    float *Ks = sm + AT_S * AT_LQ;     // [S][D+4]
    float *Ps = sm;                    // [S][S+1], after the scores
    float *Vs = sm + AT_QK;            // [S][D]
    const int64_t b = blockIdx.x / heads, h = blockIdx.x % heads;
    const int t = threadIdx.x;
    const int S = (int)seq, D = (int)d;
    const float *base = qkv + b * seq * ld + h * d;
    const int64_t H = heads * d;
    const bool vec = ((D | ld | H | h * d) & 3) == 0 && (reinterpret_cast<uintptr_t>(qkv) & 15) == 0;
    if (vec) {
        // 16-byte loads, all of a thread's loads in flight before the stores
        const int D4 = D >> 2, n4 = S * D4;
        for (int e0 = t; e0 < n4; e0 += 256 * 4) {
            float4 q[4], k[4], v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 256;
                if (e < n4) {
                    const int i = e / D4, p4 = e - i * D4;
                    const float4 *row = reinterpret_cast<const float4 *>(base + i * ld) + p4;
                    q[u] = __ldg(row);
                    k[u] = __ldg(row + H / 4);
                    v[u] = __ldg(row + H / 2);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 256;
                if (e < n4) {
                    const int i = e / D4, p = (e - i * D4) * 4;
                    *reinterpret_cast<float4 *>(Qs + i * AT_LQ + p) = q[u];
                    *reinterpret_cast<float4 *>(Ks + i * AT_LQ + p) = k[u];
                    *reinterpret_cast<float4 *>(Vs + i * AT_D + p) = v[u];
                }
            }
        }
    } else {
        for (int e = t; e < S * D; e += 256) {
            const int i = e / D, p = e - i * D;
            const float *row = base + i * ld;
            Qs[i * AT_LQ + p] = row[p];
            Ks[i * AT_LQ + p] = row[H + p];
            Vs[i * AT_D + p] = row[2 * H + p];
        }
    }
    __syncthreads();
    // scores: rows 4*ib + r, columns jb + 8*c; every output still sums
    // p = 0..D-1 in order with separate mul and add
    const int jb = t & 7, ib = t >> 3;
    {
        float acc[4][16];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[r][c] = 0.0f;
        const int D4 = D & ~3;
#pragma unroll 1
        for (int p = 0; p < D4; p += 4) {
            float4 q[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) q[r] = *reinterpret_cast<const float4 *>(Qs + (ib * 4 + r) * AT_LQ + p);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const float4 k = *reinterpret_cast<const float4 *>(Ks + (jb + 8 * c) * AT_LQ + p);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    float a = acc[r][c];
                    a = __fadd_rn(a, __fmul_rn(q[r].x, k.x));
                    a = __fadd_rn(a, __fmul_rn(q[r].y, k.y));
                    a = __fadd_rn(a, __fmul_rn(q[r].z, k.z));
                    acc[r][c] = __fadd_rn(a, __fmul_rn(q[r].w, k.w));
                }
            }
        }
#pragma unroll 1
        for (int p = D4; p < D; ++p) {
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const float k = Ks[(jb + 8 * c) * AT_LQ + p];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    acc[r][c] = __fadd_rn(acc[r][c], __fmul_rn(Qs[(ib * 4 + r) * AT_LQ + p], k));
            }
        }
        __syncthreads();   // Q / K dead: P takes their place
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = ib * 4 + r;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const int j = jb + 8 * c;
                if (i < S && j < S) Ps[i * AT_LP + j] = __fmul_rn(acc[r][c], alpha);
            }
        }
    }
    __syncthreads();
    // softmax in the reference's order: the row max and the f64 sum stay
    // sequential per row; the exps and the final scaling are elementwise
    __shared__ float rmax[AT_S], rinv[AT_S];
    if (t < S) {
        const float *r = Ps + t * AT_LP;
        float m = r[0];
        for (int c = 1; c < S; ++c)
            if (r[c] > m) m = r[c];
        rmax[t] = m;
    }
    __syncthreads();
    for (int e = t; e < S * S; e += 256) {
        const int i = e / S, c = e - i * S;
        Ps[i * AT_LP + c] = (float)exp((double)Ps[i * AT_LP + c] - (double)rmax[i]);
    }
    __syncthreads();
    if (t < S) {
        const float *r = Ps + t * AT_LP;
        double s = 0.0;
        for (int c = 0; c < S; ++c) s = __dadd_rn(s, (double)r[c]);
        rinv[t] = (float)(1.0 / s);
    }
    __syncthreads();
    for (int e = t; e < S * S; e += 256) {
        const int i = e / S, c = e - i * S;
        Ps[i * AT_LP + c] = __fmul_rn(Ps[i * AT_LP + c], rinv[i]);
    }
    __syncthreads();
    // context: rows 4*ib + r, columns 4*jb + {0..3} and 32 + 4*jb + {0..3};
    // p = 0..S-1 in order
    {
        float acc[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r][c] = 0.0f;
        for (int p = 0; p < S; ++p) {
            float pv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) pv[r] = Ps[min(ib * 4 + r, AT_S - 1) * AT_LP + p];
            const float4 v0 = *reinterpret_cast<const float4 *>(Vs + p * AT_D + jb * 4);
            const float4 v1 = *reinterpret_cast<const float4 *>(Vs + p * AT_D + 32 + jb * 4);
            const float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = __fadd_rn(acc[r][c], __fmul_rn(pv[r], vv[c]));
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = ib * 4 + r;
            if (i >= S) continue;
            float *o = ctx + (b * seq + i) * ldo + h * d;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int j = (c < 4 ? 0 : 32) + jb * 4 + (c & 3);
                if (j < D) o[j] = __fmul_rn(acc[r][c], 1.0f);
            }
        }
    }
}
}  // namespace

extern "C" int32_t si_attention_f32(const float *qkv, float *ctx, int64_t batch, int64_t seq, int64_t heads,
                                    int64_t head_dim, int64_t ld_qkv, int64_t ld_ctx, float alpha, void *stream)
{
    if (!qkv || !ctx || batch < 0 || seq <= 0 || heads <= 0 || head_dim <= 0) {
        si_set_error("attention: bad arguments");
        return SI_EINVAL;
    }
    if (seq > AT_S || head_dim > AT_D || head_dim > 64) {
        si_set_error("attention: fused kernel supports seq <= 128 and head_dim <= 64");
        return SI_EUNSUPPORTED;
    }
    if (batch == 0) return SI_OK;
    const int smem = AT_SMEM;
    // (cheap; set on every call so every device of the process has it)
    cudaFuncSetAttribute(k_attention, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    launch_pdl(k_attention, dim3((unsigned)(batch * heads)), dim3(256), smem, (cudaStream_t)stream, qkv, ctx, seq, heads, head_dim, ld_qkv,
                                                                               ld_ctx, alpha);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { si_set_error(cudaGetErrorString(e)); return SI_ECUDA; }
    return SI_OK;
}
