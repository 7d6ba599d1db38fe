// spmm_gather.cu -- K1, the CUDA-core gather SpMM, plus the naive per-element
// reference kernel and the token-major transpose.
//
// K1 replaces _acc_group_panel + _spmm_task_* (spmm.py:192-280).  The
// reference's micro-tile (sparse.py:28-31) is kept as the device weight
// format because it is already dp4a-shaped: tile row r is the s8x4 word of
// row r over the tile's 4 block columns.  One warp owns one 4-row group and
// 128 tokens (4 per lane).  Per micro-tile a lane issues 4 coalesced 32-bit
// loads of the gathered activation rows X[idx_c][n..n+3], byte-transposes
// them with 8 PRMT into 4 per-token words X[idx_0..3][n+t], and issues 16
// dp4a.u32.s32 (4 rows x 4 tokens) -- the VNNI step of Alg. 1 (PAPER.md:
// 123-158) on 32-lane warps.  Integer accumulation wraps mod 2^32, exactly as
// the reference, and is order independent, so any schedule gives the same
// bits.  The epilogue runs in registers; a CTA (8 warps = 32 output rows)
// stages its [128 tokens x 32 rows] tile in shared memory and writes it out
// token-major ([N, M], spmm.py:236) with coalesced row segments.  K1s (below)
// is the same kernel reading its gathered rows from a cp.async-staged slab.
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <set>

#include "epilogue.cuh"
#include "si_internal.h"

namespace {

constexpr int K1_WARPS = 8;          // groups per CTA
constexpr int K1_TOK = 128;          // tokens per CTA (4 per lane)
constexpr int K1_ROWS = 4 * K1_WARPS;

__device__ __forceinline__ int32_t dp4a_us(uint32_t a_u8x4, uint32_t b_s8x4, int32_t c)
{
    int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_u8x4), "r"(b_s8x4), "r"(c));
    return d;
}

template <bool VEC>
__device__ __forceinline__ uint32_t load_x4(const uint8_t *__restrict__ x, int64_t row_off, int64_t n0,
                                            int64_t N)
{
    const uint8_t *p = x + row_off + n0;
    if (VEC && n0 + 3 < N) return __ldg(reinterpret_cast<const uint32_t *>(p));
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (n0 + i < N) v |= (uint32_t)__ldg(p + i) << (8 * i);
    return v;
}

template <int MODE, int OUTB, bool VEC>
__global__ void __launch_bounds__(K1_WARPS * 32)
k1_gather_kernel(const int32_t *__restrict__ tile_ptr, const uint4 *__restrict__ tile_w,
                 const int4 *__restrict__ tile_idx, int32_t groups, const uint8_t *__restrict__ x,
                 int64_t ldx, int64_t N, void *__restrict__ out, int64_t ldo, EpiParams E)
{
    SI_PDL_ENTRY();
    __shared__ uint32_t stage[K1_ROWS][K1_TOK + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t g = blockIdx.y * K1_WARPS + warp;
    const int64_t nb = (int64_t)blockIdx.x * K1_TOK;
    const int64_t n0 = nb + lane * 4;

    int32_t acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[r][t] = 0;

    if (g < groups) {
        const int32_t t0 = __ldg(tile_ptr + g), t1 = __ldg(tile_ptr + g + 1);
#pragma unroll 4
        for (int32_t t = t0; t < t1; ++t) {
            const uint4 w = __ldg(tile_w + t);
            const int4 ix = __ldg(tile_idx + t);
            const uint32_t x0 = load_x4<VEC>(x, (int64_t)ix.x * ldx, n0, N);
            const uint32_t x1 = load_x4<VEC>(x, (int64_t)ix.y * ldx, n0, N);
            const uint32_t x2 = load_x4<VEC>(x, (int64_t)ix.z * ldx, n0, N);
            const uint32_t x3 = load_x4<VEC>(x, (int64_t)ix.w * ldx, n0, N);
            // 4x4 byte transpose: tok[t] = (x0.b_t, x1.b_t, x2.b_t, x3.b_t)
            const uint32_t lo01 = __byte_perm(x0, x1, 0x5140), lo23 = __byte_perm(x2, x3, 0x5140);
            const uint32_t hi01 = __byte_perm(x0, x1, 0x7362), hi23 = __byte_perm(x2, x3, 0x7362);
            const uint32_t tok[4] = {__byte_perm(lo01, lo23, 0x5410), __byte_perm(lo01, lo23, 0x7632),
                                     __byte_perm(hi01, hi23, 0x5410), __byte_perm(hi01, hi23, 0x7632)};
            const uint32_t wr[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) acc[r][tt] = dp4a_us(tok[tt], wr[r], acc[r][tt]);
        }
        // epilogue in registers (spmm.py:227-236)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int32_t m = g * 4 + r;
            if (m < E.M) {
                const int32_t adj = __ldg(E.adj + m);
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                    const int64_t n = n0 + tt;
                    uint32_t v = 0;
                    if (n < N) v = epi_apply<MODE>((int32_t)((uint32_t)acc[r][tt] + (uint32_t)adj), m, n, E);
                    stage[warp * 4 + r][lane * 4 + tt] = v;
                }
            }
        }
    }
    __syncthreads();
    // token-major store: each warp writes whole token rows of the 32-row slab
    const int32_t m0 = blockIdx.y * K1_ROWS;
    const int32_t mrow = m0 + lane;
    for (int t = warp; t < K1_TOK; t += K1_WARPS) {
        const int64_t n = nb + t;
        if (n >= N) break;
        if (mrow < E.M) {
            const uint32_t v = stage[lane][t];
            if (OUTB == 4)
                reinterpret_cast<uint32_t *>(out)[n * ldo + mrow] = v;
            else
                reinterpret_cast<uint8_t *>(out)[n * ldo + mrow] = (uint8_t)(v & 0xFF);
        }
    }
}

// K1s: the same kernel with the CTA's activation tile staged in shared memory.
// The whole [K x 128 tokens] slab the CTA's 8 groups gather from is brought in
// once with 16-byte cp.async (K * 128 B <= K1S_SLAB), and each warp's first
// K1S_TILES micro-tiles (weights + column indices) with it, so the gathered row
// loads of the block loop are conflict-free LDS.32 instead of dependent L2
// round trips (the small-N cells are latency-bound: 24 CTAs of config 1 each
// walk ~20 micro-tiles).  Needs [K, N] activations with a 16-byte-aligned
// base and leading dimension (the transposed workspace of the [N, K] path
// qualifies); everything after the block loop is K1's.
constexpr int K1S_TILES = 128;                        // micro-tiles per group staged next to the slab
constexpr int K1S_WBYTES = K1_WARPS * K1S_TILES * 32; // their weights + column indices (32 KB)
constexpr int K1S_SLAB = 160 * 1024;                  // largest activation slab (K <= 1280)

__device__ __forceinline__ void cp_async_16(uint32_t dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <int MODE, int OUTB>
__global__ void __launch_bounds__(K1_WARPS * 32)
k1s_gather_kernel(const int32_t *__restrict__ tile_ptr, const uint4 *__restrict__ tile_w,
                  const int4 *__restrict__ tile_idx, int32_t groups, int32_t K, const uint8_t *__restrict__ x,
                  int64_t ldx, int64_t N, void *__restrict__ out, int64_t ldo, EpiParams E)
{
    extern __shared__ __align__(16) uint8_t dyn[];
    uint4 *ws_w = reinterpret_cast<uint4 *>(dyn);                       // [warp][K1S_TILES] weights
    int4 *ws_i = reinterpret_cast<int4 *>(dyn + K1S_WBYTES / 2);        // [warp][K1S_TILES] column indices
    uint8_t *xs = dyn + K1S_WBYTES;                                     // [K][K1_TOK]
    __shared__ uint32_t stage[K1_ROWS][K1_TOK + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t g = blockIdx.y * K1_WARPS + warp;
    const int64_t nb = (int64_t)blockIdx.x * K1_TOK;
    const int64_t n0 = nb + lane * 4;
    // this warp's micro-tiles (weights, column indices) do not depend on the
    // previous kernel: their copy starts before the grid dependency wait
    int32_t t0 = 0, t1 = 0;
    if (g < groups) {
        t0 = __ldg(tile_ptr + g);
        t1 = __ldg(tile_ptr + g + 1);
    }
    const int32_t nst = min(t1 - t0, K1S_TILES);
    {
        const uint32_t w_u = (uint32_t)__cvta_generic_to_shared(ws_w + warp * K1S_TILES);
        const uint32_t i_u = (uint32_t)__cvta_generic_to_shared(ws_i + warp * K1S_TILES);
        for (int t = lane; t < nst; t += 32) {
            cp_async_16(w_u + 16 * t, tile_w + t0 + t);
            cp_async_16(i_u + 16 * t, tile_idx + t0 + t);
        }
    }
    SI_PDL_ENTRY();
    {
        // stage the slab: 8 chunks of 16 B per activation row (chunks wholly
        // past the leading dimension are skipped; their tokens are never stored)
        const uint32_t xs_u = (uint32_t)__cvta_generic_to_shared(xs);
        const int chunks = K * (K1_TOK / 16);
        for (int c = threadIdx.x; c < chunks; c += K1_WARPS * 32) {
            const int k = c >> 3, j = c & 7;
            const int64_t col = nb + 16 * j;
            if (col < ldx) cp_async_16(xs_u + (uint32_t)c * 16, x + (int64_t)k * ldx + col);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
    }

    int32_t acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[r][t] = 0;

    if (g < groups) {
        const uint32_t *xw = reinterpret_cast<const uint32_t *>(xs) + lane;   // this lane's 4 tokens of row 0
        const uint4 *sw = ws_w + warp * K1S_TILES;
        const int4 *si = ws_i + warp * K1S_TILES;
#pragma unroll 4
        for (int32_t t = 0; t < t1 - t0; ++t) {
            // (staged tiles from shared memory, a longer group's tail straight from L2)
            const uint4 w = t < nst ? sw[t] : __ldg(tile_w + t0 + t);
            const int4 ix = t < nst ? si[t] : __ldg(tile_idx + t0 + t);
            const uint32_t x0 = xw[ix.x * (K1_TOK / 4)], x1 = xw[ix.y * (K1_TOK / 4)];
            const uint32_t x2 = xw[ix.z * (K1_TOK / 4)], x3 = xw[ix.w * (K1_TOK / 4)];
            const uint32_t lo01 = __byte_perm(x0, x1, 0x5140), lo23 = __byte_perm(x2, x3, 0x5140);
            const uint32_t hi01 = __byte_perm(x0, x1, 0x7362), hi23 = __byte_perm(x2, x3, 0x7362);
            const uint32_t tok[4] = {__byte_perm(lo01, lo23, 0x5410), __byte_perm(lo01, lo23, 0x7632),
                                     __byte_perm(hi01, hi23, 0x5410), __byte_perm(hi01, hi23, 0x7632)};
            const uint32_t wr[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) acc[r][tt] = dp4a_us(tok[tt], wr[r], acc[r][tt]);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int32_t m = g * 4 + r;
            if (m < E.M) {
                const int32_t adj = __ldg(E.adj + m);
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                    const int64_t n = n0 + tt;
                    uint32_t v = 0;
                    if (n < N) v = epi_apply<MODE>((int32_t)((uint32_t)acc[r][tt] + (uint32_t)adj), m, n, E);
                    stage[warp * 4 + r][lane * 4 + tt] = v;
                }
            }
        }
    }
    __syncthreads();
    const int32_t m0 = blockIdx.y * K1_ROWS;
    const int32_t mrow = m0 + lane;
    for (int t = warp; t < K1_TOK; t += K1_WARPS) {
        const int64_t n = nb + t;
        if (n >= N) break;
        if (mrow < E.M) {
            const uint32_t v = stage[lane][t];
            if (OUTB == 4)
                reinterpret_cast<uint32_t *>(out)[n * ldo + mrow] = v;
            else
                reinterpret_cast<uint8_t *>(out)[n * ldo + mrow] = (uint8_t)(v & 0xFF);
        }
    }
}

// [N, K] token-major -> [K, ldt] (ldt = N rounded up to 16) through smem
__global__ void transpose_nk_kernel(const uint8_t *__restrict__ x, int64_t ldx, int64_t N, int32_t K,
                                    uint8_t *__restrict__ xt, int64_t ldt)
{
    SI_PDL_ENTRY();
    __shared__ uint8_t tile[64][65];
    const int64_t n0 = (int64_t)blockIdx.x * 64;
    const int32_t k0 = blockIdx.y * 64;
    for (int i = threadIdx.y; i < 64; i += blockDim.y) {
        for (int j = threadIdx.x; j < 64; j += blockDim.x) {
            const int64_t n = n0 + i;
            const int32_t k = k0 + j;
            tile[i][j] = (n < N && k < K) ? x[n * ldx + k] : 0;
        }
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 64; i += blockDim.y) {
        for (int j = threadIdx.x; j < 64; j += blockDim.x) {
            const int32_t k = k0 + i;
            const int64_t n = n0 + j;
            if (k < K && n < ldt) xt[(int64_t)k * ldt + n] = tile[j][i];
        }
    }
}

// naive reference (spmm_ref, spmm.py:401-427): one thread per output
// element, plain loop over the group's blocks, generic interpreter epilogue.
__global__ void ref_kernel(const int32_t *__restrict__ tile_ptr, const int8_t *__restrict__ vals,
                           const int32_t *__restrict__ idx, const uint8_t *__restrict__ x, int32_t layout,
                           int64_t ldx, int64_t N, void *__restrict__ out, int64_t ldo, EpiParams E)
{
    SI_PDL_ENTRY();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= N * (int64_t)E.M) return;
    const int64_t n = e / E.M;
    const int32_t m = (int32_t)(e % E.M);
    const int32_t g = m >> 2, r = m & 3;
    uint32_t acc = 0;
    for (int64_t p = 4 * (int64_t)tile_ptr[g]; p < 4 * (int64_t)tile_ptr[g + 1]; ++p) {
        const int32_t w = vals[(p >> 2) * 16 + r * 4 + (p & 3)];
        const int64_t k = idx[p];
        const uint32_t xv = layout == 0 ? x[k * ldx + n] : x[n * ldx + k];
        acc += (uint32_t)(w * (int32_t)xv);
    }
    const int32_t a32 = (int32_t)(acc + (uint32_t)E.adj[m]);
    uint32_t v = E.mode == EPI_S32 ? (uint32_t)a32 : epi_generic(a32, m, n, E);
    if (E.out_dtype == 0 || E.out_dtype == 3)
        reinterpret_cast<uint32_t *>(out)[n * ldo + m] = v;
    else
        reinterpret_cast<uint8_t *>(out)[n * ldo + m] = (uint8_t)(v & 0xFF);
}

template <int MODE, int OUTB>
void launch_k1_mode(const SpmmArgs &a, const uint8_t *x, int64_t ldx, bool vec, cudaStream_t st)
{
    const SiImage *h = a.h;
    EpiParams E = make_epi(h, a.img, a.sides, a.n);
    dim3 grid((unsigned)((a.n + K1_TOK - 1) / K1_TOK), (unsigned)((h->groups + K1_WARPS - 1) / K1_WARPS));
    auto tp = img_sec<int32_t>(a.img, h->off_tile_ptr);
    auto tw = img_sec<uint4>(a.img, h->off_tile_w);
    auto ti = img_sec<int4>(a.img, h->off_tile_idx);
    // staged variant: 16-byte-aligned [K, N] activations whose slab fits
    const size_t slab = (size_t)h->K * K1_TOK;
    if (ldx % 16 == 0 && ((uintptr_t)x) % 16 == 0 && slab <= (size_t)K1S_SLAB) {
        auto kern = k1s_gather_kernel<MODE, OUTB>;
        static std::mutex mu;
        static std::set<int> done;
        int dev = 0;
        cudaGetDevice(&dev);
        {
            std::lock_guard<std::mutex> lk(mu);
            if (done.insert(dev).second)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K1S_WBYTES + K1S_SLAB);
        }
        launch_pdl(kern, dim3(grid), dim3(K1_WARPS * 32), K1S_WBYTES + slab, st, tp, tw, ti, h->groups, h->K, x, ldx, a.n, a.out,
                   a.ldo, E);
        return;
    }
    if (vec)
        launch_pdl(k1_gather_kernel<MODE, OUTB, true>, dim3(grid), dim3(K1_WARPS * 32), 0, st, tp, tw, ti, h->groups, x, ldx, a.n,
                                                                          a.out, a.ldo, E);
    else
        launch_pdl(k1_gather_kernel<MODE, OUTB, false>, dim3(grid), dim3(K1_WARPS * 32), 0, st, tp, tw, ti, h->groups, x, ldx, a.n,
                                                                           a.out, a.ldo, E);
}

template <int OUTB>
void launch_k1_outb(const SpmmArgs &a, const uint8_t *x, int64_t ldx, bool vec, cudaStream_t st)
{
    switch (a.h->epi_mode) {
    case EPI_S32: launch_k1_mode<EPI_S32, OUTB>(a, x, ldx, vec, st); break;
    case EPI_DEQ_F32: launch_k1_mode<EPI_DEQ_F32, OUTB>(a, x, ldx, vec, st); break;
    case EPI_REQUANT: launch_k1_mode<EPI_REQUANT, OUTB>(a, x, ldx, vec, st); break;
    case EPI_REQUANT_LUT: launch_k1_mode<EPI_REQUANT_LUT, OUTB>(a, x, ldx, vec, st); break;
    case EPI_DEQ_TABLE: launch_k1_mode<EPI_DEQ_TABLE, OUTB>(a, x, ldx, vec, st); break;
    default: launch_k1_mode<EPI_GENERIC, OUTB>(a, x, ldx, vec, st); break;
    }
}

inline int64_t tpad(int64_t n) { return (n + 15) / 16 * 16; }

}  // namespace

bool k1s_preferred(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx)
{
    // the staged kernel wins where its CTAs fit one wave (one CTA per SM: the
    // slab takes most of the shared memory) and a group holds few blocks: the
    // config-2 grid at N = 128 / 512 (profiles/r02c_config2_{gather,tc}.md)
    // crosses over at ~120 blocks per group (768 @85%, 1024 @90%)
    if (layout != SI_ACT_KN || ldx % 16 || ((uintptr_t)x) % 16) return false;
    if ((size_t)h->K * K1_TOK > (size_t)K1S_SLAB) return false;
    static std::atomic<int> sm_count{0};   // (every GPU of a node is the same part)
    int sms = sm_count.load(std::memory_order_relaxed);
    if (sms == 0) {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sms = v > 0 ? v : 148;
        sm_count.store(sms, std::memory_order_relaxed);
    }
    const int64_t ctas = ((n + K1_TOK - 1) / K1_TOK) * ((h->groups + K1_WARPS - 1) / K1_WARPS);
    if (ctas > sms) return false;
    const uint64_t tiles = (h->off_tile_idx - h->off_tile_w) / 16;   // (section padding included: < 64 tiles)
    return 4 * tiles <= 120ull * (uint64_t)h->groups;
}

uint64_t k1_workspace(const SiImage *h, int64_t n, int32_t layout)
{
    return layout == 1 ? (uint64_t)h->K * (uint64_t)tpad(n) : 0;
}

int k1_launch_count(const SiImage *, int32_t layout) { return layout == 1 ? 2 : 1; }

int k1_launch(const SpmmArgs &a)
{
    cudaStream_t st = (cudaStream_t)a.stream;
    const uint8_t *x = a.x;
    int64_t ldx = a.ldx;
    if (a.layout == 1) {
        const int64_t ldt = tpad(a.n);
        dim3 grid((unsigned)((ldt + 63) / 64), (unsigned)((a.h->K + 63) / 64));
        launch_pdl(transpose_nk_kernel, dim3(grid), dim3(dim3(32, 8)), 0, st, a.x, a.ldx, a.n, a.h->K, (uint8_t *)a.ws, ldt);
        x = (const uint8_t *)a.ws;
        ldx = ldt;
    }
    const bool vec = (ldx % 4 == 0) && (((uintptr_t)x) % 4 == 0);
    const int outb = (a.h->out_dtype == 0 || a.h->out_dtype == 3) ? 4 : 1;
    if (outb == 4)
        launch_k1_outb<4>(a, x, ldx, vec, st);
    else
        launch_k1_outb<1>(a, x, ldx, vec, st);
    return (int)cudaGetLastError();
}

int kref_launch(const SpmmArgs &a)
{
    cudaStream_t st = (cudaStream_t)a.stream;
    const SiImage *h = a.h;
    EpiParams E = make_epi(h, a.img, a.sides, a.n);
    const int64_t total = a.n * (int64_t)h->M;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    launch_pdl(ref_kernel, dim3(blocks), dim3(256), 0, st, img_sec<int32_t>(a.img, h->off_tile_ptr),
                                       img_sec<int8_t>(a.img, h->off_tile_w),
                                       img_sec<int32_t>(a.img, h->off_tile_idx), a.x, a.layout, a.ldx, a.n,
                                       a.out, a.ldo, E);
    return (int)cudaGetLastError();
}
