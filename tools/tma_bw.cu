// tma_bw.cu -- experiment harness (not part of the product library): TMA
// streaming throughput vs ring depth / box size.  Every CTA streams boxes of
// [rows x 128 B] from a 2D u8 tensor through a ring of S slots; a consumer
// thread waits for each slot and releases it at once.  Built by tools/tma_bw.py.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2306_16601_b200/csrc/tc_ptx.cuh"

__global__ void tma_bw_kernel(const __grid_constant__ CUtensorMap tm, int S, int box_rows, int iters, int rows_total,
                              int stride_ctas, int nprod, int ncols)
{
    // nprod >= 1000: warp-converged producers (whole warp loops, one elected
    // lane issues, tcw::), nprod - 1000 of them
    const bool conv = nprod >= 1000;
    if (conv) nprod -= 1000;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    const int slot_bytes = box_rows * 128;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * slot_bytes);
    uint64_t *empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tm);
    }
    __syncthreads();
    const int nboxes = rows_total / box_rows;
    const int w = threadIdx.x >> 5;
    if (w >= 2 && w < 2 + (nprod < 0 ? -nprod : nprod) && (conv || (threadIdx.x & 31) == 0)) {
        // producer p issues iterations i = p, p + nprod, ... (slot i % S)
        for (int i = w - 2; i < iters; i += (nprod < 0 ? -nprod : nprod)) {
            const int stage = i % S;
            const uint32_t phase = (uint32_t)((i / S) & 1);
            tc::mbar_spin(&empty[stage], phase ^ 1);
            if (conv) tcw::mbar_expect_tx(&full[stage], slot_bytes);
            else tc::mbar_expect_tx(&full[stage], slot_bytes);
            int b, col;
            if (stride_ctas == 0) {
                // disjoint: CTA c streams its own slice of the buffer
                const int per = nboxes / (int)gridDim.x;
                b = (int)blockIdx.x * per + (per ? i % per : 0);
                col = 0;
            } else {
                const unsigned q = (unsigned)blockIdx.x * (unsigned)stride_ctas + (unsigned)i;
                b = (int)(q & (unsigned)(nboxes - 1));
                col = (int)((q >> 4) & (unsigned)(ncols - 1));
            }
            if (conv) tcw::tma_load_2d(smem + stage * slot_bytes, &tm, &full[stage], col * 128, b * box_rows);
            else tc::tma_load_2d(smem + stage * slot_bytes, &tm, &full[stage], col * 128, b * box_rows);
        }
    } else if (threadIdx.x == 32) {
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < iters; ++i) {
            tc::mbar_wait(&full[stage], phase);
            if (nprod < 0) tc::mma_commit(&empty[stage]);   // release through the tensor pipe
            else tc::mbar_arrive(&empty[stage]);
            if (++stage == S) { stage = 0; phase ^= 1; }
        }
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// returns GB/s (bytes delivered to smem / time), or < 0 on error
extern "C" double tma_bw(const void *buf, long rows_total, int S, int box_rows, int iters, int ctas, int stride_ctas,
                         int reps, int nprod, long pitch)
{
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) return -1;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows_total};
    cuuint64_t strides[1] = {(cuuint64_t)pitch};
    const int ncols = (int)(pitch / 128);
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    if (reinterpret_cast<EncodeTiledFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(buf), dims,
                                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -2;
    const int smem = S * box_rows * 128 + 1024 + 2048;
    if (cudaFuncSetAttribute(tma_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return -3;
    const int np = nprod >= 1000 ? nprod - 1000 : (nprod < 0 ? -nprod : nprod);
    tma_bw_kernel<<<ctas, 64 + 32 * np, smem>>>(tm, S, box_rows, iters, (int)rows_total, stride_ctas, nprod, ncols);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) tma_bw_kernel<<<ctas, 64 + 32 * np, smem>>>(tm, S, box_rows, iters, (int)rows_total, stride_ctas, nprod, ncols);
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess) return -4;
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return (double)ctas * iters * box_rows * 128.0 * reps / (ms * 1e-3) / 1e9;
}

// ---- pair mode: cluster of 2, each CTA issues .cta_group::2 loads that
// complete on the leader's barrier (as k2p does); the leader's consumer
// releases the slot in both CTAs
__global__ void __cluster_dims__(2, 1, 1) tma_bw2_kernel(const __grid_constant__ CUtensorMap tm, int S, int box_rows,
                                                         int iters, int rows_total, int nprod, int boxes_per_stage)
{
    const bool release_commit = nprod < 0;
    if (nprod < 0) nprod = -nprod;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    const int box_bytes = box_rows * 128;
    const int slot_bytes = box_bytes * boxes_per_stage;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * slot_bytes);
    uint64_t *empty = full + S;
    const uint32_t rank = tc::cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tm);
    }
    tc::cluster_sync();
    const int nboxes = rows_total / box_rows;
    const int per = nboxes / (int)gridDim.x;
    const int w = threadIdx.x >> 5;
    const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
    if (w >= 2 && w < 2 + nprod && (threadIdx.x & 31) == 0) {
        for (int i = w - 2; i < iters; i += nprod) {
            const int stage = i % S;
            const uint32_t phase = (uint32_t)((i / S) & 1);
            tc::mbar_spin(&empty[stage], phase ^ 1);
            if (rank == 0) tc::mbar_expect_tx(&full[stage], 2 * slot_bytes);
            for (int j = 0; j < boxes_per_stage; ++j) {
                const int b = (int)blockIdx.x * per + (per ? (i * boxes_per_stage + j) % per : 0);
                tc::tma_load_2d_2sm(smem + stage * slot_bytes + j * box_bytes, &tm, full0 + 8 * stage, 0,
                                    b * box_rows);
            }
        }
    } else if (threadIdx.x == 32 && rank == 0) {
        const uint32_t empty1 = tc::mapa(tc::smem_u32(empty), 1);
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < iters; ++i) {
            tc::mbar_wait(&full[stage], phase);
            if (release_commit) {
                // release through the tensor pipe: 2-SM commit multicast to both CTAs
                tc::mma_commit_2sm_mc(&empty[stage], 0x3);
            } else {
                tc::mbar_arrive(&empty[stage]);
                tc::mbar_arrive_cluster(empty1 + 8 * stage);
            }
            if (++stage == S) { stage = 0; phase ^= 1; }
        }
    }
    tc::cluster_sync();
}

extern "C" double tma_bw2(const void *buf, long rows_total, int S, int box_rows, int iters, int ctas, int reps,
                          int nprod, int boxes_per_stage)
{
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) return -1;
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, (cuuint64_t)rows_total};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    if (reinterpret_cast<EncodeTiledFn>(fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(buf), dims,
                                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -2;
    const int smem = S * box_rows * 128 * boxes_per_stage + 1024 + 2048;
    if (cudaFuncSetAttribute(tma_bw2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return -3;
    const int nthr = 64 + 32 * (nprod < 0 ? -nprod : nprod);
    tma_bw2_kernel<<<ctas, nthr, smem>>>(tm, S, box_rows, iters, (int)rows_total, nprod, boxes_per_stage);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r)
        tma_bw2_kernel<<<ctas, nthr, smem>>>(tm, S, box_rows, iters, (int)rows_total, nprod, boxes_per_stage);
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess) return -4;
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return (double)ctas * iters * box_rows * 128.0 * boxes_per_stage * reps / (ms * 1e-3) / 1e9;
}

// ---- the pair kernel's exact TMA stream (BASELINE 5b geometry) without its
// other roles: units (token tile nt, 256-row tile mt), m fastest, strided over
// the pairs; per 128-k stage each CTA loads its W^T half box {128 m, 128 k}
// and its X half box {128 tok, 128 k} (SWIZZLE_128B) onto the leader's barrier.
__global__ void __cluster_dims__(2, 1, 1) tma_pairk_kernel(const __grid_constant__ CUtensorMap tw,
                                                           const __grid_constant__ CUtensorMap tx, int S, int mtiles,
                                                           int ntiles, int kchunks, int nprod, int mode)
{
    // mode bits: 1 allocate 512 TMEM columns (pair), 2 sixteen extra warps
    // parked on a barrier until the end (the kernel's epilogue warps)
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    constexpr int SLOT = 32768;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * SLOT);
    uint64_t *empty = full + S;
    uint64_t *done = empty + S;
    uint32_t *tslot = reinterpret_cast<uint32_t *>(done + 1);
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_init(done, 1);
        tc::mbar_fence_init();
    }
    const int w = threadIdx.x >> 5;
    if ((mode & 1) && w == 0) tc::tmem_alloc_2sm(tslot, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const int units = mtiles * ntiles;
    const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
    if (w >= 2 && w < 2 + nprod) {
        const int prod = w - 2;
        int stage = 0, it = 0;
        uint32_t phase = 0;
        for (int u = pair; u < units; u += npairs) {
            const int nt = u / mtiles, mt = u % mtiles;
            for (int kc = 0; kc < kchunks; ++kc, ++it) {
                if (it % nprod == prod) {
                    tc::mbar_spin(&empty[stage], phase ^ 1);
                    if (rank == 0) tcw::mbar_expect_tx(&full[stage], 2 * SLOT);
                    uint8_t *a = smem + stage * SLOT;
                    tcw::tma_load_2d_2sm(a, &tw, full0 + 8 * stage, mt * 256 + 128 * (int)rank, kc * 128);
                    tcw::tma_load_2d_2sm(a + 16384, &tx, full0 + 8 * stage, nt * 256 + 128 * (int)rank, kc * 128);
                }
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
        }
    } else if (w == 1 && rank == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int u = pair; u < units; u += npairs)
            for (int kc = 0; kc < kchunks; ++kc) {
                tc::mbar_spin(&full[stage], phase);
                tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
        if ((threadIdx.x & 31) == 0) {
            tc::mbar_arrive(done);
            tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(done), 1));
        }
    } else if (w >= 2 + nprod && (mode & 2)) {
        tc::mbar_wait(done, 0);
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if ((mode & 1) && w == 0) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(*tslot, 512);
    }
}

extern "C" double tma_pairk(const void *wt, const void *x, int M, int K, int N, int S, int nprod, int reps, int mode)
{
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) return -1;
    auto enc = reinterpret_cast<EncodeTiledFn>(fn);
    CUtensorMap tw, tx;
    cuuint64_t dw[2] = {(cuuint64_t)M, (cuuint64_t)K}, sw[1] = {(cuuint64_t)M};
    cuuint64_t dx[2] = {(cuuint64_t)N, (cuuint64_t)K}, sx[1] = {(cuuint64_t)N};
    cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(wt), dw, sw, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
        enc(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(x), dx, sx, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
        return -2;
    const int smem = S * 32768 + 1024 + 1024;
    if (cudaFuncSetAttribute(tma_pairk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return -3;
    const int mtiles = M / 256, ntiles = N / 256, kchunks = K / 128;
    const int threads = 64 + 32 * nprod + ((mode & 2) ? 32 * 16 : 0);
    tma_pairk_kernel<<<148, threads, smem>>>(tw, tx, S, mtiles, ntiles, kchunks, nprod, mode);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) tma_pairk_kernel<<<148, threads, smem>>>(tw, tx, S, mtiles, ntiles, kchunks, nprod, mode);
    cudaEventRecord(b);
    if (cudaEventSynchronize(b) != cudaSuccess) return -4;
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3 / reps;   // us per sweep
}
