// mma_rate.cu -- experiment harness (not part of the product library):
// tcgen05 kind::i8 issue-rate microbenchmark over CTA pairs (cta_group::2),
// operands static in shared memory / tensor memory, optionally with a
// concurrent bulk-copy stream into a separate shared-memory ring.  Answers:
// what MMA rate do dense and 2:4-sparse M256 x N x K tiles reach, with A
// from shared memory (SS) or from tensor memory (TS), and does a concurrent
// shared-memory write stream slow them down.  Built by tools/mma_rate.py.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2306_16601_b200/csrc/tc_ptx.cuh"

namespace {

__device__ __forceinline__ void mma_ts_i8_2sm(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
        "elect.sync r|p, 0xffffffff;\n\t"
        "setp.ne.b32 q, %4, 0;\n\t"
        "@p tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, q;\n}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_sp_ts_i8_2sm(uint32_t d, uint32_t a, uint64_t b, uint32_t e, uint32_t idesc,
                                                 uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
        "elect.sync r|p, 0xffffffff;\n\t"
        "setp.ne.b32 q, %5, 0;\n\t"
        "@p tcgen05.mma.sp.cta_group::2.kind::i8 [%0], [%1], %2, [%3], %4, q;\n}" ::"r"(d),
        "r"(a), "l"(b), "r"(e), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void cp_256_2sm(uint32_t taddr, uint64_t sdesc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\t"
        "elect.sync r|p, 0xffffffff;\n\t"
        "@p tcgen05.cp.cta_group::2.128x256b [%0], %1;\n}" ::"r"(taddr), "l"(sdesc)
        : "memory");
}

constexpr uint32_t SM_A = 0, SM_B = 16384, SM_E = 49152, SM_RING = 53248, RING_SLOT = 16384, RING_N = 4;
constexpr uint32_t SM_BAR = SM_RING + RING_SLOT * RING_N;  // 118784
constexpr uint32_t SMEM_BYTES = SM_BAR + 256 + 1024;

}  // namespace

// mode: 0 dense SS, 1 dense TS, 2 sparse SS, 3 sparse TS.  Every CTA pair
// issues `iters` M256 x N MMAs (K32 dense, K64 sparse) into one accumulator,
// committing every 16 and keeping at most two groups in flight.
// stream > 0: one warp per CTA bulk-copies `stream` 16 KB chunks of gsrc
// into a 4-slot ring concurrently with the MMAs (its own cycle count is
// reported, so the overlap is checked from both durations).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    mma_rate_kernel(int mode, int iters, int N, int stream, const uint8_t *gsrc, long gchunks,
                    unsigned long long *out, int ldw, int ld_iters)
{
    extern __shared__ __align__(1024) uint8_t smraw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    uint64_t *bars = (uint64_t *)(sm + SM_BAR);  // [2..5] ring, [6..9] mma groups per issuer
    uint32_t *tslot = (uint32_t *)(sm + SM_BAR + 96);
    const int t = threadIdx.x, warp = t >> 5;
    const uint32_t rank = tc::cluster_ctarank();
    for (int i = t; i < 49152 / 4; i += blockDim.x) ((uint32_t *)sm)[i] = 0x01020304u * (uint32_t)(i * 2654435761u);
    for (int i = t; i < 4096 / 4; i += blockDim.x) ((uint32_t *)(sm + SM_E))[i] = 0x44444444u;
    if (t == 0) {
        for (int i = 0; i < 11; ++i) tc::mbar_init(&bars[i], 1);
        tc::mbar_fence_init();
    }
    if (warp == 1) tc::tmem_alloc_2sm(tslot, 512);
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tb = *tslot;
    const bool sparse = mode & 2, ts = mode & 1;
    uint32_t idesc = tc::idesc_i8(256, N, 0, 0) | (sparse ? (1u << 2) : 0u);
    unsigned long long t0 = 0, t1 = 0, g0 = 0, g1 = 0;
    // issuers: warp 0 (and warp 3 with mode & 4, on a second accumulator at
    // column 128; N <= 128 then).  mode & 16: the 16-MMA group is unrolled
    // with descriptors precomputed outside the loop.
    const int nissue = (mode & 4) ? 2 : 1;
    if ((warp == 0 || (warp == 3 && nissue == 2)) && rank == 0) {
        const int me = warp == 0 ? 0 : 1;
        uint64_t *gb = &bars[6 + 2 * me];
        const uint32_t dacc = (mode & 8192) ? tb : tb + 128 * me;   // 8192: both issuers on one accumulator
        const int my_iters = iters / nissue;
        if (sparse && me == 0) tcw::tmem_cp_128x128b_2sm(tb + 384, tc::smem_desc(tc::smem_u32(sm + SM_E), 2048, 128, 0));
        uint64_t bd[4], ad[4];
        const uint64_t ed = tc::smem_desc(tc::smem_u32(sm + SM_E), 2048, 128, 0);
        for (int ks = 0; ks < 4; ++ks) {
            bd[ks] = tc::smem_desc_sw128(tc::smem_u32(sm + SM_B) + (sparse ? 64 * (ks & 1) : 32 * ks), 16, 1024);
            if (mode & 16384) {    // four distinct A tiles (two 2:4 images) and B tiles (two 96-row stages)
                ad[ks] = tc::smem_desc(tc::smem_u32(sm + SM_A) + 8192 * (ks >> 1) + 256 * (ks & 1), 128, 512, 0);
                bd[ks] = tc::smem_desc_sw128(tc::smem_u32(sm + SM_B) + 12288 * (ks >> 1) + 64 * (ks & 1), 16, 1024);
            } else if (mode & 512)        // K3's 2:4 image: SWIZZLE_NONE core matrices, LBO 128, SBO 512
                ad[ks] = tc::smem_desc(tc::smem_u32(sm + SM_A) + 256 * (ks & 1), 128, 512, 0);
            else if (mode & 1024)  // SWIZZLE_64B K-major rows of 64 B
                ad[ks] = tc::smem_desc(tc::smem_u32(sm + SM_A) + 32 * (ks & 1), 16, 512, 4);
            else
                ad[ks] = tc::smem_desc_sw128(tc::smem_u32(sm + SM_A) + 32 * ks, 16, 1024);
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        t0 = clock64();
        if (mode & 16) {
            for (int g = 0; g < my_iters / 16; ++g) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int ks = j & 3;
                    if (mode & 32) tcw::tmem_cp_128x128b_2sm(tb + 384 + 4 * (j & 3), ed);
                    if ((mode & 64) && (j & 3) == 0) cp_256_2sm(tb + 384 + 8 * ((j >> 2) & 1), ed);
                    const uint32_t acc = (g | j) ? 1u : 0u;
                    const uint32_t dA = (mode & 256) ? dacc + 128 * (j & 1) : dacc;
                    if (!sparse) {
                        if (ts) mma_ts_i8_2sm(dA, tb + 256 + 8 * ks, bd[ks], idesc, acc);
                        else tcw::mma_i8_2sm(dA, ad[ks], bd[ks], idesc, acc);
                    } else {
                        if (ts) mma_sp_ts_i8_2sm(dA, tb + 256 + 8 * ks, bd[ks], tb + 384, idesc, acc);
                        else tcw::mma_sp_i8_2sm(dA, ad[ks], bd[ks], tb + 384 + ((mode & 32768) ? 4 * (j & 7) : 0), idesc, acc);
                    }
                    if ((mode & 128) && (j & 1)) tcw::mma_commit_2sm_mc(&bars[10], 0x3);
                }
                tcw::mma_commit_2sm_mc(&gb[g & 1], 0x3);
                if (g >= 1) tc::mbar_wait(&gb[(g - 1) & 1], ((g - 1) >> 1) & 1);
            }
        } else {
            for (int i = 0; i < my_iters; ++i) {
                const int ks = i & 3;
                if (!sparse) {
                    if (ts) mma_ts_i8_2sm(dacc, tb + 256 + 8 * ks, bd[ks], idesc, i > 0);
                    else tcw::mma_i8_2sm(dacc, ad[ks], bd[ks], idesc, i > 0);
                } else {
                    if (ts) mma_sp_ts_i8_2sm(dacc, tb + 256 + 8 * ks, bd[ks], tb + 384, idesc, i > 0);
                    else tcw::mma_sp_i8_2sm(dacc, ad[ks], bd[ks], tb + 384, idesc, i > 0);
                }
                if ((i & 15) == 15) {
                    const int g = i >> 4;
                    tcw::mma_commit_2sm_mc(&gb[g & 1], 0x3);
                    if (g >= 1) tc::mbar_wait(&gb[(g - 1) & 1], ((g - 1) >> 1) & 1);
                }
            }
        }
        const int glast = (my_iters >> 4) - 1;
        tc::mbar_wait(&gb[glast & 1], (glast >> 1) & 1);
        t1 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        if ((t & 31) == 0 && me == 0) {
            out[blockIdx.x * 4 + 0] = t1 - t0;
            out[blockIdx.x * 4 + 1] = g1 - g0;
        }
        __threadfence_block();
    }
    if ((mode & (2048 | 4096)) && warp >= 4 && warp < 12 && !((mode & 4096) && (warp & 3) == 1)) {
        // busy neighbours: dependent-chain-free FMA/ALU/SHFL mix, like an epilogue
        float a0 = threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
        uint32_t u = threadIdx.x;
        unsigned long long b0 = clock64();
        while (clock64() - b0 < (unsigned long long)ld_iters) {
#pragma unroll 16
            for (int i = 0; i < 64; ++i) {
                a0 = __fmaf_rn(a0, 1.0001f, 0.5f); a1 = __fmaf_rn(a1, 0.9999f, 0.25f);
                a2 = __fadd_rn(a2, a3); a3 = __fmul_rn(a3, 1.00001f);
                u = __byte_perm(u, (uint32_t)i, 0x3715) + __shfl_xor_sync(0xffffffffu, u, 1);
            }
        }
        if (a0 + a1 + a2 + a3 == 1.2345f && u == 7) out[0] = u;
    }
    if (warp >= 4 && warp < 4 + ldw) {
        // TMEM reader: this warp's lane quarter, 32 columns per load, cycling
        // over the first 256 columns
        const int q = warp & 3;
        uint32_t r[32], acc = 0;
        unsigned long long l0 = clock64();
        for (int i = 0; i < ld_iters; ++i) {
            tc::tmem_ld_32x32b_x32(tb + ((uint32_t)(q * 32) << 16) + 32 * (i & 7), r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += r[j];
        }
        unsigned long long l1 = clock64();
        if ((t & 31) == 0 && warp == 4) {
            out[blockIdx.x * 4 + 2] = (unsigned long long)ld_iters * 4096 * ldw;
            out[blockIdx.x * 4 + 3] = l1 - l0 + (acc == 0x12345678u);
        }
    }
    if (warp == 2 && stream > 0) {
        // ring producer: 16 KB bulk copies from an L2-resident source
        unsigned long long nbytes = 0, s0 = clock64();
        long c = (long)(blockIdx.x * 97) % gchunks;
        uint32_t j = 0;
        while (j < (uint32_t)stream) {
            const uint32_t slot = j % RING_N;
            if (j >= RING_N) tc::mbar_wait(&bars[2 + slot], ((j / RING_N) - 1) & 1);
            if ((t & 31) == 0) {
                tc::mbar_expect_tx(&bars[2 + slot], RING_SLOT);
                tc::bulk_load(sm + SM_RING + slot * RING_SLOT, gsrc + c * RING_SLOT, RING_SLOT, &bars[2 + slot]);
            }
            __syncwarp();
            c = (c + 1) % gchunks;
            ++j;
            nbytes += RING_SLOT;
        }
        for (uint32_t q = (j > RING_N ? j - RING_N : 0); q < j; ++q)
            tc::mbar_wait(&bars[2 + q % RING_N], (q / RING_N) & 1);
        unsigned long long s1 = clock64();
        if ((t & 31) == 0) {
            out[blockIdx.x * 4 + 2] = nbytes;
            out[blockIdx.x * 4 + 3] = s1 - s0;
        }
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) tc::tmem_dealloc_2sm(tb, 512);
}

extern "C" int mma_rate(int mode, int iters, int N, int stream, int ctas, const uint8_t *gsrc, long gchunks,
                        unsigned long long *out_host, float *ms, int ldw, int ld_iters)
{
    unsigned long long *dout;
    cudaMalloc(&dout, (size_t)ctas * 4 * sizeof(unsigned long long));
    cudaMemset(dout, 0, (size_t)ctas * 4 * sizeof(unsigned long long));
    cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES + 65536);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_rate_kernel<<<ctas, 384, SMEM_BYTES + 65536>>>(mode, iters, N, stream, gsrc, gchunks, dout, ldw, ld_iters);
    cudaEventRecord(e1);
    int err = (int)cudaDeviceSynchronize();
    if (err == 0) err = (int)cudaGetLastError();
    cudaEventElapsedTime(ms, e0, e1);
    cudaMemcpy(out_host, dout, (size_t)ctas * 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(dout);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return err;
}
