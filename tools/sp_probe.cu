// sp_probe.cu -- experiment harness (not part of the product library):
// one CTA runs a single tcgen05.mma.sp.kind::i8 (M128 x N64 x K64) from
// operands laid out in smem by the host, to pin down the sparse A layout and
// the metadata (E) format in TMEM.  Built by tools/sp_probe.py with nvcc.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2306_16601_b200/csrc/tc_ptx.cuh"

namespace {
__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t sdesc)
{
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_sp_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t e, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%3], %4, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(e), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;  // layout type 0 = SWIZZLE_NONE
}
}  // namespace

// a_img: 4 KB smem image of A, b_img: 4 KB smem image of B (N64 x K64, K-major),
// e_img: 2 KB smem image of E; out: int32 [128][64]
// params: a_lbo, a_sbo, b_lbo, b_sbo, e_lbo, e_sbo, sparse_id2, e_col
__global__ void sp_probe_kernel(const uint8_t *a_img, const uint8_t *b_img, const uint8_t *e_img, int32_t *out,
                                const int *prm)
{
    __shared__ __align__(1024) uint8_t sa[4096];
    __shared__ __align__(1024) uint8_t sb[4096];
    __shared__ __align__(1024) uint8_t se[2048];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    for (int i = t; i < 4096; i += blockDim.x) { sa[i] = a_img[i]; sb[i] = b_img[i]; }
    for (int i = t; i < 2048; i += blockDim.x) se[i] = e_img[i];
    if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
    if ((t >> 5) == 0) tc::tmem_alloc(&tslot, 256);
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tb = tslot;
    if (t == 0) {
        const uint64_t ad = desc_none(tc::smem_u32(sa), prm[0], prm[1]);
        const uint64_t bd = desc_none(tc::smem_u32(sb), prm[2], prm[3]);
        const uint64_t ed = desc_none(tc::smem_u32(se), prm[4], prm[5]);
        const uint32_t ecol = tb + prm[7];
        tmem_cp_128x128b(ecol, ed);
        // kind::i8, A s8 (sparse), B u8, K-major both, M128 N64, sparse flag
        uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | (0u << 15) | (0u << 16) | ((64u >> 3) << 17) |
                         ((128u >> 4) << 24) | (1u << 2) | ((uint32_t)prm[6] & 3u);
        mma_sp_i8(tb, ad, bd, ecol, idesc, 0);
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::tc_fence_after();
    const int w = t >> 5, l = t & 31;
    uint32_t r[32];
    for (int half = 0; half < 2; ++half) {
        tc::tmem_ld_32x32b_x32(tb + ((uint32_t)(w * 32) << 16) + half * 32, r);
        tc::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[(w * 32 + l) * 64 + half * 32 + j] = (int32_t)r[j];
    }
    tc::tc_fence_before();
    __syncthreads();
    if ((t >> 5) == 0) tc::tmem_dealloc(tb, 256);
}

extern "C" int sp_probe(const uint8_t *a, const uint8_t *b, const uint8_t *e, int32_t *out, const int *prm)
{
    uint8_t *da, *db, *de;
    int32_t *dout;
    int *dp;
    cudaMalloc(&da, 4096);
    cudaMalloc(&db, 4096);
    cudaMalloc(&de, 2048);
    cudaMalloc(&dout, 128 * 64 * 4);
    cudaMalloc(&dp, 8 * sizeof(int));
    cudaMemcpy(da, a, 4096, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b, 4096, cudaMemcpyHostToDevice);
    cudaMemcpy(de, e, 2048, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, prm, 8 * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, 128 * 64 * 4);
    sp_probe_kernel<<<1, 128>>>(da, db, de, dout, dp);
    int err = (int)cudaDeviceSynchronize();
    cudaMemcpy(out, dout, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    cudaFree(da); cudaFree(db); cudaFree(de); cudaFree(dout); cudaFree(dp);
    return err;
}

// ---- pair probe: cluster of 2, tcgen05.cp/mma.sp with cta_group::2 (M256 x N64 x K64)
namespace {
__device__ __forceinline__ void tmem_cp_128x128b_2sm(uint32_t taddr, uint64_t sdesc)
{
    asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void mma_sp_i8_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t e, uint32_t idesc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.sp.cta_group::2.kind::i8 [%0], %1, %2, [%3], %4, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(e), "r"(idesc)
        : "memory");
}
}  // namespace

// a_img: [2][4096] A halves; b_img: [2][2048] B halves (32 tokens x K64 each);
// e_img: [2][2048]; out: int32 [256][64]
__global__ void __cluster_dims__(2, 1, 1) sp_probe_pair_kernel(const uint8_t *a_img, const uint8_t *b_img,
                                                               const uint8_t *e_img, int32_t *out, int bsbo)
{
    __shared__ __align__(1024) uint8_t sa[4096];
    __shared__ __align__(1024) uint8_t sb[2048];
    __shared__ __align__(1024) uint8_t se[2048];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    const uint32_t rank = tc::cluster_ctarank();
    for (int i = t; i < 4096; i += blockDim.x) sa[i] = a_img[rank * 4096 + i];
    for (int i = t; i < 2048; i += blockDim.x) { sb[i] = b_img[rank * 2048 + i]; se[i] = e_img[rank * 2048 + i]; }
    if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
    if ((t >> 5) == 0) tc::tmem_alloc_2sm(&tslot, 256);
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tb = tslot;
    if (t == 0 && rank == 0) {
        const uint64_t ad = desc_none(tc::smem_u32(sa), 128, 256);
        const uint64_t bd = desc_none(tc::smem_u32(sb), 128, bsbo);
        const uint64_t ed = desc_none(tc::smem_u32(se), 2048, 128);
        tmem_cp_128x128b_2sm(tb + 128, ed);
        uint32_t idesc = (2u << 4) | (1u << 7) | ((64u >> 3) << 17) | ((256u >> 4) << 24) | (1u << 2);
        mma_sp_i8_2sm(tb, ad, bd, tb + 128, idesc);
        tc::mma_commit_2sm_mc(&bar, 0x3);
    }
    tc::mbar_wait(&bar, 0);
    tc::tc_fence_after();
    const int w = t >> 5, l = t & 31;
    uint32_t r[32];
    for (int half = 0; half < 2; ++half) {
        tc::tmem_ld_32x32b_x32(tb + ((uint32_t)(w * 32) << 16) + half * 32, r);
        tc::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[(rank * 128 + w * 32 + l) * 64 + half * 32 + j] = (int32_t)r[j];
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if ((t >> 5) == 0) tc::tmem_dealloc_2sm(tb, 256);
}

extern "C" int sp_probe_pair(const uint8_t *a, const uint8_t *b, const uint8_t *e, int32_t *out, int bsbo)
{
    uint8_t *da, *db, *de;
    int32_t *dout;
    cudaMalloc(&da, 8192);
    cudaMalloc(&db, 4096);
    cudaMalloc(&de, 4096);
    cudaMalloc(&dout, 256 * 64 * 4);
    cudaMemcpy(da, a, 8192, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b, 4096, cudaMemcpyHostToDevice);
    cudaMemcpy(de, e, 4096, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, 256 * 64 * 4);
    sp_probe_pair_kernel<<<2, 128>>>(da, db, de, dout, bsbo);
    int err = (int)cudaDeviceSynchronize();
    cudaMemcpy(out, dout, 256 * 64 * 4, cudaMemcpyDeviceToHost);
    cudaFree(da); cudaFree(db); cudaFree(de); cudaFree(dout);
    return err;
}
