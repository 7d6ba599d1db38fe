// atmem_probe.cu -- experiment harness (not part of the product library):
// pins down tcgen05.mma.kind::i8 with the A operand in tensor memory.  One
// CTA writes A [128 x 32] s8 into TMEM with tcgen05.st (lane = row m, 32-bit
// column c = bytes k = 4c..4c+3 in the order chosen by `order`), B [64 x 32]
// u8 is K-major SWIZZLE_NONE in smem, one M128 x N64 x K32 MMA runs and D is
// read back.  Built by tools/atmem_probe.py.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2306_16601_b200/csrc/tc_ptx.cuh"

namespace {
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void mma_i8_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
}  // namespace

// a: s8 [128][32] row-major; b_img: 2 KB smem image of B (N64 x K32 K-major,
// core matrices, LBO 128, SBO 256); out: int32 [128][64]
__global__ void atmem_kernel(const int8_t *a, const uint8_t *b_img, int32_t *out, int order)
{
    __shared__ __align__(1024) uint8_t sb[2048];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    for (int i = t; i < 2048; i += blockDim.x) sb[i] = b_img[i];
    if (t == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
    if (w == 0) tc::tmem_alloc(&tslot, 128);
    tc::fence_proxy_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tb = tslot;
    // A into TMEM columns [64, 72): lane = row
    {
        const int m = w * 32 + l;
        uint32_t v[8];
        for (int c = 0; c < 8; ++c) {
            uint32_t word = 0;
            for (int j = 0; j < 4; ++j) {
                const int k = order ? 4 * c + (3 - j) : 4 * c + j;
                word |= (uint32_t)(uint8_t)a[m * 32 + k] << (8 * j);
            }
            v[c] = word;
        }
        tmem_st_32x32b_x8(tb + ((uint32_t)(w * 32) << 16) + 64, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (t == 0) {
        const uint64_t bd = desc_none(tc::smem_u32(sb), 128, 256);
        const uint32_t idesc = tc::idesc_i8(128, 64, 0, 0);
        mma_i8_ta(tb, tb + 64, bd, idesc, 0);
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::tc_fence_after();
    uint32_t r[32];
    for (int half = 0; half < 2; ++half) {
        tc::tmem_ld_32x32b_x32(tb + ((uint32_t)(w * 32) << 16) + half * 32, r);
        tc::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[(w * 32 + l) * 64 + half * 32 + j] = (int32_t)r[j];
    }
    tc::tc_fence_before();
    __syncthreads();
    if (w == 0) tc::tmem_dealloc(tb, 128);
}

extern "C" int atmem_probe(const int8_t *a, const uint8_t *b, int32_t *out, int order)
{
    int8_t *da;
    uint8_t *db;
    int32_t *dout;
    cudaMalloc(&da, 4096);
    cudaMalloc(&db, 2048);
    cudaMalloc(&dout, 128 * 64 * 4);
    cudaMemcpy(da, a, 4096, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b, 2048, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, 128 * 64 * 4);
    atmem_kernel<<<1, 128>>>(da, db, dout, order);
    int err = (int)cudaDeviceSynchronize();
    cudaMemcpy(out, dout, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    cudaFree(da); cudaFree(db); cudaFree(dout);
    return err;
}
