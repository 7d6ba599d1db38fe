// spmm_tc.cu -- K2: the tensor-core SpMM (tcgen05.mma kind::i8, TMA, TMEM).
//
// Replaces the same reference functions as K1 (_acc_group_panel +
// _spmm_task_*, spmm.py:192-280) for token counts where a 128-row weight
// tile against a 256-token activation tile is worth a tensor-core pass.
// The 4x1 blocks are expanded into dense 128 x K weight tiles (W^T, m
// contiguous, built once by the plan builder); X is read in its native
// orientation ([K, N] -> MN-major B operand, [N, K] -> K-major B operand),
// so no relayout pass exists.  Integer MACs are exact and wrap mod 2^32,
// so the expansion changes no bit of the accumulator.
//
// Structure (one persistent CTA per SM, warp-specialised):
//   warp 0      TMA producer: W^T chunk [128 m x 128 k] and X chunk
//               [256 n x 128 k] per stage, 4-stage mbarrier ring
//   warp 1      TMEM allocator + single-thread MMA issuer:
//               4 x tcgen05.mma.cta_group::1.kind::i8 M128 N256 K32 per stage
//   warps 2-9   epilogue: tcgen05.ld 32x32b -> registers -> fused epilogue ->
//               8-bit outputs: saturating pack, 4x4 quad byte transpose,
//               128B-swizzled smem tile, TMA store of [128 tokens x 128 m];
//               32-bit outputs: coalesced 128-byte row stores
// TMEM holds two 128 x 256 s32 accumulators (all 512 columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1.  Tiles are ordered
// m-fastest so the CTAs working on one token tile run together and share
// its X chunks through L2.
//
// Requant fast path (EPI_REQUANT, the BASELINE config-5 epilogue): no
// conversion instruction (those run on the quarter-rate XU pipe).  The
// accumulator becomes an f32 by the 1.5*2^23 magic-number trick (exact for
// |a| < 2^22), r = a * c[m] with c = f32(scale_in/fp), rint(r) by the same
// magic, and the exactness certificate |r - rint(r)| + 2^-20|r| < 1/2 is
// max-reduced over each 32-element chunk; a chunk that fails it (or has an
// out-of-range accumulator) recomputes the flagged elements with the
// reference's f64 expression (epilogue.py:218-228).  See epilogue.cuh for
// the error bound.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <mutex>

#include "epilogue.cuh"
#include "si_internal.h"
#include "tc_ptx.cuh"

namespace {

constexpr int BM = 128;     // weight rows per tile (MMA M)
constexpr int BN = 256;     // tokens per tile (MMA N)
constexpr int BK = 128;     // k per pipeline stage
constexpr int A_BYTES = BM * BK;           // 16 KB
constexpr int B_BYTES = BN * BK;           // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr int STG_HALF = 128 * 128;        // staging bytes per token half (8-bit outputs)
constexpr int TABLE_BYTES = 16 * 1024;    // breakpoint tables staged in smem (EPI_DEQ_TABLE)

// pipeline depth: 4 stages for the fast epilogues, 3 when the epilogue
// needs shared-memory tables (the L1 carve-out is otherwise ~2 KB)
template <int MODE>
constexpr int stages_for() { return (MODE == EPI_DEQ_TABLE || MODE == EPI_REQUANT_LUT || MODE == EPI_GENERIC) ? 3 : 4; }
template <int MODE, int OUTK>
constexpr int smem_bytes()
{
    return stages_for<MODE>() * STAGE_BYTES + ((OUTK == 1 || OUTK == 2) ? 2 * STG_HALF : 0) +
           (MODE == EPI_DEQ_TABLE ? TABLE_BYTES : 0) + 1024 + 256;
}

enum OutKind { OUT_32 = 0, OUT_U8_TMA = 1, OUT_S8_TMA = 2, OUT_8_DIRECT = 3 };

struct K2Params {
    int32_t mtiles, ntiles, kchunks;
    int32_t b_mn_major;  // 1: X is [K, N] (MN-major B), 0: [N, K] (K-major B)
    int64_t N;
    void *out;
    int64_t ldo;
    const float *rqc;    // requant c[m] = f32(scale_in[m] / fp)
};

constexpr float MAGIC_F = 12582912.0f;     // 1.5 * 2^23
constexpr int32_t MAGIC_I = 0x4B400000;

__device__ __noinline__ int32_t requant_exact(int32_t a, float s, float fp, int32_t zp, int32_t lo, int32_t hi)
{
    double y = __ddiv_rn(__dmul_rn((double)a, (double)s), (double)fp);
    double q = rint(y) + (double)zp;
    q = fmin(fmax(q, (double)lo), (double)hi);
    return (int32_t)q;
}

__device__ __noinline__ float deq_exact(int32_t a, float s) { return dev_deq_acc(a, s); }

// 4x4 byte transpose inside each quad of lanes: lane 4i+u holds word w = bytes
// (m = 4i+u; tokens 4w..4w+3) and gets (m = 4i..4i+3; token 4w+u).
__device__ __forceinline__ uint32_t quad_transpose(uint32_t w, uint32_t selA, uint32_t selB)
{
    uint32_t o = __shfl_xor_sync(0xffffffffu, w, 1);
    uint32_t x = __byte_perm(w, o, selA);
    uint32_t y = __shfl_xor_sync(0xffffffffu, x, 2);
    return __byte_perm(x, y, selB);
}

template <int MODE, int OUTK>
__global__ void __launch_bounds__(THREADS, 1)
k2_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
             const __grid_constant__ CUtensorMap tmap_o, const K2Params P, const EpiParams E)
{
    constexpr bool STAGED = (OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA);
    constexpr int STAGES = stages_for<MODE>();
    constexpr int SMEM_RING = STAGES * STAGE_BYTES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = tc::smem_u32(smem_raw);
    uint8_t *smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
    uint8_t *stage_base = smem;
    uint8_t *staging = smem + SMEM_RING;
    uint8_t *tables = smem + SMEM_RING + (STAGED ? 2 * STG_HALF : 0);
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + (MODE == EPI_DEQ_TABLE ? TABLE_BYTES : 0));
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int total_tiles = P.mtiles * P.ntiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], EPI_WARPS);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_w);
        tc::tma_prefetch_desc(&tmap_x);
        if (STAGED) tc::tma_prefetch_desc(&tmap_o);
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
                const int mt = tile % P.mtiles, nt = tile / P.mtiles;
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t *a_s = stage_base + stage * STAGE_BYTES;
                    uint8_t *b_s = a_s + A_BYTES;
                    tc::mbar_expect_tx(&full[stage], STAGE_BYTES);
                    tc::tma_load_2d(a_s, &tmap_w, &full[stage], mt * BM, kc * BK);
                    if (P.b_mn_major) {
                        tc::tma_load_2d(b_s, &tmap_x, &full[stage], nt * BN, kc * BK);
                        tc::tma_load_2d(b_s + B_BYTES / 2, &tmap_x, &full[stage], nt * BN + 128, kc * BK);
                    } else {
                        tc::tma_load_2d(b_s, &tmap_x, &full[stage], kc * BK, nt * BN);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (one thread)
            const uint32_t idesc = tc::idesc_i8(BM, BN, 1, P.b_mn_major ? 1 : 0);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_addr = tc::smem_u32(stage_base + stage * STAGE_BYTES);
                    const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk) {
                        const uint64_t adesc = tc::smem_desc_sw128(a_addr + kk * 4096, A_BYTES, 1024);
                        const uint64_t bdesc = P.b_mn_major
                                                   ? tc::smem_desc_sw128(b_addr + kk * 4096, B_BYTES / 2, 1024)
                                                   : tc::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
                        tc::mma_i8(d_tmem, adesc, bdesc, idesc, (kc | kk) ? 1u : 0u);
                    }
                    tc::mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else {
        // ---------------- epilogue warps
        const int q = warp & 3;             // TMEM lane quarter this warp may access (m sub-block)
        const int h = (warp - 2) >> 2;      // token half of the 256-token tile
        const int u = lane & 3, i4 = lane >> 2;
        const uint32_t selA = (u & 1) ? 0x3715u : 0x6240u;
        const uint32_t selB = (u & 2) ? 0x3276u : 0x5410u;
        uint8_t *stg = staging + h * STG_HALF;
        // breakpoint tables -> smem (keys | values | buckets)
        int32_t *s_key = reinterpret_cast<int32_t *>(tables);
        uint32_t *s_val = reinterpret_cast<uint32_t *>(tables + 4 * E.n_bp);
        uint16_t *s_bkt = reinterpret_cast<uint16_t *>(tables + 8 * E.n_bp + 4);
        if constexpr (MODE == EPI_DEQ_TABLE) {
            const int et = threadIdx.x - 64;
            for (int i = et; i < E.n_bp; i += 32 * EPI_WARPS) s_key[i] = __ldg(E.bp_key + i);
            for (int i = et; i <= E.n_bp; i += 32 * EPI_WARPS) s_val[i] = __ldg(E.bp_v + i);
            for (int i = et; i < E.bp_nbucket; i += 32 * EPI_WARPS) s_bkt[i] = __ldg(E.bp_bucket + i);
            tc::named_bar_sync(3, 32 * EPI_WARPS);
        }
        const bool leader = (q == ((2 + 4 * h) & 3)) && lane == 0;  // first warp of the half
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const int mt = tile % P.mtiles, nt = tile / P.mtiles;
            const int32_t m = mt * BM + q * 32 + lane;
            const bool mok = m < E.M;
            const int32_t adj = mok ? __ldg(E.adj + m) : 0;
            const float s_in = mok ? __ldg(E.scale_in + m) : 0.0f;
            float cq = 0.0f;
            if (MODE == EPI_REQUANT) cq = mok ? __ldg(P.rqc + m) : 0.0f;
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < 128 / 32; ++c) {
                const int col = h * 128 + c * 32;
                uint32_t r[32];
                tc::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + col, r);
                tc::tmem_ld_wait();
                const int64_t n0 = (int64_t)nt * BN + col;
                int32_t v[32];
                if constexpr (MODE == EPI_REQUANT) {
                    const int32_t adjM = (int32_t)((uint32_t)adj + (uint32_t)MAGIC_I);
                    const int32_t qoff = MAGIC_I - E.q_zp;
                    float emax = 0.0f;
                    uint32_t umax = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int32_t b = (int32_t)(r[j] + (uint32_t)adjM);
                        umax = max(umax, (uint32_t)(b - 0x4B000000));
                        const float af = __fsub_rn(__int_as_float(b), MAGIC_F);
                        const float rf = __fmul_rn(af, cq);
                        const float uu = __fadd_rn(rf, MAGIC_F);
                        const float d = __fsub_rn(rf, __fsub_rn(uu, MAGIC_F));
                        emax = fmaxf(emax, __fmaf_rn(fabsf(rf), 9.5367431640625e-07f, fabsf(d)));
                        v[j] = __float_as_int(uu) - qoff;
                    }
                    if (__any_sync(0xffffffffu, emax >= 0.5f || umax >= 0x800000u)) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int32_t a = (int32_t)(r[j] + (uint32_t)adj);
                            const int32_t b = (int32_t)((uint32_t)a + (uint32_t)MAGIC_I);
                            const float rf = __fmul_rn(__fsub_rn(__int_as_float(b), MAGIC_F), cq);
                            const float d = __fsub_rn(rf, __fsub_rn(__fadd_rn(rf, MAGIC_F), MAGIC_F));
                            const bool bad = ((uint32_t)(b - 0x4B000000) >= 0x800000u) ||
                                             !(__fmaf_rn(fabsf(rf), 9.5367431640625e-07f, fabsf(d)) < 0.5f);
                            if (bad && mok) v[j] = requant_exact(a, s_in, E.q_scale, E.q_zp, E.q_lo, E.q_hi);
                        }
                    }
                    if (OUTK == OUT_32 || OUTK == OUT_8_DIRECT) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = min(max(v[j], E.q_lo), E.q_hi);
                    }
                } else if constexpr (MODE == EPI_S32) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = (int32_t)(r[j] + (uint32_t)adj);
                } else if constexpr (MODE == EPI_DEQ_F32) {
                    const int32_t adjM = (int32_t)((uint32_t)adj + (uint32_t)MAGIC_I);
                    uint32_t umax = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int32_t b = (int32_t)(r[j] + (uint32_t)adjM);
                        umax = max(umax, (uint32_t)(b - 0x4B000000));
                        v[j] = __float_as_int(__fmul_rn(__fsub_rn(__int_as_float(b), MAGIC_F), s_in));
                    }
                    if (__any_sync(0xffffffffu, umax >= 0x800000u)) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int32_t a = (int32_t)(r[j] + (uint32_t)adj);
                            if ((uint32_t)(a + 0x400000) >= 0x800000u) v[j] = __float_as_int(deq_exact(a, s_in));
                        }
                    }
                } else if constexpr (MODE == EPI_DEQ_TABLE) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float x = dev_deq_acc((int32_t)(r[j] + (uint32_t)adj), s_in);
                        v[j] = (int32_t)bp_lookup_bucketed(x, s_key, s_bkt, s_val, E.n_bp, E.bp_key_lo, E.bp_shift,
                                                           E.bp_nbucket);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int64_t n = n0 + j;
                        v[j] = (mok && n < P.N)
                                   ? (int32_t)epi_apply<MODE>((int32_t)(r[j] + (uint32_t)adj), m, n, E)
                                   : 0;
                    }
                }

                if constexpr (OUTK == OUT_32) {
                    if (mok) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n0 + j < P.N) reinterpret_cast<int32_t *>(P.out)[(n0 + j) * P.ldo + m] = v[j];
                    }
                } else if constexpr (OUTK == OUT_8_DIRECT) {
                    if (mok) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n0 + j < P.N)
                                reinterpret_cast<uint8_t *>(P.out)[(n0 + j) * P.ldo + m] = (uint8_t)(v[j] & 0xFF);
                    }
                } else {
                    // saturating pack of 4 consecutive tokens, quad transpose to
                    // 4 consecutive m, swizzled STS into the [token][128 m] tile
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        uint32_t word;
                        if (OUTK == OUT_U8_TMA)
                            word = tc::pack_sat_u8(v[4 * w + 1], v[4 * w], tc::pack_sat_u8(v[4 * w + 3], v[4 * w + 2], 0));
                        else
                            word = tc::pack_sat_s8(v[4 * w + 1], v[4 * w], tc::pack_sat_s8(v[4 * w + 3], v[4 * w + 2], 0));
                        word = quad_transpose(word, selA, selB);
                        const int t = c * 32 + 4 * w + u;                // token row within the half
                        const int chunk = 2 * q + (i4 >> 2);              // 16B chunk of the 128B row
                        const int off = t * 128 + (((chunk ^ (t & 7)) << 4)) + 4 * (i4 & 3);
                        *reinterpret_cast<uint32_t *>(stg + off) = word;
                    }
                }
            }
            // this warp's TMEM reads are complete: release the accumulator
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            if constexpr (STAGED) {
                tc::fence_proxy_async_smem();
                tc::named_bar_sync(1 + h, 128);
                if (leader) {
                    tc::tma_store_2d(&tmap_o, stg, mt * BM, nt * BN + h * 128);
                    tc::tma_store_commit();
                    tc::tma_store_wait_read0();
                }
                tc::named_bar_sync(1 + h, 128);
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (STAGED && leader) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

// ---- host side ------------------------------------------------------------------
int g_num_sms = 0;
std::once_flag g_sms_once;

int num_sms()
{
    std::call_once(g_sms_once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    });
    return g_num_sms;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library does not link libcuda (it must load on GPU-less build hosts).
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

EncodeTiledFn encode_fn()
{
    std::call_once(g_encode_once, [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = reinterpret_cast<EncodeTiledFn>(fn);
    });
    return g_encode;
}

bool encode_2d(CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
               uint32_t box_inner, uint32_t box_outer)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {pitch_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(ptr), dims, strides,
                                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int MODE, int OUTK>
int launch_mode(const SpmmArgs &a, const CUtensorMap &tw, const CUtensorMap &tx, const CUtensorMap &to,
                const K2Params &p)
{
    auto kern = k2_tc_kernel<MODE, OUTK>;
    constexpr int smem = smem_bytes<MODE, OUTK>();
    static_assert(smem <= 232448, "shared memory budget");
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr_set = true;
    }
    EpiParams E = make_epi(a.h, a.img, a.sides, a.n);
    const int tiles = p.mtiles * p.ntiles;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    kern<<<grid, THREADS, smem, (cudaStream_t)a.stream>>>(tw, tx, to, p, E);
    return (int)cudaGetLastError();
}

template <int OUTK>
int launch_outk(const SpmmArgs &a, const CUtensorMap &tw, const CUtensorMap &tx, const CUtensorMap &to,
                const K2Params &p)
{
    switch (a.h->epi_mode) {
    case EPI_S32: return launch_mode<EPI_S32, OUTK>(a, tw, tx, to, p);
    case EPI_DEQ_F32: return launch_mode<EPI_DEQ_F32, OUTK>(a, tw, tx, to, p);
    case EPI_REQUANT: return launch_mode<EPI_REQUANT, OUTK>(a, tw, tx, to, p);
    case EPI_REQUANT_LUT: return launch_mode<EPI_REQUANT_LUT, OUTK>(a, tw, tx, to, p);
    case EPI_DEQ_TABLE: return launch_mode<EPI_DEQ_TABLE, OUTK>(a, tw, tx, to, p);
    default: return launch_mode<EPI_GENERIC, OUTK>(a, tw, tx, to, p);
    }
}

}  // namespace

bool k2_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx, int64_t)
{
    if (n < 1 || n > (int64_t)INT32_MAX - BN) return false;
    if (((uintptr_t)x) % 16) return false;
    if (ldx % 16) return false;
    if (layout == 1 && h->K % 16) return false;  // K-major rows: TMA inner extent granularity
    return h->tc_mtiles > 0;
}

uint64_t k2_workspace(const SiImage *, int64_t, int32_t) { return 0; }

int k2_launch_count(const SiImage *, int32_t) { return 1; }

int k2_launch(const SpmmArgs &a)
{
    const SiImage *h = a.h;
    CUtensorMap tw, tx, to;
    const void *wt = img_sec<uint8_t>(a.img, h->off_tc_wt);
    const uint64_t mpad = (uint64_t)h->tc_mtiles * 128;
    if (!encode_2d(&tw, wt, mpad, (uint64_t)h->tc_kpad, mpad, 128, BK)) return (int)cudaErrorInvalidValue;
    bool ok;
    if (a.layout == 0)
        ok = encode_2d(&tx, a.x, (uint64_t)a.n, (uint64_t)h->K, (uint64_t)a.ldx, 128, BK);
    else
        ok = encode_2d(&tx, a.x, (uint64_t)h->K, (uint64_t)a.n, (uint64_t)a.ldx, BK, BN);
    if (!ok) return (int)cudaErrorInvalidValue;
    K2Params p;
    p.mtiles = h->tc_mtiles;
    p.ntiles = (int32_t)((a.n + BN - 1) / BN);
    p.kchunks = h->tc_kpad / BK;
    p.b_mn_major = a.layout == 0 ? 1 : 0;
    p.N = a.n;
    p.out = a.out;
    p.ldo = a.ldo;
    p.rqc = img_sec<float>(a.img, h->off_rqc);
    const bool out32 = h->out_dtype == 0 || h->out_dtype == 3;
    if (out32) {
        std::memset(&to, 0, sizeof(to));
        return launch_outk<OUT_32>(a, tw, tx, to, p);
    }
    const bool tma_ok = (a.ldo % 16 == 0) && ((uintptr_t)a.out % 16 == 0) &&
                        encode_2d(&to, a.out, (uint64_t)h->M, (uint64_t)a.n, (uint64_t)a.ldo, 128, 128);
    if (!tma_ok) {
        std::memset(&to, 0, sizeof(to));
        return launch_outk<OUT_8_DIRECT>(a, tw, tx, to, p);
    }
    return h->out_dtype == 2 ? launch_outk<OUT_U8_TMA>(a, tw, tx, to, p) : launch_outk<OUT_S8_TMA>(a, tw, tx, to, p);
}
