// spmm_tca.cu -- K2a: the weight-stationary tensor-core SpMM with W in TMEM.
//
// Same reference functions as K1/K2 (_acc_group_panel + _spmm_task_*,
// spmm.py:192-280).  The dense pair kernel (K2, spmm_tc.cu) streams both
// operands through shared memory: per CTA 128 W rows x 128 k and 128 tokens x
// 128 k per stage, 64 B/clk of operand reads plus 64 B/clk of TMA writes on
// the 128 B/clk shared-memory crossbar, and 2.15 GB of L2 -> SM traffic for
// BASELINE 5b.  K2a keeps the CTA pair's 256 W rows resident in *tensor
// memory* (tcgen05.mma with the A operand in TMEM: lane = row, 4 k-bytes per
// 32-bit column, pinned by tools/atmem_probe.py) and streams only X:
//
//   * TMEM per CTA: W rows (K/4 columns, K <= 1024) + two 128-token s32
//     accumulators (the epilogue of tile i overlaps the MMAs of tile i+1);
//   * the per-stage smem stream is the X half alone (64 tokens x 128 k = 8
//     KB per CTA), so the tensor pipe reads 32 B/clk of B from smem and the
//     TMA writes 32 B/clk;
//   * each pair walks a contiguous run of (row tile, token tile) work, row
//     tile major, so W is loaded into TMEM once or twice per pair and the
//     epilogue's per-row constants are fixed for the whole row tile.
//
// Roles (20 warps): warps 0, 18, 19 TMA producers (stage i on producer i mod
// 3), warp 1 TMEM allocator + MMA issuer (leader CTA, warp-converged,
// elect.sync issue), warps 2-17 the epilogue (4 token groups of 32 x 4 TMEM
// lane quarters), which also load W rows into TMEM (tcgen05.st) at a row-tile
// switch.
#include <cstdio>

#include "k2_common.cuh"

namespace {

constexpr int A_TN = 128;                       // tokens per accumulator tile (pair)
constexpr int A_TNH = 64;                       // tokens per CTA half
constexpr int A_EPI_WARPS = 16;
constexpr int A_NPROD = 3;                      // warp 0 + warps 18, 19 (20 warps keep the 96-register cap)
constexpr int A_THREADS = 32 * (2 + A_EPI_WARPS + A_NPROD - 1);
constexpr int A_KMAX = 1024;
constexpr int A_STAGE_MAX = A_TNH * 256;        // X half of one 256-k stage (16 KB)
constexpr int A_STG = 128 * 32;                 // 8-bit staging: 128 m x 32 tokens
constexpr uint32_t A_COL_A = 2 * A_TN;          // W rows start at TMEM column 256

template <int OUTK>
constexpr int a_staged() { return (OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) ? 2 * 4 * A_STG : 0; }
// KS: k per pipeline stage (256: one 16 KB box per CTA -- a TMA-issuing warp
// sustains about one box per ~340 ns whatever its size, tools/tma_bw.py prod;
// 128 for token-major X whose K is not a multiple of 128)
template <int MODE, int OUTK, int KS>
constexpr int a_stages()
{
    constexpr int s = (SMEM_MAX - a_staged<OUTK>() - table_bytes<MODE>() - 2048) / (A_TNH * KS);
    return s > 16 ? 16 : s;
}
template <int MODE, int OUTK, int KS>
constexpr int a_smem()
{
    return a_stages<MODE, OUTK, KS>() * (A_TNH * KS) + a_staged<OUTK>() + table_bytes<MODE>() + 1024 + 512;
}

struct AParams {
    const int8_t *wrow;   // dense W row-major [mtiles*256][kpad] (image off_tc_wrow)
    int32_t kpad;
    int32_t total;        // work tiles = mtiles * ntiles
};

__device__ __forceinline__ void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// M256 x N x K32 over the pair with A in TMEM (warp-converged, elected issue)
__device__ __forceinline__ void mma_i8_2sm_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accum)
{
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .b32 r;\n\t"
        "elect.sync r|p, 0xffffffff;\n\t"
        "setp.ne.b32 q, %4, 0;\n\t"
        "@p tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, q;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
}

struct RowConst {
    int32_t adj;
    float s_in, cq, gm;
    bool fast;
};

template <int MODE>
__device__ __forceinline__ RowConst row_const(int32_t m, const K2Params &P, const EpiParams &E)
{
    RowConst k;
    const bool mok = m < E.M;
    k.adj = mok ? __ldg(E.adj + m) : 0;
    k.s_in = mok ? __ldg(E.scale_in + m) : 0.0f;
    float cq = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqc + m) : 0.0f;
    const float cp = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqp + m) : 0.0f;
    const float gr = mok ? __ldg(P.rqg + m) : 1.0f;
    const bool proven = !(P.debug & 256) && __all_sync(0xffffffffu, gr >= 1.0f);
    const bool wide = __any_sync(0xffffffffu, gr >= 2.0f);
    k.fast = !(P.debug & 256) && !wide && __all_sync(0xffffffffu, gr >= 0.0f);
    k.gm = proven ? (wide ? 2.0f : 1.0f) : (gr >= 1.0f ? 0.0f : fmaxf(gr, 0.0f));
    k.cq = proven ? cp : cq;
    return k;
}

template <int MODE, int OUTK, bool MN, int KS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(A_THREADS, 1)
k2a_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_o, const K2Params P,
           const EpiParams E, const AParams A)
{
    constexpr int STAGES = a_stages<MODE, OUTK, KS>();
    constexpr int A_STAGE = A_TNH * KS;
    const int kstages = (A.kpad + KS - 1) / KS;
    constexpr bool STAGED = (OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA);
    static_assert(STAGES >= 4, "shared memory budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *ring = smem;                                  // [STAGES][64 tok x 128 k]
    uint8_t *staging = ring + STAGES * A_STAGE;            // [2 slots][4 groups][128 m x 32 tok]
    uint8_t *tables = staging + a_staged<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;                      // [2]
    uint64_t *tempty = tfull + 2;                          // [2] (leader)
    uint64_t *afull = tempty + 2;                          // (leader) both CTAs' W rows in TMEM
    uint64_t *aempty = afull + 1;                          // MMAs on the resident W rows retired
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(aempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    // this pair's contiguous run of work tiles t = mt * ntiles + nt (row tile
    // major: W is loaded into TMEM once or twice per pair).  Grouping pairs per
    // row tile so all row tiles walk the same token tiles together (X from L2)
    // measured slower (idle pairs; the X stream is not DRAM-bound).
    const int t0 = (int)(((int64_t)A.total * pair) / npairs), t1 = (int)(((int64_t)A.total * (pair + 1)) / npairs);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 2 * A_EPI_WARPS);
        }
        tc::mbar_init(afull, 2 * A_EPI_WARPS);
        tc::mbar_init(aempty, 1);
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_x);
    }
    if (warp == 1) tc::tmem_alloc_2sm(tmem_slot, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 || warp >= 2 + A_EPI_WARPS) {
        // ---------------- TMA producers (both CTAs, whole warp, elected issue): X halves
        const int prod = warp == 0 ? 0 : warp - (2 + A_EPI_WARPS) + 1;
        const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
        // X is re-read once per 256-row tile: keep it in L2 (evict_last) while
        // the outputs stream past it (evict_first, epilogue)
        const uint64_t keep = tc::policy_evict_last();
        int stage = 0, it = 0;
        uint32_t phase = 0;
        for (int t = t0; t < t1; ++t) {
            const int nt = t % P.ntiles;
            const int tok = nt * A_TN + A_TNH * (int)rank;
            for (int ks = 0; ks < kstages; ++ks, ++it) {
                if (it % A_NPROD == prod) {
                    tc::mbar_spin(&empty[stage], phase ^ 1);
                    if (rank == 0) tcw::mbar_expect_tx(&full[stage], 2 * A_STAGE);
                    if (MN)   // [K, N]: one {64 tokens, KS k} SWIZZLE_64B box
                        tcw::tma_load_2d_2sm_hint(ring + stage * A_STAGE, &tmap_x, full0 + 8 * stage, tok, ks * KS, keep);
                    else if (KS == 256)   // [N, K]: {128 k, 64 tokens, 2 k-blocks} -> two SW128 tiles
                        tcw::tma_load_3d_2sm_hint(ring + stage * A_STAGE, &tmap_x, full0 + 8 * stage, 0, tok, 2 * ks,
                                                  keep);
                    else
                        tcw::tma_load_2d_2sm_hint(ring + stage * A_STAGE, &tmap_x, full0 + 8 * stage, ks * KS, tok, keep);
                }
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ---------------- MMA issuer: leader CTA, whole warp, elected issue; M256 x N128 x K32, A in TMEM
            const uint32_t idesc = tc::idesc_i8(256, A_TN, 0, MN ? 1 : 0);
            int stage = 0, acc = 0, mt_cur = -1;
            uint32_t phase = 0, acc_phase = 0, aphase = 0;
            for (int t = t0; t < t1; ++t) {
                const int mt = t / P.ntiles;
                if (mt != mt_cur) {
                    if (mt_cur >= 0) tcw::mma_commit_2sm_mc(aempty, 0x3);   // old rows free once their MMAs retire
                    tc::mbar_spin_cluster(afull, aphase);
                    aphase ^= 1;
                    mt_cur = mt;
                }
                tc::mbar_spin(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * A_TN;
                for (int ks = 0; ks < kstages; ++ks) {
                    tc::mbar_spin(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t b_addr = tc::smem_u32(ring + stage * A_STAGE);
                    const int nk = min(KS, A.kpad - ks * KS) / 32;
#pragma unroll 8
                    for (int kk = 0; kk < nk; ++kk) {
                        // K-major: 32 k-bytes along the 128 B swizzle row, next 64-row
                        // tile every 128 k; MN-major SWIZZLE_64B: four 8-k core-matrix
                        // groups (512 B each) per 32 k
                        const uint64_t bdesc =
                            MN ? tc::smem_desc(b_addr + kk * 2048, 4096, 512, 4)
                               : tc::smem_desc_sw128(b_addr + (kk >> 2) * (A_TNH * 128) + (kk & 3) * 32, 16, 1024);
                        if (!(P.debug & 16))
                            mma_i8_2sm_ta(d_tmem, tmem_base + A_COL_A + ks * (KS / 4) + kk * 8, bdesc, idesc,
                                          (ks | kk) ? 1u : 0u);
                    }
                    tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tcw::mma_commit_2sm_mc(&tfull[acc], 0x3);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else {
        // ---------------- epilogue warps (both CTAs): W rows into TMEM at a row-tile
        // switch, then each accumulator tile's 32-token chunk of this warp's group
        EpiWarp W = make_epi_warp<MODE, A_EPI_WARPS>(warp, lane, staging, tables, E);
        const int g = W.g, q = W.q;
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        const uint32_t afull0 = tc::mapa(tc::smem_u32(afull), 0);
        const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
        const int gbytes = A.kpad / 4;                       // k-bytes of W this warp loads per row
        int acc = 0, slot = 0, mt_cur = -1;
        uint32_t acc_phase = 0, aphase = 0;
        RowConst k{};
        const uint64_t stream_out = tc::policy_evict_first();
        for (int t = t0; t < t1; ++t) {
            const int mt = t / P.ntiles, nt = t % P.ntiles;
            const int32_t row0 = mt * 256 + 128 * (int)rank;
            const int32_t m = row0 + q * 32 + lane;
            if (mt != mt_cur) {
                // the MMAs on the previous rows must have retired before they are overwritten
                tc::mbar_wait(aempty, aphase ^ 1);
                aphase ^= 1;
                tc::tc_fence_after();
                const int8_t *src = A.wrow + (int64_t)m * A.kpad + g * gbytes;
                for (int b = 0; b < gbytes; b += 32) {
                    const uint4 v0 = __ldg(reinterpret_cast<const uint4 *>(src + b));
                    const uint4 v1 = __ldg(reinterpret_cast<const uint4 *>(src + b) + 1);
                    const uint32_t v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                    tmem_st_32x32b_x8(lane_base + A_COL_A + (uint32_t)((g * gbytes + b) >> 2), v);
                }
                tmem_st_wait();
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_cluster(afull0);
                k = row_const<MODE>(m, P, E);
                mt_cur = mt;
            }
            // ---- epilogue of tile t (this warp: 32 rows x tokens [32g, 32g + 32))
            const int64_t tok0 = (int64_t)nt * A_TN;
            tc::mbar_wait(&tfull[acc], acc_phase);
            tc::tc_fence_after();
            uint8_t *const stg0 = W.stg;
            if constexpr (STAGED) {
                if (q == 2 && lane == 0) tc::tma_store_wait_read1();
                tc::named_bar_sync(1 + g, 128);
                W.stg = staging + slot * (4 * A_STG) + g * A_STG;
            }
            // token order inside the accumulator: columns [0, 64) are CTA 0's
            // 64 tokens, [64, 128) CTA 1's (the pair MMA's N halves)
            const int64_t n0 = tok0 + (g >> 1) * A_TNH + (g & 1) * 32;
            // the accumulator is released as soon as this warp's chunk is in
            // registers: with 128-token tiles the MMAs of a tile take ~1 us, so
            // the math and stores must not sit on the accumulator's critical path
            const uint32_t te = tempty0 + 8 * acc;
            auto release = [te, lane]() {
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_cluster(te);
            };
            if (!(P.debug & 1))
                epi_chunk<MODE, OUTK, false>(lane_base + acc * A_TN + g * 32, m, m < E.M, k.adj, k.s_in, k.cq, k.gm,
                                             k.fast, n0, 0, P, E, W, 0, 0, release);
            else
                release();
            if constexpr (STAGED) {
                tc::fence_proxy_async_smem();
                tc::named_bar_sync(1 + g, 128);
                if (q == 2 && lane == 0 && !(P.debug & 8192)) {
                    tc::tma_store_2d_hint(&tmap_o, W.stg, row0, (int32_t)n0, stream_out);
                    tc::tma_store_commit();
                }
                slot ^= 1;
            }
            W.stg = stg0;
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (STAGED && q == 2 && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(tmem_base, 512);
    }
}

template <int MODE, int OUTK, bool MN, int KS>
void k2a_go(const SpmmArgs &a, const CUtensorMap &tx, const CUtensorMap &to, const K2Params &p, const EpiParams &E,
            const AParams &A, int pairs)
{
    auto kern = k2a_kernel<MODE, OUTK, MN, KS>;
    constexpr int smem = a_smem<MODE, OUTK, KS>();
    static_assert(smem <= SMEM_MAX, "shared memory budget");
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); attr = true; }
    kern<<<2 * pairs, A_THREADS, smem, (cudaStream_t)a.stream>>>(tx, to, p, E, A);
}

template <int MODE, int OUTK>
int k2a_launch_mode(const SpmmArgs &a, const CUtensorMap &tx, const CUtensorMap &to, const K2Params &p,
                    const AParams &A)
{
    EpiParams E = make_epi(a.h, a.img, a.sides, a.n);
    const int npairs = num_sms() / 2;
    const int pairs = A.total < npairs ? A.total : npairs;
    if (a.layout == 0) k2a_go<MODE, OUTK, true, 256>(a, tx, to, p, E, A, pairs);
    else if (a.h->K % 128 == 0) k2a_go<MODE, OUTK, false, 256>(a, tx, to, p, E, A, pairs);
    else k2a_go<MODE, OUTK, false, 128>(a, tx, to, p, E, A, pairs);
    return (int)cudaGetLastError();
}

template <int OUTK>
int k2a_launch_outk(const SpmmArgs &a, const CUtensorMap &tx, const CUtensorMap &to, const K2Params &p,
                    const AParams &A)
{
    switch (a.h->epi_mode) {
    case EPI_S32: return k2a_launch_mode<EPI_S32, OUTK>(a, tx, to, p, A);
    case EPI_DEQ_F32: return k2a_launch_mode<EPI_DEQ_F32, OUTK>(a, tx, to, p, A);
    case EPI_REQUANT: return k2a_launch_mode<EPI_REQUANT, OUTK>(a, tx, to, p, A);
    case EPI_REQUANT_LUT: return k2a_launch_mode<EPI_REQUANT_LUT, OUTK>(a, tx, to, p, A);
    case EPI_DEQ_TABLE: return k2a_launch_mode<EPI_DEQ_TABLE, OUTK>(a, tx, to, p, A);
    default: return k2a_launch_mode<EPI_GENERIC, OUTK>(a, tx, to, p, A);
    }
}

}  // namespace

bool k2a_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx)
{
    if (h->tc_kpad > A_KMAX || h->tc_mtiles < 2) return false;
    if (n < 1 || n > (int64_t)INT32_MAX - A_TN) return false;
    if (((uintptr_t)x) % 16 || ldx % 16) return false;
    if (layout == 1 && h->K % 16) return false;
    return true;
}

int k2a_launch(const SpmmArgs &a)
{
    const SiImage *h = a.h;
    static const int dbg = env_int("SI_K2_DEBUG", 0);
    CUtensorMap tx, to;
    bool ok = a.layout == 0   ? encode_2d(&tx, a.x, (uint64_t)a.n, (uint64_t)h->K, (uint64_t)a.ldx, A_TNH, 256,
                                            CU_TENSOR_MAP_SWIZZLE_64B)
              : h->K % 128 == 0 ? encode_3d_kblocks(&tx, a.x, (uint64_t)a.n, (uint64_t)h->K, (uint64_t)a.ldx, A_TNH, 2)
                                : encode_2d(&tx, a.x, (uint64_t)h->K, (uint64_t)a.n, (uint64_t)a.ldx, 128, A_TNH);
    if (!ok) return (int)cudaErrorInvalidValue;
    K2Params p;
    std::memset(&p, 0, sizeof(p));
    p.mtiles = (h->tc_mtiles + 1) / 2;
    p.ntiles = (int32_t)((a.n + A_TN - 1) / A_TN);
    p.kchunks = h->tc_kpad / 128;
    p.b_mn_major = a.layout == 0 ? 1 : 0;
    p.mgroups = 1;
    p.N = a.n;
    p.out = a.out;
    p.ldo = a.ldo;
    p.rqc = img_sec<float>(a.img, h->off_rqc);
    p.rqg = img_sec<float>(a.img, h->off_rqg);
    p.rqp = img_sec<float>(a.img, h->off_rqp);
    p.debug = dbg;
    AParams A;
    A.wrow = img_sec<int8_t>(a.img, h->off_tc_wrow);
    A.kpad = h->tc_kpad;
    A.total = p.mtiles * p.ntiles;
    const bool out32 = h->out_dtype == 0 || h->out_dtype == 3;
    if (out32) {
        std::memset(&to, 0, sizeof(to));
        return k2a_launch_outk<OUT_32>(a, tx, to, p, A);
    }
    const bool tma_ok = (a.ldo % 16 == 0) && ((uintptr_t)a.out % 16 == 0) &&
                        encode_2d(&to, a.out, (uint64_t)h->M, (uint64_t)a.n, (uint64_t)a.ldo, 128, 32);
    if (!tma_ok) {
        std::memset(&to, 0, sizeof(to));
        return k2a_launch_outk<OUT_8_DIRECT>(a, tx, to, p, A);
    }
    return h->out_dtype == 2 ? k2a_launch_outk<OUT_U8_TMA>(a, tx, to, p, A)
                             : k2a_launch_outk<OUT_S8_TMA>(a, tx, to, p, A);
}
