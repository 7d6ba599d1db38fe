// spmm_tc.cu -- K2: the dense-expanded tensor-core SpMM (tcgen05.mma kind::i8, TMA, TMEM).
//
// Replaces the same reference functions as K1 (_acc_group_panel +
// _spmm_task_*, spmm.py:192-280) for token counts where tensor-core tiles
// pay and the 2:4 kernel (K3, spmm_xs.cu) does not apply: [K, N]
// activations, K > 1024, or a single 128-row weight tile.  The 4x1 blocks
// are expanded into dense weight tiles (W^T, m contiguous, built once by the
// plan builder); X is read in its native orientation ([K, N] -> MN-major B
// operand, [N, K] -> K-major B operand), so no relayout pass exists.  Integer
// MACs are exact and wrap mod 2^32, so the expansion changes no bit of the
// accumulator.
//
//  k2   single CTA, M128 x N256 tiles, both operands streamed through a TMA
//       ring (weights of one 128-row tile).
//  k2p  a CTA *pair* (cluster of 2, tcgen05 cta_group::2) computing
//       D[256 W rows x 256 tokens] per tile with 256-k stages; each CTA holds
//       half of A and half of B, so every SM moves half the operand bytes.
//
// Every single-thread role waits with mbarrier.try_wait (the hardware
// suspends the warp) rather than a test_wait polling loop: the kernel is
// power-limited (profiles/r02_k2_experiments.md), and the polling warps cost
// 0.3-0.5% of every config-5 linear.
//
// Roles: warp 0 and warps 18-19 TMA producers, warp 1 TMEM allocator + MMA
// issuer (one elected lane; in a pair only the leader CTA issues), warps
// 2-17 the epilogue (4 per TMEM lane quarter, 64 tokens each).  TMEM holds
// two accumulators so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// Epilogue (all compiled forms of the reference's _run_chain,
// epilogue.py:207-249; k2_common.cuh): tcgen05.ld 32x32b.x32 -> registers ->
// the form's math -> 8-bit outputs: saturating pack, 4x4 quad byte
// transpose, a per-warp [32 tokens][32 m] smem tile, one TMA store per warp
// and chunk; 32-bit outputs: coalesced 128-byte rows.  The requant form (BASELINE config 5) uses the plan's proven
// per-row multipliers (one fma onto the magic number 1.5*2^23 + zp) or the
// f32 certificate path with an exact f64 fallback (k2_common.cuh epi_chunk).
#include "k2_common.cuh"

namespace {

// ================================================================ single CTA
constexpr int S_BM = 128;
constexpr int S_A = S_BM * BK;       // 16 KB
constexpr int S_B = TILE_N * BK;     // 32 KB
constexpr int S_STAGE = S_A + S_B;

template <int MODE, int OUTK>
constexpr int single_stages()
{
    return (SMEM_MAX - 2048 - staged_bytes<OUTK>() - table_bytes<MODE>()) / S_STAGE > 4
               ? 4
               : (SMEM_MAX - 2048 - staged_bytes<OUTK>() - table_bytes<MODE>()) / S_STAGE;
}
template <int MODE, int OUTK>
constexpr int single_smem()
{
    return single_stages<MODE, OUTK>() * S_STAGE + staged_bytes<OUTK>() + table_bytes<MODE>() + 1024 + 512;
}

template <int MODE, int OUTK>
__global__ void __launch_bounds__(MT_THREADS, 1)
k2_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
             const __grid_constant__ CUtensorMap tmap_o, const K2Params P, const EpiParams E)
{
    constexpr int STAGES = single_stages<MODE, OUTK>();
    constexpr int RING = STAGES * S_STAGE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *staging = smem + RING;
    uint8_t *tables = staging + staged_bytes<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
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
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    tc::pdl_wait();                 // X may come from the previous kernel
    tc::pdl_launch_dependents();

    const int prod = producer_index(warp, 2 + EPI_WARPS);
    // (a producer must never run more than one ring round ahead of the
    // slot it waits on: parity waits cannot tell rounds r-1 and r-3 apart)
    const int nprod = NPROD < STAGES ? NPROD : STAGES;
    if (prod >= 0) {
        if (lane == 0) {
            int stage = 0, it = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
                const int mt = tile % P.mtiles, nt = tile / P.mtiles;
                for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                    if (it % nprod != prod) {
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    tc::mbar_wait(&empty[stage], phase ^ 1);   // (try_wait: no polling traffic on the shared-memory pipe)
                    uint8_t *a_s = smem + stage * S_STAGE;
                    uint8_t *b_s = a_s + S_A;
                    tc::mbar_expect_tx(&full[stage], S_STAGE);
                    tc::tma_load_2d(a_s, &tmap_w, &full[stage], mt * S_BM, kc * BK);
                    if (P.b_mn_major) {
                        tc::tma_load_2d(b_s, &tmap_x, &full[stage], nt * TILE_N, kc * BK);
                        tc::tma_load_2d(b_s + S_B / 2, &tmap_x, &full[stage], nt * TILE_N + 128, kc * BK);
                    } else {
                        tc::tma_load_2d(b_s, &tmap_x, &full[stage], kc * BK, nt * TILE_N);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_i8(S_BM, TILE_N, 1, P.b_mn_major ? 1 : 0);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * TILE_N;
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_addr = tc::smem_u32(smem + stage * S_STAGE);
                    const uint32_t b_addr = a_addr + S_A;
#pragma unroll
                    for (int kk = 0; kk < BK / 32; ++kk) {
                        const uint64_t adesc = tc::smem_desc_sw128(a_addr + kk * 4096, S_A, 1024);
                        const uint64_t bdesc = P.b_mn_major ? tc::smem_desc_sw128(b_addr + kk * 4096, S_B / 2, 1024)
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
    } else if (warp < 2 + EPI_WARPS) {
        const EpiWarp W = make_epi_warp<MODE>(warp, lane, staging, tables, E);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const int mt = tile % P.mtiles, nt = tile / P.mtiles;
            uint64_t *te = &tempty[acc];
            uint64_t *tf = &tfull[acc];
            const uint32_t ph = acc_phase;
            epi_tile<MODE, OUTK>(tmem_base, acc * TILE_N, mt * S_BM, (int64_t)nt * TILE_N, &tmap_o, P, E, W,
                                 [tf, ph] { tc::mbar_wait(tf, ph); }, [te] { tc::mbar_arrive(te); });
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if ((OUTK == OUT_U8_W || OUTK == OUT_S8_W) && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

// ================================================================ CTA pair
// Per CTA and BKS-k stage: A half = 128 W rows x BKS k, B half = 128 tokens x
// BKS k.  BKS = 256 (32 KB + 32 KB per stage: fewest barriers per byte, the
// large-N default) or 128 (twice the stages in the same shared memory: a work
// unit of few k chunks no longer fills the whole ring, so the next unit's
// loads overlap this one's MMAs -- the small-N variant).
template <int BKS>
struct PairGeom {
    static constexpr int A = 128 * BKS;
    static constexpr int B = 128 * BKS;
    static constexpr int SLOT = A + B;
};

template <int MODE, int OUTK, int BKS>
constexpr int pair_stages()
{
    constexpr int s = (SMEM_MAX - staged_bytes<OUTK>() - table_bytes<MODE>() - 2048) / PairGeom<BKS>::SLOT;
    return s > 8 ? 8 : s;
}
template <int MODE, int OUTK, int BKS>
constexpr int pair_smem()
{
    return pair_stages<MODE, OUTK, BKS>() * PairGeom<BKS>::SLOT + staged_bytes<OUTK>() + table_bytes<MODE>() + 1024 + 512;
}

template <int MODE, int OUTK, int BKS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(MT_THREADS, 1)
k2p_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
           const __grid_constant__ CUtensorMap tmap_o, const K2Params P, const EpiParams E)
{
    constexpr int STAGES = pair_stages<MODE, OUTK, BKS>();
    constexpr int P_A = PairGeom<BKS>::A, P_B = PairGeom<BKS>::B, P_SLOT = PairGeom<BKS>::SLOT;
    static_assert(STAGES >= 2, "shared memory budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *ring = smem;
    uint8_t *staging = ring + STAGES * P_SLOT;
    uint8_t *tables = staging + staged_bytes<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int units = P.ntiles * P.mtiles;   // (token tile, pair tile), pair tile fastest

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 2 * EPI_WARPS);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_w);
        tc::tma_prefetch_desc(&tmap_x);
    }
    if (warp == 1) tc::tmem_alloc_2sm(tmem_slot, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    tc::pdl_wait();                 // X may come from the previous kernel
    tc::pdl_launch_dependents();

    const int prod = producer_index(warp, 2 + EPI_WARPS);
    // (a producer must never run more than one ring round ahead of the
    // slot it waits on: parity waits cannot tell rounds r-1 and r-3 apart)
    const int nprod = NPROD < STAGES ? NPROD : STAGES;
    if (prod >= 0) {
        // ---------------- TMA producers (both CTAs; bytes land on the leader's
        // barriers), whole warp, one elected lane issues (tcw::)
        if (prod < nprod) {
            const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
            int stage = 0, it = 0;
            uint32_t phase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                const int nt = unit / P.mtiles, mt = unit % P.mtiles;
                const int tok = nt * TILE_N + 128 * (int)rank;
                for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                    if (it % nprod != prod) {
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    tc::mbar_wait(&empty[stage], phase ^ 1);   // (try_wait: no polling traffic on the shared-memory pipe)
                    uint8_t *a_s = ring + stage * P_SLOT;
                    const uint32_t fb = full0 + 8 * stage;
                    if (rank == 0) tcw::mbar_expect_tx(&full[stage], 2 * P_SLOT);
                    tcw::tma_load_2d_2sm(a_s, &tmap_w, fb, mt * 256 + 128 * (int)rank, kc * BKS);
                    if (P.b_mn_major)
                        tcw::tma_load_2d_2sm(a_s + P_A, &tmap_x, fb, tok, kc * BKS);
                    else
                        // token-major X: K-major boxes span at most 128 k (one
                        // SWIZZLE_128B row), so a 256-k stage is two stacked tiles
                        for (int h = 0; h < BKS / BK; ++h)
                            tcw::tma_load_2d_2sm(a_s + P_A + h * (128 * BK), &tmap_x, fb, kc * BKS + h * BK, tok);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ---------------- MMA issuer: leader CTA, whole warp, one elected lane issues, M256 x N256 x K32
            const uint32_t idesc = tc::idesc_i8(256, TILE_N, 1, P.b_mn_major ? 1 : 0);
            const uint32_t ring_u = tc::smem_u32(ring);
            const uint64_t adesc0 = tc::smem_desc_sw128(ring_u, P_A, 1024);
            const uint64_t bdesc0 = P.b_mn_major ? tc::smem_desc_sw128(ring_u + P_A, P_B, 1024)
                                                 : tc::smem_desc_sw128(ring_u + P_A, 16, 1024);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * TILE_N;
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint64_t so = (uint64_t)((stage * P_SLOT) >> 4);
#ifdef SI_EXPERIMENTS
                    if (P.exp & 2) {
                    } else
#endif
                    if (P.b_mn_major) {
#pragma unroll
                        for (int kk = 0; kk < BKS / 32; ++kk)
                            tcw::mma_i8_2sm(d_tmem, adesc0 + so + kk * 256, bdesc0 + so + kk * 256, idesc,
                                            (kc | kk) ? 1u : 0u);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < BKS / 32; ++kk)
                            tcw::mma_i8_2sm(d_tmem, adesc0 + so + kk * 256,
                                            bdesc0 + so + (kk >> 2) * (128 * BK / 16) + (kk & 3) * 2, idesc,
                                            (kc | kk) ? 1u : 0u);
                    }
                    tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tcw::mma_commit_2sm_mc(&tfull[acc], 0x3);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp < 2 + EPI_WARPS) {
        // ---------------- epilogue warps (both CTAs; each reads its own TMEM half)
        const EpiWarp W = make_epi_warp<MODE>(warp, lane, staging, tables, E);
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            const int nt = unit / P.mtiles, mt = unit % P.mtiles;
            const uint32_t te = tempty0 + 8 * acc;
            uint64_t *tf = &tfull[acc];
            const uint32_t ph = acc_phase;
            epi_tile<MODE, OUTK>(tmem_base, acc * TILE_N, mt * 256 + 128 * (int)rank, (int64_t)nt * TILE_N, &tmap_o,
                                 P, E, W, [tf, ph] { tc::mbar_wait(tf, ph); }, [te] { tc::mbar_arrive_cluster(te); });
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if ((OUTK == OUT_U8_W || OUTK == OUT_S8_W) && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(tmem_base, 512);
    }
}

template <int MODE, int OUTK>
int launch_mode(const SpmmArgs &a, const CUtensorMap &tw, const CUtensorMap &tx, const CUtensorMap &to, K2Params p,
                bool single)
{
    EpiParams E = make_epi(a.h, a.img, a.sides, a.n);
    cudaStream_t st = (cudaStream_t)a.stream;
    const int sms = num_sms();
    if (single) {
        auto kern = k2_tc_kernel<MODE, OUTK>;
        constexpr int smem = single_smem<MODE, OUTK>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        set_smem_attr(kern, smem);
        const int tiles = p.mtiles * p.ntiles;
        return (int)launch_pdl(kern, dim3(tiles < sms ? tiles : sms), dim3(MT_THREADS), smem, st, tw, tx, to, p, E);
    } else if (p.bks == 128) {
        auto kern = k2p_kernel<MODE, OUTK, 128>;
        constexpr int smem = pair_smem<MODE, OUTK, 128>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        set_smem_attr(kern, smem);
        const int units = p.mtiles * p.ntiles;
        const int pairs = units < sms / 2 ? units : sms / 2;
        return (int)launch_pdl(kern, dim3(2 * pairs), dim3(MT_THREADS), smem, st, tw, tx, to, p, E);
    } else {
        auto kern = k2p_kernel<MODE, OUTK, 256>;
        constexpr int smem = pair_smem<MODE, OUTK, 256>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        set_smem_attr(kern, smem);
        const int units = p.mtiles * p.ntiles;
        const int pairs = units < sms / 2 ? units : sms / 2;
        return (int)launch_pdl(kern, dim3(2 * pairs), dim3(MT_THREADS), smem, st, tw, tx, to, p, E);
    }
    return (int)cudaGetLastError();
}

template <int OUTK>
int launch_outk(const SpmmArgs &a, const CUtensorMap &tw, const CUtensorMap &tx, const CUtensorMap &to,
                const K2Params &p, bool single)
{
    switch (a.h->epi_mode) {
    case EPI_S32: return launch_mode<EPI_S32, OUTK>(a, tw, tx, to, p, single);
    case EPI_DEQ_F32: return launch_mode<EPI_DEQ_F32, OUTK>(a, tw, tx, to, p, single);
    case EPI_REQUANT: return launch_mode<EPI_REQUANT, OUTK>(a, tw, tx, to, p, single);
    case EPI_REQUANT_LUT: return launch_mode<EPI_REQUANT_LUT, OUTK>(a, tw, tx, to, p, single);
    case EPI_DEQ_TABLE: return launch_mode<EPI_DEQ_TABLE, OUTK>(a, tw, tx, to, p, single);
    case EPI_DEQ_SIDE: return launch_mode<EPI_DEQ_SIDE, OUTK>(a, tw, tx, to, p, single);
    default: return launch_mode<EPI_GENERIC, OUTK>(a, tw, tx, to, p, single);
    }
}

}  // namespace

bool k2_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx, int64_t)
{
    if (n < 1 || n > (int64_t)INT32_MAX - TILE_N) return false;
    if (((uintptr_t)x) % 16) return false;
    if (ldx % 16) return false;
    if (layout == SI_ACT_NK && h->K % 16) return false;  // K-major rows: TMA inner extent granularity
    return h->tc_mtiles > 0;
}

uint64_t k2_workspace(const SiImage *, int64_t, int32_t) { return 0; }

int k2_launch_count(const SiImage *, int32_t) { return 1; }

int k2_launch(const SpmmArgs &a)
{
    const SiImage *h = a.h;
    // the pair tiles W rows by 256 (an odd count of 128-row tiles reads one
    // tile of TMA out-of-bounds zero fill); a single 128-row tile takes the
    // one-CTA kernel
    const bool single = h->tc_mtiles <= 1;
    CUtensorMap tw, tx, to;
    const void *wt = img_sec<uint8_t>(a.img, h->off_tc_wt);
    const uint64_t mpad = (uint64_t)h->tc_mtiles * 128;
    // pair kernel: 256-k stages, or 128-k stages when a pair gets only a few
    // work units (the ring then holds more than one unit's k chunks, so the
    // next unit's loads overlap this one's MMAs)
    const int32_t ntiles = (int32_t)((a.n + TILE_N - 1) / TILE_N);
    const long pair_units = (long)((h->tc_mtiles + 1) / 2) * ntiles;
    uint32_t bks = single ? BK : (pair_units <= 6L * (num_sms() / 2) ? 128 : 256);
#ifdef SI_EXPERIMENTS
    if (!single)
        if (const char *e = getenv("SI_K2_BKS")) bks = (uint32_t)atoi(e) == 128 ? 128 : 256;
#endif
    bool ok = encode_2d(&tw, wt, mpad, (uint64_t)h->tc_kpad, mpad, 128, bks);
    if (a.layout == SI_ACT_KN)
        ok = ok && encode_2d(&tx, a.x, (uint64_t)a.n, (uint64_t)h->K, (uint64_t)a.ldx, 128, bks);
    else
        ok = ok && encode_2d(&tx, a.x, (uint64_t)h->K, (uint64_t)a.n, (uint64_t)a.ldx, BK, single ? TILE_N : 128);
    if (!ok) return (int)cudaErrorInvalidValue;
    K2Params p;
    std::memset(&p, 0, sizeof(p));
    p.mtiles = single ? h->tc_mtiles : (h->tc_mtiles + 1) / 2;
    p.ntiles = ntiles;
    p.kchunks = single ? h->tc_kpad / BK : (h->tc_kpad + (int)bks - 1) / (int)bks;
    p.bks = (int32_t)bks;
#ifdef SI_EXPERIMENTS
    if (const char *e = getenv("SI_K2_EXP")) p.exp = atoi(e);
#endif
    p.b_mn_major = a.layout == SI_ACT_KN ? 1 : 0;
    p.N = a.n;
    p.out = a.out;
    p.ldo = a.ldo;
    p.rqc = img_sec<float>(a.img, h->off_rqc);
    p.rqg = img_sec<float>(a.img, h->off_rqg);
    p.rqp = img_sec<float>(a.img, h->off_rqp);
    if (h->out_dtype == SI_F32 || h->out_dtype == SI_S32) {
        std::memset(&to, 0, sizeof(to));
        return launch_outk<OUT_32>(a, tw, tx, to, p, single);
    }
    // 8-bit outputs: every epilogue warp stages its own [32 tokens][32 m]
    // chunk and TMA-stores it as a 32 x 32 box (no cross-warp barrier on the
    // output path: 1-4% faster than one swizzled 128-row tile per column
    // group, profiles/r02_k2_experiments.md)
    const bool tma_ok = (a.ldo % 16 == 0) && ((uintptr_t)a.out % 16 == 0) &&
                        encode_2d(&to, a.out, (uint64_t)h->M, (uint64_t)a.n, (uint64_t)a.ldo, 32, 32,
                                  CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!tma_ok) {
        std::memset(&to, 0, sizeof(to));
        return launch_outk<OUT_8_DIRECT>(a, tw, tx, to, p, single);
    }
    return h->out_dtype == SI_U8 ? launch_outk<OUT_U8_W>(a, tw, tx, to, p, single)
                                 : launch_outk<OUT_S8_W>(a, tw, tx, to, p, single);
}
