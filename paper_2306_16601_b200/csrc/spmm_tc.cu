// spmm_tc.cu -- K2: the tensor-core SpMM (tcgen05.mma kind::i8, TMA, TMEM).
//
// Replaces the same reference functions as K1 (_acc_group_panel +
// _spmm_task_*, spmm.py:192-280) for token counts where tensor-core tiles
// pay.  The 4x1 blocks are expanded into dense weight tiles (W^T, m
// contiguous, built once by the plan builder); X is read in its native
// orientation ([K, N] -> MN-major B operand, [N, K] -> K-major B operand),
// so no relayout pass exists.  Integer MACs are exact and wrap mod 2^32, so
// the expansion changes no bit of the accumulator.
//
// Kernels sharing one epilogue:
//
//  k2   single CTA, M128 x N256 tiles, both operands streamed through a TMA
//       ring (default for K <= 1024).
//  k2p  a CTA *pair* (cluster of 2, tcgen05 cta_group::2) computing
//       D[256 W rows x 256 tokens] per tile; each CTA holds half of A and
//       half of B, so every SM moves half the operand bytes (default for
//       K > 1024).  XSTAT keeps the pair's activation tile resident while W
//       streams (SI_K2_VARIANT=xstat).
//  k2x  pair + expander warps that build the dense W tile in smem from the
//       block lists (SI_K2_VARIANT=expand[_xstat]).
//  k2s  pair on the 2:4 sparse tensor-core path (tcgen05.mma.sp): the plan
//       packs each 4-wide k window's first two nonzero columns into the
//       compressed operand + metadata; columns beyond two per window are
//       added in the epilogue from per-row residual lists.  M256 x N192
//       tiles so the metadata fits TMEM next to two accumulators.
//
// Roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer (one
// thread; in a pair only the leader CTA issues), then the epilogue warps (4
// per TMEM lane quarter, 64 tokens each).  TMEM holds two accumulators so the
// epilogue of tile i overlaps the MMAs of tile i+1.
//
// Epilogue (all compiled forms of the reference's _run_chain,
// epilogue.py:207-249): tcgen05.ld 32x32b.x32 -> registers -> the form's
// math -> 8-bit outputs: saturating pack, 4x4 quad byte transpose, 128B-
// swizzled smem tile, TMA store; 32-bit outputs: coalesced 128-byte rows.
// The requant form (BASELINE config 5) uses no conversion instruction (those
// run on the quarter-rate XU pipe): the accumulator becomes an f32 by the
// 1.5*2^23 magic-number trick (exact for |a| < 2^22), r = a * c[m] with
// c = f32(scale_in/fp) in packed f32x2 ops, rint(r) by the same magic, and
// the certificate |r - rint(r)| + 2^-22|r| < 1/2 is max-reduced per 32
// elements; a chunk that fails it (or holds an out-of-range accumulator)
// recomputes the flagged elements with the reference's f64 expression.
// Error bound: |r - y| <= (2^-23 + 2^-48)|y| (a exact, one rounding each for
// c and a*c; y = the reference's f64 value), so outside the certificate's
// band rint(r) == rint(y) and the output bits match.
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

    const int prod = producer_index(warp, 2 + EPI_WARPS);
    // (a producer must never run more than one ring round ahead of the
    // slot it waits on: parity waits cannot tell rounds r-1 and r-3 apart)
    const int nprod = (P.debug & 4096) ? 1 : (NPROD < STAGES ? NPROD : STAGES);   // 4096: single producer
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
                    tc::mbar_spin(&empty[stage], phase ^ 1);
                    uint8_t *a_s = smem + stage * S_STAGE;
                    uint8_t *b_s = a_s + S_A;
                    if (P.debug & 8) {
                        tc::mbar_arrive(&full[stage]);
                    } else {
                        const int lmt = (P.debug & 2) ? 0 : mt, lnt = (P.debug & 4) ? 0 : nt;
                        tc::mbar_expect_tx(&full[stage], S_STAGE);
                        tc::tma_load_2d(a_s, &tmap_w, &full[stage], lmt * S_BM, kc * BK);
                        if (P.b_mn_major) {
                            tc::tma_load_2d(b_s, &tmap_x, &full[stage], lnt * TILE_N, kc * BK);
                            tc::tma_load_2d(b_s + S_B / 2, &tmap_x, &full[stage], lnt * TILE_N + 128, kc * BK);
                        } else {
                            tc::tma_load_2d(b_s, &tmap_x, &full[stage], kc * BK, lnt * TILE_N);
                        }
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
                tc::mbar_spin(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * TILE_N;
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_spin(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_addr = tc::smem_u32(smem + stage * S_STAGE);
                    const uint32_t b_addr = a_addr + S_A;
#pragma unroll
                    for (int kk = 0; kk < ((P.debug & 16) ? 0 : BK / 32); ++kk) {
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
        if ((OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) && W.q == 2 && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

// ================================================================ CTA pair
// Per CTA: A half = 128 W rows x 128 k (16 KB), B half = 128 tokens x 128 k
// (16 KB).  X-stationary: B halves for all k chunks stay resident.
constexpr int P_A = 128 * BK;        // 16 KB
constexpr int P_B = 128 * BK;        // 16 KB
constexpr int KMAX_XSTAT = 1024;     // resident X: 128 tokens x K <= 128 KB per CTA

// BKS: k per pipeline stage (128, or 256 for the big-stage variant pair256)
template <int MODE, int OUTK, bool XSTAT, int BKS = BK>
constexpr int pair_stages()
{
    constexpr int fixed = staged_bytes<OUTK>() + table_bytes<MODE>() + 2048 + (XSTAT ? KMAX_XSTAT * 128 : 0);
    constexpr int per = XSTAT ? 128 * BKS : 2 * 128 * BKS;
    constexpr int s = (SMEM_MAX - fixed) / per;
    return s > 8 ? 8 : s;
}
template <int MODE, int OUTK, bool XSTAT, int BKS = BK>
constexpr int pair_smem()
{
    return pair_stages<MODE, OUTK, XSTAT, BKS>() * (XSTAT ? 128 * BKS : 2 * 128 * BKS) +
           (XSTAT ? KMAX_XSTAT * 128 : 0) + staged_bytes<OUTK>() + table_bytes<MODE>() + 1024 + 512;
}

template <int MODE, int OUTK, bool XSTAT, int BKS = BK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(MT_THREADS, 1)
k2p_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
           const __grid_constant__ CUtensorMap tmap_o, const K2Params P, const EpiParams E)
{
    static_assert(!XSTAT || BKS == BK, "X-stationary uses 128-k stages");
    constexpr int P_A = 128 * BKS, P_B = 128 * BKS;
    constexpr int STAGES = pair_stages<MODE, OUTK, XSTAT, BKS>();
    constexpr int SLOT = XSTAT ? P_A : (P_A + P_B);
    constexpr int XBYTES = XSTAT ? KMAX_XSTAT * 128 : 0;
    constexpr int XCH = KMAX_XSTAT / BK;             // 8 resident X chunks
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *xbuf = smem;                            // XSTAT: [kchunks][128 tok x 128 k]
    uint8_t *ring = smem + XBYTES;
    uint8_t *staging = ring + STAGES * SLOT;
    uint8_t *tables = staging + staged_bytes<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint64_t *xfull = tempty + 2;                    // per K chunk of the resident X tile
    uint64_t *xempty = xfull + XCH;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(xempty + XCH);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    // work units: XSTAT -> (token tile, m-group); else (token tile, m-tile), m fastest
    const int units = XSTAT ? P.ntiles * P.mgroups : P.ntiles * P.mtiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 2 * EPI_WARPS);
        }
        for (int c = 0; c < XCH; ++c) {
            tc::mbar_init(&xfull[c], 1);
            tc::mbar_init(&xempty[c], 1);
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

    auto unit_range = [&](int unit, int &nt, int &m_lo, int &m_hi) {
        if (XSTAT) {
            nt = unit / P.mgroups;
            const int mg = unit % P.mgroups;
            const int base = P.mtiles / P.mgroups, rem = P.mtiles % P.mgroups;
            m_lo = mg * base + (mg < rem ? mg : rem);
            m_hi = m_lo + base + (mg < rem ? 1 : 0);
        } else {
            nt = unit / P.mtiles;
            m_lo = unit % P.mtiles;
            m_hi = m_lo + 1;
        }
    };

    const int prod = producer_index(warp, 2 + EPI_WARPS);
    // (a producer must never run more than one ring round ahead of the
    // slot it waits on: parity waits cannot tell rounds r-1 and r-3 apart)
    const int nprod = (P.debug & 4096) ? 1 : (NPROD < STAGES ? NPROD : STAGES);   // 4096: single producer
    if (prod >= 0) {
        {   // whole warp, one elected lane issues (tcw::)
            // ---------------- TMA producers (both CTAs; bytes land on the leader's barriers)
            const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
            const uint32_t xfull0 = tc::mapa(tc::smem_u32(xfull), 0);
            int stage = 0, it = 0;
            uint32_t phase = 0, xphase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, m_lo, m_hi;
                unit_range(unit, nt, m_lo, m_hi);
                const int tok = nt * TILE_N + 128 * (int)rank;
                for (int mt = m_lo; mt < m_hi; ++mt) {
                    for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                        if (it % nprod != prod) {
                            if (++stage == STAGES) { stage = 0; phase ^= 1; }
                            continue;
                        }
                        if (XSTAT && mt == m_lo) {
                            // roll the resident X tile chunk by chunk: chunk kc is
                            // reloaded as soon as the previous unit's last MMA on it retires
                            tc::mbar_spin(&xempty[kc], xphase ^ 1);
                            if (rank == 0) tcw::mbar_expect_tx(&xfull[kc], 2 * P_B);
                            if (P.b_mn_major)
                                tcw::tma_load_2d_2sm(xbuf + kc * P_B, &tmap_x, xfull0 + 8 * kc, tok, kc * BK);
                            else
                                tcw::tma_load_2d_2sm(xbuf + kc * P_B, &tmap_x, xfull0 + 8 * kc, kc * BK, tok);
                        }
                        tc::mbar_spin(&empty[stage], phase ^ 1);
                        uint8_t *a_s = ring + stage * SLOT;
                        const uint32_t fb = full0 + 8 * stage;
                        if (rank == 0) tcw::mbar_expect_tx(&full[stage], 2 * SLOT);
                        // (debug 2 / 4: every W / X load from tile 0 -- experiments)
                        const int lmt = (P.debug & 2) ? 0 : mt, ltok = (P.debug & 4) ? 128 * (int)rank : tok;
                        tcw::tma_load_2d_2sm(a_s, &tmap_w, fb, lmt * 256 + 128 * (int)rank, kc * BKS);
                        if (!XSTAT) {
                            if (P.b_mn_major)
                                tcw::tma_load_2d_2sm(a_s + P_A, &tmap_x, fb, ltok, kc * BKS);
                            else
                                // token-major X: K-major boxes span at most 128 k (one
                                // SWIZZLE_128B row), so a 256-k stage is two stacked tiles
                                for (int h = 0; h < BKS / BK; ++h)
                                    tcw::tma_load_2d_2sm(a_s + P_A + h * (128 * BK), &tmap_x, fb, kc * BKS + h * BK, ltok);
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                xphase ^= 1;
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ---------------- MMA issuer: leader CTA, whole warp, one elected lane issues, M256 x N256 x K32
            const uint32_t idesc = tc::idesc_i8(256, TILE_N, 1, P.b_mn_major ? 1 : 0);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0, xphase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, m_lo, m_hi;
                unit_range(unit, nt, m_lo, m_hi);
                for (int mt = m_lo; mt < m_hi; ++mt) {
                    if (!(P.debug & 262144)) tc::mbar_spin(&tempty[acc], acc_phase ^ 1);   // experiment: no wait
                    tc::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * TILE_N;
                    for (int kc = 0; kc < P.kchunks; ++kc) {
                        if (XSTAT && mt == m_lo) tc::mbar_spin(&xfull[kc], xphase);
                        tc::mbar_spin(&full[stage], phase);
                        tc::tc_fence_after();
                        const uint32_t a_addr = tc::smem_u32(ring + stage * SLOT);
                        const uint32_t b_addr = XSTAT ? tc::smem_u32(xbuf + kc * P_B) : a_addr + P_A;
#pragma unroll
                        for (int kk = 0; kk < ((P.debug & 16) ? 0 : BKS / 32); ++kk) {
                            const uint64_t adesc = tc::smem_desc_sw128(a_addr + kk * 4096, P_A, 1024);
                            const uint64_t bdesc =
                                P.b_mn_major ? tc::smem_desc_sw128(b_addr + kk * 4096, P_B, 1024)
                                             : tc::smem_desc_sw128(b_addr + (kk >> 2) * (128 * BK) + (kk & 3) * 32, 16, 1024);
                            tcw::mma_i8_2sm(d_tmem, adesc, bdesc, idesc, (kc | kk) ? 1u : 0u);
                        }
                        if (P.debug & 65536) {
                            // experiment (with debug 16): release by plain mbarrier arrives
                            if (lane == 0) {
                                tc::mbar_arrive(&empty[stage]);
                                tc::mbar_arrive_cluster(tc::mapa(tc::smem_u32(&empty[stage]), 1));
                            }
                        } else {
                            tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                        }
                        if (XSTAT && mt == m_hi - 1) tcw::mma_commit_2sm_mc(&xempty[kc], 0x3);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    tcw::mma_commit_2sm_mc(&tfull[acc], 0x3);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
                xphase ^= 1;
            }
        }
    } else if (warp < 2 + EPI_WARPS) {
        // ---------------- epilogue warps (both CTAs; each reads its own TMEM half)
        const EpiWarp W = make_epi_warp<MODE>(warp, lane, staging, tables, E);
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            int nt, m_lo, m_hi;
            unit_range(unit, nt, m_lo, m_hi);
            for (int mt = m_lo; mt < m_hi; ++mt) {
                const uint32_t te = tempty0 + 8 * acc;
                uint64_t *tf = &tfull[acc];
                const uint32_t ph = acc_phase;
                if (P.debug & 524288) {   // experiment: bare handshake (wait, release)
                    tc::mbar_wait(tf, ph);
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_cluster(te);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                    continue;
                }
                epi_tile<MODE, OUTK>(tmem_base, acc * TILE_N, mt * 256 + 128 * (int)rank, (int64_t)nt * TILE_N,
                                     &tmap_o, P, E, W, [tf, ph] { tc::mbar_wait(tf, ph); },
                                     [te] { tc::mbar_arrive_cluster(te); });
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
        if ((OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) && W.q == 2 && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(tmem_base, 512);
    }
}


// ================================================================ clusters of CTA pairs sharing X
// XM pairs (cluster of 2*XM CTAs) compute the same 256-token tile for XM
// consecutive 256-row tiles.  Every CTA loads its own W half (2SM TMA, to its
// pair leader's barrier) and a 128/XM-row k-slice of its token half of X,
// multicast to the CTAs holding the same token half in all XM pairs: the
// L2 -> crossbar traffic for X drops by XM (the pair kernel's TMA-only
// mainloop runs at the lts2xbar peak, profiles/).  A non-leader CTA's X
// slices complete on its own barrier; its warp 1 (idle there) forwards the
// completion to the pair leader.  A stage is free again once all XM pair
// leaders committed it (empty barrier count XM, commit multicast to the cluster).
template <int MODE, int OUTK, int XM>
constexpr int mc_stages()
{
    constexpr int s = (SMEM_MAX - staged_bytes<OUTK>() - table_bytes<MODE>() - 2048) / (P_A + P_B);
    return s > 8 ? 8 : s;
}
template <int MODE, int OUTK, int XM>
constexpr int mc_smem()
{
    return mc_stages<MODE, OUTK, XM>() * (P_A + P_B) + staged_bytes<OUTK>() + table_bytes<MODE>() + 1024 + 512;
}

template <int MODE, int OUTK, int XM>
__global__ void __cluster_dims__(2 * XM, 1, 1) __launch_bounds__(MT_THREADS, 1)
k2m_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
           const __grid_constant__ CUtensorMap tmap_o, const K2Params P, const EpiParams E)
{
    constexpr int STAGES = mc_stages<MODE, OUTK, XM>();
    constexpr int SLOT = P_A + P_B;
    constexpr int XROWS = BK / XM;                   // k rows of each X slice
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *ring = smem;
    uint8_t *staging = ring + STAGES * SLOT;
    uint8_t *tables = staging + staged_bytes<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = tc::cluster_ctarank();
    const uint32_t q = crank >> 1, r = crank & 1, lead = 2 * q;
    const int cl = blockIdx.x / (2 * XM), ncl = gridDim.x / (2 * XM);
    const int mgroups = P.mtiles / XM;
    const int units = P.ntiles * mgroups;
    const uint16_t pair_mask = (uint16_t)(3u << lead);
    const uint16_t all_mask = (uint16_t)((1u << (2 * XM)) - 1);
    uint16_t xmask = 0;
#pragma unroll
    for (int i = 0; i < XM; ++i) xmask |= (uint16_t)(1u << (2 * i + r));

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            // leader: its producer's arrive.expect_tx + the peer's forward; peer: its producer
            tc::mbar_init(&full[s], r == 0 ? 2 : 1);
            tc::mbar_init(&empty[s], XM);
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

    const int prod = producer_index(warp, 2 + EPI_WARPS);
    // (a producer must never run more than one ring round ahead of the
    // slot it waits on: parity waits cannot tell rounds r-1 and r-3 apart)
    const int nprod = (P.debug & 4096) ? 1 : (NPROD < STAGES ? NPROD : STAGES);   // 4096: single producer
    if (prod >= 0) {
        {   // ---------------- TMA producers (whole warp, one elected lane issues)
            const uint32_t full_lead = tc::mapa(tc::smem_u32(full), lead);
            int stage = 0, it = 0;
            uint32_t phase = 0;
            for (int unit = cl; unit < units; unit += ncl) {
                const int nt = unit / mgroups, mt = (unit % mgroups) * XM + (int)q;
                const int tok = nt * TILE_N + 128 * (int)r;
                for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                    if (it % nprod != prod) {
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    tc::mbar_spin(&empty[stage], phase ^ 1);
                    uint8_t *a_s = ring + stage * SLOT;
                    // leader barrier: both W halves + its X half; peer barrier: its X half
                    tcw::mbar_expect_tx(&full[stage], r == 0 ? 2 * P_A + P_B : P_B);
                    tcw::tma_load_2d_2sm(a_s, &tmap_w, full_lead + 8 * stage, mt * 256 + 128 * (int)r, kc * BK);
                    tcw::tma_load_2d_mc(a_s + P_A + q * XROWS * 128, &tmap_x, &full[stage], tok,
                                       kc * BK + (int)q * XROWS, xmask);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (r == 0) {
            // ---------------- MMA issuer: pair leader, whole warp, one elected lane issues, M256 x N256 x K32
            const uint32_t idesc = tc::idesc_i8(256, TILE_N, 1, 1);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int unit = cl; unit < units; unit += ncl) {
                tc::mbar_spin(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * TILE_N;
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_spin(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_addr = tc::smem_u32(ring + stage * SLOT);
                    const uint32_t b_addr = a_addr + P_A;
#pragma unroll
                    for (int kk = 0; kk < ((P.debug & 16) ? 0 : BK / 32); ++kk) {
                        const uint64_t adesc = tc::smem_desc_sw128(a_addr + kk * 4096, P_A, 1024);
                        const uint64_t bdesc = tc::smem_desc_sw128(b_addr + kk * 4096, P_B, 1024);
                        tcw::mma_i8_2sm(d_tmem, adesc, bdesc, idesc, (kc | kk) ? 1u : 0u);
                    }
                    tcw::mma_commit_2sm_mc(&empty[stage], all_mask);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tcw::mma_commit_2sm_mc(&tfull[acc], pair_mask);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        } else if (lane == 0) {
            // ---------------- peer CTA: forward X-slice completion to the pair leader
            const uint32_t full_lead = tc::mapa(tc::smem_u32(full), lead);
            int stage = 0;
            uint32_t phase = 0;
            for (int unit = cl; unit < units; unit += ncl) {
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_spin(&full[stage], phase);
                    tc::mbar_arrive_cluster(full_lead + 8 * stage);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp < 2 + EPI_WARPS) {
        // ---------------- epilogue warps (each CTA reads its own TMEM half)
        const EpiWarp W = make_epi_warp<MODE>(warp, lane, staging, tables, E);
        const uint32_t tempty_lead = tc::mapa(tc::smem_u32(tempty), lead);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int unit = cl; unit < units; unit += ncl) {
            const int nt = unit / mgroups, mt = (unit % mgroups) * XM + (int)q;
            const uint32_t te = tempty_lead + 8 * acc;
            uint64_t *tf = &tfull[acc];
            const uint32_t ph = acc_phase;
            epi_tile<MODE, OUTK>(tmem_base, acc * TILE_N, mt * 256 + 128 * (int)r, (int64_t)nt * TILE_N, &tmap_o, P,
                                 E, W, [tf, ph] { tc::mbar_wait(tf, ph); }, [te] { tc::mbar_arrive_cluster(te); });
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if ((OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) && W.q == 2 && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(tmem_base, 512);
    }
}


// ================================================================ CTA pair, expanded W
// As k2p, but the weight operand never streams densely: per (128-row tile,
// 128-k chunk) the plan holds the nonzero 4x1 blocks as (smem word offset,
// 4-row value word) lists (csrc/plan.cpp build_expand_lists).  The producer
// bulk-copies a stage's two lists (k rows 0-63 / 64-127) into an entry ring;
// two expander warps zero their half of the MN-major SWIZZLE_128B A tile and
// scatter the words.  W traffic per token tile drops from M*K bytes to
// ~6 bytes per nonzero block, and a stage is ready a few hundred cycles after
// its lists land instead of after a 16 KB L2->smem TMA round trip.
struct XLayout {
    int32_t nstages;      // W (and streamed-X) ring slots
    int32_t neslots;      // entry-list ring slots
    int32_t eslot_bytes;  // bytes per entry slot (two half lists)
    int32_t ehalf_bytes;  // offset of the second half list in a slot
    int32_t xbytes;       // resident X bytes (X-stationary) or 0
    int32_t slot_bytes;   // W (+X) bytes per ring slot
    int32_t staged;       // staging bytes
    int32_t tables;       // table bytes
};
constexpr int X_MAXSLOTS = 12;
constexpr int EXP_WARPS = 2;
constexpr int X_THREADS = THREADS + 32 * EXP_WARPS;

template <int MODE, int OUTK, bool XSTAT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(X_THREADS, 1)
k2x_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_o, const K2Params P,
           const EpiParams E, const XLayout L, const uint32_t *__restrict__ eptr, const uint8_t *__restrict__ ent)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *xbuf = smem;
    uint8_t *ring = smem + L.xbytes;
    uint8_t *staging = ring + L.nstages * L.slot_bytes;
    uint8_t *tables = staging + L.staged;
    uint8_t *eslots = tables + L.tables;
    uint64_t *full = reinterpret_cast<uint64_t *>(eslots + L.neslots * L.eslot_bytes);
    uint64_t *empty = full + X_MAXSLOTS;
    uint64_t *efull = empty + X_MAXSLOTS;
    uint64_t *eempty = efull + X_MAXSLOTS;
    uint64_t *tfull = eempty + X_MAXSLOTS;
    uint64_t *tempty = tfull + 2;
    uint64_t *xfull = tempty + 2;
    uint64_t *xempty = xfull + 8;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(xempty + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int units = XSTAT ? P.ntiles * P.mgroups : P.ntiles * P.mtiles;
    const int S = L.nstages, ES = L.neslots;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(&full[s], 2 + (XSTAT ? 0 : 1));
            tc::mbar_init(&empty[s], 1);
        }
        for (int e = 0; e < ES; ++e) {
            tc::mbar_init(&efull[e], 1);
            tc::mbar_init(&eempty[e], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 2 * EPI_WARPS);
        }
        for (int c = 0; c < 8; ++c) {
            tc::mbar_init(&xfull[c], 1);
            tc::mbar_init(&xempty[c], 1);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_x);
    }
    if (warp == 1) tc::tmem_alloc_2sm(tmem_slot, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto unit_range = [&](int unit, int &nt, int &m_lo, int &m_hi) {
        if (XSTAT) {
            nt = unit / P.mgroups;
            const int mg = unit % P.mgroups;
            const int base = P.mtiles / P.mgroups, rem = P.mtiles % P.mgroups;
            m_lo = mg * base + (mg < rem ? mg : rem);
            m_hi = m_lo + base + (mg < rem ? 1 : 0);
        } else {
            nt = unit / P.mtiles;
            m_lo = unit % P.mtiles;
            m_hi = m_lo + 1;
        }
    };

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer: entry lists (own CTA) + X (TMA, bytes on the leader)
            const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
            const uint32_t xfull0 = tc::mapa(tc::smem_u32(xfull), 0);
            int stage = 0, es = 0;
            uint32_t phase = 0, ephase = 0, xphase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, m_lo, m_hi;
                unit_range(unit, nt, m_lo, m_hi);
                const int tok = nt * TILE_N + 128 * (int)rank;
                for (int mt = m_lo; mt < m_hi; ++mt) {
                    const int rt = 2 * mt + (int)rank;
                    for (int kc = 0; kc < P.kchunks; ++kc) {
                        // entry lists of this CTA's half of the stage
                        tc::mbar_spin(&eempty[es], ephase ^ 1);
                        uint32_t b0 = 0, b1 = 0, o0 = 0, o1 = 0;
                        if (rt < P.rtiles) {
                            const int j = (rt * P.kchunks + kc) * 2;
                            o0 = __ldg(eptr + j);
                            o1 = __ldg(eptr + j + 1);
                            b0 = o1 - o0;
                            b1 = __ldg(eptr + j + 2) - o1;
                        }
                        tc::mbar_expect_tx(&efull[es], b0 + b1);
                        uint8_t *dst = eslots + es * L.eslot_bytes;
                        if (b0) tc::bulk_load(dst, ent + o0, b0, &efull[es]);
                        if (b1) tc::bulk_load(dst + L.ehalf_bytes, ent + o1, b1, &efull[es]);
                        if (++es == ES) { es = 0; ephase ^= 1; }
                        if (XSTAT) {
                            if (mt == m_lo) {
                                tc::mbar_spin(&xempty[kc], xphase ^ 1);
                                if (rank == 0) tc::mbar_expect_tx(&xfull[kc], 2 * P_B);
                                if (P.b_mn_major)
                                    tc::tma_load_2d_2sm(xbuf + kc * P_B, &tmap_x, xfull0 + 8 * kc, tok, kc * BK);
                                else
                                    tc::tma_load_2d_2sm(xbuf + kc * P_B, &tmap_x, xfull0 + 8 * kc, kc * BK, tok);
                            }
                        } else {
                            tc::mbar_spin(&empty[stage], phase ^ 1);
                            uint8_t *b_s = ring + stage * L.slot_bytes + P_A;
                            const uint32_t fb = full0 + 8 * stage;
                            if (rank == 0) tc::mbar_expect_tx(&full[stage], 2 * P_B);
                            if (P.b_mn_major)
                                tc::tma_load_2d_2sm(b_s, &tmap_x, fb, tok, kc * BK);
                            else
                                tc::tma_load_2d_2sm(b_s, &tmap_x, fb, kc * BK, tok);
                            if (++stage == S) { stage = 0; phase ^= 1; }
                        }
                    }
                }
                xphase ^= 1;
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // ---------------- MMA issuer: leader CTA, one thread, M256 x N256 x K32
            const uint32_t idesc = tc::idesc_i8(256, TILE_N, 1, P.b_mn_major ? 1 : 0);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0, xphase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, m_lo, m_hi;
                unit_range(unit, nt, m_lo, m_hi);
                for (int mt = m_lo; mt < m_hi; ++mt) {
                    tc::mbar_spin(&tempty[acc], acc_phase ^ 1);
                    tc::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * TILE_N;
                    for (int kc = 0; kc < P.kchunks; ++kc) {
                        if (XSTAT && mt == m_lo) tc::mbar_spin(&xfull[kc], xphase);
                        tc::mbar_spin(&full[stage], phase);
                        tc::tc_fence_after();
                        const uint32_t a_addr = tc::smem_u32(ring + stage * L.slot_bytes);
                        const uint32_t b_addr = XSTAT ? tc::smem_u32(xbuf + kc * P_B) : a_addr + P_A;
#pragma unroll
                        for (int kk = 0; kk < ((P.debug & 16) ? 0 : BK / 32); ++kk) {
                            const uint64_t adesc = tc::smem_desc_sw128(a_addr + kk * 4096, P_A, 1024);
                            const uint64_t bdesc = P.b_mn_major ? tc::smem_desc_sw128(b_addr + kk * 4096, P_B, 1024)
                                                                : tc::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
                            tc::mma_i8_2sm(d_tmem, adesc, bdesc, idesc, (kc | kk) ? 1u : 0u);
                        }
                        tc::mma_commit_2sm_mc(&empty[stage], 0x3);
                        if (XSTAT && mt == m_hi - 1) tc::mma_commit_2sm_mc(&xempty[kc], 0x3);
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                    tc::mma_commit_2sm_mc(&tfull[acc], 0x3);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
                xphase ^= 1;
            }
        }
    } else if (warp >= 2 + EPI_WARPS) {
        // ---------------- expanders: warp e builds every EXP_WARPS-th stage's
        // whole A tile (zero 16 KB, scatter the two half lists), so each warp
        // has EXP_WARPS MMA-stage times to finish one stage
        const int e = warp - (2 + EPI_WARPS);
        const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
        long it = 0;  // global stage counter (same sequence as producer / MMA)
        for (int unit = pair; unit < units; unit += npairs) {
            int nt, m_lo, m_hi;
            unit_range(unit, nt, m_lo, m_hi);
            for (int mt = m_lo; mt < m_hi; ++mt) {
                const int rt = 2 * mt + (int)rank;
                for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                    if ((int)(it % EXP_WARPS) != e) continue;
                    const int stage = (int)(it % S), es = (int)(it % ES);
                    const uint32_t phase = (uint32_t)((it / S) & 1), ephase = (uint32_t)((it / ES) & 1);
                    int n0 = 0, n1 = 0;
                    if (rt < P.rtiles) {
                        const int j = (rt * P.kchunks + kc) * 2;
                        const uint32_t o0 = __ldg(eptr + j), o1 = __ldg(eptr + j + 1), o2 = __ldg(eptr + j + 2);
                        n0 = (int)((o1 - o0) / 6);
                        n1 = (int)((o2 - o1) / 6);
                    }
                    tc::mbar_spin(&empty[stage], phase ^ 1);
                    uint8_t *a_s = ring + stage * L.slot_bytes;
                    if (!(P.debug & 32)) {
                        uint4 *z = reinterpret_cast<uint4 *>(a_s);
#pragma unroll 8
                        for (int i = lane; i < P_A / 16; i += 32) z[i] = make_uint4(0, 0, 0, 0);
                    }
                    tc::mbar_spin(&efull[es], ephase);
                    __syncwarp();
                    uint32_t *w32 = reinterpret_cast<uint32_t *>(a_s);
                    if (!(P.debug & 64)) {
#pragma unroll 1
                        for (int hh = 0; hh < 2; ++hh) {
                            const int n = hh ? n1 : n0;
                            const uint8_t *el = eslots + es * L.eslot_bytes + hh * L.ehalf_bytes;
                            // 4 entries per lane per step: 16 B of values, 8 B of offsets
                            const uint4 *v4 = reinterpret_cast<const uint4 *>(el);
                            const uint2 *o4 = reinterpret_cast<const uint2 *>(el + 4 * n);
                            for (int i = lane; i < n / 4; i += 32) {
                                const uint4 v = v4[i];
                                const uint2 o = o4[i];
                                w32[o.x & 0xFFFF] = v.x;
                                w32[o.x >> 16] = v.y;
                                w32[o.y & 0xFFFF] = v.z;
                                w32[o.y >> 16] = v.w;
                            }
                        }
                    }
                    if (!(P.debug & 128)) tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tc::mbar_arrive(&eempty[es]);
                        tc::mbar_arrive_cluster(full0 + 8 * stage);
                    }
                }
            }
        }
    } else {
        // ---------------- epilogue warps (both CTAs; each reads its own TMEM half)
        const EpiWarp W = make_epi_warp<MODE>(warp, lane, staging, tables, E);
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            int nt, m_lo, m_hi;
            unit_range(unit, nt, m_lo, m_hi);
            for (int mt = m_lo; mt < m_hi; ++mt) {
                const uint32_t te = tempty0 + 8 * acc;
                uint64_t *tf = &tfull[acc];
                const uint32_t ph = acc_phase;
                epi_tile<MODE, OUTK>(tmem_base, acc * TILE_N, mt * 256 + 128 * (int)rank, (int64_t)nt * TILE_N,
                                     &tmap_o, P, E, W, [tf, ph] { tc::mbar_wait(tf, ph); },
                                     [te] { tc::mbar_arrive_cluster(te); });
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
        if ((OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) && W.q == 2 && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(tmem_base, 512);
    }
}

// ================================================================ CTA pair, 2:4 sparse A
// Per CTA and k chunk: the plan's 12 KB image of its 128 W rows (compressed
// A 8 KB, K-major SWIZZLE_NONE, + two 2 KB metadata tiles) and 96 tokens x
// 128 k of X as three SWIZZLE_32B atoms (32 tokens wide).  Per stage the
// leader copies both metadata tiles into TMEM (tcgen05.cp, 4 columns each)
// and issues two M256 x N192 x K64 tcgen05.mma.sp.  TMEM: accumulators at
// columns [0,192) and [192,384), metadata slots at 384 and 392 (alternating
// stages).
constexpr int SP_TILE_N = 192;
constexpr int SP_EPI_WARPS = 12;
constexpr int SP_THREADS = 32 * (2 + SP_EPI_WARPS + NPROD - 1);
constexpr int SP_IMG = 12288;
constexpr int SP_BATOM = 32 * BK;          // 32 tokens x 128 k = 4 KB
#ifdef SP_XEXP
constexpr int SP_B = 4 * SP_BATOM;
#else
constexpr int SP_B = 3 * SP_BATOM;
#endif
constexpr int SP_SLOT = SP_IMG + SP_B;     // 24 KB
constexpr uint32_t SP_ECOL = 2 * SP_TILE_N;

template <int OUTK>
constexpr int sp_staged() { return (OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) ? 3 * STG_GROUP : 0; }
template <int MODE, int OUTK>
constexpr int sp_stages()
{
    constexpr int s = (SMEM_MAX - sp_staged<OUTK>() - table_bytes<MODE>() - 2048) / SP_SLOT;
    return s > 8 ? 8 : s;
}
template <int MODE, int OUTK>
constexpr int sp_smem()
{
    return sp_stages<MODE, OUTK>() * SP_SLOT + sp_staged<OUTK>() + table_bytes<MODE>() + 1024 + 512;
}

template <int MODE, int OUTK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SP_THREADS, 1)
k2s_kernel(const __grid_constant__ CUtensorMap tmap_s, const __grid_constant__ CUtensorMap tmap_x,
           const __grid_constant__ CUtensorMap tmap_o, const K2Params P, const EpiParams E)
{
    constexpr int STAGES = sp_stages<MODE, OUTK>();
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *ring = smem;
    uint8_t *staging = ring + STAGES * SP_SLOT;
    uint8_t *tables = staging + sp_staged<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int units = P.ntiles * P.mtiles;          // (token tile, 256-row tile), rows fastest

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 2 * SP_EPI_WARPS);
        }
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_s);
        tc::tma_prefetch_desc(&tmap_x);
    }
    if (warp == 1) tc::tmem_alloc_2sm(tmem_slot, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int prod = producer_index(warp, 2 + SP_EPI_WARPS);
    // (a producer must never run more than one ring round ahead of the
    // slot it waits on: parity waits cannot tell rounds r-1 and r-3 apart)
    const int nprod = (P.debug & 4096) ? 1 : (NPROD < STAGES ? NPROD : STAGES);   // 4096: single producer
    if (prod >= 0) {
        if (lane == 0) {
            // ---------------- TMA producers (both CTAs; bytes land on the leader's barriers)
            const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
            int stage = 0, it = 0;
            uint32_t phase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                const int nt = unit / P.mtiles, mt = unit % P.mtiles;
                const int tok = nt * SP_TILE_N + 96 * (int)rank;
                const int rt = 2 * mt + (int)rank;
                for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                    if (it % nprod != prod) {
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    tc::mbar_spin(&empty[stage], phase ^ 1);
                    uint8_t *slot = ring + stage * SP_SLOT;
                    const uint32_t fb = full0 + 8 * stage;
                    if (rank == 0) tc::mbar_expect_tx(&full[stage], 2 * ((P.debug & 1024) ? SP_B : SP_SLOT));
                    if (!(P.debug & 1024))
                        tc::tma_load_2d_2sm(slot, &tmap_s, fb, 0, (rt * P.kchunks + kc) * (SP_IMG / 128));
#ifdef SP_XEXP
                    tc::tma_load_2d_2sm(slot + SP_IMG, &tmap_x, fb, tok, kc * BK);
#else
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        tc::tma_load_2d_2sm(slot + SP_IMG + i * SP_BATOM, &tmap_x, fb, tok + 32 * i, kc * BK);
#endif
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // ---------------- MMA issuer: leader CTA, one thread
            const uint32_t idesc = tc::idesc_i8(256, SP_TILE_N, 0, 1) | (1u << 2);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0, eslot = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                tc::mbar_spin(&tempty[acc], acc_phase ^ 1);
                tc::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * SP_TILE_N;
                for (int kc = 0; kc < P.kchunks; ++kc) {
                    tc::mbar_spin(&full[stage], phase);
                    tc::tc_fence_after();
                    const uint32_t a_addr = tc::smem_u32(ring + stage * SP_SLOT);
                    const uint32_t e_tmem = tmem_base + SP_ECOL + 8 * eslot;
                    tc::tmem_cp_128x128b_2sm(e_tmem, tc::smem_desc(a_addr + 8192, 2048, 128, 0));
                    tc::tmem_cp_128x128b_2sm(e_tmem + 4, tc::smem_desc(a_addr + 10240, 2048, 128, 0));
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const uint64_t adesc = tc::smem_desc(a_addr + 256 * j, 128, 512, 0);
                        const uint64_t bdesc = tc::smem_desc(a_addr + SP_IMG + 2048 * j, SP_BATOM, 256, 6);
                        if (!(P.debug & 16))
                            tc::mma_sp_i8_2sm(d_tmem, adesc, bdesc, e_tmem + 4 * j, idesc, (kc | j) ? 1u : 0u);
                    }
                    tc::mma_commit_2sm_mc(&empty[stage], 0x3);
                    eslot ^= 1;
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tc::mma_commit_2sm_mc(&tfull[acc], 0x3);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp < 2 + SP_EPI_WARPS) {
        // ---------------- epilogue warps (both CTAs; each reads its own TMEM half)
        const EpiWarp W = make_epi_warp<MODE, SP_EPI_WARPS>(warp, lane, staging, tables, E);
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            const int nt = unit / P.mtiles, mt = unit % P.mtiles;
            const uint32_t te = tempty0 + 8 * acc;
            uint64_t *tf = &tfull[acc];
            const uint32_t ph = acc_phase;
            epi_tile<MODE, OUTK, true>(tmem_base, acc * SP_TILE_N, mt * 256 + 128 * (int)rank,
                                       (int64_t)nt * SP_TILE_N, &tmap_o, P, E, W,
                                       [tf, ph] { tc::mbar_wait(tf, ph); }, [te] { tc::mbar_arrive_cluster(te); });
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if ((OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) && W.q == 2 && lane == 0) tc::tma_store_wait_all0();
    }
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(tmem_base, 512);
    }
}

// shared-memory plan of k2x for this image; false if it does not fit
template <int MODE, int OUTK>
bool plan_xlayout(const SiImage *h, bool xstat, XLayout &L, int &smem)
{
    const int kch = h->tc_kpad / BK;
    L.staged = staged_bytes<OUTK>();
    L.tables = table_bytes<MODE>();
    L.xbytes = xstat ? kch * P_B : 0;
    L.slot_bytes = xstat ? P_A : P_A + P_B;
    L.ehalf_bytes = ((h->tc_emax * 6 + 127) / 128) * 128;
    L.eslot_bytes = 2 * L.ehalf_bytes;
    const int fixed = 1024 + 1024 + L.xbytes + L.staged + L.tables;
    // deep entry ring first (bulk-copy latency ~2 us), then W slots (>= 3)
    for (int es = X_MAXSLOTS; es >= 2; --es) {
        const int room = SMEM_MAX - fixed - es * L.eslot_bytes;
        int st = room / L.slot_bytes;
        if (st > 4) st = 4;
        if (st >= 3 || (es == 2 && st >= 2)) {
            L.nstages = st;
            L.neslots = es;
            smem = fixed + es * L.eslot_bytes + st * L.slot_bytes;
            return true;
        }
    }
    return false;
}

template <int MODE, int OUTK>
int launch_mode(const SpmmArgs &a, const CUtensorMap &tw, const CUtensorMap &tx, const CUtensorMap &to, K2Params p,
                int variant)
{
    EpiParams E = make_epi(a.h, a.img, a.sides, a.n);
    cudaStream_t st = (cudaStream_t)a.stream;
    const int sms = num_sms();
    if (variant == V_EXPAND || variant == V_EXPAND_XSTAT) {
        const bool xstat = variant == V_EXPAND_XSTAT;
        XLayout L;
        int smem = 0;
        if (!plan_xlayout<MODE, OUTK>(a.h, xstat, L, smem)) variant = xstat ? V_PAIR_XSTAT : V_PAIR;
        else {
            const uint32_t *eptr = img_sec<uint32_t>(a.img, a.h->off_tc_eptr);
            const uint8_t *ent = img_sec<uint8_t>(a.img, a.h->off_tc_ent);
            const int npairs = sms / 2;
            if (xstat) p.mgroups = pick_mgroups(p.mtiles, p.ntiles, npairs);
            const long units = xstat ? (long)p.ntiles * p.mgroups : (long)p.ntiles * p.mtiles;
            const int pairs = units < npairs ? (int)units : npairs;
            if (xstat) {
                auto kern = k2x_kernel<MODE, OUTK, true>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                kern<<<2 * pairs, X_THREADS, smem, st>>>(tx, to, p, E, L, eptr, ent);
            } else {
                auto kern = k2x_kernel<MODE, OUTK, false>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                kern<<<2 * pairs, X_THREADS, smem, st>>>(tx, to, p, E, L, eptr, ent);
            }
            return (int)cudaGetLastError();
        }
    }
    if (variant == V_MC2 || variant == V_MC4) {
        const int XM = variant == V_MC2 ? 2 : 4;
        const long units = (long)p.ntiles * (p.mtiles / XM);
        if (XM == 2) {
            auto kern = k2m_kernel<MODE, OUTK, 2>;
            constexpr int smem = mc_smem<MODE, OUTK, 2>();
            static_assert(smem <= SMEM_MAX, "shared memory budget");
            static int ncl = 0;
            if (!ncl) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                ncl = max_clusters(kern, 4, MT_THREADS, smem, sms / 4);
            }
            const int g = units < ncl ? (int)units : ncl;
            kern<<<4 * g, MT_THREADS, smem, st>>>(tw, tx, to, p, E);
        } else {
            auto kern = k2m_kernel<MODE, OUTK, 4>;
            constexpr int smem = mc_smem<MODE, OUTK, 4>();
            static_assert(smem <= SMEM_MAX, "shared memory budget");
            static int ncl = 0;
            if (!ncl) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                ncl = max_clusters(kern, 8, MT_THREADS, smem, sms / 8);
            }
            const int g = units < ncl ? (int)units : ncl;
            kern<<<8 * g, MT_THREADS, smem, st>>>(tw, tx, to, p, E);
        }
    } else if (variant == V_SPARSE) {
        auto kern = k2s_kernel<MODE, OUTK>;
        constexpr int smem = sp_smem<MODE, OUTK>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        static bool attr = false;
        if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); attr = true; }
        const int units = p.mtiles * p.ntiles;
        const int pairs = units < sms / 2 ? units : sms / 2;
        kern<<<2 * pairs, SP_THREADS, smem, st>>>(tw, tx, to, p, E);
    } else if (variant == V_SINGLE) {
        auto kern = k2_tc_kernel<MODE, OUTK>;
        constexpr int smem = single_smem<MODE, OUTK>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        static bool attr = false;
        if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); attr = true; }
        const int tiles = p.mtiles * p.ntiles;
        kern<<<tiles < sms ? tiles : sms, MT_THREADS, smem, st>>>(tw, tx, to, p, E);
    } else if (variant == V_PAIR256) {
        auto kern = k2p_kernel<MODE, OUTK, false, 256>;
        constexpr int smem = pair_smem<MODE, OUTK, false, 256>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        static bool attr = false;
        if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); attr = true; }
        const int units = p.mtiles * p.ntiles;
        const int pairs = units < sms / 2 ? units : sms / 2;
        kern<<<2 * pairs, MT_THREADS, smem, st>>>(tw, tx, to, p, E);
    } else if (variant == V_PAIR) {
        auto kern = k2p_kernel<MODE, OUTK, false>;
        constexpr int smem = pair_smem<MODE, OUTK, false>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        static bool attr = false;
        if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); attr = true; }
        const int units = p.mtiles * p.ntiles;
        const int pairs = units < sms / 2 ? units : sms / 2;
        kern<<<2 * pairs, MT_THREADS, smem, st>>>(tw, tx, to, p, E);
    } else {
        auto kern = k2p_kernel<MODE, OUTK, true>;
        constexpr int smem = pair_smem<MODE, OUTK, true>();
        static_assert(smem <= SMEM_MAX, "shared memory budget");
        static bool attr = false;
        if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); attr = true; }
        const int npairs = sms / 2;
        p.mgroups = pick_mgroups(p.mtiles, p.ntiles, npairs);
        const long units = (long)p.ntiles * p.mgroups;
        const int pairs = units < npairs ? (int)units : npairs;
        kern<<<2 * pairs, MT_THREADS, smem, st>>>(tw, tx, to, p, E);
    }
    return (int)cudaGetLastError();
}

template <int OUTK>
int launch_outk(const SpmmArgs &a, const CUtensorMap &tw, const CUtensorMap &tx, const CUtensorMap &to,
                const K2Params &p, int variant)
{
    switch (a.h->epi_mode) {
    case EPI_S32: return launch_mode<EPI_S32, OUTK>(a, tw, tx, to, p, variant);
    case EPI_DEQ_F32: return launch_mode<EPI_DEQ_F32, OUTK>(a, tw, tx, to, p, variant);
    case EPI_REQUANT: return launch_mode<EPI_REQUANT, OUTK>(a, tw, tx, to, p, variant);
    case EPI_REQUANT_LUT: return launch_mode<EPI_REQUANT_LUT, OUTK>(a, tw, tx, to, p, variant);
    case EPI_DEQ_TABLE: return launch_mode<EPI_DEQ_TABLE, OUTK>(a, tw, tx, to, p, variant);
    default: return launch_mode<EPI_GENERIC, OUTK>(a, tw, tx, to, p, variant);
    }
}

}  // namespace

bool k2_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx, int64_t)
{
    if (n < 1 || n > (int64_t)INT32_MAX - TILE_N) return false;
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
    static const int dbg = env_int("SI_K2_DEBUG", 0);
    static const int forced = [] {
        const char *e = getenv("SI_K2_VARIANT");
        if (!e) return -1;
        std::string s(e);
        return s == "single" ? (int)V_SINGLE : s == "pair" ? (int)V_PAIR : s == "xstat" ? (int)V_PAIR_XSTAT
             : s == "expand" ? (int)V_EXPAND : s == "expand_xstat" ? (int)V_EXPAND_XSTAT
             : s == "sparse" ? (int)V_SPARSE : s == "mc2" ? (int)V_MC2 : s == "mc4" ? (int)V_MC4
             : s == "pair256" ? (int)V_PAIR256 : s == "xsparse" ? 100 : s == "tmemw" ? 101 : -1;
    }();
    if (forced == 101) {
        if (k2a_supported(h, a.n, a.layout, a.x, a.ldx)) return k2a_launch(a);
        return (int)cudaErrorInvalidValue;
    }
    // K2t (X-stationary 2:4, spmm_tcx.cu; SI_K2_VARIANT=xsparse): token-major
    // X, K <= 1024, every pair tile's residual fits its slots.  Opt-in: on the
    // config-5 shapes it measures slower than the dense pair.
    if (forced == 100) {
        if (k2t_supported(h, a.n, a.layout, a.x, a.ldx)) return k2t_launch(a);
        return (int)cudaErrorInvalidValue;
    }
    // the pair kernels tile W rows by 256; an odd count of 128-row tiles reads
    // one tile of TMA out-of-bounds zero fill
    // measured default ("K2 variants"): the CTA pair unless the
    // weight has a single 128-row tile; the other variants stay selectable
    // (SI_K2_VARIANT) for tuning
    // [K, N] activations take the 256-k-stage pair (after the plan-image
    // alignment fix it measures best on every config-5 linear: 52.4 / 177.5 /
    // 167.9 us vs pair 54.5 / 197.0 / 169.4); token-major X the 128-k pair
    int variant = forced >= 0 ? forced : h->tc_mtiles <= 1 ? V_SINGLE : V_PAIR256;
    if (variant == V_PAIR_XSTAT && h->tc_kpad > KMAX_XSTAT) variant = V_PAIR;
    if (variant == V_EXPAND_XSTAT && h->tc_kpad > KMAX_XSTAT) variant = V_EXPAND;
    if (variant == V_SPARSE && a.layout != 0) variant = V_PAIR;   // k2s reads X as [K, N]
    // X-sharing clusters: [K, N] activations and whole groups of XM pair tiles
    if ((variant == V_MC2 || variant == V_MC4) && a.layout != 0) variant = V_PAIR;
    if (variant == V_MC4 && ((h->tc_mtiles + 1) / 2) % 4) variant = V_MC2;
    if (variant == V_MC2 && ((h->tc_mtiles + 1) / 2) % 2) variant = V_PAIR;

    CUtensorMap tw, tx, to;
    bool ok;
    if (variant == V_SPARSE) {
        // the 2:4 images viewed as rows of 128 B, one 96-row box per (tile, chunk)
        const uint64_t rows = (uint64_t)((h->tc_mtiles + 1) / 2 * 2) * (h->tc_kpad / BK) * (SP_IMG / 128);
        ok = encode_2d(&tw, img_sec<uint8_t>(a.img, h->off_sp_img), 128, rows, 128, 128, SP_IMG / 128,
                       CU_TENSOR_MAP_SWIZZLE_NONE) &&
#ifdef SP_XEXP
             encode_2d(&tx, a.x, (uint64_t)a.n, (uint64_t)h->K, (uint64_t)a.ldx, 128, BK);
#else
             encode_2d(&tx, a.x, (uint64_t)a.n, (uint64_t)h->K, (uint64_t)a.ldx, 32, BK, CU_TENSOR_MAP_SWIZZLE_32B);
#endif
    } else {
        const void *wt = img_sec<uint8_t>(a.img, h->off_tc_wt);
        const uint64_t mpad = (uint64_t)h->tc_mtiles * 128;
        const uint32_t xbox_tok = variant == V_SINGLE ? TILE_N : 128;
        const uint32_t bks = variant == V_PAIR256 ? 256 : BK;
        const uint32_t xbox_k = variant == V_MC2 ? BK / 2 : variant == V_MC4 ? BK / 4 : bks;
        ok = encode_2d(&tw, wt, mpad, (uint64_t)h->tc_kpad, mpad, 128, bks);
        if (a.layout == 0)
            ok = ok && encode_2d(&tx, a.x, (uint64_t)a.n, (uint64_t)h->K, (uint64_t)a.ldx, 128, xbox_k);
        else
            ok = ok && encode_2d(&tx, a.x, (uint64_t)h->K, (uint64_t)a.n, (uint64_t)a.ldx, BK, xbox_tok);
    }
    if (!ok) return (int)cudaErrorInvalidValue;
    K2Params p;
    const int tile_n = variant == V_SPARSE ? SP_TILE_N : TILE_N;
    p.mtiles = variant == V_SINGLE ? h->tc_mtiles : (h->tc_mtiles + 1) / 2;
    p.ntiles = (int32_t)((a.n + tile_n - 1) / tile_n);
    p.kchunks = variant == V_PAIR256 ? (h->tc_kpad + 255) / 256 : h->tc_kpad / BK;
    p.b_mn_major = a.layout == 0 ? 1 : 0;
    p.mgroups = 1;
    p.N = a.n;
    p.out = a.out;
    p.ldo = a.ldo;
    p.rqc = img_sec<float>(a.img, h->off_rqc);
    p.rqg = img_sec<float>(a.img, h->off_rqg);
    p.rqp = img_sec<float>(a.img, h->off_rqp);
    p.rtiles = h->tc_mtiles;
    p.x = static_cast<const uint8_t *>(a.x);
    p.ldx = a.ldx;
    p.sp_rptr = img_sec<int32_t>(a.img, h->off_sp_rptr);
    p.sp_res = img_sec<int32_t>(a.img, h->off_sp_res);
    p.debug = dbg;
    const bool out32 = h->out_dtype == 0 || h->out_dtype == 3;
    if (out32) {
        std::memset(&to, 0, sizeof(to));
        return launch_outk<OUT_32>(a, tw, tx, to, p, variant);
    }
    // 8-bit stores: TMA store of a swizzled smem tile (default; measured
    // fastest) or quad-transposed direct 32-bit stores (SI_K2_STORE=direct)
    static const bool use_direct = [] { const char *e = getenv("SI_K2_STORE"); return e && std::string(e) == "direct"; }();
    if (use_direct && a.ldo % 4 == 0 && (uintptr_t)a.out % 4 == 0) {
        std::memset(&to, 0, sizeof(to));
        return h->out_dtype == 2 ? launch_outk<OUT_U8_Q>(a, tw, tx, to, p, variant)
                                 : launch_outk<OUT_S8_Q>(a, tw, tx, to, p, variant);
    }
    const bool tma_ok = (a.ldo % 16 == 0) && ((uintptr_t)a.out % 16 == 0) &&
                        encode_2d(&to, a.out, (uint64_t)h->M, (uint64_t)a.n, (uint64_t)a.ldo, 128, COLS);
    if (!tma_ok) {
        std::memset(&to, 0, sizeof(to));
        return launch_outk<OUT_8_DIRECT>(a, tw, tx, to, p, variant);
    }
    return h->out_dtype == 2 ? launch_outk<OUT_U8_TMA>(a, tw, tx, to, p, variant)
                             : launch_outk<OUT_S8_TMA>(a, tw, tx, to, p, variant);
}
