// spmm_tcx.cu -- K2t: the X-stationary 2:4 sparse tensor-core SpMM.
//
// Same reference functions as K1/K2 (_acc_group_panel + _spmm_task_*,
// spmm.py:192-280).  Designed from the per-SM data budget of the dense pair
// kernel: there, every SM streams both the dense W tile and
// the X tile through shared memory, and the L2 -> SM stream (~11.6 TB/s chip
// wide) bounds the main loop.  K2t cuts both terms:
//
//  * W enters as the plan's 2:4 images (tcgen05.mma.sp.kind::i8): a 4-wide k
//    window of a 4x1-block group keeps its first two nonzero columns, so the
//    operand is half the bytes of dense W and the tensor pipe does half the
//    MACs.  Columns beyond two per window (~1 per 4-row group at K = 1024,
//    90% sparsity) form a second, tiny 2:4 operand per 256-row pair tile
//    over "slots" (plan.cpp build_tr_sections): a gather warp copies the
//    slot columns out of the resident X tile into a small K-major buffer and
//    the leader issues one or two extra sparse MMAs into the same
//    accumulator.  Every MAC is an exact integer MAC; the result is bit-equal
//    to the dense product.
//  * X stays resident: a CTA pair owns a tile of TN = 2*TNH tokens (token-
//    major X, K-major SWIZZLE_128B, TNH x K bytes per CTA, K <= 1024) and
//    walks all 256-row W tiles over it, so X crosses L2 -> SM once and W once
//    per token tile.  The tile rolls chunk by chunk into the next unit.
//
// Roles (18 warps): warps 0 and 15-17 TMA producers (stage i on producer
// i mod 4), warp 1 TMEM allocator + single-thread MMA issuer (leader CTA),
// warps 2-13 the epilogue (3 column groups x 4 TMEM lane quarters; the shared
// compiled _run_chain forms of k2_common.cuh), warp 14 the residual gather
// warp (also forwards the peer CTA's X arrival to the leader).  TMEM: two TN-column accumulators
// (the epilogue of tile i overlaps the MMAs of tile i+1) + metadata slots.
#include <cstdio>

#include "k2_common.cuh"

namespace {

// TMA issue: one issuing warp keeps about two boxes in flight (one box per
// ~311 ns whatever its size, tools/tma_bw.py prod), so the 12 KB W images
// need several producer warps to reach the ~133 GB/s per-SM TMA ceiling
constexpr int T_EPI_WARPS = 12;                  // 3 column groups x 4 TMEM lane quarters
constexpr int T_EPI_GROUPS = T_EPI_WARPS / 4;
constexpr int T_GATHER_WARP = 2 + T_EPI_WARPS;   // 14 (the gather warp that also forwards X arrival)
constexpr int T_NPROD = 4;                       // warp 0 + warps 15..17
constexpr int T_NGATHER = 3;                     // warps 14, 18, 19
constexpr int T_THREADS = 32 * (2 + T_EPI_WARPS + T_NPROD - 1 + T_NGATHER);
constexpr int T_IMG = 12288;                     // one (128-row tile, 128-k chunk) 2:4 image
constexpr int T_KMAX = 1024;
constexpr int T_XCHUNKS = T_KMAX / 128;
constexpr int T_STG = 128 * 32;                  // 8-bit staging: 128 m x 32 tokens per column group
constexpr int T_MAXPAIRS = 512;                  // residual MMA counts staged in smem (M <= 131072)

template <int TNH>
struct TGeom {
    static constexpr int TN = 2 * TNH;
    static constexpr int XCH = TNH * 128;        // one resident 128-k chunk of this CTA's tokens
    static constexpr int XBYTES = T_XCHUNKS * XCH;
    static constexpr int NCH = TN / 32;          // 32-token epilogue chunks per accumulator
    static constexpr uint32_t ECOL = 2 * TN;     // metadata TMEM columns (two 8-column slots)
    static_assert(TNH % 16 == 0, "token half must keep 1024-byte SW128 atoms and N % 16 == 0");
    static_assert(ECOL + 16 <= 512, "TMEM budget");
};

template <int OUTK>
constexpr int t_staged() { return (OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA) ? 2 * T_EPI_GROUPS * T_STG : 0; }
template <int MODE, int OUTK, int TNH>
constexpr int t_fixed()
{
    return TGeom<TNH>::XBYTES + TGeom<TNH>::XCH + t_staged<OUTK>() + table_bytes<MODE>() + 1024 + 512 + 4 * T_MAXPAIRS;
}
template <int MODE, int OUTK, int TNH>
constexpr int t_stages()
{
    constexpr int s = (SMEM_MAX - t_fixed<MODE, OUTK, TNH>()) / T_IMG;
    return s > 8 ? 8 : s;
}
template <int MODE, int OUTK, int TNH>
constexpr int t_smem() { return t_fixed<MODE, OUTK, TNH>() + t_stages<MODE, OUTK, TNH>() * T_IMG; }

struct TParams {
    const uint16_t *tr_k;    // [pairs][TR_SLOTS] activation column per residual slot
    const int32_t *tr_cnt;   // [pairs] residual MMAs (64 slots each)
    unsigned long long *trace;   // experiment (SI_K2T_TRACE): role timelines of pair 0, else null
};

// experiment timeline: role r of pair 0 appends (kind << 56 | globaltimer ns)
constexpr int T_TRACE_N = 8192;
__device__ __forceinline__ void trace_ev(unsigned long long *tr, int role, int &cnt, unsigned kind)
{
    if (!tr || cnt >= T_TRACE_N) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[role * T_TRACE_N + cnt++] = ((unsigned long long)kind << 56) | (t & 0x00FFFFFFFFFFFFFFull);
}

// Per-row epilogue constants of one accumulator tile (loaded one tile ahead:
// the epilogue is the critical role, so their global-load latency must not
// sit between two tiles).
struct RowK {
    int32_t adj;
    float s_in, cq, cp, gr;
};

template <int MODE>
__device__ __forceinline__ RowK load_rowk(int32_t m, const K2Params &P, const EpiParams &E)
{
    RowK k;
    const bool mok = m < E.M;
    k.adj = mok ? __ldg(E.adj + m) : 0;
    k.s_in = mok ? __ldg(E.scale_in + m) : 0.0f;
    k.cq = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqc + m) : 0.0f;
    k.cp = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqp + m) : 0.0f;
    k.gr = mok ? __ldg(P.rqg + m) : 1.0f;
    return k;
}

// Epilogue of one accumulator (this warp: 32 rows x the column group's
// chunks); per-chunk TMA stores from two alternating staging slots per group
// (a slot is rewritten only once the store issued from it two chunks earlier
// has read it).
template <int MODE, int OUTK, int TNH, typename Wait, typename Release>
__device__ __forceinline__ void epi_tile_t(uint32_t tmem_base, uint32_t tmem_col, int32_t row0, int64_t tok0,
                                           const CUtensorMap *tmap_o, const K2Params &P, const EpiParams &E,
                                           EpiWarp &W, const RowK &k, int &slot, Wait wait_full, Release release,
                                           unsigned long long *trc = nullptr, int trole = 0, int *tcnt = nullptr)
{
    using G = TGeom<TNH>;
    constexpr bool STAGED = (OUTK == OUT_U8_TMA || OUTK == OUT_S8_TMA);
    const int32_t m = row0 + W.q * 32 + W.lane;
    const bool mok = m < E.M;
    const bool proven = !(P.debug & 256) && __all_sync(0xffffffffu, k.gr >= 1.0f);
    const bool wide = __any_sync(0xffffffffu, k.gr >= 2.0f);
    const bool fast = !(P.debug & 256) && !wide && __all_sync(0xffffffffu, k.gr >= 0.0f);
    const float gm = proven ? (wide ? 2.0f : 1.0f) : (k.gr >= 1.0f ? 0.0f : fmaxf(k.gr, 0.0f));
    const float cq = proven ? k.cp : k.cq;
    wait_full();
    tc::tc_fence_after();
    const uint32_t lane_base = tmem_base + ((uint32_t)(W.q * 32) << 16) + tmem_col;
    uint8_t *const stg0 = W.stg;
#pragma unroll 1
    for (int ch = W.g; ch < G::NCH; ch += T_EPI_GROUPS) {
        if constexpr (STAGED) {
            // the store issued from this slot two chunks ago must have read it
            if (trc) trace_ev(trc, trole, *tcnt, 22);
            if (W.q == 2 && W.lane == 0) tc::tma_store_wait_read1();
            tc::named_bar_sync(1 + W.g, 128);
            if (trc) trace_ev(trc, trole, *tcnt, 23);
            W.stg = stg0 + slot * (T_EPI_GROUPS * T_STG);
        }
        if (!(P.debug & 1))
            epi_chunk<MODE, OUTK>(lane_base + ch * 32, m, mok, k.adj, k.s_in, cq, gm, fast, tok0 + ch * 32, 0, P, E,
                                  W);
        if constexpr (STAGED) {
            if (trc) trace_ev(trc, trole, *tcnt, 24);
            if (!(P.debug & 16384)) tc::fence_proxy_async_smem();   // 16384: experiment, no proxy fence
            if (trc) trace_ev(trc, trole, *tcnt, 26);
            tc::named_bar_sync(1 + W.g, 128);
            if (W.q == 2 && W.lane == 0 && !(P.debug & 8192)) {
                tc::tma_store_2d(tmap_o, W.stg, row0, (int32_t)(tok0 + ch * 32));
                tc::tma_store_commit();
            }
            if (trc) trace_ev(trc, trole, *tcnt, 25);
            slot ^= 1;
        }
    }
    W.stg = stg0;
    tc::tc_fence_before();
    __syncwarp();
    if (W.lane == 0) release();
}

template <int MODE, int OUTK, int TNH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(T_THREADS, 1)
k2t_kernel(const __grid_constant__ CUtensorMap tmap_s, const __grid_constant__ CUtensorMap tmap_r,
           const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_o, const K2Params P,
           const EpiParams E, const TParams T)
{
    using G = TGeom<TNH>;
    constexpr int STAGES = t_stages<MODE, OUTK, TNH>();
    static_assert(STAGES >= 3, "shared memory budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *xbuf = smem;                          // [T_XCHUNKS][TNH tok x 128 k] SW128 K-major
    uint8_t *rbuf = xbuf + G::XBYTES;              // gathered residual slots, same layout
    uint8_t *ring = rbuf + G::XCH;                 // [STAGES][T_IMG]
    uint8_t *staging = ring + STAGES * T_IMG;
    uint8_t *tables = staging + t_staged<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;              // [2]
    uint64_t *tempty = tfull + 2;                  // [2] (leader)
    uint64_t *xfull = tempty + 2;                  // [T_XCHUNKS] this CTA's X chunk landed
    uint64_t *xpeer = xfull + T_XCHUNKS;           // [T_XCHUNKS] (leader) the peer's X chunk landed
    uint64_t *xempty = xpeer + T_XCHUNKS;          // [T_XCHUNKS] MMAs + gathers of the unit done with it
    uint64_t *rfull = xempty + T_XCHUNKS;          // (leader) both CTAs' residual slots gathered
    uint64_t *rempty = rfull + 1;                  // residual MMAs retired
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rempty + 1);
    // per pair tile residual MMA counts, read by every role once per row tile:
    // staged in smem so no role waits on a global load there
    int32_t *s_rcnt = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(full) + 512);
    for (int i = threadIdx.x; i < P.mtiles; i += blockDim.x) s_rcnt[i] = __ldg(T.tr_cnt + i);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int units = P.ntiles * P.mgroups;
    unsigned long long *trc = (pair == 0) ? T.trace : nullptr;
    int tcnt = 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 2 * T_EPI_WARPS);
        }
        for (int c = 0; c < T_XCHUNKS; ++c) {
            tc::mbar_init(&xfull[c], 1);
            tc::mbar_init(&xpeer[c], 1);
            tc::mbar_init(&xempty[c], 1 + T_NGATHER);
        }
        tc::mbar_init(rfull, 2 * T_NGATHER);
        tc::mbar_init(rempty, 1);
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_s);
        tc::tma_prefetch_desc(&tmap_r);
        tc::tma_prefetch_desc(&tmap_x);
    }
    if (warp == 1) tc::tmem_alloc_2sm(tmem_slot, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto unit_range = [&](int unit, int &nt, int &m_lo, int &m_hi) {
        nt = unit / P.mgroups;
        const int mg = unit % P.mgroups;
        const int base = P.mtiles / P.mgroups, rem = P.mtiles % P.mgroups;
        m_lo = mg * base + (mg < rem ? mg : rem);
        m_hi = m_lo + base + (mg < rem ? 1 : 0);
    };
    // row tiles of a unit are walked from a pair-dependent start: pairs in
    // lock step would otherwise all read the same 12 KB W image at once and
    // pile onto the few L2 slices holding it
    auto row_tile = [&](int m_lo, int m_hi, int i) { return m_lo + (i + pair) % (m_hi - m_lo); };

    if (warp == 0 || (warp > T_GATHER_WARP && warp < T_GATHER_WARP + T_NPROD)) {
        {   // whole warp, one elected lane issues (tcw::)
            // ---------------- TMA producers (both CTAs): W images onto the leader's
            // barriers, this CTA's X chunks onto its own
            const int prod = warp == 0 ? 0 : warp - T_GATHER_WARP;
            const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
            int stage = 0, it = 0;
            uint32_t phase = 0, xphase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, m_lo, m_hi;
                unit_range(unit, nt, m_lo, m_hi);
                const int tok = nt * G::TN + TNH * (int)rank;
                for (int i = 0; i < m_hi - m_lo; ++i) {
                    const int mt = row_tile(m_lo, m_hi, i);
                    const int nres = (P.debug & 1024) ? 0 : s_rcnt[mt];   // 1024: experiment, no residual stage
                    const int nst = P.kchunks + (nres ? 1 : 0);
                    for (int s = 0; s < nst; ++s, ++it) {
                        if (it % T_NPROD == prod) {
                            if (i == 0 && s < P.kchunks && !(P.debug & 8)) {   // 8: experiment, no X loads
                                tc::mbar_spin(&xempty[s], xphase ^ 1);
                                tcw::mbar_expect_tx(&xfull[s], G::XCH);
                                // (debug 4: every unit loads token tile 0 -- experiment)
                                tcw::tma_load_2d(xbuf + s * G::XCH, &tmap_x, &xfull[s], s * 128,
                                                (P.debug & 4) ? TNH * (int)rank : tok);
                            }
                            tc::mbar_spin(&empty[stage], phase ^ 1);
                            if (lane == 0) trace_ev(trc, 2 * prod + (int)rank, tcnt, 10 + prod);
                            if (rank == 0) tcw::mbar_expect_tx(&full[stage], 2 * T_IMG);
                            // (debug 2: every row tile loads pair tile 0's images -- experiment)
                            const int rt = 2 * ((P.debug & 2) ? 0 : mt) + (int)rank;
                            if (s < P.kchunks)
                                tcw::tma_load_2d_2sm(ring + stage * T_IMG, &tmap_s, full0 + 8 * stage, 0,
                                                    (rt * P.kchunks + s) * (T_IMG / 128));
                            else
                                tcw::tma_load_2d_2sm(ring + stage * T_IMG, &tmap_r, full0 + 8 * stage, 0,
                                                    rt * (T_IMG / 128));
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                xphase ^= 1;
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && (P.debug & 4096)) {
            // experiment (with 2048 | 1024 | 8): minimal consumer, wait full -> release
            int stage = 0;
            uint32_t phase = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, m_lo, m_hi;
                unit_range(unit, nt, m_lo, m_hi);
                for (int q = 0; q < (m_hi - m_lo) * P.kchunks; ++q) {
                    tc::mbar_wait(&full[stage], phase);
                    tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        } else if (rank == 0) {
            // ---------------- MMA issuer: leader CTA, whole warp, one elected lane issues, M256 x N(TN) x K64 sparse
            const uint32_t idesc = tc::idesc_i8(256, G::TN, 0, 0) | (1u << 2);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0, xphase = 0, rphase = 0, eslot = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, m_lo, m_hi;
                unit_range(unit, nt, m_lo, m_hi);
                for (int i = 0; i < m_hi - m_lo; ++i) {
                    const int mt = row_tile(m_lo, m_hi, i);
                    const int nres = (P.debug & 1024) ? 0 : s_rcnt[mt];   // 1024: experiment, no residual stage
                    if (!(P.debug & 2048)) tc::mbar_spin(&tempty[acc], acc_phase ^ 1);
                    if (lane == 0) trace_ev(trc, 8, tcnt, 2);
                    tc::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * G::TN;
                    for (int kc = 0; kc < P.kchunks; ++kc) {
                        if (i == 0 && !(P.debug & 8)) {
                            tc::mbar_spin(&xfull[kc], xphase);
                            tc::mbar_spin_cluster(&xpeer[kc], xphase);
                        }
                        tc::mbar_spin(&full[stage], phase);
                        if (lane == 0) trace_ev(trc, 8, tcnt, 1);
                        tc::tc_fence_after();
                        const uint32_t a_addr = tc::smem_u32(ring + stage * T_IMG);
                        const uint32_t b_addr = tc::smem_u32(xbuf + kc * G::XCH);
                        const uint32_t e_tmem = tmem_base + G::ECOL + 8 * eslot;
                        if (!(P.debug & 32)) {   // 32: experiment, no metadata copies
                            tcw::tmem_cp_128x128b_2sm(e_tmem, tc::smem_desc(a_addr + 8192, 2048, 128, 0));
                            tcw::tmem_cp_128x128b_2sm(e_tmem + 4, tc::smem_desc(a_addr + 10240, 2048, 128, 0));
                        }
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            const uint64_t adesc = tc::smem_desc(a_addr + 256 * j, 128, 512, 0);
                            const uint64_t bdesc = tc::smem_desc_sw128(b_addr + 64 * j, 16, 1024);
                            if (!(P.debug & 16))
                                tcw::mma_sp_i8_2sm(d_tmem, adesc, bdesc, e_tmem + 4 * j, idesc, (kc | j) ? 1u : 0u);
                        }
                        tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                        if (i == m_hi - m_lo - 1) tcw::mma_commit_2sm_mc(&xempty[kc], 0x3);
                        eslot ^= 1;
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (nres) {
                        // residual slots: B from the gathered buffer of both CTAs
                        tc::mbar_spin(&full[stage], phase);
                        if (lane == 0) trace_ev(trc, 8, tcnt, 1);
                        tc::mbar_spin_cluster(rfull, rphase);
                        if (lane == 0) trace_ev(trc, 8, tcnt, 3);
                        tc::tc_fence_after();
                        const uint32_t a_addr = tc::smem_u32(ring + stage * T_IMG);
                        const uint32_t b_addr = tc::smem_u32(rbuf);
                        const uint32_t e_tmem = tmem_base + G::ECOL + 8 * eslot;
                        tcw::tmem_cp_128x128b_2sm(e_tmem, tc::smem_desc(a_addr + 8192, 2048, 128, 0));
                        if (nres > 1)
                            tcw::tmem_cp_128x128b_2sm(e_tmem + 4, tc::smem_desc(a_addr + 10240, 2048, 128, 0));
                        for (int j = 0; j < nres; ++j) {
                            const uint64_t adesc = tc::smem_desc(a_addr + 256 * j, 128, 512, 0);
                            const uint64_t bdesc = tc::smem_desc_sw128(b_addr + 64 * j, 16, 1024);
                            if (!(P.debug & 16) && !(P.debug & 512))
                                tcw::mma_sp_i8_2sm(d_tmem, adesc, bdesc, e_tmem + 4 * j, idesc, 1u);
                        }
                        tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                        tcw::mma_commit_2sm_mc(rempty, 0x3);
                        rphase ^= 1;
                        eslot ^= 1;
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    tcw::mma_commit_2sm_mc(&tfull[acc], 0x3);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
                xphase ^= 1;
            }
        }
    } else if (P.debug & 2048) {
        // experiment: epilogue and gather warps idle; the leader's accumulator
        // barriers are released once per tile by the MMA thread itself (below)
    } else if (warp == T_GATHER_WARP || warp >= T_GATHER_WARP + T_NPROD) {
        // ---------------- residual gather (both CTAs, T_NGATHER warps): slot s
        // of the residual operand = X column tr_k[s] of this CTA's tokens,
        // copied from the resident SW128 X tile into the same layout
        const int gi = warp == T_GATHER_WARP ? 0 : warp - (T_GATHER_WARP + T_NPROD) + 1;
        const uint32_t rfull0 = tc::mapa(tc::smem_u32(rfull), 0);
        const uint32_t xpeer0 = tc::mapa(tc::smem_u32(xpeer), 0);
        uint32_t xphase = 0, rphase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            int nt, m_lo, m_hi;
            unit_range(unit, nt, m_lo, m_hi);
            for (int kc = 0; kc < P.kchunks && !(P.debug & 8); ++kc) {
                tc::mbar_wait(&xfull[kc], xphase);
                if (rank == 1 && gi == 0 && lane == 0) tc::mbar_arrive_cluster(xpeer0 + 8 * kc);
            }
            for (int i = 0; i < m_hi - m_lo; ++i) {
                    const int mt = row_tile(m_lo, m_hi, i);
                const int nres = (P.debug & 1024) ? 0 : s_rcnt[mt];   // 1024: experiment, no residual stage
                if (!nres) continue;
                const int w4 = nres * 16;                  // 4-slot words per token (16 or 32)
                const int j4 = lane % w4, tstep = 32 / w4;
                // this lane's 4 slots: source offsets inside the X tile
                uint32_t kofs[4], kx[4];
                const uint16_t *kp = T.tr_k + (size_t)mt * TR_SLOTS + 4 * j4;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t k = __ldg(kp + b);
                    kofs[b] = (k >> 7) * G::XCH + (k & 15);
                    kx[b] = (k >> 4) & 7;
                }
                tc::mbar_wait(rempty, rphase ^ 1);
                if (lane == 0 && gi == 0) trace_ev(trc, 10 + (int)rank, tcnt, 30);
                if (!(P.debug & 512)) {
#pragma unroll 4
                    for (int t = lane / w4 + tstep * gi; t < TNH; t += tstep * T_NGATHER) {
                        const uint32_t r8 = (uint32_t)(t & 7);
                        const uint32_t rowb = (uint32_t)(t >> 3) * 1024 + r8 * 128;
                        uint32_t word = 0;
#pragma unroll
                        for (int b = 0; b < 4; ++b)
                            word |= (uint32_t)xbuf[rowb + ((kx[b] ^ r8) << 4) + kofs[b]] << (8 * b);
                        *reinterpret_cast<uint32_t *>(rbuf + rowb + ((((uint32_t)j4 >> 2) ^ r8) << 4) +
                                                      4 * (j4 & 3)) = word;
                    }
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (gi == 0) trace_ev(trc, 10 + (int)rank, tcnt, 31);
                    tc::mbar_arrive_cluster(rfull0);
                }
                rphase ^= 1;
            }
            // every read of this unit's X tile is done: second arrival on the chunks
            __syncwarp();
            if (lane == 0)
                for (int kc = 0; kc < P.kchunks; ++kc) tc::mbar_arrive(&xempty[kc]);
            xphase ^= 1;
        }
    } else {
        // ---------------- epilogue warps (both CTAs; each reads its own TMEM half)
        EpiWarp W = make_epi_warp<MODE, T_EPI_WARPS>(warp, lane, staging, tables, E);
        W.stg = staging + W.g * T_STG;
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        const int32_t mrow = 128 * (int)rank + W.q * 32 + lane;   // this lane's row within a pair tile
        int acc = 0, slot = 0;
        uint32_t acc_phase = 0;
        // (unit, row tile) sequence of this pair, walked one tile ahead for the row constants
        int unit = pair, i = 0, nt = 0, m_lo = 0, m_hi = 0;
        if (unit < units) unit_range(unit, nt, m_lo, m_hi);
        RowK k = load_rowk<MODE>(row_tile(m_lo, m_hi, 0) * 256 + mrow, P, E);
        while (unit < units) {
            const int mt = row_tile(m_lo, m_hi, i);
            const int cur_nt = nt;
            // advance to the next tile and prefetch its row constants
            int nunit = unit, ni = i + 1, nnt = nt, nlo = m_lo, nhi = m_hi;
            if (ni == m_hi - m_lo) {
                nunit += npairs;
                ni = 0;
                if (nunit < units) unit_range(nunit, nnt, nlo, nhi);
            }
            const RowK kn = nunit < units ? load_rowk<MODE>(row_tile(nlo, nhi, ni) * 256 + mrow, P, E) : k;
            const uint32_t te = tempty0 + 8 * acc;
            uint64_t *tf = &tfull[acc];
            const uint32_t ph = acc_phase;
            const bool tw = (warp == 2 && lane == 0);
            epi_tile_t<MODE, OUTK, TNH>(tmem_base, acc * G::TN, mt * 256 + 128 * (int)rank, (int64_t)cur_nt * G::TN,
                                        &tmap_o, P, E, W, k, slot,
                                        [&, tf, ph] { tc::mbar_wait(tf, ph); if (tw) trace_ev(trc, 12 + (int)rank, tcnt, 20); },
                                        [&, te] { if (tw) trace_ev(trc, 12 + (int)rank, tcnt, 21); tc::mbar_arrive_cluster(te); },
                                        tw ? trc : nullptr, 12 + (int)rank, &tcnt);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
            k = kn;
            unit = nunit; i = ni; nt = nnt; m_lo = nlo; m_hi = nhi;
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

constexpr int T_TNH = 112;

template <int MODE, int OUTK>
int k2t_launch_mode(const SpmmArgs &a, const CUtensorMap &ts, const CUtensorMap &tr, const CUtensorMap &tx,
                    const CUtensorMap &to, K2Params p, const TParams &T)
{
    EpiParams E = make_epi(a.h, a.img, a.sides, a.n);
    cudaStream_t st = (cudaStream_t)a.stream;
    const int npairs = num_sms() / 2;
    auto kern = k2t_kernel<MODE, OUTK, T_TNH>;
    constexpr int smem = t_smem<MODE, OUTK, T_TNH>();
    static_assert(smem <= SMEM_MAX, "shared memory budget");
    static bool attr = false;
    if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); attr = true; }
    p.mgroups = pick_mgroups(p.mtiles, p.ntiles, npairs);
    const long units = (long)p.ntiles * p.mgroups;
    const int pairs = units < npairs ? (int)units : npairs;
    kern<<<2 * pairs, T_THREADS, smem, st>>>(ts, tr, tx, to, p, E, T);
    return (int)cudaGetLastError();
}

template <int OUTK>
int k2t_launch_outk(const SpmmArgs &a, const CUtensorMap &ts, const CUtensorMap &tr, const CUtensorMap &tx,
                    const CUtensorMap &to, const K2Params &p, const TParams &T)
{
    switch (a.h->epi_mode) {
    case EPI_S32: return k2t_launch_mode<EPI_S32, OUTK>(a, ts, tr, tx, to, p, T);
    case EPI_DEQ_F32: return k2t_launch_mode<EPI_DEQ_F32, OUTK>(a, ts, tr, tx, to, p, T);
    case EPI_REQUANT: return k2t_launch_mode<EPI_REQUANT, OUTK>(a, ts, tr, tx, to, p, T);
    case EPI_REQUANT_LUT: return k2t_launch_mode<EPI_REQUANT_LUT, OUTK>(a, ts, tr, tx, to, p, T);
    case EPI_DEQ_TABLE: return k2t_launch_mode<EPI_DEQ_TABLE, OUTK>(a, ts, tr, tx, to, p, T);
    default: return k2t_launch_mode<EPI_GENERIC, OUTK>(a, ts, tr, tx, to, p, T);
    }
}

}  // namespace

bool k2t_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx)
{
    if (layout != 1 || !h->tr_ok || h->tc_kpad > T_KMAX || h->tc_mtiles < 2) return false;
    if ((h->tc_mtiles + 1) / 2 > T_MAXPAIRS) return false;
    if (n < 1 || n > (int64_t)INT32_MAX - 2 * T_TNH) return false;
    if (((uintptr_t)x) % 16 || ldx % 16 || h->K % 16) return false;
    return true;
}

int k2t_launch(const SpmmArgs &a)
{
    const SiImage *h = a.h;
    static const int dbg = env_int("SI_K2_DEBUG", 0);
    const int kch = h->tc_kpad / 128;
    const int pt_n = (h->tc_mtiles + 1) / 2;
    CUtensorMap ts, tr, tx, to;
    // (SI_K2T_SWZ=1: experiment only -- W images through SWIZZLE_128B boxes,
    // wrong results, to time the TMA path)
    static const CUtensorMapSwizzle iswz = env_int("SI_K2T_SWZ", 0) ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    bool ok = encode_2d(&ts, img_sec<uint8_t>(a.img, h->off_sp_img), 128, (uint64_t)2 * pt_n * kch * (T_IMG / 128), 128,
                        128, T_IMG / 128, iswz) &&
              encode_2d(&tr, img_sec<uint8_t>(a.img, h->off_tr_img), 128, (uint64_t)2 * pt_n * (T_IMG / 128), 128, 128,
                        T_IMG / 128, iswz) &&
              encode_2d(&tx, a.x, (uint64_t)h->K, (uint64_t)a.n, (uint64_t)a.ldx, 128, T_TNH);
    if (!ok) return (int)cudaErrorInvalidValue;
    K2Params p;
    std::memset(&p, 0, sizeof(p));
    p.mtiles = pt_n;
    p.ntiles = (int32_t)((a.n + 2 * T_TNH - 1) / (2 * T_TNH));
    p.kchunks = kch;
    p.b_mn_major = 0;
    p.mgroups = 1;
    p.N = a.n;
    p.out = a.out;
    p.ldo = a.ldo;
    p.rqc = img_sec<float>(a.img, h->off_rqc);
    p.rqg = img_sec<float>(a.img, h->off_rqg);
    p.rqp = img_sec<float>(a.img, h->off_rqp);
    p.x = static_cast<const uint8_t *>(a.x);
    p.ldx = a.ldx;
    p.debug = dbg;
    TParams T;
    T.tr_k = img_sec<uint16_t>(a.img, h->off_tr_k);
    T.tr_cnt = img_sec<int32_t>(a.img, h->off_tr_cnt);
    T.trace = nullptr;
    static const char *trace_path = getenv("SI_K2T_TRACE");   // experiment: dump pair 0's role timelines
    static unsigned long long *trace_buf = nullptr;
    const size_t trace_bytes = (size_t)16 * T_TRACE_N * 8;
    if (trace_path) {
        if (!trace_buf) cudaMalloc(&trace_buf, trace_bytes);
        cudaMemsetAsync(trace_buf, 0, trace_bytes, (cudaStream_t)a.stream);
        T.trace = trace_buf;
    }
    struct TraceDump {
        const char *path; unsigned long long *buf; size_t bytes; cudaStream_t st;
        ~TraceDump()
        {
            if (!path || !buf) return;
            std::string hb(bytes, '\0');
            cudaStreamSynchronize(st);
            cudaMemcpy(&hb[0], buf, bytes, cudaMemcpyDeviceToHost);
            if (FILE *f = fopen(path, "wb")) { fwrite(hb.data(), 1, bytes, f); fclose(f); }
        }
    } dump{trace_path, trace_buf, trace_bytes, (cudaStream_t)a.stream};
    const bool out32 = h->out_dtype == 0 || h->out_dtype == 3;
    if (out32) {
        std::memset(&to, 0, sizeof(to));
        return k2t_launch_outk<OUT_32>(a, ts, tr, tx, to, p, T);
    }
    // 8-bit stores: TMA store of a swizzled smem tile (default) or quad-
    // transposed direct 32-bit stores (SI_K2_STORE=direct)
    static const bool use_direct = [] { const char *e = getenv("SI_K2_STORE"); return e && std::string(e) == "direct"; }();
    if (use_direct && a.ldo % 4 == 0 && (uintptr_t)a.out % 4 == 0) {
        std::memset(&to, 0, sizeof(to));
        return h->out_dtype == 2 ? k2t_launch_outk<OUT_U8_Q>(a, ts, tr, tx, to, p, T)
                                 : k2t_launch_outk<OUT_S8_Q>(a, ts, tr, tx, to, p, T);
    }
    const bool tma_ok = (a.ldo % 16 == 0) && ((uintptr_t)a.out % 16 == 0) &&
                        encode_2d(&to, a.out, (uint64_t)h->M, (uint64_t)a.n, (uint64_t)a.ldo, 128, 32);
    if (!tma_ok) {
        std::memset(&to, 0, sizeof(to));
        return k2t_launch_outk<OUT_8_DIRECT>(a, ts, tr, tx, to, p, T);
    }
    return h->out_dtype == 2 ? k2t_launch_outk<OUT_U8_TMA>(a, ts, tr, tx, to, p, T)
                             : k2t_launch_outk<OUT_S8_TMA>(a, ts, tr, tx, to, p, T);
}
