// spmm_xs.cu -- K3: the X-stationary 2:4-sparse tensor-core SpMM.
//
// Same reference functions as K1/K2 (_acc_group_panel + _spmm_task_*,
// spmm.py:192-280): out[n, m] = epilogue(sum_k W[m,k] x[k,n] + adj[m]).
//
// Why this shape (tools/mma_rate.py, profiles/r02_*):
//  * Dense-expanded W (K2) multiplies 10x the algorithmic MACs at 90% block
//    sparsity and streams both operand tiles through L2 -> SM (2.15 GB for
//    config 5b); it is bound there and by the dense MMA.
//  * W enters as the plan's 2:4 images (tcgen05.mma.sp.kind::i8, measured
//    at 2x the dense rate on B200: M256 x N256 x K64 per ~130-150 clk): a
//    4-wide k window of a 4x1-block group keeps its first two nonzero
//    columns.  Columns beyond two per window (~1 per group at K = 1024, 90%)
//    form a small second 2:4 operand per 256-row pair tile over "slots"
//    (plan.cpp build_tr_sections): the gather warp copies those activation
//    columns out of the resident X tile, and the MMA warp issues one or two
//    extra sparse MMAs into the same accumulator.  Every MAC is an exact
//    integer MAC, so the result is bit-equal to the dense product.
//  * X stays resident: a CTA pair owns 2 x 112 tokens of token-major X
//    (K-major SWIZZLE_128B, 112 x K bytes per CTA, K <= 1024) and walks its
//    unit's 256-row W tiles over it; X crosses L2 -> SM once, W once per
//    token tile.  The tile rolls chunk by chunk into the next unit.
//  * Issue path: a single thread's tcgen05 instructions serialise (~130-150
//    clk per MMA regardless of N, tools/mma_rate.py), so each 128-k stage is
//    one tcgen05.cp (both metadata tiles, 128x256b) + two MMAs with
//    descriptors formed by adding offsets to precomputed bases.
//
// Roles (20 warps, 96 registers each): warps 0, 14 and 17 TMA producers
// (stage i on producer i mod 3), warp 1 TMEM allocator + MMA issuer (leader
// CTA), warps 2-13 the epilogue (3 token-column groups x 4 TMEM lane
// quarters; the compiled _run_chain forms of k2_common.cuh), warps 15, 16,
// 18, 19 the residual gather (the first also forwards this CTA's X-chunk
// arrivals to the leader).  8-bit outputs leave per warp: each warp stages its own 32
// rows x 32 tokens (1 KB, no cross-warp barrier) and TMA-stores them.  TMEM: two 224-column
// accumulators (the epilogue of tile i overlaps the MMAs of tile i+1) + two
// 8-column metadata slots.
#include <cstdio>

#include "k2_common.cuh"

namespace {

// Experiment switches exist only in experiment builds (SI_BUILD_DEFS=
// -DSI_EXPERIMENTS, a separate library selected with SI_LIB); the product
// library compiles every XS_EXP(...) to false.
#ifdef SI_EXPERIMENTS
#define XS_EXP(bit) ((X.exp & (bit)) != 0)
#else
#define XS_EXP(bit) false
#endif
enum XsExp : int32_t {
    XE_NO_EPI = 1,      // epilogue: wait and release only
    XE_NO_GATHER = 2,   // gather: handshakes only
    XE_NO_MMA = 4,      // MMA warp: commits only
    XE_W_TILE0 = 8,     // every W load reads pair tile 0 (L2 hot-spot test)
    XE_NO_STORE = 16,   // epilogue: no TMA stores
    XE_EPI_LDONLY = 32, // epilogue: TMEM loads + release only (no math, staging, stores)
};

constexpr int XS_TNH = 112;                          // tokens per CTA
constexpr int XS_TN = 2 * XS_TNH;                    // MMA N (pair)
constexpr int XS_KMAX = 1024;
constexpr int XS_XCHUNKS = XS_KMAX / 128;
constexpr int XS_XCH = XS_TNH * 128;                 // one resident 128-k chunk of this CTA's tokens
constexpr int XS_XBYTES = XS_XCHUNKS * XS_XCH;
constexpr int XS_IMG = 12288;                        // one (128-row tile, 128-k chunk) 2:4 image
constexpr int XS_EPI_WARPS = 12;
constexpr int XS_EPI_GROUPS = XS_EPI_WARPS / 4;
constexpr int XS_NCH = XS_TN / 32;                   // 32-token epilogue chunks per accumulator (7)
// Warp placement: a warp's scheduler (SMSP) is warp % 4.  The MMA issuer
// (warp 1, SMSP 1) is the critical role: its tcgen05 issue slows when the
// warps beside it keep the scheduler busy, so no gather warp shares SMSP 1
// and the producer there (17) sleeps in try_wait instead of spinning.
constexpr int XS_NPROD = 3;                          // warps 0, 14, 17
constexpr int XS_PROD1_WARP = 2 + XS_EPI_WARPS;      // 14
constexpr int XS_PROD2_WARP = 17;
constexpr int XS_NGATHER = 4;                        // warps 15, 16, 18, 19
constexpr int XS_THREADS = 32 * 20;                  // 20 warps: 96 registers each
__device__ __forceinline__ int xs_gather_index(int warp)
{
    return warp == 15 ? 0 : warp == 16 ? 1 : warp == 18 ? 2 : warp == 19 ? 3 : -1;
}
constexpr int XS_WSTG = 32 * 32;                     // 8-bit staging slot of one warp: 32 tokens x 32 m
constexpr int XS_MAXPAIRS = 512;                     // residual MMA counts staged in smem (M <= 131072)
constexpr uint32_t XS_ECOL = 2 * XS_TN;              // metadata slots: TMEM columns 448..463
static_assert(XS_ECOL + 16 <= 512, "TMEM budget");
static_assert(XS_TNH % 8 == 0, "token half must keep whole 8-row SW128 atoms");

template <int OUTK>
constexpr int xs_staged() { return (OUTK == OUT_U8_W || OUTK == OUT_S8_W) ? XS_EPI_WARPS * XS_WSTG : 0; }
template <int MODE, int OUTK>
constexpr int xs_fixed()
{
    // + 1024 alignment slack, 1024 barriers, the per-pair-tile residual counts
    return XS_XBYTES + XS_XCH + xs_staged<OUTK>() + table_bytes<MODE>() + 1024 + 1024 + 4 * XS_MAXPAIRS;
}
template <int MODE, int OUTK>
constexpr int xs_stages()
{
    constexpr int s = (SMEM_MAX - xs_fixed<MODE, OUTK>()) / XS_IMG;
    return s > 8 ? 8 : s;
}
template <int MODE, int OUTK>
constexpr int xs_smem() { return xs_fixed<MODE, OUTK>() + xs_stages<MODE, OUTK>() * XS_IMG; }

struct XsParams {
    int32_t ptiles;          // 256-row pair tiles
    int32_t ntiles;          // 224-token tiles
    int32_t kchunks;         // 128-k chunks (<= 8)
    int32_t mgroups;         // pair tiles of a token tile split into this many work units
    const uint16_t *tr_k;    // [ptiles][TR_SLOTS] activation column per residual slot
    const int32_t *tr_cnt;   // [ptiles] residual MMAs (64 slots each)
    int32_t exp;             // experiment switches (XsExp; experiment builds only)
    unsigned long long *trace;   // experiment builds: pair 0's role timelines, else null
};

// experiment builds only: (event << 56 | globaltimer ns) per role of pair 0
#ifdef SI_EXPERIMENTS
constexpr int XS_TRACE_N = 4096;
__device__ __forceinline__ void xs_trace(const XsParams &X, int role, int &cnt, unsigned ev)
{
    if (!X.trace || cnt >= XS_TRACE_N || (blockIdx.x >> 1) != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    X.trace[role * XS_TRACE_N + cnt++] = ((unsigned long long)ev << 56) | (t & 0x00FFFFFFFFFFFFFFull);
}
#define XS_TRACE(role, cnt, ev) xs_trace(X, role, cnt, ev)
#else
#define XS_TRACE(role, cnt, ev) ((void)0)
#endif

// per-row epilogue constants of one accumulator tile, loaded a tile ahead
struct XsRow {
    int32_t adj;
    float s_in, cq, cp, gr;
};

template <int MODE>
__device__ __forceinline__ XsRow xs_row(int32_t m, const K2Params &P, const EpiParams &E)
{
    XsRow k;
    const bool mok = m < E.M;
    k.adj = mok ? __ldg(E.adj + m) : 0;
    k.s_in = mok ? __ldg(E.scale_in + m) : 0.0f;
    k.cq = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqc + m) : 0.0f;
    k.cp = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqp + m) : 0.0f;
    k.gr = mok ? __ldg(P.rqg + m) : 1.0f;
    return k;
}

// Epilogue of one accumulator for one warp: its 32 rows x the column group's
// 32-token chunks (g, g+3, g+6), each staged in this warp's own 1 KB tile and
// TMA-stored by its lane 0 (the tile is rewritten once that store has read
// it).  The accumulator is released once this warp's last chunk is in
// registers.
template <int MODE, int OUTK, typename Release>
__device__ __forceinline__ void xs_epi_tile(uint32_t lane_base, int32_t row0, int64_t tok0,
                                            const CUtensorMap *tmap_o, const K2Params &P, const EpiParams &E,
                                            EpiWarp &W, const XsRow &k, Release release,
                                            const XsParams &X)
{
    if (XS_EXP(XE_NO_EPI)) {
        tc::tc_fence_before();
        __syncwarp();
        if (W.lane == 0) release();
        return;
    }
    if (XS_EXP(XE_EPI_LDONLY)) {
        uint32_t acc = 0;
#pragma unroll 1
        for (int ch = W.g; ch < XS_NCH; ch += XS_EPI_GROUPS) {
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32(lane_base + ch * 32, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= r[j];
        }
        tc::tc_fence_before();
        __syncwarp();
        if (W.lane == 0) release();
        if (acc == 0x9e3779b9u && W.lane == 33) *reinterpret_cast<uint32_t *>(P.out) = acc;
        return;
    }
    constexpr bool STAGED = (OUTK == OUT_U8_W || OUTK == OUT_S8_W);
    const int32_t m = row0 + W.q * 32 + W.lane;
    const bool mok = m < E.M;
    const bool proven = __all_sync(0xffffffffu, k.gr >= 1.0f);
    const bool wide = __any_sync(0xffffffffu, k.gr >= 2.0f);
    const bool fast = !wide && __all_sync(0xffffffffu, k.gr >= 0.0f);
    const float gm = proven ? (wide ? 2.0f : 1.0f) : (k.gr >= 1.0f ? 0.0f : fmaxf(k.gr, 0.0f));
    const float cq = proven ? k.cp : k.cq;
    auto rel = [&]() {
        tc::tc_fence_before();
        __syncwarp();
        if (W.lane == 0) release();
    };
#pragma unroll 1
    for (int ch = W.g; ch < XS_NCH; ch += XS_EPI_GROUPS) {
        const bool last = ch + XS_EPI_GROUPS >= XS_NCH;
        if constexpr (STAGED) {
            // this warp's previous store must have read its staging tile
            if (W.lane == 0) tc::tma_store_wait_read0();
            __syncwarp();
        }
        if (last)
            epi_chunk<MODE, OUTK>(lane_base + ch * 32, m, mok, k.adj, k.s_in, cq, gm, fast, tok0 + ch * 32, 0, P, E,
                                  W, rel);
        else
            epi_chunk<MODE, OUTK>(lane_base + ch * 32, m, mok, k.adj, k.s_in, cq, gm, fast, tok0 + ch * 32, 0, P, E,
                                  W);
        if constexpr (STAGED) {
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (W.lane == 0 && !XS_EXP(XE_NO_STORE)) {
                tc::tma_store_2d(tmap_o, W.stg, row0 + W.q * 32, (int32_t)(tok0 + ch * 32));
                tc::tma_store_commit();
            }
        }
    }
}

template <int MODE, int OUTK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(XS_THREADS, 1)
k3_kernel(const __grid_constant__ CUtensorMap tmap_s, const __grid_constant__ CUtensorMap tmap_r,
          const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_o, const K2Params P,
          const EpiParams E, const XsParams X)
{
    constexpr int STAGES = xs_stages<MODE, OUTK>();
    static_assert(STAGES >= 3, "shared memory budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *xbuf = smem;                          // [XS_XCHUNKS][112 tok x 128 k] SW128 K-major
    uint8_t *rbuf = xbuf + XS_XBYTES;              // gathered residual slots, same layout
    uint8_t *ring = rbuf + XS_XCH;                 // [STAGES][XS_IMG]
    uint8_t *staging = ring + STAGES * XS_IMG;
    uint8_t *tables = staging + xs_staged<OUTK>();
    uint64_t *full = reinterpret_cast<uint64_t *>(tables + table_bytes<MODE>());
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;              // [2]
    uint64_t *tempty = tfull + 2;                  // [2] (leader)
    uint64_t *xfull = tempty + 2;                  // [XS_XCHUNKS] this CTA's X chunk landed
    uint64_t *xpeer = xfull + XS_XCHUNKS;          // [XS_XCHUNKS] (leader) the peer's X chunk landed
    uint64_t *xempty = xpeer + XS_XCHUNKS;         // [XS_XCHUNKS] MMAs + gather of the unit done with it
    uint64_t *rfull = xempty + XS_XCHUNKS;         // (leader) both CTAs' residual slots gathered
    uint64_t *rempty = rfull + 1;                  // residual MMAs retired
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rempty + 1);
    // per pair tile residual MMA counts, read by every role once per row tile
    int32_t *s_rcnt = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(full) + 1024);
    tc::pdl_wait();                 // X may come from the previous kernel (PDL launch)
    tc::pdl_launch_dependents();
    for (int i = threadIdx.x; i < X.ptiles; i += blockDim.x) s_rcnt[i] = __ldg(X.tr_cnt + i);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int units = X.ntiles * X.mgroups;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], 1);
            tc::mbar_init(&tempty[a], 2 * XS_EPI_WARPS);
        }
        for (int c = 0; c < XS_XCHUNKS; ++c) {
            tc::mbar_init(&xfull[c], 1);
            tc::mbar_init(&xpeer[c], 1);
            tc::mbar_init(&xempty[c], 1 + XS_NGATHER);   // the unit's last MMA commit + the gather warps
        }
        tc::mbar_init(rfull, 2 * XS_NGATHER);
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

    auto unit_range = [&](int unit, int &nt, int &p_lo, int &p_hi) {
        nt = unit / X.mgroups;
        const int mg = unit % X.mgroups;
        const int base = X.ptiles / X.mgroups, rem = X.ptiles % X.mgroups;
        p_lo = mg * base + (mg < rem ? mg : rem);
        p_hi = p_lo + base + (mg < rem ? 1 : 0);
    };
    // a unit's pair tiles are walked from a pair-dependent start, so pairs
    // in lock step do not all read the same W image at once
    auto pair_tile = [&](int p_lo, int p_hi, int i) { return p_lo + (i + pair) % (p_hi - p_lo); };

    if (warp == 0 || warp == XS_PROD1_WARP || warp == XS_PROD2_WARP) {
        // ---------------- TMA producers (both CTAs): W images onto the leader's
        // barriers (stage i on producer i mod 3), this CTA's X chunks onto its own
        const int prod = warp == 0 ? 0 : warp == XS_PROD1_WARP ? 1 : 2;
        const uint32_t full0 = tc::mapa(tc::smem_u32(full), 0);
        int stage = 0, it = 0;
        uint32_t phase = 0, xphase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            int nt, p_lo, p_hi;
            unit_range(unit, nt, p_lo, p_hi);
            const int tok = nt * XS_TN + XS_TNH * (int)rank;
            for (int i = 0; i < p_hi - p_lo; ++i) {
                const int pt = pair_tile(p_lo, p_hi, i);
                const int nst = X.kchunks + (s_rcnt[pt] ? 1 : 0);
                for (int s = 0; s < nst; ++s, ++it) {
                    if (it % XS_NPROD != prod) {
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if (i == 0 && s < X.kchunks) {
                        tc::mbar_wait(&xempty[s], xphase ^ 1);
                        tcw::mbar_expect_tx(&xfull[s], XS_XCH);
                        tcw::tma_load_2d(xbuf + s * XS_XCH, &tmap_x, &xfull[s], s * 128, tok);
                    }
                    tc::mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0) tcw::mbar_expect_tx(&full[stage], 2 * XS_IMG);
                    const int rt = 2 * (XS_EXP(XE_W_TILE0) ? 0 : pt) + (int)rank;
                    if (s < X.kchunks)
                        tcw::tma_load_2d_2sm(ring + stage * XS_IMG, &tmap_s, full0 + 8 * stage, 0,
                                             (rt * X.kchunks + s) * (XS_IMG / 128));
                    else
                        tcw::tma_load_2d_2sm(ring + stage * XS_IMG, &tmap_r, full0 + 8 * stage, 0,
                                             rt * (XS_IMG / 128));
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
            xphase ^= 1;
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ---------------- MMA issuer: leader CTA, whole warp (one elected lane
            // issues), M256 x N224 x K64 sparse; per stage one metadata copy
            const uint32_t idesc = tc::idesc_i8(256, XS_TN, 0, 0) | (1u << 2);
            const uint32_t ring_u = tc::smem_u32(ring);
            const uint64_t adesc0 = tc::smem_desc(ring_u, 128, 512, 0);
            const uint64_t edesc0 = tc::smem_desc(ring_u + 8192, 2048, 128, 0);
            const uint64_t bdesc0 = tc::smem_desc_sw128(tc::smem_u32(xbuf), 16, 1024);
            const uint64_t rdesc0 = tc::smem_desc_sw128(tc::smem_u32(rbuf), 16, 1024);
            int stage = 0, acc = 0, tcnt = 0;
            uint32_t phase = 0, acc_phase = 0, xphase = 0, rphase = 0, eslot = 0;
            for (int unit = pair; unit < units; unit += npairs) {
                int nt, p_lo, p_hi;
                unit_range(unit, nt, p_lo, p_hi);
                for (int i = 0; i < p_hi - p_lo; ++i) {
                    const int pt = pair_tile(p_lo, p_hi, i);
                    const int nres = s_rcnt[pt];
                    tc::mbar_spin(&tempty[acc], acc_phase ^ 1);
                    if (lane == 0) XS_TRACE(0, tcnt, 1);
                    tc::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * XS_TN;
                    for (int kc = 0; kc < X.kchunks; ++kc) {
                        if (i == 0) {
                            tc::mbar_spin(&xfull[kc], xphase);
                            tc::mbar_spin_cluster(&xpeer[kc], xphase);
                        }
                        if (lane == 0) XS_TRACE(0, tcnt, 10);
                        tc::mbar_spin(&full[stage], phase);
                        if (lane == 0) XS_TRACE(0, tcnt, 2);
                        tc::tc_fence_after();
                        const uint64_t so = (uint64_t)((stage * XS_IMG) >> 4);
                        const uint32_t e_tmem = tmem_base + XS_ECOL + 8 * eslot;
                        if (!XS_EXP(XE_NO_MMA)) {
                            tcw::tmem_cp_128x256b_2sm(e_tmem, edesc0 + so);
                            const uint64_t bo = bdesc0 + (uint64_t)((kc * XS_XCH) >> 4);
                            tcw::mma_sp_i8_2sm(d_tmem, adesc0 + so, bo, e_tmem, idesc, kc ? 1u : 0u);
                            tcw::mma_sp_i8_2sm(d_tmem, adesc0 + so + 16, bo + 4, e_tmem + 4, idesc, 1u);
                        }
                        tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                        if (i == p_hi - p_lo - 1) tcw::mma_commit_2sm_mc(&xempty[kc], 0x3);
                        eslot ^= 1;
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (nres) {
                        // residual slots: B from the gathered buffers of both CTAs
                        tc::mbar_spin(&full[stage], phase);
                        tc::mbar_spin_cluster(rfull, rphase);
                        if (lane == 0) XS_TRACE(0, tcnt, 3);
                        tc::tc_fence_after();
                        const uint64_t so = (uint64_t)((stage * XS_IMG) >> 4);
                        const uint32_t e_tmem = tmem_base + XS_ECOL + 8 * eslot;
                        if (!XS_EXP(XE_NO_MMA)) {
                            tcw::tmem_cp_128x256b_2sm(e_tmem, edesc0 + so);
                            tcw::mma_sp_i8_2sm(d_tmem, adesc0 + so, rdesc0, e_tmem, idesc, 1u);
                            if (nres > 1)
                                tcw::mma_sp_i8_2sm(d_tmem, adesc0 + so + 16, rdesc0 + 4, e_tmem + 4, idesc, 1u);
                        }
                        tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                        tcw::mma_commit_2sm_mc(rempty, 0x3);
                        rphase ^= 1;
                        eslot ^= 1;
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    tcw::mma_commit_2sm_mc(&tfull[acc], 0x3);
                    if (lane == 0) XS_TRACE(0, tcnt, 4);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
                xphase ^= 1;
            }
        }
    } else if (xs_gather_index(warp) >= 0) {
        // ---------------- residual gather (both CTAs): slot s of the residual
        // operand = activation column tr_k[s] of this CTA's tokens, copied from
        // the resident SW128 X tile into the same layout; forwards this CTA's
        // X-chunk arrivals to the leader (its MMA cannot wait on a peer barrier)
        const int gi = xs_gather_index(warp);
        int tcnt = 0;
        const uint32_t rfull0 = tc::mapa(tc::smem_u32(rfull), 0);
        const uint32_t xpeer0 = tc::mapa(tc::smem_u32(xpeer), 0);
        uint32_t xphase = 0, rphase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            int nt, p_lo, p_hi;
            unit_range(unit, nt, p_lo, p_hi);
            for (int kc = 0; kc < X.kchunks; ++kc) {
                tc::mbar_wait(&xfull[kc], xphase);
                if (rank == 1 && gi == 0 && lane == 0) tc::mbar_arrive_cluster(xpeer0 + 8 * kc);
            }
            for (int i = 0; i < p_hi - p_lo; ++i) {
                const int pt = pair_tile(p_lo, p_hi, i);
                const int nres = s_rcnt[pt];
                if (!nres) continue;
                const int w4 = nres * 16;                  // 4-slot words per token (16 or 32)
                const int j4 = lane % w4, tstep = 32 / w4;
                // this lane's 4 slots: column loads issued before the wait for
                // the residual buffer, their use after it
                uint32_t kk4[4], kofs[4], kx[4];
                const uint16_t *kp = X.tr_k + (size_t)pt * TR_SLOTS + 4 * j4;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    kk4[b] = __ldg(kp + b);
                    if (kk4[b] == 0xFFFFu) kk4[b] = 0;     // unused slot: any column (its weights are zero)
                }
                tc::mbar_wait(rempty, rphase ^ 1);
                if (lane == 0 && rank == 0) XS_TRACE(13 + gi, tcnt, 8);
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    kofs[b] = (kk4[b] >> 7) * XS_XCH + (kk4[b] & 15);
                    kx[b] = (kk4[b] >> 4) & 7;
                }
#pragma unroll 4
                for (int t = lane / w4 + tstep * gi; t < (XS_EXP(XE_NO_GATHER) ? 0 : XS_TNH); t += tstep * XS_NGATHER) {
                    const uint32_t r8 = (uint32_t)(t & 7);
                    const uint32_t rowb = (uint32_t)(t >> 3) * 1024 + r8 * 128;
                    uint32_t word = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b) word |= (uint32_t)xbuf[rowb + ((kx[b] ^ r8) << 4) + kofs[b]] << (8 * b);
                    *reinterpret_cast<uint32_t *>(rbuf + rowb + ((((uint32_t)j4 >> 2) ^ r8) << 4) + 4 * (j4 & 3)) =
                        word;
                }
                tc::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_cluster(rfull0);
                if (lane == 0 && rank == 0) XS_TRACE(13 + gi, tcnt, 9);
                rphase ^= 1;
            }
            // every read of this unit's X tile is done: second arrival on the chunks
            __syncwarp();
            if (lane == 0)
                for (int kc = 0; kc < X.kchunks; ++kc) tc::mbar_arrive(&xempty[kc]);
            xphase ^= 1;
        }
    } else {
        // ---------------- epilogue warps (both CTAs; each reads its own TMEM half)
        EpiWarp W = make_epi_warp<MODE, XS_EPI_WARPS>(warp, lane, staging, tables, E);
        W.stg = staging + (warp - 2) * XS_WSTG;
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        const int32_t mrow = 128 * (int)rank + W.q * 32 + lane;   // this lane's row within a pair tile
        const uint32_t lane_off = (uint32_t)(W.q * 32) << 16;
        int acc = 0, tcnt = 0;
        uint32_t acc_phase = 0;
        for (int unit = pair; unit < units; unit += npairs) {
            int nt, p_lo, p_hi;
            unit_range(unit, nt, p_lo, p_hi);
            for (int i = 0; i < p_hi - p_lo; ++i) {
                const int pt = pair_tile(p_lo, p_hi, i);
                // row constants: loads issued before blocking on the accumulator
                const XsRow k = xs_row<MODE>(pt * 256 + mrow, P, E);
                const uint32_t te = tempty0 + 8 * acc;
                const int role = 1 + (warp - 2);
                tc::mbar_wait(&tfull[acc], acc_phase);
                if (lane == 0 && rank == 0) XS_TRACE(role, tcnt, 5);
                tc::tc_fence_after();
                xs_epi_tile<MODE, OUTK>(tmem_base + lane_off + acc * XS_TN, pt * 256 + 128 * (int)rank,
                                        (int64_t)nt * XS_TN, &tmap_o, P, E, W, k,
                                        [&, te] { tc::mbar_arrive_cluster(te); if (rank == 0) XS_TRACE(role, tcnt, 6); }, X);
                if (lane == 0 && rank == 0) XS_TRACE(role, tcnt, 7);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
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
int k3_launch_mode(const SpmmArgs &a, const CUtensorMap &ts, const CUtensorMap &tr, const CUtensorMap &tx,
                   const CUtensorMap &to, const K2Params &p, XsParams X)
{
    EpiParams E = make_epi(a.h, a.img, a.sides, a.n);
    cudaStream_t st = (cudaStream_t)a.stream;
    const int npairs = num_sms() / 2;
    auto kern = k3_kernel<MODE, OUTK>;
    constexpr int smem = xs_smem<MODE, OUTK>();
    static_assert(smem <= SMEM_MAX, "shared memory budget");
    set_smem_attr(kern, smem);
    X.mgroups = pick_mgroups(X.ptiles, X.ntiles, npairs);
    const long units = (long)X.ntiles * X.mgroups;
    const int pairs = units < npairs ? (int)units : npairs;
    return (int)launch_pdl(kern, dim3(2 * pairs), dim3(XS_THREADS), smem, st, ts, tr, tx, to, p, E, X);
}

template <int OUTK>
int k3_launch_outk(const SpmmArgs &a, const CUtensorMap &ts, const CUtensorMap &tr, const CUtensorMap &tx,
                   const CUtensorMap &to, const K2Params &p, const XsParams &X)
{
    switch (a.h->epi_mode) {
    case EPI_S32: return k3_launch_mode<EPI_S32, OUTK>(a, ts, tr, tx, to, p, X);
    case EPI_DEQ_F32: return k3_launch_mode<EPI_DEQ_F32, OUTK>(a, ts, tr, tx, to, p, X);
    case EPI_REQUANT: return k3_launch_mode<EPI_REQUANT, OUTK>(a, ts, tr, tx, to, p, X);
    case EPI_REQUANT_LUT: return k3_launch_mode<EPI_REQUANT_LUT, OUTK>(a, ts, tr, tx, to, p, X);
    case EPI_DEQ_TABLE: return k3_launch_mode<EPI_DEQ_TABLE, OUTK>(a, ts, tr, tx, to, p, X);
    case EPI_DEQ_SIDE: return k3_launch_mode<EPI_DEQ_SIDE, OUTK>(a, ts, tr, tx, to, p, X);
    default: return k3_launch_mode<EPI_GENERIC, OUTK>(a, ts, tr, tx, to, p, X);
    }
}

}  // namespace

bool k3_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx)
{
    if (layout != SI_ACT_NK || !h->tr_ok || h->tc_kpad > XS_KMAX || h->tc_mtiles < 2) return false;
    if ((h->tc_mtiles + 1) / 2 > XS_MAXPAIRS) return false;
    if (n < 1 || n > (int64_t)INT32_MAX - XS_TN) return false;
    if (((uintptr_t)x) % 16 || ldx % 16 || h->K % 16) return false;
    return true;
}

int k3_launch(const SpmmArgs &a)
{
    const SiImage *h = a.h;
    const int kch = h->tc_kpad / 128;
    const int pt_n = (h->tc_mtiles + 1) / 2;
    CUtensorMap ts, tr, tx, to;
    bool ok = encode_2d(&ts, img_sec<uint8_t>(a.img, h->off_sp_img), 128, (uint64_t)2 * pt_n * kch * (XS_IMG / 128),
                        128, 128, XS_IMG / 128, CU_TENSOR_MAP_SWIZZLE_NONE) &&
              encode_2d(&tr, img_sec<uint8_t>(a.img, h->off_tr_img), 128, (uint64_t)2 * pt_n * (XS_IMG / 128), 128,
                        128, XS_IMG / 128, CU_TENSOR_MAP_SWIZZLE_NONE) &&
              encode_2d(&tx, a.x, (uint64_t)h->K, (uint64_t)a.n, (uint64_t)a.ldx, 128, XS_TNH);
    if (!ok) return (int)cudaErrorInvalidValue;
    K2Params p;
    std::memset(&p, 0, sizeof(p));
    p.N = a.n;
    p.out = a.out;
    p.ldo = a.ldo;
    p.rqc = img_sec<float>(a.img, h->off_rqc);
    p.rqg = img_sec<float>(a.img, h->off_rqg);
    p.rqp = img_sec<float>(a.img, h->off_rqp);
    XsParams X;
    X.ptiles = pt_n;
    X.ntiles = (int32_t)((a.n + XS_TN - 1) / XS_TN);
    X.kchunks = kch;
    X.mgroups = 1;
    X.tr_k = img_sec<uint16_t>(a.img, h->off_tr_k);
    X.tr_cnt = img_sec<int32_t>(a.img, h->off_tr_cnt);
    X.exp = 0;
    X.trace = nullptr;
#ifdef SI_EXPERIMENTS
    if (const char *e = getenv("SI_XS_EXP")) X.exp = atoi(e);
    static unsigned long long *trace_buf = nullptr;
    const char *trace_path = getenv("SI_XS_TRACE");
    const size_t trace_bytes = (size_t)20 * XS_TRACE_N * 8;
    if (trace_path) {
        if (!trace_buf) cudaMalloc(&trace_buf, trace_bytes);
        cudaMemsetAsync(trace_buf, 0, trace_bytes, (cudaStream_t)a.stream);
        X.trace = trace_buf;
    }
    // (the launch below; then, tracing: wait for it and write the timeline)
    struct Dump {
        const char *path; unsigned long long *buf; size_t bytes; cudaStream_t st;
        ~Dump()
        {
            if (!path || !buf) return;
            std::string hb(bytes, '\0');
            cudaStreamSynchronize(st);
            cudaMemcpy(&hb[0], buf, bytes, cudaMemcpyDeviceToHost);
            if (FILE *f = fopen(path, "wb")) { fwrite(hb.data(), 1, bytes, f); fclose(f); }
        }
    } dump{trace_path, trace_buf, trace_bytes, (cudaStream_t)a.stream};
#endif
    if (h->out_dtype == SI_F32 || h->out_dtype == SI_S32) {
        std::memset(&to, 0, sizeof(to));
        return k3_launch_outk<OUT_32>(a, ts, tr, tx, to, p, X);
    }
    // 8-bit outputs: per-warp boxes of 32 rows x 32 tokens
    const bool tma_ok = (a.ldo % 16 == 0) && ((uintptr_t)a.out % 16 == 0) &&
                        encode_2d(&to, a.out, (uint64_t)h->M, (uint64_t)a.n, (uint64_t)a.ldo, 32, 32,
                                  CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!tma_ok) {
        std::memset(&to, 0, sizeof(to));
        return k3_launch_outk<OUT_8_DIRECT>(a, ts, tr, tx, to, p, X);
    }
    return h->out_dtype == SI_U8 ? k3_launch_outk<OUT_U8_W>(a, ts, tr, tx, to, p, X)
                                 : k3_launch_outk<OUT_S8_W>(a, ts, tr, tx, to, p, X);
}
