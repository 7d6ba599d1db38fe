// spmm_ws.cu -- K4: the W-stationary 2:4-sparse tensor-core SpMM.
//
// Same reference functions as K1/K2/K3 (_acc_group_panel + _spmm_task_*,
// spmm.py:192-280): out[n, m] = epilogue(sum_k W[m,k] x[k,n] + adj[m]).
//
// Why this shape (profiles/r02_k3_analysis.md):
//  * K3 (X-stationary) streams every 2:4 W image once per token tile: each
//    128-k stage costs the MMA thread a metadata copy, two MMAs and a commit,
//    and the resident X tile leaves a shallow W ring.
//  * Here a CTA pair keeps one 256-row W tile resident for a long run of
//    token tiles: the compressed A images (64 B per row and 128-k chunk) stay
//    in shared memory, their metadata in tensor memory, copied there once
//    per W tile.  Only X streams (token-major, K-major SWIZZLE_128B boxes of
//    96 tokens x 128 k per CTA), through a ring that owns all the shared
//    memory W does not use, and the MMA thread issues nothing but MMAs and
//    one commit per stage.
//  * The columns that do not fit the 2:4 images (plan.cpp build_tr_sections)
//    are gathered per stage out of the streamed X boxes into a residual B
//    tile; one or two extra sparse MMAs per tile add them in.  Every MAC is
//    an exact integer MAC, so the result is bit-equal to the dense product.
//
// Work split: the (W tile, token tile) grid is walked W-tile-major and cut
// into one contiguous range per pair, so a pair loads at most two W tiles.
//
// Roles (20 warps, 96 registers each): warps 0 and 14 TMA producers (ring
// iteration i on producer i mod 2; X boxes, and at a W change the W images
// and metadata), warp 1 TMEM allocator + MMA issuer (leader CTA), warps 2-13
// the epilogue (3 token-column groups x 4 TMEM lane quarters), warps 15, 16,
// 18, 19 the residual gather (after the stage's MMAs retired: the commit
// reaches both CTAs, so no arrival has to be forwarded), warp 17 idle.  TMEM: two
// 192-column accumulators + 72 metadata columns.
#include "k2_common.cuh"

namespace {

// Experiment switches exist only in experiment builds (SI_BUILD_DEFS=
// -DSI_EXPERIMENTS, a separate library selected with SI_LIB); the product
// library compiles every WS_EXP(...) to false.
#ifdef SI_EXPERIMENTS
#define WS_EXP(bit) ((X.exp & (bit)) != 0)
#else
#define WS_EXP(bit) false
#endif
#ifdef SI_EXPERIMENTS
// wait-time accounting: cycles a role spends in each of its waits (slots
// 0..3) and in the kernel (slot 4), written per (CTA, warp) to X.stats
#define WS_T0() const long long _t0 = clock64()
#define WS_ACC(slot) wstat[slot] += clock64() - _t0
#else
#define WS_T0() ((void)0)
#define WS_ACC(slot) ((void)0)
#endif
enum WsExp : int32_t {
    WE_NO_EPI = 1,      // epilogue: wait and release only
    WE_NO_GATHER = 2,   // gather: handshakes only
    WE_NO_MMA = 4,      // MMA warp: commits only
    WE_NO_STORE = 16,   // epilogue: no TMA stores
    WE_EPI_LDONLY = 32, // epilogue: TMEM loads + release only
};

constexpr int WS_TNH = 96;                           // tokens per CTA
constexpr int WS_TN = 2 * WS_TNH;                    // MMA N (pair)
constexpr int WS_KMAX = 1024;
constexpr int WS_KCH = WS_KMAX / 128;                // 128-k chunks of a W tile (<= 8)
constexpr int WS_XST = WS_TNH * 128;                 // one ring stage: this CTA's tokens x 128 k
constexpr int WS_AIMG = 8192;                        // compressed A part of a 12 KB 2:4 image
constexpr int WS_EIMG = 4096;                        // its two metadata tiles
constexpr int WS_IMG_ROWS = 96;                      // 128-byte rows per image (64 A + 32 metadata)
constexpr int WS_WBYTES = (WS_KCH + 1) * WS_AIMG;    // resident A: the W tile's chunks + the residual image
constexpr int WS_META_PER_STAGE = WS_XST / WS_EIMG;  // metadata chunks one ring stage carries (3)
constexpr int WS_EPI_WARPS = 12;
constexpr int WS_EPI_GROUPS = WS_EPI_WARPS / 4;
constexpr int WS_NCH = WS_TN / 32;                   // 32-token epilogue chunks per accumulator
constexpr int WS_NPROD = 2;                          // warps 0, 14
constexpr int WS_PROD1_WARP = 2 + WS_EPI_WARPS;      // 14
constexpr int WS_NGATHER = 2;                        // warps 15, 17
constexpr int WS_NISSUE = 4;                         // MMA issuers: warps 1, 16, 18, 19 (one per scheduler)
constexpr int WS_THREADS = 32 * 20;
constexpr int WS_WSTG = 32 * 32;                     // 8-bit staging slot of one warp: 32 tokens x 32 m
constexpr uint32_t WS_ECOL = 2 * WS_TN;              // metadata: TMEM columns 384 .. 384 + 8 * 9
constexpr int WS_LCAP = 4 * TR_SLOTS;                // gather list capacity per 128-k chunk (class-interleaved)
constexpr int WS_LIST = 8 * WS_LCAP * 2 + 256;       // per-chunk gather lists (u16) + class counters + lengths
static_assert(WS_ECOL + 8 * (WS_KCH + 1) <= 512, "TMEM budget");
static_assert(WS_TNH % 8 == 0 && WS_TN % 32 == 0 && WS_TN % 16 == 0, "tile shape");
static_assert(WS_NCH % WS_EPI_GROUPS == 0, "epilogue chunks split evenly over the column groups");
static_assert(WS_XST % 1024 == 0 && WS_META_PER_STAGE >= 1, "ring stage");

__device__ __forceinline__ int ws_issuer_index(int warp)
{
    return warp == 1 ? 0 : warp == 16 ? 1 : warp == 18 ? 2 : warp == 19 ? 3 : -1;
}
__device__ __forceinline__ int ws_gather_index(int warp)
{
    return warp == 15 ? 0 : warp == 17 ? 1 : -1;
}

template <int OUTK>
constexpr int ws_staged() { return (OUTK == OUT_U8_W || OUTK == OUT_S8_W) ? WS_EPI_WARPS * WS_WSTG : 0; }
// residual B tiles: double-buffered unless the epilogue's table needs the room
template <int MODE>
constexpr int ws_rbufs() { return table_bytes<MODE>() ? 1 : 2; }
template <int MODE, int OUTK>
constexpr int ws_fixed()
{
    // + 1024 alignment slack, 1024 barriers
    return WS_WBYTES + ws_rbufs<MODE>() * WS_XST + ws_staged<OUTK>() + table_bytes<MODE>() + WS_LIST + 1024 + 1024;
}
template <int MODE, int OUTK>
constexpr int ws_stages()
{
    // a multiple of 4: a ring stage always belongs to the same producer (stage
    // mod 2), MMA issuer (stage mod 2) and gather warp (stage mod 4), so every
    // role waits on its own stages only, round after round (a parity wait
    // cannot tell round r from round r-2, and must never skip a round)
    constexpr int s = (SMEM_MAX - ws_fixed<MODE, OUTK>()) / WS_XST;
    return s >= 12 ? 12 : s >= 8 ? 8 : 4;
}
template <int MODE, int OUTK>
constexpr int ws_smem() { return ws_fixed<MODE, OUTK>() + ws_stages<MODE, OUTK>() * WS_XST; }

struct WsParams {
    int32_t ptiles;          // 256-row pair tiles
    int32_t ntiles;          // 192-token tiles
    int32_t kchunks;         // 128-k chunks (<= 8)
    int32_t nmeta;           // ring iterations that carry a W tile's metadata
    int32_t q, n_main, H;    // tile schedule (WsIter): main pairs per W tile, their token tiles, helper pairs
    const uint16_t *tr_k;    // [ptiles][TR_SLOTS] activation column per residual slot (0xFFFF: unused)
    const int32_t *tr_cnt;   // [ptiles] residual MMAs (64 slots each)
    int32_t exp;             // experiment switches (WsExp; experiment builds only)
    long long *stats;        // experiment builds: per (CTA, warp) wait-cycle counters (mapped host memory)
};

struct WsRow {
    int32_t adj;
    float s_in, cq, cp, gr;
};

template <int MODE>
__device__ __forceinline__ WsRow ws_row(int32_t m, const K2Params &P, const EpiParams &E)
{
    WsRow k;
    const bool mok = m < E.M;
    k.adj = mok ? __ldg(E.adj + m) : 0;
    k.s_in = mok ? __ldg(E.scale_in + m) : 0.0f;
    k.cq = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqc + m) : 0.0f;
    k.cp = (MODE == EPI_REQUANT && mok) ? __ldg(P.rqp + m) : 0.0f;
    k.gr = mok ? __ldg(P.rqg + m) : 1.0f;
    return k;
}

// Epilogue of one accumulator for one warp: its 32 rows x the column group's
// 32-token chunks (g, g+3), each staged in this warp's own 1 KB tile and
// TMA-stored by its lane 0.  Every chunk, once in registers, is overwritten
// with `adj_next` (adj[m] of the rows the tile after next accumulates here:
// the MMAs only ever accumulate), and the accumulator is released once this
// warp's last chunk is refilled.
template <int MODE, int OUTK, typename Release>
__device__ __forceinline__ void ws_epi_tile(uint32_t lane_base, int32_t row0, int64_t tok0, const CUtensorMap *tmap_o,
                                            const K2Params &P, const EpiParams &E, EpiWarp &W, const WsRow &k,
                                            int32_t adj_next, Release release, const WsParams &X,
                                            long long *wstat = nullptr)
{
    (void)wstat;
    auto rel = [&]() {
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (W.lane == 0) release();
    };
    if (WS_EXP(WE_NO_EPI) || WS_EXP(WE_EPI_LDONLY)) {
        uint32_t acc = 0;
#pragma unroll 1
        for (int ch = W.g; ch < WS_NCH; ch += WS_EPI_GROUPS) {
            if (WS_EXP(WE_EPI_LDONLY)) {
                uint32_t r[32];
                tc::tmem_ld_32x32b_x32(lane_base + ch * 32, r);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc ^= r[j];
            }
            tc::tmem_st_32x32b_x32_fill(lane_base + ch * 32, (uint32_t)adj_next);
        }
        rel();
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
#pragma unroll 1
    for (int ch = W.g; ch < WS_NCH; ch += WS_EPI_GROUPS) {
        const bool last = ch + WS_EPI_GROUPS >= WS_NCH;
        const uint32_t ta = lane_base + ch * 32;
        if constexpr (STAGED) {
            // this warp's previous store must have read its staging tile
            WS_T0();
            if (W.lane == 0) tc::tma_store_wait_read0();
            __syncwarp();
            WS_ACC(2);
        }
#ifdef SI_EXPERIMENTS
        const long long t_ld = clock64();
#endif
        // (adj is already in the accumulator: the chunk's math adds 0)
        epi_chunk<MODE, OUTK>(ta, m, mok, 0, k.s_in, cq, gm, fast, tok0 + ch * 32, 0, P, E, W, [&]() {
#ifdef SI_EXPERIMENTS
            wstat[3] += clock64() - t_ld;
#endif
            tc::tmem_st_32x32b_x32_fill(ta, (uint32_t)adj_next);
            if (last) rel();
        });
        if constexpr (STAGED) {
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (W.lane == 0 && !WS_EXP(WE_NO_STORE)) {
                tc::tma_store_2d(tmap_o, W.stg, row0 + W.q * 32, (int32_t)(tok0 + ch * 32));
                tc::tma_store_commit();
            }
        }
    }
}

// Tile schedule.  Every token tile's X boxes should be read by all the W
// tiles at about the same time (X is re-streamed once per W tile: 16 x 67 MB
// for config 5b, which only stays L2-resident if the pairs sweep the tokens
// together).  `q` = pairs / ptiles "main" pairs per W tile keep that tile for
// the whole kernel and take the token tiles j, j+q, j+2q, ... below n_main;
// the remaining H pairs split the token tiles [n_main, ntiles) of all W tiles
// W-tile-major.  n_main balances the two groups' tile counts.  A pair's work
// is a short list of segments (one W tile, token tiles nt0, nt0+step, ... <
// nt1): one for a main pair, one per W tile touched for a helper.
struct WsSeg {
    int pt, nt0, nt1, step;
};
struct WsPlan {
    int nsegs, pt_first;
    int nh;            // helper: token tiles per W tile in the helper region
    int a0, a1;        // helper: first tile offset in the first segment, end offset in the last
    bool main;
    int j;             // main: first token tile
};
__device__ __forceinline__ WsPlan ws_plan(const WsParams &X, int pair)
{
    WsPlan W;
    const int main_pairs = X.q * X.ptiles;
    W.main = pair < main_pairs;
    W.nh = X.ntiles - X.n_main;
    W.a0 = W.a1 = W.j = 0;
    if (W.main) {
        W.pt_first = pair % X.ptiles;
        W.j = pair / X.ptiles;
        W.nsegs = W.j < X.n_main ? 1 : 0;
    } else {
        const long Th = (long)W.nh * X.ptiles;
        const int h = pair - main_pairs;
        const long i0 = Th * h / X.H, i1 = Th * (h + 1) / X.H;
        if (i1 <= i0) {
            W.nsegs = 0;
            W.pt_first = 0;
        } else {
            W.pt_first = (int)(i0 / W.nh);
            const int pt_last = (int)((i1 - 1) / W.nh);
            W.nsegs = pt_last - W.pt_first + 1;
            W.a0 = (int)(i0 % W.nh);
            W.a1 = (int)((i1 - 1) % W.nh) + 1;
        }
    }
    return W;
}
__device__ __forceinline__ WsSeg ws_seg(const WsParams &X, const WsPlan &W, int s)
{
    WsSeg g;
    if (W.main) {
        g.pt = W.pt_first;
        g.nt0 = W.j;
        g.nt1 = X.n_main;
        g.step = X.q;
    } else {
        g.pt = W.pt_first + s;
        g.nt0 = X.n_main + (s == 0 ? W.a0 : 0);
        g.nt1 = X.n_main + (s == W.nsegs - 1 ? W.a1 : W.nh);
        g.step = 1;
    }
    return g;
}
// W tile of the tile `ahead` (1 or 2) tiles after (segment s, token tile nt), or -1
__device__ __forceinline__ int ws_pt_ahead(const WsParams &X, const WsPlan &W, int s, const WsSeg &g, int nt, int ahead)
{
    int left = (g.nt1 - 1 - nt) / g.step;           // tiles after nt in this segment
    if (ahead <= left) return g.pt;
    ahead -= left;
    for (int t = s + 1; t < W.nsegs; ++t) {
        const WsSeg h = ws_seg(X, W, t);
        const int cnt = (h.nt1 - h.nt0 + h.step - 1) / h.step;
        if (ahead <= cnt) return h.pt;
        ahead -= cnt;
    }
    return -1;
}

// Ring bookkeeping.  Iteration i of the ring (metadata iterations at a W
// change, then kch X boxes per tile) uses stage i mod 8 in round i / 8.  The
// ring has exactly 8 stages so that an iteration's owner is a function of its
// stage: producer i mod 2, MMA issuer i mod 4, gather warp i mod 2.  Every
// role therefore waits on its own stages only, round after round -- a parity
// wait cannot tell round r from round r-2, so no role may skip a round of a
// barrier it waits on -- and walks its iterations without a loop over the
// others (single-warp control flow costs ~25 clk per branch: the issuers'
// per-stage loop used to be the kernel's critical path).
constexpr int WS_STAGES = 8;

template <int MODE, int OUTK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(WS_THREADS, 1)
k4_kernel(const __grid_constant__ CUtensorMap tmap_sa, const __grid_constant__ CUtensorMap tmap_se,
          const __grid_constant__ CUtensorMap tmap_ra, const __grid_constant__ CUtensorMap tmap_re,
          const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_o, const K2Params P,
          const EpiParams E, const WsParams X)
{
    constexpr int STAGES = WS_STAGES;
    static_assert(ws_stages<MODE, OUTK>() >= WS_STAGES, "shared memory budget");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *wbuf = smem;                          // [WS_KCH + 1][8 KB] compressed A (last: residual image)
    uint8_t *rbuf = wbuf + WS_WBYTES;              // [2] gathered residual slots [96 tok x 128 slots] SW128 K-major
    constexpr int RB = ws_rbufs<MODE>();
    uint8_t *ring = rbuf + RB * WS_XST;            // [STAGES][WS_XST]
    uint8_t *staging = ring + STAGES * WS_XST;
    uint8_t *tables = staging + ws_staged<OUTK>();
    uint16_t *glist = reinterpret_cast<uint16_t *>(tables + table_bytes<MODE>());   // [8][WS_LCAP]
    int32_t *gcnt = reinterpret_cast<int32_t *>(glist + 8 * WS_LCAP);               // [8][4] entries per word class
    int32_t *glen = gcnt + 32;                                                      // [8] list length (multiple of 4)
    uint64_t *xfull = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(glist) + WS_LIST);
    uint64_t *xpeer = xfull + STAGES;              // (peer) the stage landed: forwarded by the leader's gather warp
    uint64_t *empty = xpeer + STAGES;              // this CTA's stage: its issuer's MMAs retired + its gather warp done
    uint64_t *tfull = empty + STAGES;              // [2]
    uint64_t *tempty = tfull + 2;                  // [2] (leader)
    uint64_t *rfull = tempty + 2;                  // [2] (leader) both CTAs' residual slots gathered
    uint64_t *rempty = rfull + 2;                  // [2] residual MMAs retired
    uint64_t *wfull = rempty + 2;                  // (leader) both CTAs' resident A images landed
    uint64_t *wfree = wfull + 1;                   // every MMA of the W tile retired
    uint64_t *wmeta = wfree + 1;                   // (leader) the W tile's metadata copies retired
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(wmeta + 1);
    tc::pdl_wait();                 // X may come from the previous kernel (PDL launch)
    tc::pdl_launch_dependents();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_ctarank();
    const int pair = blockIdx.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            tc::mbar_init(&xfull[s], 1);
            tc::mbar_init(&xpeer[s], 1);
            tc::mbar_init(&empty[s], 2);                      // the owning issuer's commit + the owning gather warp
        }
        for (int a = 0; a < 2; ++a) {
            tc::mbar_init(&tfull[a], WS_NISSUE);              // every MMA issuer commits
            tc::mbar_init(&tempty[a], 2 * WS_EPI_WARPS);
            tc::mbar_init(&rfull[a], 2 * WS_NGATHER);
            tc::mbar_init(&rempty[a], 1);
        }
        tc::mbar_init(wfull, 1);
        tc::mbar_init(wfree, WS_NISSUE);                      // every MMA issuer commits
        tc::mbar_init(wmeta, WS_NISSUE);                      // every MMA issuer's metadata copies
        tc::mbar_fence_init();
        tc::tma_prefetch_desc(&tmap_sa);
        tc::tma_prefetch_desc(&tmap_se);
        tc::tma_prefetch_desc(&tmap_ra);
        tc::tma_prefetch_desc(&tmap_re);
        tc::tma_prefetch_desc(&tmap_x);
    }
    if (warp == 1) tc::tmem_alloc_2sm(tmem_slot, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int kch = X.kchunks, nmeta = X.nmeta;
    const WsPlan Wp = ws_plan(X, pair);
#ifdef SI_EXPERIMENTS
    long long wstat[5] = {0, 0, 0, 0, 0};
    const long long t_start = clock64();
#endif

    if (warp == 0 || warp == WS_PROD1_WARP) {
        // ---------------- TMA producers (both CTAs): producer p loads the ring
        // iterations i = p (mod 2); both CTAs' boxes complete on the leader's
        // barrier.  Producer 0 also loads the resident A images at a W change.
        const int prod = warp == 0 ? 0 : 1;
        const uint32_t wfull0 = tc::mapa(tc::smem_u32(wfull), 0);
        const uint32_t xfull0 = tc::mapa(tc::smem_u32(xfull), 0);
        int it = 0;
        for (int sg = 0; sg < Wp.nsegs; ++sg) {
            const WsSeg g = ws_seg(X, Wp, sg);
            const int rt = 2 * g.pt + (int)rank;
            if (prod == 0) {
                // the previous W tile's MMAs must have retired
                if (sg > 0) tc::mbar_wait(wfree, (uint32_t)(sg - 1) & 1);
                if (rank == 0) tcw::mbar_expect_tx(wfull, 2 * (kch + 1) * WS_AIMG);
                for (int c = 0; c < kch; ++c)
                    tcw::tma_load_2d_2sm(wbuf + c * WS_AIMG, &tmap_sa, wfull0, 0, (rt * kch + c) * WS_IMG_ROWS);
                tcw::tma_load_2d_2sm(wbuf + WS_KCH * WS_AIMG, &tmap_ra, wfull0, 0, rt * WS_IMG_ROWS);
            }
            for (int j = (prod - it) & 1; j < nmeta; j += 2) {
                const int itn = it + j, stage = itn & 7;
                tc::mbar_wait(&empty[stage], (((uint32_t)itn >> 3) & 1) ^ 1);
                const int c0 = j * WS_META_PER_STAGE;
                const int c1 = c0 + WS_META_PER_STAGE < kch + 1 ? c0 + WS_META_PER_STAGE : kch + 1;
                if (rank == 0) tcw::mbar_expect_tx(&xfull[stage], 2 * (c1 - c0) * WS_EIMG);
                for (int c = c0; c < c1; ++c) {
                    uint8_t *dst = ring + stage * WS_XST + (c - c0) * WS_EIMG;
                    if (c < kch)
                        tcw::tma_load_2d_2sm(dst, &tmap_se, xfull0 + 8 * stage, 0, (rt * kch + c) * WS_IMG_ROWS + 64);
                    else
                        tcw::tma_load_2d_2sm(dst, &tmap_re, xfull0 + 8 * stage, 0, rt * WS_IMG_ROWS + 64);
                }
            }
            it += nmeta;
            for (int nt = g.nt0; nt < g.nt1; nt += g.step) {
                const int tok = nt * WS_TN + WS_TNH * (int)rank;
                for (int kc = (prod - it) & 1; kc < kch; kc += 2) {
                    const int itn = it + kc, stage = itn & 7;
                    {
                        WS_T0();
                        tc::mbar_wait(&empty[stage], (((uint32_t)itn >> 3) & 1) ^ 1);
                        WS_ACC(0);
                    }
                    if (rank == 0) tcw::mbar_expect_tx(&xfull[stage], 2 * WS_XST);
                    tcw::tma_load_2d_2sm(ring + stage * WS_XST, &tmap_x, xfull0 + 8 * stage, kc * 128, tok);
                }
                it += kch;
            }
        }
    } else if (ws_issuer_index(warp) >= 0) {
        if (rank == 0) {
            // ---------------- MMA issuers: leader CTA, four warps (one elected lane
            // each issues), M256 x N192 x K64 sparse, A and metadata resident.
            // One thread issues an MMA per ~160 clk whatever N is and its own
            // control flow adds as much again (tools/mma_rate.py), so
            // issuer m takes the ring iterations i = m (mod 4): at most two
            // stages per tile, straight-line.  Every MMA accumulates (the
            // epilogue leaves adj[m] in the accumulator it releases), integer
            // adds commute, so the issue streams need no order between them; a
            // stage is complete when its issuer's commit arrives, an accumulator
            // and a W tile when all four issuers' commits have.
            const int mi = ws_issuer_index(warp);
            const uint32_t idesc = tc::idesc_i8(256, WS_TN, 0, 0) | (1u << 2);
            const uint32_t ring_u = tc::smem_u32(ring);
            const uint64_t adesc0 = tc::smem_desc(tc::smem_u32(wbuf), 128, 512, 0);
            const uint64_t edesc0 = tc::smem_desc(ring_u, 2048, 128, 0);
            const uint64_t bdesc0 = tc::smem_desc_sw128(ring_u, 16, 1024);
            const uint64_t rdesc0 = tc::smem_desc_sw128(tc::smem_u32(rbuf), 16, 1024);
            const uint32_t e_base = tmem_base + WS_ECOL;
            int it = 0, acc = 0, rcount = 0, pend_nres = 0, pend_acc = 0;
            uint32_t acc_phase = 0;
            // one owned X stage: wait for it, two MMAs, commit
            auto do_stage = [&](int itn, int kc, uint32_t d_tmem) {
                const int stage = itn & 7;
                const uint64_t bo = bdesc0 + (uint64_t)((stage * WS_XST) >> 4);
                const uint64_t ao = adesc0 + (uint64_t)((kc * WS_AIMG) >> 4);
                {
                    WS_T0();
                    tc::mbar_spin(&xfull[stage], ((uint32_t)itn >> 3) & 1);
                    WS_ACC(0);
                }
                // (TMA -> mbarrier -> MMA needs no tcgen05 fence)
                if (!WS_EXP(WE_NO_MMA)) {
                    tcw::mma_sp_i8_2sm(d_tmem, ao, bo, e_base + 8 * kc, idesc, 1u);
                    tcw::mma_sp_i8_2sm(d_tmem, ao + 16, bo + 4, e_base + 8 * kc + 4, idesc, 1u);
                }
                tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
            };
            // (issuer 0) residual slots of the pending tile: B from the gathered
            // buffers of both CTAs, then its share of that accumulator is complete
            auto flush_residual = [&]() {
                const int rb_sel = rcount % RB;
                {
                    WS_T0();
                    tc::mbar_spin_cluster(&rfull[rb_sel], (uint32_t)(rcount / RB) & 1);
                    WS_ACC(2);
                }
                const uint32_t d_pend = tmem_base + pend_acc * WS_TN;
                const uint64_t ao = adesc0 + (uint64_t)((WS_KCH * WS_AIMG) >> 4);
                const uint64_t ro = rdesc0 + (uint64_t)((rb_sel * WS_XST) >> 4);
                tcw::mma_sp_i8_2sm(d_pend, ao, ro, e_base + 8 * WS_KCH, idesc, 1u);
                if (pend_nres > 1) tcw::mma_sp_i8_2sm(d_pend, ao + 16, ro + 4, e_base + 8 * WS_KCH + 4, idesc, 1u);
                tcw::mma_commit_2sm_mc(&rempty[rb_sel], 0x3);
                tcw::mma_commit_2sm_mc(&tfull[pend_acc], 0x3);
                ++rcount;
                pend_nres = 0;
            };
            for (int sg = 0; sg < Wp.nsegs; ++sg) {
                const WsSeg g = ws_seg(X, Wp, sg);
                // metadata of the new W tile -> TMEM (each issuer copies the
                // stages it owns), once every issuer's MMAs on the previous tile
                // have retired; MMAs start when every issuer's copies have
                if (sg > 0) {
                    tc::mbar_spin(wfree, (uint32_t)(sg - 1) & 1);
                    tc::tc_fence_after();
                }
                for (int j = (mi - it) & 3; j < nmeta; j += 4) {
                    const int itn = it + j, stage = itn & 7;
                    tc::mbar_spin(&xfull[stage], ((uint32_t)itn >> 3) & 1);
                    const uint64_t so = (uint64_t)((stage * WS_XST) >> 4);
                    const int c0 = j * WS_META_PER_STAGE;
                    const int c1 = c0 + WS_META_PER_STAGE < kch + 1 ? c0 + WS_META_PER_STAGE : kch + 1;
                    for (int c = c0; c < c1; ++c)
                        tcw::tmem_cp_128x256b_2sm(e_base + 8 * (c < kch ? c : WS_KCH),
                                                  edesc0 + so + (uint64_t)(((c - c0) * WS_EIMG) >> 4));
                    tcw::mma_commit_2sm_mc(&empty[stage], 0x3);
                }
                it += nmeta;
                tcw::mma_commit_2sm_mc(wmeta, 0x1);
                tc::mbar_spin(wmeta, (uint32_t)sg & 1);
                tc::mbar_spin(wfull, (uint32_t)sg & 1);
                tc::tc_fence_after();
                const int nres = mi == 0 ? __ldg(X.tr_cnt + g.pt) : 0;
                for (int nt = g.nt0; nt < g.nt1; nt += g.step) {
                    {
                        WS_T0();
                        tc::mbar_spin(&tempty[acc], acc_phase);      // (the epilogue's initial fill is completion 0)
                        WS_ACC(1);
                    }
                    tc::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * WS_TN;
                    int kc = (mi - it) & 3;
                    if (kc < kch) do_stage(it + kc, kc, d_tmem);
                    // the previous tile's residual MMAs (its last columns are
                    // gathered when its last stage lands: one stage of slack)
                    if (pend_nres) flush_residual();
                    kc += 4;
                    if (kc < kch) do_stage(it + kc, kc, d_tmem);
                    it += kch;
                    if (nres) {
                        pend_nres = nres;
                        pend_acc = acc;
                        // now if the tile's slots are already gathered (the gather
                        // runs at landing time, ahead of the MMAs), else one stage
                        // into the next tile; the residual image leaves with the W tile
                        if (nt + g.step >= g.nt1 ||
                            tc::mbar_test_cluster(&rfull[rcount % RB], (uint32_t)(rcount / RB) & 1))
                            flush_residual();
                    } else {
                        tcw::mma_commit_2sm_mc(&tfull[acc], 0x3);
                    }
                    if (nt + g.step >= g.nt1) tcw::mma_commit_2sm_mc(wfree, 0x3);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
            }
            if (pend_nres) flush_residual();
        }
    } else if (ws_gather_index(warp) >= 0) {
        // ---------------- residual gather (both CTAs): slot s of the residual
        // operand = activation column tr_k[s] of this CTA's tokens, copied out
        // of the streamed X box that carries it into the same SW128 layout.
        // Gather warp g owns the ring iterations i = g (mod 2): it waits for
        // the stage to land, copies the stage's entries and releases the
        // stage.  The leader sees both CTAs' boxes complete on its barrier and
        // forwards that to the peer.
        //
        // One instruction moves 8 tokens x 4 entries (lane = 8 * entry + token):
        // the 8 rows of a SWIZZLE_128B atom put one column into 8 different
        // 16-byte segments, and the four entries of a quad have four different
        // words within the segment, so the byte loads hit 32 different banks.
        // Per W tile the slots are bucketed by 128-k chunk and word class once:
        // list position 4 * i + c holds the i-th entry of class c (0xFFFF: none).
        const int gi = ws_gather_index(warp);
        const int gtid = gi * 32 + lane;
        const uint32_t rfull0 = tc::mapa(tc::smem_u32(rfull), 0);
        const uint32_t r8 = (uint32_t)(lane & 7), eq = (uint32_t)(lane >> 3);
        uint64_t *landed = rank == 0 ? xfull : xpeer;
        const uint32_t xpeer1 = tc::mapa(tc::smem_u32(xpeer), 1);
        int it = 0, rcount = 0;
        auto stage_landed = [&](int itn) {
            const int stage = itn & 7;
            WS_T0();
            tc::mbar_wait_cluster(&landed[stage], ((uint32_t)itn >> 3) & 1);
            WS_ACC(0);
            if (rank == 0 && lane == 0) tc::mbar_arrive_cluster(xpeer1 + 8 * stage);
        };
        for (int sg = 0; sg < Wp.nsegs; ++sg) {
            const WsSeg g = ws_seg(X, Wp, sg);
            const int nres = __ldg(X.tr_cnt + g.pt);
            tc::named_bar_sync(8, 32 * WS_NGATHER);
            if (gtid < 32) gcnt[gtid] = 0;
            for (int i = gtid; i < 8 * WS_LCAP / 2; i += 32 * WS_NGATHER) reinterpret_cast<uint32_t *>(glist)[i] = 0xFFFFFFFFu;
            tc::named_bar_sync(8, 32 * WS_NGATHER);
            for (int sl = gtid; sl < 64 * nres; sl += 32 * WS_NGATHER) {
                const uint32_t k = __ldg(X.tr_k + (size_t)g.pt * TR_SLOTS + sl);
                if (k != 0xFFFFu) {
                    const int c = (int)(k >> 7), wc = (int)((k & 15u) >> 2);
                    const int pos = atomicAdd(&gcnt[c * 4 + wc], 1);
                    glist[c * WS_LCAP + 4 * pos + wc] = (uint16_t)(((k & 127u) << 8) | (uint32_t)sl);
                }
            }
            tc::named_bar_sync(8, 32 * WS_NGATHER);
            if (gtid < 8) {
                int mx = 0;
                for (int wc = 0; wc < 4; ++wc) mx = max(mx, gcnt[gtid * 4 + wc]);
                glen[gtid] = 4 * mx;
            }
            tc::named_bar_sync(8, 32 * WS_NGATHER);
            for (int j = (gi - it) & 1; j < nmeta; j += 2) {
                stage_landed(it + j);
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&empty[(it + j) & 7]);
            }
            it += nmeta;
            for (int nt = g.nt0; nt < g.nt1; nt += g.step) {
                const int rb_sel = rcount % RB;
                uint8_t *rb = rbuf + rb_sel * WS_XST + r8 * 128;
                bool first = true;
                for (int kc = (gi - it) & 1; kc < kch; kc += 2) {
                    const int itn = it + kc, stage = itn & 7;
                    // this lane's entries of the stage's first four quads: loaded
                    // in the shadow of the wait for the stage
                    const uint16_t *gl = glist + kc * WS_LCAP + eq;
                    const int np = nres ? glen[kc] : 0;
                    uint32_t ent[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) ent[j] = 4 * j < np ? gl[4 * j] : 0xFFFFu;
                    stage_landed(itn);
                    if (nres && first) {
                        // the residual MMAs two tiles back must have read this buffer
                        WS_T0();
                        tc::mbar_wait(&rempty[rb_sel], ((uint32_t)(rcount / RB) & 1) ^ 1);
                        WS_ACC(1);
                        first = false;
                    }
                    WS_T0();
                    if (nres) {
                        if (!WS_EXP(WE_NO_GATHER)) {
                            const uint8_t *xs = ring + stage * WS_XST + r8 * 128;
                            for (int p0 = 0; p0 < np; p0 += 16) {
                                if (p0) {
#pragma unroll
                                    for (int j = 0; j < 4; ++j) ent[j] = p0 + 4 * j < np ? gl[p0 + 4 * j] : 0xFFFFu;
                                }
                                // (a missing entry reads column 0 and stores nothing)
                                const uint8_t *src[4];
                                uint8_t *dst[4];
                                uint8_t v[4][WS_TNH / 8];
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    const uint32_t ko = ent[j] == 0xFFFFu ? 0u : ent[j] >> 8, sl = ent[j] & 127u;
                                    src[j] = xs + (((ko >> 4) ^ r8) << 4) + (ko & 15u);
                                    dst[j] = rb + (((sl >> 4) ^ r8) << 4) + (sl & 15u);
                                }
#pragma unroll
                                for (int j = 0; j < 4; ++j)
#pragma unroll
                                    for (int tg = 0; tg < WS_TNH / 8; ++tg) v[j][tg] = src[j][tg * 1024];
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (ent[j] != 0xFFFFu) {
#pragma unroll
                                        for (int tg = 0; tg < WS_TNH / 8; ++tg) dst[j][tg * 1024] = v[j][tg];
                                    }
                            }
                        }
                    }
                    __syncwarp();
                    WS_ACC(2);
                    if (lane == 0) tc::mbar_arrive(&empty[stage]);
                }
                it += kch;
                if (nres) {
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_cluster(rfull0 + 8 * rb_sel);
                    ++rcount;
                }
            }
        }
    } else if (warp >= 2 && warp < 2 + WS_EPI_WARPS) {
        // ---------------- epilogue warps (both CTAs; each reads its own TMEM half)
        EpiWarp W = make_epi_warp<MODE, WS_EPI_WARPS>(warp, lane, staging, tables, E);
        W.stg = staging + (warp - 2) * WS_WSTG;
        const uint32_t tempty0 = tc::mapa(tc::smem_u32(tempty), 0);
        const int32_t mrow = 128 * (int)rank + W.q * 32 + lane;   // this lane's row within a pair tile
        const uint32_t lane_off = (uint32_t)(W.q * 32) << 16;
        int acc = 0;
        uint32_t acc_phase = 0;
        // adj[m] of this lane's row in pair tile pt (the accumulators' initial value)
        auto adj_of = [&](int pt) -> int32_t {
            const int32_t m2 = pt * 256 + mrow;
            return (pt >= 0 && m2 < E.M) ? __ldg(E.adj + m2) : 0;
        };
        // initial fill of both accumulators for the first two tiles, then the
        // first completion of tempty[0..1]
        if (Wp.nsegs > 0) {
            const WsSeg g0 = ws_seg(X, Wp, 0);
            for (int a = 0; a < 2; ++a) {
                const int32_t v = adj_of(a == 0 ? g0.pt : ws_pt_ahead(X, Wp, 0, g0, g0.nt0, 1));
                for (int ch = W.g; ch < WS_NCH; ch += WS_EPI_GROUPS)
                    tc::tmem_st_32x32b_x32_fill(tmem_base + lane_off + a * WS_TN + ch * 32, (uint32_t)v);
            }
            tc::tmem_st_wait();
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive_cluster(tempty0);
                tc::mbar_arrive_cluster(tempty0 + 8);
            }
        }
        for (int sg = 0; sg < Wp.nsegs; ++sg) {
            const WsSeg g = ws_seg(X, Wp, sg);
            const WsRow k = ws_row<MODE>(g.pt * 256 + mrow, P, E);
            for (int nt = g.nt0; nt < g.nt1; nt += g.step) {
                // the accumulator released here next holds the tile two ahead
                int32_t adj_next = k.adj;
                if (nt + 2 * g.step >= g.nt1) adj_next = adj_of(ws_pt_ahead(X, Wp, sg, g, nt, 2));
                const uint32_t te = tempty0 + 8 * acc;
                {
                    WS_T0();
                    tc::mbar_wait(&tfull[acc], acc_phase);
                    WS_ACC(0);
                }
                tc::tc_fence_after();
                WS_T0();
                ws_epi_tile<MODE, OUTK>(tmem_base + lane_off + acc * WS_TN, g.pt * 256 + 128 * (int)rank,
                                        (int64_t)nt * WS_TN, &tmap_o, P, E, W, k, adj_next,
                                        [te] { tc::mbar_arrive_cluster(te); }, X
#ifdef SI_EXPERIMENTS
                                        , wstat
#endif
                );
                WS_ACC(1);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
        if ((OUTK == OUT_U8_W || OUTK == OUT_S8_W) && lane == 0) tc::tma_store_wait_all0();
    }
#ifdef SI_EXPERIMENTS
    if (X.stats && lane == 0) {
        wstat[4] = clock64() - t_start;
        for (int i = 0; i < 5; ++i) X.stats[((size_t)blockIdx.x * 20 + warp) * 5 + i] = wstat[i];
    }
#endif
    tc::tc_fence_before();
    tc::cluster_sync();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc_2sm(tmem_base, 512);
    }
}

template <int MODE, int OUTK>
int k4_launch_mode(const SpmmArgs &a, const CUtensorMap *tm, const K2Params &p, const WsParams &X)
{
    EpiParams E = make_epi(a.h, a.img, a.sides, a.n);
    cudaStream_t st = (cudaStream_t)a.stream;
    const int npairs = num_sms() / 2;
    auto kern = k4_kernel<MODE, OUTK>;
    constexpr int smem = ws_smem<MODE, OUTK>();
    static_assert(smem <= SMEM_MAX, "shared memory budget");
    set_smem_attr(kern, smem);
    const long tiles = (long)X.ptiles * X.ntiles;
    const int pairs = tiles < npairs ? (int)tiles : npairs;
    WsParams S = X;
    S.q = pairs / X.ptiles;
    S.H = pairs - S.q * X.ptiles;
    if (S.q == 0)
        S.n_main = 0;
    else if (S.H == 0)
        S.n_main = X.ntiles;
    else {
        // tiles per main pair n_main / q ~ tiles per helper (ntiles - n_main) * ptiles / H
        S.n_main = (int)(((long)X.ntiles * S.q * X.ptiles + pairs / 2) / pairs);
        if (S.n_main > X.ntiles) S.n_main = X.ntiles;
    }
    if (S.n_main == X.ntiles) S.H = 0;       // nothing left for helpers
    const int launch_pairs = S.q * X.ptiles + S.H;
    return (int)launch_pdl(kern, dim3(2 * launch_pairs), dim3(WS_THREADS), smem, st, tm[0], tm[1], tm[2], tm[3], tm[4],
                           tm[5], p, E, S);
}

template <int OUTK>
int k4_launch_outk(const SpmmArgs &a, const CUtensorMap *tm, const K2Params &p, const WsParams &X)
{
    switch (a.h->epi_mode) {
    case EPI_S32: return k4_launch_mode<EPI_S32, OUTK>(a, tm, p, X);
    case EPI_DEQ_F32: return k4_launch_mode<EPI_DEQ_F32, OUTK>(a, tm, p, X);
    case EPI_REQUANT: return k4_launch_mode<EPI_REQUANT, OUTK>(a, tm, p, X);
    case EPI_REQUANT_LUT: return k4_launch_mode<EPI_REQUANT_LUT, OUTK>(a, tm, p, X);
    case EPI_DEQ_TABLE: return k4_launch_mode<EPI_DEQ_TABLE, OUTK>(a, tm, p, X);
    case EPI_DEQ_SIDE: return k4_launch_mode<EPI_DEQ_SIDE, OUTK>(a, tm, p, X);
    default: return k4_launch_mode<EPI_GENERIC, OUTK>(a, tm, p, X);
    }
}

}  // namespace

bool k4_supported(const SiImage *h, int64_t n, int32_t layout, const void *x, int64_t ldx)
{
    if (layout != SI_ACT_NK || !h->tr_ok || h->tc_kpad > WS_KMAX || h->tc_mtiles < 2) return false;
    if (n < 1 || n > (int64_t)INT32_MAX - WS_TN) return false;
    if (((uintptr_t)x) % 16 || ldx % 16 || h->K % 16) return false;
    return true;
}

int k4_launch(const SpmmArgs &a)
{
    const SiImage *h = a.h;
    const int kch = h->tc_kpad / 128;
    const int pt_n = (h->tc_mtiles + 1) / 2;
    CUtensorMap tm[6];
    const uint8_t *sp = img_sec<uint8_t>(a.img, h->off_sp_img);
    const uint8_t *tr = img_sec<uint8_t>(a.img, h->off_tr_img);
    const uint64_t sp_rows = (uint64_t)2 * pt_n * kch * WS_IMG_ROWS, tr_rows = (uint64_t)2 * pt_n * WS_IMG_ROWS;
    bool ok = encode_2d(&tm[0], sp, 128, sp_rows, 128, 128, 64, CU_TENSOR_MAP_SWIZZLE_NONE) &&
              encode_2d(&tm[1], sp, 128, sp_rows, 128, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE) &&
              encode_2d(&tm[2], tr, 128, tr_rows, 128, 128, 64, CU_TENSOR_MAP_SWIZZLE_NONE) &&
              encode_2d(&tm[3], tr, 128, tr_rows, 128, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE) &&
              encode_2d(&tm[4], a.x, (uint64_t)h->K, (uint64_t)a.n, (uint64_t)a.ldx, 128, WS_TNH);
    if (!ok) return (int)cudaErrorInvalidValue;
    K2Params p;
    std::memset(&p, 0, sizeof(p));
    p.N = a.n;
    p.out = a.out;
    p.ldo = a.ldo;
    p.rqc = img_sec<float>(a.img, h->off_rqc);
    p.rqg = img_sec<float>(a.img, h->off_rqg);
    p.rqp = img_sec<float>(a.img, h->off_rqp);
    WsParams X;
    X.ptiles = pt_n;
    X.ntiles = (int32_t)((a.n + WS_TN - 1) / WS_TN);
    X.kchunks = kch;
    X.nmeta = (kch + 1 + WS_META_PER_STAGE - 1) / WS_META_PER_STAGE;
    X.tr_k = img_sec<uint16_t>(a.img, h->off_tr_k);
    X.tr_cnt = img_sec<int32_t>(a.img, h->off_tr_cnt);
    X.exp = 0;
    X.stats = nullptr;
#ifdef SI_EXPERIMENTS
    if (const char *e = getenv("SI_WS_EXP")) X.exp = atoi(e);
    if (const char *e = getenv("SI_WS_STATS")) X.stats = (long long *)strtoull(e, nullptr, 0);
#endif
    if (h->out_dtype == SI_F32 || h->out_dtype == SI_S32) {
        std::memset(&tm[5], 0, sizeof(tm[5]));
        return k4_launch_outk<OUT_32>(a, tm, p, X);
    }
    // 8-bit outputs: per-warp boxes of 32 rows x 32 tokens
    const bool tma_ok = (a.ldo % 16 == 0) && ((uintptr_t)a.out % 16 == 0) &&
                        encode_2d(&tm[5], a.out, (uint64_t)h->M, (uint64_t)a.n, (uint64_t)a.ldo, 32, 32,
                                  CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!tma_ok) {
        std::memset(&tm[5], 0, sizeof(tm[5]));
        return k4_launch_outk<OUT_8_DIRECT>(a, tm, p, X);
    }
    return h->out_dtype == SI_U8 ? k4_launch_outk<OUT_U8_W>(a, tm, p, X) : k4_launch_outk<OUT_S8_W>(a, tm, p, X);
}
