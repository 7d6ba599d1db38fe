// k2_common.cuh -- shared by the tensor-core kernels (spmm_tc.cu, spmm_xs.cu):
// tile constants, kernel parameters, the compiled epilogue forms of the
// reference's _run_chain (epilogue.py:207-249) and the host-side launch helpers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>
#include <string>

#include "epilogue.cuh"
#include "si_internal.h"
#include "tc_ptx.cuh"

namespace {


constexpr int BK = 128;                     // k per pipeline stage (one 128B swizzle row)
constexpr int EPI_WARPS = 16;               // 4 per TMEM lane quarter
constexpr int EPI_GROUPS = EPI_WARPS / 4;   // token column groups
constexpr int TILE_N = 256;                 // tokens per accumulator tile
constexpr int COLS = TILE_N / EPI_GROUPS;   // tokens per epilogue warp (64)
constexpr int THREADS = 32 * (2 + EPI_WARPS);
// TMA issue: one issuing warp sustains about one box per ~200 ns (tools/
// tma_bw.py), so the single/pair/sparse kernels spread their loads over
// NPROD producer warps (warp 0 + NPROD-1 warps after the epilogue warps),
// producer p taking the ring iterations it == p (mod NPROD)
constexpr int NPROD = 3;   // 20 warps: keeps the 96-register cap (warps allocate in groups of 4)
constexpr int MT_THREADS = THREADS + 32 * (NPROD - 1);
__device__ __forceinline__ int producer_index(int warp, int first_extra)
{
    return warp == 0 ? 0 : (warp >= first_extra && warp < first_extra + NPROD - 1) ? warp - first_extra + 1 : -1;
}
constexpr int WSTG = 32 * 32;               // one per-warp staging buffer (8-bit outputs): 32 tokens x 32 m
constexpr int STG_BYTES = EPI_WARPS * 2 * WSTG;
constexpr int TABLE_BYTES = 16 * 1024;      // breakpoint tables staged in smem (EPI_DEQ_TABLE)
constexpr int SMEM_MAX = 232448;

// 8-bit outputs: *_W stage a per-warp tile of 32 tokens x 32 rows (row-major
// 32 B) and store it with one TMA store per warp and chunk (no cross-warp
// barrier); OUT_8_DIRECT writes bytes (outputs TMA cannot address)
enum OutKind { OUT_32 = 0, OUT_8_DIRECT = 3, OUT_U8_W = 4, OUT_S8_W = 5 };

struct K2Params {
    int32_t mtiles;      // weight-row tiles (128 rows single-CTA, 256 rows per pair)
    int32_t ntiles;      // 256-token tiles
    int32_t kchunks;     // k stages
    int32_t b_mn_major;  // 1: X is [K, N] (MN-major B), 0: [N, K] (K-major B)
    int32_t bks;         // pair kernel: k per stage (256, or 128 for few work units per pair)
    int32_t exp;         // experiment builds only (SI_K2_EXP): 1 no epilogue work, 2 no MMAs
    int64_t N;
    void *out;
    int64_t ldo;
    const float *rqc;    // requant c[m] = f32(scale_in[m] / fp)
    const float *rqg;    // per-row class (image off_rqg): < 0 unsafe, >= 1 proven, else requant guard
    const float *rqp;    // proven rows' requant multiplier (image off_rqp)
};

constexpr float MAGIC_F = 12582912.0f;     // 1.5 * 2^23
// certificate guard: with |a| < 2^22 the magic conversion is exact, so
// r = RN(a * RN(s/fp)) has |r - y| <= (2^-23 + 2^-48)|y| against the
// reference's f64 value y; 2^-22 |r| leaves a 2x margin
constexpr float CERT_G = 2.384185791015625e-07f;  // 2^-22
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

// per-warp epilogue state
struct EpiWarp {
    int q, g, lane, u, i4;
    uint32_t selA, selB;
    uint8_t *stg;
    const int32_t *s_key;
    const uint32_t *s_val;
    const uint16_t *s_bkt;
};

// One 32-token chunk of one warp: TMEM columns -> outputs.  m is this
// lane's weight row, n0 the chunk's first token, c the chunk index within the
// warp's 64 columns (staging row offset).
struct NoOp {
    __device__ __forceinline__ void operator()() const {}
};

// on_loaded() runs once the chunk's accumulators are in registers (the
// accumulator can be released there, before the math and the stores).
template <int MODE, int OUTK, typename OnLoaded = NoOp>
__device__ __forceinline__ void epi_chunk(uint32_t taddr, int32_t m, bool mok, int32_t adj, float s_in, float cq,
                                          float gm, bool fast, int64_t n0, int c, const K2Params &P,
                                          const EpiParams &E, const EpiWarp &W, OnLoaded on_loaded = OnLoaded())
{
    uint32_t r[32];
    tc::tmem_ld_32x32b_x32(taddr, r);
    tc::tmem_ld_wait();
    on_loaded();
    int32_t v[32];
    if constexpr (MODE == EPI_REQUANT) {
        const int32_t adjM = (int32_t)((uint32_t)adj + (uint32_t)MAGIC_I);
        const int32_t qoff = MAGIC_I - E.q_zp;
        float emax = 0.0f;
        uint32_t umax = 0;
        const unsigned long long M2 = tc::f2pack(MAGIC_F, MAGIC_F), C2 = tc::f2pack(cq, cq);
        if (gm >= 1.0f) {   // (warp-uniform: all rows proven)
            // every row of this warp has a plan-time multiplier c' (rqp) under
            // which rint(a * c' + zp) (one fma rounding onto the magic number
            // 1.5*2^23 + zp) equals the reference's output for every reachable
            // accumulator (plan.cpp requant_fma_exact): no certificate
            const unsigned long long MZ2 = tc::f2pack(MAGIC_F + (float)E.q_zp, MAGIC_F + (float)E.q_zp);
            if (gm >= 2.0f) {
                // some row may exceed the magic range (|a| < 2^24): I2F conversion
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    const float a0 = __int2float_rn((int32_t)(r[j] + (uint32_t)adj));
                    const float a1 = __int2float_rn((int32_t)(r[j + 1] + (uint32_t)adj));
                    const unsigned long long uu = tc::fma_f32x2(tc::f2pack(a0, a1), C2, MZ2);
                    v[j] = __float_as_int(tc::f2lo(uu)) - MAGIC_I;
                    v[j + 1] = __float_as_int(tc::f2hi(uu)) - MAGIC_I;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    const int32_t b0 = (int32_t)(r[j] + (uint32_t)adjM);
                    const int32_t b1 = (int32_t)(r[j + 1] + (uint32_t)adjM);
                    const unsigned long long af =
                        tc::sub_f32x2(tc::f2pack(__int_as_float(b0), __int_as_float(b1)), M2);
                    const unsigned long long uu = tc::fma_f32x2(af, C2, MZ2);
                    v[j] = __float_as_int(tc::f2lo(uu)) - MAGIC_I;
                    v[j + 1] = __float_as_int(tc::f2hi(uu)) - MAGIC_I;
                }
            }
        } else if (fast) {
            // every row of this warp provably stays within the magic-number
            // range (plan-time bound 255*sum|w| + |adj| < 2^22) and |r| <= the
            // row's max|r|: the certificate |d| + 2^-22|r| < 1/2 reduces to
            // max|d| < 1/2 - guard (guard = 2^-22 max|r|, rqg; proven rows 0)
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                const int32_t b0 = (int32_t)(r[j] + (uint32_t)adjM);
                const int32_t b1 = (int32_t)(r[j + 1] + (uint32_t)adjM);
                const unsigned long long af = tc::sub_f32x2(tc::f2pack(__int_as_float(b0), __int_as_float(b1)), M2);
                const unsigned long long rf = tc::mul_f32x2(af, C2);
                const unsigned long long uu = tc::add_f32x2(rf, M2);
                const unsigned long long d = tc::sub_f32x2(rf, tc::sub_f32x2(uu, M2));
                emax = fmaxf(emax, fmaxf(fabsf(tc::f2lo(d)), fabsf(tc::f2hi(d))));
                v[j] = __float_as_int(tc::f2lo(uu)) - qoff;
                v[j + 1] = __float_as_int(tc::f2hi(uu)) - qoff;
            }
            emax += gm;
        } else
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const int32_t b0 = (int32_t)(r[j] + (uint32_t)adjM);
            const int32_t b1 = (int32_t)(r[j + 1] + (uint32_t)adjM);
            umax = max(umax, (uint32_t)(b0 - 0x4B000000));
            umax = max(umax, (uint32_t)(b1 - 0x4B000000));
            const unsigned long long af = tc::sub_f32x2(tc::f2pack(__int_as_float(b0), __int_as_float(b1)), M2);
            const unsigned long long rf = tc::mul_f32x2(af, C2);
            const unsigned long long uu = tc::add_f32x2(rf, M2);
            const unsigned long long d = tc::sub_f32x2(rf, tc::sub_f32x2(uu, M2));
            emax = fmaxf(emax, __fmaf_rn(fabsf(tc::f2lo(rf)), CERT_G, fabsf(tc::f2lo(d))));
            emax = fmaxf(emax, __fmaf_rn(fabsf(tc::f2hi(rf)), CERT_G, fabsf(tc::f2hi(d))));
            v[j] = __float_as_int(tc::f2lo(uu)) - qoff;
            v[j + 1] = __float_as_int(tc::f2hi(uu)) - qoff;
        }
        if (__any_sync(0xffffffffu, emax >= 0.5f || umax >= 0x800000u)) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int32_t a = (int32_t)(r[j] + (uint32_t)adj);
                const int32_t b = (int32_t)((uint32_t)a + (uint32_t)MAGIC_I);
                const float rf = __fmul_rn(__fsub_rn(__int_as_float(b), MAGIC_F), cq);
                const float d = __fsub_rn(rf, __fsub_rn(__fadd_rn(rf, MAGIC_F), MAGIC_F));
                const bool bad = ((uint32_t)(b - 0x4B000000) >= 0x800000u) ||
                                 !(__fmaf_rn(fabsf(rf), CERT_G, fabsf(d)) < 0.5f);
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
        if (fast) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int32_t b = (int32_t)(r[j] + (uint32_t)adjM);
                v[j] = __float_as_int(__fmul_rn(__fsub_rn(__int_as_float(b), MAGIC_F), s_in));
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int32_t b = (int32_t)(r[j] + (uint32_t)adjM);
                umax = max(umax, (uint32_t)(b - 0x4B000000));
                v[j] = __float_as_int(__fmul_rn(__fsub_rn(__int_as_float(b), MAGIC_F), s_in));
            }
        }
        if (!fast && __any_sync(0xffffffffu, umax >= 0x800000u)) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int32_t a = (int32_t)(r[j] + (uint32_t)adj);
                if ((uint32_t)(a + 0x400000) >= 0x800000u) v[j] = __float_as_int(deq_exact(a, s_in));
            }
        }
    } else if constexpr (MODE == EPI_DEQ_TABLE) {
        // dequantized value f32(f64(a) * f64(s)) = RN(a * s) exactly while
        // |a| <= 2^24; when every row of the warp provably stays below 2^22
        // (`fast`, the plan's row bound) the magic-number conversion replaces
        // I2F and the f64 fallback disappears from the loop
        float x[32];
        if (fast) {
            const int32_t adjM = (int32_t)((uint32_t)adj + (uint32_t)MAGIC_I);
#pragma unroll
            for (int j = 0; j < 32; ++j)
                x[j] = __fmul_rn(__fsub_rn(__int_as_float((int32_t)(r[j] + (uint32_t)adjM)), MAGIC_F), s_in);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) x[j] = dev_deq_acc((int32_t)(r[j] + (uint32_t)adj), s_in);
        }
        if (E.bp_lin_n > 0) {
            // (uniform) linear buckets with one threshold each: one compare
            const uint32_t lin = tc::smem_u32(W.s_key) - (0x4B000000u << 3);
            const float nbm1 = (float)(E.bp_lin_n - 1);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = bp_lookup_linear_smem(x[j], lin, E.bp_lin_inv, E.bp_lin_off, nbm1);
        } else
        // (uniform branch on the plan's bucket occupancy) fixed-step lookups
#define SI_BP_CHUNK(S)                                                                                          \
    for (int j = 0; j < 32; ++j)                                                                                \
        v[j] = (int32_t)bp_lookup_fixed<S>(x[j], W.s_key, W.s_bkt, W.s_val, E.n_bp, E.bp_key_lo, E.bp_shift,     \
                                           E.bp_nbucket);
        if (E.n_bp > 0 && E.bp_occ < 4) {
#pragma unroll
            SI_BP_CHUNK(2)
        } else if (E.n_bp > 0 && E.bp_occ < 16) {
#pragma unroll
            SI_BP_CHUNK(4)
        } else if (E.n_bp > 0 && E.bp_occ < 64) {
#pragma unroll
            SI_BP_CHUNK(6)
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                v[j] = (int32_t)bp_lookup_bucketed(x[j], W.s_key, W.s_bkt, W.s_val, E.n_bp, E.bp_key_lo, E.bp_shift,
                                                   E.bp_nbucket);
        }
#undef SI_BP_CHUNK
    } else if constexpr (MODE == EPI_DEQ_SIDE) {
        // [DEQ_ACC, ADD_SIDE(i)] (residual connection): f32(f64(a) * f64(s))
        // + side[i][n][m] in f32, the interpreter's two steps without it
        const float *sd = E.sides + (int64_t)__ldg(E.iparams + 3) * E.N * E.M + m;
        const int32_t adjM = (int32_t)((uint32_t)adj + (uint32_t)MAGIC_I);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int64_t n = n0 + j;
            const float d = fast ? __fmul_rn(__fsub_rn(__int_as_float((int32_t)(r[j] + (uint32_t)adjM)), MAGIC_F), s_in)
                                 : dev_deq_acc((int32_t)(r[j] + (uint32_t)adj), s_in);
            v[j] = (mok && n < P.N) ? __float_as_int(__fadd_rn(d, __ldg(sd + n * E.M))) : 0;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int64_t n = n0 + j;
            v[j] = (mok && n < P.N) ? (int32_t)epi_apply<MODE>((int32_t)(r[j] + (uint32_t)adj), m, n, E) : 0;
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
                if (n0 + j < P.N) reinterpret_cast<uint8_t *>(P.out)[(n0 + j) * P.ldo + m] = (uint8_t)(v[j] & 0xFF);
        }
    } else if constexpr (OUTK == OUT_U8_W || OUTK == OUT_S8_W) {
        // saturating pack of 4 consecutive tokens, quad transpose to 4
        // consecutive m, STS into this warp's [32 token][32 m] tile: the
        // lanes of one store cover 4 token rows x 32 bytes (conflict-free)
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            uint32_t word;
            if (OUTK == OUT_U8_W)
                word = tc::pack_sat_u8(v[4 * w + 1], v[4 * w], tc::pack_sat_u8(v[4 * w + 3], v[4 * w + 2], 0));
            else
                word = tc::pack_sat_s8(v[4 * w + 1], v[4 * w], tc::pack_sat_s8(v[4 * w + 3], v[4 * w + 2], 0));
            word = quad_transpose(word, W.selA, W.selB);
            *reinterpret_cast<uint32_t *>(W.stg + c * WSTG + (4 * w + W.u) * 32 + 4 * W.i4) = word;
        }
    }
}

// Epilogue of one accumulator tile for one warp (its 32 rows x 64 tokens),
// followed by the release of the accumulator and (8-bit) the TMA store of
// the group's staging tile.  row0 = first weight row of this CTA's 128-row
// half, tmem_col = accumulator column base.  release(): arrive on tempty.
template <int MODE, int OUTK, typename Wait, typename Release>
__device__ __forceinline__ void epi_tile(uint32_t tmem_base, uint32_t tmem_col, int32_t row0, int64_t tok0,
                                         const CUtensorMap *tmap_o, const K2Params &P, const EpiParams &E,
                                         const EpiWarp &W, Wait wait_full, Release release)
{
    // per-warp output: each warp stages its own [32 tokens][32 m] chunk (two
    // buffers) and stores it with its own TMA store: no cross-warp barrier
    constexpr bool PERWARP = (OUTK == OUT_U8_W || OUTK == OUT_S8_W);
    const int32_t m = row0 + W.q * 32 + W.lane;
    const bool mok = m < E.M;
    // per-row constants: issue the loads before blocking on the accumulator
    const int32_t adj = mok ? __ldg(E.adj + m) : 0;
    const float s_in = mok ? __ldg(E.scale_in + m) : 0.0f;
    float cq = 0.0f, cp = 0.0f;
    if (MODE == EPI_REQUANT) {
        cq = mok ? __ldg(P.rqc + m) : 0.0f;
        cp = mok ? __ldg(P.rqp + m) : 0.0f;
    }
    const float gr = mok ? __ldg(P.rqg + m) : 1.0f;
    // gm: 1 (2: I2F conversion) when every row of the warp is proven exact
    // (no certificate), else this row's certificate guard (proven rows: 0);
    // fast: every row stays inside the magic-number range
#ifdef SI_EXPERIMENTS
    if (P.exp & 1) {
        wait_full();
        tc::tc_fence_after();
        tc::tc_fence_before();
        __syncwarp();
        if (W.lane == 0) release();
        return;
    }
#endif
    const bool proven = __all_sync(0xffffffffu, gr >= 1.0f);
    const bool wide = __any_sync(0xffffffffu, gr >= 2.0f);
    const bool fast = !wide && __all_sync(0xffffffffu, gr >= 0.0f);
    const float gm = proven ? (wide ? 2.0f : 1.0f) : (gr >= 1.0f ? 0.0f : fmaxf(gr, 0.0f));
    if (proven) cq = cp;
    wait_full();
    tc::tc_fence_after();
    // the accumulator is released as soon as the last chunk is in registers
    // (before its math and staging), so the MMAs of the tile after next can
    // start that much earlier
    auto rel = [&]() {
        tc::tc_fence_before();
        __syncwarp();
        if (W.lane == 0) release();
    };
#pragma unroll 1
    for (int c = 0; c < COLS / 32; ++c) {
        const int col = W.g * COLS + c * 32;
        const uint32_t ta = tmem_base + ((uint32_t)(W.q * 32) << 16) + tmem_col + col;
        if constexpr (PERWARP) {
            // the store that last used this buffer (two chunks ago) has read it
            if (W.lane == 0) tc::tma_store_wait_read1();
            __syncwarp();
        }
        if (c == COLS / 32 - 1)
            epi_chunk<MODE, OUTK>(ta, m, mok, adj, s_in, cq, gm, fast, tok0 + col, c, P, E, W, rel);
        else
            epi_chunk<MODE, OUTK>(ta, m, mok, adj, s_in, cq, gm, fast, tok0 + col, c, P, E, W);
        if constexpr (PERWARP) {
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (W.lane == 0) {
                tc::tma_store_2d(tmap_o, W.stg + c * WSTG, row0 + W.q * 32, (int32_t)(tok0 + col));
                tc::tma_store_commit();
            }
        }
    }
}

template <int MODE, int NEPI = EPI_WARPS>
__device__ __forceinline__ EpiWarp make_epi_warp(int warp, int lane, uint8_t *staging, uint8_t *tables,
                                                 const EpiParams &E)
{
    EpiWarp W;
    W.q = warp & 3;
    W.g = (warp - 2) >> 2;
    W.lane = lane;
    W.u = lane & 3;
    W.i4 = lane >> 2;
    W.selA = (W.u & 1) ? 0x3715u : 0x6240u;
    W.selB = (W.u & 2) ? 0x3276u : 0x5410u;
    W.stg = staging + (warp - 2) * (2 * WSTG);   // this warp's two [32 tokens][32 m] staging buffers
    int32_t *s_key = reinterpret_cast<int32_t *>(tables);
    uint32_t *s_val = reinterpret_cast<uint32_t *>(tables + 4 * E.n_bp);
    uint16_t *s_bkt = reinterpret_cast<uint16_t *>(tables + 8 * E.n_bp + 4);
    if constexpr (MODE == EPI_DEQ_TABLE) {
        const int et = threadIdx.x - 64;
        if (E.bp_lin_n > 0) {
            // the linear table (<= 2048 entries of 8 bytes) takes the whole region
            uint2 *s_lin = reinterpret_cast<uint2 *>(tables);
            for (int i = et; i < E.bp_lin_n; i += 32 * NEPI) s_lin[i] = __ldg(E.bp_lin + i);
        } else {
            for (int i = et; i < E.n_bp; i += 32 * NEPI) s_key[i] = __ldg(E.bp_key + i);
            for (int i = et; i <= E.n_bp; i += 32 * NEPI) s_val[i] = __ldg(E.bp_v + i);
            for (int i = et; i < E.bp_nbucket; i += 32 * NEPI) s_bkt[i] = __ldg(E.bp_bucket + i);
        }
        tc::named_bar_sync(1 + EPI_GROUPS, 32 * NEPI);
    }
    W.s_key = s_key;
    W.s_val = s_val;
    W.s_bkt = s_bkt;
    return W;
}

template <int OUTK>
constexpr int staged_bytes() { return (OUTK == OUT_32 || OUTK == OUT_8_DIRECT) ? 0 : STG_BYTES; }
template <int MODE>
constexpr int table_bytes() { return MODE == EPI_DEQ_TABLE ? TABLE_BYTES : 0; }

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
               uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {pitch_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 3-D view for a token-major [N][K] activation: dims {128 (k in block), N,
// K/128 (block)}, so one box of {128, rows, blocks} lands as `blocks`
// consecutive K-major SWIZZLE_128B tiles of `rows` x 128 B.  Needs K % 128 == 0.
bool encode_3d_kblocks(CUtensorMap *m, const void *ptr, uint64_t n, uint64_t k, uint64_t pitch_bytes, uint32_t rows,
                       uint32_t blocks)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc || k % 128) return false;
    cuuint64_t dims[3] = {128, n, k / 128};
    cuuint64_t strides[2] = {pitch_bytes, 128};
    cuuint32_t box[3] = {128, rows, blocks};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// the dynamic shared-memory limit is a property of (function, device): set
// once per (kernel, device), under a lock (every instantiation of a kernel
// template has the same pointer type, so the key is the pointer value)
template <typename Kern>
void set_smem_attr(Kern kern, int smem)
{
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    const std::pair<const void *, int> key((const void *)kern, dev);
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert(key).second) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

int pick_mgroups(int mtiles, int ntiles, int npairs)
{
    // split each token tile's m-tiles into groups so units load-balance over
    // the pairs: minimise waves * (m-tiles per unit + X reload cost)
    int best_g = 1;
    double best = 1e30;
    for (int g = 1; g <= mtiles; ++g) {
        const long units = (long)ntiles * g;
        const long waves = (units + npairs - 1) / npairs;
        const double cost = (double)waves * ((double)((mtiles + g - 1) / g) + 0.25);
        if (cost < best - 1e-9) { best = cost; best_g = g; }
    }
    return best_g;
}

}  // namespace
