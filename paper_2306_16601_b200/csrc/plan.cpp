// plan.cpp -- host side of the C ABI: plan-image builder and program compiler.
//
// Replaces plan_spmm (spmm.py:160-189) + the device-facing half of
// build_program (epilogue.py:61-182).  Compiled with -ffp-contract=off so
// every host evaluation of the epilogue follows the reference's pinned f64
// expression trees (tensor.py:9-17, epilogue.py:190-249), calling the same
// glibc tanh/erf the reference's numba code calls.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <array>
#include <map>
#include <cfloat>
#include <string>
#include <vector>

#include "../../include/sparseinfer_b200.h"
#include "image.h"
#include "si_internal.h"

namespace {

thread_local std::string g_err;

uint64_t align16(uint64_t v) { return (v + 15) & ~uint64_t(15); }

inline int32_t wrap32(int64_t v) { return (int32_t)(uint32_t)(uint64_t)v; }

// ---- host evaluation of the reference's per-element chain ops -------------
// (_gelu_scalar epilogue.py:190-194; _quant_scalar :197-204; _run_chain :207-249)
float h_gelu_tanh(float x)
{
    double xd = (double)x;
    double t = 0.7978845608028654 * (xd + 0.044715 * xd * xd * xd);
    return (float)(0.5 * xd * (1.0 + std::tanh(t)));
}

float h_gelu_erf(float x)
{
    double xd = (double)x;
    return (float)(0.5 * xd * (1.0 + std::erf(xd * 0.7071067811865476)));
}

int32_t h_quant(double x, double scale, int32_t zp, int32_t lo, int32_t hi)
{
    double q = std::rint(x / scale) + (double)zp;
    if (q < (double)lo) q = (double)lo;
    if (q > (double)hi) q = (double)hi;
    return (int32_t)q;
}

struct State {
    int32_t xi = 0;
    float xf = 0.0f;
};

// Applies ops[s0:s1) (all per-tensor unary: LUT, DEQ, GELU*, QUANT) to a state.
void run_unary(const si_program *p, int s0, int s1, State &st)
{
    for (int s = s0; s < s1; ++s) {
        const int32_t *ip = p->iparams + 3 * s;
        switch (p->ops[s]) {
        case SI_OP_LUT: {
            int32_t key = ip[1] == 1 ? st.xi + 128 : st.xi;
            uint8_t b = p->luts[(int64_t)ip[0] * 256 + key];
            st.xi = ip[2] == 1 ? (int32_t)(int8_t)b : (int32_t)b;
            break;
        }
        case SI_OP_DEQ: {
            float t = (float)st.xi - (float)ip[0];
            st.xf = t * p->fparams[s];
            break;
        }
        case SI_OP_GELU: st.xf = h_gelu_tanh(st.xf); break;
        case SI_OP_GELU_ERF: st.xf = h_gelu_erf(st.xf); break;
        case SI_OP_QUANT:
            st.xi = h_quant((double)st.xf, (double)p->fparams[s], ip[0], ip[1], ip[2]);
            break;
        default: break;
        }
    }
}

bool is_unary(int32_t op)
{
    return op == SI_OP_LUT || op == SI_OP_DEQ || op == SI_OP_GELU || op == SI_OP_GELU_ERF ||
           op == SI_OP_QUANT;
}

// the live value after the program, as the 32-bit word the kernel stores
uint32_t final_word(const si_program *p, const State &st)
{
    if (p->out_dtype == SI_F32) {
        uint32_t u;
        std::memcpy(&u, &st.xf, 4);
        return u;
    }
    return (uint32_t)st.xi;
}

// ---- breakpoint table: x (f32 after DEQ_ACC) -> final word ---------------
// f32 values in total order via an int64 key.
int64_t f2key(float x)
{
    uint32_t u;
    std::memcpy(&u, &x, 4);
    return (u & 0x80000000u) ? -(int64_t)(u & 0x7fffffffu) : (int64_t)u;
}

float key2f(int64_t k)
{
    uint32_t u = k < 0 ? (0x80000000u | (uint32_t)(-k)) : (uint32_t)k;
    float x;
    std::memcpy(&x, &u, 4);
    return x;
}

struct BpTable {
    std::vector<float> x;     // thresholds: smallest x at which the value changes
    std::vector<uint32_t> v;  // v[i] for x in [x[i-1], x[i])
};

// f(x) = ops[1:) applied to xf = x.  Scans the whole finite f32 line at a
// fixed key stride and bisects every interval whose ends differ.  Exact as
// long as no value is entered and left again inside one stride (4096 ulps),
// which the program checks it cannot have been by re-evaluating 64 keys on
// each side of every threshold.
bool build_breakpoints(const si_program *p, BpTable &t)
{
    auto f = [&](int64_t key) {
        State st;
        st.xf = key2f(key);
        run_unary(p, 1, p->n_ops, st);
        return final_word(p, st);
    };
    const int64_t kmin = f2key(-FLT_MAX), kmax = f2key(FLT_MAX);
    const int64_t stride = 4096;
    t.x.clear();
    t.v.clear();
    int64_t prev_k = kmin;
    uint32_t prev_v = f(kmin);
    t.v.push_back(prev_v);
    for (int64_t k = kmin + stride;; k += stride) {
        if (k > kmax) k = kmax;
        uint32_t v = f(k);
        if (v != prev_v) {
            // bisect (prev_k, k]: find the smallest key with value != prev_v
            int64_t lo = prev_k, hi = k;
            while (hi - lo > 1) {
                int64_t mid = lo + (hi - lo) / 2;
                if (f(mid) == prev_v) lo = mid; else hi = mid;
            }
            uint32_t vh = f(hi);
            // the stretch (hi, k] must be constant vh, else a level was skipped
            for (int64_t q = hi; q <= k; q += (k - hi) / 64 + 1)
                if (f(q) != vh) return false;
            t.x.push_back(key2f(hi));
            t.v.push_back(vh);
            prev_v = vh;
            if (vh != v) return false;
        }
        prev_k = k;
        if (k == kmax) break;
        if (t.x.size() > 4096) return false;
    }
    // local re-check around every threshold
    for (size_t i = 0; i < t.x.size(); ++i) {
        int64_t k0 = f2key(t.x[i]);
        for (int64_t d = -64; d < 64; ++d) {
            int64_t k = k0 + d;
            if (k < kmin || k > kmax) continue;
            uint32_t want = d < 0 ? t.v[i] : t.v[i + 1];
            if (f(k) != want) return false;
        }
    }
    return true;
}

struct Compiled {
    int32_t mode = EPI_GENERIC;
    int32_t exact = 1;
    float q_scale = 0, q_inv = 0;
    int32_t q_zp = 0, q_lo = 0, q_hi = 0;
    std::vector<uint32_t> clut;
    BpTable bp;
    int32_t bp_key_lo = 0, bp_shift = 0, bp_occ = 0;
    std::vector<uint16_t> bp_bucket;
    // linear buckets with at most one threshold each (device fast path)
    std::vector<uint32_t> bp_lin;   // 2 words per bucket
    float bp_lin_inv = 0, bp_lin_off = 0;
};

// Coarse index over the thresholds in f32 key space: bucket b covers keys
// [key_lo + (b << shift), key_lo + ((b+1) << shift)); bucket[b] is the number
// of thresholds with key < bucket start.  A lookup then scans a handful of
// thresholds instead of a 9-step binary search.
void build_buckets(Compiled &c)
{
    const size_t n = c.bp.x.size();
    if (n == 0) return;
    const int64_t lo = f2key(c.bp.x[0]), hi = f2key(c.bp.x[n - 1]);
    int shift = 0;
    while (((hi - lo) >> shift) >= 2048) ++shift;
    const int64_t nb = ((hi - lo) >> shift) + 1;
    c.bp_key_lo = (int32_t)lo;
    c.bp_shift = shift;
    c.bp_bucket.assign((size_t)nb, 0);
    size_t i = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t start = lo + (b << shift);
        while (i < n && f2key(c.bp.x[i]) < start) ++i;
        c.bp_bucket[(size_t)b] = (uint16_t)i;
    }
    // most thresholds any bucket holds: a lookup never advances further than
    // that from bucket[b], so the device can take a fixed, divergence-free
    // number of steps
    int32_t occ = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t next = b + 1 < nb ? c.bp_bucket[(size_t)b + 1] : (int64_t)n;
        occ = std::max<int32_t>(occ, (int32_t)(next - c.bp_bucket[(size_t)b]));
    }
    c.bp_occ = occ;
}

// The device's bucket function (k2_common.cuh epi_chunk, EPI_DEQ_TABLE): one
// f32 fma, a clamp and round-to-nearest-even.  It is monotone in x, so for x
// in bucket b every threshold in a lower bucket is < x and every threshold in
// a higher bucket is > x: with at most one threshold per bucket the piece of x
// is decided by one compare.
static inline int32_t lin_bucket(float x, float inv, float off, int32_t nb)
{
    float t = fmaf(x, inv, off);
    t = fminf(fmaxf(t, 0.0f), (float)(nb - 1));
    return (int32_t)nearbyintf(t);
}

// Smallest power-of-two bucket count (<= 2048: 16 KB of 8-byte entries) under
// which no bucket holds two thresholds; values must fit 16 bits.
void build_linear(Compiled &c)
{
    const size_t n = c.bp.x.size();
    if (n == 0) return;
    for (uint32_t v : c.bp.v) {
        const int32_t sv = (int32_t)v;
        if (sv < -32768 || sv > 32767) return;
    }
    const float lo = c.bp.x[0], hi = c.bp.x[n - 1];
    if (!(hi > lo) && n > 1) return;
    for (int32_t nb = 64; nb <= 2048; nb *= 2) {
        const float inv = n > 1 ? (float)((double)(nb - 1) / ((double)hi - (double)lo)) : 0.0f;
        const float off = -lo * inv;
        if (!std::isfinite(inv) || !std::isfinite(off)) continue;
        std::vector<int32_t> first((size_t)nb, -1);
        bool ok = true;
        int32_t prev = -1;
        for (size_t i = 0; i < n && ok; ++i) {
            const int32_t b = lin_bucket(c.bp.x[i], inv, off, nb);
            ok = b > prev;            // strictly increasing: one threshold per bucket, order kept
            prev = b;
            if (ok) first[(size_t)b] = (int32_t)i;
        }
        if (!ok) continue;
        c.bp_lin.assign((size_t)2 * nb, 0);
        size_t before = 0;           // thresholds in lower buckets
        for (int32_t b = 0; b < nb; ++b) {
            float thr = INFINITY;
            uint32_t vlo = c.bp.v[before], vhi = vlo;
            if (first[(size_t)b] >= 0) {
                thr = c.bp.x[(size_t)first[(size_t)b]];
                vhi = c.bp.v[before + 1];
                ++before;
            }
            uint32_t tb;
            std::memcpy(&tb, &thr, 4);
            c.bp_lin[(size_t)2 * b] = tb;
            c.bp_lin[(size_t)2 * b + 1] = (vlo & 0xFFFFu) | (vhi << 16);
        }
        c.bp_lin_inv = inv;
        c.bp_lin_off = off;
        return;
    }
}

Compiled compile_program(const si_program *p)
{
    Compiled c;
    const int L = p->n_ops;
    bool has_gelu = false, has_side = false;
    for (int s = 0; s < L; ++s) {
        has_gelu |= p->ops[s] == SI_OP_GELU || p->ops[s] == SI_OP_GELU_ERF;
        has_side |= p->ops[s] == SI_OP_ADD_SIDE || p->ops[s] == SI_OP_ADD_CHAN;
    }
    if (L == 0) { c.mode = EPI_S32; return c; }
    if (L == 1 && p->ops[0] == SI_OP_DEQ_ACC && p->out_dtype == SI_F32) {
        c.mode = EPI_DEQ_F32;
        return c;
    }
    if (L == 2 && p->ops[0] == SI_OP_DEQ_ACC && p->ops[1] == SI_OP_ADD_SIDE && p->out_dtype == SI_F32) {
        c.mode = EPI_DEQ_SIDE;
        return c;
    }
    bool tail_unary = true;
    for (int s = 1; s < L; ++s) tail_unary &= is_unary(p->ops[s]);
    if (p->ops[0] == SI_OP_REQUANT) {
        const int32_t *ip = p->iparams;
        c.q_scale = p->fparams[0];
        c.q_inv = (float)(1.0 / (double)p->fparams[0]);
        c.q_zp = ip[0]; c.q_lo = ip[1]; c.q_hi = ip[2];
        if (L == 1) { c.mode = EPI_REQUANT; return c; }
        if (tail_unary && c.q_hi - c.q_lo < 256) {
            c.mode = EPI_REQUANT_LUT;
            c.clut.assign(256, 0);
            for (int32_t q = c.q_lo; q <= c.q_hi; ++q) {
                State st;
                st.xi = q;
                run_unary(p, 1, L, st);
                c.clut[q - c.q_lo] = final_word(p, st);
            }
            return c;
        }
    }
    if (p->ops[0] == SI_OP_DEQ_ACC && tail_unary) {
        // the f32 chain must end in an integer state for a finite table
        bool reaches_int = false;
        for (int s = 1; s < L; ++s) reaches_int |= p->ops[s] == SI_OP_QUANT;
        if (reaches_int && build_breakpoints(p, c.bp)) {
            build_buckets(c);
            // keys + values + buckets must fit the kernels' 16 KB smem table
            if (8 * c.bp.x.size() + 4 + 2 * c.bp_bucket.size() <= 16384) {
                c.mode = EPI_DEQ_TABLE;
                build_linear(c);
                return c;
            }
            c.bp = BpTable();
            c.bp_bucket.clear();
        }
    }
    c.mode = EPI_GENERIC;
    c.exact = has_gelu ? 0 : 1;
    (void)has_side;
    return c;
}

struct Layout {
    uint64_t off[30];
    uint64_t total;
};



// True when the device's proven-row requant, n(a) = bits(fma(f32(a), c,
// 1.5*2^23 + zp)) - bits(1.5*2^23) = rint(a*c + zp) (one rounding, exact while
// |a*c + zp| < 2^22) saturated to [lo, hi], equals the reference's
// rint((f64(a) * s) / fp) + zp clamped (epilogue.py:218-228) for every
// integer |a| <= A.  Both are monotone in a, so they agree everywhere iff
// every output step (k-1 -> k, lo < k <= hi) happens at the same a; each
// step is located from its estimate by exact evaluation of both sides.
static bool requant_fma_exact(int64_t A, float s_in, float fp, float c, int32_t zp, int32_t lo, int32_t hi)
{
    const double q = (double)s_in / (double)fp;
    if (!(c != 0.0f) || !std::isfinite(c) || !std::isfinite(q) || q == 0.0 || (c > 0) != (q > 0)) return false;
    if ((double)A * std::fabs((double)c) + std::fabs((double)zp) >= 2097152.0) return false;
    const float mz = 12582912.0f + (float)zp;
    const int64_t sg = c > 0 ? 1 : -1;
    auto Rd = [&](int64_t t) {
        const float u = std::fmaf((float)(sg * t), c, mz);
        return (int64_t)u - 12582912;
    };
    auto Ry = [&](int64_t t) {
        const double y = ((double)(sg * t) * (double)s_in) / (double)fp;
        return (int64_t)std::nearbyint(y) + zp;
    };
    auto step = [&](auto R, int64_t k, int64_t &out) {
        // smallest t in [-A, A + 1] with R(t) >= k (A + 1: never)
        double est = std::ceil(((double)(k - zp) - 0.5) / std::fabs(q));
        est = std::min(std::max(est, (double)-A), (double)(A + 1));
        int64_t t = (int64_t)est;
        int steps = 0;
        while (t > -A && R(t - 1) >= k) { --t; if (++steps > 4096) return false; }
        while (t <= A && R(t) < k) { ++t; if (++steps > 4096) return false; }
        out = t;
        return true;
    };
    for (int64_t k = (int64_t)lo + 1; k <= (int64_t)hi; ++k) {
        int64_t tr = 0, ty = 0;
        if (!step(Rd, k, tr) || !step(Ry, k, ty) || tr != ty) return false;
    }
    return true;
}

// Search f32 multipliers near f32(s / fp) for one that makes the proven-row
// requant exact for this row (requant_fma_exact); 0 if none within 32 ulps.
static float requant_find_multiplier(int64_t A, float s_in, float fp, int32_t zp, int32_t lo, int32_t hi)
{
    const float c0 = (float)((double)s_in / (double)fp);
    if (requant_fma_exact(A, s_in, fp, c0, zp, lo, hi)) return c0;
    float up = c0, dn = c0;
    for (int i = 0; i < 32; ++i) {
        up = std::nextafter(up, INFINITY);
        dn = std::nextafter(dn, -INFINITY);
        if (requant_fma_exact(A, s_in, fp, up, zp, lo, hi)) return up;
        if (requant_fma_exact(A, s_in, fp, dn, zp, lo, hi)) return dn;
    }
    return 0.0f;
}

// 2:4 images of K3 (see image.h).  A window (group, 4 consecutive k) keeps
// its first two nonzero columns in the compressed operand; further columns
// go to the per-row residual lists.
struct SparseImages {
    std::vector<uint8_t> img;
    std::vector<int32_t> rptr;
    std::vector<int32_t> res;
    int32_t maxres = 0;
    // K3 residual operand (image.h): per 256-row pair tile
    std::vector<uint8_t> tr_img;    // [pair tiles * 2][12288]
    std::vector<uint16_t> tr_k;     // [pair tiles][TR_SLOTS]
    std::vector<int32_t> tr_cnt;    // [pair tiles] residual MMAs (64 slots each)
    int32_t tr_ok = 1;
};

// Write one 4-wide window of a 2:4 image tile (12 KB: compressed A
// [128 rows x 64 B] K-major SWIZZLE_NONE core matrices + two metadata tiles):
// window wl (0..31) of row `row`, entries (position in window, value) sorted by
// position, at most two.
static void sp_put_window(uint8_t *tile, int32_t row, int32_t wl, const std::pair<int32_t, uint8_t> *ent, int n)
{
    int32_t idx0 = 0, idx1 = 1;
    uint8_t v0 = 0, v1 = 0;
    if (n == 2) {
        idx0 = ent[0].first; v0 = ent[0].second;
        idx1 = ent[1].first; v1 = ent[1].second;
    } else if (n == 1) {
        if (ent[0].first == 3) { idx0 = 0; idx1 = 3; v1 = ent[0].second; }
        else { idx0 = ent[0].first; idx1 = 3; v0 = ent[0].second; }
    }
    auto aoff = [&](int32_t pb) { return (row / 8) * 512 + (pb / 16) * 128 + (row % 8) * 16 + (pb % 16); };
    tile[aoff(2 * wl)] = v0;
    tile[aoff(2 * wl + 1)] = v1;
    const int32_t mma = wl / 16, wm = wl % 16;
    const uint8_t nib = (uint8_t)(idx0 | (idx1 << 2));
    uint8_t *e = tile + 8192 + mma * 2048 + (row / 8) * 128 + (row % 8) * 16 + wm / 2;
    *e = (uint8_t)((*e & ((wm % 2) ? 0x0F : 0xF0)) | ((wm % 2) ? (nib << 4) : nib));
}

// K3: the residual columns of a 256-row pair tile become one more 2:4
// operand over "slots": slot s holds activation column tr_k[s] (gathered
// on-chip from the resident X tile), so the residual is one or two extra
// sparse MMAs instead of per-element epilogue work.  Slots are assigned
// greedily so that no row holds more than two entries in any 4-slot window;
// a pair tile needing more than TR_SLOTS slots disables K3 (tr_ok = 0).
static void build_tr_sections(SparseImages &S, const std::vector<std::vector<int32_t>> &rres, int32_t rt_n,
                              int32_t rt_pad)
{
    const int32_t pt_n = rt_pad / 2;
    S.tr_img.assign((size_t)rt_pad * 12288, 0);
    S.tr_k.assign((size_t)pt_n * TR_SLOTS, 0);
    S.tr_cnt.assign((size_t)pt_n, 0);
    for (int32_t pt = 0; pt < pt_n; ++pt) {
        // column -> rows (local 0..255) holding a residual there
        std::map<int32_t, std::vector<std::pair<int32_t, uint8_t>>> bycol;
        for (int32_t lr = 0; lr < 256; ++lr) {
            const int32_t rt = 2 * pt + lr / 128;
            if (rt >= rt_n) continue;
            for (int32_t ent : rres[(size_t)rt * 128 + lr % 128]) bycol[ent >> 8].emplace_back(lr, (uint8_t)(ent & 0xFF));
        }
        std::vector<std::array<uint8_t, TR_SLOTS / 4>> cnt(256);
        for (auto &c : cnt) c.fill(0);
        std::vector<int32_t> slot_col(TR_SLOTS, -1);
        std::vector<std::vector<std::pair<int32_t, uint8_t>>> slot_rows(TR_SLOTS);
        int32_t used = 0;
        for (auto &kv : bycol) {
            int32_t s = 0;
            for (; s < TR_SLOTS; ++s) {
                if (slot_col[s] >= 0) continue;
                bool ok = true;
                for (auto &rv : kv.second)
                    if (cnt[rv.first][s / 4] >= 2) { ok = false; break; }
                if (ok) break;
            }
            if (s == TR_SLOTS) { S.tr_ok = 0; break; }
            slot_col[s] = kv.first;
            slot_rows[s] = kv.second;
            for (auto &rv : kv.second) ++cnt[rv.first][s / 4];
            used = std::max(used, s + 1);
        }
        if (!S.tr_ok) break;
        S.tr_cnt[pt] = (used + 63) / 64;
        for (int32_t s = 0; s < TR_SLOTS; ++s) S.tr_k[(size_t)pt * TR_SLOTS + s] = slot_col[s] >= 0 ? (uint16_t)slot_col[s] : (uint16_t)0xFFFF;
        // per row and window: the (position, value) entries
        std::vector<std::vector<std::pair<int32_t, uint8_t>>> win((size_t)256 * (TR_SLOTS / 4));
        for (int32_t s = 0; s < TR_SLOTS; ++s)
            for (auto &rv : slot_rows[s]) win[(size_t)rv.first * (TR_SLOTS / 4) + s / 4].emplace_back(s % 4, rv.second);
        for (int32_t lr = 0; lr < 256; ++lr) {
            uint8_t *tile = S.tr_img.data() + ((size_t)2 * pt + lr / 128) * 12288;
            for (int32_t wl = 0; wl < TR_SLOTS / 4; ++wl) {
                auto &e = win[(size_t)lr * (TR_SLOTS / 4) + wl];
                std::sort(e.begin(), e.end());
                sp_put_window(tile, lr % 128, wl, e.data(), (int)e.size());
            }
        }
    }
    if (!S.tr_ok) {
        std::fill(S.tr_cnt.begin(), S.tr_cnt.end(), 0);
        std::fill(S.tr_img.begin(), S.tr_img.end(), 0);
    }
}

SparseImages build_sparse_images(const si_weight *w)
{
    SparseImages S;
    const int32_t G = w->rows / 4;
    const int32_t rt_n = (w->logical_rows + 127) / 128;
    const int32_t kch = (w->cols + 127) / 128;
    const int32_t rt_pad = (rt_n + 1) / 2 * 2;   // whole 256-row pair tiles
    S.img.assign((size_t)rt_pad * kch * 12288, 0);
    std::vector<std::vector<int32_t>> rres((size_t)rt_n * 128);
    for (int32_t g = 0; g < G && g / 32 < rt_n; ++g) {
        const int32_t rt = g / 32, gl = g % 32;
        // dense 4-row strip of this group: column -> 4 values (summing duplicates, int8 wrap)
        std::vector<std::pair<int32_t, uint32_t>> cols;
        for (int64_t q = w->group_ptr[g]; q < w->group_ptr[g + 1]; ++q) {
            uint32_t word = 0;
            for (int r = 0; r < 4; ++r) {
                uint8_t b = (uint8_t)w->vals[(q / 4) * 16 + r * 4 + (q % 4)];
                if (g * 4 + r >= w->logical_rows) b = 0;
                word |= (uint32_t)b << (8 * r);
            }
            if (!word) continue;
            bool merged = false;
            for (auto &c : cols)
                if (c.first == w->idx[q]) {
                    uint32_t sum = 0;
                    for (int r = 0; r < 4; ++r)
                        sum |= (uint32_t)(uint8_t)((int8_t)(c.second >> (8 * r)) + (int8_t)(word >> (8 * r))) << (8 * r);
                    c.second = sum;
                    merged = true;
                    break;
                }
            if (!merged) cols.emplace_back(w->idx[q], word);
        }
        std::sort(cols.begin(), cols.end());
        size_t i = 0;
        while (i < cols.size()) {
            const int32_t win = cols[i].first / 4;
            size_t j = i;
            while (j < cols.size() && cols[j].first / 4 == win) ++j;
            const int32_t kc = win / 32, wl = win % 32;     // window within the 128-k chunk
            uint8_t *tile = S.img.data() + ((size_t)rt * kch + kc) * 12288;
            // slots: up to two kept columns, ascending window index
            int32_t idx0 = 0, idx1 = 1;
            uint32_t v0 = 0, v1 = 0;
            const size_t kept = std::min<size_t>(2, j - i);
            if (kept == 2) {
                idx0 = cols[i].first % 4; v0 = cols[i].second;
                idx1 = cols[i + 1].first % 4; v1 = cols[i + 1].second;
            } else if (kept == 1) {
                const int32_t ii = cols[i].first % 4;
                if (ii == 3) { idx0 = 0; idx1 = 3; v1 = cols[i].second; }
                else { idx0 = ii; idx1 = 3; v0 = cols[i].second; }
            }
            for (size_t e = i + kept; e < j; ++e)
                for (int r = 0; r < 4; ++r) {
                    const int8_t v = (int8_t)(cols[e].second >> (8 * r));
                    if (v) rres[(size_t)rt * 128 + gl * 4 + r].push_back((cols[e].first << 8) | (uint8_t)v);
                }
            const int32_t mma = wl / 16, wm = wl % 16;        // MMA (64 logical k) and window in it
            const uint8_t nib = (uint8_t)(idx0 | (idx1 << 2));
            for (int r = 0; r < 4; ++r) {
                const int32_t row = gl * 4 + r;
                const int32_t pb0 = 2 * wl, pb1 = 2 * wl + 1;  // physical bytes of the window
                auto aoff = [&](int32_t pb) {
                    return (row / 8) * 512 + (pb / 16) * 128 + (row % 8) * 16 + (pb % 16);
                };
                tile[aoff(pb0)] = (uint8_t)(v0 >> (8 * r));
                tile[aoff(pb1)] = (uint8_t)(v1 >> (8 * r));
                uint8_t *e = tile + 8192 + mma * 2048 + (row / 8) * 128 + (row % 8) * 16 + wm / 2;
                *e |= (wm % 2) ? (uint8_t)(nib << 4) : nib;
            }
            i = j;
        }
    }
    // windows never touched keep metadata 0 = (idx 0, idx 0) over zero values:
    // rewrite them to the canonical (0, 1)
    for (size_t t = 0; t < (size_t)rt_pad * kch; ++t)
        for (int mma = 0; mma < 2; ++mma)
            for (int row = 0; row < 128; ++row) {
                uint8_t *e = S.img.data() + t * 12288 + 8192 + mma * 2048 + (row / 8) * 128 + (row % 8) * 16;
                for (int b = 0; b < 8; ++b)
                    for (int h = 0; h < 2; ++h) {
                        const uint8_t nib = (e[b] >> (4 * h)) & 0xF;
                        if (nib == 0) e[b] |= (uint8_t)(0x4 << (4 * h));
                    }
            }
    S.rptr.assign((size_t)rt_n * 128 + 1, 0);
    for (size_t r = 0; r < rres.size(); ++r) {
        S.rptr[r] = (int32_t)S.res.size();
        S.maxres = std::max<int32_t>(S.maxres, (int32_t)rres[r].size());
        S.res.insert(S.res.end(), rres[r].begin(), rres[r].end());
    }
    S.rptr[rres.size()] = (int32_t)S.res.size();
    build_tr_sections(S, rres, rt_n, rt_pad);
    return S;
}


}  // namespace

void si_set_error(const std::string &msg) { g_err = msg; }

extern "C" const char *si_last_error(void) { return g_err.c_str(); }

extern "C" int32_t si_abi_version(void) { return SI_ABI_VERSION; }

static int32_t validate(const si_weight *w, const si_program *p)
{
    if (!w || !p) { si_set_error("null weight/program"); return SI_EINVAL; }
    if (w->rows <= 0 || w->rows % 4 || w->cols <= 0 || w->logical_rows <= 0 ||
        w->logical_rows > w->rows || w->rows - w->logical_rows >= 4) {
        si_set_error("bad weight geometry");
        return SI_EINVAL;
    }
    if (p->m != w->logical_rows) {
        si_set_error("program channel count must match weight rows");
        return SI_EINVAL;
    }
    const int32_t G = w->rows / 4;
    if (w->group_ptr[0] != 0) { si_set_error("group_ptr[0] != 0"); return SI_EFORMAT; }
    for (int32_t g = 0; g < G; ++g) {
        int32_t a = w->group_ptr[g], b = w->group_ptr[g + 1];
        if (b < a || (b - a) % 4) {
            si_set_error("group_ptr must be non-decreasing multiples of 4");
            return SI_EFORMAT;
        }
    }
    int64_t T = w->group_ptr[G];
    for (int64_t t = 0; t < T; ++t)
        if (w->idx[t] < 0 || w->idx[t] >= w->cols) {
            si_set_error("column index out of range");
            return SI_EFORMAT;
        }
    for (int s = 0; s < p->n_ops; ++s) {
        int32_t op = p->ops[s];
        if (op < 0 || op > SI_OP_GELU_ERF) { si_set_error("unknown opcode"); return SI_EINVAL; }
        if (op == SI_OP_LUT && (p->iparams[3 * s] < 0 || p->iparams[3 * s] >= p->n_luts)) {
            si_set_error("lut index out of range");
            return SI_EINVAL;
        }
        if (op == SI_OP_ADD_CHAN && (p->iparams[3 * s] < 0 || p->iparams[3 * s] >= p->n_chans)) {
            si_set_error("channel vector index out of range");
            return SI_EINVAL;
        }
        if ((op == SI_OP_REQUANT || op == SI_OP_QUANT || op == SI_OP_DEQ) && !(p->fparams[s] > 0)) {
            si_set_error("quantization scale must be positive");
            return SI_EINVAL;
        }
    }
    return SI_OK;
}

static Layout make_layout(const si_weight *w, const si_program *p, const Compiled &c, const SparseImages &sp)
{
    Layout l{};
    const int64_t G = w->rows / 4, T = w->group_ptr[G], tiles = T / 4;
    const int64_t M = w->logical_rows;
    const int64_t mt = (M + 127) / 128, kp = (w->cols + 127) / 128 * 128;
    // every section starts on a 1024-byte boundary: the TMA boxes of the
    // tensor-core operand sections read 128-byte rows, and a row straddling two
    // L2 lines doubles the line requests (the W^T section used to sit at 16 or
    // 80 mod 128)
    auto align1k = [](uint64_t v) { return (v + 1023) & ~uint64_t(1023); };
    uint64_t cur = align1k(sizeof(SiImage));
    auto put = [&](int i, uint64_t bytes) { l.off[i] = cur; cur = align1k(cur + bytes); };
    put(0, 4 * (G + 1));
    put(1, 16 * tiles);
    put(2, 16 * tiles);
    put(3, 4 * M);
    put(4, 4 * M);
    put(5, 4 * (uint64_t)p->n_ops);
    put(6, 4 * (uint64_t)p->n_ops);
    put(7, 4 * (uint64_t)p->n_ops);
    put(8, 12 * (uint64_t)p->n_ops);
    put(9, 256 * (uint64_t)p->n_luts);
    put(10, 4 * (uint64_t)p->n_chans * M);
    put(11, 4 * 256);
    put(12, 4 * c.bp.x.size());
    put(13, 4 * (c.bp.v.size() + 1));
    put(14, (uint64_t)kp * mt * 128);
    put(15, 4 * M);
    put(16, 4 * c.bp.x.size());
    put(17, 2 * c.bp_bucket.size());
    put(18, 0);   // (image v4: K2x expansion lists, retired)
    put(19, 0);
    put(20, 4 * M);
    put(21, sp.img.size());
    put(22, 4 * sp.rptr.size());
    put(23, 4 * sp.res.size());
    put(24, 4 * M);
    put(25, sp.tr_img.size());
    put(26, 2 * sp.tr_k.size());
    put(27, 4 * sp.tr_cnt.size());
    put(28, 0);   // (image v4: K2a row-major W, retired)
    put(29, 4 * c.bp_lin.size());
    l.total = cur;
    return l;
}

extern "C" int32_t si_plan_image_size(const si_weight *w, const si_program *p, uint64_t *bytes)
{
    int32_t rc = validate(w, p);
    if (rc) return rc;
    Compiled c = compile_program(p);
    SparseImages sp = build_sparse_images(w);
    *bytes = make_layout(w, p, c, sp).total;
    return SI_OK;
}

extern "C" int32_t si_plan_image_build(const si_weight *w, const si_program *p, const int32_t *bias,
                                       void *host_image, uint64_t bytes)
{
    int32_t rc = validate(w, p);
    if (rc) return rc;
    Compiled c = compile_program(p);
    SparseImages sp = build_sparse_images(w);
    Layout l = make_layout(w, p, c, sp);
    if (bytes < l.total) { si_set_error("image buffer too small"); return SI_ENOSPACE; }
    uint8_t *base = (uint8_t *)host_image;
    std::memset(base, 0, l.total);
    SiImage *h = (SiImage *)base;
    const int32_t G = w->rows / 4;
    const int64_t T = w->group_ptr[G], tiles = T / 4, M = w->logical_rows, K = w->cols;
    h->magic = SI_IMG_MAGIC;
    h->version = SI_IMG_VERSION;
    h->M = (int32_t)M; h->K = (int32_t)K; h->rows = w->rows; h->groups = G;
    h->padded_blocks = T; h->tiles = tiles;
    h->out_dtype = p->out_dtype; h->a_zp = p->a_zp;
    h->n_ops = p->n_ops; h->n_luts = p->n_luts; h->n_chans = p->n_chans; h->n_sides = p->n_sides;
    h->epi_mode = c.mode; h->exact = c.exact;
    h->q_scale = c.q_scale; h->q_inv = c.q_inv; h->q_zp = c.q_zp; h->q_lo = c.q_lo; h->q_hi = c.q_hi;
    h->n_bp = (int32_t)c.bp.x.size();
    h->tc_mtiles = (int32_t)((M + 127) / 128);
    h->tc_kpad = (int32_t)((K + 127) / 128 * 128);
    uint64_t *offs = &h->off_tile_ptr;
    for (int i = 0; i < 15; ++i) offs[i] = l.off[i];
    h->total_bytes = l.total;
    h->off_rqc = l.off[15];
    h->off_bp_key = l.off[16];
    h->off_bp_bucket = l.off[17];
    h->bp_key_lo = c.bp_key_lo;
    h->bp_shift = c.bp_shift;
    h->bp_occ = c.bp_occ;
    h->bp_nbucket = (int32_t)c.bp_bucket.size();
    h->off_bp_lin = l.off[29];
    h->bp_lin_n = (int32_t)(c.bp_lin.size() / 2);
    h->bp_lin_inv = c.bp_lin_inv;
    h->bp_lin_off = c.bp_lin_off;
    h->off_rqg = l.off[20];
    h->off_sp_img = l.off[21];
    h->off_sp_rptr = l.off[22];
    h->off_sp_res = l.off[23];
    h->off_rqp = l.off[24];
    h->sp_nres = (int32_t)sp.res.size();
    h->sp_maxres = sp.maxres;
    h->off_tr_img = l.off[25];
    h->off_tr_k = l.off[26];
    h->off_tr_cnt = l.off[27];
    h->tr_ok = sp.tr_ok;
    h->tr_pairs = (int32_t)sp.tr_cnt.size();
    h->off_tc_wrow = l.off[28];
    std::memcpy(base + h->off_tr_img, sp.tr_img.data(), sp.tr_img.size());
    std::memcpy(base + h->off_tr_k, sp.tr_k.data(), 2 * sp.tr_k.size());
    std::memcpy(base + h->off_tr_cnt, sp.tr_cnt.data(), 4 * sp.tr_cnt.size());
    std::memcpy(base + h->off_sp_img, sp.img.data(), sp.img.size());
    std::memcpy(base + h->off_sp_rptr, sp.rptr.data(), 4 * sp.rptr.size());
    if (!sp.res.empty()) std::memcpy(base + h->off_sp_res, sp.res.data(), 4 * sp.res.size());
    h->off_tc_eptr = l.off[18];
    h->off_tc_ent = l.off[19];
    h->tc_emax = 0;
    h->tc_nlists = 0;

    // micro-tiles: reference layout kept verbatim (sparse.py:28-31)
    int32_t *tp = (int32_t *)(base + h->off_tile_ptr);
    for (int32_t g = 0; g <= G; ++g) tp[g] = w->group_ptr[g] / 4;
    std::memcpy(base + h->off_tile_w, w->vals, (size_t)(16 * tiles));
    std::memcpy(base + h->off_tile_idx, w->idx, (size_t)(4 * T));

    // compensation (sparse.py:51-62) and adj (spmm.py:231), int32 wrap
    int64_t nnz = 0;
    int32_t *adj = (int32_t *)(base + h->off_adj);
    for (int32_t g = 0; g < G; ++g) {
        int64_t s[4] = {0, 0, 0, 0};
        for (int64_t q = w->group_ptr[g]; q < w->group_ptr[g + 1]; ++q) {
            bool any = false;
            for (int r = 0; r < 4; ++r) {
                int8_t v = w->vals[(q / 4) * 16 + r * 4 + (q % 4)];
                s[r] += v;
                any |= v != 0;
            }
            nnz += any;
        }
        for (int r = 0; r < 4; ++r) {
            int64_t m = (int64_t)g * 4 + r;
            if (m >= M) break;
            int32_t comp = wrap32(s[r]);
            int64_t b = bias ? bias[m] : 0;
            adj[m] = wrap32(b - (int64_t)p->a_zp * (int64_t)comp);
        }
    }
    h->nnz_blocks = nnz;

    // per-row bound on |acc + adj| (u8 activations <= 255): rows whose bound
    // stays below 2^22 never leave the magic-number range (rqg >= 0).  For
    // requant, rows with a multiplier c' (rqp) under which the one-rounding
    // fma form provably matches the reference's f64 rounding for every
    // reachable accumulator get rqg = 1 (no certificate); the other rows get
    // the certificate guard 2^-22 * max|r| as a per-row constant (0 <= rqg <= 1/4).
    {
        float *rqg = (float *)(base + h->off_rqg);
        float *rqp = (float *)(base + h->off_rqp);
        for (int32_t g = 0; g < G; ++g) {
            int64_t sabs[4] = {0, 0, 0, 0};
            for (int64_t q = w->group_ptr[g]; q < w->group_ptr[g + 1]; ++q)
                for (int r = 0; r < 4; ++r) {
                    const int v = w->vals[(q / 4) * 16 + r * 4 + (q % 4)];
                    sabs[r] += v < 0 ? -v : v;
                }
            for (int r = 0; r < 4; ++r) {
                const int64_t m = (int64_t)g * 4 + r;
                if (m >= M) break;
                const int64_t a = adj[m] < 0 ? -(int64_t)adj[m] : (int64_t)adj[m];
                const int64_t bound = 255 * sabs[r] + a;
                if (c.mode == EPI_REQUANT && bound < 16777216) {
                    // proven rows: 1 = accumulator converts by the magic number
                    // (|a| < 2^22), 2 = by I2F (|a| < 2^24, exact)
                    const float cp = requant_find_multiplier(bound, p->scale_in[m], c.q_scale, c.q_zp, c.q_lo, c.q_hi);
                    rqp[m] = cp;
                    if (cp != 0.0f) rqg[m] = bound < 4194304 ? 1.0f : 2.0f;
                }
                if (rqg[m] >= 1.0f) {
                } else if (bound >= 4194304) {
                    rqg[m] = -1.0f;
                } else if (c.mode == EPI_REQUANT) {
                    const float cm = (float)((double)p->scale_in[m] / (double)c.q_scale);
                    {
                        // certificate guard 2^-22 * max|r| (max|r| <= bound * |c|), rounded up
                        const double g = (double)bound * std::fabs((double)cm) * 2.384185791015625e-07 * (1.0 + 1.0 / 1024);
                        rqg[m] = (float)std::min(g * (1.0 + 1e-6) + 1e-30, 0.25);
                    }
                } else {
                    rqg[m] = 0.0f;
                }
            }
        }
    }

    std::memcpy(base + h->off_scale_in, p->scale_in, 4 * (size_t)M);
    if (p->n_ops) {
        std::memcpy(base + h->off_ops, p->ops, 4 * (size_t)p->n_ops);
        std::memcpy(base + h->off_fparams, p->fparams, 4 * (size_t)p->n_ops);
        float *finv = (float *)(base + h->off_finv);
        for (int s = 0; s < p->n_ops; ++s)
            finv[s] = p->fparams[s] > 0 ? (float)(1.0 / (double)p->fparams[s]) : 0.0f;
        std::memcpy(base + h->off_iparams, p->iparams, 12 * (size_t)p->n_ops);
    }
    if (c.mode == EPI_REQUANT || c.mode == EPI_REQUANT_LUT) {
        float *rqc = (float *)(base + h->off_rqc);
        for (int64_t m = 0; m < M; ++m) rqc[m] = (float)((double)p->scale_in[m] / (double)c.q_scale);
    }
    if (p->n_luts) std::memcpy(base + h->off_luts, p->luts, 256 * (size_t)p->n_luts);
    if (p->n_chans) std::memcpy(base + h->off_chans, p->chans, 4 * (size_t)p->n_chans * M);
    if (!c.clut.empty()) std::memcpy(base + h->off_clut, c.clut.data(), 4 * 256);
    if (!c.bp.x.empty()) {
        int32_t *keys = (int32_t *)(base + h->off_bp_key);
        for (size_t i = 0; i < c.bp.x.size(); ++i) keys[i] = (int32_t)f2key(c.bp.x[i]);
        std::memcpy(base + h->off_bp_bucket, c.bp_bucket.data(), 2 * c.bp_bucket.size());
        std::memcpy(base + h->off_bp_x, c.bp.x.data(), 4 * c.bp.x.size());
        std::memcpy(base + h->off_bp_v, c.bp.v.data(), 4 * c.bp.v.size());
    } else if (!c.bp.v.empty()) {
        std::memcpy(base + h->off_bp_v, c.bp.v.data(), 4 * c.bp.v.size());
    }
    if (!c.bp_lin.empty()) std::memcpy(base + h->off_bp_lin, c.bp_lin.data(), 4 * c.bp_lin.size());

    // K2 source: dense W^T [kpad][mtiles*128] int8, m contiguous
    int8_t *wt = (int8_t *)(base + h->off_tc_wt);
    const int64_t ldm = (int64_t)h->tc_mtiles * 128;
    for (int32_t g = 0; g < G; ++g)
        for (int64_t q = w->group_ptr[g]; q < w->group_ptr[g + 1]; ++q)
            for (int r = 0; r < 4; ++r) {
                int64_t m = (int64_t)g * 4 + r;
                int8_t v = w->vals[(q / 4) * 16 + r * 4 + (q % 4)];
                if (m < M && v) wt[(int64_t)w->idx[q] * ldm + m] += v;
            }
    return SI_OK;
}

// Structural check of an image of `bytes` bytes from an untrusted source (a
// plan file): header present, magic / version known, every section inside
// total_bytes, total_bytes inside the buffer, and the section extents the
// header's own counts imply (the kernels index sections by those counts).
extern "C" int32_t si_plan_image_validate(const void *image, uint64_t bytes)
{
    const SiImage *h = (const SiImage *)image;
    if (!h || bytes < sizeof(SiImage)) {
        si_set_error("plan image shorter than its header");
        return SI_EFORMAT;
    }
    if (h->magic != SI_IMG_MAGIC || h->version != SI_IMG_VERSION) {
        si_set_error("not a plan image (magic/version mismatch)");
        return SI_EFORMAT;
    }
    if (h->total_bytes > bytes || h->total_bytes < sizeof(SiImage)) {
        si_set_error("plan image total size exceeds the buffer");
        return SI_EFORMAT;
    }
    if (h->M < 1 || h->K < 1 || h->rows < h->M || h->rows % 4 || h->groups != h->rows / 4 || h->padded_blocks < 0 ||
        h->padded_blocks % 4 || h->tiles * 4 != h->padded_blocks || h->n_ops < 0 || h->n_luts < 0 || h->n_chans < 0 ||
        h->n_sides < 0 || h->n_bp < 0 || h->tc_mtiles != (h->M + 127) / 128 || h->tc_kpad != (h->K + 127) / 128 * 128) {
        si_set_error("plan image header fields are inconsistent");
        return SI_EFORMAT;
    }
    const uint64_t M = (uint64_t)h->M, T = (uint64_t)h->padded_blocks, kch = (uint64_t)h->tc_kpad / 128;
    const uint64_t rt_pad = ((uint64_t)h->tc_mtiles + 1) / 2 * 2;
    struct Sec { uint64_t off, len; };
    const Sec secs[] = {
        {h->off_tile_ptr, 4 * ((uint64_t)h->groups + 1)}, {h->off_tile_w, 4 * T}, {h->off_tile_idx, 4 * T},
        {h->off_adj, 4 * M}, {h->off_scale_in, 4 * M}, {h->off_ops, 4 * (uint64_t)h->n_ops},
        {h->off_fparams, 4 * (uint64_t)h->n_ops}, {h->off_finv, 4 * (uint64_t)h->n_ops},
        {h->off_iparams, 12 * (uint64_t)h->n_ops}, {h->off_luts, 256 * (uint64_t)h->n_luts},
        {h->off_chans, 4 * (uint64_t)h->n_chans * M}, {h->off_clut, 4 * 256}, {h->off_bp_x, 4 * (uint64_t)h->n_bp},
        {h->off_bp_v, 4 * ((uint64_t)h->n_bp + 1)}, {h->off_tc_wt, (uint64_t)h->tc_kpad * h->tc_mtiles * 128},
        {h->off_rqc, 4 * M}, {h->off_bp_key, 4 * (uint64_t)h->n_bp},
        {h->off_bp_bucket, 2 * (uint64_t)(h->bp_nbucket > 0 ? h->bp_nbucket : 0)}, {h->off_rqg, 4 * M},
        {h->off_bp_lin, 8 * (uint64_t)(h->bp_lin_n > 0 ? h->bp_lin_n : 0)},
        {h->off_sp_img, rt_pad * kch * 12288}, {h->off_sp_rptr, 4 * ((uint64_t)h->tc_mtiles * 128 + 1)},
        {h->off_sp_res, 4 * (uint64_t)(h->sp_nres > 0 ? h->sp_nres : 0)}, {h->off_rqp, 4 * M},
        {h->off_tr_img, rt_pad * 12288}, {h->off_tr_k, 2 * (rt_pad / 2) * TR_SLOTS}, {h->off_tr_cnt, 4 * (rt_pad / 2)},
    };
    for (const Sec &sc : secs)
        if (sc.off > h->total_bytes || sc.len > h->total_bytes - sc.off || sc.off % 16) {
            si_set_error("plan image section outside the image");
            return SI_EFORMAT;
        }
    if (h->sp_nres < 0 || h->tr_pairs != (int32_t)(rt_pad / 2)) {
        si_set_error("plan image header fields are inconsistent");
        return SI_EFORMAT;
    }
    return SI_OK;
}

extern "C" int32_t si_plan_info_get(const void *host_image, si_plan_info *info)
{
    const SiImage *h = (const SiImage *)host_image;
    if (!h || h->magic != SI_IMG_MAGIC || h->version != SI_IMG_VERSION) {
        si_set_error("not a plan image");
        return SI_EINVAL;
    }
    info->m = h->M; info->k = h->K; info->groups = h->groups; info->out_dtype = h->out_dtype;
    info->epi_mode = h->epi_mode; info->exact = h->exact;
    info->nnz_blocks = h->nnz_blocks; info->padded_blocks = h->padded_blocks;
    info->image_bytes = h->total_bytes;
    return SI_OK;
}
