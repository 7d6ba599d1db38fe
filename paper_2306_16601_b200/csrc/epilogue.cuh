// epilogue.cuh -- the fused SpMM epilogue on the device.
//
// Bit-exact restatement of the reference's per-element chain
// (_run_chain, epilogue.py:207-249) for every compiled form, with two
// tricks that keep f64 division off the hot path:
//
//  * DEQ_ACC  f32(f64(a)*f64(s)): for |a| <= 2^24 the f64 product of a
//    24-bit integer and a 24-bit significand is exact, so one f32 rounding
//    of the f32 product gives the same bits.  Larger |a| take the f64 path.
//  * REQUANT / QUANT  clamp(rint(f64 expr) + zp): evaluated in f32 with a
//    proven relative error < 4*2^-24; when the f32 value is farther than
//    2^-20*|r| from a half-integer its rounding equals the f64 one, else the
//    exact f64 expression (IEEE-correct __dmul_rn/__ddiv_rn/rint) decides.
//
// GELU (epilogue.py:190-194) is never evaluated on the device when it feeds
// an integer output: the plan compiles such chains to a 256-entry table or
// an f32 breakpoint table built on the host with glibc tanh (plan.cpp).
// Only f32-output / residual chains run the device tanh (documented as
// within 1e-5 relative, not bit-exact).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

#include "image.h"

struct EpiParams {
    int32_t mode, out_dtype, M, n_ops;
    float q_scale, q_inv;
    int32_t q_zp, q_lo, q_hi, n_bp;
    const int32_t *adj;
    const float *scale_in;
    const int32_t *ops;
    const float *fparams;
    const float *finv;
    const int32_t *iparams;
    const uint8_t *luts;
    const float *chans;
    const uint32_t *clut;
    const float *bp_x;
    const uint32_t *bp_v;
    const float *sides;   // f32 [n_sides, N, M]
    int64_t N;
    const int32_t *bp_key;
    const uint16_t *bp_bucket;
    int32_t bp_key_lo, bp_shift, bp_nbucket, bp_occ;
    // linear buckets, at most one threshold each (image.h off_bp_lin); 0 entries: none
    const uint2 *bp_lin;
    int32_t bp_lin_n;
    float bp_lin_inv, bp_lin_off;
};

static inline EpiParams make_epi(const SiImage *h, const void *img, const float *sides, int64_t n)
{
    EpiParams e;
    e.mode = h->epi_mode;
    e.out_dtype = h->out_dtype;
    e.M = h->M;
    e.n_ops = h->n_ops;
    e.q_scale = h->q_scale;
    e.q_inv = h->q_inv;
    e.q_zp = h->q_zp;
    e.q_lo = h->q_lo;
    e.q_hi = h->q_hi;
    e.n_bp = h->n_bp;
    e.adj = img_sec<int32_t>(img, h->off_adj);
    e.scale_in = img_sec<float>(img, h->off_scale_in);
    e.ops = img_sec<int32_t>(img, h->off_ops);
    e.fparams = img_sec<float>(img, h->off_fparams);
    e.finv = img_sec<float>(img, h->off_finv);
    e.iparams = img_sec<int32_t>(img, h->off_iparams);
    e.luts = img_sec<uint8_t>(img, h->off_luts);
    e.chans = img_sec<float>(img, h->off_chans);
    e.clut = img_sec<uint32_t>(img, h->off_clut);
    e.bp_x = img_sec<float>(img, h->off_bp_x);
    e.bp_v = img_sec<uint32_t>(img, h->off_bp_v);
    e.sides = sides;
    e.N = n;
    e.bp_key = img_sec<int32_t>(img, h->off_bp_key);
    e.bp_bucket = img_sec<uint16_t>(img, h->off_bp_bucket);
    e.bp_key_lo = h->bp_key_lo;
    e.bp_shift = h->bp_shift;
    e.bp_nbucket = h->bp_nbucket;
    e.bp_occ = h->bp_occ;
    e.bp_lin = img_sec<uint2>(img, h->off_bp_lin);
    e.bp_lin_n = h->bp_lin_n;
    e.bp_lin_inv = h->bp_lin_inv;
    e.bp_lin_off = h->bp_lin_off;
    return e;
}

// OP_DEQ_ACC, epilogue.py:247-248
__device__ __forceinline__ float dev_deq_acc(int32_t a, float s)
{
    if (a <= (1 << 24) && a >= -(1 << 24)) return __fmul_rn(__int2float_rn(a), s);
    return __double2float_rn(__dmul_rn((double)a, (double)s));
}

// rint(y)+zp clamped, from an f32 estimate r of y with |r-y| < 2^-21 |y|.
__device__ __forceinline__ bool fast_round(float r, int32_t zp, int32_t lo, int32_t hi, int32_t &out)
{
    float ar = fabsf(r);
    if (ar >= 4194304.0f) {  // 2^22: beyond any 8-bit range after zp
        if (hi - lo > 65535) return false;
        out = r > 0.0f ? hi : lo;
        return true;
    }
    if (ar != 0.0f && ar < 1e-30f) return false;  // subnormal territory: no bound
    float fl = floorf(r);
    float fr = __fsub_rn(r, fl);
    float d = fabsf(__fsub_rn(fr, 0.5f));
    if (d <= __fmaf_rn(ar, 9.5367431640625e-07f, 1e-30f)) return false;
    int32_t q = (int32_t)fl + (fr > 0.5f ? 1 : 0) + zp;
    out = min(max(q, lo), hi);
    return true;
}

// OP_REQUANT, epilogue.py:218-228
__device__ __forceinline__ int32_t dev_requant(int32_t a, float s, float fp, float inv, int32_t zp,
                                               int32_t lo, int32_t hi)
{
    int32_t out;
    if (inv != 0.0f) {
        float r = __fmul_rn(__fmul_rn(__int2float_rn(a), s), inv);
        if (fast_round(r, zp, lo, hi, out)) return out;
    }
    double y = __ddiv_rn(__dmul_rn((double)a, (double)s), (double)fp);
    double q = rint(y) + (double)zp;
    q = fmin(fmax(q, (double)lo), (double)hi);
    return (int32_t)q;
}

// OP_QUANT, _quant_scalar epilogue.py:197-204
__device__ __forceinline__ int32_t dev_quant(float x, float fp, float inv, int32_t zp, int32_t lo,
                                             int32_t hi)
{
    int32_t out;
    if (inv != 0.0f) {
        float r = __fmul_rn(x, inv);
        if (fast_round(r, zp, lo, hi, out)) return out;
    }
    double q = rint(__ddiv_rn((double)x, (double)fp)) + (double)zp;
    q = fmin(fmax(q, (double)lo), (double)hi);
    return (int32_t)q;
}

// OP_GELU (tanh form, epilogue.py:190-194) -- device tanh, not bit-pinned
__device__ __forceinline__ float dev_gelu_tanh(float x)
{
    double xd = (double)x;
    double c = __dmul_rn(__dmul_rn(__dmul_rn(0.044715, xd), xd), xd);
    double t = __dmul_rn(0.7978845608028654, __dadd_rn(xd, c));
    return __double2float_rn(__dmul_rn(__dmul_rn(0.5, xd), __dadd_rn(1.0, tanh(t))));
}

// OP_GELU_ERF (extension)
__device__ __forceinline__ float dev_gelu_erf(float x)
{
    double xd = (double)x;
    double e = erf(__dmul_rn(xd, 0.7071067811865476));
    return __double2float_rn(__dmul_rn(__dmul_rn(0.5, xd), __dadd_rn(1.0, e)));
}

// number of thresholds <= x, then the value of that piece
__device__ __forceinline__ uint32_t bp_lookup(float x, const float *bx, const uint32_t *bv, int n)
{
    int base = 0, len = n;
    while (len > 0) {
        int half = len >> 1;
        if (__ldg(bx + base + half) <= x) {
            base += half + 1;
            len -= half + 1;
        } else {
            len = half;
        }
    }
    return __ldg(bv + base);
}

__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }

// f32 -> int32 key preserving the total order of finite floats (+0 == -0)
__device__ __forceinline__ int32_t f32_key(float x)
{
    const uint32_t u = __float_as_uint(x);
    return (u & 0x80000000u) ? -(int32_t)(u & 0x7fffffffu) : (int32_t)u;
}

// bucketed breakpoint lookup: value of the piece containing x.  The tables
// may live in global (read-only path) or shared memory.
__device__ __forceinline__ uint32_t bp_lookup_bucketed(float x, const int32_t *keys, const uint16_t *bucket,
                                                       const uint32_t *vals, int n, int32_t key_lo, int shift,
                                                       int nbucket)
{
    const int32_t k = f32_key(x);
    if (n == 0 || k < key_lo) return vals[0];
    uint32_t b = ((uint32_t)k - (uint32_t)key_lo) >> shift;
    b = min(b, (uint32_t)(nbucket - 1));
    int i = bucket[b];
    while (i < n && keys[i] <= k) ++i;
    return vals[i];
}

// The same lookup as a fixed-length branchless binary search inside the
// bucket: the answer lies in [bucket[b], bucket[b] + occ] (occ = the most
// thresholds any bucket holds, plan.cpp), so S steps with 2^S > occ find it.
// Every lane runs the same straight-line code: the 32 lookups of an epilogue
// chunk neither diverge nor loop.
template <int S>
__device__ __forceinline__ uint32_t bp_lookup_fixed(float x, const int32_t *keys, const uint16_t *bucket,
                                                    const uint32_t *vals, int n, int32_t key_lo, int shift,
                                                    int nbucket)
{
    const int32_t k = f32_key(x);
    const uint32_t d = k < key_lo ? 0u : (uint32_t)k - (uint32_t)key_lo;
    const uint32_t b = min(d >> shift, (uint32_t)(nbucket - 1));
    int i = bucket[b];
#pragma unroll
    for (int st = 1 << (S - 1); st >= 1; st >>= 1) {
        const int j = i + st;   // take the step if keys[j - 1] <= k
        const int32_t kk = keys[min(j, n) - 1];
        i = (j <= n && kk <= k) ? j : i;
    }
    return vals[i];
}

// Linear-bucket lookup (plan.cpp build_linear): the bucket function is one
// fma, a clamp and the magic-number round-to-nearest-even; the bucket's one
// threshold decides between its two 16-bit values.
__device__ __forceinline__ int32_t bp_lookup_linear(float x, const uint2 *tab, float inv, float off, float nbm1)
{
    float t = __fmaf_rn(x, inv, off);
    t = fminf(fmaxf(t, 0.0f), nbm1);
    const uint32_t b = __float_as_uint(__fadd_rn(t, 8388608.0f)) & 0x7FFFFFu;
    const uint2 e = tab[b];
    // sign-extended 16-bit half of e.y picked by one PRMT (selector nibble msb:
    // replicate the byte's sign): 0xBB32 = upper half, 0x9910 = lower half
    const uint32_t sel = x >= __uint_as_float(e.x) ? 0xBB32u : 0x9910u;
    uint32_t r;
    asm("prmt.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(e.y), "r"(sel));
    return (int32_t)r;
}

// The same lookup for a table staged in shared memory.  `biased` is the
// table's 32-bit shared address minus (0x4B000000 << 3): the float bits of
// t + 2^23 are 0x4B000000 + b, so (bits << 3) + biased wraps to the address of
// entry b in one shift-add (no mask, no separate base add).
__device__ __forceinline__ int32_t bp_lookup_linear_smem(float x, uint32_t biased, float inv, float off, float nbm1)
{
    float t = __fmaf_rn(x, inv, off);
    t = fminf(fmaxf(t, 0.0f), nbm1);
    const uint32_t addr = (__float_as_uint(__fadd_rn(t, 8388608.0f)) << 3) + biased;
    uint32_t ex, ey;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(ex), "=r"(ey) : "r"(addr));
    const uint32_t sel = x >= __uint_as_float(ex) ? 0xBB32u : 0x9910u;
    uint32_t r;
    asm("prmt.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(ey), "r"(sel));
    return (int32_t)r;
}

// _run_chain interpreter (epilogue.py:207-249) for EPI_GENERIC
static __device__ __noinline__ uint32_t epi_generic(int32_t acc, int32_t m, int64_t n, const EpiParams &E)
{
    int32_t xi = 0;
    float xf = 0.0f;
    for (int s = 0; s < E.n_ops; ++s) {
        const int32_t op = __ldg(E.ops + s);
        const int32_t i0 = __ldg(E.iparams + 3 * s), i1 = __ldg(E.iparams + 3 * s + 1),
                      i2 = __ldg(E.iparams + 3 * s + 2);
        const float fp = __ldg(E.fparams + s), inv = __ldg(E.finv + s);
        switch (op) {
        case 0: xi = dev_requant(acc, __ldg(E.scale_in + m), fp, inv, i0, i1, i2); break;
        case 1: {
            int32_t key = i1 == 1 ? xi + 128 : xi;
            uint8_t b = __ldg(E.luts + (int64_t)i0 * 256 + key);
            xi = i2 == 1 ? (int32_t)(int8_t)b : (int32_t)b;
            break;
        }
        case 2: xf = __fmul_rn(__fsub_rn((float)xi, (float)i0), fp); break;
        case 3: xf = dev_gelu_tanh(xf); break;
        case 4: xf = __fadd_rn(xf, __ldg(E.sides + ((int64_t)i0 * E.N + n) * E.M + m)); break;
        case 5: xf = __fadd_rn(xf, __ldg(E.chans + (int64_t)i0 * E.M + m)); break;
        case 6: xi = dev_quant(xf, fp, inv, i0, i1, i2); break;
        case 7: xf = dev_deq_acc(acc, __ldg(E.scale_in + m)); break;
        case 8: xf = dev_gelu_erf(xf); break;
        default: break;
        }
    }
    return E.out_dtype == 0 ? f2u(xf) : (uint32_t)xi;
}

// One output element: a32 already includes adj[m].  Returns the 32-bit word
// to store (s32 / f32 bits, or the int state whose low byte is stored).
template <int MODE>
__device__ __forceinline__ uint32_t epi_apply(int32_t a32, int32_t m, int64_t n, const EpiParams &E)
{
    if constexpr (MODE == EPI_S32) {
        return (uint32_t)a32;
    } else if constexpr (MODE == EPI_DEQ_F32) {
        return f2u(dev_deq_acc(a32, __ldg(E.scale_in + m)));
    } else if constexpr (MODE == EPI_REQUANT) {
        return (uint32_t)dev_requant(a32, __ldg(E.scale_in + m), E.q_scale, E.q_inv, E.q_zp, E.q_lo,
                                     E.q_hi);
    } else if constexpr (MODE == EPI_REQUANT_LUT) {
        int32_t q = dev_requant(a32, __ldg(E.scale_in + m), E.q_scale, E.q_inv, E.q_zp, E.q_lo,
                                E.q_hi);
        return __ldg(E.clut + (q - E.q_lo));
    } else if constexpr (MODE == EPI_DEQ_TABLE) {
        float x = dev_deq_acc(a32, __ldg(E.scale_in + m));
        return bp_lookup_bucketed(x, E.bp_key, E.bp_bucket, E.bp_v, E.n_bp, E.bp_key_lo, E.bp_shift,
                                  E.bp_nbucket);
    } else {
        return epi_generic(a32, m, n, E);
    }
}
