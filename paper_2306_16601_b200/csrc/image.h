// image.h -- layout of the plan image (host builder <-> device kernels).
//
// One position-independent blob per plan: the host builds it
// (plan.cpp, si_plan_image_build), Python copies it to a CUDA tensor, the
// kernels read their sections through byte offsets.  Everything the
// reference's SpmmPlan holds (spmm.py:110-133) is in here: the weight in
// the GPU tile formats, adj[m] = bias[m] - a_zp*comp[m] (spmm.py:231), the
// per-channel scale_in and the compiled epilogue program.
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

#define SI_IMG_MAGIC 0x58344953u /* "SI4X" */
#define SI_IMG_VERSION 7u   /* 6: unused residual slots carry tr_k = 0xFFFF; 7: linear breakpoint table */
#define TR_SLOTS 128 /* K3 residual slots per 256-row pair tile */

// compiled epilogue forms (see plan.cpp: compile_program)
enum EpiMode : int32_t {
    EPI_S32 = 0,         // []                     -> s32 acc+adj (spmm.py:280)
    EPI_DEQ_F32 = 1,     // [DEQ_ACC]              -> f32
    EPI_REQUANT = 2,     // [REQUANT]              -> 8-bit
    EPI_REQUANT_LUT = 3, // [REQUANT, int chain]   -> 256-entry composite table
    EPI_DEQ_TABLE = 4,   // [DEQ_ACC, f32 unary*, QUANT, int chain] -> breakpoint table over f32
    EPI_GENERIC = 5,     // anything else: device interpreter of _run_chain
    EPI_DEQ_SIDE = 6     // [DEQ_ACC, ADD_SIDE] -> f32 (residual); kernels run it in their
                         // EPI_GENERIC instantiation (K2: compiled branch, K1/KREF: interpreter)
};

struct SiImage {
    uint32_t magic, version;
    int32_t M, K, rows, groups;
    int64_t padded_blocks, nnz_blocks, tiles;  // tiles = padded_blocks / 4
    int32_t out_dtype, a_zp, n_ops, n_luts, n_chans, n_sides;
    int32_t epi_mode, exact;
    // single-op fast paths (EPI_REQUANT / first op of EPI_REQUANT_LUT)
    float q_scale, q_inv;
    int32_t q_zp, q_lo, q_hi;
    int32_t n_bp;          // breakpoints in the EPI_DEQ_TABLE table
    // tensor-core (K2) geometry
    int32_t tc_mtiles;     // ceil(M / 128)
    int32_t tc_kpad;       // K rounded up to 128
    int32_t pad0, pad1;
    // section offsets in bytes from the image start (16-byte aligned)
    uint64_t off_tile_ptr;   // int32 [groups+1]        micro-tile offsets per group
    uint64_t off_tile_w;     // uint4 [tiles]           reference micro-tiles (sparse.py:28-31)
    uint64_t off_tile_idx;   // int4  [tiles]           the 4 block columns of each tile
    uint64_t off_adj;        // int32 [M]               bias - a_zp*comp (wrapped)
    uint64_t off_scale_in;   // f32   [M]
    uint64_t off_ops;        // int32 [n_ops]
    uint64_t off_fparams;    // f32   [n_ops]
    uint64_t off_finv;       // f32   [n_ops]           f32(1/fparam) for the guard-band fast path
    uint64_t off_iparams;    // int32 [n_ops*3]
    uint64_t off_luts;       // u8    [n_luts*256]
    uint64_t off_chans;      // f32   [n_chans*M]
    uint64_t off_clut;       // u32   [256]             composite table (EPI_REQUANT_LUT)
    uint64_t off_bp_x;       // f32   [n_bp]            thresholds (EPI_DEQ_TABLE)
    uint64_t off_bp_v;       // u32   [n_bp+1]          values (bits of the final state)
    uint64_t off_tc_wt;      // int8  [tc_kpad][tc_mtiles*128]  W^T dense (K2 B/A operand source)
    uint64_t total_bytes;
    uint64_t off_rqc;        // f32   [M]               f32(f64(scale_in)/f64(fp)) for the requant fast path
    // bucketed index over the breakpoint thresholds (f32 total-order keys)
    int32_t bp_key_lo, bp_shift, bp_nbucket, bp_occ;   // bp_occ: most thresholds in one bucket
    uint64_t off_bp_key;     // i32   [n_bp]            threshold keys
    uint64_t off_bp_bucket;  // u16   [bp_nbucket]      first threshold index per key bucket
    // K2 on-chip expansion lists: for every (128-row tile rt, 128-k chunk kc,
    // 64-k half) the nonzero 4x1 blocks as smem word offsets into the
    // MN-major SWIZZLE_128B [128 k x 128 m] operand tile plus the 4-row value
    // word.  List j: u32 values[n] then u16 offsets[n], n padded to 8 by
    // repeating the last entry, starting at byte tc_eptr[j].
    int32_t tc_emax;         // max padded entries of any list
    int32_t tc_nlists;       // tc_mtiles * kchunks * 2
    uint64_t off_tc_eptr;    // u32   [tc_nlists + 1]   byte offsets into the entry section
    uint64_t off_tc_ent;     // bytes                   entry lists
    uint64_t off_rqg;        // f32   [M]               per-row epilogue class: -1 if |acc+adj| may reach 2^22,
                             //                         1 requant rounding proven exact (plan.cpp
                             //                         requant_row_exact), else the requant certificate
                             //                         guard 2^-22 max|r| (<= 1/4; 0 for other modes)
    // 2:4 images (K3, spmm_xs.cu): per (128-row tile, 128-k chunk) a 12 KB
    // image = compressed A [128 rows x 64 B] (K-major, SWIZZLE_NONE core
    // matrices, LBO 128 / SBO 512) + two metadata tiles [128 rows x 16 B]
    // (bytes 0-7: 4-bit idx0|idx1<<2 per 4-wide k window; SBO 128), and
    // per-row residual lists for windows with > 2 nonzero columns.
    uint64_t off_sp_img;     // bytes [even(tc_mtiles) * kchunks * 12288]
    uint64_t off_sp_rptr;    // i32   [tc_mtiles * 128 + 1] residual entry offsets per padded row
    uint64_t off_sp_res;     // i32   [n_res]  (k << 8) | (uint8)w
    int32_t sp_nres, sp_maxres;  // residual entries, max per row
    uint64_t off_rqp;        // f32   [M]               requant multiplier c' of rows proven exact (rqg == 1):
                             //                         out = bits(fma(f32(a), c', 1.5*2^23 + zp)) - bits(1.5*2^23)
    // K3 (X-stationary 2:4 kernel) residual operand, per 256-row pair tile
    // pt: the columns that did not fit the main 2:4 images, gathered on-chip
    // into TR_SLOTS slots of a second 2:4 operand (plan.cpp build_tr_sections)
    uint64_t off_tr_img;     // bytes [2*pairs][12288]   residual 2:4 images (same format as sp_img)
    uint64_t off_tr_k;       // u16   [pairs][TR_SLOTS]   activation column of each slot (0xFFFF: unused)
    uint64_t off_tr_cnt;     // i32   [pairs]             residual MMAs (64 slots each; 0..TR_SLOTS/64)
    int32_t tr_ok, tr_pairs; // tr_ok 0: some pair tile needs more than TR_SLOTS slots (K3 unavailable)
    uint64_t off_tc_wrow;    // (image v4: row-major W of the retired K2a; empty since v5)
    // EPI_DEQ_TABLE fast path (plan.cpp build_linear): bucket b = rn(clamp(fma(x,
    // bp_lin_inv, bp_lin_off), 0, bp_lin_n - 1)) holds at most one threshold:
    // entry {f32 thr, i16 value below | i16 value at/above << 16}.  bp_lin_n = 0:
    // no such table (thresholds too close, or values beyond 16 bits).
    uint64_t off_bp_lin;     // u32x2 [bp_lin_n]
    int32_t bp_lin_n;
    float bp_lin_inv, bp_lin_off;
    int32_t pad2;
    uint64_t reserved0;
};

static_assert(sizeof(SiImage) % 16 == 0, "image header must stay 16-byte aligned");

template <typename T>
static inline __host__ __device__ const T *img_sec(const void *img, uint64_t off)
{
    return reinterpret_cast<const T *>(reinterpret_cast<const uint8_t *>(img) + off);
}
