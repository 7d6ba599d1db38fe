"""Probe the tcgen05.mma.sp.kind::i8 operand formats (experiment, GPU box).

    python tools/sp_probe.py

Builds tools/_sp_probe.so and runs one M128xN64xK64 sparse MMA per layout
hypothesis, comparing with the dense product of the logical 2:4 matrix."""

import ctypes
import itertools
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_sp_probe.so")


def build():
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-shared", "-Xcompiler",
           "-fPIC", "-o", SO, os.path.join(HERE, "sp_probe.cu")]
    subprocess.run(cmd, check=True)


def core_image(mat, rows, row_bytes, lbo, sbo, size):
    """K-major SWIZZLE_NONE canonical layout: 8-row x 16-byte core matrices."""
    img = np.zeros(size, np.uint8)
    for r in range(rows):
        for b in range(row_bytes):
            off = (r // 8) * sbo + (b // 16) * lbo + (r % 8) * 16 + (b % 16)
            img[off] = mat[r, b]
    return img


def make_problem(seed=0):
    rng = np.random.default_rng(seed)
    A = np.zeros((128, 64), np.int8)
    idx = np.zeros((128, 16, 2), np.int64)
    for m in range(128):
        for c in range(16):
            i0, i1 = sorted(rng.choice(4, 2, replace=False))
            idx[m, c] = (i0, i1)
            A[m, 4 * c + i0] = rng.integers(-127, 128)
            A[m, 4 * c + i1] = rng.integers(-127, 128)
    B = rng.integers(0, 256, (64, 64), dtype=np.uint8)  # [n][k]
    D = A.astype(np.int64) @ B.astype(np.int64).T
    return A, idx, B, D


def compress(A, idx):
    P = np.zeros((128, 32), np.int8)
    for m in range(128):
        for c in range(16):
            P[m, 2 * c] = A[m, 4 * c + idx[m, c, 0]]
            P[m, 2 * c + 1] = A[m, 4 * c + idx[m, c, 1]]
    return P


def meta_rows(idx, hi_first=False, swap=False):
    E = np.zeros((128, 16), np.uint8)
    for m in range(128):
        for c in range(16):
            a, b = idx[m, c]
            nib = (b | (a << 2)) if swap else (a | (b << 2))
            byte, hi = c // 2, (c % 2 == 1)
            if hi_first:
                hi = not hi
            E[m, byte] |= (nib << 4) if hi else nib
    return E


def main():
    if not os.path.exists(SO):
        build()
    L = ctypes.CDLL(SO)
    A, idx, B, D = make_problem()
    P = compress(A, idx)
    a_img = core_image(P.view(np.uint8), 128, 32, 128, 256, 4096)
    b_img = core_image(B, 64, 64, 128, 512, 4096)
    out = np.zeros((128, 64), np.int32)
    for hi_first, swap, id2, ecol in itertools.product([False, True], [False, True], [0], [128]):
        E = meta_rows(idx, hi_first, swap)
        e_img = core_image(E, 128, 16, 2048, 128, 2048)
        prm = np.array([128, 256, 128, 512, 2048, 128, id2, ecol], np.int32)
        rc = L.sp_probe(a_img.ctypes.data, b_img.ctypes.data, e_img.ctypes.data, out.ctypes.data, prm.ctypes.data)
        bad = int((out != D).sum())
        print(f"hi_first={hi_first} swap={swap} id2={id2} ecol={ecol} rc={rc} mismatches={bad}", flush=True)
        if bad and bad < 8192:
            mm = np.argwhere(out != D)[:3]
            print("   e.g.", [(tuple(x), int(out[tuple(x)]), int(D[tuple(x)])) for x in mm])
    # sanity: dense result with everything = check the B/A layouts via a second
    # probe where the metadata selects (0, 1) everywhere
    idx01 = np.zeros_like(idx)
    idx01[..., 1] = 1
    A01 = np.zeros_like(A)
    for m in range(128):
        for c in range(16):
            A01[m, 4 * c] = A[m, 4 * c + idx[m, c, 0]]
            A01[m, 4 * c + 1] = A[m, 4 * c + idx[m, c, 1]]
    D01 = A01.astype(np.int64) @ B.astype(np.int64).T
    E = meta_rows(idx01)
    e_img = core_image(E, 128, 16, 2048, 128, 2048)
    prm = np.array([128, 256, 128, 512, 2048, 128, 0, 128], np.int32)
    L.sp_probe(a_img.ctypes.data, b_img.ctypes.data, e_img.ctypes.data, out.ctypes.data, prm.ctypes.data)
    print("idx(0,1) everywhere: mismatches", int((out != D01).sum()))


def probe_second_half():
    """Metadata for the second 64-k MMA of a stage lives in bytes 8..15 of
    each row (TMEM columns +2,+3): address it by column offset or id2?"""
    L = ctypes.CDLL(SO)
    A, idx, B, D = make_problem(1)
    P = compress(A, idx)
    a_img = core_image(P.view(np.uint8), 128, 32, 128, 256, 4096)
    b_img = core_image(B, 64, 64, 128, 512, 4096)
    E8 = meta_rows(idx)
    E = np.zeros((128, 16), np.uint8)
    E[:, 8:16] = E8[:, 0:8]
    e_img = core_image(E, 128, 16, 2048, 128, 2048)
    out = np.zeros((128, 64), np.int32)
    sel = [tuple(int(v) for v in a.split(",")) for a in sys.argv[2:]] or [(1, 128)]
    for id2, ecol in sel:
        prm = np.array([128, 256, 128, 512, 2048, 128, id2, ecol], np.int32)
        rc = L.sp_probe(a_img.ctypes.data, b_img.ctypes.data, e_img.ctypes.data, out.ctypes.data, prm.ctypes.data)
        print(f"second-half metadata: id2={id2} ecol={ecol} rc={rc} mismatches={int((out != D).sum())}", flush=True)


def probe_pair():
    """cluster of 2: each CTA holds 128 rows of A (+ its metadata) and 32 of
    the 64 tokens of B; the leader issues cp + mma.sp with cta_group::2."""
    L = ctypes.CDLL(SO)
    A0, idx0, B, _ = make_problem(2)
    A1, idx1, _, _ = make_problem(3)
    A = np.concatenate([A0, A1])
    D = A.astype(np.int64) @ B.astype(np.int64).T          # [256, 64]
    a_img = np.concatenate([core_image(compress(A0, idx0).view(np.uint8), 128, 32, 128, 256, 4096),
                            core_image(compress(A1, idx1).view(np.uint8), 128, 32, 128, 256, 4096)])
    e_img = np.concatenate([core_image(meta_rows(idx0), 128, 16, 2048, 128, 2048),
                            core_image(meta_rows(idx1), 128, 16, 2048, 128, 2048)])
    b_img = np.concatenate([core_image(B[:32], 32, 64, 128, 512, 2048), core_image(B[32:], 32, 64, 128, 512, 2048)])
    out = np.zeros((256, 64), np.int32)
    rc = L.sp_probe_pair(a_img.ctypes.data, b_img.ctypes.data, e_img.ctypes.data, out.ctypes.data, 512)
    print(f"pair sparse: rc={rc} mismatches={int((out != D).sum())}", flush=True)
    if (out != D).any():
        mm = np.argwhere(out != D)[:4]
        print("   e.g.", [(tuple(int(v) for v in x), int(out[tuple(x)]), int(D[tuple(x)])) for x in mm])


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "pair":
        probe_pair()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "half":
        probe_second_half()
        sys.exit(0)
    sys.exit(main())
