"""Probe tcgen05.mma.kind::i8 with A in tensor memory (experiment, GPU box).

    python tools/atmem_probe.py

Builds tools/_atmem_probe.so and runs one M128 x N64 x K32 MMA whose A was
written into TMEM by tcgen05.st (lane = row, 4 k-bytes per 32-bit column,
little- or big-endian within the column), against numpy."""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_atmem_probe.so")


def build():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-shared",
                    "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "atmem_probe.cu")], check=True)


def core_image(mat, rows, row_bytes, lbo, sbo, size):
    img = np.zeros(size, np.uint8)
    for r in range(rows):
        for b in range(row_bytes):
            img[(r // 8) * sbo + (b // 16) * lbo + (r % 8) * 16 + (b % 16)] = mat[r, b]
    return img


def main():
    if not os.path.exists(SO):
        build()
    L = ctypes.CDLL(SO)
    rng = np.random.default_rng(0)
    A = rng.integers(-128, 128, (128, 32)).astype(np.int8)
    B = rng.integers(0, 256, (64, 32)).astype(np.uint8)   # [n][k]
    D = A.astype(np.int64) @ B.astype(np.int64).T
    b_img = core_image(B, 64, 32, 128, 256, 2048)
    out = np.zeros((128, 64), np.int32)
    for order in (0, 1):
        rc = L.atmem_probe(A.ctypes.data, b_img.ctypes.data, out.ctypes.data, order)
        print(f"A in TMEM, byte order {'le' if order == 0 else 'be'}: rc={rc} mismatches={int((out != D).sum())}",
              flush=True)


if __name__ == "__main__":
    main()
