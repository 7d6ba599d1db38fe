"""TMA streaming throughput vs ring depth and box size (experiment, GPU box).

    python tools/tma_bw.py
"""
import ctypes, os, subprocess, sys
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_tma_bw.so")


def build():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-shared",
                    "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "tma_bw.cu")], check=True)


if __name__ == "__main__":
    if not os.path.exists(SO):
        build()
    L = ctypes.CDLL(SO)
    L.tma_bw.restype = ctypes.c_double
    L.tma_bw.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7 + [ctypes.c_long]
    L.tma_bw2.restype = ctypes.c_double
    L.tma_bw2.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    rows = (96 << 20) // 128
    print("--- disjoint 96 MB, 148 CTAs: 1-CTA loads vs pair (.cta_group::2) loads", flush=True)
    for S in (6, 12):
        for nprod in (1, 3):
            bw = L.tma_bw(buf.data_ptr(), rows, S, 128, 1024, 148, 0, 5, nprod, 128)
            print(f"1-CTA  S {S:2d} x 16 KB, producers {nprod}: {bw/148:6.1f} GB/s per SM", flush=True)
    for (S, bps) in ((6, 2), (12, 1), (3, 4)):
        for nprod in (1, 3):
            bw = L.tma_bw2(buf.data_ptr(), rows, S, 128, 1024 // bps, 148, 5, nprod, bps)
            print(f"pair   S {S:2d} x {bps} boxes of 16 KB, producers {nprod}: {bw/148:6.1f} GB/s per SM", flush=True)
