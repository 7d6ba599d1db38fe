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
    buf = torch.randint(0, 255, (64 << 20,), dtype=torch.uint8, device="cuda")
    print("--- L2-resident 64 MB, 148 CTAs, box rows x 128 B, pitch 64 KB; producers < 0: tcgen05.commit release", flush=True)
    pitch = 65536
    rows = (64 << 20) // pitch
    for box in (128, 256):
        for S in (4, 8, 12):
            if S * box * 128 > 200 * 1024:
                continue
            for nprod in (1, 2, 4, -1, -2):
                bw = L.tma_bw(buf.data_ptr(), rows, S, box, 1024 * 128 // box, 148, 97, 5, nprod, pitch)
                print(f"box {box} S {S:2d} producers {nprod:2d}: {bw:8.1f} GB/s", flush=True)
