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


def producer_sweep(conv=False):
    """Per-SM TMA throughput vs producer warps and box size (148 CTAs, S slots);
    conv: warp-converged producers (tcw::) instead of lone lane-0 threads."""
    L = ctypes.CDLL(SO)
    L.tma_bw.restype = ctypes.c_double
    L.tma_bw.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7 + [ctypes.c_long]
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    rows = (96 << 20) // 128
    for box in (64, 96, 128, 256):
        for nprod in (1, 2, 4):
            S = max(2, min(16, (192 * 1024) // (box * 128)))
            bw = L.tma_bw(buf.data_ptr(), rows, S, box, 2048, 148, 0, 5, nprod + (1000 if conv else 0), 128) / 148
            print(f"box {box * 128 // 1024:2d} KB S {S:2d} producers {nprod}{' (converged)' if conv else ''}: "
                  f"{bw:6.1f} GB/s per SM", flush=True)


def commit_sweep():
    """Slot release by plain mbarrier arrive vs tcgen05.commit (148 CTAs)."""
    L = ctypes.CDLL(SO)
    L.tma_bw.restype = ctypes.c_double
    L.tma_bw.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7 + [ctypes.c_long]
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    rows = (96 << 20) // 128
    for box in (96, 128):
        for nprod in (4, -4):
            for S in (4, 8, 12):
                bw = L.tma_bw(buf.data_ptr(), rows, S, box, 2048, 148, 0, 5, nprod, 128) / 148
                print(f"box {box * 128 // 1024:2d} KB S {S:2d} producers {abs(nprod)} release "
                      f"{'commit' if nprod < 0 else 'arrive'}: {bw:6.1f} GB/s per SM", flush=True)


def pair_sweep():
    """CTA-pair loads (.cta_group::2 onto the leader's barrier), plain-arrive release."""
    L = ctypes.CDLL(SO)
    L.tma_bw2.restype = ctypes.c_double
    L.tma_bw2.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    rows = (96 << 20) // 128
    for box in (96, 128):
        for nprod in (4, -4):
            for S in (4, 7, 12):
                bw = L.tma_bw2(buf.data_ptr(), rows, S, box, 2048, 148, 5, nprod, 1) / 148
                print(f"pair box {box * 128 // 1024:2d} KB S {S:2d} producers {abs(nprod)} release "
                      f"{'commit-mc' if nprod < 0 else 'arrive'}: {bw:6.1f} GB/s per SM", flush=True)


def shared_sweep():
    """148 CTAs reading one small L2-resident set of boxes (like K2t's W images:
    ~3 MB read by every pair) vs disjoint slices."""
    L = ctypes.CDLL(SO)
    L.tma_bw.restype = ctypes.c_double
    L.tma_bw.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7 + [ctypes.c_long]
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    for nbox in (256, 2048, 8192):
        rows = nbox * 96
        for stride in (1, 8, 64):
            bw = L.tma_bw(buf.data_ptr(), rows, 8, 96, 2048, 148, stride, 5, 4, 128) / 148
            print(f"shared set {nbox * 12 // 1024:3d} MB stride {stride:2d}: {bw:6.1f} GB/s per SM", flush=True)
    bw = L.tma_bw(buf.data_ptr(), (96 << 20) // 128, 8, 96, 2048, 148, 0, 5, 4, 128) / 148
    print(f"disjoint: {bw:6.1f} GB/s per SM", flush=True)


def pair_small():
    L = ctypes.CDLL(SO)
    L.tma_bw2.restype = ctypes.c_double
    L.tma_bw2.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    for mb in (96, 24, 3):
        rows = (mb << 20) // 128
        for nprod in (4, -4):
            bw = L.tma_bw2(buf.data_ptr(), rows, 7, 96, 2048, 148, 5, nprod, 1) / 148
            print(f"pair {mb} MB set, 12 KB boxes S 7 producers 4 {'commit' if nprod < 0 else 'arrive'}: "
                  f"{bw:6.1f} GB/s per SM", flush=True)


def pitch_sweep():
    """Box rows contiguous (pitch 128 B) vs strided like the kernels' operand
    tiles (X [N][K] rows K bytes apart, [K][N] rows N bytes apart)."""
    L = ctypes.CDLL(SO)
    L.tma_bw.restype = ctypes.c_double
    L.tma_bw.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7 + [ctypes.c_long]
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    for pitch in (128, 1024, 4096, 65536):
        rows = (96 << 20) // pitch
        for box, S in ((64, 16), (128, 12)):
            bw = L.tma_bw(buf.data_ptr(), rows, S, box, 2048, 148, 0, 5, 4, pitch) / 148
            print(f"pitch {pitch:6d} B, box {box} rows x 128 B, S {S}, 4 producers: {bw:6.1f} GB/s per SM", flush=True)


def pairk(S=4, nprod=3, mode=0):
    """The pair kernel's TMA stream for BASELINE 5b (W^T 1024x4096, X 1024x65536)
    with no other roles: microseconds per sweep, vs the kernel's TMA-only run.
    mode bits: 1 TMEM allocated, 2 sixteen parked warps."""
    L = ctypes.CDLL(SO)
    L.tma_pairk.restype = ctypes.c_double
    L.tma_pairk.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_int] * 7
    M, K, N = 4096, 1024, 65536
    wt = torch.randint(0, 255, (K * M,), dtype=torch.uint8, device="cuda")
    x = torch.randint(0, 255, (K * N,), dtype=torch.uint8, device="cuda")
    us = L.tma_pairk(wt.data_ptr(), x.data_ptr(), M, K, N, S, nprod, 5, mode)
    gb = (K * N * (M // 256) + K * M * (N // 256)) / (us * 1e-6) / 1e9
    print(f"5b pair TMA stream S {S} producers {nprod} mode {mode}: {us:7.1f} us  ({gb / 148:5.1f} GB/s per SM)",
          flush=True)


def latency_sweep():
    """Per-SM TMA throughput vs ring depth, 1 CTA vs 148 CTAs (disjoint L2-resident
    slices): the implied round trip S * box / (bytes/s per SM)."""
    L = ctypes.CDLL(SO)
    L.tma_bw.restype = ctypes.c_double
    L.tma_bw.argtypes = [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_int] * 7 + [ctypes.c_long]
    buf = torch.randint(0, 255, (96 << 20,), dtype=torch.uint8, device="cuda")
    rows = (96 << 20) // 128
    for ctas in (1, 148):
        for box in (96, 128):
            for S in (1, 2, 4, 6, 8, 12):
                if S * box * 128 > 200 * 1024:
                    continue
                bw = L.tma_bw(buf.data_ptr(), rows, S, box, 2048, ctas, 0, 5, 1, 128) / ctas
                rt = S * box * 128 / (bw * 1e9) * 1e6
                print(f"ctas {ctas:3d} box {box * 128 // 1024:2d} KB S {S:2d}: {bw:6.1f} GB/s per SM, "
                      f"round trip {rt:5.2f} us", flush=True)


if __name__ == "__main__":
    if not os.path.exists(SO):
        build()
    if len(sys.argv) > 1 and sys.argv[1] == "commit":
        commit_sweep()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "shared":
        shared_sweep()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pairk":
        pairk(*[int(v) for v in sys.argv[2:5]])
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pitch":
        pitch_sweep()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pairsmall":
        pair_small()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pair":
        pair_sweep()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "prod":
        producer_sweep(conv=len(sys.argv) > 2)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "lat":
        latency_sweep()
        sys.exit(0)
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

