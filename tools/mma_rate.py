"""tcgen05 kind::i8 issue-rate microbenchmark (experiment, GPU box).

    python tools/mma_rate.py

Dense (K32) and 2:4-sparse (K64) M256 x N MMAs over CTA pairs on all 148
SMs, A from shared memory (SS) or tensor memory (TS), with and without a
concurrent 16 KB bulk-copy stream into shared memory.  Prints MACs per clock
per SM (logical MACs, zeros of the 2:4 operand included) and the stream's
per-SM rate."""
import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_mma_rate.so")
MODES = {0: "dense SS", 1: "dense TS", 2: "sparse SS", 3: "sparse TS"}


def build():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-shared",
                    "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "mma_rate.cu")], check=True)


def run(L, buf, mode, N, stream, iters=8192, ctas=148, ldw=0, ld_iters=0):
    out = (ctypes.c_ulonglong * (ctas * 4))()
    ms = ctypes.c_float()
    err = L.mma_rate(mode, iters, N, stream, ctas, ctypes.c_void_p(buf.data_ptr()), buf.numel() // 16384, out,
                     ctypes.byref(ms), ldw, ld_iters)
    if err:
        raise RuntimeError(f"mma_rate mode {mode} N {N}: cuda error {err}")
    kl = 64 if mode & 2 else 32
    cyc = [out[4 * c] for c in range(0, ctas, 2)]
    cyc = sum(cyc) / len(cyc)
    macs_clk_sm = 256 * N * kl * iters / cyc / 2
    res = {"mode": MODES[mode & 3], "N": N, "cyc_per_mma": cyc / iters, "mac_clk_sm": macs_clk_sm, "ms": ms.value}
    if ldw:
        res["ld_B_clk"] = sum(out[4 * c + 2] / max(1, out[4 * c + 3]) for c in range(ctas)) / ctas
    if stream:
        sb = [out[4 * c + 2] / max(1, out[4 * c + 3]) for c in range(ctas)]
        res["stream_B_clk"] = sum(sb) / len(sb)
        res["stream_cyc"] = sum(out[4 * c + 3] for c in range(ctas)) / ctas
    return res


def main():
    if not os.path.exists(SO):
        build()
    L = ctypes.CDLL(SO)
    L.mma_rate.restype = ctypes.c_int
    L.mma_rate.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p,
                                               ctypes.POINTER(ctypes.c_float), ctypes.c_int, ctypes.c_int]
    buf = torch.randint(0, 255, (32 << 20,), dtype=torch.uint8, device="cuda")
    import sys
    if len(sys.argv) > 1 and sys.argv[1] == "ws":
        # K4's question: sparse SS MMAs with the 2:4 image's SWIZZLE_NONE A (512),
        # one or two issuers on ONE accumulator (4 | 8192), with and without a
        # concurrent bulk-copy stream into shared memory
        for N in (128, 192, 256):
            for two in (0, 1):
                for a_none in (0, 512):
                    for stream in (0, 4096):
                        mode = 2 | 16 | a_none | ((4 | 8192) if two else 0)
                        run(L, buf, mode, N, stream, iters=1024)
                        r = run(L, buf, mode, N, stream)
                        extra = f"  stream {r['stream_B_clk']:5.1f} B/clk/SM" if stream else ""
                        print(f"sparse SS N{N:3d} issuers {1 + two} A {'none' if a_none else 'sw128'}: "
                              f"{r['cyc_per_mma']:7.1f} clk/MMA (combined){extra}", flush=True)
        for N in (192,):
            for extra, tag in ((128, "commit (multicast) per 2 MMAs"), (128 | 2048, "commit per 2 + busy neighbour warps"),
                               (16384, "4 distinct A and B tiles"), (32768, "8 metadata addresses"),
                               (16384 | 32768, "distinct A, B and metadata")):
                mode = 2 | 16 | 512 | 4 | 8192 | extra
                run(L, buf, mode, N, 4096, iters=1024, ld_iters=200000)
                r = run(L, buf, mode, N, 4096, ld_iters=3000000)
                print(f"sparse SS N{N} issuers 2, {tag}: {r['cyc_per_mma']:7.1f} clk/MMA (combined)", flush=True)
        return
    for N, extra, tag in ((224, 16 | 64 | 128, "K3 stage pattern, idle neighbours"),
                          (224, 16 | 64 | 128 | 2048, "K3 stage, busy warps on all 4 SMSPs"),
                          (224, 16 | 64 | 128 | 4096, "K3 stage, busy warps off the issuer's SMSP")):
        mode = 2 | extra
        run(L, buf, mode, N, 0, iters=1024, ld_iters=200000)
        r = run(L, buf, mode, N, 0, ld_iters=3000000)
        print(f"{tag:44s} N{N:3d}: {r['cyc_per_mma']:7.1f} clk/MMA  {r['mac_clk_sm']:7.0f} MAC/clk/SM", flush=True)


if __name__ == "__main__":
    main()
