"""Dense / sparse tcgen05 kind::i8 MMA rate with one and two issuers, and the SM clock
under a sustained MMA load (clock64 / %globaltimer), on the GPU box:

    python tools/dense_rate.py

Uses the microbenchmark kernel of tools/mma_rate.cu (profiles/r02_k2_experiments.md, section 2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ctypes, torch
import mma_rate as M
if not os.path.exists(M.SO): M.build()
L = ctypes.CDLL(M.SO)
L.mma_rate.restype = ctypes.c_int
L.mma_rate.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int, ctypes.c_int]
buf = torch.randint(0, 255, (32 << 20,), dtype=torch.uint8, device="cuda")
for sparse in (0, 2):
  for N in (128, 256):
    for two in (0, 1):
        for stream in (0, 4096):
            mode = sparse | 16 | ((4 | 8192) if two else 0)
            M.run(L, buf, mode, N, stream, iters=1024)
            r = M.run(L, buf, mode, N, stream)
            extra = f"  stream {r['stream_B_clk']:5.1f} B/clk/SM" if stream else ""
            print(f"{'sparse' if sparse else 'dense'} SS N{N} issuers {1+two}: {r['cyc_per_mma']:7.1f} clk/MMA  {r['mac_clk_sm']:7.0f} MAC/clk/SM{extra}", flush=True)
print("--- sustained: dense SS N256, 2 issuers, stream; SM clock = cycles / globaltimer")
for iters in (8192, 65536, 524288):
    mode = 0 | 16 | 4 | 8192
    out = (ctypes.c_ulonglong * (148 * 4))()
    ms = ctypes.c_float()
    err = L.mma_rate(mode, iters, 256, 4096, 148, ctypes.c_void_p(buf.data_ptr()), buf.numel() // 16384, out, ctypes.byref(ms), 0, 0)
    cyc = out[0]; ns = out[1]
    print(f"iters {iters}: {cyc/iters:.1f} clk/MMA, {ns/1e3:.0f} us, SM clock {cyc/ns*1e3:.0f} MHz, rc {err}", flush=True)
