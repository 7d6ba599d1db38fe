"""Host <-> device copy bandwidth on the box (pinned buffers, CUDA events):
H2D alone, D2H alone, and both directions at once on two streams -- the
ceiling of bench.py's e2e (host-buffer) number.

    python tools/pcie_bw.py
"""
import torch

MB = 1 << 20


def bw(nbytes=256 * MB, reps=5):
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, dirs in (("h2d", ("in",)), ("d2h", ("out",)), ("both", ("in", "out"))):
        best = 0.0
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_event(e0)
            s2.wait_event(e0)
            if "in" in dirs:
                with torch.cuda.stream(s1):
                    d_a.copy_(h_in, non_blocking=True)
            if "out" in dirs:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_b, non_blocking=True)
            cur = torch.cuda.current_stream()
            cur.wait_stream(s1)
            cur.wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = max(best, nbytes / (ms / 1e3) / 1e9)
        res[name] = best
    return res


if __name__ == "__main__":
    r = bw()
    print(f"pinned 256 MB copies, GB/s per direction: H2D {r['h2d']:.1f}, D2H {r['d2h']:.1f}, "
          f"both at once {r['both']:.1f} (each direction)")
