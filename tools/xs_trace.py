"""Summarise a K3 role timeline (experiment builds: SI_LIB=<exp lib>
SI_XS_TRACE=<file> python tests/prof_one.py c5b sp 1 nk).

Roles: 0 MMA issuer (1 tile start after tempty, 2 stage full, 3 rfull,
4 tile issued); 1..12 epilogue warps of the leader CTA (5 tfull, 6 release,
7 tile done); 13..16 gather warps (8 rempty ok, 9 gathered)."""
import sys
import numpy as np

N = 4096
raw = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(20, N)
ev = (raw >> np.uint64(56)).astype(np.int64)
t = (raw & np.uint64((1 << 56) - 1)).astype(np.int64)
t0 = t[t > 0].min()


def events(role, kind):
    m = (ev[role] == kind) & (t[role] > 0)
    return (t[role][m] - t0) / 1e3   # us


ts, ti = events(0, 1), events(0, 4)
print(f"MMA tiles: {len(ts)}; span {ti[-1]:.1f} us")
print("tile issue time (start->issued) us: median", np.median(ti - ts[:len(ti)]))
print("gap tile issued -> next start (tempty wait) us: median", np.median(ts[1:len(ti)] - ti[:-1]))
full, pre = events(0, 2), events(0, 10)
k = min(len(full), len(pre))
w = full[:k] - pre[:k]
print(f"stage full waits: n {k}, median {np.median(w) * 1e3:.0f} ns, mean {np.mean(w) * 1e3:.0f} ns, "
      f"total {np.sum(w):.1f} us; issue between stages median {np.median(pre[1:k] - full[:k - 1]) * 1e3:.0f} ns")
for r in (1, 2, 3, 4):
    tf, rl, dn = events(r, 5), events(r, 6), events(r, 7)
    k = min(len(tf), len(rl), len(dn))
    if k:
        print(f"epi warp {r + 1}: tiles {k}, tfull->release {np.median(rl[:k] - tf[:k]):.2f} us, "
              f"tfull->done {np.median(dn[:k] - tf[:k]):.2f} us, idle before tfull {np.median(tf[1:k] - dn[:k-1]):.2f} us")
for r in (13, 14):
    a, b = events(r, 8), events(r, 9)
    k = min(len(a), len(b))
    if k:
        print(f"gather warp {r - 12}: {k} tiles, gather {np.median(b[:k] - a[:k]):.2f} us")
# MMA tile timeline vs epilogue of the same accumulator
print("first 12 tiles (start, issued) us:", [(round(a, 2), round(b, 2)) for a, b in zip(ts[:12], ti[:12])])
print("epi warp 2 (tfull, release, done):", [(round(a, 2), round(b, 2), round(c, 2)) for a, b, c in zip(events(1, 5)[:8], events(1, 6)[:8], events(1, 7)[:8])])
