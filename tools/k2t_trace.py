"""Analyse a K2t role timeline (SI_K2T_TRACE=<file>, experiment builds): per-role
event streams of pair 0 -> waits and intervals.

    SI_K2T_TRACE=/tmp/t.bin python tests/prof_one.py c5b tc 1 nk; python tools/k2t_trace.py /tmp/t.bin
"""
import sys

import numpy as np

N = 8192
NAMES = {1: "mma:full", 2: "mma:tempty", 3: "mma:rfull", 20: "epi:tfull", 21: "epi:release", 30: "gat:rempty",
         31: "gat:done", 22: "epi:ch_start", 23: "epi:slot_ok", 24: "epi:math_done", 26: "epi:fenced",
         25: "epi:stored"}


def main(path):
    a = np.fromfile(path, dtype=np.uint64).reshape(16, N)
    t0 = min(int(v & ((1 << 56) - 1)) for v in a.ravel() if v)
    roles = {}
    for r in range(16):
        v = a[r][a[r] != 0]
        if len(v) == 0:
            continue
        kind = (v >> np.uint64(56)).astype(int)
        t = (v & np.uint64((1 << 56) - 1)).astype(np.int64) - t0
        roles[r] = (kind, t)
    end = max(t.max() for _, t in roles.values())
    print(f"span {end / 1e3:.1f} us")
    for r, (kind, t) in sorted(roles.items()):
        for k in sorted(set(kind)):
            tk = t[kind == k]
            d = np.diff(tk)
            nm = NAMES.get(k, f"prod{k - 10}")
            print(f"role {r:2d} {nm:12s} n={len(tk):5d} first={tk[0] / 1e3:7.2f}us "
                  f"interval mean={d.mean() if len(d) else 0:7.1f}ns p50={np.median(d) if len(d) else 0:7.1f} "
                  f"p90={np.percentile(d, 90) if len(d) else 0:7.1f}")
    # MMA thread: per stage, how long did it wait on full? (gap between consecutive events of role 8)
    if 8 in roles:
        kind, t = roles[8]
        gaps = np.diff(t)
        nxt = kind[1:]
        for k in sorted(set(nxt)):
            g = gaps[nxt == k]
            print(f"mma gap before {NAMES.get(k, k):11s}: n={len(g)} mean={g.mean():7.1f}ns sum={g.sum() / 1e3:7.1f}us")
    if 12 in roles:
        kind, t = roles[12]
        gaps = np.diff(t)
        nxt = kind[1:]
        for k in sorted(set(nxt)):
            g = gaps[nxt == k]
            print(f"epi gap before {NAMES.get(k, k):13s}: n={len(g)} mean={g.mean():7.1f}ns sum={g.sum() / 1e3:7.1f}us")
    if len(sys.argv) > 2:
        kind, t = roles[8]
        for k, tt in list(zip(kind, t))[:int(sys.argv[2])]:
            print(NAMES.get(k, k), tt)




def latency(path):
    """TMA latency per stage: leader's full-ok minus the later of the two CTAs' issue times."""
    a = np.fromfile(path, dtype=np.uint64).reshape(16, N)
    msk = np.uint64((1 << 56) - 1)

    def ev(r, k):
        v = a[r][a[r] != 0]
        return (v[(v >> np.uint64(56)) == k] & msk).astype(np.int64)
    full = ev(8, 1)
    iss = []
    for j in range(len(full)):
        p = j % 4
        t0 = ev(2 * p, 10 + p)
        t1 = ev(2 * p + 1, 10 + p)
        if j // 4 < min(len(t0), len(t1)):
            iss.append(max(t0[j // 4], t1[j // 4]))
    iss = np.array(iss)
    lat = full[:len(iss)] - iss
    print(f"stage latency issue->full: mean {lat.mean():.0f} ns p10 {np.percentile(lat, 10):.0f} "
          f"p50 {np.median(lat):.0f} p90 {np.percentile(lat, 90):.0f}")
    # how long a slot waits between its release... (full of stage j -> empty-ok of j+S at the producer)
    skew = np.array([abs(ev(2 * (j % 4), 10 + j % 4)[j // 4] - ev(2 * (j % 4) + 1, 10 + j % 4)[j // 4])
                     for j in range(min(len(full), 4 * len(ev(0, 10))))])
    print(f"rank0/rank1 producer skew: mean {skew.mean():.0f} ns p90 {np.percentile(skew, 90):.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
    latency(sys.argv[1])
