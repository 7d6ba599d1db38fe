"""Summarise a GPU round's ncu output into profiles/ (tracked).

    python tools/summarize_profiles.py r01

Reads gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum launch
list of a bench run) and gpurun_out/prof_top.ncu-rep (ncu --set full of the
dominant kernel), writes profiles/<tag>_launches.md, profiles/<tag>_top.md
and profiles/dram_traffic.json (per-launch DRAM bytes of the dominant
kernel, read by bench.py for the roofline "traffic" field).
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return None
    text = [ln for ln in open(path) if not ln.startswith("==")]
    rows = [r for r in csv.DictReader(text) if r.get("Metric Name") == "gpu__time_duration.sum"]
    per = defaultdict(list)
    for r in rows:
        name = r["Kernel Name"]
        short = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        per[(short, r["Grid Size"], r["Block Size"])].append(float(r["Metric Value"].replace(",", "")))
    total = sum(sum(v) for v in per.values())
    lines = [f"# {tag}: ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1`",
             "", "Cold-cache, serialised per-launch times (ncu `gpu__time_duration.sum`, `--clock-control none`).",
             "Compare shares, not absolute times.", "",
             "| kernel | grid | block | launches | mean us | share |", "|---|---|---|---|---|---|"]
    for (k, g, b), v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {g} | {b} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / total:.1%} |")
    lines.append("")
    ours = sum(len(v) for (k, _, _), v in per.items() if k.startswith(("k1", "k2", "k3", "k4", "kref")))
    lines.append(f"Total launches: {len(rows)}; {ours} of them are this repo's kernels, the rest are torch "
                 f"utility kernels outside the SpMM (buffer fills of the host pipeline's setup).")
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    return per


def ncu_raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return {}
    return dict(zip(rows[0], rows[2]))


def raw_csv(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return {}
    return dict(zip(rows[0], rows[2]))


def top(tag, cell="c5b_4096x1024", which="top", traffic_file=True):
    rep = os.path.join(OUT, f"prof_{which}.ncu-rep")
    csvp = os.path.join(OUT, f"prof_{which}_raw.csv")   # exported on the box (tools/gpu_round.sh)
    if os.path.exists(csvp):
        m = raw_csv(csvp)
    elif os.path.exists(rep):
        m = ncu_raw(rep)
    else:
        return
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.sum.per_cycle_active", "lts__t_sectors_srcunit_tex_op_read.sum",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.pct_of_peak_sustained_elapsed",
            "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
            "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_on.avg.pct_of_peak_sustained_elapsed",
            "derived__lts__lts2xbar_bytes.sum.per_second", "derived__lts__lts2xbar_bytes.sum.peak_sustained",
            "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "Kernel Name"]
    kern = {"top": "tc", "sp": "sp", "ws": "ws"}.get(which, which)
    what = "the dominant kernel" if which == "top" else f"kernel=\"{kern}\" on the same linear"
    lines = [f"# {tag}: ncu --set full of {what} ({cell}, `tests/prof_one.py c5b {kern} 3 nk`)", "",
             "| metric | value |", "|---|---|"]
    for k in keys:
        if k in m:
            lines.append(f"| `{k}` | {m[k]} |")
    with open(os.path.join(PROF, f"{tag}_{which}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if not traffic_file:
        return

    def mb(k):
        try:
            v = float(m[k].replace(",", ""))
        except (KeyError, ValueError):
            return None
        return v

    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    if rd is not None and wr is not None:
        # ncu reports MB in the raw page for these byte counters
        traffic = {cell: {"dram_read_MB": rd, "dram_write_MB": wr, "per_launch_bytes": (rd + wr) * 1e6,
                          "source": f"profiles/{tag}_top.md"}}
        with open(os.path.join(PROF, "dram_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    top(tag)
    for which in ("sp", "ws"):
        if os.path.exists(os.path.join(OUT, f"prof_{which}_raw.csv")):
            top(tag, which=which, traffic_file=False)
    print("ok")
