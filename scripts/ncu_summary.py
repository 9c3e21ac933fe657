"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into plain text for profiles/.

python scripts/ncu_summary.py report.ncu-rep        # key SOL / memory / stall metrics
python scripts/ncu_summary.py launches.csv          # per-kernel device-time shares
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate", "No Eligible",
        "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    kn, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    print(f"kernel: {rows[1][kn][:150]}")
    for r in rows[1:]:
        if r[mi] in KEEP:
            print(f"  {r[mi]:40s} {r[vi]:>16s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    for i, n in enumerate(rr[0]):
        if n in RAW:
            print(f"  {n:40s} {rr[2][i]:>16s} {rr[1][i]}")
    stalls = []
    for i, n in enumerate(rr[0]):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                stalls.append((float(rr[2][i]), n[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    print("  stall samples: " + ", ".join(f"{n} {v / tot * 100:.1f}%" for v, n in sorted(stalls, reverse=True)[:6]))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    kn, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[kn].split("(")[0].replace("void ", "")
            tot[name] += float(r[vi].replace(",", ""))
            cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e3:10.1f} {v / s * 100:6.1f}%")


if __name__ == "__main__":
    p = sys.argv[1]
    rep(p) if p.endswith(".ncu-rep") else launches(p)
