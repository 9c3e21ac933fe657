"""Per-step kernel shares from an ncu launch list (--metrics gpu__time_duration.sum --csv):
median time per launch of each step kernel, and the other launches of the run.

python scripts/launch_shares.py launches.csv "mc_mesh_kernel<3, 0, 4," pack_grad reduce_nodes pcg_ell
"""
import csv
import statistics
import sys
from collections import defaultdict

path, step = sys.argv[1], sys.argv[2:]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
kn, vi = rows[hi].index("Kernel Name"), rows[hi].index("Metric Value")
t = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        t[r[kn].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")) / 1e3)
per = {}
for pat in step:
    names = [k for k in t if pat in k]
    per[pat] = (statistics.median([v for k in names for v in t[k]]), sum(len(t[k]) for k in names), names)
tot = sum(v[0] for v in per.values())
for pat, (us, n, names) in per.items():
    print(f"{names[0][:60]:60s} {us:9.1f} us {us / tot * 100:6.1f} %   ({n} launches)")
print(f"{'step total':60s} {tot:9.1f} us")
print("\nOther launches in the run (setup, sweep variants, bench probes, torch's L2 flush):")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    if not any(k in names for _, _, names in per.values()):
        print(f"  {k[:70]:70s} x{len(v):3d}  median {statistics.median(v):9.1f} us")
