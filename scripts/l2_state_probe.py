"""Diagnostic: how much of a streaming kernel's time after bench.py's L2 flush is the
write-back of the flush's own dirty lines.  Times the C5 folded-R SpMV (b = R c) after
(a) the bench flush (256 MB zero_, leaves L2 full of dirty lines), (b) the same flush
followed by a 256 MB read (L2 left full of clean lines), (c) no flush (R partly L2-resident).
python scripts/l2_state_probe.py   (GPU)"""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_00538_b200 as tt  # noqa: E402

sys.argv = ["bench.py", "--config", "c5"]
args = bench.parse_args()
args.samples = 50
tgt, src, fs, loc, mass = bench.build_problem(args, tt)
plan = tt.SamplePlan.build(args.samples, "sobol", 0, dim=3)
op = tt.MCTransferOperator(tgt, src, plan, source_locator=loc)
rp, ci, va = op.R
alg = 8 * (tgt.n_nodes + 1) + 12 * va.numel() + 8 * src.n_nodes + 8 * tgt.n_nodes
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")


def run(mode, reps=30):
    ts = []
    for i in range(reps + 3):
        if mode in ("dirty", "clean"):
            flush.zero_()
        if mode == "clean":
            flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        op.load(fs, check=False)
        e.record()
        if i >= 3:
            ts.append((s, e))
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ts)
    print(f"{mode:6s} {ms * 1e3:6.1f} us  {alg / (ms * 1e-3) / 1e9:7.0f} GB/s (algorithmic {alg / 1e6:.1f} MB)")


for m in ("dirty", "clean", "none"):
    run(m)
