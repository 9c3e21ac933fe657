"""Where the end-to-end coupling step's time goes beyond the device step (C2): CUDA-event
times of the H2D copy alone, the D2H copy alone, the graph replay alone and the whole
CouplingStep call (pinned host buffers; L2 flushed before each, as the bench)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402

tgt = tt.generate_cube_mesh(55, 0.2, seed=20, split="kuhn")
src = tt.generate_cube_mesh(55, 0.2, seed=10, split="kuhn_mirror")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
loc = tt.UniformGridLocator.build(src)
plan = tt.SamplePlan.build(64, "sobol", 0, dim=3)
step = tt.CouplingStep(tgt, src, plan, source_locator=loc)
c_host = torch.as_tensor(fs.coeffs).pin_memory()
x_host = torch.empty(tgt.n_nodes, dtype=torch.float64).pin_memory()
x_dev = torch.empty(tgt.n_nodes, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    step(c_host)
torch.cuda.synchronize()


def timed(fn, reps=30):
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return round(float(np.median(ts)), 1)


def spin_call():
    step.c_dev.copy_(c_host, non_blocking=True)
    step._graph.replay()
    ev = torch.cuda.Event()
    ev.record()
    while not ev.query():
        pass


def yield_call():
    step.c_dev.copy_(c_host, non_blocking=True)
    step._graph.replay()
    torch.cuda.current_stream().synchronize()


out = {
    "copy_replay_sync_us": timed(yield_call),
    "copy_replay_spin_us": timed(spin_call),
    "h2d_us": timed(lambda: step.c_dev.copy_(c_host, non_blocking=True)),
    "d2h_us": timed(lambda: x_host.copy_(x_dev, non_blocking=True)),
    "replay_us": timed(lambda: step._graph.replay()),
    "replay_sync_us": timed(lambda: (step._graph.replay(), torch.cuda.current_stream().synchronize())),
    "call_us": timed(lambda: step(c_host)),
    "bytes_each_way": int(c_host.numel() * 8),
}
print(json.dumps(out))
