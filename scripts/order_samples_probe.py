"""Does the order of a shared plan's samples change the fused kernel's time?  The C2 load
with the Sobol plan as generated, sorted by nearest walk anchor (slot), and sorted along a
Morton curve of the barycentric point (spatially coherent consecutive samples).  Same sums in
another order: b agrees to rounding."""
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200.montecarlo import element_contributions  # noqa: E402

root = Path(__file__).resolve().parents[1]
txt = (root / "paper_2603_00538_b200/csrc/tt_common.cuh").read_text()
blk = txt[txt.index("kAnchor3[16][4] = {"):]
blk = blk[:blk.index("};")]
A = np.array([[float(v) for v in re.findall(r"[-\d.]+", r)] for r in re.findall(r"\{([^{}]+)\}", blk)])

tgt = tt.generate_cube_mesh(55, 0.2, seed=20, split="kuhn")
src = tt.generate_cube_mesh(55, 0.2, seed=10, split="kuhn_mirror")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
box = tt.MeshBackedField(fs, tt.UniformGridLocator.build(src))
N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
base = tt.SamplePlan.build(N, "sobol", 0, dim=3)
lam = base.barycentric
slot = ((lam[:, None, :] - A[None]) ** 2).sum(-1).argmin(1)
q = np.clip((lam[:, :3] * 1024).astype(np.int64), 0, 1023)
morton = np.zeros(N, np.int64)
for bit in range(10):
    for c in range(3):
        morton |= ((q[:, c] >> bit) & 1) << (3 * bit + c)
orders = {"generated": np.arange(N), "by_slot": np.argsort(slot, kind="stable"), "morton": np.argsort(morton, kind="stable"),
          "slot_then_morton": np.lexsort((morton, slot)),
          "slot_then_distance": np.lexsort((((lam - A[slot]) ** 2).sum(1), slot))}
out = {}
ref = None
for name, perm in orders.items():
    plan = tt.SamplePlan(N, "sobol", 0, barycentric=lam[perm], dim=3)
    for _ in range(3):
        element_contributions(tgt, box, plan)
    ts = []
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); c = element_contributions(tgt, box, plan); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    b = tgt.device.reduce_nodes(c).cpu().numpy()
    ref = b if ref is None else ref
    out[name] = {"ms": round(float(np.median(ts)), 4), "db": float(np.max(np.abs(b - ref)) / np.max(np.abs(ref)))}
print(json.dumps({"N": N, **out}))
