"""Does the target's element ORDER matter for the fused kernel?  The C3 torus pair (file
order: phi fastest, whole circles) and the same target with its elements in Morton order of
their centroids; also the C2 cube.  Kernel time per load (CUDA events), N = 64.
python scripts/order_probe.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200.dist import morton_codes  # noqa: E402
from paper_2603_00538_b200.montecarlo import element_contributions  # noqa: E402


def timed(tgt, box, plan, reps=10):
    out = torch.empty((tgt.n_elems, 4), dtype=torch.float64, device="cuda")
    for _ in range(3):
        element_contributions(tgt, box, plan, out=out)
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); element_contributions(tgt, box, plan, out=out); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


for name, (t, s) in {"c3": (tt.generate_torus_mesh(40, 80, 260, perturbation=0.2, seed=20),
                            tt.generate_torus_mesh(36, 88, 240, perturbation=0.2, seed=10, split="kuhn_mirror")),
                     "c2": (tt.generate_cube_mesh(55, 0.2, seed=20), tt.generate_cube_mesh(55, 0.2, seed=10, split="kuhn_mirror"))}.items():
    fs = tt.NodalField.from_function(s, tt.get_field("smooth", dim=3).fn)
    box = tt.MeshBackedField(fs, tt.UniformGridLocator.build(s))
    plan = tt.SamplePlan.build(64, "sobol", 0, dim=3)
    perm = np.argsort(morton_codes(t.centroids), kind="stable")
    tm = tt.TetMesh.from_arrays(t.nodes, t.elements[perm])
    print(name, "file order %.3f ms" % timed(t, box, plan), "morton order %.3f ms" % timed(tm, box, plan), flush=True)
