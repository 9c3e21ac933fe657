"""Walk/schedule statistics of the fused kernel from the instrumented build
(TT_LIB_PATH=<lib built with -DTT_MC_STATS>): lane utilisation of the flattened loop,
walk steps, exact fallbacks and snaps (outside samples) per sample.
python scripts/mc_stats.py [3 | 2 | torus]"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200 import _lib  # noqa: E402
from paper_2603_00538_b200.montecarlo import load_vector  # noqa: E402

lib = _lib.lib()
get = lib.tt_debug_mc_stats
get.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 8)()
arg = sys.argv[1] if len(sys.argv) > 1 else "3"
dim = 2 if arg == "2" else 3
if arg == "torus":   # C3: non-matching faceted tori, outside samples snapped
    tgt = tt.generate_torus_mesh(40, 80, 260, perturbation=0.2, seed=20)
    src = tt.generate_torus_mesh(36, 88, 240, perturbation=0.2, seed=10, split="kuhn_mirror")
elif dim == 3:
    tgt = tt.generate_cube_mesh(55, 0.2, seed=20, split="kuhn")
    src = tt.generate_cube_mesh(55, 0.2, seed=10, split="kuhn_mirror")
else:
    tgt = tt.generate_square_mesh(707, 0.2, seed=20, diagonal="right")
    src = tt.generate_square_mesh(707, 0.2, seed=10, diagonal="left")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=dim).fn)
box = tt.MeshBackedField(fs, tt.UniformGridLocator.build(src))
for n in (16, 64, 256, 1024):
    plan = tt.SamplePlan.build(n, "sobol", 0, dim=dim)
    load_vector(tgt, box, plan)
    torch.cuda.synchronize()
    get(buf, 1)
    load_vector(tgt, box, plan)
    torch.cuda.synchronize()
    get(buf, 1)
    it, busy, samples, steps, slow, snaps = list(buf)[:6]
    print(json.dumps({"dim": dim, "N": n, "lane_util": round(busy / (32 * it), 4),
                      "iters_per_sample_lane": round(32 * it / samples, 3),
                      "steps_per_sample": round(steps / samples, 4),
                      "fallback_per_sample": round(slow / samples, 6),
                      "snap_per_sample": round(snaps / samples, 7), "samples": samples}))
