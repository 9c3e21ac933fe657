"""Per-iteration phase split of the textbook slab PCG (path="slab") from the instrumented build
(TT_LIB_PATH=<lib built with -DTT_PCG_TRACE>): globaltimer marks of block 0."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200 import _lib  # noqa: E402
from paper_2603_00538_b200.fem import pcg_device  # noqa: E402
from paper_2603_00538_b200.montecarlo import load_vector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 55
tgt = tt.generate_cube_mesh(n, 0.2, seed=20, split="kuhn")
src = tt.generate_cube_mesh(n, 0.2, seed=10, split="kuhn_mirror")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
b = load_vector(tgt, tt.MeshBackedField(fs), tt.SamplePlan.build(64, "sobol", 0, dim=3))
mass = tgt.device.mass
for _ in range(3):
    pcg_device(mass, b, tol=1e-12, path="slab")
torch.cuda.synchronize()
buf = (C.c_ulonglong * (64 * 6))()
_lib.lib().tt_debug_pcg_trace(buf)
t = np.array(buf, dtype=np.float64).reshape(64, 6)
t = t[t[:, 0] > 0]
it = len(t)
ph = np.diff(t, axis=1) / 1e3                       # us: spmv, syncA, totalA, vecB, syncB
nxt = (t[1:, 0] - t[:-1, 5]) / 1e3                 # totalsB + tests + beta until next iteration
names = ["spmv (phase A)", "block sum + grid sync A", "grid total A", "vector update (phase B)",
         "block sums + grid sync B"]
print(f"rows {tgt.n_nodes}, iterations traced {it}")
for k, nm in enumerate(names):
    print(f"  {nm:28s} {np.median(ph[:, k]):7.2f} us")
print(f"  {'grid totals B + tests':28s} {np.median(nxt):7.2f} us")
print(f"  {'iteration':28s} {np.median(np.diff(t[:, 0])) / 1e3:7.2f} us")
