"""Per-iteration phase split of the pipelined slab PCG (the default C2 solve) from the
instrumented build: TT_LIB_PATH=<lib built with -DTT_PCG_TRACE> python scripts/pcg_pipe_trace.py
(globaltimer marks of block 0)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200 import _lib  # noqa: E402
from paper_2603_00538_b200.fem import pcg_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 55
tgt = tt.generate_cube_mesh(n, 0.2, seed=20, split="kuhn")
mass = tgt.device.mass
b = mass.matvec(torch.as_tensor(np.sin(3 * tgt.nodes[:, 0]) + 2.0, device="cuda"))
for _ in range(3):
    pcg_device(mass, b, tol=1e-12, path="auto")
torch.cuda.synchronize()
buf = (C.c_ulonglong * (64 * 6))()
_lib.lib().tt_debug_pcg_trace(buf)
t = np.array(buf, dtype=np.float64).reshape(64, 6)
t = t[t[:, 1] > 0]
ph = np.diff(t, axis=1) / 1e3
names = ["residual test + alpha/beta", "SpMV + own-row updates", "block partial sums",
         "wait for slowest block + grid sync", "grid totals (3)"]
print(f"rows {tgt.n_nodes}, iterations traced {len(t)}")
for k, nm in enumerate(names):
    print(f"  {nm:36s} {np.median(ph[:, k]):7.2f} us")
print(f"  {'iteration':36s} {np.median(np.diff(t[:, 0])) / 1e3:7.2f} us")
