"""Driver for ncu / timing of the supermesh metrics kernel: the C1-size 2-D pair (1M / 1M
triangles), E_L2 and E_mass of an MC transfer.  python scripts/profile_supermesh.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402

tgt = tt.generate_square_mesh(707, 0.2, seed=20, diagonal="right")
src = tt.generate_square_mesh(707, 0.2, seed=10, diagonal="left")
fs = tt.NodalField.from_function(src, tt.get_field("smooth").fn)
ft = tt.transfer_mc(tgt, tt.MeshBackedField(fs), tt.SamplePlan.build(64, "sobol", 0))
iset = tt.find_intersections(tgt, src)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    iset._cache.clear()
    e = tt.supermesh_l2_error(fs, ft, iset)
torch.cuda.synchronize()
print(f"E_L2 {e:.6e}  E_mass {tt.supermesh_mass_error(fs, ft, iset):.3e}  "
      f"{(time.perf_counter() - t) / 5 * 1e3:.2f} ms per metric evaluation (1M x 1M triangles)")
