"""C3 study: conservation error vs samples per element on the ~5M-tet torus pair
(BASELINE.json configs[2]).  Writes one JSON object to stdout."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402
from paper_2603_00538_b200.montecarlo import map_points  # noqa: E402

t0 = time.time()
tgt = tt.generate_torus_mesh(40, 80, 260, perturbation=0.2, seed=20)
src = tt.generate_torus_mesh(36, 88, 240, perturbation=0.2, seed=10, split="kuhn_mirror")
fs = tt.NodalField.from_function(src, tt.get_field("smooth", dim=3).fn)
box = tt.MeshBackedField(fs)
_ = tgt.device.mass
setup = time.time() - t0
out = {"target_tets": tgt.n_elems, "source_tets": src.n_elems, "setup_s": round(setup, 1), "rows": []}
# reference value of the sampled integral: a high-N per-element Philox estimate
ref_plan = tt.SamplePlan.build(4096, "philox", 12345, dim=3)
i_ref = float(tt.assemble_load_mc(tgt, box, ref_plan, device=True).sum())
out["sampled_integral_ref"] = {"plan": "philox N=4096 seed 12345", "value": i_ref}
out["domain_mismatch_e_mass"] = abs(tt.integrate_field(fs) - i_ref) / abs(tt.integrate_field(fs))
tt.transfer_mc(tgt, box, tt.SamplePlan.build(16, "sobol", 0, dim=3))   # warm-up (seeds, setup)
for mode in ("sobol", "philox"):
    for N in (16, 64, 256, 400, 800, 1600):
        plan = tt.SamplePlan.build(N, mode, 0, dim=3)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ft = tt.transfer_mc(tgt, box, plan, cg_tol=1e-12)
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        b_sum = float(tt.assemble_load_mc(tgt, box, plan, device=True).sum())
        i_t = tt.integrate_field(ft)
        row = {"mode": mode, "N": N, "samples": tgt.n_elems * N, "ms": round(ms, 2),
               "samples_per_s": tgt.n_elems * N / (ms * 1e-3),
               "solve_conservation": abs(i_t - b_sum) / abs(b_sum),
               "mc_mass_error_vs_ref": abs(i_t - i_ref) / abs(i_ref),
               "e_mass_vs_source": tt.mass_error(fs, ft)}
        if N == 64:
            # fraction of samples outside the faceted source boundary (snapped)
            loc = box.locator
            pts = map_points(tgt, plan, 0, 200000).reshape(-1, 3)
            el, _ = loc.locate_many(pts)
            row["outside_fraction_first200k_elems"] = float((el < 0).float().mean())
        out["rows"].append(row)
print(json.dumps(out))
