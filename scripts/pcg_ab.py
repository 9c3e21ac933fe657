"""A/B of PCG builds: median cg_solve time (device, CUDA events) on the C1 (2-D, 501k rows,
slab), C2 (3-D, 176k rows, slab) and C4 (3-D, 1.77M rows, L2-streaming) mass matrices.
python scripts/pcg_ab.py libA.so libB.so ...   (each in its own process via TT_LIB_PATH)"""
import json
import os
import subprocess
import sys

CODE = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_00538_b200 as tt
from paper_2603_00538_b200.fem import pcg_device, decode_result
out = {}
for name, mk in (("c1", lambda: tt.generate_square_mesh(707, 0.2, seed=20, diagonal="right")),
                 ("c2", lambda: tt.generate_cube_mesh(55, 0.2, seed=20)),
                 ("c4", lambda: tt.generate_cube_mesh(120, 0.2, seed=20))):
    m = mk()
    M = m.device.mass
    f = np.sin(3 * m.nodes[:, 0]) * np.cos(2 * m.nodes[:, 1]) + 2.0
    b = M.matvec(torch.as_tensor(f, device="cuda"))
    ts = []
    for k in range(23):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); x, bx, res = pcg_device(M, b, tol=1e-12); e.record(); e.synchronize()
        if k >= 3: ts.append(s.elapsed_time(e))
    r = decode_result(res)
    err = float((x - torch.as_tensor(f, device="cuda")).abs().max())
    out[name] = {"ms": float(np.median(ts)), "iters": int(r.iterations), "conv": int(r.converged), "err_vs_f": err}
print(json.dumps(out))
'''
res = {}
for lib in sys.argv[1:]:
    env = dict(os.environ, TT_LIB_PATH=os.path.abspath(lib))
    p = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env)
    res[os.path.basename(lib)] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else p.stderr[-800:]
print(json.dumps(res, indent=1))
