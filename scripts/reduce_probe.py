"""Node gather (tt_reduce_nodes) timing at C1/C2/C4 size: CUDA events per launch, with the
contributions freshly rewritten (L2-resident, as after the fused load kernel) and after an
L2 flush; checks b against np.add.at bitwise.  Runs the package of the current directory
(tree A/B: cd <tree> && python <this script>)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00538_b200 as tt  # noqa: E402


def run(name, m, reps=50):
    dm = m.device
    g = torch.Generator(device="cuda").manual_seed(1)
    contrib = torch.randn((m.n_elems, dm.k), dtype=torch.float64, device="cuda", generator=g)
    b = dm.reduce_nodes(contrib)
    ref = np.zeros(m.n_nodes)
    np.add.at(ref, m.elements, contrib.cpu().numpy())
    out = {"config": name, "bitwise_add_at": bool(np.array_equal(b.cpu().numpy(), ref))}
    half = m.n_elems // 2
    bh = dm.reduce_nodes(contrib[half:], half, m.n_elems)
    refh = np.zeros(m.n_nodes)
    np.add.at(refh, m.elements[half:], contrib[half:].cpu().numpy())
    out["range_bitwise"] = bool(np.array_equal(bh.cpu().numpy(), refh))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    layouts = [("rowmajor", contrib)]
    if hasattr(tt._lib, "contrib_ld"):          # trees with the transposed layout
        ct = contrib.t().contiguous().t()
        out["transposed_bitwise"] = bool(np.array_equal(dm.reduce_nodes(ct).cpu().numpy(), ref))
        bt = dm.reduce_nodes(ct[half:], half, m.n_elems)
        out["transposed_range_bitwise"] = bool(np.array_equal(bt.cpu().numpy(), refh))
        layouts.append(("transposed", ct))
    for (lay, cb), warm in [(l_, w_) for l_ in layouts for w_ in (True, False)]:
        ts = []
        for _ in range(reps):
            if warm:
                cb.mul_(1.0)
            else:
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dm.reduce_nodes(cb, out=b)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        out[f"{lay}_{'l2' if warm else 'cold'}_us"] = round(ts[len(ts) // 2], 2)
    out["alg_bytes"] = m.n_elems * dm.k * 12 + m.n_nodes * 16
    return out


for name, m in [("C2", tt.generate_cube_mesh(55, 0.2, seed=20, split="kuhn")),
                ("C1", tt.generate_square_mesh(500, 0.2, seed=20)),
                ("C4", tt.generate_cube_mesh(120, 0.2, seed=20, split="kuhn"))]:
    print(json.dumps(run(name, m)), flush=True)
