"""Walk-seed anchors of the fused MC kernel (tt_common.cuh kAnchor2 / kAnchor3).

A target element stores the source elements containing 16 anchor points (barycentric
coordinates below); a sample starts its facet walk at the anchor nearest to it in
barycentric space (per-block slot table, tt_mc.cu).  The first k+1 anchors are the
centroid and the corner points (v_i + c)/2 (the cheap closed-form slot rule used when
there is no table); the other 16-(k+1) are k-means centres of uniform samples of the
reference simplex with those fixed.  Measured match rate "sample in its anchor's source
element" on the C2-style cube pair (n=12, N=64 Sobol): 56.5 % -> 66.7 % (3-D); 2-D square
pair (n=150): 71.7 % -> 83.6 %.

python scripts/seed_anchors.py   # prints the C tables
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
import tt_oracle as O  # noqa: E402  (bary_map only: uniform samples of the simplex)


def anchors(D, m=16, n=200000, iters=80):
    K = D + 1
    fixed = np.array([[1 / K] * K] + [[(1 + K) / (2 * K) if i == j else 1 / (2 * K) for j in range(K)]
                                     for i in range(K)])
    rng = np.random.default_rng(0)
    U = O.bary_map(rng.random((n, D)))
    C = U[rng.choice(n, m, replace=False)]
    C[:K + 1] = fixed
    for _ in range(iters):
        a = ((U[:, None, :] - C[None]) ** 2).sum(-1).argmin(1)
        C = np.array([U[a == k].mean(0) if (a == k).any() else C[k] for k in range(m)])
        C[:K + 1] = fixed
    return C


if __name__ == "__main__":
    for D in (2, 3):
        C = anchors(D)
        print(f"__constant__ double kAnchor{D}[16][{D + 1}] = {{")
        for r in C:
            print("    {" + ", ".join(f"{v:.6f}" for v in r) + "},")
        print("};")
