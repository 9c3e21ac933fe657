"""Walk-seed anchors of the fused MC kernel (tt_common.cuh kAnchor2 / kAnchor3).

A target element stores the source elements containing 48 anchor points (barycentric
coordinates below); a sample starts its facet walk at the anchor nearest to it in
barycentric space among the first 16 (N < 32) or all 48 (per-block slot table, tt_mc.cu).  The first k+1 anchors are the
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


def anchors(D, m=16, n=200000, iters=80, fixed=None):
    """m anchors: the rows of ``fixed`` (default: centroid and corner points) kept, the rest
    k-means centres of uniform samples of the reference simplex."""
    K = D + 1
    if fixed is None:
        fixed = np.array([[1 / K] * K] + [[(1 + K) / (2 * K) if i == j else 1 / (2 * K) for j in range(K)]
                                         for i in range(K)])
    nf = len(fixed)
    rng = np.random.default_rng(0)
    U = O.bary_map(rng.random((n, D)))
    C = U[rng.choice(n, m, replace=False)]
    C[:nf] = fixed
    for _ in range(iters):
        # nearest centre, in chunks (the same arithmetic as one (n, m, K) array, cache-sized)
        a = np.concatenate([((U[i:i + 8192, None, :] - C[None]) ** 2).sum(-1).argmin(1)
                            for i in range(0, n, 8192)])
        order = np.argsort(a, kind="stable")
        bounds = np.searchsorted(a[order], np.arange(m + 1))
        C = np.array([U[order[bounds[k]:bounds[k + 1]]].mean(0) if bounds[k + 1] > bounds[k] else C[k]
                      for k in range(m)])
        C[:nf] = fixed
    return C


def round6(C):
    return np.array([[float(f"{v:.6f}") for v in r] for r in C])


if __name__ == "__main__":
    # 48 anchors (TT_SEED_ANCHORS): the first 16 are the 16-anchor set (what the fused kernel
    # uses below N = 32), the other 32 k-means centres with those 16 fixed.  --first16 prints
    # only the 16-anchor set (seconds instead of minutes)
    first16 = "--first16" in sys.argv
    for D in (2, 3):
        C16 = round6(anchors(D, 16))
        C = C16 if first16 else round6(anchors(D, 48, fixed=C16))
        print(f"static __constant__ double kAnchor{D}[TT_SEED_ANCHORS][{D + 1}] = {{")
        for r in C:
            print("    {" + ", ".join(f"{v:.6f}" for v in r) + "},")
        print("};")
