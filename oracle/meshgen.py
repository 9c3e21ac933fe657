"""Synthetic benchmark meshes for the CPU reference arm -- TEST / BASELINE
INFRASTRUCTURE ONLY (bench.py --impl reference, tests).

The reference package generates only 2-D squares (mesh.py:186-232, used directly from
oracle/_ref for C1).  BASELINE.json's 3-D configs are defined by two generators -- a
Kuhn-split jittered unit cube (C2, C4) and a swept-annulus torus (C3) -- restated here in
plain numpy so the reference arm builds its inputs without importing the product
package.  ``tests/test_oracle.py`` checks they produce the product's meshes exactly
(same nodes, same connectivity, same orientation).
"""

import numpy as np

PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def _orient(nodes, elems):
    """Swap two vertices of negatively oriented tets (positive signed volume)."""
    v = nodes[elems]
    a = v[:, 0]
    u, w, t = v[:, 1] - a, v[:, 2] - a, v[:, 3] - a
    cx = w[:, 1] * t[:, 2] - w[:, 2] * t[:, 1]
    cy = w[:, 2] * t[:, 0] - w[:, 0] * t[:, 2]
    cz = w[:, 0] * t[:, 1] - w[:, 1] * t[:, 0]
    vol = ((u[:, 0] * cx + u[:, 1] * cy) + u[:, 2] * cz) / 6.0
    neg = vol < 0
    elems = elems.copy()
    elems[neg] = elems[neg][:, [0, 2, 1, 3]]
    return elems


def _kuhn(corner):
    tets = []
    for p in PERMS:
        off = [0, 0, 0]
        verts = [corner(*off)]
        for axis in p[:2]:
            off[axis] = 1
            verts.append(corner(*off))
        verts.append(corner(1, 1, 1))
        tets.append(np.stack(verts, axis=-1))
    return np.stack(tets, axis=1).reshape(-1, 4).astype(np.int32)


def cube(n, perturbation=0.2, seed=0, split="kuhn"):
    """(nodes (n+1)^3 x 3, tets 6 n^3 x 4): unit cube, interior nodes jittered by
    U(-p h, p h) from default_rng(seed); split 'kuhn' (000-111 diagonal) or 'kuhn_mirror'."""
    g = np.linspace(0, 1, n + 1)
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    nodes = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
    h = 1.0 / n
    if perturbation > 0:
        jit = np.random.default_rng(seed).uniform(-perturbation * h, perturbation * h, size=nodes.shape)
        inner = np.all((nodes > 0) & (nodes < 1), axis=1)
        nodes[inner] += jit[inner]
    i, j, k = (a.ravel() for a in np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij"))
    m = n + 1

    def corner(a, b, c):
        if split == "kuhn_mirror":
            a = 1 - a
        return ((i + a) * m + (j + b)) * m + (k + c)
    return nodes, _orient(nodes, _kuhn(corner))


def torus(n_rho, n_theta, n_phi, perturbation=0.2, seed=0, split="kuhn", R=1.0, a_in=0.15, a_out=0.45):
    """Swept annulus a_in <= rho <= a_out around the z axis, (rho, theta, phi) hexes
    Kuhn-split; interior radii and all angles jittered by U(-p h, p h)."""
    i, j, k = np.meshgrid(np.arange(n_rho + 1), np.arange(n_theta), np.arange(n_phi), indexing="ij")
    rho = a_in + (a_out - a_in) * i / n_rho
    th = 2 * np.pi * j / n_theta
    ph = 2 * np.pi * k / n_phi
    if perturbation > 0:
        jit = np.random.default_rng(seed).uniform(-perturbation, perturbation, size=(3,) + rho.shape)
        inner = (i > 0) & (i < n_rho)
        rho = rho + np.where(inner, jit[0] * (a_out - a_in) / n_rho, 0.0)
        th = th + jit[1] * 2 * np.pi / n_theta
        ph = ph + jit[2] * 2 * np.pi / n_phi
    rr = R + rho * np.cos(th)
    nodes = np.column_stack([(rr * np.cos(ph)).ravel(), (rr * np.sin(ph)).ravel(), (rho * np.sin(th)).ravel()])
    ci, cj, ck = (a.ravel() for a in np.meshgrid(np.arange(n_rho), np.arange(n_theta), np.arange(n_phi),
                                                 indexing="ij"))

    def corner(a, b, c):
        if split == "kuhn_mirror":
            a = 1 - a
        return ((ci + a) * n_theta + (cj + b) % n_theta) * n_phi + (ck + c) % n_phi
    return nodes, _orient(nodes, _kuhn(corner))
