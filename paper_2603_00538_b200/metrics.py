"""Conservation and accuracy reporting (reference: metrics.py:1-94).

DoF and single-mesh metrics run on the device.  The supermesh metrics need the
mesh-intersection subsystem (intersect.py), which is out of scope for this
framework; they raise ``NotImplementedError``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .errors import ZeroDenominator
from .fem import NodalField, check_same_mesh, integrate_field


@dataclass
class ErrorReport:
    """One row of transfer-quality metrics plus run metadata (metrics.py:16-32)."""

    method: str = ""
    e_l2_supermesh: float = np.nan
    e_mass_supermesh: float = np.nan
    e_l2_dof: float = np.nan
    e_mass_mesh: float = np.nan
    meta: dict = field(default_factory=dict)

    CSV_FIELDS = ("method", "e_l2_supermesh", "e_mass_supermesh", "e_l2_dof", "e_mass_mesh")

    def to_csv_row(self) -> str:
        vals = [getattr(self, f) for f in self.CSV_FIELDS[1:]]
        return ",".join([self.method] + [repr(v) for v in vals])


def dof_l2_error(approx: NodalField, reference: NodalField) -> float:
    """Relative l2 error over the DoF vectors of two fields on one mesh (metrics.py:77-83)."""
    check_same_mesh(approx, reference)
    den = torch.linalg.vector_norm(reference.coeffs_dev)
    if float(den) == 0.0:
        raise ZeroDenominator("reference field has zero l2 norm")
    return float(torch.linalg.vector_norm(approx.coeffs_dev - reference.coeffs_dev) / den)


def mesh_mass_error(approx: NodalField, reference: NodalField, rule=None) -> float:
    """Relative conservation error, both integrals on the shared mesh (metrics.py:86-94)."""
    check_same_mesh(approx, reference)
    mass_ref = integrate_field(reference, rule)
    if mass_ref == 0.0:
        raise ZeroDenominator("reference field has zero mass")
    return float(abs(integrate_field(approx, rule) - mass_ref) / abs(mass_ref))


def mass_error(source: NodalField, target: NodalField) -> float:
    """Relative conservation error between fields on different meshes, each
    integrated exactly on its own mesh (P1 integrals are exact)."""
    ms = integrate_field(source)
    if ms == 0.0:
        raise ZeroDenominator("source field has zero mass")
    return float(abs(ms - integrate_field(target)) / abs(ms))


def supermesh_l2_error(*args, **kwargs):
    raise NotImplementedError("supermesh metrics need mesh intersection (out of scope)")


def supermesh_mass_error(*args, **kwargs):
    raise NotImplementedError("supermesh metrics need mesh intersection (out of scope)")
