"""Sobol sequences on the device (reference: sobol.py:1-52).

Gray-code construction with Joe-Kuo direction numbers, dimensions 1-3 (d = 3 extends
the reference for tetrahedra: s=2, a=1, m=(1,3)); the all-zeros point is skipped and
``skip`` discards further points.  Integer-exact, so identical to the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import InvalidParameter


def sobol(count: int, dim: int = 2, skip: int = 0, device: bool = False):
    if count < 1:
        raise InvalidParameter(f"count must be >= 1, got {count}")
    if skip < 0:
        raise InvalidParameter(f"skip must be >= 0, got {skip}")
    out = torch.empty((count, dim), dtype=torch.float64, device=_lib.device())
    _lib.call("tt_plan_sobol", dim, count, skip, _lib.ptr(out), _lib.stream_handle())
    return out if device else out.cpu().numpy()


def sobol_2d(count: int, skip: int = 0) -> np.ndarray:
    """First ``count`` points of the 2-D Sobol sequence in [0, 1)^2 (sobol.py:34-52)."""
    return sobol(count, 2, skip)
