"""CPU: libtt_b200.so loads without a GPU, exports every entry point declared in
include/tt_b200.h, and the ctypes struct layouts match the C compiler's."""

import re
import subprocess
import tempfile
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "tt_b200.h"


def _declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_seam():
    names = _declared()
    for must in ("tt_locate_many", "tt_locate", "tt_grid_count", "tt_grid_fill", "tt_mc_load",
                 "tt_plan_sobol", "tt_plan_pcg64", "tt_plan_philox", "tt_reduce_nodes",
                 "tt_mass_pattern", "tt_mass_fill", "tt_pcg", "tt_snap", "tt_nearest"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2603_00538_b200 import _lib
    lib = _lib.load_library(require_device=False)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(_lib.EXPORTED)
    assert lib.tt_version() >= 100


def test_library_is_sm100a_only():
    so = ROOT / "paper_2603_00538_b200" / "libtt_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_struct_layouts_match_c():
    from paper_2603_00538_b200 import _lib
    import ctypes as C
    structs = {"tt_mesh_t": _lib.tt_mesh_t, "tt_grid_t": _lib.tt_grid_t, "tt_plan_t": _lib.tt_plan_t,
               "tt_expr_t": _lib.tt_expr_t, "tt_source_t": _lib.tt_source_t,
               "tt_pcg_result_t": _lib.tt_pcg_result_t, "tt_dpcg_t": _lib.tt_dpcg_t}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src, exe = Path(d) / "l.c", Path(d) / "l"
        src.write_text("\n".join(lines))
        subprocess.run(["gcc", "-std=c11", str(src), "-o", str(exe)], check=True)
        got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                            text=True, check=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, f"{name}.{fname}"


def test_no_device_raises_loudly():
    import torch
    from paper_2603_00538_b200 import _lib
    from paper_2603_00538_b200.errors import DeviceUnavailable
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(DeviceUnavailable):
        _lib.lib()


def test_contrib_ld_layouts():
    """The C ABI's contribution layout argument: 0 for a row-major (n, k) tensor (including
    empty and one-row tensors), ld for the transpose of a (k, ld) buffer and its row slices;
    anything else is refused."""
    import pytest
    import torch
    from paper_2603_00538_b200._lib import contrib_ld
    for n in (0, 1, 2, 7):
        assert contrib_ld(torch.empty((n, 4), dtype=torch.float64)) == 0
        t = torch.empty((4, n), dtype=torch.float64).t()
        assert contrib_ld(t) in ((0,) if n <= 1 else (n,))
    t = torch.empty((3, 10), dtype=torch.float64).t()
    assert contrib_ld(t[4:]) == 10 and contrib_ld(t[4:]) >= t[4:].shape[0]
    with pytest.raises(ValueError):
        contrib_ld(torch.empty((10, 8), dtype=torch.float64)[:, ::2])
