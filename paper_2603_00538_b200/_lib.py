"""ctypes binding of the C ABI in ``include/tt_b200.h`` (libtt_b200.so).

This is the only place the host layer crosses into native code.  There is no CPU
fallback: if the library or a CUDA device is missing every entry point raises
``DeviceUnavailable`` (loudly, at first use).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import torch

from .errors import (DeviceUnavailable, DimensionMismatch, InvalidParameter,
                     TransferError)

# TT_LIB_PATH: load another build of the library (same-box A/B measurements)
LIB_PATH = Path(os.environ.get("TT_LIB_PATH") or Path(__file__).resolve().parent / "libtt_b200.so")

TT_OK, TT_ERR_INVALID_PARAMETER, TT_ERR_DIMENSION_MISMATCH, TT_ERR_CUDA, TT_ERR_CAPACITY = 0, 1, 2, 3, 4
TT_FLAG_NONFINITE, TT_FLAG_OUTSIDE_STRICT, TT_FLAG_CAPACITY, TT_FLAG_INVALID_DENSITY = 1, 2, 4, 8
TT_FLAG_NONMANIFOLD = 16
TT_FLAG_WIDE_ROWS = 32
TT_SEED_ANCHORS = 48
TT_FLAG_SNAPPED = 64
TT_FLAG_PEER_TIMEOUT = 128
TT_HINT_DEFER_SNAP = 1
TT_PLAN_SHARED, TT_PLAN_PHILOX = 0, 1
TT_SRC_EXPR, TT_SRC_MESH, TT_SRC_VALUES, TT_SRC_CACHED = 0, 1, 2, 3
TT_OUTSIDE_SNAP, TT_OUTSIDE_STRICT = 0, 1
TT_EXPR_MAX_OPS, TT_EXPR_MAX_STACK = 64, 16

OPS = {"const": 0, "x": 1, "y": 2, "z": 3, "add": 4, "sub": 5, "mul": 6, "div": 7,
       "pow": 8, "neg": 9, "sin": 10, "cos": 11, "exp": 12, "sqrt": 13, "log": 14,
       "tan": 15, "abs": 16, "square": 17}


def rec_stride(dim: int) -> int:
    return 8 if dim == 2 else 16


def wrec_stride(dim: int) -> int:
    return 6 if dim == 2 else 10


class tt_mesh_t(C.Structure):
    _fields_ = [("dim", C.c_int32), ("reserved", C.c_int32), ("n_nodes", C.c_int64),
                ("n_elems", C.c_int64), ("nodes", C.c_void_p), ("elems", C.c_void_p),
                ("measure", C.c_void_p), ("gid", C.c_void_p)]


class tt_grid_t(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int32 * 3), ("walk", C.c_int32),
                ("reserved", C.c_int32), ("lo", C.c_double * 3),
                ("hi", C.c_double * 3), ("n_elems", C.c_int64), ("cell_start", C.c_void_p),
                ("cell_elems", C.c_void_p), ("rec", C.c_void_p), ("centroids", C.c_void_p),
                ("wrec", C.c_void_p)]


class tt_plan_t(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim", C.c_int32), ("n_samples", C.c_int64),
                ("lam", C.c_void_p), ("seed", C.c_uint64), ("order", C.c_void_p),
                ("lam_walk", C.c_void_p)]


class tt_expr_t(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("ops", C.c_int32 * TT_EXPR_MAX_OPS),
                ("consts", C.c_double * TT_EXPR_MAX_OPS)]


class tt_source_t(C.Structure):
    _fields_ = [("kind", C.c_int32), ("outside", C.c_int32), ("dim", C.c_int32),
                ("hints", C.c_int32), ("expr", tt_expr_t), ("grid", tt_grid_t),
                ("src_elems", C.c_void_p), ("coeffs", C.c_void_p), ("values", C.c_void_p),
                ("cached_ids", C.c_void_p), ("seeds", C.c_void_p), ("elem_coeffs", C.c_void_p),
                ("elem_grad", C.c_void_p)]


class tt_pcg_result_t(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("residual", C.c_double),
                ("best_residual", C.c_double), ("converged", C.c_int32),
                ("zero_rhs", C.c_int32)]


class tt_dpcg_t(C.Structure):
    _fields_ = [("n_own", C.c_int64), ("n_ext", C.c_int64), ("width", C.c_int32), ("reserved", C.c_int32),
                ("ell_cols", C.c_void_p), ("ell_vals", C.c_void_p), ("diag", C.c_void_p), ("b", C.c_void_p),
                ("x", C.c_void_p), ("best_x", C.c_void_p), ("r", C.c_void_p), ("w", C.c_void_p),
                ("p", C.c_void_p), ("s", C.c_void_p), ("dinv", C.c_void_p), ("u", C.c_void_p),
                ("send_start", C.c_void_p), ("send_pos", C.c_void_p), ("n_send", C.c_int64),
                ("send_buf", C.c_void_p),
                ("part", C.c_void_p), ("sums", C.c_void_p), ("state", C.c_void_p),
                ("tol", C.c_double), ("maxiter", C.c_int64)]


_P = C.c_void_p
_I64 = C.c_int64
_I = C.c_int
_D = C.c_double
_U64 = C.c_uint64

_SIGNATURES = {
    "tt_last_error": ([], C.c_char_p),
    "tt_version": ([], _I),
    "tt_device_sm_count": ([C.POINTER(_I)], _I),
    "tt_plan_sobol": ([_I, _I64, _I64, _P, _P], _I),
    "tt_plan_pcg64": ([_I, _I64, _U64, _U64, _U64, _U64, _P, _P], _I),
    "tt_bary_map": ([_I, _I64, _P, _P, _P], _I),
    "tt_plan_philox": ([_I, _I64, _I64, _I64, _U64, _P, _P], _I),
    "tt_geometry": ([C.POINTER(tt_mesh_t), _P, _P, _P, _P], _I),
    "tt_bbox": ([_I, _I64, _P, _P, _P], _I),
    "tt_grid_count": ([C.POINTER(tt_mesh_t), C.POINTER(tt_grid_t), _P, _P], _I),
    "tt_grid_fill": ([C.POINTER(tt_mesh_t), C.POINTER(tt_grid_t), _P, _P, _P], _I),
    "tt_locate": ([C.POINTER(tt_grid_t), _P, _I64, _D, _P, _P, _P], _I),
    "tt_locate_many": ([_P, _I64, _I, _I, C.POINTER(_D), _P, _P, _P, _P, _D, _P, _P, _P], _I),
    "tt_grid_walk_prep": ([C.POINTER(tt_mesh_t), _P, _P, _D, _P, _P, _P, _P], _I),
    "tt_seed_elements": ([C.POINTER(tt_grid_t), C.POINTER(tt_mesh_t), _I64, _I64, _P, _P, _P], _I),
    "tt_nearest": ([C.POINTER(tt_grid_t), _P, _I64, _P, _P], _I),
    "tt_snap": ([C.POINTER(tt_grid_t), _P, _I64, _P, _P, _P], _I),
    "tt_map_points": ([C.POINTER(tt_mesh_t), _I64, _I64, C.POINTER(tt_plan_t), _P, _P], _I),
    "tt_eval_points": ([C.POINTER(tt_source_t), _P, _I64, _P, _P, _P], _I),
    "tt_plan_walk_order": ([_I, _I64, _P, _P, _P, _P], _I),
    "tt_mc_load": ([C.POINTER(tt_mesh_t), _I64, _I64, C.POINTER(tt_plan_t),
                    C.POINTER(tt_source_t), _P, _P, _P, _P], _I),
    "tt_mc_load_ld": ([C.POINTER(tt_mesh_t), _I64, _I64, C.POINTER(tt_plan_t),
                       C.POINTER(tt_source_t), _P, _I64, _P, _P, _P], _I),
    "tt_mc_load_density": ([C.POINTER(tt_mesh_t), _I64, _I64, C.POINTER(tt_plan_t),
                            C.POINTER(tt_source_t), _P, _P, _P, _P], _I),
    "tt_mc_cache_ids": ([C.POINTER(tt_mesh_t), _I64, _I64, C.POINTER(tt_plan_t),
                         C.POINTER(tt_grid_t), _P, _P, _P], _I),
    "tt_pack_coeffs": ([C.POINTER(tt_mesh_t), _P, _P, _P], _I),
    "tt_pack_grad": ([C.POINTER(tt_mesh_t), _P, _P, _P], _I),
    "tt_mc_fold": ([C.POINTER(tt_mesh_t), C.POINTER(tt_plan_t), C.POINTER(tt_mesh_t), _P, _P,
                    C.POINTER(_I64), C.POINTER(_P), _P], _I),
    "tt_mc_fold_finish": ([_P, _P, _P, _P, _P], _I),
    "tt_spmv_rect": ([_I64, _P, _P, _P, _P, _P, _P], _I),
    "tt_incidence_count": ([C.POINTER(tt_mesh_t), _P, _P], _I),
    "tt_incidence_fill": ([C.POINTER(tt_mesh_t), _P, _P, _P, _P], _I),
    "tt_reduce_nodes": ([_I64, _I, _P, _P, _I64, _I64, _P, _P, _P], _I),
    "tt_reduce_nodes_ld": ([_I64, _I, _P, _P, _I64, _I64, _P, _I64, _P, _P], _I),
    "tt_mass_pattern": ([C.POINTER(tt_mesh_t), _P, _P, _P, _P, _P], _I),
    "tt_mass_fill": ([C.POINTER(tt_mesh_t), _P, _P, C.POINTER(_D), _P, _P, _P, _P], _I),
    "tt_pcg_workspace_doubles": ([_I64], _I64),
    "tt_pcg": ([_I64, _P, _P, _P, _P, _D, _I64, _P, _P, _P, _P, _P], _I),
    "tt_csr_to_ell": ([_I64, _P, _P, _P, _I, _P, _P, _P, _P, _P], _I),
    "tt_pcg_ell": ([_I64, _I, _P, _P, _P, _P, _D, _I64, _P, _P, _P, _P, _P], _I),
    "tt_pcg_ell_slab": ([_I64, _I, _P, _P, _P, _P, _D, _I64, _P, _P, _P, _P, _P], _I),
    "tt_pcg_ell_slab_pipelined": ([_I64, _I, _P, _P, _P, _P, _D, _I64, _P, _P, _P, _P, _P], _I),
    "tt_spmv": ([_I64, _P, _P, _P, _P, _P, _P], _I),
    "tt_integrate_p1": ([C.POINTER(tt_mesh_t), _P, _P, _P], _I),
    "tt_supermesh_integrals": ([C.POINTER(tt_mesh_t), _P, C.POINTER(tt_mesh_t), _P, C.POINTER(tt_grid_t),
                                _D, _P, _P, _P], _I),
    "tt_dpcg_part_doubles": ([], _I64),
    "tt_dpcg_start": ([_P, _P], _I),
    "tt_dpcg_update": ([_P, _I, _P], _I),
    "tt_dpcg_spmv": ([_P, _I, _P], _I),
    "tt_dpcg_finish": ([_P, _P, _P], _I),
    "tt_reduce_nodes_ranked": ([_I64, _P, _P, _P, _P, _P, _P], _I),
    "tt_dpcg_peer_solve": ([_P, _P, _P, _P, _P, _I64, _I, _I, _P, _P, _P, _P], _I),
    "tt_gather_rows": ([_I64, _I, _P, _P, _P, _P], _I),
    "tt_scatter_rows": ([_I64, _I, _P, _P, _P, _P], _I),
    "tt_fp64_peak_probe": ([_I64, _P, C.POINTER(_I), C.POINTER(_I), _P], _I),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load_library(require_device: bool = True):
    """Load libtt_b200.so (and check for a CUDA device unless told otherwise)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceUnavailable(
                f"{LIB_PATH.name} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    if require_device and not torch.cuda.is_available():
        raise DeviceUnavailable("no CUDA device visible: this framework has no CPU path")
    return _lib


_lib_dev = None


def lib():
    """The library, with a CUDA device checked once per process (hot path: every call)."""
    global _lib_dev
    if _lib_dev is None:
        _lib_dev = load_library(True)
    return _lib_dev


def stream_handle(stream=None):
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    # the current stream's raw handle straight from the CUDA context torch keeps: this is
    # on every ABI call, and torch.cuda.current_stream() builds a Stream object through
    # device-index normalisation (~5-15 us of host time per call)
    lib()
    torch.cuda.init()   # no-op once initialised; the raw query needs the lazy init done
    return C.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def check(code: int, what: str = ""):
    if code == TT_OK:
        return
    msg = (_lib.tt_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if code == TT_ERR_INVALID_PARAMETER:
        raise InvalidParameter(text)
    if code == TT_ERR_DIMENSION_MISMATCH:
        raise DimensionMismatch(text)
    raise TransferError(f"CUDA library error {code}: {text}")


def call(name: str, *args):
    fn = getattr(lib(), name)
    check(fn(*args), name)


def call_status(name: str, *args) -> int:
    """Call an entry point that reports TT_ERR_CAPACITY as a normal outcome (nothing was
    launched, the caller picks another kernel); any other error raises."""
    code = getattr(lib(), name)(*args)
    if code != TT_ERR_CAPACITY:
        check(code, name)
    return code


def contrib_ld(t) -> int:
    """Layout of an (n, k) element-contribution tensor for the C ABI: 0 when row-major
    (contiguous), ld when it is the transpose of a (k, ld) buffer (strides (1, ld), ld >= n)."""
    n, k = t.shape
    if t.is_contiguous():
        return 0
    if t.stride(0) == 1 and t.stride(1) >= n:
        return int(t.stride(1))
    raise ValueError(f"contribution tensor with strides {t.stride()}: need row-major or transposed")


def ptr(t) -> C.c_void_p:
    if t is None:
        return C.c_void_p(None)
    return C.c_void_p(t.data_ptr())


def device() -> torch.device:
    lib()
    torch.cuda.init()
    return torch.device("cuda", torch._C._cuda_getDevice())


def sm_count() -> int:
    out = C.c_int(0)
    lib().tt_device_sm_count(C.byref(out))
    return out.value


def status_word() -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device())


def mesh_desc(dim, n_nodes, n_elems, nodes, elems, measure=None, gid=None) -> tt_mesh_t:
    return tt_mesh_t(dim, 0, n_nodes, n_elems, ptr(nodes).value, ptr(elems).value,
                     ptr(measure).value, ptr(gid).value)


if os.environ.get("TT_B200_EAGER_LOAD"):
    load_library(False)
