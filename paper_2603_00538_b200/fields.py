"""Analytic source fields compiled for in-kernel evaluation (reference: fields.py:1-67).

``parse_field`` accepts the reference's whitelisted expression language (+ - * / **,
unary minus, sin/cos/exp, numeric constants, pi, e; x, y and -- for 3-D -- z) and
compiles it to a postfix program (``tt_expr_t``) that the fused Monte-Carlo kernel
interprets per sample in registers.  Plain Python callables written with numpy
ufuncs (``lambda x, y: np.sin(5*x*y)``) are *traced* into the same program by
calling them once with symbolic arguments; a callable that cannot be traced stays a
host black box and is evaluated through the materialised-points path.
"""

from __future__ import annotations

import ast
import math

import numpy as np

from .errors import InvalidParameter

_ALLOWED_CALLS = {"sin": np.sin, "cos": np.cos, "exp": np.exp}
_ALLOWED_NAMES = {"x", "y", "z", "pi", "e"}
_ALLOWED_NODES = (
    ast.Expression, ast.BinOp, ast.UnaryOp, ast.Constant, ast.Name, ast.Call,
    ast.Load, ast.Add, ast.Sub, ast.Mult, ast.Div, ast.Pow, ast.USub, ast.UAdd,
)

Program = list  # [(opname, const)]


def _validate(node: ast.AST) -> None:
    for sub in ast.walk(node):
        if not isinstance(sub, _ALLOWED_NODES):
            raise InvalidParameter(
                f"unsupported syntax in field expression: {type(sub).__name__}")
        if isinstance(sub, ast.Name) and sub.id not in _ALLOWED_NAMES | set(_ALLOWED_CALLS):
            raise InvalidParameter(f"unknown name {sub.id!r} in field expression")
        if isinstance(sub, ast.Call):
            if not isinstance(sub.func, ast.Name) or sub.func.id not in _ALLOWED_CALLS:
                raise InvalidParameter("only sin, cos, exp calls are allowed")
        if isinstance(sub, ast.Constant) and not isinstance(sub.value, (int, float)):
            raise InvalidParameter("only numeric constants are allowed")


def _pow_ops(exponent_prog: Program) -> Program:
    """numpy power fast paths: x**2 -> square, x**0.5 -> sqrt (exact like np.power)."""
    if len(exponent_prog) == 1 and exponent_prog[0][0] == "const":
        c = exponent_prog[0][1]
        if c == 2.0:
            return [("square", 0.0)]
        if c == 0.5:
            return [("sqrt", 0.0)]
    return exponent_prog + [("pow", 0.0)]


def _compile(node) -> Program:
    if isinstance(node, ast.Expression):
        return _compile(node.body)
    if isinstance(node, ast.Constant):
        return [("const", float(node.value))]
    if isinstance(node, ast.Name):
        if node.id in ("x", "y", "z"):
            return [(node.id, 0.0)]
        return [("const", math.pi if node.id == "pi" else math.e)]
    if isinstance(node, ast.UnaryOp):
        inner = _compile(node.operand)
        return inner + [("neg", 0.0)] if isinstance(node.op, ast.USub) else inner
    if isinstance(node, ast.BinOp):
        left, right = _compile(node.left), _compile(node.right)
        if isinstance(node.op, ast.Pow):
            return left + _pow_ops(right)
        op = {ast.Add: "add", ast.Sub: "sub", ast.Mult: "mul", ast.Div: "div"}[type(node.op)]
        return left + right + [(op, 0.0)]
    if isinstance(node, ast.Call):
        return _compile(node.args[0]) + [(node.func.id, 0.0)]
    raise InvalidParameter(f"cannot compile {type(node).__name__}")


def stack_depth(prog: Program) -> int:
    depth = best = 0
    for op, _ in prog:
        if op in ("const", "x", "y", "z"):
            depth += 1
        elif op in ("add", "sub", "mul", "div", "pow"):
            depth -= 1
        best = max(best, depth)
    return best


# ------------------------------------------------------------------ tracing
class _TraceError(Exception):
    pass


_UFUNC_UNARY = {np.sin: "sin", np.cos: "cos", np.exp: "exp", np.sqrt: "sqrt", np.log: "log",
                np.tan: "tan", np.absolute: "abs", np.negative: "neg", np.square: "square"}
_UFUNC_BINARY = {np.add: "add", np.subtract: "sub", np.multiply: "mul",
                 np.true_divide: "div", np.power: "pow"}


class _Sym:
    """Symbolic array stand-in that records numpy arithmetic as a postfix program."""

    __array_priority__ = 10000

    def __init__(self, prog: Program):
        self.prog = prog

    @staticmethod
    def lift(v) -> Program:
        if isinstance(v, _Sym):
            return v.prog
        if isinstance(v, (int, float, np.floating, np.integer)) and not isinstance(v, bool):
            return [("const", float(v))]
        if isinstance(v, np.ndarray) and v.ndim == 0:
            return [("const", float(v))]
        raise _TraceError(f"cannot trace operand of type {type(v).__name__}")

    def _bin(self, other, op, swap=False):
        a, b = self.lift(self), self.lift(other)
        if swap:
            a, b = b, a
        if op == "pow":
            return _Sym(a + _pow_ops(b))
        return _Sym(a + b + [(op, 0.0)])

    def __add__(self, o): return self._bin(o, "add")
    def __radd__(self, o): return self._bin(o, "add", True)
    def __sub__(self, o): return self._bin(o, "sub")
    def __rsub__(self, o): return self._bin(o, "sub", True)
    def __mul__(self, o): return self._bin(o, "mul")
    def __rmul__(self, o): return self._bin(o, "mul", True)
    def __truediv__(self, o): return self._bin(o, "div")
    def __rtruediv__(self, o): return self._bin(o, "div", True)
    def __pow__(self, o): return self._bin(o, "pow")
    def __rpow__(self, o): return self._bin(o, "pow", True)
    def __neg__(self): return _Sym(self.prog + [("neg", 0.0)])
    def __pos__(self): return self

    def __bool__(self):
        raise _TraceError("data-dependent control flow")

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        if method != "__call__" or kwargs:
            raise _TraceError(f"unsupported ufunc use {ufunc.__name__}.{method}")
        if ufunc in _UFUNC_UNARY and len(inputs) == 1:
            return _Sym(self.lift(inputs[0]) + [(_UFUNC_UNARY[ufunc], 0.0)])
        if ufunc in _UFUNC_BINARY and len(inputs) == 2:
            a, b = self.lift(inputs[0]), self.lift(inputs[1])
            if _UFUNC_BINARY[ufunc] == "pow":
                return _Sym(a + _pow_ops(b))
            return _Sym(a + b + [(_UFUNC_BINARY[ufunc], 0.0)])
        raise _TraceError(f"unsupported ufunc {ufunc.__name__}")

    def __array_function__(self, func, types, args, kwargs):
        if func in (np.full_like,):
            return _Sym([("const", float(args[1] if len(args) > 1 else kwargs["fill_value"]))])
        if func is np.ones_like:
            return _Sym([("const", 1.0)])
        if func is np.zeros_like:
            return _Sym([("const", 0.0)])
        if func in (np.asarray, np.asanyarray, np.broadcast_to, np.copy):
            return args[0]
        raise _TraceError(f"unsupported numpy function {func.__name__}")


def trace_callable(fn, dim: int) -> Program | None:
    """Postfix program of ``fn(x, y[, z])`` or None if it cannot be traced."""
    args = [_Sym([(n, 0.0)]) for n in ("x", "y", "z")[:dim]]
    try:
        out = fn(*args)
        prog = _Sym.lift(out)
    except Exception:  # anything untraceable stays a host black box
        return None
    if len(prog) > 64 or stack_depth(prog) > 16:
        return None
    return prog


def parse_field(expr: str, dim: int | None = None):
    """Compile an arithmetic expression in x, y (and z) into an analytic field whose
    device program is the compiled postfix code (fields.py:34-52)."""
    from .montecarlo import AnalyticField
    try:
        tree = ast.parse(expr, mode="eval")
    except SyntaxError as exc:
        raise InvalidParameter(f"invalid field expression {expr!r}: {exc}") from exc
    _validate(tree)
    prog = _compile(tree)
    if len(prog) > 64 or stack_depth(prog) > 16:
        raise InvalidParameter(f"field expression {expr!r} is too long for the device program")
    code = compile(tree, "<field>", "eval")
    env = dict(_ALLOWED_CALLS, pi=np.pi, e=np.e)

    def fn(x, y, z=None):
        out = eval(code, {"__builtins__": {}}, dict(env, x=x, y=y, z=z if z is not None else 0.0 * x))
        return np.broadcast_to(np.asarray(out, dtype=np.float64), np.shape(x)).copy() \
            if np.ndim(out) == 0 else out
    uses_z = any(op == "z" for op, _ in prog)
    if dim is None:
        dim = 3 if uses_z else None
    return AnalyticField(fn, name=expr, program=prog, dim=dim)


#: the two test fields used throughout the experiment harnesses (fields.py:56-59)
NAMED_FIELDS = {
    "linear": "x + y",
    "smooth": "sin(x)*cos(y) + 2",
}

#: 3-D variants (builder-defined; the reference is 2-D only)
NAMED_FIELDS_3D = {
    "linear": "x + y + z",
    "smooth": "sin(x)*cos(y)*cos(z) + 2",
}


def get_field(name_or_expr: str, dim: int | None = None):
    """Named field (``linear``, ``smooth``) or a custom expression (fields.py:62-67)."""
    table = NAMED_FIELDS_3D if dim == 3 else NAMED_FIELDS
    expr = table.get(name_or_expr, name_or_expr)
    f = parse_field(expr, dim=dim)
    f.name = name_or_expr
    return f
