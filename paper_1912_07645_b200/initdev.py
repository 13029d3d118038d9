"""Initial data on the device.

The reference evaluates its initial-data expression language on the host
with numpy (iodsl/expr.py:338-386 ``eval_init``) once per sample; for MC/QMC
ensembles that host work and the H2D copy dominate short runs.  Here the
per-component expression trees are compiled once into a small stack
bytecode and evaluated by ``fvb_init_eval`` at every cell centre of every
sample of a batch, straight into the padded device buffer the solver runs
on.

Parity: IEEE + - * / and sqrt, the comparisons, the ternary and numpy's
array fast paths of ``np.power`` (exponent 2 -> square, 0.5 -> sqrt, -1 ->
reciprocal) are reproduced operation by operation, so expressions built from
them evaluate bitwise like the reference; sin / cos / exp / general pow are
CUDA's (<= 2 ulp from glibc), so expressions using them agree to rounding
level (a ternary threshold sitting within an ulp of a cell centre could
flip -- the reference's own caveat).

``DeviceInit`` accepts the reference's AST nodes (duck-typed on the class
names Num/Var/Rand/Unary/Binary/Ternary/Call of iodsl/expr.py:28-70) or
expression strings (parsed by ``parse_expr`` below, same grammar).  It is a
drop-in ``evaluate_init(grid, vector)`` for ``run_mc`` / ``run_mlmc``, which
recognise it and skip the host entirely.
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import errors as E
from .grid import Field

# --- the expression language (grammar of iodsl/expr.py:1-12) ---------------


@dataclass(frozen=True)
class Num:
    value: float


@dataclass(frozen=True)
class Var:
    name: str


@dataclass(frozen=True)
class Rand:
    index: int


@dataclass(frozen=True)
class Unary:
    op: str
    operand: object


@dataclass(frozen=True)
class Binary:
    op: str
    left: object
    right: object


@dataclass(frozen=True)
class Ternary:
    cond: object
    then: object
    otherwise: object


@dataclass(frozen=True)
class Call:
    name: str
    args: tuple


ARITY = {"sin": 1, "cos": 1, "exp": 1, "abs": 1, "sqrt": 1, "min": 2, "max": 2}
_TOK = re.compile(r"\s*(?:(?P<num>(?:\d+\.\d*|\.\d+|\d+)(?:[eE][+-]?\d+)?)|(?P<ident>[A-Za-z_]\w*)"
                  r"|(?P<op><=|>=|==|!=|[-+*/^<>()?:,]))")
_CMP = ("<", "<=", ">", ">=", "==", "!=")


def parse_expr(text: str):
    """Text -> AST.  Precedence, loosest first: ternary (right assoc.),
    comparisons, + -, * /, unary minus, ^ (right assoc., tighter than unary
    minus); functions sin cos exp abs sqrt min max; x y z pi X<k>."""
    toks, pos = [], 0
    while True:
        m = _TOK.match(text, pos)
        if m is None:
            rest = text[pos:].lstrip()
            if not rest:
                break
            at = len(text) - len(rest)
            raise E.ExprError(f"unexpected character {text[at]!r}", pos=at)
        toks.append((m.lastgroup, m.group(m.lastgroup), m.start(m.lastgroup)))
        pos = m.end()
    toks.append(("end", "", len(text)))
    i = [0]

    def peek():
        return toks[i[0]]

    def take():
        i[0] += 1
        return toks[i[0] - 1]

    def expect(v):
        k, val, p = peek()
        if val != v:
            raise E.ExprError(f"expected {v!r}, found {val or 'end of input'!r}", pos=p)
        take()

    def ternary():
        c = binary(0)
        if peek()[1] == "?":
            take()
            a = ternary()
            expect(":")
            return Ternary(c, a, ternary())
        return c

    levels = (_CMP, ("+", "-"), ("*", "/"))

    def binary(lv):
        if lv == len(levels):
            return unary()
        node = binary(lv + 1)
        while peek()[1] in levels[lv]:
            node = Binary(take()[1], node, binary(lv + 1))
        return node

    def unary():
        if peek()[1] == "-":
            take()
            return Unary("-", unary())
        base = atom()
        if peek()[1] == "^":
            take()
            return Binary("^", base, unary())
        return base

    def atom():
        kind, val, p = take()
        if kind == "num":
            return Num(float(val))
        if kind == "ident":
            if peek()[1] == "(":
                if val not in ARITY:
                    raise E.ExprError(f"unknown function {val!r}", pos=p)
                take()
                args = [ternary()]
                while peek()[1] == ",":
                    take()
                    args.append(ternary())
                expect(")")
                if len(args) != ARITY[val]:
                    raise E.ExprError(f"{val} takes {ARITY[val]} argument(s), got {len(args)}", pos=p)
                return Call(val, tuple(args))
            if val in ("x", "y", "z", "pi"):
                return Var(val)
            m = re.match(r"X(\d+)$", val)
            if m:
                return Rand(int(m.group(1)))
            raise E.ExprError(f"unknown identifier {val!r}", pos=p)
        if val == "(":
            node = ternary()
            expect(")")
            return node
        raise E.ExprError(f"unexpected {val or 'end of input'!r}", pos=p)

    node = ternary()
    if peek()[0] != "end":
        raise E.ExprError(f"unexpected {peek()[1]!r}", pos=peek()[2])
    return node


_PREC = {"?": 1, **{c: 2 for c in _CMP}, "+": 3, "-": 3, "*": 4, "/": 4, "neg": 5, "^": 6}


def print_expr(node, parent: int = 0) -> str:
    """AST -> text with minimal parentheses (the reference's message format,
    iodsl/expr.py print_expr)."""
    k = type(node).__name__
    if k == "Num":
        return repr(node.value)
    if k == "Var":
        return node.name
    if k == "Rand":
        return f"X{node.index}"
    if k == "Call":
        return f"{node.name}({', '.join(print_expr(a, 0) for a in node.args)})"
    if k == "Unary":
        s = "-" + print_expr(node.operand, _PREC["neg"])
        return f"({s})" if parent > _PREC["neg"] else s
    if k == "Ternary":
        s = (f"{print_expr(node.cond, _PREC['?'] + 1)} ? {print_expr(node.then, _PREC['?'])} : "
             f"{print_expr(node.otherwise, _PREC['?'])}")
        return f"({s})" if parent > _PREC["?"] else s
    if k == "Binary":
        p = _PREC[node.op]
        lp, rp = (p + 1, p) if node.op == "^" else (p, p + 1)
        s = f"{print_expr(node.left, lp)} {node.op} {print_expr(node.right, rp)}"
        return f"({s})" if parent > p else s
    raise TypeError(f"not an initial-data expression node: {node!r}")


# --- bytecode (op codes of fvb_aux.cu InitOp) --------------------------------

OP = {n: i for i, n in enumerate(
    ["const", "x", "y", "z", "rand", "neg", "add", "sub", "mul", "div", "pow", "lt", "le", "gt", "ge", "eq", "ne",
     "sel", "sin", "cos", "exp", "abs", "sqrt", "min", "max", "sqr", "recip"])}
_BIN = {"+": "add", "-": "sub", "*": "mul", "/": "div", "<": "lt", "<=": "le", ">": "gt", ">=": "ge",
        "==": "eq", "!=": "ne"}


class _Compiler:
    def __init__(self, dim: int):
        self.dim = dim
        self.code: list[int] = []
        self.consts: list[float] = []
        self.nrand = 0

    def const(self, v: float):
        v = float(v)
        for j, c in enumerate(self.consts):
            if c == v and math.copysign(1.0, c) == math.copysign(1.0, v):
                return j
        self.consts.append(v)
        return len(self.consts) - 1

    def emit(self, op: str, arg: int = 0):
        self.code.append(OP[op] | (arg << 8))

    def node(self, n):
        """Emit n; returns (stack depth needed, depends on the coordinates)."""
        k = type(n).__name__
        if k == "Num":
            self.emit("const", self.const(n.value))
            return 1, False
        if k == "Var":
            if n.name == "pi":
                self.emit("const", self.const(np.pi))
                return 1, False
            axis = "xyz".index(n.name)
            if axis >= self.dim:
                raise E.ExprError(f"coordinate {n.name!r} is not available here")
            self.emit(n.name)
            return 1, True
        if k == "Rand":
            self.nrand = max(self.nrand, int(n.index) + 1)
            self.emit("rand", int(n.index))
            return 1, False
        if k == "Unary":
            d, arr = self.node(n.operand)
            self.emit("neg")
            return d, arr
        if k == "Call":
            if len(n.args) == 1:
                d, arr = self.node(n.args[0])
                self.emit(n.name)
                return d, arr
            d0, a0 = self.node(n.args[0])
            d1, a1 = self.node(n.args[1])
            self.emit(n.name)
            return max(d0, 1 + d1), a0 or a1
        if k == "Ternary":
            d0, a0 = self.node(n.cond)
            d1, a1 = self.node(n.then)
            d2, a2 = self.node(n.otherwise)
            self.emit("sel")
            return max(d0, 1 + d1, 2 + d2), a0 or a1 or a2
        if k == "Binary":
            if n.op == "^":
                d0, a0 = self.node(n.left)
                r = n.right
                # numpy's array fast paths of np.power with a scalar exponent
                if a0 and type(r).__name__ == "Num" and float(r.value) in (2.0, 0.5, -1.0):
                    self.emit({2.0: "sqr", 0.5: "sqrt", -1.0: "recip"}[float(r.value)])
                    return d0, True
                d1, a1 = self.node(r)
                self.emit("pow")
                return max(d0, 1 + d1), a0 or a1
            d0, a0 = self.node(n.left)
            d1, a1 = self.node(n.right)
            self.emit(_BIN[n.op])
            return max(d0, 1 + d1), a0 or a1
        raise TypeError(f"not an initial-data expression node: {n!r}")


def _eq_code(model) -> int:
    return {"euler": 0, "burgers": 1, "advection": 2}[str(getattr(model, "kind", "euler"))]


class DeviceInit:
    """``evaluate_init`` replacement evaluated on the GPU (see module doc).

    ``DeviceInit(exprs, model, primitive=True)`` with ``exprs`` the
    per-component ASTs (``rc.initial_exprs`` of the reference's parsed
    config) or strings, ``model`` the EquationModel, ``primitive`` as in
    ``eval_init``."""

    def __init__(self, exprs, model, primitive: bool = True):
        self.exprs = [parse_expr(e) if isinstance(e, str) else e for e in exprs]
        self.model = model
        self.primitive = bool(primitive)
        self._prog = {}

    # -- compile once per dimension -----------------------------------------
    def _program(self, dim: int):
        prog = self._prog.get(dim)
        if prog is None:
            import torch

            comp = _Compiler(dim)
            offs, depth = [0], 1
            for ex in self.exprs:
                d, _ = comp.node(ex)
                depth = max(depth, d)
                offs.append(len(comp.code))
            code = torch.tensor(comp.code or [0], dtype=torch.int32, device="cuda")
            consts = torch.tensor(comp.consts or [0.0], dtype=torch.float64, device="cuda")
            prog = self._prog[dim] = (code, consts, (N.C.c_int32 * len(offs))(*offs), depth, comp.nrand)
        return prog

    def _scheme(self, grid):
        s = N.Scheme()
        s.dim = grid.dim
        s.ncomp = self.model.ncomp
        s.eq = _eq_code(self.model)
        s.ghost = grid.ghost_width
        s.rk_order = 1
        s.gamma = float(getattr(self.model, "gamma", 1.4))
        for k in range(3):
            s.cells[k] = grid.cells[k] if k < grid.dim else 1
            s.deltas[k] = grid.deltas[k] if k < grid.dim else 1.0
        return s

    def evaluate_batch(self, grid, vectors, out):
        """Evaluate samples ``vectors`` (sequence of random vectors) into the
        device tensor ``out`` (len(vectors), ncomp, *padded).  Returns one
        exception (or None) per sample, in the reference's check order."""
        import torch

        from .solver import make_layout

        N._require_cuda()
        ncomp = self.model.ncomp
        if len(self.exprs) != ncomp:
            err = E.ExprError(f"need {ncomp} component expressions, got {len(self.exprs)}")
            return [err] * len(vectors)
        code, consts, offs, depth, nrand = self._program(grid.dim)
        errs = [None] * len(vectors)
        for i, v in enumerate(vectors):
            if nrand > len(v):
                errs[i] = E.ExprError(f"random symbol X{nrand - 1} exceeds the stochastic dimension")
        width = max(1, nrand)
        vec = np.zeros((len(vectors), width))
        for i, v in enumerate(vectors):
            vv = np.asarray(v, dtype=np.float64)[:width]
            vec[i, :len(vv)] = vv
        d_vec = torch.from_numpy(vec).to("cuda")
        bad = torch.empty((len(vectors), ncomp + 2), dtype=torch.int64, device="cuda")
        ctx = N.context()
        origin = (N.C.c_double * 3)(*([float(o) for o in grid.origin] + [0.0] * (3 - grid.dim)))
        ctx.check(ctx.lib.fvb_init_eval(ctx.h, N.C.byref(self._scheme(grid)), N.C.byref(make_layout(grid, ncomp)),
                                        origin, N.C.c_void_p(code.data_ptr()), offs,
                                        N.C.c_void_p(consts.data_ptr()), depth, int(self.primitive),
                                        N.C.c_void_p(d_vec.data_ptr()), width, len(vectors),
                                        N.C.c_void_p(out.data_ptr()), N.C.c_void_p(bad.data_ptr())))
        flags = bad.cpu().numpy().view(np.uint64)
        none = np.uint64(0xFFFFFFFFFFFFFFFF)
        shape = tuple(grid.interior_shape)
        for i in range(len(vectors)):
            if errs[i] is not None:
                continue
            f = flags[i]
            for c in range(ncomp):
                if f[c] != none:
                    cell = tuple(int(j) for j in np.unravel_index(int(f[c]), shape))
                    errs[i] = E.ExprError(f"component {c} evaluates to a non-finite value at cell {cell}: "
                                          f"{print_expr(self.exprs[c])}")
                    break
            if errs[i] is None and _eq_code(self.model) == 0 and self.primitive and f[ncomp] != none:
                errs[i] = E.UnphysicalStateError("non-positive density or pressure in primitive state")
            if errs[i] is None and f[ncomp + 1] != none:
                errs[i] = E.UnphysicalStateError("initial data is unphysical")
        return errs

    def __call__(self, grid, random_vector=()):
        """eval_init(exprs, model, grid, random_vector, primitive) -> host Field."""
        import torch

        from .solver import DeviceField

        out = torch.empty((1, self.model.ncomp) + tuple(grid.padded[::-1]), dtype=torch.float64, device="cuda")
        err = self.evaluate_batch(grid, [tuple(random_vector)], out)[0]
        if err is not None:
            raise err
        return DeviceField(grid, self.model.ncomp, out[0]).to_host()


__all__ = ["DeviceInit", "parse_expr", "print_expr", "Num", "Var", "Rand", "Unary", "Binary", "Ternary", "Call",
           "Field"]
