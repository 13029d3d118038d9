"""Device initial data, host side: the expression parser/printer against the
reference's (golden fingerprints from iodsl/expr.py), and the compiled
bytecode -- run here by a numpy restatement of the device interpreter
(fvb_aux.cu init_run) -- against the reference's pointwise values."""
import numpy as np
import pytest

from paper_1912_07645_b200 import errors as E
from paper_1912_07645_b200 import initdev as I


def run_bytecode(comp, env):
    """numpy restatement of fvb_aux.cu init_run (same op semantics)."""
    inv = {v: k for k, v in I.OP.items()}
    st = []
    un = {"neg": np.negative, "sin": np.sin, "cos": np.cos, "exp": np.exp, "abs": np.abs, "sqrt": np.sqrt,
          "sqr": lambda a: a * a, "recip": lambda a: 1.0 / a}
    bi = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide, "pow": np.power,
          "min": np.minimum, "max": np.maximum}
    cmp = {"lt": np.less, "le": np.less_equal, "gt": np.greater, "ge": np.greater_equal, "eq": np.equal,
           "ne": np.not_equal}
    for w in comp.code:
        op, arg = inv[w & 0xFF], w >> 8
        if op == "const":
            st.append(comp.consts[arg])
        elif op in ("x", "y", "z"):
            st.append(env[op])
        elif op == "rand":
            st.append(env[f"X{arg}"])
        elif op in un:
            st.append(un[op](st.pop()))
        elif op == "sel":
            b, a, q = st.pop(), st.pop(), st.pop()
            st.append(np.where(np.asarray(q) != 0.0, a, b))
        else:
            b, a = st.pop(), st.pop()
            st.append(bi[op](a, b) if op in bi else cmp[op](a, b).astype(float))
    assert len(st) == 1
    return st[0]


def test_parser_printer_match_reference(golden):
    for case in golden["exprs"]:
        node = I.parse_expr(case["text"])
        assert I.print_expr(node) == case["print"], case["text"]
        assert repr(node).replace("paper_1912_07645_b200.initdev.", "") == case["repr"], case["text"]
        assert I.print_expr(I.parse_expr(case["print"])) == case["print"]  # round trip


def test_bytecode_matches_reference_values(golden):
    xs = np.array([0.1, 0.37, 0.5, 0.81])
    env = {"x": xs, "y": xs[::-1].copy(), "z": xs * 0.5, "X0": 0.3, "X1": 0.7, "X2": 0.1, "X3": 0.9}
    for case in golden["exprs"]:
        comp = I._Compiler(3)
        depth, _ = comp.node(I.parse_expr(case["text"]))
        assert 1 <= depth <= 32
        got = np.broadcast_to(np.asarray(run_bytecode(comp, env), dtype=float), xs.shape)
        ref = np.array(case["values"])
        assert np.array_equal(got, ref, equal_nan=True), (case["text"], got, ref)


def test_initial_programs_of_every_golden_run_compile(golden):
    for case in golden["runs"]:
        comp = I._Compiler(case["scheme"]["dim"])
        for t in case["init_exprs"]:
            comp.node(I.parse_expr(t))
        assert comp.nrand <= 4


def test_parse_errors_and_unavailable_coordinate():
    with pytest.raises(E.ExprError, match="unknown function 'tan'"):
        I.parse_expr("tan(x)")
    with pytest.raises(E.ExprError, match=r"position 4: expected '\)'"):
        I.parse_expr("(1+2")
    with pytest.raises(E.ExprError, match="sin takes 1 argument"):
        I.parse_expr("sin(x, y)")
    with pytest.raises(E.ExprError, match="coordinate 'z' is not available here"):
        I._Compiler(2).node(I.parse_expr("x + z"))
