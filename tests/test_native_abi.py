"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU
and exports every symbol include/fvb200.h declares; the ctypes structs match
the header layout; the product refuses to compute without CUDA (no CPU
fallback)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "fvb200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(fvb_\w+)\(", text, re.M)))


def test_header_declares_what_ctypes_binds():
    from paper_1912_07645_b200 import _native as N

    assert set(_declared()) == set(N.EXPORTS)


def test_library_exports_every_symbol():
    from paper_1912_07645_b200 import _native as N

    if not N.LIB_PATH.exists():  # fresh checkout: build it (nvcc cross-compiles, no GPU needed)
        from paper_1912_07645_b200 import build as B

        B.build()
    lib = N.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.fvb_version() == 1


def test_struct_layout_matches_header():
    from paper_1912_07645_b200 import _native as N

    # fvb_scheme: 12 int32 (48 B) + 3 int64 + 3 double + 4 double + 3 double
    assert ctypes.sizeof(N.Scheme) == 48 + 24 + 24 + 32 + 24
    assert ctypes.sizeof(N.Layout) == 40
    assert ctypes.sizeof(N.RunInfo) == 40


def test_halo_count_host_only():
    """fvb_halo_count is pure host arithmetic: g * ncomp * prod(padded other axes)."""
    from paper_1912_07645_b200 import _native as N

    lib = N.load_library()
    s = N.Scheme()
    s.dim, s.ncomp, s.ghost = 3, 5, 2
    for k, n in enumerate((16, 12, 8)):
        s.cells[k] = n
    assert lib.fvb_halo_count(ctypes.byref(s), 0) == 2 * 5 * (12 + 4) * (8 + 4)
    assert lib.fvb_halo_count(ctypes.byref(s), 2) == 2 * 5 * (16 + 4) * (12 + 4)


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200._native import NativeUnavailable

    grid = P.GridSpec(1, (8,), (0.0,), (1.0,), ghost_width=1)
    cfg = P.SchemeConfig(P.EquationModel("burgers", 1), P.FluxKind.RUSANOV, P.Reconstruction(), 1)
    with pytest.raises(NativeUnavailable):
        P.run_simulation(P.field_from_interior(grid, np.ones((1, 8))), cfg)
