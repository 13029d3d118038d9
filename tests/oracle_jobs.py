"""Oracle work units for the benchmark-size parity tests -- TEST
INFRASTRUCTURE ONLY (the checker side).  Each function is a pure numpy
computation (oracle/fv_oracle.py) picklable into a spawned worker process,
so the large oracle references of tests/test_gpu_benchsize.py run
concurrently on the host cores while the GPU does its part."""
from __future__ import annotations

import numpy as np

from oracle import fv_oracle as O


def simulate_checkpoints(u_pad, scheme: dict, checkpoints):
    """O.simulate from u_pad, returning (interior, dts) after each step count
    in ``checkpoints`` (ascending): chained runs restart t at 0, exactly
    like the GPU side (t_end >> the steps' total, so min(dt, t_end - t)
    never binds)."""
    sc = O.Scheme(**scheme)
    out = {}
    cur = np.array(u_pad, dtype=np.float64)
    done = 0
    dts = []
    for n in checkpoints:
        if n > done:
            cur, log = O.simulate(cur, sc, n - done)
            dts += [d for (_, _, d) in log]
            done = n
        out[n] = (np.array(O.interior(cur, sc)), list(dts))
    return out


def sample_final(kind: str, cells, vec, scheme: dict):
    """Final interior of one UQ sample (run_mc's _run_one_sample, uq.py:281-290)."""
    sc = O.Scheme(**scheme)
    u0 = O.kelvin_helmholtz(tuple(cells), vec) if kind == "kh" else O.burgers_sines(tuple(cells), vec)
    final, _ = O.simulate(u0, sc)
    return np.array(O.interior(final, sc))


def structure_sums(w, p: float, H: int):
    return O.structure_sums(np.asarray(w), p, H)
