"""Shared test helpers: build oracle schemes from golden case records."""
import numpy as np

from oracle import fv_oracle as O


def oracle_scheme(d: dict) -> O.Scheme:
    return O.Scheme(
        dim=d["dim"], cells=tuple(d["cells"]), deltas=tuple(d["deltas"]), eq=d["eq"],
        gamma=d["gamma"], adv=tuple(d["adv"]), flux=d["flux"], recon=d["recon"],
        eps=d["eps"], rk=d["rk"], cfl=d["cfl"], t_end=d["t_end"], bcs=tuple(d["bcs"]),
        ghost=d["ghost"],
    )


def rel_l1(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = np.abs(b).sum()
    return float(np.abs(a - b).sum() / den) if den else float(np.abs(a - b).sum())
