"""Process-per-rank decomposition (run_parallel_nccl) exercised on ONE GPU:
several processes share the device and exchange halos / reduce dt through
gloo on host memory (cpu_comm), so no kernel ever waits on another rank.
The stitched result must be bitwise equal to the serial oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, lay, n_steps, overlap, out):
    import json
    from pathlib import Path

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1912_07645_b200 as P
    from oracle import fv_oracle as O
    from paper_1912_07645_b200.parallel import run_parallel
    from tests.helpers import oracle_scheme, product_objects

    root = Path(__file__).resolve().parent / "golden"
    golden = json.loads((root / "golden.json").read_text())
    arrays = np.load(root / "golden.npz")
    case = next(r for r in golden["runs"] if r["name"] == name)
    grid, cfg = product_objects(case["scheme"])
    data = np.array(arrays[name + "__init"])
    init = P.Field(grid, data.shape[0], data)
    res, recs = run_parallel(init, cfg, lay, n_steps=n_steps, overlap=overlap, arith="exact")
    if rank == 0:
        sc = oracle_scheme(case["scheme"])
        if n_steps is None:
            ok = O.sha16(res.interior) == case["final_sha"] and len(recs[0]) == case["steps"]
        else:
            ref, log = O.simulate_fixed(data, sc, n_steps)
            ok = (O.sha16(res.interior) == O.sha16(O.interior(ref, sc))
                  and [r.dt for r in recs[0]] == [d for (_, _, d) in log])
        out["ok"] = ok
        out["recs"] = len(recs)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,lay,n_steps,overlap", [
    ("kh2d64_weno2_50", (2, 1), 4, True),
    ("kh2d64_weno2_50", (1, 2), 4, True),     # march axis split: inner box overlaps the exchange
    ("kh2d64_weno2_50", (1, 2), 4, False),
    ("euler2d_hllc_weno3_outflow", (2, 2), 3, True),
    ("burgers1d_weno2_rk1_periodic", (2,), 7, True),
    ("burgers1d_weno3_rk3_outflow", (2,), None, True),
    ("kh3d16_weno2_5", (1, 1, 2), 2, True),
    ("euler3d_hllc_none_outflow", (1, 2, 2), 3, True)])
def test_run_parallel_process_per_rank(name, lay, n_steps, overlap):
    world = int(np.prod(lay))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _port(), name, lay, n_steps, overlap, out), nprocs=world, join=True)
    assert out.get("ok"), (name, lay)
    assert out["recs"] == world
