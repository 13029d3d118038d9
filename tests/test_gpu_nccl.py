"""Process-per-GPU paths over NCCL (needs >= 2 visible GPUs; skipped
otherwise -- this pool's boxes have one).  Each rank owns its own device:

* run_parallel over NCCL (DecomposedRun: march-axis halos in place and
  overlapped with the inner box; x halos packed), stitched on rank 0 and
  bitwise equal to the serial oracle;
* run_mc sharded over the ranks with the NCCL all-gather merge, equal to the
  single-process estimate up to the merge association (<= 1e-14);
* bench.py --gpus 2 for the sharded (mc) and decomposed (kh3d) workloads:
  one JSON line with n_gpus == 2.
"""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs (one process per GPU over NCCL)")]

ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, lay, n_steps, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_1912_07645_b200 as P
    from oracle import fv_oracle as O
    from paper_1912_07645_b200.parallel import run_parallel
    from tests.helpers import oracle_scheme, product_objects

    golden = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
    arrays = np.load(ROOT / "tests" / "golden" / "golden.npz")
    case = next(r for r in golden["runs"] if r["name"] == name)
    grid, cfg = product_objects(case["scheme"])
    data = np.array(arrays[name + "__init"])
    res, recs = run_parallel(P.Field(grid, data.shape[0], data), cfg, lay, n_steps=n_steps, arith="exact")
    if rank == 0:
        ref, log = O.simulate_fixed(data, oracle_scheme(case["scheme"]), n_steps)
        sc = oracle_scheme(case["scheme"])
        out["ok"] = (O.sha16(res.interior) == O.sha16(O.interior(ref, sc))
                     and [r.dt for r in recs[0]] == [d for (_, _, d) in log] and len(recs) == world)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,lay,n_steps", [("kh2d64_weno2_50", (1, 2), 4), ("kh2d64_weno2_50", (2, 1), 4),
                                              ("kh3d16_weno2_5", (1, 1, 2), 2)])
def test_run_parallel_nccl(name, lay, n_steps):
    world = int(np.prod(lay))
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _port(), name, lay, n_steps, out), nprocs=world, join=True)
    assert out.get("ok")


def _mc_worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import kelvin_helmholtz

    grid = P.GridSpec(2, (128, 128), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=0.01)
    plan = uq.SamplePlan("mc", 8, 42, 4)
    m, = uq.run_mc(plan, grid, cfg, kelvin_helmholtz, [uq.FieldMoments(grid, 4)], arith="exact")
    if rank == 0:
        out["mean"], out["m2"], out["count"] = m.acc.mean, m.acc.m2, m.acc.count
    dist.destroy_process_group()


def test_run_mc_sharded_nccl():
    out = mp.Manager().dict()
    mp.spawn(_mc_worker, args=(2, _port(), out), nprocs=2, join=True)
    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200 import uq
    from paper_1912_07645_b200.initial import kelvin_helmholtz
    from tests.helpers import rel_l1

    grid = P.GridSpec(2, (128, 128), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
    cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC,
                         P.Reconstruction(P.ReconstructionKind.WENO2), rk_order=3, cfl=0.475, t_end=0.01)
    m1, = uq.run_mc(uq.SamplePlan("mc", 8, 42, 4), grid, cfg, kelvin_helmholtz, [uq.FieldMoments(grid, 4)],
                    arith="exact")
    assert out["count"] == 8
    assert rel_l1(out["mean"], m1.acc.mean) <= 1e-14
    assert rel_l1(out["m2"], m1.acc.m2) <= 1e-12


@pytest.mark.parametrize("config,extra", [("mc", ["--mc-samples", "64", "--mc-steps", "4", "--cells", "128"]),
                                          ("kh3d", ["--cells", "64"])])
def test_bench_two_gpus(config, extra):
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", config, "--steps", "2",
           "--warmup", "3"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
