"""Where does the time of one run_simulation(host Field) call go?"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1912_07645_b200 as P
from paper_1912_07645_b200 import _native as N
from paper_1912_07645_b200.initial import kelvin_helmholtz
from paper_1912_07645_b200.solver import DeviceField, DeviceRun, pinned_field

n = 1024
grid = P.GridSpec(2, (n, n), (0.0, 0.0), (1.0, 1.0), ghost_width=2)
cfg = P.SchemeConfig(P.EquationModel("euler", 2), P.FluxKind.HLLC, P.Reconstruction(P.ReconstructionKind.WENO2),
                     rk_order=3, cfl=0.475, t_end=2.0)
init = pinned_field(kelvin_helmholtz(grid, [0.82, 0.19, 0.87, 0.39]))
P.run_simulation(init, cfg, max_steps=2, arith="fast")
torch.cuda.synchronize()


def t(f, label, reps=5):
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - a) / reps * 1e3:8.3f} ms")
    return r


t(lambda: P.run_simulation(init, cfg, max_steps=10, arith="fast"), "run_simulation(max_steps=10)")
dev = t(lambda: DeviceField.from_host(init), "from_host (pinned)")
t(lambda: DeviceField.from_host(P.Field(grid, 4, np.array(init.data))), "from_host (pageable)")
t(lambda: dev.to_host(), "to_host")
t(lambda: dev.data.cpu(), "data.cpu()")
bufs = [dev.data, torch.empty_like(dev.data), torch.empty_like(dev.data)]


def run10():
    r = DeviceRun(grid, cfg, bufs, 1, N.MODE_T_END, 10, "fast")
    r.steps(10)
    infos, done = r.poll()
    r.read_log(infos, 0.0)
    r.end()


t(run10, "DeviceRun begin+10 steps+poll+log+end")


def begin_end():
    r = DeviceRun(grid, cfg, bufs, 1, N.MODE_T_END, 10, "fast")
    r.end()


t(begin_end, "DeviceRun begin+end")

import ctypes
libc = ctypes.CDLL("libc.so.6")
M_TRIM_THRESHOLD, M_MMAP_THRESHOLD = -1, -3
libc.mallopt(M_MMAP_THRESHOLD, 1 << 30)
libc.mallopt(M_TRIM_THRESHOLD, 1 << 31)
t(lambda: dev.data.cpu(), "data.cpu() after mallopt")
t(lambda: dev.to_host(), "to_host after mallopt")
stage = torch.empty(tuple(dev.data.shape), dtype=torch.float64, pin_memory=True)


def staged():
    stage.copy_(dev.data)
    return stage.numpy().copy()


t(staged, "pinned staging + numpy copy (mallopt)")
t(lambda: torch.empty(tuple(dev.data.shape), dtype=torch.float64, pin_memory=True).copy_(dev.data), "fresh pinned each call")
t(lambda: P.run_simulation(init, cfg, max_steps=10, arith="fast"), "run_simulation(max_steps=10) mallopt")
