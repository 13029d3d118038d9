"""Debug: fused peer halo stores on one GPU (2 subdomains, KH2D 64^2 periodic)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1912_07645_b200 as P  # noqa: E402
from paper_1912_07645_b200 import _native as N  # noqa: E402
from paper_1912_07645_b200.parallel import RankTopology, decompose, scatter_field  # noqa: E402
from paper_1912_07645_b200.solver import DeviceField, DeviceRun  # noqa: E402
from tests.helpers import product_objects  # noqa: E402

golden = json.loads((ROOT / "tests/golden/golden.json").read_text())
arrays = np.load(ROOT / "tests/golden/golden.npz")
name = sys.argv[1] if len(sys.argv) > 1 else "kh2d64_weno2_50"
case = next(r for r in golden["runs"] if r["name"] == name)
grid, cfg = product_objects(case["scheme"])
init = P.Field(grid, 4 if grid.dim == 2 else 5, np.array(arrays[name + "__init"]))
march = grid.dim - 1
topo = RankTopology(tuple(2 if k == march else 1 for k in range(grid.dim)))
parts = decompose(grid, topo)
locs = scatter_field(init, parts)
g = grid.ghost_width
stream = torch.cuda.current_stream()
ctxs, bufs = [], []
for r in range(2):
    ctx = N.Context(0, stream)
    b0 = DeviceField.from_host(locs[r]).data.unsqueeze(0).contiguous()
    b = [b0, torch.zeros_like(b0), torch.zeros_like(b0)]
    ctx.check(ctx.lib.fvb_run_set_external_reduce(ctx.h, 1))
    DeviceRun(parts[r].grid, cfg, b, 1, N.MODE_FIXED, 4, "exact", halo_axes=(march,), ctx=ctx, log=False)
    ctxs.append(ctx)
    bufs.append(b)
keep = []
for r in range(2):
    q = 1 - r
    arr = (N.C.c_void_p * 3)(*[N.C.c_void_p(x.data_ptr()) for x in bufs[q]])
    keep.append(arr)
    ctxs[r].check(ctxs[r].lib.fvb_run_set_peers(ctxs[r].h, arr, arr))
n = parts[0].grid.cells[march]
for r in range(2):  # initial ghosts
    q = 1 - r
    u = bufs[r][0][0]
    u[:, 0:g] = bufs[q][0][0][:, n:n + g]
    u[:, n + g:n + 2 * g] = bufs[q][0][0][:, g:2 * g]
red = [torch.zeros(grid.dim + 2, dtype=torch.float64, device="cuda") for _ in range(2)]
for r in range(2):
    ctxs[r].check(ctxs[r].lib.fvb_run_export(ctxs[r].h, N.C.c_void_p(red[r].data_ptr())))
m = torch.stack(red).max(0).values
for r in range(2):
    red[r].copy_(m)
    ctxs[r].check(ctxs[r].lib.fvb_run_finalize(ctxs[r].h, N.C.c_void_p(red[r].data_ptr()), 0))
for st in range(3):
    for r in range(2):
        ctxs[r].check(ctxs[r].lib.fvb_run_stage(ctxs[r].h, st))
    torch.cuda.synchronize()
    k = (1, 2, 0)[st]
    for r in range(2):
        q = 1 - r
        u = bufs[r][k][0]
        lo_ok = torch.equal(u[:, 0:g], bufs[q][k][0][:, n:n + g])
        hi_ok = torch.equal(u[:, n + g:n + 2 * g], bufs[q][k][0][:, g:2 * g])
        diff_lo = (u[:, 0:g] - bufs[q][k][0][:, n:n + g]).abs().max().item()
        diff_hi = (u[:, n + g:n + 2 * g] - bufs[q][k][0][:, g:2 * g]).abs().max().item()
        print(f"stage {st} out buf {k} rank {r}: low ghosts ok {lo_ok} ({diff_lo:.3e}) high ghosts ok {hi_ok} ({diff_hi:.3e})")

# --- determinism / serialisation experiment
import os  # noqa: E402
from tests.test_gpu_fused_halo import _fused_run  # noqa: E402
from paper_1912_07645_b200.parallel import run_parallel  # noqa: E402
import paper_1912_07645_b200._native as NN  # noqa: E402

orig_ctx_check = NN.Context.check
lay = tuple(2 if k == march else 1 for k in range(grid.dim))
ref, _ = run_parallel(init, cfg, lay, n_steps=4, arith="exact")
for trial in range(3):
    out, _ = _fused_run(P, init, cfg, 2, 4, "exact")
    d = np.abs(out.interior - ref.interior)
    print(f"trial {trial}: max diff {d.max():.3e} bad {int((d > 0).sum())}")
# serialise: synchronize after every library call
def sync_check(self, rc):
    torch.cuda.synchronize()
    return orig_ctx_check(self, rc)
NN.Context.check = sync_check
for trial in range(2):
    out, _ = _fused_run(P, init, cfg, 2, 4, "exact")
    d = np.abs(out.interior - ref.interior)
    print(f"synced trial {trial}: max diff {d.max():.3e} bad {int((d > 0).sum())}")
NN.Context.check = orig_ctx_check
