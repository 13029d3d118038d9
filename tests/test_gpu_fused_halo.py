"""The fused halo exchange (fvb_run_set_peers): with the march axis split,
every stage kernel also stores its first / last g march rows into the
neighbours' ghost rows, so a decomposed step needs no exchange step at all.
Multi-GPU runs map the neighbours' buffers over NVLink (symmetric memory,
parallel.DecomposedRun(peer_halos=...)); here the subdomains live on ONE GPU
in one process, each with its own context, their stages issued one after the
other on one stream (no kernel waits on another), the peers being plain
device pointers -- the same kernel code path.  Bitwise equal to the serial
oracle (exact) / to the undecomposed run (fast)."""
import numpy as np
import pytest

from oracle import fv_oracle as O
from tests.helpers import oracle_scheme, product_objects

pytestmark = pytest.mark.gpu


def _fused_run(P, init, cfg, nrank, n_steps, arith):
    """All subdomains' contexts on ONE explicit stream (the legacy default
    stream would give each context its own stream: no ordering between
    them)."""
    import torch

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        out = _fused_run_on_stream(P, init, cfg, nrank, n_steps, arith)
    torch.cuda.current_stream().wait_stream(stream)
    return out


def _fused_run_on_stream(P, init, cfg, nrank, n_steps, arith):
    import torch

    from paper_1912_07645_b200 import _native as N
    from paper_1912_07645_b200.parallel import RankTopology, decompose, scatter_field, stitch_fields
    from paper_1912_07645_b200.solver import DeviceField, DeviceRun, _v

    grid = init.grid
    march = grid.dim - 1
    lay = tuple(nrank if k == march else 1 for k in range(grid.dim))
    topo = RankTopology(lay)
    parts = decompose(grid, topo)
    locs = scatter_field(init, parts)
    periodic = _v(cfg.bc[march]) == "periodic"
    g = grid.ghost_width
    stream = torch.cuda.current_stream()
    runs, ctxs, bufs = [], [], []
    for r in range(nrank):
        ctx = N.Context(torch.cuda.current_device(), stream)  # one plan per subdomain
        b0 = DeviceField.from_host(locs[r]).data.unsqueeze(0).contiguous()
        b = [b0, torch.empty_like(b0), torch.empty_like(b0)]
        for x in b[1:]:
            x.zero_()
        ctx.check(ctx.lib.fvb_run_set_external_reduce(ctx.h, 1))
        runs.append(DeviceRun(parts[r].grid, cfg, b, 1, N.MODE_FIXED, n_steps, arith, halo_axes=(march,), ctx=ctx,
                              log=True))
        ctxs.append(ctx)
        bufs.append(b)
    n = parts[0].grid.cells[march]
    ax = 1  # numpy axis of the march axis in (ncomp, *padded) is 1 (slowest)

    def nb(r, side):
        return topo.neighbor(r, march, side, periodic)

    keep = []
    for r in range(nrank):
        lo, hi = nb(r, 0), nb(r, 1)
        arr = lambda q: None if q is None else (N.C.c_void_p * 3)(*[N.C.c_void_p(x.data_ptr()) for x in bufs[q]])  # noqa
        keep.append((arr(lo), arr(hi)))
        ctxs[r].check(ctxs[r].lib.fvb_run_set_peers(ctxs[r].h, keep[-1][0], keep[-1][1]))

    def slab(t, lo, hi):
        s = [slice(None)] * t.dim()
        s[ax] = slice(lo, hi)
        return tuple(s)

    def fill_ghosts(k):
        # the first stage's input: neighbours' layers (a device copy), outflow at world edges
        for r in range(nrank):
            u = bufs[r][k][0]
            lo, hi = nb(r, 0), nb(r, 1)
            if lo is not None:
                u[slab(u, 0, g)] = bufs[lo][k][0][slab(u, n, n + g)]
            else:
                u[slab(u, 0, g)] = u[slab(u, g, g + 1)].expand_as(u[slab(u, 0, g)])
            if hi is not None:
                u[slab(u, n + g, n + 2 * g)] = bufs[hi][k][0][slab(u, g, 2 * g)]
            else:
                u[slab(u, n + g, n + 2 * g)] = u[slab(u, n + g - 1, n + g)].expand_as(u[slab(u, n + g, n + 2 * g)])

    def outflow_edges(k):
        for r in range(nrank):
            u = bufs[r][k][0]
            if nb(r, 0) is None:
                u[slab(u, 0, g)] = u[slab(u, g, g + 1)].expand_as(u[slab(u, 0, g)])
            if nb(r, 1) is None:
                u[slab(u, n + g, n + 2 * g)] = u[slab(u, n + g - 1, n + g)].expand_as(u[slab(u, n + g, n + 2 * g)])

    red = [torch.zeros(grid.dim + 2, dtype=torch.float64, device="cuda") for _ in range(nrank)]

    def reduce_finalize(post):
        for r in range(nrank):
            ctxs[r].check(ctxs[r].lib.fvb_run_export(ctxs[r].h, N.C.c_void_p(red[r].data_ptr())))
        m = torch.stack(red).max(dim=0).values
        for r in range(nrank):
            red[r].copy_(m)
            ctxs[r].check(ctxs[r].lib.fvb_run_finalize(ctxs[r].h, N.C.c_void_p(red[r].data_ptr()), post))

    fill_ghosts(0)
    reduce_finalize(0)
    nst = cfg.rk_order
    for step in range(n_steps):
        for st in range(nst):
            k = step % 2 if nst == 1 else st
            if step or st:
                outflow_edges(k)
            for r in range(nrank):
                ctxs[r].check(ctxs[r].lib.fvb_run_stage(ctxs[r].h, st))
        reduce_finalize(1)
    finals = []
    for r in range(nrank):
        infos, _ = runs[r].poll()
        runs[r].read_log(infos, 0.0)
        info = runs[r].end()[0]
        assert info.err == 0, info.err
        finals.append(DeviceField(parts[r].grid, init.ncomp, bufs[r][0 if nst > 1 else n_steps % 2][0]).to_host())
    return stitch_fields(grid, parts, finals), [rec.dt for rec in runs[0].records[0]]


@pytest.mark.parametrize("name,nrank", [("kh2d64_weno2_50", 2), ("kh2d64_weno2_50", 4),
                                        ("euler2d_hllc_weno3_outflow", 2), ("kh3d16_weno2_5", 2),
                                        ("euler3d_hllc_none_outflow", 2)])
def test_fused_halo_exact_bitwise(golden, golden_arrays, name, nrank):
    import paper_1912_07645_b200 as P

    case = next(r for r in golden["runs"] if r["name"] == name)
    grid, cfg = product_objects(case["scheme"])
    data = np.array(golden_arrays[name + "__init"])
    init = P.Field(grid, data.shape[0], data)
    if grid.cells[grid.dim - 1] % nrank:
        pytest.skip("not divisible")
    out, dts = _fused_run(P, init, cfg, nrank, 4, "exact")
    ref, log = O.simulate_fixed(init.data, oracle_scheme(case["scheme"]), 4)
    assert dts == [d for (_, _, d) in log]
    assert O.sha16(out.interior) == O.sha16(O.interior(ref, oracle_scheme(case["scheme"]))), (name, nrank)


@pytest.mark.parametrize("name", ["kh2d64_weno2_50", "kh3d16_weno2_5"])
def test_fused_halo_fast_equals_undecomposed(golden, golden_arrays, name):
    """Fast mode (pair kernel in 2D, ring3i in 3D): the fused decomposed run
    equals the undecomposed fast run bitwise."""
    import paper_1912_07645_b200 as P
    from paper_1912_07645_b200.parallel import run_parallel

    case = next(r for r in golden["runs"] if r["name"] == name)
    grid, cfg = product_objects(case["scheme"])
    data = np.array(golden_arrays[name + "__init"])
    init = P.Field(grid, data.shape[0], data)
    whole, _ = run_parallel(init, cfg, (1,) * grid.dim, n_steps=4, arith="fast")
    out, _ = _fused_run(P, init, cfg, 2, 4, "fast")
    assert O.sha16(out.interior) == O.sha16(whole.interior)
