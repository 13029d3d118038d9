"""Multi-process host logic on CPU (gloo, world_size 2): contiguous sample
sharding and the rank-ordered all_gather used to merge per-GPU UQ
accumulators (paper_1912_07645_b200/uq.py), and the halo exchange protocol
of the domain decomposition (paper_1912_07645_b200/parallel.py).  The
per-rank statistics are computed with the oracle on CPU (test-side only);
what is under test is the product's collective plumbing and ordering."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_07645_b200.uq import gather_ordered, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_tiles_exactly():
    for n in (1, 7, 8, 1024, 1000):
        for w in (1, 2, 3, 4, 8):
            blocks = [shard_range(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1


def _moments_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import fv_oracle as O

    rng = np.random.default_rng(7)
    fields = rng.standard_normal((10, 3, 5, 6))
    lo, hi = shard_range(len(fields), world, rank)
    local = O.Moments(fields.shape[1:])
    for k in range(lo, hi):
        local.push(fields[k])
    blocks = gather_ordered([torch.from_numpy(local.mean), torch.from_numpy(local.m2)], local.count, dist, None,
                            world)
    tot = O.Moments(fields.shape[1:])
    for cnt, (mean, m2) in blocks:
        part = O.Moments(fields.shape[1:])
        part.count, part.mean, part.m2 = cnt, mean.numpy(), m2.numpy()
        tot.merge(part)
    seq = O.Moments(fields.shape[1:])
    for f in fields:
        seq.push(f)
    out[rank] = (tot.count == seq.count and
                 float(np.abs(tot.mean - seq.mean).max()) <= 1e-15 and
                 float(np.abs(tot.m2 - seq.m2).max()) <= 1e-13)
    dist.destroy_process_group()


def test_rank_ordered_moment_merge_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_moments_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] and out[1]


def _halo_worker(rank, world, port, lay, periodic, out, listy=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import fv_oracle as O
    from paper_1912_07645_b200 import parallel as PP

    g = 2
    cells = (12, 10)
    rng = np.random.default_rng(3)
    inner = rng.standard_normal((3, cells[1], cells[0]))
    sc = O.Scheme(dim=2, cells=cells, deltas=(1 / 12, 1 / 10), eq="burgers", recon="weno2",
                  bcs=tuple("periodic" if p else "outflow" for p in periodic))
    want = O.ghost_fill(O.padded_from_interior(sc, inner), sc)
    topo = PP.RankTopology(lay)
    loc_cells = (cells[0] // lay[0], cells[1] // lay[1])
    cx, cy = topo.coords(rank)
    ox, oy = cx * loc_cells[0], cy * loc_cells[1]
    u = np.zeros((3, loc_cells[1] + 2 * g, loc_cells[0] + 2 * g))
    u[:, g:g + loc_cells[1], g:g + loc_cells[0]] = inner[:, oy:oy + loc_cells[1], ox:ox + loc_cells[0]]

    def sl(axis, lo, hi):  # slab over the padded extent of the other axis
        s = [slice(None), slice(None), slice(None)]
        s[2 - axis] = slice(lo, hi)
        return tuple(s)

    def pack(axis, side):
        n = loc_cells[axis]
        slab = np.ascontiguousarray(u[sl(axis, g, 2 * g) if side == 0 else sl(axis, n, n + g)])
        if listy and axis == 1:  # march axis: one contiguous message per component (parallel._Halos)
            return [torch.from_numpy(np.ascontiguousarray(slab[c])) for c in range(slab.shape[0])]
        return torch.from_numpy(slab)

    def alloc(axis, side):
        b = pack(axis, 0)
        return [torch.empty_like(x) for x in b] if isinstance(b, list) else torch.empty_like(b)

    def unpack(axis, side, buf):
        n = loc_cells[axis]
        val = np.stack([x.numpy() for x in buf]) if isinstance(buf, list) else buf.numpy()
        u[sl(axis, 0, g) if side == 0 else sl(axis, n + g, n + 2 * g)] = val

    PP.halo_exchange_dist(topo, rank, periodic, pack, unpack, alloc, dist)
    ok = True
    for axis in range(2):
        n = loc_cells[axis]
        if topo.ranks_per_axis[axis] == 1:
            continue
        for side in (0, 1):
            if topo.neighbor(rank, axis, side, periodic[axis]) is None:
                continue
            # face ghosts over the transverse interior must equal the serial fill
            gh = slice(0, g) if side == 0 else slice(n + g, n + 2 * g)
            if axis == 0:
                mine = u[:, g:g + loc_cells[1], gh]
                ref = want[:, g + oy:g + oy + loc_cells[1], (ox + gh.start):(ox + gh.stop)]
            else:
                mine = u[:, gh, g:g + loc_cells[0]]
                ref = want[:, (oy + gh.start):(oy + gh.stop), g + ox:g + ox + loc_cells[0]]
            ok &= bool(np.array_equal(mine, ref))
    out[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("lay,periodic,listy", [((2, 1), (True, True), False), ((2, 2), (True, True), False),
                                                ((2, 2), (False, True), False), ((1, 2), (True, False), False),
                                                ((1, 2), (True, True), True), ((2, 2), (True, False), True)])
def test_halo_exchange_dist_gloo(lay, periodic, listy):
    world = lay[0] * lay[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_halo_worker, args=(world, _free_port(), lay, periodic, out, listy), nprocs=world, join=True)
    assert all(out[r] for r in range(world))


class _CountFunctional:
    """A host-side functional of the duck-typed reference protocol
    (fresh/update/merge/name, uq.py:161-273) that run_mc feeds host fields."""

    name = "count_max"

    def __init__(self):
        self.samples = 0
        self.maxima = []

    def fresh(self):
        return _CountFunctional()

    def update(self, field):
        self.samples += 1
        self.maxima.append(float(np.max(field.data)))

    def merge(self, other):
        self.samples += other.samples
        self.maxima += other.maxima


def _merge_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1912_07645_b200 import uq

    proto_h = uq.Histogram([(1, 2), (3, 0)], 0, 0.0, 1.0, bins=4)
    proto_c = _CountFunctional()
    slots = [uq._Slot(proto_h, None, 1), uq._Slot(proto_c, None, 1)]
    rng = np.random.default_rng(11)
    vals = rng.uniform(-0.2, 1.2, size=(9, 2))  # 9 samples, 2 probes each
    lo, hi = shard_range(len(vals), world, rank)
    for k in range(lo, hi):
        slots[0].hist.add_values(vals[k])
        slots[1].host.samples += 1
        slots[1].host.maxima.append(float(vals[k].max()))
    uq._merge_ranks(slots, dist, None, world)
    ref = uq.Histogram([(1, 2), (3, 0)], 0, 0.0, 1.0, bins=4)
    for v in vals:
        ref.add_values(v)
    h, c = slots[0].result(), slots[1].result()
    out[rank] = (bool(np.array_equal(h.counts, ref.counts)) and h.samples == 9 and c.samples == 9
                 and c.maxima == [float(v.max()) for v in vals])
    dist.destroy_process_group()


def test_histogram_and_host_functional_merge_gloo():
    """run_mc's cross-rank merge of a Histogram (counts and samples add) and
    of an arbitrary host functional (gathered, merged in rank order =
    sample order), ADVICE r01."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_merge_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] and out[1]
