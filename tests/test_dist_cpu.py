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
