"""Multi-rank host logic of the node-sharded integrals on CPU (gloo, world size 2).

The device kernels cannot run here; the test drives the same protocol with a
deterministic stand-in for the per-tile partials: each rank fills only its
contiguous tile range, one all-reduce(sum) assembles the vector, and the
result must be bit-identical to the single-process vector for every world size.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_11989_b200.distributed import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tile_partials(n_tiles, ncomp, lo, hi):
    """Stand-in for tile_kernel: slot t gets a fixed pseudo-random value, others stay zero."""
    rng = np.random.default_rng(1234)
    full = rng.standard_normal(n_tiles * ncomp) * np.exp(rng.uniform(-30, 30, n_tiles * ncomp))
    out = np.zeros_like(full)
    out[lo * ncomp:hi * ncomp] = full[lo * ncomp:hi * ncomp]
    return out, full


def _worker(rank, world, port, n_tiles, ncomp, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n_tiles, rank, world)
    part, full = _tile_partials(n_tiles, ncomp, lo, hi)
    t = torch.tensor(part, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    ok = bool(torch.equal(t, torch.tensor(full)))
    # max-over-ranks timing reduction used by bench.py
    tm = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    q.put((rank, ok, float(tm[0])))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slot_disjoint_allreduce_is_exact(world):
    n_tiles, ncomp = 98304 // 64, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_tiles, ncomp, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert all(tm == float(world) for _, _, tm in res)


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 98304, 1000003):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert all(hi >= lo for lo, hi in ranges)
