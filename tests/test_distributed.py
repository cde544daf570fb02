"""Multi-rank logic of the node-sharded integrals.

* CPU (gloo, world size 2): the chunk protocol with real integrand values -- every rank sums
  the ATM integrand over the nodes of its own chunks (CPU oracle, the checker), writes them into
  its slots of the chunk vector, one all-reduce(sum) assembles it, and the fixed-order total is
  bit-identical to the one-process run.
* GPU (gloo, world size 2, both ranks on the box's one GPU): the real ShardedIntegral -- each
  process runs the tile kernel on its chunk range, the chunk vector is all-reduced through a
  host copy, and the result matches the one-process C-ABI value bit for bit.  The two processes'
  kernels never wait on each other (the exchange is on the host), so sharing one GPU is safe.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_11989_b200.distributed import MAX_CHUNKS, ChunkLayout, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(worker, world, *args, timeout=300):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    # collect results, failing fast when a worker dies (its peer would otherwise wait in the
    # rendezvous or a collective until the timeout)
    import queue
    import time
    res, deadline = [], time.monotonic() + timeout
    while len(res) < len(procs):
        try:
            res.append(q.get(timeout=2.0))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or time.monotonic() > deadline:
                for p in procs:
                    if p.is_alive():
                        p.kill()
                raise RuntimeError(f"distributed worker failed (exit codes {dead})" if dead else "timeout")
    for p in procs:
        p.join(timeout=60)
    return sorted(res)


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# grid of the CPU protocol test: fcc ATM, 2 radial x 3^2 angular nodes per cell
_N_U, _N_V, _Q = 2, 3, 3


def _oracle_chunk_sums(rank, world):
    """This rank's slots of the chunk vector: ATM integrand sums over the oracle's nodes of each
    owned chunk (nodes play the role of tiles here)."""
    from oracle import oracle as O
    from paper_2504_11989_b200 import named_lattice
    fcc = named_lattice("fcc")
    n = O.grid_nodes(3, _N_U, _N_V)
    lay = ChunkLayout(n)
    vec = np.zeros(lay.n_chunks * 2)
    c_lo, c_hi = lay.chunks_of(rank, world)
    for c in range(c_lo, c_hi):
        lo, hi = c * lay.chunk_tiles, min((c + 1) * lay.chunk_tiles, n)
        vec[2 * c:2 * c + 2] = O.atm_grid(fcc.a, _N_U, _N_V, _Q, lo, hi)
    return vec


def _cpu_worker(rank, world, port, q):
    _init(rank, world, port)
    t = torch.tensor(_oracle_chunk_sums(rank, world), dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    tot = [math.fsum(t[j::2].tolist()) for j in range(2)]
    # max-over-ranks timing reduction used by bench.py
    tm = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    q.put((rank, t.numpy().tobytes(), tot, float(tm[0])))
    dist.destroy_process_group()


def test_chunk_allreduce_with_oracle_partials_is_exact():
    world = 2
    res = _run(_cpu_worker, world)
    single = _oracle_chunk_sums(0, 1)
    for _, vec, tot, tm in res:
        assert vec == single.tobytes()       # assembled chunk vector: bit-identical to W = 1
        assert tot == [math.fsum(single[j::2]) for j in range(2)]
        assert tm == float(world)
    from oracle import oracle as O
    from paper_2504_11989_b200 import named_lattice
    full = O.atm_grid(named_lattice("fcc").a, _N_U, _N_V, _Q)
    assert np.allclose(res[0][2], full, rtol=1e-14, atol=0)


def test_chunk_layout_matches_the_library():
    """ChunkLayout (Python) and lz_chunk_layout (C, used by the one-call host entry point) agree;
    ranks own whole chunks that cover the tiles exactly."""
    import ctypes as C

    from paper_2504_11989_b200 import _native as N
    for n in (1, 5, 95, 96, 97, 192, 1000, 98304, 98305, 1000003):
        lay = ChunkLayout(n)
        ct, nc = C.c_int64(0), C.c_int64(0)
        assert N.lib().lz_chunk_layout(n, C.byref(ct), C.byref(nc)) == 0
        assert (lay.chunk_tiles, lay.n_chunks) == (ct.value, nc.value)
        assert lay.n_chunks <= MAX_CHUNKS and (lay.n_chunks - 1) * lay.chunk_tiles < n
        for world in (1, 2, 3, 4, 8):
            tiles = [lay.tiles_of(r, world) for r in range(world)]
            assert tiles[0][0] == 0 and tiles[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(tiles, tiles[1:]))
    assert ChunkLayout(98304).chunk_tiles == 1024   # C3: 96 chunks of 1,024 tiles
    assert N.lib().lz_reduce_chunks(None, 10, 2, 1, 0, 11, None, None) == N.LZ_EINVAL


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 98304, 1000003):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert all(hi >= lo for lo, hi in ranges)


def _gpu_worker(rank, world, port, q, n_u, n_v):
    _init(rank, world, port)
    torch.cuda.set_device(0)
    from paper_2504_11989_b200 import named_lattice
    from paper_2504_11989_b200.distributed import ShardedIntegral
    from paper_2504_11989_b200.quadrature import atm_plan
    s = ShardedIntegral(atm_plan(named_lattice("fcc")), n_u, n_v, 3)
    out = s.run().cpu().numpy()
    q.put((rank, s.world, s.tile_lo, s.tile_hi, out.tobytes()))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("n_u,n_v", [(16, 8), (32, 16)])
def test_sharded_integral_two_processes(n_u, n_v):
    from paper_2504_11989_b200 import named_lattice
    from paper_2504_11989_b200.manybody import ATMGrid, atm_integrals
    res = _run(_gpu_worker, 2, n_u, n_v, timeout=600)
    ref = atm_integrals(named_lattice("fcc"), ATMGrid(n_u, n_v, 3))
    assert [r[1] for r in res] == [2, 2]
    assert res[0][3] == res[1][2] and res[0][2] == 0   # contiguous whole-chunk shards
    for _, _, _, _, buf in res:
        out = np.frombuffer(buf, dtype=np.float64)
        assert out[0] * 8 == ref.zeta333 and out[1] * 8 == ref.dot_term
