"""Multi-GPU node sharding of the fused BZ integrals (one process per GPU).

Every fixed Duffy grid is a flat list of 256-node tiles; each tile reduces
deterministically to one partial per component.  The tiles are grouped into at
most ``MAX_CHUNKS`` = 96 fixed chunks that depend only on the grid (C3: 96
chunks of 1,024 tiles).  Rank r of W owns the contiguous chunk range
[r C / W, (r+1) C / W): it runs the tile kernel on its tiles, reduces each of
its chunks in a fixed order (``lz_reduce_chunks``) into its own slots of a
C x ncomp vector, and ONE all-reduce (sum, FP64) over NCCL/NVLink assembles
that vector exactly (every other slot is zero, and adding zeros is exact) --
1.5 KB for C3 instead of the 1.5 MB of tile partials.  The fixed-order
compensated reduction of the chunk vector then gives bit-identical results
for any W.  This replaces the reference's ThreadPoolExecutor over Duffy cells
and its fsum of their values (L/quadrature.py:482-490).
"""
from __future__ import annotations

import warnings
from dataclasses import dataclass

import torch
import torch.distributed as dist

from .lattice import Lattice
from .manybody import ATMGrid, ATMResult
from .quadrature import Plan, atm_plan, product_plan


MAX_CHUNKS = 96  # divisible by 1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48: balanced ranks for those W


def shard_range(n: int, rank: int, world: int):
    """Contiguous index range [lo, hi) of one rank out of ``n`` units."""
    return n * rank // world, n * (rank + 1) // world


@dataclass(frozen=True)
class ChunkLayout:
    """Fixed grouping of ``n_tiles`` tile partials into chunks (a function of the grid only)."""

    n_tiles: int
    max_chunks: int = MAX_CHUNKS

    @property
    def chunk_tiles(self) -> int:
        return max(1, -(-self.n_tiles // self.max_chunks))

    @property
    def n_chunks(self) -> int:
        return -(-self.n_tiles // self.chunk_tiles) if self.n_tiles else 0

    def chunks_of(self, rank: int, world: int):
        """Chunk range [c_lo, c_hi) owned by ``rank``."""
        return shard_range(self.n_chunks, rank, world)

    def tiles_of(self, rank: int, world: int):
        """Tile range [t_lo, t_hi) owned by ``rank`` (whole chunks)."""
        c_lo, c_hi = self.chunks_of(rank, world)
        return min(c_lo * self.chunk_tiles, self.n_tiles), min(c_hi * self.chunk_tiles, self.n_tiles)


def nccl_comm_ptr(group=None, device=None) -> int:
    """Raw ncclComm_t of a NCCL process group (0 if the group is not NCCL or not yet connected).
    The communicator is created lazily by the first collective."""
    if not (dist.is_available() and dist.is_initialized()):
        return 0
    pg = group if group is not None else dist.group.WORLD
    try:
        if dist.get_backend(pg) != "nccl":
            return 0
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        return int(pg._get_backend(dev)._comm_ptr())
    except (AttributeError, RuntimeError):
        return 0


def allreduce_partials(partials: torch.Tensor, group=None, stream=None) -> None:
    """Sum the slot-disjoint partials of every rank in place: through the C ABI
    (lz_allreduce_partials: one ncclAllReduce on the library's stream order) when the group is
    NCCL, else torch.distributed on a host copy (gloo groups: CPU tests and the two-process
    one-GPU test)."""
    comm = nccl_comm_ptr(group, partials.device) if partials.is_cuda else 0
    if comm:
        from . import _native as N
        st = stream if stream is not None else torch.cuda.current_stream(partials.device).cuda_stream
        rc = N.lib().lz_allreduce_partials(partials.data_ptr(), partials.numel(), comm, st)
        if rc == N.LZ_OK:
            return
        if rc != N.LZ_ENCCL:
            N.check(rc, "all-reduce")
        # NCCL could not be resolved or refused the call before enqueueing: torch's collective
        warnings.warn(f"lz_allreduce_partials unavailable ({N.last_error()}); using dist.all_reduce")
    if partials.is_cuda and dist.get_backend(group) != "nccl":
        host = partials.cpu()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        partials.copy_(host)
        return
    dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)


def _world(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


class ShardedIntegral:
    """Reusable device buffers + plan for repeated sharded evaluation of one integral."""

    def __init__(self, plan: Plan, n_u: int, n_v: int, grading: int, device=None, group=None,
                 world=None, rank=None):
        self.plan = plan
        self.n_u, self.n_v, self.grading = n_u, n_v, grading
        self.group = group
        r, w = _world(group)
        # rank/world overrides: time one rank's shard of a larger job on this process's GPU
        self.rank = r if rank is None else rank
        self.world = w if world is None else world
        self.n_nodes, self.n_tiles = plan.tiles(n_u, n_v, grading)
        self.ncomp = plan.ncomp
        self.layout = ChunkLayout(self.n_tiles)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        # tile partials at their global slots (only this rank's range is written and read)
        self.partials = torch.empty(self.n_tiles * self.ncomp, dtype=torch.float64, device=self.device)
        self.chunks = torch.zeros(self.layout.n_chunks * self.ncomp, dtype=torch.float64, device=self.device)
        self.out = torch.zeros(self.ncomp, dtype=torch.float64, device=self.device)
        self.chunk_lo, self.chunk_hi = self.layout.chunks_of(self.rank, self.world)
        self.tile_lo, self.tile_hi = self.layout.tiles_of(self.rank, self.world)

    @property
    def local_nodes(self) -> int:
        return (self.tile_hi - self.tile_lo) * 256

    @property
    def exchange_bytes(self) -> int:
        return self.chunks.numel() * 8

    def _stream(self, stream):
        return stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream

    def integrate(self, stream=None) -> None:
        """Enqueue the tile kernel on this rank's tiles."""
        if self.tile_hi > self.tile_lo:
            self.plan.integrate_device(self.partials, self.n_u, self.n_v, self.grading,
                                       self.tile_lo, self.tile_hi, stream=stream)

    def reduce(self, stream=None) -> torch.Tensor:
        """Chunk sums of this rank, the all-reduce of the chunk vector, the fixed-order total."""
        from . import _native as N
        st = self._stream(stream)
        if self.world > 1:
            self.chunks.zero_()
        N.check(N.lib().lz_reduce_chunks(self.partials.data_ptr(), self.n_tiles, self.ncomp,
                                         self.layout.chunk_tiles, self.chunk_lo, self.chunk_hi,
                                         self.chunks.data_ptr(), st), "chunk reduce")
        if self.world > 1:
            allreduce_partials(self.chunks, self.group, stream)
        Plan.reduce_device(self.chunks, self.layout.n_chunks, self.ncomp, self.out, stream=stream)
        return self.out

    def run(self, stream=None) -> torch.Tensor:
        """Enqueue one evaluation; returns the device tensor of component sums (before 2^d)."""
        self.integrate(stream)
        return self.reduce(stream)


def atm_energy_distributed(lattice: Lattice, grid: ATMGrid | None = None, group=None) -> ATMResult:
    """ATM energy with the node grid sharded over the process group (one GPU per rank)."""
    grid = grid or ATMGrid()
    s = ShardedIntegral(atm_plan(lattice), grid.n_u, grid.n_v, grid.grading, group=group)
    out = s.run().cpu().numpy()
    scale = 2.0 ** lattice.d
    z333, dot = scale * out[0], scale * out[1]
    return ATMResult((z333 - 3.0 * dot) / 6.0, z333, dot, grid, s.n_nodes)


def product_integral_distributed(lattice: Lattice, nus_key: tuple, n_u: int, n_v: int, grading: int = 1,
                                 group=None) -> float:
    """2^d * sum of prod_j Z_j^{m_j} over the sharded fixed grid; nus_key = ((nu, m), ...)."""
    s = ShardedIntegral(product_plan(lattice, nus_key), n_u, n_v, grading, group=group)
    return float(2.0 ** lattice.d * s.run().cpu().numpy()[0])
