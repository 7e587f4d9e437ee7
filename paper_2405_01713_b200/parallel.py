"""Multi-GPU plumbing for the per-cell path (one process per GPU).

Cells are independent, so ranks integrate disjoint sets of cells
with no collective on the data path: one fixed grid dealt in block-cyclic tiles
(strong scaling, the BASELINE configuration "256^3 cells sharded over 2/4/8
B200") or one slab of a fixed size per rank (weak scaling).  The only communication is
host-side plumbing over torch.distributed: a barrier around the timed region,
the max over ranks of the timed duration, and the sum of the aggregate
integrator statistics.  (The global-norm mode's WRMS allreduce is the one
collective that belongs to the method; it is not part of this module.)
"""
from __future__ import annotations

import os

STAT_SUM = ("n_cells", "n_failed", "nst", "nfe", "nje", "nsetups", "nni", "netf", "ncfn", "nli")
STAT_MAX = ("nst_max", "nfe_max")


def env_rank():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, world: int, cells_per_rank: int):
    """Global cell indices [start, stop) of `rank`'s slab (weak scaling: every rank
    owns cells_per_rank cells of one seeded field of world * cells_per_rank cells)."""
    if not (0 <= rank < world) or cells_per_rank < 1:
        raise ValueError("bad shard request")
    return rank * cells_per_rank, (rank + 1) * cells_per_rank


def block_cyclic_cells(rank: int, world: int, L: int, tile: int = 16):
    """Strong scaling of one L^3 grid: the grid is cut into (L/tile)^3 tiles of tile^3 cells,
    numbered x-fastest, and tile t is dealt to rank t mod world, so every rank gets a spatially spread share of
    any stiffness gradient (an ignition front, a temperature ramp).  Returns the sorted global cell indices
    (x-fastest: c = (k L + j) L + i, the synth.fields grid order) of `rank`'s tiles.  Requires tile | L; when
    world does not divide the tile count the first (count mod world) ranks get one tile more."""
    import numpy as np
    if not (0 <= rank < world) or L < 1 or tile < 1 or L % tile:
        raise ValueError("bad block-cyclic request")
    T = L // tile
    tiles = np.arange(rank, T ** 3, world, dtype=np.int64)
    ti, tj, tk = tiles % T, (tiles // T) % T, tiles // (T * T)
    o = np.arange(tile, dtype=np.int64)
    ii = (ti[:, None] * tile + o[None, :])                     # [tiles, tile]
    jj = (tj[:, None] * tile + o[None, :])
    kk = (tk[:, None] * tile + o[None, :])
    c = (kk[:, :, None, None] * L + jj[:, None, :, None]) * L + ii[:, None, None, :]
    return np.sort(c.reshape(-1))


def contiguous_cells(rank: int, world: int, total: int, align: int = 1):
    """[start, stop) of rank's contiguous part of `total` cells, part sizes multiples of `align` except the last
    (the global-norm mode keeps whole 256-cell reduction blocks per rank, reading R15)."""
    if not (0 <= rank < world) or total < 1:
        raise ValueError("bad contiguous request")
    per = -(-total // world)
    per = -(-per // align) * align
    a = min(total, rank * per)
    return a, min(total, a + per)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (timed durations are reported as the slowest rank)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    """Sum of a per-rank scalar (e.g. the cells each rank integrated)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def reduce_stats(stats: dict, dist=None, device=None) -> dict:
    """Whole-job aggregate of bdfb_get_stats dictionaries (sums and maxima)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return dict(stats)
    import torch
    s = torch.tensor([float(stats[k]) for k in STAT_SUM], dtype=torch.float64, device=device)
    m = torch.tensor([float(stats[k]) for k in STAT_MAX], dtype=torch.float64, device=device)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    out = {k: int(v) for k, v in zip(STAT_SUM, s.tolist())}
    out.update({k: int(v) for k, v in zip(STAT_MAX, m.tolist())})
    return out


def job_throughput(cells_per_rank: int, world: int, max_seconds_per_step: float) -> float:
    """Whole-job cells/s: all ranks' cells over the slowest rank's time."""
    return cells_per_rank * world / max_seconds_per_step


def allreduce_minmax(lo, hi, group=None):
    """Typical values over the whole domain (Eq. 7, "taken over the entire computational domain"):
    element-wise MIN of the per-rank minima and MAX of the maxima over the ranks of `group`
    (torch.distributed; NCCL for device tensors, gloo on CPU).  n doubles each: statistics-sized plumbing,
    not a data-path collective.  No-op without an initialised process group."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return lo, hi
    lo, hi = lo.clone(), hi.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return lo, hi
