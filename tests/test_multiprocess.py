"""World-size-2 gloo test of the multi-GPU host logic (CPU): sharding covers the
field exactly once, per-cell results do not depend on the sharding, the timed
duration is the max over ranks and the statistics aggregate to the
single-process totals.  The per-rank integration uses the CPU oracle (there is
no GPU here); the logic under test is paper_2405_01713_b200.parallel."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cells_per_rank, out):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2405_01713_b200 import parallel as PL
    from synth import robertson_field
    r, w, lr = PL.env_rank()
    a, b = PL.shard(r, w, cells_per_rank)
    y0 = robertson_field(w * cells_per_rank, cells=np.arange(a, b))
    y, st = O.integrate_batch(O.Model.robertson(), y0, 0.0, 40.0, 1e-6, 1e-10)
    stats = {k: 0 for k in PL.STAT_SUM + PL.STAT_MAX}
    stats.update(n_cells=y.shape[1], n_failed=int((st["status"] != 0).sum()), nst=int(st["nst"].sum()),
                 nfe=int(st["nfe"].sum()), nje=int(st["nje"].sum()), nsetups=int(st["nsetups"].sum()),
                 nni=int(st["nni"].sum()), netf=int(st["netf"].sum()), ncfn=int(st["ncfn"].sum()),
                 nst_max=int(st["nst"].max()), nfe_max=int(st["nfe"].max()))
    agg = PL.reduce_stats(stats, dist)
    tmax = PL.max_over_ranks(1.0 + rank, dist)
    out[rank] = (a, b, y, agg, tmax)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    world, cpr = 2, 48
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), cpr, out), nprocs=world, join=True)
    sys.path.insert(0, REPO)
    from oracle import oracle as O
    from synth import robertson_field
    y0 = robertson_field(world * cpr)
    yref, st = O.integrate_batch(O.Model.robertson(), y0, 0.0, 40.0, 1e-6, 1e-10)
    got = np.zeros_like(yref)
    covered = np.zeros(world * cpr, int)
    for r in range(world):
        a, b, y, agg, tmax = out[r]
        got[:, a:b] = y
        covered[a:b] += 1
        assert tmax == float(world)                       # max over ranks
        assert agg["n_cells"] == world * cpr
        assert agg["nst"] == int(st["nst"].sum()) and agg["nfe"] == int(st["nfe"].sum())
        assert agg["nst_max"] == int(st["nst"].max())
    assert np.all(covered == 1)
    assert np.array_equal(got, yref)                       # sharding-invariant, bit for bit


def test_shard_arithmetic():
    from paper_2405_01713_b200 import parallel as PL
    assert PL.shard(0, 4, 10) == (0, 10) and PL.shard(3, 4, 10) == (30, 40)
    with pytest.raises(ValueError):
        PL.shard(4, 4, 10)
    assert PL.job_throughput(100, 8, 2.0) == 400.0


def _tv_worker(rank, world, port, cells_per_rank, out):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_01713_b200 import parallel as PL
    from synth import flame_field
    a, b = PL.shard(rank, world, cells_per_rank)
    y, _, _, _ = flame_field("h2_lidryer", 8, cells=np.arange(a, b))
    # each rank's own min/max (what bdfb_minmax returns on its GPU), then the MIN/MAX over ranks
    lo, hi = torch.tensor(y.min(axis=1)), torch.tensor(y.max(axis=1))
    glo, ghi = PL.allreduce_minmax(lo, hi)
    out[rank] = (glo.numpy(), ghi.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_typical_values_gloo():
    """Eq. 7 typical values over the whole domain: the per-rank min/max combined with MIN/MAX over 2 ranks
    give the oracle's typical values of the unsharded field, bit for bit, on every rank."""
    world, cpr = 2, 256
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_tv_worker, args=(world, _free_port(), cpr, out), nprocs=world, join=True)
    sys.path.insert(0, REPO)
    from oracle import oracle as O
    from synth import flame_field
    y, _, _, _ = flame_field("h2_lidryer", 8, cells=np.arange(world * cpr))
    tv = O.typical_values(y)
    for r in range(world):
        lo, hi = out[r]
        assert np.array_equal(0.5 * (lo + hi), tv)


# ---------------------------------------------------------------- strong scaling: block-cyclic tiles
def test_block_cyclic_partition_covers_grid_once():
    """Tiles of 16^3 dealt round-robin: every cell of the grid exactly once, balanced to one tile, and each
    rank's cells spread over the whole grid (every z-slab of tiles is represented when world <= tiles/slab)."""
    sys.path.insert(0, REPO)
    from paper_2405_01713_b200 import parallel as PL
    L, tile = 64, 16
    for world in (1, 2, 3, 4, 8):
        parts = [PL.block_cyclic_cells(r, world, L, tile) for r in range(world)]
        allc = np.concatenate(parts)
        assert len(allc) == L ** 3 and len(np.unique(allc)) == L ** 3
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= tile ** 3
        for p in parts:
            assert len(np.unique(p // (L * L * tile))) == L // tile      # every z-slab of tiles
    with pytest.raises(ValueError):
        PL.block_cyclic_cells(0, 2, 60, 16)


def _strong_worker(rank, world, port, L, tile, out):
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2405_01713_b200 import parallel as PL
    from synth import robertson_field
    cells = PL.block_cyclic_cells(rank, world, L, tile)
    y0 = robertson_field(L ** 3, cells=cells)
    y, st = O.integrate_batch(O.Model.robertson(), y0, 0.0, 4.0, 1e-6, 1e-10)
    total = PL.sum_over_ranks(len(cells), dist)
    out[rank] = (cells, y, total)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_strong_scaling_block_cyclic_gloo():
    """bench.py's default multi-GPU mode on the CPU: two ranks integrate their block-cyclic tiles of one fixed
    grid; the union is the whole grid, the cell count sums to L^3 over the ranks, and every cell equals the
    single-process result bit for bit (the seeded inputs do not depend on the partition)."""
    world, L, tile = 2, 8, 4
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_strong_worker, args=(world, _free_port(), L, tile, out), nprocs=world, join=True)
    sys.path.insert(0, REPO)
    from oracle import oracle as O
    from synth import robertson_field
    y0 = robertson_field(L ** 3)
    yref, _ = O.integrate_batch(O.Model.robertson(), y0, 0.0, 4.0, 1e-6, 1e-10)
    seen = np.zeros(L ** 3, int)
    for r in range(world):
        cells, y, total = out[r]
        assert total == L ** 3
        seen[cells] += 1
        assert np.array_equal(y, yref[:, cells])
    assert np.all(seen == 1)
