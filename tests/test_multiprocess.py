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
