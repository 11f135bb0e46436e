"""Multi-rank host logic on CPU (gloo, world size 2): trajectory sharding with
global ids (inputs independent of the rank count), the config-4 ensemble sum
(the engine's only collective) and max-over-ranks timing as bench.py does it."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

B_TOTAL = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_18052_b200 as lbg

    b = B_TOTAL // world
    # shard of global trajectory ids [rank*b, (rank+1)*b)
    rho = lbg.ginibre_batch(2, rank * b, b, 9, threads=1)
    delta, scale = lbg.sweep_params(rank * b, b)
    # stand-in for the per-rank ensemble partial sum (the allreduce'd quantity)
    part = torch.from_numpy(rho.sum(axis=0).view(np.float64).copy())
    dist.all_reduce(part)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, (rho, delta, scale))
    if rank == 0:
        out.put((part.numpy().view(np.complex128).reshape(9, 9), float(t.item()), gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharding_and_ensemble_reduce(world, lbg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ens, tmax, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = lbg.ginibre_batch(2, 0, B_TOTAL, 9, threads=2)
    rho = np.concatenate([g[0] for g in gathered])
    assert np.array_equal(rho, whole)  # inputs independent of the number of ranks
    d0, s0 = lbg.sweep_params(0, B_TOTAL)
    assert np.array_equal(np.concatenate([g[1] for g in gathered]), d0)
    assert np.array_equal(np.concatenate([g[2] for g in gathered]), s0)
    assert np.abs(ens - whole.sum(axis=0)).max() <= 1e-12  # reduction order differs only
    assert abs(np.trace(ens).real - B_TOTAL) <= 1e-12
    assert tmax == float(world)


@pytest.mark.parametrize("B", [1, 7, 4096, 65536, 1 << 20])
def test_strong_scaling_partition_tiles_the_global_batch(B):
    """bench.py's strong-scaling shares [floor(rB/W), floor((r+1)B/W)) tile
    [0, B) exactly for every W, with sizes differing by <= 1."""
    import bench
    for W in (1, 2, 3, 4, 8):
        shares = [bench.share(r, W, B) for r in range(W)]
        assert shares[0][0] == 0 and shares[-1][1] == B
        assert all(shares[r][1] == shares[r + 1][0] for r in range(W - 1))
        sizes = [hi - lo for lo, hi in shares]
        assert max(sizes) - min(sizes) <= 1
        assert bench.config_dict(2, W, "strong")["global_batch"] == 4096
