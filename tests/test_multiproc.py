"""N>1 host logic on CPU (gloo, world_size 2): batch sharding of a conv program is exact
(each rank's shard program over its slice == the corresponding slice of the full program),
and the max-over-ranks reduction the bench uses."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_06498_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch

    from oracle import Port, Rng, wrap
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, H, Wd, C, K = 4, 5, 6, 8, 4
    rng = Rng(99)
    I = wrap(8, rng.bulk(N * H * Wd * C)).reshape(N, H * Wd * C)
    F = wrap(8, rng.bulk(9 * K * C))
    lo, hi = W.shard_range(N, world, rank)
    text = W.conv2d(hi - lo, H, Wd, C, K)
    o = Port.execute(text, {"I": I[lo:hi].ravel(), "F": F, "O": np.zeros((hi - lo) * H * Wd * K, np.int64)})["O"]
    objs = [None] * world
    dist.all_gather_object(objs, o)
    gathered = [torch.from_numpy(x.astype(np.float64)) for x in objs]
    elapsed = torch.tensor([1.0 + rank])  # bench.py: device time reduced with MAX over ranks
    dist.all_reduce(elapsed, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = Port.execute(W.conv2d(N, H, Wd, C, K), {"I": I.ravel(), "F": F,
                                                       "O": np.zeros(N * H * Wd * K, np.int64)})["O"]
        out["ok"] = bool(np.array_equal(torch.cat(gathered).numpy().astype(np.int64), full))
        out["max"] = float(elapsed.item())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_batch_sharding_gloo_world2():
    from oracle import Port
    if not Port.available():
        pytest.skip("oracle/_port not built")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["ok"]
    assert out["max"] == 2.0


def test_shard_range_partitions():
    for total in (1, 5, 32, 1024):
        for world in (1, 2, 3, 8):
            spans = [W.shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
