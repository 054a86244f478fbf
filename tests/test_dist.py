"""Multi-process (world_size 2, gloo, CPU) checks of the frame sharding used by
bench.py on N GPUs: shards are disjoint and contiguous, each rank's generated
shard is bit-identical to the same global frames generated in one process, and
the max/sum reductions of the timed region give the job-wide numbers."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import bsidgen
from paper_1802_08483_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, per_rank, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, local = sharding.dist_env()
    first, count = sharding.frame_range(r, w, per_rank)
    cfg = bsidgen.configs()["C2"]
    b = bsidgen.make_batch(cfg, first, count)
    sharding.barrier()
    t_max = sharding.max_over_ranks(10.0 + r)
    n_tot = sharding.sum_over_ranks(count)
    out[rank] = dict(first=first, count=count, rx=b.rx.copy(), rho=b.rho.copy(), msg=b.msg.copy(),
                     t_max=t_max, n_tot=n_tot, local=local)
    dist.destroy_process_group()


def test_two_rank_sharding_gloo():
    world, per_rank = 2, 24
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), per_rank, out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]
    assert [x["first"] for x in res] == [0, per_rank]
    assert all(x["count"] == per_rank for x in res)
    assert all(x["t_max"] == 11.0 for x in res)
    assert all(x["n_tot"] == world * per_rank for x in res)
    assert [x["local"] for x in res] == [0, 1]
    full = bsidgen.make_batch(bsidgen.configs()["C2"], 0, world * per_rank)
    for r, x in enumerate(res):
        sl = slice(r * per_rank, (r + 1) * per_rank)
        np.testing.assert_array_equal(x["rx"], full.rx[sl])
        np.testing.assert_array_equal(x["rho"], full.rho[sl])
        np.testing.assert_array_equal(x["msg"], full.msg[sl])


def test_frame_seeds_independent_of_batch_split():
    cfg = bsidgen.configs()["C3"]
    a = bsidgen.make_batch(cfg, 100, 6)
    b = bsidgen.make_batch(cfg, 103, 3)
    np.testing.assert_array_equal(a.rx[3:], b.rx)
    np.testing.assert_array_equal(a.rho[3:], b.rho)


def test_single_process_reductions_are_identity():
    assert sharding.max_over_ranks(3.5) == 3.5
    assert sharding.sum_over_ranks(7) == 7.0
    assert sharding.frame_range(0, 1, 10) == (0, 10)


def test_strong_scaling_partition():
    """bench.py --total-frames: contiguous, disjoint, covering, sizes within one frame."""
    for total in (0, 1, 7, 256, 1001):
        for world in (1, 2, 3, 8):
            parts = [sharding.frame_range_strong(r, world, total) for r in range(world)]
            assert sum(c for _, c in parts) == total
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(world - 1))
            assert parts[0][0] == 0
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
