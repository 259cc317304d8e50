"""Multi-process (gloo, world size 2, CPU) tests of the N>1 host paths:
shard ranges, global-index RNG keying, the BPTT all-reduce."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_14783_b200.sharding import reduce_bptt, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(rank, world, total)
    # per-env streams keyed by GLOBAL index: what qb_env_reset seeds on device
    seeds = np.array([np.random.PCG64(7 + i).state["state"]["state"] % (1 << 64) for i in range(lo, hi)], np.uint64)
    # BPTT: each rank's env-summed action gradient + its loss share
    T = 5
    rng = np.random.default_rng(100 + rank)
    per_env = torch.as_tensor(rng.normal(size=(hi - lo, T, 4)))
    loss, g = reduce_bptt(torch.tensor(float(rank + 1)), per_env.sum(0))
    result_q.put((rank, lo, hi, seeds, per_env.numpy(), float(loss), g.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [10, 1001])
def test_two_rank_sharding_and_bptt_reduce(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shards tile [0, total) exactly
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == total
    # streams are those of the single-process run
    full = np.array([np.random.PCG64(7 + i).state["state"]["state"] % (1 << 64) for i in range(total)], np.uint64)
    assert np.array_equal(np.concatenate([res[0][3], res[1][3]]), full)
    # all-reduced loss and shared gradient equal the single-process sums
    all_envs = np.concatenate([res[0][4], res[1][4]])
    for r in res:
        assert r[5] == 3.0
        np.testing.assert_allclose(r[6], all_envs.sum(0), rtol=1e-12)


def test_shard_range_single():
    assert shard_range(0, 1, 7) == (0, 7)
    with pytest.raises(ValueError):
        shard_range(2, 2, 7)
