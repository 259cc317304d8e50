"""Multi-GPU contract of the env-parallel path on one GPU (SURVEY 8-E,
SPEC.md:485): env i evolves identically whatever the world size.

  * make_env(cfg, shard=(r, W)) for r = 0, 1 equals the unsharded env's
    slices bit for bit -- states, flags, rewards, nearest points, depth and
    segmentation images -- over 50 steps with respawns (per-env streams keyed
    by the GLOBAL index, reference base.py:95 default_rng(seed + i))
  * config 4: the sharded forward + adjoint equals the unsharded one per env,
    the env-summed shared-action gradient is bitwise reproducible, and two
    processes (gloo) reducing their shards with reduce_bptt get the
    single-process sums
  * bench.py --gpus 2 launches its own ranks (plumbing; its numbers are not
    benchmark values on a shared GPU)

Two shards of one env on one GPU are independent envs: no kernel of one waits
on the other (the only collective is the host-side BPTT all-reduce)."""

import dataclasses
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2407_14783_b200 import gradients as G  # noqa: E402
from paper_2407_14783_b200.control import LV  # noqa: E402
from paper_2407_14783_b200.env import make_env, navigation_config  # noqa: E402
from paper_2407_14783_b200.params import native_params  # noqa: E402
from paper_2407_14783_b200.sharding import reduce_bptt, shard_range  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sharded_env_equals_unsharded_slices():
    n, W = 100, 2
    cfg = dataclasses.replace(navigation_config(0, n, with_segmentation=True), episode_max_steps=12)
    full = make_env(cfg)
    shards = [make_env(cfg, shard=(r, W)) for r in range(W)]
    ranges = [shard_range(r, W, n) for r in range(W)]
    assert [s.index_offset for s in shards] == [lo for lo, _ in ranges]
    full.reset(seed=4)
    for s in shards:
        s.reset(seed=4)
    g = torch.Generator(device="cuda").manual_seed(3)
    respawns = 0
    for t in range(50):
        v = torch.randn(n, 3, device="cuda", generator=g) * 2.0
        yaw = torch.randn(n, device="cuda", generator=g)
        rf = full.step(LV(v, yaw))
        rs = [s.step(LV(v[lo:hi].contiguous(), yaw[lo:hi].contiguous())) for s, (lo, hi) in zip(shards, ranges)]
        torch.cuda.synchronize()
        respawns += int(rf.terminated.sum() + rf.truncated.sum())
        for s, r, (lo, hi) in zip(shards, rs, ranges):
            assert torch.equal(s._planes, full._planes[:, lo:hi]), t
            for a, b in ((r.reward, rf.reward), (r.terminated, rf.terminated), (r.truncated, rf.truncated),
                         (s.nearest_pt, full.nearest_pt), (s.nearest_dist, full.nearest_dist),
                         (s.step_counts, full.step_counts), (s._rng, full._rng)):
                assert torch.equal(a, b[lo:hi]), t
            for k in ("depth", "segmentation"):
                assert torch.equal(r.observations[k], rf.observations[k][lo:hi]), (t, k)
    assert respawns > 0


def _bptt_inputs(n, T, seed=7):
    g = torch.Generator(device="cuda").manual_seed(seed)
    init = torch.zeros((17, n), device="cuda")
    init[0:3] = (torch.rand((3, n), device="cuda", generator=g) - 0.5) * 0.2
    init[6] = 1.0
    init[13:17] = 900.0
    acts = 900.0 + torch.randn((T, n, 4), device="cuda", generator=g) * 20.0
    return init, acts


def _bptt(init, acts, total):
    P = native_params()
    tape, _ = G.rollout_planes(P, "rotor", init, acts)
    d = tape[-1, 0:3] - torch.tensor([1.0, 0.0, 2.0], device="cuda")[:, None]
    gtraj = torch.zeros_like(tape)
    gtraj[-1, 0:3] = 2.0 * d / total
    gsum = torch.zeros(acts.shape[0] * 4, dtype=torch.float64, device="cuda")
    ga, gi, _ = G.backward_planes(P, "rotor", tape, acts, gtraj, action_grad_sum=gsum)
    loss = float((d.double() ** 2).sum() / total)
    return ga, gi, gsum, loss


def test_sharded_bptt_equals_unsharded():
    n, T, W = 2048, 64, 2
    init, acts = _bptt_inputs(n, T)
    ga, gi, gsum, _ = _bptt(init, acts, n)
    ga2, gi2, gsum2, _ = _bptt(init, acts, n)
    assert torch.equal(gsum, gsum2)  # deterministic env-sum (no atomics)
    assert torch.equal(ga, ga2) and torch.equal(gi, gi2)
    np.testing.assert_allclose(gsum.cpu().numpy().reshape(T, 4), ga.double().sum(1).cpu().numpy(), rtol=1e-10,
                               atol=1e-15)
    parts = []
    for r in range(W):
        lo, hi = shard_range(r, W, n)
        a, i, s, _ = _bptt(init[:, lo:hi].contiguous(), acts[:, lo:hi].contiguous(), n)
        assert torch.equal(a, ga[:, lo:hi]) and torch.equal(i, gi[:, lo:hi])
        parts.append(s)
    np.testing.assert_allclose((parts[0] + parts[1]).cpu().numpy(), gsum.cpu().numpy(), rtol=1e-12, atol=1e-18)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, n, T, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    init, acts = _bptt_inputs(n, T)
    lo, hi = shard_range(rank, world, n)
    _, _, gsum, loss = _bptt(init[:, lo:hi].contiguous(), acts[:, lo:hi].contiguous(), n)
    buf = torch.zeros(T * 4 + 1, dtype=torch.float64)  # gloo: a host buffer
    loss_all, g_all = reduce_bptt(loss, gsum, out=buf)
    q.put((rank, float(loss_all), g_all.numpy().copy()))
    dist.destroy_process_group()


def test_two_process_bptt_reduce():
    import torch.multiprocessing as mp

    n, T, world = 2048, 64, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    init, acts = _bptt_inputs(n, T)
    _, _, gsum, loss = _bptt(init, acts, n)
    for _, l, g in res:
        np.testing.assert_allclose(l, loss, rtol=1e-12)
        np.testing.assert_allclose(g, gsum.cpu().numpy(), rtol=1e-12, atol=1e-18)


def test_bench_spawns_its_own_ranks():
    env = dict(os.environ, QB_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "c1", "--steps", "10",
                          "--warmup", "3", "--no-cpu", "--no-e2e"], capture_output=True, text=True, timeout=600, env=env,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["global_envs"] == 200 and line["value"] > 0


def test_bench_two_ranks_end_to_end_leg():
    """The e2e leg under two ranks: each rank's flat-bindings handle owns its
    shard (bindings.make_env(shard=...)); the whole-job e2e value counts both."""
    env = dict(os.environ, QB_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "c2a", "--steps", "10",
                          "--warmup", "3", "--no-cpu"], capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["global_envs"] == 200
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 100 * 16
