"""Benchmark of the VisFly/quadsim hot path on B200.

BASELINE.json metric: env-steps/s and 64x64 depth frames/s (whole box) at
1/2/4/8 B200 vs the CPU reference.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c1|c2|c2a|c4|c5|c3n|swarm] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Default workload = BASELINE config 3, the largest single-GPU config:
navigation, 65,536 envs per GPU, 64x64 depth + segmentation from one camera,
seeded LV actions, the full env.step (lazy auto-reset, controller, RK4 x2
dynamics, proximity / collision / out-of-bounds, reward, termination) plus
the observation render.  One env-step renders one 64x64 depth frame, so
env-steps/s == depth frames/s.  Multi-GPU: envs sharded by global index,
no per-step collective ("scaling": "weak"); time = max over ranks of the
CUDA-event time; value = all ranks' env-steps / that time.

One JSON line (rank 0).  Besides the contract keys:
  roofline            dominant kernel of the step (K2 render) vs HBM
  roofline_dynamics   K1 alone at 16.7M envs (HBM-bound design target)
  cpu_baseline        CPU oracle (C restatement, OpenMP, all host cores) on a
                      bounded sample of the same workload
  e2e                 public API with host buffers (pinned H2D actions, D2H of
                      observations + reward/flags) inside the timed region
  clocks, gpu_launches, kernel_ms
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "env-steps/sec (= 64x64 depth frames/sec), whole box"
WORKLOADS = {
    "c1": "hover free flight (garage), dynamics only, 100 envs/GPU (BASELINE config 1)",
    "c2": "navigation, 64x64 depth, 100 envs/GPU, procedural box/cylinder triangle-mesh room (BASELINE config 2)",
    "c2a": "config 2 on the analytic scene (the same room and obstacles as spheres / oriented boxes)",
    "c3": "navigation, 64x64 depth+segmentation, 65536 envs/GPU (BASELINE config 3)",
    "c4": "BPTT through dynamics, 16384 envs/GPU, horizon 64, loss/grad all-reduce (BASELINE config 4)",
    "c5": "landing on a 5e5-triangle indoor mesh, 64x64 down depth+seg, 131072 envs/GPU (BASELINE config 5, 1M on 8 GPUs)",
    "c3n": "config 3 + sensor noise (SURVEY F1): depth N(0, 0.02) -> Redwood, segmentation salt-and-pepper 2%, "
           "IMU N(0, 0.05); 65536 envs/GPU",
    "swarm": "swarm gap crossing (SURVEY F2): one swarm of 256 agents, 64x64 depth with the other 255 agents "
             "rendered as spheres, pairwise collisions",
}
ENVS = {"c1": 100, "c2": 100, "c2a": 100, "c3": 65536, "c4": 16384, "c5": 131072, "c3n": 65536, "swarm": 256}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi SM clock + throttle reasons, sampled during the timed region."""

    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index=0):
        self.samples, self.index, self._stop, self._t = [], index, threading.Event(), None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                          "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.1)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        good = [s for s in self.samples if len(s) >= 3]
        sm = [float(s[0]) for s in good if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in good if s[1].replace(".", "").isdigit()]
        reasons = set()
        for s in good:
            try:
                v = int(s[2], 16)
            except Exception:
                continue
            reasons.update(name for bit, name in self.BITS.items() if v & bit)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- distributed


# plumbing test hook only (tests/test_gpu_sharding.py): QB_BENCH_SHARE_GPU=1 puts
# every rank on cuda:0 with the gloo backend, to exercise the launcher and the
# max-over-ranks timing on a one-GPU box; its numbers are not benchmark values
SHARE_GPU = os.environ.get("QB_BENCH_SHARE_GPU") == "1"


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARE_GPU:
        local = 0
    torch.cuda.set_device(local if world > 1 else 0)
    if world > 1:
        import torch.distributed as dist

        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARE_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def profile_traffic(kernel_key):
    """Per-unit DRAM traffic (bytes) of a kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d[kernel_key]["dram_bytes_per_unit"], d[kernel_key]
    except Exception:
        return None, None


# ---------------------------------------------------------------- our arm


def workload_config(kind, n):
    """The EnvConfig of a workload for n agents (one swarm of n for 'swarm')."""
    import dataclasses

    from paper_2407_14783_b200.env import (DistSpec, EnvConfig, InitRandomization, SceneSpec, SensorSpec,
                                           gap_crossing_config, navigation_config)
    from paper_2407_14783_b200.sensing import NoiseSpec

    if kind == "c1":
        return EnvConfig(num_agents=n, command_type="ctbr", episode_max_steps=1000)
    if kind == "c2":  # the tessellated variant (SURVEY 8-D C2 b): 69 objects, 2076 triangles
        cfg = navigation_config(scene_seed=0, num_agents=n)
        return dataclasses.replace(cfg, scenes=(dataclasses.replace(cfg.scenes[0], kind="cluttered_mesh"),))
    if kind == "c2a":
        return navigation_config(scene_seed=0, num_agents=n)
    if kind == "c3":
        return navigation_config(scene_seed=0, num_agents=n, with_segmentation=True)
    if kind == "c3n":
        cfg = navigation_config(scene_seed=0, num_agents=n, with_segmentation=True)
        return dataclasses.replace(cfg, sensors=(
            SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("normal", sigma=0.02),
                                                          NoiseSpec("redwood", sigma_disparity=0.002))),
            SensorSpec(kind="segmentation", name="vision", noise=(NoiseSpec("saltpepper", p=0.02),)),
            SensorSpec(kind="imu", name="imu", noise=(NoiseSpec("normal", sigma=0.05),))))
    if kind == "swarm":
        cfg = gap_crossing_config(num_agents=n)
        return dataclasses.replace(cfg, randomization=InitRandomization(
            position=DistSpec("uniform", low=[-5.5, -5.5, 0.5], high=[-1.0, 5.5, 3.5])))
    if kind == "c5":
        return EnvConfig(num_agents=n, task="landing", command_type="lv", episode_max_steps=512,
                         scenes=(SceneSpec(kind="indoor", seed=0),),
                         randomization=InitRandomization(position=DistSpec("uniform", low=[-12, -12, 1.0],
                                                                           high=[12, 12, 4.5])),
                         min_spawn_clearance=0.3,
                         sensors=(SensorSpec(kind="depth", name="depth", orientation="down"),
                                  SensorSpec(kind="segmentation", name="vision", orientation="down")))
    raise ValueError(kind)


def env_workload(kind, rank, world, total):
    from paper_2407_14783_b200.env import make_env

    if kind == "swarm":  # one swarm per rank (swarms do not shard: every agent sees every other)
        cfg = workload_config(kind, total // world)
        return make_env(cfg), cfg
    cfg = workload_config(kind, total)
    # config 5's 5e5-triangle hall: built on the device (LBVH + SAH treelet refinement, ~26 ms; its tree
    # renders as fast as the host binned-SAH tree, which takes ~0.45 s to build)
    build = "device" if kind == "c5" else "host"
    return make_env(cfg, shard=(rank, world), scene_build=build), cfg


def make_actions(kind, n, count, rank):
    import torch

    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    a = torch.empty((count, n, 4), device="cuda")
    if kind == "c1":  # hover CTBR + seeded body-rate perturbation
        a[..., 0] = 9.81
        a[..., 1:] = torch.randn((count, n, 3), device="cuda", generator=g) * 0.5
    else:  # LV set-points + yaw
        a[..., :3] = torch.randn((count, n, 3), device="cuda", generator=g) * 1.5
        a[..., 0] += 1.0
        a[..., 3] = (torch.rand((count, n), device="cuda", generator=g) * 2 - 1) * math.pi
    return a  # (count, n, 4) contiguous; a[i] is step i's (n, 4) action


def run_env(args, rank, world, kind):
    import torch

    import paper_2407_14783_b200._native as nat

    total = ENVS[kind] * world
    env, cfg = env_workload(kind, rank, world, total)
    env.reset(seed=args.seed)
    n, K, W = env.num_agents, args.steps, args.warmup
    acts = make_actions(kind, n, K + W, rank)
    small = n <= 4096  # latency-bound configs (1, 2): replay 10-step CUDA graphs
    G = 10
    graph = None
    if small:
        K = max(G, (K + G - 1) // G * G)
        args.steps = K
        acts = make_actions(kind, n, K + W, rank)
        static_a = torch.zeros((G, n, 4), device="cuda")
        graph = env.make_step_graph(static_a)

    def launch(a, events=None):
        env._bufs.action = a.data_ptr()
        if events:
            events[0].record()
        nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))
        if events:
            events[1].record()
        env._render()
        if events:
            events[2].record()
        env._observe()
        if events:
            events[3].record()

    def launch_graph(first):
        static_a.copy_(acts[first:first + G])  # stage the next G steps' actions (one device copy)
        graph()

    for i in range(W):
        launch(acts[i])
    if small:
        launch_graph(0)
    torch.cuda.synchronize()
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(K)]
    barrier(world)
    torch.cuda.synchronize()
    clk = ClockSampler(0 if SHARE_GPU else int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    if small:
        for k in range(0, K, G):
            launch_graph(W + k)
    else:
        for k in range(K):
            launch(acts[W + k], ev[k])
    t1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = max_over_ranks(t0.elapsed_time(t1), world)
    k3 = 2 if (small and env.split_step) else 1  # the graph path launches the split step's two phases
    launches = K * (k3 + len(env._cams) + (1 if env._obs_sensors else 0))
    out = dict(env=env, cfg=cfg, n=n, total=total, ms=ms, clocks=clocks, launches=launches, graph=small)
    if not small:
        out["step_ms"] = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
        out["render_ms"] = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
        if env._obs_sensors:
            out["observe_ms"] = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    return out


def run_e2e(cfg, rank, world, kind):
    """End to end through the reference-facing flat-array boundary
    (bindings.step: SPEC.md:566-605 -> qb_env_step_io, one native call per
    step): actions from pinned host memory, observations + reward / flags /
    info back in pinned host memory before the call returns.  Host clock
    around K steps (a host-to-host number), max over ranks."""
    import torch

    from paper_2407_14783_b200 import bindings

    h = bindings.make_env(cfg, shard=(rank, world), scene_build="device" if kind == "c5" else "host")
    n = h.num_agents
    K = 6 if n > 4096 else 200
    rng = np.random.default_rng(rank)
    acts = []
    for _ in range(K + 2):
        a = torch.empty((n, 4), dtype=torch.float32, pin_memory=True).numpy()
        if cfg.command_type == "ctbr":
            a[:, 0] = 9.81
            a[:, 1:] = rng.normal(scale=0.5, size=(n, 3))
        else:
            a[:, :3] = rng.normal(scale=1.5, size=(n, 3))
            a[:, 0] += 1.0
            a[:, 3] = rng.uniform(-math.pi, math.pi, n)
        acts.append(a)
    out = h.outputs(pinned=True)
    bindings.reset(h, 0, out=out)
    for k in range(2):
        bindings.step(h, acts[k], out=out)
    barrier(world)
    t = time.perf_counter()
    for k in range(K):
        res = bindings.step(h, acts[k + 2], out=out)
    dt = max_over_ranks(time.perf_counter() - t, world)
    d2h = sum(v.nbytes for k, v in out.items() if not k.startswith("_") and hasattr(v, "nbytes")) + out["_small"].nbytes
    h2d = acts[0].nbytes
    seg = {k: str(v.dtype) for k, v in res[0].arrays.items()}
    bindings.close(h)
    return {"value": n * world * K / dt, "unit": "env-steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": K, "ms_per_step": dt / K * 1e3, "dtypes": seg,
            "path": "bindings.step(handle, pinned (N,4) actions) -> qb_env_step_io: action read in place, env step, "
                    "render, state rows + flags/reward packed into pinned host memory, images D2H (segmentation as "
                    "uint8 when every id < 256, lossless; >= 4,096 envs: rendered in up to 16 camera slices, each "
                    "slice's D2H overlapping the next slices' renders), stream synchronised before returning"}


def run_e2e_device_obs(env, world, kind, K=50):
    """A GPU-resident policy's loop (Isaac-Gym style): the public env.step
    with host actions from pinned memory (H2D inside the timed region) and
    the step's reward / terminated / truncated read back to the host every
    step (D2H), while the observations stay on the device for the policy.
    A secondary figure beside `e2e` (which ships every observation back)."""
    import torch

    from paper_2407_14783_b200.control import CTBR, LV

    n = env.num_agents
    rng = np.random.default_rng(1)
    acts = []
    for _ in range(K + 2):
        a = torch.empty((n, 4), dtype=torch.float32, pin_memory=True)
        a[:, :3] = torch.as_tensor(rng.normal(scale=1.5, size=(n, 3)), dtype=torch.float32)
        a[:, 3] = torch.as_tensor(rng.uniform(-math.pi, math.pi, n), dtype=torch.float32)
        acts.append(a)
    host = torch.empty(n * 6, dtype=torch.uint8, pin_memory=True)

    def one(a):
        cmd = CTBR(a[:, 0] + 9.81, a[:, 1:]) if kind == "c1" else LV(a[:, :3], a[:, 3])
        r = env.step(cmd)
        host[:4 * n].view(torch.float32).copy_(r.reward, non_blocking=True)
        host[4 * n:5 * n].copy_(r.terminated.view(torch.uint8), non_blocking=True)
        host[5 * n:].copy_(r.truncated.view(torch.uint8), non_blocking=True)
        torch.cuda.current_stream().synchronize()  # the host reads the step's result

    for k in range(2):
        one(acts[k])
    barrier(world)
    t = time.perf_counter()
    for k in range(K):
        one(acts[k + 2])
    dt = max_over_ranks(time.perf_counter() - t, world)
    return {"value": n * world * K / dt, "unit": "env-steps/s", "h2d_bytes_per_step": n * 16,
            "d2h_bytes_per_step": n * 6, "steps": K,
            "path": "env.step(LV from pinned host actions) -> reward / terminated / truncated read back each step; "
                    "observations stay on the device (a GPU-resident policy)"}


def run_env_step_roofline(pk):
    """K1+K3 fused env step alone (qb_env_step) at 4M envs, free flight in the
    garage: per env-step it reads the state (68 B) + action (16 B) + step
    count, scene, respawn flag (9 B) and writes state + prev_state (136 B),
    7 flags, reward, nearest distance + point (7 + 4 + 32 B), step count (4 B):
    272 algorithmic B/env-step; the exact-double proximity query and reward
    are computed, not read.  L2 (126 MB) << the 1.1 GB of planes touched."""
    import torch

    import paper_2407_14783_b200._native as nat
    from paper_2407_14783_b200.env import EnvConfig, make_env

    n = 1 << 22
    env = make_env(EnvConfig(num_agents=n, command_type="ctbr", episode_max_steps=10**6))
    env.reset(seed=0)
    act = torch.zeros((n, 4), device="cuda")
    act[:, 0] = 9.81
    act[:, 1:] = torch.randn((n, 3), device="cuda") * 0.3
    env._bufs.action = act.data_ptr()

    def launch():
        nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))

    for _ in range(3):
        launch()
    ev = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    gbs = n * 272 / (ms / 1e3) / 1e9
    del env
    return {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
            "traffic": None, "envs": n, "ms": ms, "env_steps_per_sec": n / (ms / 1e3),
            "note": "K1+K3 fused env step (CTBR, RK4 x2, exact-double nearest point over the garage, flags, reward), "
                    "272 algorithmic B/env-step"}


def run_dynamics_roofline(pk):
    """K1 alone at 16.7M envs: 152 B/env-step (read 17 + 4 floats, write 17)."""
    import torch

    import paper_2407_14783_b200._native as nat
    from paper_2407_14783_b200.params import native_params

    n = 1 << 24
    P = native_params()
    pl = torch.zeros((17, n), device="cuda")
    pl[0:3] = torch.rand((3, n), device="cuda")
    pl[6] = 1.0
    pl[13:17] = 900.0
    act = torch.empty((n, 4), device="cuda")
    act[:, 0] = 9.81
    act[:, 1:] = torch.randn((n, 3), device="cuda") * 0.3
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def launch():
        nat.check(nat.lib().qb_dynamics_step(P, nat.CMD["ctbr"], nat.QB_F32, n, n, nat.ptr(pl), nat.ptr(act), None, None,
                                             nat.stream_of()))

    for _ in range(3):
        launch()
    ev = []
    for _ in range(10):
        flush.zero_()  # L2 flushed between launches
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch()
        b.record()
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    gbs = n * 152 / (ms / 1e3) / 1e9
    traffic, _ = profile_traffic("k_dyn_step")
    return {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
            "traffic": traffic * n if traffic else None, "envs": n, "ms": ms, "env_steps_per_sec": n / (ms / 1e3),
            "note": "K1 (CTBR controller + mixer + RK4 x2 + renorm), 152 algorithmic B/env-step, L2 flushed"}


def run_bptt(args, rank, world):
    """Config 4: BPTT through the dynamics, horizon 64, 16384 envs/GPU.
    One iteration = forward rollout (1 launch) + loss and its trajectory
    gradient + adjoint sweep (1 launch) + fixed-order env-sum of the shared
    action gradient, replayed as one CUDA graph, then all_reduce(SUM) of loss
    and shared gradient over NCCL."""
    import torch

    from paper_2407_14783_b200 import gradients as G
    from paper_2407_14783_b200.params import native_params
    from paper_2407_14783_b200.sharding import reduce_bptt

    # weak scaling: 16384 envs per GPU; --strong: 16384 envs in total, split over the ranks
    n, T = (ENVS["c4"] // world if args.strong else ENVS["c4"]), 64
    P = native_params()
    g = torch.Generator(device="cuda").manual_seed(7 + rank)
    init = torch.zeros((17, n), device="cuda")
    init[0:3] = (torch.rand((3, n), device="cuda", generator=g) - 0.5) * 0.2
    init[6] = 1.0
    init[13:17] = 900.0
    acts = 900.0 + torch.randn((T, n, 4), device="cuda", generator=g) * 20.0
    target = torch.tensor([1.0, 0.0, 2.0], device="cuda")
    gsum = torch.zeros(T * 4, dtype=torch.float64, device="cuda")
    red = torch.zeros(T * 4 + 1, dtype=torch.float64, device="cpu" if SHARE_GPU else "cuda")
    # dL/dtrajectory: the loss reads only the final positions, so every other block stays zero (written once)
    gtraj = torch.zeros((T + 1, 17, n), device="cuda")

    loss_buf = torch.zeros((), dtype=torch.float64, device="cuda")

    def local():
        """Everything of an iteration but the collective: forward rollout, loss and
        its trajectory gradient, adjoint sweep, env-sum of the action gradient."""
        tape, _ = G.rollout_planes(P, "rotor", init, acts)
        d = tape[-1, 0:3] - target[:, None]
        loss_buf.copy_((d * d).sum() / (n * world) + 1e-6 * ((acts - 900.0) ** 2).sum())
        gtraj[-1, 0:3] = 2.0 * d / (n * world)
        gsum.zero_()
        G.backward_planes(P, "rotor", tape, acts, gtraj, action_grad_sum=gsum)

    for _ in range(2):  # warm-up (allocator, module loading) before capture
        local()
    torch.cuda.synchronize()
    # the iteration's ~15 launches replayed as one CUDA graph (static shapes); the
    # NCCL all-reduce stays outside the graph
    graph = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs):
        with torch.cuda.graph(graph, stream=cs):
            local()
    torch.cuda.current_stream().wait_stream(cs)

    def iteration():
        graph.replay()
        reduce_bptt(loss_buf, gsum, out=red)  # one all_reduce(SUM) of [shared grad, loss] over NCCL

    for _ in range(args.warmup):
        iteration()
    torch.cuda.synchronize()
    barrier(world)
    K = args.steps
    clk = ClockSampler(0 if SHARE_GPU else int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(K):
        iteration()
    t1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = max_over_ranks(t0.elapsed_time(t1), world)
    # per-kernel device time: each direction captured alone in a CUDA graph and
    # replayed back to back (an eager call's host overhead and allocations
    # would otherwise be timed with a 0.05 ms kernel)
    tape_s, _ = G.rollout_planes(P, "rotor", init, acts)
    gz = torch.zeros_like(tape_s)

    def graph_ms(fn, R=20):
        gr, s = torch.cuda.CUDAGraph(), torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()  # warm-up outside the capture
            with torch.cuda.graph(gr, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        gr.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(R):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / R

    fwd_ms = graph_ms(lambda: G.rollout_planes(P, "rotor", init, acts))
    bwd_ms = graph_ms(lambda: G.backward_planes(P, "rotor", tape_s, acts, gz, action_grad_sum=gsum))
    return dict(n=n, T=T, ms=ms, clocks=clocks, fwd_ms=fwd_ms, bwd_ms=bwd_ms)


def cpu_baseline_env(kind="c3", n_sample=1024, steps=12):
    """The CPU oracle (C restatement of the reference, OpenMP on all host
    cores) on a bounded sample of the same workload: env-steps/s."""
    import oracle
    from oracle.env import OracleEnv
    from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig

    cfg = workload_config(kind, n_sample)
    scenes = []
    for spec in cfg.scenes:
        t = spec.materialize().arrays
        scenes.append(oracle.OracleScene(t.prim_type, t.prim_data, t.prim_object_id, t.prim_aabb_lo, t.prim_aabb_hi))
    env = OracleEnv(cfg, scenes, QuadParams(), SimConfig(), ControllerGains())
    env.reset(seed=0)
    rng = np.random.default_rng(0)

    def act():
        if cfg.command_type == "ctbr":
            return np.concatenate([np.full((n_sample, 1), 9.81), rng.normal(scale=0.5, size=(n_sample, 3))], 1)
        return np.concatenate([rng.normal(scale=1.5, size=(n_sample, 3)), rng.uniform(-3, 3, (n_sample, 1))], 1)

    env.step(act())
    t = time.perf_counter()
    for _ in range(steps):
        env.step(act())
    dt = time.perf_counter() - t
    return n_sample * steps / dt, dt


def reference_python_env(kind, n_sample, steps):
    """The reference ITSELF -- quadsim (numpy + numba) installed unmodified in
    baseline/_ref (`pip install --no-index --target baseline/_ref`) -- on a
    bounded sample of the same workload, timed beside the C port (the port
    is the reference arm; this shows how the port compares with the real
    thing).  numba's JIT compile (first render / query) is timed separately
    and excluded.  Returns None when baseline/_ref is absent."""
    import dataclasses

    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "quadsim")):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    import numba
    from quadsim.control import CTBR as RCTBR, LV as RLV
    from quadsim.env.config import EnvConfig as REnvConfig, SensorSpec as RSensorSpec
    from quadsim.env.tasks import make_env as rmake_env, navigation_config as rnav

    if kind == "c1":
        cfg = REnvConfig(num_agents=n_sample, command_type="ctbr", episode_max_steps=1000)
    elif kind == "c3":
        cfg = rnav(scene_seed=0, num_agents=n_sample)
        cfg = dataclasses.replace(cfg, sensors=cfg.sensors + (RSensorSpec(kind="segmentation", name="segmentation",
                                                                          width=64, height=64),))
    else:
        return None
    rng = np.random.default_rng(0)

    def act():
        if kind == "c1":
            return RCTBR(np.full(n_sample, 9.81), rng.normal(scale=0.5, size=(n_sample, 3)))
        return RLV(rng.normal(scale=1.5, size=(n_sample, 3)), rng.uniform(-3, 3, n_sample))

    t = time.perf_counter()
    env = rmake_env(cfg)
    env.reset(seed=0)
    env.step(act())  # numba JIT compile of the render / nearest-point kernels
    compile_s = time.perf_counter() - t
    env.step(act())
    t = time.perf_counter()
    for _ in range(steps):
        env.step(act())
    dt = time.perf_counter() - t
    return {"value": n_sample * steps / dt, "unit": "env-steps/s", "cores": int(numba.get_num_threads()),
            "kind": "reference (quadsim, numpy + numba, unmodified, baseline/_ref)",
            "sample": f"{n_sample} envs x {steps} steps ({dt:.1f} s; numba compile {compile_s:.1f} s excluded)",
            "threading_layer": str(numba.threading_layer()) if hasattr(numba, "threading_layer") else None}


def cpu_baseline_bptt(n_sample=8, T=64):
    """Oracle rollout_grad (dense 17x17 Jacobian chain, gradients.py:218-237)."""
    import oracle
    from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig

    P = oracle.pack_params(QuadParams(), SimConfig(), ControllerGains())
    rng = np.random.default_rng(0)
    x0 = np.zeros(17); x0[6] = 1.0; x0[13:] = P.hover_speed

    def loss(tr):
        g = np.zeros_like(tr)
        g[-1, 0:3] = 2 * (tr[-1, 0:3] - [1.0, 0, 2.0])
        return 0.0, g

    t = time.perf_counter()
    for _ in range(n_sample):
        oracle.rollout_grad(P, x0, 900 + rng.normal(scale=20, size=(T, 4)), loss)
    dt = time.perf_counter() - t
    return n_sample * T / dt, dt


def render_rooflines(kind, r, pk, steps):
    """K2's two roofline figures.  Primary: SM instruction issue, the bound
    the renderer actually has: warp-instructions per camera from
    the committed ncu capture x cameras / live kernel time, against 148 SMs x
    4 schedulers x the SM clock sampled under load.  Secondary: HBM, the
    algorithmic bytes (depth + seg writes, pose reads) / kernel time."""
    px = r["n"] * 64 * 64
    nbytes = px * sum(4 for s in r["cfg"].sensors) + r["n"] * 40
    gbs = nbytes / (r["render_ms"] / 1e3) / 1e9
    traffic, meta = profile_traffic("k_render_cull" if kind != "c5" else "k_render_f")
    hbm = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
           "traffic": traffic * r["n"] if traffic else None,
           "note": "K2 render: algorithmic bytes = depth+seg writes + pose reads; far below HBM by design"}
    mhz = (r["clocks"] or {}).get("sm_mhz") or 1965.0
    rays = px / (r["render_ms"] / 1e3)
    issue = None
    if meta and meta.get("warp_instructions_per_unit"):
        wips = meta["warp_instructions_per_unit"] * r["n"] / (r["render_ms"] / 1e3)
        peak_wi = 148 * 4 * mhz * 1e6
        ref_ops = 4360.0 if kind == "c5" else 1470.0
        issue = {"bound": "issue", "achieved": wips, "peak": peak_wi, "unit": "warp-instr/s", "frac": wips / peak_wi,
                 "traffic": traffic * r["n"] if traffic else None,
                 "kernel": "k_render_cull" if kind != "c5" else "k_render_f",
                 "kernel_ms": r["render_ms"], "step_ms": r["ms"] / steps, "rays_per_s": rays,
                 "warp_instr_per_camera": meta["warp_instructions_per_unit"],
                 "reference_ops_per_ray": ref_ops,
                 "reference_equiv_frac": rays * ref_ops / (148 * 128 * mhz * 1e6),
                 "ncu": {k: meta[k] for k in ("issue_active_pct", "warps_active_pct", "l1_hit_pct", "l2_hit_pct",
                                              "registers", "source") if k in meta},
                 "note": f"dominant kernel of the step ({r['render_ms']:.3f} of {r['ms'] / steps:.3f} ms); "
                         "peak = 148 SMs x 4 issue slots x the SM clock sampled in the timed region"}
    return issue, hbm


def env_line(kind, args, rank, world, pk, cpu=True, e2e=True):
    """Bench line body of one env workload (configs 1, 2, 3, 5, ...)."""
    r = run_env(args, rank, world, kind)
    value = r["total"] * args.steps / (r["ms"] / 1e3)
    line = {"value": value, "ms_per_step": r["ms"] / args.steps, "steps": args.steps, "clocks": r["clocks"],
            "gpu_launches": r["launches"],
            "config": {"workload": WORKLOADS[kind], "envs_per_gpu": r["n"], "global_envs": r["total"],
                       "resolution": "64x64", "integrator": "rk4, 2 substeps",
                       "sensors": ",".join(f"{s.name}:{s.kind}" for s in r["cfg"].sensors) or "none",
                       "l2": "per-step output (depth+seg, 2.1 GB at c3) >> 126 MB L2; no flush needed"
                       if not r["graph"] else "100 envs: latency-bound; 10 env steps per CUDA-graph replay "
                                              "(actions staged by device copies inside the timed region)",
                       "parallelism": f"env shards x{world}, no per-step collective"}}
    if "render_ms" in r:
        line["kernel_ms"] = {"env_step_k1k3": r["step_ms"], "render_k2": r["render_ms"]}
        if "observe_ms" in r:
            line["kernel_ms"]["observe_imu_noise"] = r["observe_ms"]
        issue, hbm = render_rooflines(kind, r, pk, args.steps)
        line["roofline"] = issue or hbm
        line["roofline_render_hbm"] = hbm
    elif r["graph"]:
        # latency-bound small batch: per-step device time of the whole graph-replayed step
        line["roofline"] = {"bound": "latency", "achieved": r["ms"] / args.steps * 1e3, "unit": "us/step",
                            "peak": None, "frac": None, "traffic": None,
                            "note": "100 envs = 100 warps on 148 SMs: one dependent chain of ~2.6k instructions "
                                    "per env-step; no throughput roofline applies (see roofline_env_step for K1+K3 "
                                    "at 4M envs)"}
    if e2e:
        line["e2e"] = run_e2e(r["cfg"], rank, world, kind)
        if kind == "c3" and r.get("env") is not None:
            line["e2e_obs_on_device"] = run_e2e_device_obs(r["env"], world, kind)
    if rank == 0 and cpu:
        ns = {"c5": 64, "c3n": 256, "swarm": 256}.get(kind, min(1024, ENVS[kind]))
        steps = {"c5": 2, "swarm": 4}.get(kind, 12 if ns > 100 else 400)
        v, dt = cpu_baseline_env(kind, n_sample=ns, steps=steps)
        line["cpu_baseline"] = {"value": v, "unit": "env-steps/s", "cores": os.cpu_count(), "kind": "port",
                                "sample": f"{ns} envs x {steps} steps of the same env step on the C oracle "
                                          f"(OpenMP), {dt:.1f} s"}
    line["_r"] = r
    return line


def bptt_line(args, rank, world, pk, cpu=True):
    r = run_bptt(args, rank, world)
    steps_total = r["n"] * r["T"] * world * args.steps
    line = {"metric": "BPTT env-steps/sec (forward + adjoint), whole box", "value": steps_total / (r["ms"] / 1e3),
            "ms_per_step": r["ms"] / args.steps, "steps": args.steps, "clocks": r["clocks"],
            "scaling": "strong" if args.strong else "weak", "gpu_launches": 3 * args.steps,
            "graph": "forward + loss + adjoint + env-sum captured as one CUDA graph per iteration",
            "config": {"workload": WORKLOADS["c4"], "envs_per_gpu": r["n"], "horizon": r["T"],
                       "parallelism": f"env shards x{world}, all_reduce(SUM) of loss + shared action grad"},
            "kernel_ms": {"rollout_forward": r["fwd_ms"], "rollout_backward": r["bwd_ms"]}}
    fwd_b, bwd_b = 152 + 68, 236  # algorithmic B/env-step (tape write, tape/action read, grad write)
    gbs = r["n"] * r["T"] * (fwd_b + bwd_b) / ((r["fwd_ms"] + r["bwd_ms"]) / 1e3) / 1e9
    hbm = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
           "traffic": None, "note": "forward+adjoint, (220+236) algorithmic B/env-step"}
    line["roofline"] = hbm
    _, meta = profile_traffic("k_rollout_bwd")
    if meta and meta.get("warp_instructions_per_unit"):
        mhz = (r["clocks"] or {}).get("sm_mhz") or 1965.0
        wips = meta["warp_instructions_per_unit"] * r["n"] * r["T"] / (r["bwd_ms"] / 1e3)
        line["roofline_adjoint_issue"] = {
            "bound": "issue", "achieved": wips, "peak": 148 * 4 * mhz * 1e6, "unit": "warp-instr/s",
            "frac": wips / (148 * 4 * mhz * 1e6), "kernel": "k_rollout_bwd",
            "note": "the adjoint recomputes each step's RK4 stages and runs the hand-derived VJP: "
                    f"{meta['warp_instructions_per_unit']:.0f} warp-instr/env-step (ncu) -- issue, not HBM, bounds it"}
    if rank == 0 and cpu:
        v, dt = cpu_baseline_bptt()
        line["cpu_baseline"] = {"value": v, "unit": "env-steps/s", "cores": 1, "kind": "port",
                                "sample": f"8 agents x H=64 oracle rollout_grad ({dt:.1f} s)"}
    return line


def parity_leg(line, kind):
    """Checker run after the timed region (never inside it): one more env
    step of the benchmark env through env.step, re-evaluated by the CPU
    oracle on the GPU's own pre/post-step states (oracle/parity.py): flags /
    nearest point / reward bit-exact, dynamics per north-star tolerance, a
    seeded 512-camera sample re-rendered (mismatch and grazing fractions)."""
    import torch

    from oracle.parity import env_step_parity, oracle_scenes
    from paper_2407_14783_b200.control import CTBR, LV
    from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig

    r = line["_r"]
    env, cfg = r["env"], r["cfg"]
    n = env.num_agents
    rng = np.random.default_rng(99)
    a = np.concatenate([rng.normal(scale=1.5, size=(n, 3)) + [1.0, 0, 0], rng.uniform(-np.pi, np.pi, (n, 1))], 1)
    cmd = LV(a[:, :3], a[:, 3]) if cfg.command_type == "lv" else CTBR(a[:, 0] + 9.81, a[:, 1:])
    if cfg.command_type != "lv":
        a = np.concatenate([a[:, :1] + 9.81, a[:, 1:]], 1)
    t = time.perf_counter()
    res = env.step(cmd)
    torch.cuda.synchronize()
    sample = np.sort(rng.choice(n, size=min(512, n), replace=False))
    rep = env_step_parity(env, cfg, res.observations, a, oracle_scenes(cfg), (QuadParams(), SimConfig(), ControllerGains()),
                          sample)
    keep = ("flags_equal", "flag_mismatches", "nearest_equal", "reward_equal", "state_err_max", "state_err_p99",
            "envs_over_1e-5", "over_1e-5_explained", "over_1e-5_unexplained", "render")
    out = {k: rep[k] for k in keep if k in rep}
    out["envs"] = n
    out["checker"] = "CPU oracle (oracle/parity.py) on the GPU's own states, one extra untimed step"
    out["seconds"] = time.perf_counter() - t
    return out


def sustained_leg(args, rank, world, line, seconds=5.0):
    """>= 5 s of steady-state device-timed steps with the clock
    sampler running: the long-run value beside the short headline window."""
    import torch

    import paper_2407_14783_b200._native as nat

    r = line["_r"]
    env = r["env"]
    K = max(10, int(math.ceil(seconds * 1e3 / max(line["ms_per_step"], 1e-3))))
    a = make_actions("c3", env.num_agents, 8, rank)

    def launch(i):
        env._bufs.action = a[i % 8].data_ptr()
        nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))
        env._render()
        env._observe()

    torch.cuda.synchronize()
    barrier(world)
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")) if not SHARE_GPU else 0)
    clk.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for i in range(K):
        launch(i)
    t1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = max_over_ranks(t0.elapsed_time(t1), world)
    return {"value": r["total"] * K / (ms / 1e3), "unit": "env-steps/s", "steps": K, "seconds": ms / 1e3,
            "ms_per_step": ms / K, "clocks": clocks}


def sub_args(args, kind, steps):
    ns = argparse.Namespace(**vars(args))
    ns.workload, ns.steps, ns.warmup = kind, steps, max(args.warmup, 3)
    return ns


def strip(d):
    return {k: v for k, v in d.items() if not k.startswith("_")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-sub", dest="sub", action="store_false",
                    help="config 3 only: skip the config 1/2/4/5 sub-records, the parity and the sustained legs")
    ap.add_argument("--strong", action="store_true", help="c4: fixed 16384 envs in total (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    kind = args.workload

    if args.impl == "reference":
        return reference_arm(args, kind)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)

    import torch

    rank, world, local = dist_setup()
    pk, pk_kind = peaks()
    line = {"metric": METRIC, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (procedurally generated scenes, seeded actions); no datasets offline",
            "peaks_source": pk_kind}
    if kind == "c4":
        line.update(bptt_line(args, rank, world, pk, cpu=args.cpu))
    else:
        body = env_line(kind, args, rank, world, pk, cpu=args.cpu, e2e=args.e2e)
        line.update(body)
        line["steps"] = args.steps
        if rank == 0:
            line["roofline_dynamics"] = run_dynamics_roofline(pk)
            line["roofline_env_step"] = run_env_step_roofline(pk)
        if kind == "c3" and args.sub:
            line["sustained"] = sustained_leg(args, rank, world, body)
            if rank == 0:
                line["parity"] = parity_leg(body, kind)
                if args.cpu and "cpu_baseline" in line:
                    try:
                        rp = reference_python_env("c3", 256, 2)
                    except Exception as e:  # the reference's own stack is optional here; the port is the baseline
                        rp = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
                    if rp:
                        line["cpu_baseline"]["reference_python"] = rp
    if kind == "c3" and args.sub:
        # every other BASELINE config as a sub-record (same contract keys), so the
        # driver's default run carries each config's number, e2e and CPU baseline
        del body["_r"]["env"]
        body["_r"] = None
        torch.cuda.empty_cache()
        subs = {}
        for sk, st in (("c1", 200), ("c2", 100), ("c5", 10)):
            sl = env_line(sk, sub_args(args, sk, st), rank, world, pk, cpu=args.cpu, e2e=args.e2e)
            sl["_r"] = None
            if sk == "c1" and rank == 0 and args.cpu and "cpu_baseline" in sl:
                try:
                    rp = reference_python_env("c1", 100, 300)
                except Exception as e:
                    rp = {"unavailable": f"{type(e).__name__}: {e}"[:200]}
                if rp:
                    sl["cpu_baseline"]["reference_python"] = rp
            subs[sk] = strip(sl)
            torch.cuda.empty_cache()
        subs["c4"] = bptt_line(sub_args(args, "c4", 10), rank, world, pk, cpu=args.cpu)
        line["configs"] = subs
    if rank == 0:
        print(json.dumps(strip(line)), flush=True)
    barrier(world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: re-run this script under
    torch.distributed.run with one rank per GPU (rendezvous on 127.0.0.1);
    rank 0 prints the JSON line."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n and not SHARE_GPU:
        raise SystemExit(f"--gpus {n}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, check=False).returncode


def reference_arm(args, kind):
    """--impl reference: the reference's algorithm on the host cores (the C
    oracle restatement -- the Python reference cannot be compiled and does
    not travel to the GPU box), same metric/config, each step a bounded
    sample.  Under torchrun only rank 0 runs."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if kind == "c4":
        vals = [cpu_baseline_bptt(n_sample=2)[0] for _ in range(max(1, min(args.steps, 5)))]
        unit, sample = "env-steps/s", "2 agents x H=64 oracle rollout_grad per step"
        metric = "BPTT env-steps/sec (forward + adjoint), whole box"
    else:
        vals = []
        ns = min({"c5": 64, "swarm": 256}.get(kind, 512), ENVS[kind])  # never more envs than the config has
        st = 2 if ns > 100 else 40  # small configs: enough steps for a measurable sample
        for _ in range(max(1, min(args.steps, 5))):
            vals.append(cpu_baseline_env(kind, n_sample=ns, steps=st)[0])
        unit, sample, metric = "env-steps/s", f"{ns} envs x {st} steps per step (C oracle, OpenMP)", METRIC
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": metric, "value": v, "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "config": {"workload": WORKLOADS[kind]},
            "cpu_baseline": {"value": v, "unit": unit, "cores": os.cpu_count(), "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    sys.exit(main() or 0)
