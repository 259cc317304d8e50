"""Benchmark of the VisFly/quadsim hot path on B200 (BASELINE.json metric:
env-steps/s and 64x64 depth frames/s, whole box, vs the CPU reference).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c2|c1|dyn|c5] [--impl ours|reference]

Default workload = BASELINE config 3 (the largest single-GPU config):
navigation, 65,536 envs per GPU, 64x64 depth + segmentation from one camera,
LV actions, full env.step (auto-reset, controller, RK4 dynamics, proximity,
reward, termination, render).  One env-step renders one 64x64 depth frame,
so env-steps/s == depth frames/s.  Multi-GPU (torchrun): envs sharded by
global index, no per-step collective ("scaling": "weak"), time = max over
ranks of CUDA-event time, value = all ranks' env-steps / that time.

Prints one JSON line (rank 0).  Extra keys: roofline (dominant kernel),
roofline_dynamics (K1 at HBM-relevant size), cpu_baseline (oracle on the
host cores), e2e (public API with host buffers), clocks, gpu_launches.
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

WORKLOADS = {
    "c3": dict(desc="navigation, 64x64 depth+segmentation, 65536 envs/GPU (BASELINE config 3)", envs=65536, seg=True),
    "c2": dict(desc="navigation, 64x64 depth, 100 envs (BASELINE config 2)", envs=100, seg=False),
    "c1": dict(desc="hover free flight, dynamics only, 100 envs (BASELINE config 1)", envs=100),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.samples, self.index, self._stop, self._t = [], index, threading.Event(), None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append(out.split(","))
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].strip().replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].strip().replace(".", "").isdigit()]
        reasons = set()
        bits = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}
        for s in self.samples:
            try:
                v = int(s[2].strip(), 16)
            except Exception:
                continue
            for b, name in bits.items():
                if v & b:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
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

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def l2_flush_buffer():
    import torch

    return torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


# ----------------------------------------------------------------------------
# our implementation


def bench_env(args, rank, world):
    import torch

    from paper_2407_14783_b200.control import LV
    from paper_2407_14783_b200.env import make_env, navigation_config

    wl = WORKLOADS[args.workload]
    n_per = wl["envs"]
    total = n_per * world
    cfg = navigation_config(scene_seed=0, num_agents=total, with_segmentation=wl.get("seg", False))
    env = make_env(cfg, shard=(rank, world))
    env.reset(seed=args.seed)
    n = env.num_agents
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    K, W = args.steps, args.warmup
    acts = torch.empty((K + W, n, 4), device="cuda")
    acts[..., :3] = torch.randn((K + W, n, 3), device="cuda", generator=g) * 1.5
    acts[..., 0] += 1.0
    acts[..., 3] = (torch.rand((K + W, n), device="cuda", generator=g) * 2 - 1) * math.pi
    cmds = [LV(acts[i, :, :3], acts[i, :, 3]) for i in range(K + W)]
    # pre-stage contiguous action tensors so the timed loop only launches
    staged = [acts[i].contiguous() for i in range(K + W)]

    def one(i):
        env._bufs.action = staged[i].data_ptr()
        env._launch_step()

    for i in range(W):
        one(i)
    torch.cuda.synchronize()
    # per-kernel timing inside the timed region (events on the launching stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    import paper_2407_14783_b200._native as nat
    from paper_2407_14783_b200.sensing import render_state

    barrier(world)
    torch.cuda.synchronize()
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for k in range(K):
        e0, e1, e2 = ev[k]
        env._bufs.action = staged[W + k].data_ptr()
        e0.record()
        nat.check(nat.lib().qb_env_step(env._P, env._kind, env._task, env.dev_scenes.handle, env._bufs, nat.stream_of()))
        e1.record()
        for slot in env._cams.values():
            render_state(env.dev_scenes, slot["camera"], env._planes, env_scene=env.agent_scene, depth=slot["depth"],
                         seg=slot["seg"])
        e2.record()
    t1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = t0.elapsed_time(t1)
    step_ms = [a.elapsed_time(b) for a, b, _ in ev]
    render_ms = [b.elapsed_time(c) for _, b, c in ev]
    ms = max_over_ranks(ms, world)
    launches = K * (1 + len(env._cams))
    # e2e: public API, host (pinned) actions in, observations + reward/flags out
    e2e = bench_e2e(env, cmds, args, world) if args.e2e else None
    return dict(env=env, n=n, total=total, ms=ms, step_ms=step_ms, render_ms=render_ms, clocks=clocks, launches=launches,
                e2e=e2e, cfg=cfg)


def bench_e2e(env, cmds, args, world):
    import torch

    from paper_2407_14783_b200.control import LV

    n = env.num_agents
    K = max(3, min(args.steps, 10))
    rng = np.random.default_rng(0)
    host_actions = [np.ascontiguousarray(np.concatenate([rng.normal(size=(n, 3)), rng.uniform(-3, 3, (n, 1))], 1),
                                         dtype=np.float32) for _ in range(K + 1)]
    obs_keys = [k for k in ("state", "depth", "segmentation") if k in env.get_observation().keys()]
    outs = {}

    def one(a):
        r = env.step(LV(a[:, :3], a[:, 3]))
        o = r.observations
        h2d = a.nbytes
        d2h = 0
        for k in obs_keys:
            t = o[k]
            if k not in outs:
                outs[k] = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            outs[k].copy_(t, non_blocking=True)
            d2h += t.numel() * t.element_size()
        for name, t in (("reward", r.reward), ("terminated", r.terminated), ("truncated", r.truncated)):
            if name not in outs:
                outs[name] = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            outs[name].copy_(t, non_blocking=True)
            d2h += t.numel() * t.element_size()
        torch.cuda.current_stream().synchronize()
        return h2d, d2h

    one(host_actions[0])
    barrier(world)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(K):
        h2d, d2h = one(host_actions[k + 1])
    dt = time.perf_counter() - t
    dt = max_over_ranks(dt, world)
    return {"value": n * world * K / dt, "unit": "env-steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": K}


def bench_dynamics(n, steps, warmup, rank):
    """K1 alone at an HBM-relevant size: 152 B/env-step algorithmic traffic."""
    import torch

    import paper_2407_14783_b200._native as nat
    from paper_2407_14783_b200.params import native_params

    P = native_params()
    pl = torch.zeros((17, n), device="cuda")
    pl[0:3] = torch.rand((3, n), device="cuda")
    pl[6] = 1.0
    pl[13:17] = 900.0
    act = torch.empty((n, 4), device="cuda")
    act[:, 0] = 9.81
    act[:, 1:] = torch.randn((n, 3), device="cuda") * 0.3
    flush = l2_flush_buffer()

    def launch():
        nat.check(nat.lib().qb_dynamics_step(P, nat.CMD["ctbr"], nat.QB_F32, n, n, nat.ptr(pl), nat.ptr(act), None, None,
                                             nat.stream_of()))

    for _ in range(warmup):
        launch()
    times = []
    for _ in range(steps):
        flush.zero_()  # evict L2 between launches
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch()
        b.record()
        times.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in times]))
    return n, ms


def cpu_baseline_env(cfg_total, n_sample=64, steps=3):
    """Oracle (C restatement, OpenMP on all host cores) on a bounded sample of
    the same navigation workload: env-steps/s."""
    import dataclasses

    import oracle
    from oracle.env import OracleEnv
    from paper_2407_14783_b200.env import navigation_config
    from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig

    cfg = navigation_config(scene_seed=0, num_agents=n_sample, with_segmentation=True)
    sc = cfg.scenes[0].materialize().arrays
    osc = oracle.OracleScene(sc.prim_type, sc.prim_data, sc.prim_object_id, sc.prim_aabb_lo, sc.prim_aabb_hi)
    env = OracleEnv(cfg, [osc], QuadParams(), SimConfig(), ControllerGains())
    env.reset(seed=0)
    rng = np.random.default_rng(0)
    acts = [np.concatenate([rng.normal(scale=1.5, size=(n_sample, 3)), rng.uniform(-3, 3, (n_sample, 1))], 1)
            for _ in range(steps + 1)]
    env.step(acts[0])
    t = time.perf_counter()
    for k in range(steps):
        env.step(acts[k + 1])
    dt = time.perf_counter() - t
    return n_sample * steps / dt, dt


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
    ap.add_argument("--dyn-n", type=int, default=1 << 24)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    import torch

    rank, world, local = dist_setup(args)
    pk, pk_kind = peaks()
    wl = WORKLOADS[args.workload]
    metric = "env-steps/sec (= 64x64 depth frames/sec), whole box"

    if args.impl == "reference":
        if rank == 0:
            v, dt = cpu_baseline_env(wl["envs"], n_sample=64, steps=max(1, min(args.steps, 4)))
            line = {"impl": "reference", "metric": metric, "value": v, "unit": "env-steps/s", "n_gpus": world,
                    "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                    "config": {"workload": wl["desc"]},
                    "cpu_baseline": {"value": v, "unit": "env-steps/s", "cores": os.cpu_count(), "kind": "port",
                                     "sample": "64 navigation envs (depth+seg), oracle C port with OpenMP"},
                    "e2e": {"value": v, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        return

    res = bench_env(args, rank, world)
    K = args.steps
    value = res["total"] * K / (res["ms"] / 1e3)
    # dominant kernel = K2 render: algorithmic ops/ray from the reference BVH counts
    r_ms = float(np.mean(res["render_ms"]))
    s_ms = float(np.mean(res["step_ms"]))
    rays = res["n"] * 64 * 64
    ops_per_ray = 1470.0
    achieved_ops = rays * ops_per_ray / (r_ms / 1e3)
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    peak_ops = 148 * 128 * sm_mhz * 1e6
    out_bytes = rays * (4 + (4 if wl.get("seg") else 0))
    line = {
        "metric": metric, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": res["ms"] / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (procedural cluttered room, seeded LV actions)",
        "config": {"workload": wl["desc"], "envs_per_gpu": res["n"], "global_envs": res["total"], "resolution": "64x64",
                   "sensors": "depth+segmentation" if wl.get("seg") else "depth", "integrator": "rk4 x2 substeps",
                   "l2": "per-step working set (2.1 GB of depth+seg output) >> 126 MB L2",
                   "parallelism": f"env shards x{world}, no per-step collective"},
        "kernel_ms": {"env_step_k1k3": s_ms, "render_k2": r_ms},
        "roofline": {"bound": "fp32_issue", "achieved": achieved_ops / 1e9, "peak": peak_ops / 1e9, "unit": "Gop/s",
                     "frac": achieved_ops / peak_ops, "traffic": None,
                     "note": f"K2 render: {ops_per_ray:.0f} algorithmic FP32 ops/ray (reference-BVH count, SURVEY 8-D) x "
                             f"{rays} rays per launch / launch time; peak = 148 SMs x 128 lanes x {sm_mhz:.0f} MHz "
                             f"({pk_kind}); HBM view: {out_bytes / (r_ms / 1e3) / 1e9:.1f} GB/s of "
                             f"{pk.get('hbm_gbs')} GB/s"},
        "clocks": res["clocks"], "gpu_launches": res["launches"],
    }
    if rank == 0:
        n_dyn, ms_dyn = bench_dynamics(args.dyn_n, 10, 3, rank)
        gbs = n_dyn * 152 / (ms_dyn / 1e3) / 1e9
        line["roofline_dynamics"] = {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                     "frac": gbs / pk["hbm_gbs"], "traffic": None, "envs": n_dyn, "ms": ms_dyn,
                                     "env_steps_per_sec": n_dyn / (ms_dyn / 1e3),
                                     "note": "K1 CTBR RK4x2, 152 B/env-step (read 17+4 floats, write 17), L2 flushed"}
        if res["e2e"]:
            line["e2e"] = res["e2e"]
        if args.cpu:
            v, dt = cpu_baseline_env(res["total"])
            line["cpu_baseline"] = {"value": v, "unit": "env-steps/s", "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"64 navigation envs x 3 steps (depth+seg), {dt:.1f} s of CPU work"}
        print(json.dumps(line), flush=True)
    barrier(world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
