"""One small case of every kernel family of libquadb200.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck; run by
scripts/gpu_sanitize.sh).  Sizes are chosen to hit every launch shape the
benchmarks use: warp-per-env and thread-per-env K3 (n above the warp
threshold), the culling renderer with split > 1 and split == 1, the BVH
packet renderer, the FP64 validation kernels, the observation pass (warp and
thread-per-env Poisson chains), swarm mode, the device scene build, the
adjoint with the env-sum, the bindings' pack / narrow kernels."""

import dataclasses
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_14783_b200 import bindings, gradients as G  # noqa: E402
from paper_2407_14783_b200.control import CTBR, LV  # noqa: E402
from paper_2407_14783_b200.env import (EnvConfig, SceneSpec, SensorSpec, gap_crossing_config, landing_config,  # noqa: E402
                                       make_env, navigation_config)
from paper_2407_14783_b200.geometry import queries  # noqa: E402
from paper_2407_14783_b200.geometry.device import DeviceScenes  # noqa: E402
from paper_2407_14783_b200.params import native_params  # noqa: E402
from paper_2407_14783_b200.sensing import NoiseSpec  # noqa: E402

rng = np.random.default_rng(0)


def lv(n):
    return LV(torch.randn(n, 3, device="cuda") * 2.0, torch.randn(n, device="cuda"))


def episode(cfg, steps, n_big=None, dtype=None, **kw):
    env = make_env(cfg, dtype=dtype, **kw) if dtype is not None else make_env(cfg, **kw)
    env.reset(seed=1)
    n = env.num_agents
    for _ in range(steps):
        if cfg.command_type == "ctbr":
            env.step(CTBR(torch.rand(n, device="cuda") * 10 + 5, torch.randn(n, 3, device="cuda")))
        else:
            env.step(lv(n))
    torch.cuda.synchronize()
    print(f"  {cfg.task} n={n} {dtype or 'f32'} ok", flush=True)


def main(which):
    nav = dataclasses.replace(navigation_config(0, 64, with_segmentation=True), episode_max_steps=6)
    if "env" in which:
        episode(nav, 8)                                               # warp-per-env K3 + split step + cull split>1
        episode(dataclasses.replace(nav, num_agents=10000), 3)        # thread-per-env K3 + cull split==1
        episode(nav, 4, dtype=torch.float64)                          # FP64 validation build (k_render_x)
        mesh = dataclasses.replace(nav, scenes=(dataclasses.replace(nav.scenes[0], kind="cluttered_mesh"),))
        episode(mesh, 4)                                              # BVH packet renderer (k_render_f)
        episode(dataclasses.replace(landing_config(64), episode_max_steps=5), 6)          # centroid pass
        episode(dataclasses.replace(landing_config(4000), episode_max_steps=5), 2)        # inline centroid
        episode(EnvConfig(num_agents=40, command_type="ctbr", episode_max_steps=5), 8)    # garage, warp scan
        episode(EnvConfig(num_agents=10000, command_type="ctbr", episode_max_steps=5), 3)  # nearest_point_scan
        episode(dataclasses.replace(gap_crossing_config(num_agents=6), episode_max_steps=8), 10)  # swarm
        noisy = dataclasses.replace(nav, sensors=(
            SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("normal", sigma=0.02),
                                                          NoiseSpec("redwood", sigma_disparity=0.002))),
            SensorSpec(kind="segmentation", name="seg", noise=(NoiseSpec("saltpepper", p=0.02),)),
            SensorSpec(kind="imu", name="imu", noise=(NoiseSpec("normal", sigma=0.05),))))
        episode(noisy, 3)                                             # warp-per-env observation pass
        pois = dataclasses.replace(nav, sensors=(
            SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("poisson", scaling=50.0),)),))
        episode(pois, 2)                                              # thread-per-env observation pass
        episode(mesh, 2, scene_build="device")                        # device scene build (LBVH)
    if "grad" in which:
        P = native_params()
        for kind in ("rotor", "ctbr", "srt"):
            n, T = 37, 5
            init = torch.zeros((17, n), device="cuda")
            init[6] = 1.0
            init[13:] = 900.0
            init[0:3] = torch.rand((3, n), device="cuda")
            if kind == "rotor":
                acts = 900 + torch.randn((T, n, 4), device="cuda") * 20
            elif kind == "ctbr":
                acts = torch.cat([torch.rand((T, n, 1), device="cuda") * 10 + 5, torch.randn((T, n, 3), device="cuda")], 2)
            else:
                acts = torch.rand((T, n, 4), device="cuda") * 3
            tape, _ = G.rollout_planes(P, kind, init, acts)
            gsum = torch.zeros(T * 4, dtype=torch.float64, device="cuda")
            G.backward_planes(P, kind, tape, acts, torch.randn_like(tape), action_grad_sum=gsum)
            G.step_vjp(P, kind, init, acts[0], torch.randn_like(init))
        torch.cuda.synchronize()
        print("  gradients ok", flush=True)
    if "query" in which:
        sc = nav.scenes[0].materialize()
        dev = DeviceScenes([sc])
        q = rng.uniform(-5, 5, (300, 3))
        queries.nearest_points(dev, q)
        d = rng.normal(size=(300, 3))
        queries.raycasts(dev, q, d / np.linalg.norm(d, axis=1, keepdims=True), 10.0)
        print("  queries ok", flush=True)
    if "bindings" in which:
        h = bindings.make_env(nav)
        out = h.outputs()
        bindings.reset(h, 2, out=out)
        a = np.concatenate([rng.normal(size=(64, 3)), rng.uniform(-3, 3, (64, 1))], 1).astype(np.float32)
        for _ in range(3):
            bindings.step(h, a, out=out)
            bindings.step(h, a)
        print("  bindings ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["env", "grad", "query", "bindings"])
