"""Memory / race checks without compute-sanitizer (closed on the GPU pool).

Run with the checked build (QB_LIB_PATH=scripts/_dbg/checks.so, built with
-DQB_CHECKS by scripts/gpu_checks.sh): the kernels' own bounds assertions
(csrc/qb_checks.cuh) print "QB_CHECK FAILED" lines; this script adds

  coverage     (initcheck's question) every output element of every step is
               written: the env's next observation buffers and per-step output
               block are poisoned with sentinels (NaN, -7, 0xAB) before each
               step and must hold none after it -- depth, segmentation, noisy
               observations, IMU, centroids, flags, reward, nearest points --
               for each kernel family and launch shape; the poisoned instance
               must also equal an unpoisoned twin (no stale reads)
  determinism  (racecheck's symptom) two env instances stepped with the same
               seed and actions agree bit for bit at every step; a camera set
               rendered alone (split > 1: several warps per camera) and inside
               a large batch (split == 1: several cameras per warp, shared
               lists reused) gives bit-identical frames
  adjoint      the split (two-warp, shared-memory exchange) adjoint is bitwise
               reproducible and equals itself under a different batch size

Prints one summary line per check and exits 1 on any failure."""

import dataclasses
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2407_14783_b200 import gradients as G  # noqa: E402
from paper_2407_14783_b200.control import CTBR, LV  # noqa: E402
from paper_2407_14783_b200.env import (EnvConfig, SensorSpec, gap_crossing_config, landing_config,  # noqa: E402
                                       make_env, navigation_config)
from paper_2407_14783_b200.params import native_params  # noqa: E402
from paper_2407_14783_b200.sensing import NoiseSpec, render_frames  # noqa: E402

failures = []


def check(ok, what):
    print(("ok   " if ok else "FAIL ") + what, flush=True)
    if not ok:
        failures.append(what)


def configs():
    nav = dataclasses.replace(navigation_config(0, 64, with_segmentation=True), episode_max_steps=6)
    mesh = dataclasses.replace(nav, scenes=(dataclasses.replace(nav.scenes[0], kind="cluttered_mesh"),))
    noisy = dataclasses.replace(nav, sensors=(
        SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("normal", sigma=0.02), NoiseSpec("redwood", sigma_disparity=0.002))),
        SensorSpec(kind="segmentation", name="seg", noise=(NoiseSpec("saltpepper", p=0.02),)),
        SensorSpec(kind="imu", name="imu", noise=(NoiseSpec("normal", sigma=0.05),))))
    pois = dataclasses.replace(nav, sensors=(SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("poisson", scaling=50.0),)),))
    return {
        "nav64": nav, "nav10000": dataclasses.replace(nav, num_agents=10000), "mesh64": mesh,
        "landing64": dataclasses.replace(landing_config(64), episode_max_steps=5),
        "landing4000": dataclasses.replace(landing_config(4000), episode_max_steps=5),
        "garage40": EnvConfig(num_agents=40, command_type="ctbr", episode_max_steps=5),
        "garage10000": EnvConfig(num_agents=10000, command_type="ctbr", episode_max_steps=5),
        "swarm6": dataclasses.replace(gap_crossing_config(num_agents=6), episode_max_steps=8),
        "noisy64": noisy, "poisson64": pois,
    }


def actions(cfg, n, g):
    if cfg.command_type == "ctbr":
        return CTBR(torch.rand(n, device="cuda", generator=g) * 10 + 5, torch.randn(n, 3, device="cuda", generator=g))
    return LV(torch.randn(n, 3, device="cuda", generator=g) * 2.0, torch.randn(n, device="cuda", generator=g))


def poison(env):
    """Sentinels in every buffer the next step must write."""
    nxt = env._obs_i ^ 1
    for slot in env._cams.values():
        for k in ("depth", "seg", "centroid"):
            pair = slot.get(k + "_pair")
            if pair:
                t = pair[nxt]
                t.fill_(-7) if t.dtype == torch.int32 else t.fill_(float("nan"))
    for o in env._obs_sensors:
        o["outs"][nxt].fill_(float("nan"))
    if env._swarm_obs is not None:
        env._swarm_obs_pair[nxt].fill_(float("nan"))
    # per-step outputs of the output block (needs_respawn, step counts and scene
    # indices carry state into the next step and are left alone)
    for t in (env._terminated, env._truncated, env._success, env._collision, env._oob, env._nonfinite):
        t.fill_(0xAB)
    env._reward.fill_(float("nan"))
    env.nearest_dist.fill_(float("nan"))
    env.nearest_pt.fill_(float("nan"))


def unwritten(env, res):
    bad = {}
    for k, v in res.observations.items():
        t = v
        if t.dtype == torch.int32:
            bad[k] = int((t == -7).sum())
        else:
            bad[k] = int(torch.isnan(t).sum())
    flags = env._flags
    bad["flags"] = int((flags > 1).sum())
    bad["reward"] = int(torch.isnan(env._reward).sum())
    bad["nearest"] = int(torch.isnan(env.nearest_dist).sum() + torch.isnan(env.nearest_pt).sum())
    bad["step"] = int((env.step_counts < 0).sum())
    return {k: v for k, v in bad.items() if v}


def coverage_and_determinism(name, cfg, steps=6):
    a, b = make_env(cfg), make_env(cfg)
    a.reset(seed=3)
    b.reset(seed=3)
    ga = torch.Generator(device="cuda").manual_seed(5)
    gb = torch.Generator(device="cuda").manual_seed(5)
    n = a.num_agents
    holes, diffs = {}, []
    for t in range(steps):
        poison(a)
        ra, rb = a.step(actions(cfg, n, ga)), b.step(actions(cfg, n, gb))
        torch.cuda.synchronize()
        for k, v in unwritten(a, ra).items():
            holes[k] = holes.get(k, 0) + v
        for k in ra.observations.keys():
            x, y = ra.observations[k], rb.observations[k]
            if not torch.equal(torch.nan_to_num(x.float(), nan=-1.0), torch.nan_to_num(y.float(), nan=-1.0)):
                diffs.append((t, k))
        if not (torch.equal(a._planes, b._planes) and torch.equal(a._flags, b._flags) and torch.equal(a._reward, b._reward)):
            diffs.append((t, "state/flags"))
    check(not holes, f"coverage {name}: every output written {holes or ''}")
    check(not diffs, f"determinism {name}: two instances bit-identical {diffs[:4] or ''}")


def render_split_vs_batch():
    """37 cameras alone (split > 1) vs inside 8192 (split == 1): identical frames."""
    rng = np.random.default_rng(0)
    for name, kind in (("nav", "cluttered"), ("mesh", "cluttered_mesh")):
        cfg = navigation_config(0, 8192, with_segmentation=True)
        cfg = dataclasses.replace(cfg, scenes=(dataclasses.replace(cfg.scenes[0], kind=kind),))
        env = make_env(cfg)
        cam = cfg.sensors[0].camera()
        n = 8192
        o = torch.as_tensor(rng.uniform([-4.5, -4.5, 0.3], [4.5, 4.5, 3.7], (n, 3)), device="cuda")
        q = rng.normal(size=(n, 4))
        q = torch.as_tensor(q / np.linalg.norm(q, axis=1, keepdims=True), device="cuda")
        d1, s1 = render_frames(env.dev_scenes, o, q, cam)
        idx = torch.as_tensor(np.sort(rng.choice(n, 37, replace=False)), device="cuda")
        d2, s2 = render_frames(env.dev_scenes, o[idx].contiguous(), q[idx].contiguous(), cam)
        torch.cuda.synchronize()
        check(torch.equal(d1[idx], d2) and torch.equal(s1[idx], s2), f"render {name}: 37 cameras alone == inside 8192")


def adjoint_repro():
    P = native_params()
    for n in (1000, 4096):
        T = 12
        g = torch.Generator(device="cuda").manual_seed(1)
        init = torch.zeros((17, n), device="cuda")
        init[6] = 1.0
        init[13:] = 900.0
        init[0:3] = torch.rand((3, n), device="cuda", generator=g)
        acts = 900 + torch.randn((T, n, 4), device="cuda", generator=g) * 20
        tape, _ = G.rollout_planes(P, "rotor", init, acts)
        gt = torch.randn(tape.shape, device="cuda", generator=g)
        r1 = G.backward_planes(P, "rotor", tape, acts, gt)
        r2 = G.backward_planes(P, "rotor", tape, acts, gt)
        sub = 333  # the first 333 envs as their own batch
        r3 = G.backward_planes(P, "rotor", tape[:, :, :sub].contiguous(), acts[:, :sub].contiguous(),
                               gt[:, :, :sub].contiguous())
        torch.cuda.synchronize()
        same = torch.equal(r1[0], r2[0]) and torch.equal(r1[1], r2[1])
        sub_ok = torch.equal(r1[0][:, :sub], r3[0]) and torch.equal(r1[1][:, :sub], r3[1])
        check(same and sub_ok, f"adjoint n={n}: reproducible run to run and per env independent of the batch")


if __name__ == "__main__":
    for name, cfg in configs().items():
        coverage_and_determinism(name, cfg)
    render_split_vs_batch()
    adjoint_repro()
    print(f"checks: {len(failures)} failed", flush=True)
    sys.exit(1 if failures else 0)
