"""Generate golden fixtures by RUNNING THE REFERENCE (quadsim, numpy/numba).

Run in the build container, where the read-only reference lives:

    python tests/golden/make_golden.py [/root/reference/pkg/src]

The .npz files it writes are committed; the GPU box never sees the
reference.  numpy Generator streams are not guaranteed stable across numpy
versions, so every random input is stored in the fixture itself.  Generated
with numpy 2.3.5 / numba 0.65.0.
"""

from __future__ import annotations

import dataclasses
import math
import os
import sys

import numpy as np

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import quadsim  # noqa: E402
from quadsim import control as ctl  # noqa: E402
from quadsim import dynamics as dyn  # noqa: E402
from quadsim import gradients as grd  # noqa: E402
from quadsim import sensing  # noqa: E402
from quadsim.env import tasks  # noqa: E402
from quadsim.env.config import DistSpec, EnvConfig, InitRandomization, SceneSpec, SensorSpec  # noqa: E402
from quadsim.geometry import generate, queries, shapes  # noqa: E402
from quadsim.params import ControllerGains, QuadParams, SimConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_states(rng, n, params):
    """SURVEY.md 8-D C1 parity set."""
    p = rng.uniform(-3, 3, (n, 3))
    v = rng.normal(size=(n, 3))
    q = rng.normal(size=(n, 4)) + np.array([3.0, 0, 0, 0])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    o = rng.normal(size=(n, 3))
    w = rng.uniform(600, 1200, (n, 4))
    return np.concatenate([p, v, q, o, w], axis=1)


def random_cmd(rng, kind, n):
    if kind == "ctbr":
        return np.concatenate([rng.uniform(5, 15, (n, 1)), rng.normal(size=(n, 3))], axis=1)
    if kind == "srt":
        return rng.uniform(0.5, 3.5, (n, 4))
    if kind == "lv":
        return np.concatenate([rng.normal(scale=2.0, size=(n, 3)), rng.uniform(-np.pi, np.pi, (n, 1))], axis=1)
    if kind == "ps":
        return np.concatenate([rng.uniform(-4, 4, (n, 3)), rng.uniform(-np.pi, np.pi, (n, 1))], axis=1)
    if kind == "rotor":
        return rng.uniform(0, 1600, (n, 4))
    raise ValueError(kind)


def scene_arrays(scene):
    a = scene.arrays
    return dict(prim_type=a.prim_type, prim_data=a.prim_data, prim_oid=a.prim_object_id, prim_lo=a.prim_aabb_lo,
                prim_hi=a.prim_aabb_hi, node_lo=a.node_lo, node_hi=a.node_hi, node_first=a.node_first,
                node_count=a.node_count, prim_order=a.prim_order)


def gen_dynamics():
    rng = np.random.default_rng(20240717)
    params, gains = QuadParams(), ControllerGains()
    out = {}
    n = 256
    x0 = random_states(rng, n, params)
    out["state0"] = x0
    st = dyn.QuadState.from_vector(x0)
    for kind in ("srt", "ctbr", "ps", "lv", "rotor"):
        cmd = random_cmd(rng, kind, n)
        out[f"{kind}_cmd"] = cmd
        if kind == "rotor":
            speeds = cmd
        else:
            speeds = ctl.command_to_rotor_speeds(ctl.command_from_array(kind, cmd), st, gains, params)
        out[f"{kind}_speeds"] = speeds
        for integ, sub in (("rk4", 2), ("euler", 4), ("rk4", 1)):
            sim = SimConfig(integrator=integ, substeps=sub)
            nxt = dyn.step(st.copy(), speeds, sim, params)
            out[f"{kind}_{integ}{sub}_next"] = nxt.as_vector()
    # closed-loop trajectories: 16 envs x 100 steps, fresh command every step
    m, T = 16, 100
    for kind in ("ctbr", "lv", "ps", "srt"):
        sim = SimConfig()
        x = x0[:m].copy()
        x[:, 0:3] = rng.uniform(-1, 1, (m, 3))
        x[:, 3:6] *= 0.3
        x[:, 10:13] *= 0.3
        cmds = np.empty((T, m, 4))
        traj = np.empty((T + 1, m, 17))
        traj[0] = x
        s = dyn.QuadState.from_vector(x)
        for t in range(T):
            c = random_cmd(rng, kind, m)
            if kind == "ctbr":
                c[:, 0] = rng.uniform(8.5, 11.0, m)
                c[:, 1:4] *= 0.5
            cmds[t] = c
            sp = ctl.command_to_rotor_speeds(ctl.command_from_array(kind, c), s, gains, params)
            s = dyn.step(s, sp, sim, params)
            traj[t + 1] = s.as_vector()
        out[f"traj_{kind}_cmds"] = cmds
        out[f"traj_{kind}"] = traj
    # SPEC KATs
    p10 = QuadParams(motor_decay=10.0)
    out["kat_lag"] = dyn.rotor_lag(np.zeros((1, 4)), np.full((1, 4), 100.0), 0.1, p10)
    pd = QuadParams(air_density=1.2, drag_coeffs=[0.5, 0.5, 0.5], cross_area=[0.1, 0.1, 0.1])
    out["kat_drag"] = dyn.drag_force(np.array([[1.0, 0.0, 0.0]]), pd)
    pz = QuadParams(air_density=0.0)
    s = dyn.QuadState.hover(1, pz, position=[0, 0, 10.0])
    s.rotor_speeds[:] = 0.0
    for _ in range(50):
        s = dyn.step(s, np.zeros((1, 4)), SimConfig(), pz)
    out["kat_freefall_z"] = s.position_w[0, 2]
    mix = ctl.mixer(np.array([params.mass * 9.81]), np.zeros((1, 3)), params)
    out["kat_mixer_hover"] = mix.thrusts
    h = dyn.QuadState.hover(4, params)
    for _ in range(50):
        sp = ctl.command_to_rotor_speeds(ctl.CTBR(np.full(4, 9.81), np.zeros((4, 3))), h, gains, params)
        h = dyn.step(h, sp, SimConfig(), params)
    out["kat_hover_1s"] = h.as_vector()
    out["hover_speed"] = np.array(params.hover_speed)
    np.savez_compressed(os.path.join(OUT, "dynamics.npz"), **out)


def gen_jacobian():
    rng = np.random.default_rng(7)
    params = QuadParams()
    out = {}
    for name, sim in (("rk4", SimConfig()), ("euler4", SimConfig(integrator="euler", substeps=4))):
        n = 12
        xs = random_states(rng, n, params)
        acts = rng.uniform(300, 1400, (n, 4))
        acts[0, 0] = 1500.0  # clamp boundary -> flagged
        acts[1, 1] = 1700.0  # outside -> zero column
        Js, Jas, nxt, fl = [], [], [], []
        for i in range(n):
            sj = grd.step_jacobian(dyn.QuadState.from_vector(xs[i]), acts[i], sim, params)
            Js.append(sj.full_state_jacobian); Jas.append(sj.full_action_jacobian)
            nxt.append(sj.next_state.as_vector()[0]); fl.append(sj.saturation_boundary)
        out[f"{name}_state"] = xs; out[f"{name}_action"] = acts
        out[f"{name}_J"] = np.array(Js); out[f"{name}_Ja"] = np.array(Jas)
        out[f"{name}_next"] = np.array(nxt); out[f"{name}_flag"] = np.array(fl)
    # rollout_grad (gradients.py:218-237), 3 agents x 10 steps
    target = np.array([1.0, 0.0, 2.0])

    def loss(traj):
        g = np.zeros_like(traj)
        d = traj[-1, 0:3] - target
        g[-1, 0:3] = 2.0 * d
        g[:, 3:6] = 0.02 * traj[:, 3:6]
        return float(d @ d + 0.01 * (traj[:, 3:6] ** 2).sum()), g

    sim = SimConfig()
    x0s, acts, gas, gis = [], [], [], []
    for i in range(3):
        x0 = dyn.QuadState.hover(1, params, position=rng.uniform(-0.1, 0.1, 3)).as_vector()[0]
        a = 900.0 + rng.normal(scale=20.0, size=(10, 4))
        ga, gi, tape = grd.rollout_grad(dyn.QuadState.from_vector(x0), a, loss, sim, params)
        x0s.append(x0); acts.append(a); gas.append(ga); gis.append(gi)
    out["rg_x0"] = np.array(x0s); out["rg_actions"] = np.array(acts)
    out["rg_grad_actions"] = np.array(gas); out["rg_grad_init"] = np.array(gis); out["rg_target"] = target
    np.savez_compressed(os.path.join(OUT, "jacobian.npz"), **out)


def tess_scene():
    """A TriMesh scene: a tessellated box room with a few box obstacles."""
    objs = []
    rng = np.random.default_rng(3)

    def box_mesh(c, h):
        v = np.array([[sx, sy, sz] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)], float) * h + c
        f = [(0, 1, 3), (0, 3, 2), (4, 6, 7), (4, 7, 5), (0, 4, 5), (0, 5, 1), (2, 3, 7), (2, 7, 6), (0, 2, 6), (0, 6, 4),
             (1, 5, 7), (1, 7, 3)]
        return shapes.TriMesh(v, np.array(f))

    objs.append(shapes.SceneObject(1, box_mesh(np.array([0.0, 0.0, -0.1]), np.array([5.0, 5.0, 0.1]))))
    for k in range(6):
        c = rng.uniform([-3, -3, 0.5], [3, 3, 2.5])
        objs.append(shapes.SceneObject(7 + k, box_mesh(c, rng.uniform(0.2, 0.6, 3))))
    return shapes.Scene(objs)


def gen_geometry():
    out = {}
    nav = SceneSpec(kind="cluttered", seed=0, density=0.15, volume_lo=[-5, -5, 0], volume_hi=[5, 5, 4]).materialize()
    scenes = {"nav": nav, "landing": generate.landing_scene(), "garage": generate.garage_scene(),
              "gap": generate.gap_scene(1.0), "tess": tess_scene(),
              "garage10": generate.garage_scene(shapes.AABB([-5, -5, 0], [5, 5, 4]))}
    for name, sc in scenes.items():
        for k, v in scene_arrays(sc).items():
            out[f"{name}_{k}"] = v
        out[f"{name}_bounds"] = np.stack([sc.bounds.lo, sc.bounds.hi])
    rng = np.random.default_rng(11)
    for name in ("nav", "tess"):
        sc = scenes[name]
        q = rng.uniform([-5.5, -5.5, -0.5], [5.5, 5.5, 4.5], (512, 3))
        pts, ds, ids = [], [], []
        for qq in q:
            r = queries.nearest_point(sc, qq)
            pts.append(r.point); ds.append(r.distance); ids.append(r.object_id)
        out[f"{name}_np_q"] = q; out[f"{name}_np_pt"] = np.array(pts); out[f"{name}_np_d"] = np.array(ds)
        out[f"{name}_np_id"] = np.array(ids)
        o = rng.uniform([-4.5, -4.5, 0.3], [4.5, 4.5, 3.7], (512, 3))
        d = rng.normal(size=(512, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
        ts, rid = [], []
        for oo, dd in zip(o, d):
            h = queries.raycast(sc, oo, dd, 10.0)
            ts.append(-1.0 if h is None else h.t); rid.append(-1 if h is None else h.object_id)
        out[f"{name}_rc_o"] = o; out[f"{name}_rc_d"] = d; out[f"{name}_rc_t"] = np.array(ts); out[f"{name}_rc_id"] = np.array(rid)
    # renders
    cam = sensing.CameraModel()
    pos = np.concatenate([rng.uniform([-4.4, -2.5, 1.2], [-3.8, 2.5, 2.8], (3, 3)),
                          rng.uniform([-4, -4, 0.5], [4, 4, 3.5], (3, 3))])
    yaw = rng.uniform(-np.pi, np.pi, 6)
    quat = np.stack([np.cos(yaw / 2), 0 * yaw, 0 * yaw, np.sin(yaw / 2)], axis=1)
    quat[4] = [0.9, 0.2, -0.3, 0.1]
    quat[4] /= np.linalg.norm(quat[4])
    for name in ("nav", "tess"):
        dpt, ids = sensing.render_frames(scenes[name], pos, quat, cam)
        out[f"{name}_render_pos"] = pos; out[f"{name}_render_quat"] = quat
        out[f"{name}_render_depth"] = dpt; out[f"{name}_render_ids"] = ids
    down = sensing.CameraModel(rotation=sensing.DOWNWARD)
    lpos = np.array([[0.0, 0.0, 2.0], [0.3, -0.2, 1.2], [1.5, 1.0, 3.0]])
    lq = np.array([[1.0, 0, 0, 0], [0.98, 0.1, 0.05, 0.1], [1.0, 0, 0, 0]])
    lq /= np.linalg.norm(lq, axis=1, keepdims=True)
    dpt, ids = sensing.render_frames(scenes["landing"], lpos, lq, down)
    out["landing_render_pos"] = lpos; out["landing_render_quat"] = lq
    out["landing_render_depth"] = dpt; out["landing_render_ids"] = ids
    # floor KAT: 2 m above a floor looking down -> 2.0
    floor = generate.floor_scene()
    dpt, _ = sensing.render_frames(floor, np.array([[0.0, 0.0, 2.0]]), np.array([[1.0, 0, 0, 0]]), down)
    out["kat_floor_depth"] = dpt
    np.savez_compressed(os.path.join(OUT, "geometry.npz"), **out)


def record_env(env, actions_fn, steps, seed, keep_images=(), policy=None):
    obs = env.reset(seed=seed)
    if policy is not None:
        policy.reset(obs)
    n = env.num_agents
    rec = {k: [] for k in ("state", "reward", "terminated", "truncated", "collision", "oob", "nonfinite", "success",
                           "nearest_dist", "nearest_pt", "step", "scene", "target", "full_state", "prev_state")}
    rec0 = {"state": np.stack([o["state"] for o in obs]), "full_state": env.state.as_vector().copy()}
    acts = []
    imgs = {}
    rng = np.random.default_rng(seed + 1000)
    for t in range(steps):
        if policy is not None:
            a = policy(obs, t).as_array()
        else:
            a = actions_fn(rng, t, n)
        acts.append(a)
        res = env.step(ctl.command_from_array(env.config.command_type, a))
        obs = res.observations
        rec["state"].append(np.stack([o["state"] for o in res.observations]))
        rec["full_state"].append(env.state.as_vector().copy())
        rec["prev_state"].append(env.prev_state.as_vector().copy())
        rec["reward"].append(res.reward.copy())
        rec["terminated"].append(res.terminated.copy())
        rec["truncated"].append(res.truncated.copy())
        rec["collision"].append(np.array([i["collision"] for i in res.info]))
        rec["oob"].append(np.array([i["out_of_bounds"] for i in res.info]))
        rec["nonfinite"].append(np.array([i["nonfinite"] for i in res.info]))
        rec["success"].append(np.array([i["success"] for i in res.info]))
        rec["nearest_dist"].append(np.array([i["nearest_distance"] for i in res.info]))
        rec["nearest_pt"].append(env.nearest_pt.copy())
        rec["step"].append(np.array([i["step"] for i in res.info]))
        rec["scene"].append(np.array([i["scene"] for i in res.info]))
        if "target" in res.observations[0]:
            rec["target"].append(np.stack([o["target"] for o in res.observations]))
        if t in keep_images:
            for key in res.observations[0]:
                if key in ("depth", "vision", "segmentation"):
                    imgs[f"img_{key}_{t}"] = np.stack([o[key] for o in res.observations])
    out = {k: np.array(v) for k, v in rec.items() if v}
    out.update({f"reset_{k}": v for k, v in rec0.items()})
    out["actions"] = np.array(acts)
    out.update(imgs)
    return out


def gen_env():
    # navigation: short episodes to exercise truncation, aggressive LV to hit walls/obstacles
    cfg = tasks.navigation_config(scene_seed=0, num_agents=12)
    cfg = dataclasses.replace(cfg, episode_max_steps=25)
    env = tasks.make_env(cfg)

    def lv(rng, t, n):
        v = rng.normal(scale=4.0, size=(n, 3))
        v[:, 0] += 1.5
        return np.concatenate([v, rng.uniform(-np.pi, np.pi, (n, 1))], axis=1)

    out = record_env(env, lv, 60, seed=3, keep_images=(0, 1, 59))
    out["max_steps"] = np.array(25)
    np.savez_compressed(os.path.join(OUT, "env_nav.npz"), **out)

    # landing: down-looking segmentation camera, pad-centroid target
    from quadsim.env.policies import DescendAndCenterPolicy

    cfg = dataclasses.replace(tasks.landing_config(num_agents=8), episode_max_steps=250)
    env = tasks.make_env(cfg)
    out = record_env(env, None, 330, seed=1, keep_images=(0, 60), policy=DescendAndCenterPolicy(env))
    np.savez_compressed(os.path.join(OUT, "env_landing.npz"), **out)

    # free flight (C1 semantics): garage, ctbr hover + perturbation
    cfg = EnvConfig(num_agents=8, command_type="ctbr", episode_max_steps=40,
                    randomization=InitRandomization(position=DistSpec("uniform", low=[-2, -2, 1], high=[2, 2, 3])))
    env = tasks.make_env(cfg)

    def ctbr(rng, t, n):
        return np.concatenate([rng.uniform(7.0, 16.0, (n, 1)), rng.normal(scale=4.0, size=(n, 3))], axis=1)

    out = record_env(env, ctbr, 80, seed=5)
    np.savez_compressed(os.path.join(OUT, "env_free.npz"), **out)


def gen_rng():
    out = {}
    seeds = np.array([0, 1, 7, 12345, 2**31 - 1, 2**32 + 5, 987654321012])
    states, draws, unif = [], [], []
    for s in seeds:
        bg = np.random.PCG64(int(s))
        st = bg.state["state"]
        states.append([st["state"] >> 64, st["state"] & (2**64 - 1), st["inc"] >> 64, st["inc"] & (2**64 - 1)])
        g = np.random.Generator(np.random.PCG64(int(s)))
        draws.append(g.random(8))
        g = np.random.default_rng(int(s))
        unif.append(g.uniform(np.array([-4.4, -2.5, 1.2]), np.array([-3.8, 2.5, 2.8])))
    out["seeds"] = seeds
    out["pcg_state"] = np.array(states, dtype=np.uint64)
    out["doubles"] = np.array(draws)
    out["uniform"] = np.array(unif)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **out)


NOISE_CASES = [  # (sensor, kind, params)
    ("depth", "normal", dict(sigma=0.05)), ("depth", "normal", dict(sigma=0.0)),
    ("depth", "poisson", dict(scaling=10.0)), ("depth", "poisson", dict(scaling=250.0)),
    ("depth", "saltpepper", dict(p=0.1)), ("depth", "speckle", dict(sigma=0.1)),
    ("depth", "redwood", dict(sigma_disparity=0.01, quantization=0.05)), ("depth", "redwood", dict(sigma_disparity=0.02)),
    ("segmentation", "normal", dict(sigma=0.5)), ("segmentation", "poisson", dict(scaling=1.0)),
    ("segmentation", "saltpepper", dict(p=0.2)), ("segmentation", "speckle", dict(sigma=0.05)),
    ("imu", "normal", dict(sigma=0.1)),
]


def gen_noise():
    """sensing.apply_noise per (sensor, kind), IMU readings, and a noisy env episode."""
    from quadsim.sensing import NoiseSpec

    out = {}
    rng = np.random.default_rng(77)
    for c, (sensor, kind, kw) in enumerate(NOISE_CASES):
        if sensor == "depth":
            data = rng.uniform(0.3, 10.0, (16, 12))
        elif sensor == "segmentation":
            data = rng.integers(0, 12, (16, 12)).astype(float)
        else:
            data = rng.normal(size=6)
        g = np.random.default_rng(100 + c)
        res = sensing.apply_noise(data, NoiseSpec(kind, **kw), g, sensor=sensor)
        out[f"case{c}_in"] = data
        out[f"case{c}_out"] = res
        out[f"case{c}_after"] = np.array(g.random(2))  # pins how many draws were consumed
    # IMU: body_wrench + imu_read on random states
    params = QuadParams()
    states = random_states(rng, 32, params)
    st = dyn.QuadState.from_vector(states)
    reading = sensing.imu_read(st, sensing.body_wrench(st, params), params)
    out["imu_states"] = states
    out["imu_force"] = reading.specific_force_b
    out["imu_gyro"] = reading.angvel_b
    np.savez_compressed(os.path.join(OUT, "noise.npz"), **out)

    # a noisy navigation episode: normal-distribution spawns (ziggurat in the
    # spawn path), depth + segmentation + IMU sensors with noise chains
    cfg = tasks.navigation_config(scene_seed=0, num_agents=6)
    cfg = dataclasses.replace(
        cfg, episode_max_steps=12, command_type="ctbr",  # CTBR: no trig in the controller -> FP64 bit-exact states
        randomization=dataclasses.replace(cfg.randomization,
                                          velocity=DistSpec("normal", mean=[0.2, 0.0, 0.0], sigma=[0.3, 0.3, 0.1])),
        sensors=(SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("normal", sigma=0.02),
                                                             NoiseSpec("redwood", sigma_disparity=0.005))),
                 SensorSpec(kind="imu", name="imu", noise=(NoiseSpec("normal", sigma=0.05),)),
                 SensorSpec(kind="segmentation", name="vision", noise=(NoiseSpec("saltpepper", p=0.05),))))
    env = tasks.make_env(cfg)

    def lv(rng, t, n):  # CTBR: collective thrust + body rates
        return np.concatenate([rng.uniform(6.0, 14.0, (n, 1)), rng.normal(scale=2.0, size=(n, 3))], axis=1)

    rec = record_env(env, lv, 20, seed=4, keep_images=())
    keep = (0, 1, 2, 12, 20)  # observation snapshots after reset (0) and after steps 1, 2, 12, 20
    obs_log = {"depth": [], "imu": [], "vision": []}
    env2 = tasks.make_env(cfg)
    obs = env2.reset(seed=4)
    r2 = np.random.default_rng(4 + 1000)
    for key in obs_log:
        obs_log[key].append(np.stack([o[key] for o in obs]))
    for t in range(1, 21):
        res = env2.step(ctl.command_from_array(cfg.command_type, lv(r2, t - 1, 6)))
        if t in keep:
            for key in obs_log:
                obs_log[key].append(np.stack([o[key] for o in res.observations]))
    rec.update({f"obs_{k}": np.array(v) for k, v in obs_log.items()})
    rec["obs_steps"] = np.array(keep)
    np.savez_compressed(os.path.join(OUT, "env_noise.npz"), **rec)


def gen_control():
    """Controller stages on their own: mixer (incl. saturation), LV/PS -> CTBR."""
    params, gains = QuadParams(), ControllerGains()
    rng = np.random.default_rng(21)
    n = 64
    force = rng.uniform(2.0, 18.0, n)
    force[::9] = rng.uniform(-2.0, 40.0, force[::9].shape)  # clamped collectives
    torque = rng.normal(scale=0.02, size=(n, 3))
    torque[::4] *= 40.0  # saturating torque requests
    m = ctl.mixer(force, torque, params)
    states = random_states(rng, n, params)
    st = dyn.QuadState.from_vector(states)
    lv = np.concatenate([rng.normal(scale=3.0, size=(n, 3)), rng.uniform(-np.pi, np.pi, (n, 1))], axis=1)
    ps = np.concatenate([rng.uniform(-4, 4, (n, 3)), rng.uniform(-np.pi, np.pi, (n, 1))], axis=1)
    c_lv = ctl.lv_to_ctbr(ctl.command_from_array("lv", lv), st, gains, params)
    c_ps = ctl.ps_to_ctbr(ctl.command_from_array("ps", ps), st, gains, params)
    np.savez_compressed(os.path.join(OUT, "control.npz"), force=force, torque=torque, thrusts=m.thrusts,
                        saturated=m.saturated, states=states, lv=lv, ps=ps, lv_ctbr=c_lv.as_array(),
                        ps_ctbr=c_ps.as_array())


def multiscene_config():
    """Three scenes (garage + two cluttered rooms), shuffled assignment, a
    depth + segmentation camera, CTBR (FP64-exact controller), short episodes."""
    return EnvConfig(
        num_agents=9, command_type="ctbr", episode_max_steps=15, scene_sampling="shuffled",
        scenes=(SceneSpec(kind="garage"), SceneSpec(kind="cluttered", seed=3, density=0.2),
                SceneSpec(kind="cluttered", seed=8, density=0.12)),
        randomization=InitRandomization(position=DistSpec("uniform", low=[-3.5, -3.5, 0.8], high=[3.5, 3.5, 3.0])),
        sensors=(SensorSpec(kind="depth", name="depth", width=32, height=24),
                 SensorSpec(kind="segmentation", name="vision", width=32, height=24)))


def gen_multiscene():
    env = tasks.make_env(multiscene_config())

    def ctbr(rng, t, n):
        return np.concatenate([rng.uniform(5.0, 15.0, (n, 1)), rng.normal(scale=3.0, size=(n, 3))], axis=1)

    rec = record_env(env, ctbr, 50, seed=11, keep_images=(0, 16, 49))
    np.savez_compressed(os.path.join(OUT, "env_multiscene.npz"), **rec)
    print("multiscene scenes", np.unique(rec["scene"]), "respawns", int(rec["truncated"].sum() + rec["terminated"].sum()))


def gen_logs():
    """env/logs.py episode-log bytes."""
    import tempfile

    from quadsim.env import logs

    rng = np.random.default_rng(5)
    path = os.path.join(tempfile.mkdtemp(), "ep.jsonl")
    states, actions, rewards = rng.normal(size=(3, 13)), rng.normal(size=(3, 4)), rng.normal(size=3)
    with logs.EpisodeLogWriter(path) as w:
        for i in range(3):
            w.append(7, i, states[i], actions[i], rewards[i], {"collision": bool(i == 1), "success": False})
    np.savez_compressed(os.path.join(OUT, "logs.npz"), states=states, actions=actions, rewards=rewards,
                        log=np.frombuffer(open(path, "rb").read(), np.uint8))


def gen_pgm():
    """sensing.py:238-274 PGM export bytes."""
    import tempfile

    rng = np.random.default_rng(3)
    depth = rng.uniform(0.2, 70.0, (5, 7))
    depth[0, 0], depth[1, 1] = 0.0004, 80.0
    ids = rng.integers(0, 70000, (6, 4))
    d = tempfile.mkdtemp()
    sensing.export_depth_mm(os.path.join(d, "a.pgm"), depth)
    sensing.export_segmentation(os.path.join(d, "b.pgm"), ids)
    rd = lambda f: np.frombuffer(open(os.path.join(d, f), "rb").read(), np.uint8)  # noqa: E731
    np.savez_compressed(os.path.join(OUT, "pgm.npz"), depth=depth, ids=ids, depth_pgm=rd("a.pgm"), ids_pgm=rd("b.pgm"))


def swarm_config():
    """Gap crossing in swarm mode with CTBR commands (FP64-exact controller),
    a crowded spawn box and a depth + segmentation camera (drone spheres)."""
    cfg = tasks.gap_crossing_config(gap_width=1.0, num_agents=6)
    return dataclasses.replace(
        cfg, command_type="ctbr", episode_max_steps=40,
        randomization=dataclasses.replace(cfg.randomization, position=DistSpec("uniform", low=[-3.4, -0.6, 1.3],
                                                                               high=[-2.8, 0.6, 1.7])),
        sensors=(SensorSpec(kind="depth", name="depth", width=48, height=32),
                 SensorSpec(kind="segmentation", name="vision", width=48, height=32)))


def gen_swarm():
    cfg = swarm_config()
    env = tasks.make_env(cfg)

    def ctbr(rng, t, n):
        return np.concatenate([rng.uniform(2.0, 22.0, (n, 1)), rng.normal(scale=6.0, size=(n, 3))], axis=1)

    rec = record_env(env, ctbr, 120, seed=2, keep_images=(0, 1, 17, 119))
    env2 = tasks.make_env(cfg)
    obs = env2.reset(seed=2)
    swarm = [np.stack([o["swarm"] for o in obs])]
    r2 = np.random.default_rng(2 + 1000)
    for t in range(120):
        res = env2.step(ctl.command_from_array("ctbr", ctbr(r2, t, 6)))
        swarm.append(np.stack([o["swarm"] for o in res.observations]))
    rec["swarm_obs"] = np.array(swarm)
    np.savez_compressed(os.path.join(OUT, "env_swarm.npz"), **rec)
    print("swarm collisions", rec["collision"].sum(), "terminated", rec["terminated"].sum(), "success", rec["success"].sum())


if __name__ == "__main__":
    print("reference:", quadsim.__file__, "numpy", np.__version__)
    if len(sys.argv) > 2 and sys.argv[2] == "noise":
        gen_noise()
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[2] == "multiscene":
        gen_multiscene()
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[2] == "control":
        gen_control()
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[2] == "swarm":
        gen_swarm()
        sys.exit(0)
    gen_multiscene()
    gen_control()
    gen_logs()
    gen_pgm()
    gen_swarm()
    gen_noise()
    gen_rng()
    gen_dynamics()
    gen_jacobian()
    gen_geometry()
    gen_env()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
