"""Pin the CPU oracle (oracle/) to golden fixtures produced by running the
reference itself (tests/golden/make_golden.py).  CPU only."""

import dataclasses

import numpy as np
import pytest

import oracle
from oracle.env import OracleEnv
from conftest import golden, scene_from_golden
from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig


def P(**sim):
    return oracle.pack_params(QuadParams(), SimConfig(**sim), ControllerGains())


@pytest.mark.parametrize("kind", ["srt", "ctbr", "ps", "lv"])
def test_controller_bit_exact(gdyn, kind):
    out = oracle.command_to_rotor_speeds(P(), kind, gdyn["state0"], gdyn[f"{kind}_cmd"])
    assert np.array_equal(out, gdyn[f"{kind}_speeds"])


@pytest.mark.parametrize("kind", ["srt", "ctbr", "ps", "lv", "rotor"])
@pytest.mark.parametrize("integ,sub", [("rk4", 2), ("euler", 4), ("rk4", 1)])
def test_dynamics_step_bit_exact(gdyn, kind, integ, sub):
    nxt, bad = oracle.dynamics_step(P(integrator=integ, substeps=sub), gdyn["state0"], gdyn[f"{kind}_speeds"])
    assert not bad.any()
    assert np.array_equal(nxt, gdyn[f"{kind}_{integ}{sub}_next"])


@pytest.mark.parametrize("kind", ["ctbr", "lv", "ps", "srt"])
def test_closed_loop_100_steps_bit_exact(gdyn, kind):
    traj, cmds = gdyn[f"traj_{kind}"], gdyn[f"traj_{kind}_cmds"]
    x = traj[0].copy()
    p = P()
    for t in range(cmds.shape[0]):
        sp = oracle.command_to_rotor_speeds(p, kind, x, cmds[t])
        x, bad = oracle.dynamics_step(p, x, sp)
        assert not bad.any()
    assert np.array_equal(x, traj[-1])


def test_kats(gdyn):
    # free fall and hover KATs via the oracle
    pz = oracle.pack_params(QuadParams(air_density=0.0), SimConfig(), ControllerGains())
    x = np.zeros((1, 17)); x[0, 2] = 10.0; x[0, 6] = 1.0
    for _ in range(50):
        x, _ = oracle.dynamics_step(pz, x, np.zeros((1, 4)))
    assert x[0, 2] == gdyn["kat_freefall_z"]
    assert abs(x[0, 2] - (10.0 - 4.905)) < 1e-9
    p = P()
    assert p.hover_speed == float(gdyn["hover_speed"])


def test_nonfinite_mask():
    p = P()
    x = np.zeros((3, 17)); x[:, 6] = 1.0; x[:, 13:] = 900.0
    x[1, 3] = np.inf
    nxt, bad = oracle.dynamics_step(p, x, np.full((3, 4), 900.0))
    assert bad.tolist() == [False, True, False]


@pytest.mark.parametrize("name", ["rk4", "euler4"])
def test_step_jacobian_matches_reference(gjac, name):
    sim = SimConfig() if name == "rk4" else SimConfig(integrator="euler", substeps=4)
    p = oracle.pack_params(QuadParams(), sim, ControllerGains())
    for i in range(len(gjac[f"{name}_state"])):
        J, Ja, nx, flag = oracle.step_jacobian(p, gjac[f"{name}_state"][i], gjac[f"{name}_action"][i])
        assert np.array_equal(nx, gjac[f"{name}_next"][i])  # next_state bitwise == step
        assert flag == bool(gjac[f"{name}_flag"][i])
        # BLAS-vs-loop summation order: agree to rounding
        np.testing.assert_allclose(J, gjac[f"{name}_J"][i], rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(Ja, gjac[f"{name}_Ja"][i], rtol=1e-9, atol=1e-13)


def test_rollout_grad_matches_reference(gjac):
    target = gjac["rg_target"]

    def loss(traj):
        g = np.zeros_like(traj)
        d = traj[-1, 0:3] - target
        g[-1, 0:3] = 2.0 * d
        g[:, 3:6] = 0.02 * traj[:, 3:6]
        return float(d @ d + 0.01 * (traj[:, 3:6] ** 2).sum()), g

    p = P()
    for i in range(len(gjac["rg_x0"])):
        ga, gi, _, _ = oracle.rollout_grad(p, gjac["rg_x0"][i], gjac["rg_actions"][i], loss)
        np.testing.assert_allclose(ga, gjac["rg_grad_actions"][i], rtol=1e-8, atol=1e-14)
        np.testing.assert_allclose(gi, gjac["rg_grad_init"][i], rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("name", ["nav", "landing", "garage", "gap", "tess"])
def test_bvh_build_identical(ggeo, name):
    s = scene_from_golden(ggeo, name)
    for k in ("node_lo", "node_hi", "node_first", "node_count", "prim_order"):
        assert np.array_equal(getattr(s, k), ggeo[f"{name}_{k}"]), k


@pytest.mark.parametrize("name", ["nav", "tess"])
def test_nearest_point_and_raycast_exact(ggeo, name):
    s = scene_from_golden(ggeo, name)
    pt, d, oid = s.nearest_point(ggeo[f"{name}_np_q"])
    assert np.array_equal(pt, ggeo[f"{name}_np_pt"])
    assert np.array_equal(d, ggeo[f"{name}_np_d"])
    assert np.array_equal(oid, ggeo[f"{name}_np_id"])
    # the SPEC's own oracle: brute force over all primitives
    pt_b, d_b, oid_b = s.nearest_point(ggeo[f"{name}_np_q"], brute=True)
    assert np.array_equal(oid_b, oid) and np.max(np.abs(d_b - d)) <= 1e-12
    t, rid = s.raycast(ggeo[f"{name}_rc_o"], ggeo[f"{name}_rc_d"], 10.0)
    assert np.array_equal(t, ggeo[f"{name}_rc_t"])
    assert np.array_equal(rid, ggeo[f"{name}_rc_id"])


@pytest.mark.parametrize("name,cam", [("nav", "forward"), ("tess", "forward"), ("landing", "down")])
def test_render_exact(ggeo, name, cam):
    s = scene_from_golden(ggeo, name)
    rot = oracle.FORWARD if cam == "forward" else oracle.DOWNWARD
    depth, ids = oracle.render_frames(s, ggeo[f"{name}_render_pos"], ggeo[f"{name}_render_quat"], cam_rotation=rot)
    assert np.array_equal(depth, ggeo[f"{name}_render_depth"])
    assert np.array_equal(ids, ggeo[f"{name}_render_ids"])


def _replay(gname, config, seed, scene_names):
    g = golden(gname)
    # the config's own scenes (SceneSpec volumes), flattened by the generator
    # that test_host pins bit-exact to the reference generator
    scenes = []
    for spec in config.scenes:
        t = spec.materialize().arrays
        scenes.append(oracle.OracleScene(t.prim_type, t.prim_data, t.prim_object_id, t.prim_aabb_lo, t.prim_aabb_hi))
    env = OracleEnv(config, scenes, QuadParams(), SimConfig(), ControllerGains())
    obs = env.reset(seed=seed)
    assert np.array_equal(obs["state"], g["reset_state"])
    assert np.array_equal(env.state, g["reset_full_state"])
    for t in range(g["actions"].shape[0]):
        obs, rew, term, trunc, succ = env.step(g["actions"][t])
        assert np.array_equal(env.state, g["full_state"][t]), t
        assert np.array_equal(env.prev_state, g["prev_state"][t]), t
        assert np.array_equal(rew, g["reward"][t]), t
        assert np.array_equal(term, g["terminated"][t]) and np.array_equal(trunc, g["truncated"][t]), t
        assert np.array_equal(env.collision, g["collision"][t]) and np.array_equal(env.oob, g["oob"][t]), t
        assert np.array_equal(succ, g["success"][t]), t
        assert np.array_equal(env.nearest_dist, g["nearest_dist"][t]), t
        assert np.array_equal(env.nearest_pt, g["nearest_pt"][t]), t
        assert np.array_equal(env.step_counts, g["step"][t]), t
        if "target" in g:
            assert np.array_equal(obs["target"], g["target"][t]), t
        for key in g.keys():
            if key.startswith("img_") and key.endswith(f"_{t}"):
                sensor = key[4:].rsplit("_", 1)[0]
                assert np.array_equal(obs[sensor], g[key]), (key, t)
    return env


def test_env_navigation_replay():
    from paper_2407_14783_b200.env import navigation_config

    g = golden("env_nav")
    cfg = dataclasses.replace(navigation_config(scene_seed=0, num_agents=12), episode_max_steps=int(g["max_steps"]))
    _replay("env_nav", cfg, 3, ["nav"])


def test_env_landing_replay():
    from paper_2407_14783_b200.env import landing_config

    cfg = dataclasses.replace(landing_config(num_agents=8), episode_max_steps=250)
    _replay("env_landing", cfg, 1, ["landing"])


def test_env_free_replay():
    from paper_2407_14783_b200.env import DistSpec, EnvConfig, InitRandomization

    cfg = EnvConfig(num_agents=8, command_type="ctbr", episode_max_steps=40,
                    randomization=InitRandomization(position=DistSpec("uniform", low=[-2, -2, 1], high=[2, 2, 3])))
    _replay("env_free", cfg, 5, ["garage"])


def test_pcg64_seeding_restatement():
    """qb_rng.cuh's SeedSequence + PCG64 restated in Python == numpy (rng.npz)."""
    g = golden("rng")
    M = 0xFFFFFFFF

    def seed_pcg(seed):
        ent = [seed & M] + ([seed >> 32] if seed >> 32 else [])
        hc = [0x43B0D7E5]

        def hashmix(v):
            v ^= hc[0]
            hc[0] = (hc[0] * 0x931E8875) & M
            v = (v * hc[0]) & M
            return v ^ (v >> 16)

        def mix(x, y):
            r = (0xCA01F9DD * x - 0x4973F715 * y) & M
            return r ^ (r >> 16)

        pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
        for s in range(4):
            for d in range(4):
                if s != d:
                    pool[d] = mix(pool[d], hashmix(pool[s]))
        hb, words = 0x8B51F9DD, []
        for i in range(8):
            v = pool[i & 3] ^ hb
            hb = (hb * 0x58F38DED) & M
            v = (v * hb) & M
            words.append(v ^ (v >> 16))
        val = [words[2 * i] | (words[2 * i + 1] << 32) for i in range(4)]
        mul = (2549297995355413924 << 64) + 4865540595714422341
        MM = (1 << 128) - 1
        inc = (((val[2] << 64) | val[3]) << 1 | 1) & MM
        s = inc
        s = (s + ((val[0] << 64) | val[1])) & MM
        s = (s * mul + inc) & MM
        return s, inc

    for i, seed in enumerate(g["seeds"]):
        s, inc = seed_pcg(int(seed))
        w = [int(x) for x in g["pcg_state"][i]]
        assert s == (w[0] << 64 | w[1]) and inc == (w[2] << 64 | w[3])


# ------------------------------------------------------------- F1: sensors
def noise_config():
    """The noisy navigation config make_golden.py records (env_noise.npz)."""
    from paper_2407_14783_b200.env import DistSpec, NoiseSpec, SensorSpec, navigation_config

    cfg = navigation_config(scene_seed=0, num_agents=6)
    return dataclasses.replace(
        cfg, episode_max_steps=12, command_type="ctbr",
        randomization=dataclasses.replace(cfg.randomization,
                                          velocity=DistSpec("normal", mean=[0.2, 0.0, 0.0], sigma=[0.3, 0.3, 0.1])),
        sensors=(SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("normal", sigma=0.02),
                                                             NoiseSpec("redwood", sigma_disparity=0.005))),
                 SensorSpec(kind="imu", name="imu", noise=(NoiseSpec("normal", sigma=0.05),)),
                 SensorSpec(kind="segmentation", name="vision", noise=(NoiseSpec("saltpepper", p=0.05),))))


NOISE_CASES = [
    ("depth", "normal", dict(sigma=0.05)), ("depth", "normal", dict(sigma=0.0)),
    ("depth", "poisson", dict(scaling=10.0)), ("depth", "poisson", dict(scaling=250.0)),
    ("depth", "saltpepper", dict(p=0.1)), ("depth", "speckle", dict(sigma=0.1)),
    ("depth", "redwood", dict(sigma_disparity=0.01, quantization=0.05)), ("depth", "redwood", dict(sigma_disparity=0.02)),
    ("segmentation", "normal", dict(sigma=0.5)), ("segmentation", "poisson", dict(scaling=1.0)),
    ("segmentation", "saltpepper", dict(p=0.2)), ("segmentation", "speckle", dict(sigma=0.05)),
    ("imu", "normal", dict(sigma=0.1)),
]


@pytest.mark.parametrize("case", range(len(NOISE_CASES)))
def test_apply_noise_bit_exact(case):
    from oracle.env import apply_noise
    from paper_2407_14783_b200.sensing import NoiseSpec

    g = golden("noise")
    sensor, kind, kw = NOISE_CASES[case]
    rng = np.random.default_rng(100 + case)
    out = apply_noise(g[f"case{case}_in"], NoiseSpec(kind, **kw), rng, sensor)
    assert np.array_equal(out, g[f"case{case}_out"])
    assert np.array_equal(rng.random(2), g[f"case{case}_after"])  # same number of draws consumed


def test_imu_reading_bit_exact():
    from oracle.env import imu_readings

    g = golden("noise")
    r = imu_readings(g["imu_states"], P())
    assert np.array_equal(r[:, :3], g["imu_force"])
    assert np.array_equal(r[:, 3:], g["imu_gyro"])


def test_env_noise_replay():
    """Normal-distribution spawns + depth/IMU/segmentation noise chains."""
    g = golden("env_noise")
    cfg = noise_config()
    env = _replay("env_noise", cfg, 4, ["nav"])
    # observation snapshots: replay again and compare the noisy observations
    scenes = []
    for spec in cfg.scenes:
        t = spec.materialize().arrays
        scenes.append(oracle.OracleScene(t.prim_type, t.prim_data, t.prim_object_id, t.prim_aabb_lo, t.prim_aabb_hi))
    env = OracleEnv(cfg, scenes, QuadParams(), SimConfig(), ControllerGains())
    obs = env.reset(seed=4)
    keep = list(g["obs_steps"])
    snaps = {0: obs}
    for t in range(1, 21):
        obs = env.step(g["actions"][t - 1])[0]
        if t in keep:
            snaps[t] = obs
    for j, t in enumerate(keep):
        for key in ("depth", "imu", "vision"):
            assert np.array_equal(snaps[t][key], g[f"obs_{key}"][j]), (key, t)


# ------------------------------------------------------------- F2: swarm mode
def swarm_config():
    """make_golden.py swarm_config: gap crossing, 6 agents, CTBR, depth + segmentation."""
    from paper_2407_14783_b200.env import DistSpec, SensorSpec, gap_crossing_config

    cfg = gap_crossing_config(gap_width=1.0, num_agents=6)
    return dataclasses.replace(
        cfg, command_type="ctbr", episode_max_steps=40,
        randomization=dataclasses.replace(cfg.randomization, position=DistSpec("uniform", low=[-3.4, -0.6, 1.3],
                                                                               high=[-2.8, 0.6, 1.7])),
        sensors=(SensorSpec(kind="depth", name="depth", width=48, height=32),
                 SensorSpec(kind="segmentation", name="vision", width=48, height=32)))


def test_env_swarm_gap_crossing_replay():
    """Sequential swarm spawns, pairwise collisions, drone spheres in the
    render, swarm observation and the gap-crossing reward, bit for bit."""
    g = golden("env_swarm")
    env = _replay("env_swarm", swarm_config(), 2, ["gap"])
    assert env.swarm
    cfg = swarm_config()
    scenes = []
    for spec in cfg.scenes:
        t = spec.materialize().arrays
        scenes.append(oracle.OracleScene(t.prim_type, t.prim_data, t.prim_object_id, t.prim_aabb_lo, t.prim_aabb_hi))
    env = OracleEnv(cfg, scenes, QuadParams(), SimConfig(), ControllerGains())
    obs = env.reset(seed=2)
    assert np.array_equal(obs["swarm"], g["swarm_obs"][0])
    for t in range(g["actions"].shape[0]):
        obs = env.step(g["actions"][t])[0]
        assert np.array_equal(obs["swarm"], g["swarm_obs"][t + 1]), t


def multiscene_config():
    """make_golden.py multiscene_config: 3 scenes, shuffled assignment, depth + segmentation, CTBR."""
    from paper_2407_14783_b200.env import DistSpec, EnvConfig, InitRandomization, SceneSpec, SensorSpec

    return EnvConfig(
        num_agents=9, command_type="ctbr", episode_max_steps=15, scene_sampling="shuffled",
        scenes=(SceneSpec(kind="garage"), SceneSpec(kind="cluttered", seed=3, density=0.2),
                SceneSpec(kind="cluttered", seed=8, density=0.12)),
        randomization=InitRandomization(position=DistSpec("uniform", low=[-3.5, -3.5, 0.8], high=[3.5, 3.5, 3.0])),
        sensors=(SensorSpec(kind="depth", name="depth", width=32, height=24),
                 SensorSpec(kind="segmentation", name="vision", width=32, height=24)))


def test_env_multiscene_replay():
    """Shuffled scene permutation, per-respawn scene rotation, per-scene renders."""
    _replay("env_multiscene", multiscene_config(), 11, ["garage", "c3", "c8"])
