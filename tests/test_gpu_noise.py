"""GPU parity of the sensor half of the observation: device
standard normals / Poisson draws against numpy's Generator, sensing.apply_noise
on the GPU against the reference's own outputs, the ideal IMU, and a noisy
episode (normal-distribution spawns, depth + IMU + segmentation noise chains)
replayed bit for bit in the FP64 build."""

import dataclasses

import numpy as np
import pytest

from conftest import golden
from oracle.env import apply_noise as oracle_apply_noise
from oracle.env import imu_readings
from test_oracle import NOISE_CASES, noise_config

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2407_14783_b200._native as nat  # noqa: E402
from paper_2407_14783_b200 import sensing  # noqa: E402
from paper_2407_14783_b200.control import command_from_array  # noqa: E402
from paper_2407_14783_b200.env import make_env  # noqa: E402
from paper_2407_14783_b200.sensing import NoiseSpec  # noqa: E402


def _streams(seed, n):
    rng = torch.empty((n, 4), dtype=torch.int64, device="cuda")
    nat.check(nat.lib().qb_rng_seed(seed, n, nat.ptr(rng), nat.stream_of()))
    return rng


def test_device_standard_normals_match_numpy():
    n, k, seed = 64, 4000, 31
    rng = _streams(seed, n)
    out = torch.empty((n, k), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().qb_rng_normals(n, nat.ptr(rng), k, nat.ptr(out), nat.stream_of()))
    got = out.cpu().numpy()
    ref = np.stack([np.random.default_rng(seed + i).standard_normal(k) for i in range(n)])
    bad = got != ref
    # wedge and tail draws go through log1p / exp (CUDA libm vs glibc, <= 1 ulp):
    # any difference must be an ulp-level tail value, never a shifted stream
    assert bad.sum() <= 2, np.argwhere(bad)[:5]
    if bad.any():
        np.testing.assert_allclose(got[bad], ref[bad], rtol=1e-15)
        assert np.all(np.abs(ref[bad]) > 3.6)
    # stream state after the draws: the next word equals numpy's
    nxt = torch.empty((n, 1), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().qb_rng_doubles(n, nat.ptr(rng), 1, nat.ptr(nxt), nat.stream_of()))
    g = [np.random.default_rng(seed + i) for i in range(n)]
    for gi in g:
        gi.standard_normal(k)
    assert np.array_equal(nxt.cpu().numpy()[:, 0], np.array([gi.random() for gi in g]))


def test_device_poissons_match_numpy():
    n, k, seed = 48, 300, 5
    lam = np.random.default_rng(0).uniform(0.0, 120.0, (n, k))
    lam[:, ::3] = np.random.default_rng(1).uniform(0.0, 10.0, lam[:, ::3].shape)
    lam[:, ::17] = 0.0
    rng = _streams(seed, n)
    lam_d = torch.as_tensor(lam, device="cuda")
    out = torch.empty((n, k), dtype=torch.int64, device="cuda")
    nat.check(nat.lib().qb_rng_poissons(n, nat.ptr(rng), k, nat.ptr(lam_d), nat.ptr(out), nat.stream_of()))
    ref = np.stack([np.random.default_rng(seed + i).poisson(lam[i]) for i in range(n)])
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("case", range(len(NOISE_CASES)))
def test_apply_noise_on_gpu_matches_reference(case):
    """sensing.apply_noise: the reference's outputs for the same Generator, and
    the Generator left in the same state (same number of draws)."""
    g = golden("noise")
    sensor, kind, kw = NOISE_CASES[case]
    rng = np.random.default_rng(100 + case)
    out = sensing.apply_noise(g[f"case{case}_in"], NoiseSpec(kind, **kw), rng, sensor=sensor)
    assert np.array_equal(out, g[f"case{case}_out"])
    assert np.array_equal(rng.random(2), g[f"case{case}_after"])


def test_apply_noise_rejects_invalid_sensor_kinds():
    from paper_2407_14783_b200.errors import InvalidNoiseForSensor

    with pytest.raises(InvalidNoiseForSensor):
        sensing.apply_noise(np.zeros(6), NoiseSpec("poisson", scaling=1.0), np.random.default_rng(0), sensor="imu")
    with pytest.raises(InvalidNoiseForSensor):
        sensing.apply_noise(np.zeros((4, 4)), NoiseSpec("redwood"), np.random.default_rng(0), sensor="segmentation")


def test_env_noise_episode_fp64_bit_exact():
    """Normal-distribution spawns (device ziggurat) and the noisy depth / IMU /
    segmentation observations of the reference episode, bit for bit."""
    g = golden("env_noise")
    env = make_env(noise_config(), dtype=torch.float64)
    obs = env.reset(seed=4)
    assert np.array_equal(env._planes.T.cpu().numpy(), g["reset_full_state"])
    keep = list(g["obs_steps"])
    snaps = {0: {k: obs[k].cpu().numpy() for k in ("depth", "imu", "vision")}}
    for t in range(1, 21):
        res = env.step(command_from_array("ctbr", torch.as_tensor(g["actions"][t - 1], device="cuda")))
        assert np.array_equal(env._planes.T.cpu().numpy(), g["full_state"][t - 1]), t
        if t in keep:
            snaps[t] = {k: res.observations[k].cpu().numpy() for k in ("depth", "imu", "vision")}
    for j, t in enumerate(keep):
        for key in ("depth", "imu", "vision"):
            got, ref = snaps[t][key], g[f"obs_{key}"][j]
            assert np.array_equal(got, ref), (key, t, int((got != ref).sum()))


def test_env_imu_fp32_on_own_state():
    """FP32 build: the IMU reading equals the reference formula evaluated on
    the GPU's own state (computed in double, stored as float32)."""
    from paper_2407_14783_b200.env import SensorSpec

    cfg = dataclasses.replace(noise_config(), sensors=(SensorSpec(kind="imu", name="imu"),))
    env = make_env(cfg)
    env.reset(seed=2)
    import oracle

    for _ in range(3):
        a = torch.randn((env.num_agents, 4), device="cuda")
        a[:, 0] = 9.0 + a[:, 0]
        res = env.step(command_from_array("ctbr", a))
        st = env._planes.T.double().cpu().numpy()
        ref = imu_readings(st, oracle.pack_params(env.params, env.sim, env.gains)).astype(np.float32)
        assert np.array_equal(res.observations["imu"].cpu().numpy(), ref)


def test_env_noise_fp32_close_to_fp64():
    """FP32 noisy observations follow the FP64 ones: same draws, clean values
    within the FP32 render tolerance (a few pixels may flip at grazing edges)."""
    cfg = noise_config()
    e32, e64 = make_env(cfg), make_env(cfg, dtype=torch.float64)
    o32, o64 = e32.reset(seed=4), e64.reset(seed=4)
    d32, d64 = o32["depth"].double().cpu().numpy(), o64["depth"].cpu().numpy()
    diff = np.abs(d32 - d64)
    assert np.median(diff) < 1e-5 and np.mean(diff > 1e-3) < 0.01
    v32, v64 = o32["vision"].double().cpu().numpy(), o64["vision"].cpu().numpy()
    assert np.mean(v32 != v64) < 0.01
    np.testing.assert_allclose(o32["imu"].double().cpu().numpy(), o64["imu"].cpu().numpy(), atol=1e-5, rtol=1e-5)


def test_oracle_noise_on_gpu_clean_render():
    """The env's noisy depth = the reference noise chain applied (per agent,
    on the agent's generator) to the env's own clean render."""
    from paper_2407_14783_b200.env import SensorSpec

    cfg = dataclasses.replace(noise_config(), sensors=(SensorSpec(kind="depth", name="depth", noise=(
        NoiseSpec("normal", sigma=0.02), NoiseSpec("poisson", scaling=50.0), NoiseSpec("saltpepper", p=0.02))),))
    env = make_env(cfg, dtype=torch.float64)
    obs = env.reset(seed=4)
    # advance the reference generators past the spawn draws: replay spawns on the oracle
    import oracle as orc
    from oracle.env import OracleEnv
    from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig

    scenes = []
    for spec in cfg.scenes:
        t = spec.materialize().arrays
        scenes.append(orc.OracleScene(t.prim_type, t.prim_data, t.prim_object_id, t.prim_aabb_lo, t.prim_aabb_hi))
    oenv = OracleEnv(dataclasses.replace(cfg, sensors=()), scenes, QuadParams(), SimConfig(), ControllerGains())
    oenv.reset(seed=4)
    clean = env._sensor_slot["depth"]["depth"].cpu().numpy()
    for i in range(env.num_agents):
        img = clean[i]
        for nz in cfg.sensors[0].noise:
            img = oracle_apply_noise(img, nz, oenv.rngs[i], "depth")
        assert np.array_equal(obs["depth"][i].cpu().numpy(), img), i


@pytest.mark.parametrize("size", [1, 31, 33, 91, 1000, 4099])
def test_apply_noise_ragged_sizes(size):
    """The warp-per-env sensor pass on image sizes that are not multiples of
    the 32-pixel round (partial first / last rounds, rounds restarting
    mid-window after a slow ziggurat draw), every chain kind without Poisson,
    against the reference noise model on numpy's own Generator."""
    specs = [NoiseSpec("normal", sigma=0.05), NoiseSpec("normal", sigma=0.0), NoiseSpec("speckle", sigma=0.1),
             NoiseSpec("saltpepper", p=0.1), NoiseSpec("saltpepper", p=0.0),
             NoiseSpec("redwood", sigma_disparity=0.01, quantization=0.05), NoiseSpec("redwood", quantization=0.02)]
    data = np.random.default_rng(size).uniform(0.3, 10.0, size)
    for j, spec in enumerate(specs):
        seed = 1000 * size + j
        got = sensing.apply_noise(data, spec, np.random.default_rng(seed), sensor="depth")
        r = np.random.default_rng(seed)
        ref = oracle_apply_noise(data, spec, r, "depth")
        g2 = np.random.default_rng(seed)
        sensing.apply_noise(data, spec, g2, sensor="depth")
        assert np.array_equal(g2.random(2), r.random(2)), spec  # same words consumed
        bad = got != ref
        # ziggurat wedge / tail draws use CUDA's exp / log1p (<= 1 ulp from glibc)
        assert bad.sum() <= 1, (spec, np.argwhere(bad)[:5])
        if bad.any():
            np.testing.assert_allclose(got[bad], ref[bad], rtol=1e-12)
