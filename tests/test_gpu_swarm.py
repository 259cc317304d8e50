"""GPU parity of swarm mode: sequential swarm spawns, pairwise
collisions, other agents rendered as spheres, the swarm observation and the
gap-crossing task, against the reference episode (env_swarm.npz) and the
oracle evaluated on the GPU's own state."""

import dataclasses

import numpy as np
import pytest

import oracle
from conftest import golden
from oracle.env import OracleEnv
from parity_util import state_error
from test_oracle import swarm_config

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2407_14783_b200.control import command_from_array  # noqa: E402
from paper_2407_14783_b200.env import make_env  # noqa: E402
from paper_2407_14783_b200.errors import ConfigError  # noqa: E402
from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig  # noqa: E402


def _planes(env):
    return env._planes.T.double().cpu().numpy()


def test_swarm_episode_fp64_replay():
    g = golden("env_swarm")
    cfg = swarm_config()
    env = make_env(cfg, dtype=torch.float64)
    obs = env.reset(seed=2)
    assert np.array_equal(_planes(env), g["reset_full_state"])  # sequential swarm spawns
    assert np.array_equal(obs["swarm"].cpu().numpy(), g["swarm_obs"][0])
    worst = 0.0
    for t in range(g["actions"].shape[0]):
        res = env.step(command_from_array("ctbr", g["actions"][t]))
        worst = max(worst, state_error(_planes(env), g["full_state"][t]).max())
        assert np.array_equal(env.collision.cpu().numpy(), g["collision"][t]), t
        assert np.array_equal(res.terminated.cpu().numpy(), g["terminated"][t]), t
        assert np.array_equal(res.truncated.cpu().numpy(), g["truncated"][t]), t
        assert np.array_equal(res.info["success"].cpu().numpy(), g["success"][t]), t
        np.testing.assert_allclose(res.reward.cpu().numpy(), g["reward"][t].astype(np.float32), rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(res.observations["swarm"].cpu().numpy(), g["swarm_obs"][t + 1], rtol=0, atol=1e-12)
        np.testing.assert_array_equal(res.observations["target"].cpu().numpy(), g["target"][t])
        for key in g.files:
            if key.startswith("img_") and key.endswith(f"_{t}"):
                sensor = key[4:].rsplit("_", 1)[0]
                img = res.observations[sensor].double().cpu().numpy()
                if sensor == "vision":  # ids incl. DRONE_ID0 + j spheres
                    assert np.array_equal(img, g[key]), (key, int((img != g[key]).sum()))
                else:
                    assert np.abs(img - g[key]).max() < 1e-9, key
    assert worst < 1e-12, worst


def test_swarm_fp32_flags_on_own_state():
    """FP32 build: pairwise collisions, gap rewards and flags equal the
    reference hooks evaluated on the GPU's own state."""
    cfg = swarm_config()
    env = make_env(cfg)
    env.reset(seed=2)
    scenes = []
    for spec in cfg.scenes:
        t = spec.materialize().arrays
        scenes.append(oracle.OracleScene(t.prim_type, t.prim_data, t.prim_object_id, t.prim_aabb_lo, t.prim_aabb_hi))
    orc = OracleEnv(cfg, scenes, QuadParams(), SimConfig(), ControllerGains())
    orc.reset(seed=2)
    rng = np.random.default_rng(9)
    pair_hits = 0
    for t in range(80):
        a = np.concatenate([rng.uniform(2.0, 22.0, (6, 1)), rng.normal(scale=6.0, size=(6, 3))], axis=1)
        prev = _planes(env)
        res = env.step(command_from_array("ctbr", a))
        st = _planes(env)
        orc.state, orc.prev_state = st.copy(), env._prev.T.double().cpu().numpy()
        orc.agent_scene[:] = 0
        orc._refresh_proximity()
        assert np.array_equal(env.collision.cpu().numpy(), orc.collision), t
        pair_hits += int((orc.collision & (orc.nearest_dist >= cfg.collision_radius)).sum())
        succ = orc.get_success()
        rew = orc.get_reward()
        assert np.array_equal(res.info["success"].cpu().numpy(), succ), t
        np.testing.assert_allclose(res.reward.cpu().numpy(), rew.astype(np.float32), rtol=2e-7, atol=1e-7)
        del prev
    assert pair_hits > 0  # the episode exercised agent-agent collisions


def test_swarm_mode_refuses_sharding():
    with pytest.raises(ConfigError):
        make_env(swarm_config(), shard=(0, 2))


def test_swarm_spheres_in_fp32_render():
    """Drone spheres appear in the FP32 segmentation with their ids."""
    cfg = dataclasses.replace(swarm_config(), sensors=swarm_config().sensors[1:])
    env = make_env(cfg)
    obs = env.reset(seed=2)
    seg = obs["vision"].cpu().numpy()
    assert (seg >= 60000).any()
    assert set(np.unique(seg[seg >= 60000])) <= {60000 + j for j in range(6)}
