"""The batched scripted policies drive real GPU envs end to end: commands are
built on the device from the env's device state, observation targets and
nearest points, and the tasks' success baselines are reached (reference
env/policies.py:1-8: the policies are the shipped tasks' success baselines).
The policies' arithmetic is pinned to the reference in tests/test_policies.py;
here the same policy evaluated on host copies of the inputs must agree."""

import dataclasses
from types import SimpleNamespace as NS

import pytest

from paper_2407_14783_b200.env import gap_crossing_config, landing_config, make_env, navigation_config
from paper_2407_14783_b200.env import policies as pol

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def host_env(env):
    s = env.state
    return NS(num_agents=env.num_agents, config=env.config, params=env.params, sensor_cameras=env.sensor_cameras,
              state=NS(position_w=s.position_w.double().cpu(), orientation=s.orientation.double().cpu()),
              nearest_pt=env.nearest_pt.cpu())


@pytest.mark.parametrize("task,policy,steps", [
    ("nav", "potential_field", 400), ("landing", "land", 400), ("gap", "gap_slotted", 600),
])
def test_policy_drives_env_on_device(task, policy, steps):
    cfg = {"nav": lambda: navigation_config(0, 64), "landing": lambda: landing_config(64),
           "gap": lambda: gap_crossing_config(1.0, 3)}[task]()
    env = make_env(cfg)
    obs = env.reset(seed=3)
    p = pol.make_policy(policy, env)
    p.reset(obs)
    ever = torch.zeros(env.num_agents, dtype=torch.bool, device="cuda")
    for t in range(steps):
        if t < 3 and policy != "gap_slotted":  # device evaluation == host evaluation of the same inputs
            hp = pol.make_policy(policy, host_env(env))
            hp.reset(obs)
            if policy == "potential_field":
                hp._side = p._side.cpu()
            tgt = {"target": obs["target"].double().cpu()}
            ref = hp(tgt, t)
        cmd = p(obs, t)
        assert cmd.velocity.is_cuda
        if t < 3 and policy != "gap_slotted":
            torch.testing.assert_close(cmd.velocity.cpu(), ref.velocity, rtol=0, atol=1e-12)
        res = env.step(cmd)
        obs = res.observations
        ever |= env.get_success()
    assert int(ever.sum()) >= 1, f"{policy}: no agent reached the {task} goal in {steps} steps"
