"""The two-phase env step (qb_env_step_phase: dynamics, then proximity /
reward / flags on a side stream under the observation render) gives exactly
the fused qb_env_step's results: states, rewards, flags, nearest points and
observations bit for bit, respawns included."""

import dataclasses

import numpy as np
import pytest

from paper_2407_14783_b200.control import LV
from paper_2407_14783_b200.env import landing_config, make_env, navigation_config

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _cfgs():
    nav = dataclasses.replace(navigation_config(0, 100, with_segmentation=True), episode_max_steps=40)
    mesh = dataclasses.replace(nav, scenes=tuple(dataclasses.replace(sc, kind="cluttered_mesh") for sc in nav.scenes))
    from paper_2407_14783_b200.env import SensorSpec
    from paper_2407_14783_b200.sensing import NoiseSpec

    noisy = dataclasses.replace(nav, sensors=(
        SensorSpec(kind="depth", name="depth", noise=(NoiseSpec("normal", sigma=0.02),)),
        SensorSpec(kind="segmentation", name="segmentation", noise=(NoiseSpec("saltpepper", p=0.02),)),
        SensorSpec(kind="imu", name="imu", noise=(NoiseSpec("normal", sigma=0.05),))))
    return {"nav": nav, "mesh": mesh, "landing": dataclasses.replace(landing_config(64), episode_max_steps=30),
            "noisy": noisy}


@pytest.mark.parametrize("name", ["nav", "mesh", "landing", "noisy"])
def test_split_step_equals_fused(name):
    cfg = _cfgs()[name]
    a, b = make_env(cfg), make_env(cfg)
    assert a.split_step
    b.split_step = False
    oa, ob = a.reset(seed=5), b.reset(seed=5)
    g = torch.Generator(device="cuda").manual_seed(1)
    n = cfg.num_agents
    for t in range(60):
        v = torch.randn(n, 3, device="cuda", generator=g) * 2.0
        yaw = torch.randn(n, device="cuda", generator=g)
        ra, rb = a.step(LV(v, yaw)), b.step(LV(v, yaw))
        torch.cuda.synchronize()
        for k in ("state", "depth", "segmentation", "target", "imu"):
            if k in rb.observations:
                assert torch.equal(ra.observations[k], rb.observations[k]), (t, k)
        assert torch.equal(a._planes, b._planes), t
        for x, y in ((ra.reward, rb.reward), (ra.terminated, rb.terminated), (ra.truncated, rb.truncated),
                     (a.nearest_pt, b.nearest_pt), (a.nearest_dist, b.nearest_dist), (a.collision, b.collision),
                     (a.step_counts, b.step_counts)):
            assert torch.equal(torch.as_tensor(x), torch.as_tensor(y)), t
    assert int(b.step_counts.max()) < 60  # episodes ended and respawned along the way
