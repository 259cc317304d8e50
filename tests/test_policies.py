"""Batched scripted policies (env/policies.py) against the reference's own
per-agent policies run on the same inputs (tests/golden/policies.npz,
made by tests/golden/make_policy_golden.py).  The stand-in env carries torch
tensors, as the real env's device state does; rounding differs from numpy's
per-row norms by a few ulp, so velocities are compared at 1e-12 and the
discrete state (sticky tangent side, launch latches) exactly."""

import os
from types import SimpleNamespace as NS

import numpy as np
import pytest
import torch

from paper_2407_14783_b200 import sensing
from paper_2407_14783_b200.env import policies as pol

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "policies.npz"))
T = torch.from_numpy
CALLS = 6


def fake_env(n, kind="lv"):
    cam = sensing.CameraModel(rotation=sensing.DOWNWARD)
    return NS(num_agents=n, config=NS(command_type=kind, collision_radius=0.15),
              state=NS(position_w=torch.zeros((n, 3), dtype=torch.float64),
                       orientation=torch.tensor([[1.0, 0, 0, 0]] * n, dtype=torch.float64)),
              nearest_pt=torch.zeros((n, 3), dtype=torch.float64), params=NS(hover_thrust=0.75 * 9.81 / 4.0),
              sensor_cameras=[(NS(kind="depth"), cam), (NS(kind="segmentation"), cam)])


def close(a, b):
    np.testing.assert_allclose(torch.as_tensor(a).numpy(), b, rtol=0, atol=1e-12)


def test_potential_field_matches_reference():
    env = fake_env(64)
    p = pol.make_policy("potential_field", env)
    obs = {"target": T(G["pf_target"])}
    p.reset(obs)
    for c in range(CALLS):
        env.state.position_w, env.nearest_pt = T(G[f"pf_pos_{c}"]), T(G[f"pf_near_{c}"])
        cmd = p(obs, c)
        close(cmd.velocity, G[f"pf_vel_{c}"])
        close(cmd.yaw, G[f"pf_yaw_{c}"])
        np.testing.assert_array_equal(p._side.numpy(), G[f"pf_side_{c}"])


def test_landing_matches_reference():
    env = fake_env(64)
    p = pol.make_policy("land", env)
    p.reset(None)
    for c in range(CALLS):
        env.state.position_w, env.state.orientation = T(G[f"land_pos_{c}"]), T(G[f"land_q_{c}"])
        cmd = p({"target": T(G[f"land_cen_{c}"])}, c)
        close(cmd.velocity, G[f"land_vel_{c}"])


def test_gap_slotted_matches_reference():
    env = fake_env(8)
    p = pol.make_policy("gap_slotted", env)
    env.state.position_w = T(G["gap_spawn"])
    p.reset(None)
    target = [{"target": np.array([4.0, 0.0, 1.5])} for _ in range(8)]  # list-of-dicts form also accepted
    for c in range(CALLS):
        env.state.position_w = T(G[f"gap_pos_{c}"])
        cmd = p(target, int(G[f"gap_t_{c}"]))
        close(cmd.velocity, G[f"gap_vel_{c}"])
        np.testing.assert_array_equal(p.launched.numpy(), G[f"gap_launched_{c}"])


def test_straight_and_hover():
    env = fake_env(64)
    env.state.position_w = T(G["sl_pos"])
    cmd = pol.make_policy("straight", env)({"target": T(G["sl_target"])}, 0)
    close(cmd.velocity, G["sl_vel"])
    for kind in ("ctbr", "srt", "ps", "lv"):
        env = fake_env(4, kind)
        h = pol.HoverPolicy(env)
        h.reset(None)
        c = h(None, 0)
        assert c.as_array().shape == (4, 4)
    with pytest.raises(ValueError, match="unknown policy"):
        pol.make_policy("nope", env)
    with pytest.raises(ValueError, match="LV"):
        pol.PotentialFieldPolicy(fake_env(2, "ctbr"))
