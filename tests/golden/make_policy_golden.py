"""Golden vectors for the scripted policies (reference env/policies.py:22-289),
made by RUNNING THE REFERENCE's policy classes in the build container on
seeded synthetic inputs (a stand-in env object carrying exactly the fields the
policies read: state, nearest_pt, config, params, sensor_cameras):

    python tests/golden/make_policy_golden.py [/root/reference/pkg/src]

Writes tests/golden/policies.npz.
"""

from __future__ import annotations

import os
import sys
from types import SimpleNamespace as NS

import numpy as np

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
from quadsim import quatmath as qm  # noqa: E402
from quadsim import sensing  # noqa: E402
from quadsim.env import policies as pol  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "policies.npz")
CALLS = 6


def fake_env(n, kind="lv"):
    cam = sensing.CameraModel(rotation=sensing.DOWNWARD)
    return NS(num_agents=n, config=NS(command_type=kind, collision_radius=0.15),
              state=NS(position_w=np.zeros((n, 3)), orientation=np.tile([1.0, 0, 0, 0], (n, 1))),
              nearest_pt=np.zeros((n, 3)), params=NS(hover_thrust=0.75 * 9.81 / 4.0),
              sensor_cameras=[(NS(kind="depth"), cam), (NS(kind="segmentation"), cam)])


def cmd_arrays(c):
    return {k: np.asarray(v, dtype=float) for k, v in vars(c).items()}


def main():
    rng = np.random.default_rng(14783)
    out = {}
    n = 64
    # potential field: targets fixed, positions drift, nearest points inside / outside the influence radius
    env = fake_env(n)
    p = pol.PotentialFieldPolicy(env)
    target = rng.uniform([-4, -4, 1], [4, 4, 3], size=(n, 3))
    obs = [{"target": target[i]} for i in range(n)]
    p.reset(obs)
    out["pf_target"] = target
    for c in range(CALLS):
        pos = rng.uniform([-5, -5, 0.5], [5, 5, 3.5], size=(n, 3))
        off = rng.normal(size=(n, 3))
        off *= (rng.uniform(0.05, 1.8, size=n) / np.linalg.norm(off, axis=1))[:, None]
        if c == 0:
            pos[0] = target[0]  # at the goal
            off[1] = [0.0, 0.0, 0.5]  # obstacle straight below: no tangent
        env.state.position_w, env.nearest_pt = pos, pos - off
        cmd = p(obs, c)
        out[f"pf_pos_{c}"], out[f"pf_near_{c}"] = pos, pos - off
        out[f"pf_vel_{c}"], out[f"pf_yaw_{c}"] = cmd.velocity, cmd.yaw
        out[f"pf_side_{c}"] = p._side.copy()
    # landing: level-ish down-looking cameras above the pad, centroids inside the frame or lost
    env = fake_env(n)
    p = pol.DescendAndCenterPolicy(env)
    for c in range(CALLS):
        pos = rng.uniform([-1, -1, 0.1], [1, 1, 3.0], size=(n, 3))
        q = qm.normalize(np.array([1.0, 0, 0, 0]) + rng.normal(scale=0.08, size=(n, 4)))
        cen = rng.uniform(0, 63, size=(n, 2))
        cen[rng.uniform(size=n) < 0.15] = -1.0
        env.state.position_w, env.state.orientation = pos, q
        cmd = p([{"target": cen[i]} for i in range(n)], c)
        out[f"land_pos_{c}"], out[f"land_q_{c}"], out[f"land_cen_{c}"] = pos, q, cen
        out[f"land_vel_{c}"] = cmd.velocity
    # gap: 8 agents, slotted launches
    m = 8
    env = fake_env(m)
    p = pol.TimeSlottedGapPolicy(env)
    spawn = np.column_stack([rng.uniform(-4.5, -3.5, m), rng.uniform(-2.5, 2.5, m), rng.uniform(1, 2, m)])
    env.state.position_w = spawn
    p.reset(None)
    out["gap_spawn"] = spawn
    gtarget = np.tile([4.0, 0.0, 1.5], (m, 1))
    for c, t in enumerate([0, 100, 240, 300, 480, 1000]):
        pos = np.column_stack([rng.uniform(-5, 3, m), rng.uniform(-2.5, 2.5, m), rng.uniform(1, 2, m)])
        env.state.position_w = pos
        cmd = p([{"target": gtarget[i]} for i in range(m)], t)
        out[f"gap_pos_{c}"], out[f"gap_t_{c}"] = pos, np.array(t)
        out[f"gap_vel_{c}"] = cmd.velocity
        out[f"gap_launched_{c}"] = p.launched.copy()
    # straight line
    env = fake_env(n)
    p = pol.StraightLinePolicy(env)
    pos = rng.uniform(-3, 3, size=(n, 3))
    tgt = pos + rng.normal(size=(n, 3)) * rng.uniform(0, 2, size=(n, 1))
    tgt[0] = pos[0]
    env.state.position_w = pos
    cmd = p([{"target": tgt[i]} for i in range(n)], 0)
    out["sl_pos"], out["sl_target"] = pos, tgt
    out["sl_vel"] = cmd.velocity
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
