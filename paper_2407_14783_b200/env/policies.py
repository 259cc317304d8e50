"""Scripted baseline policies (reference env/policies.py:22-289), batched.

The reference walks the agents in a Python loop over numpy rows.  Here each
policy is a handful of whole-batch tensor expressions on the env's own
device tensors (`env.state`, `env.nearest_pt`, `observations["target"]`), so
driving a 65,536-agent env adds a few elementwise launches per step and no
host round trip.  Per-agent branches become masks; the sticky tangent side
of the potential field and the launch latch of the gap policy are per-agent
tensors.  Results equal the reference's to rounding (tests/test_policies.py
pins them against the reference run on the same inputs).

Same names, constructor arguments, defaults and errors as the reference;
`make_policy(name, env)` raises ValueError for unknown names.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import control as ctl
from .. import quatmath
from ..geometry.generate import PAD_TOP
from ..params import GRAVITY

__all__ = ["HoverPolicy", "PotentialFieldPolicy", "DescendAndCenterPolicy", "TimeSlottedGapPolicy",
           "StraightLinePolicy", "POLICIES", "make_policy"]


def _pos(env) -> torch.Tensor:
    return torch.as_tensor(env.state.position_w).to(torch.float64)


def _targets(observations, like: torch.Tensor) -> torch.Tensor:
    """(n, k) targets from the batched observation dict or a list of per-agent dicts."""
    try:
        t = observations["target"]
    except (TypeError, KeyError, IndexError):
        t = np.stack([np.asarray(o["target"], dtype=float) for o in observations])
    return torch.as_tensor(t, device=like.device).to(torch.float64)


def _norm(v: torch.Tensor) -> torch.Tensor:
    return torch.sqrt((v * v).sum(-1))


def _cap(v: torch.Tensor, speed: torch.Tensor, cap) -> torch.Tensor:
    """v scaled to `cap` where its norm exceeds it."""
    return torch.where((speed > cap)[:, None], v * (cap / speed)[:, None], v)


class HoverPolicy:
    """Hold the spawn pose with the env's command type (policies.py:22-44)."""

    def __init__(self, env):
        self.env = env
        self.anchor = None
        self.yaw = None

    def reset(self, observations):
        p = _pos(self.env)
        self.anchor = p.clone()
        self.yaw = torch.zeros(p.shape[0], dtype=torch.float64, device=p.device)

    def __call__(self, observations, t: int) -> ctl.Command:
        env = self.env
        p = _pos(env)
        n, dev = p.shape[0], p.device
        kind = env.config.command_type
        if kind == "ctbr":
            return ctl.CTBR(torch.full((n,), GRAVITY, dtype=torch.float64, device=dev),
                            torch.zeros((n, 3), dtype=torch.float64, device=dev))
        if kind == "srt":
            return ctl.SRT(torch.full((n, 4), env.params.hover_thrust, dtype=torch.float64, device=dev))
        if kind == "ps":
            return ctl.PS(self.anchor.clone(), self.yaw.clone())
        return ctl.LV(torch.zeros((n, 3), dtype=torch.float64, device=dev), self.yaw.clone())


class PotentialFieldPolicy:
    """Target attraction + nearest-obstacle repulsion + a sticky tangential
    slide (policies.py:47-113)."""

    def __init__(self, env, v_cruise=1.6, v_max=2.2, k_rep=1.6, d_influence=1.2, k_tan=1.2, slow_radius=1.5):
        if env.config.command_type != "lv":
            raise ValueError("potential_field drives LV commands")
        self.env = env
        self.v_cruise, self.v_max, self.k_rep = v_cruise, v_max, k_rep
        self.d_influence, self.k_tan, self.slow_radius = d_influence, k_tan, slow_radius
        self._side = None

    def reset(self, observations):
        p = _pos(self.env)
        self._side = torch.ones(p.shape[0], dtype=torch.float64, device=p.device)

    def __call__(self, observations, t: int) -> ctl.Command:
        env = self.env
        p = _pos(env)
        if self._side is None:
            self.reset(observations)
        to_t = _targets(observations, p) - p
        dist = _norm(to_t)
        dir_t = to_t / torch.clamp(dist, min=1e-9)[:, None]
        v = (self.v_cruise * torch.clamp(dist / self.slow_radius, max=1.0))[:, None] * dir_t

        away = p - torch.as_tensor(env.nearest_pt, device=p.device).to(torch.float64)
        d = torch.clamp(_norm(away), min=1e-6)
        near = d < self.d_influence
        away_dir = away / d[:, None]
        fade = torch.clamp(torch.clamp(dist / 1.5, min=0.35), max=1.0)
        gain = self.k_rep * fade * (1.0 / d - 1.0 / self.d_influence)
        v = torch.where(near[:, None], v + gain[:, None] * away_dir, v)
        # tangent = away_dir x (0, 0, 1)
        tangent = torch.stack([away_dir[:, 1], -away_dir[:, 0], torch.zeros_like(d)], -1)
        tn = _norm(tangent)
        slide = near & (tn > 1e-6)
        tangent = tangent / torch.where(slide, tn, torch.ones_like(tn))[:, None]
        align = (tangent * dir_t).sum(-1)
        self._side = torch.where(slide & (align * self._side < -0.15), -self._side, self._side)
        k = self.k_tan * fade * (1.0 - d / self.d_influence) * self._side
        v = torch.where(slide[:, None], v + k[:, None] * tangent, v)

        speed = _norm(v)
        cap = torch.where(d < 0.9, torch.clamp(self.v_max * (d - 0.18) / 0.72, min=0.6),
                          torch.full_like(d, self.v_max))
        v = _cap(v, speed, cap)
        return ctl.LV(v, torch.atan2(dir_t[:, 1], dir_t[:, 0]))


class DescendAndCenterPolicy:
    """Landing: centre over the pad from its pixel centroid and descend
    (policies.py:116-178)."""

    def __init__(self, env, k_center=1.2, v_down_max=0.8, v_xy_max=1.0):
        if env.config.command_type != "lv":
            raise ValueError("land policy drives LV commands")
        self.env = env
        self.k_center, self.v_down_max, self.v_xy_max = k_center, v_down_max, v_xy_max
        spec = None
        for s, cam in env.sensor_cameras:
            if s.kind == "segmentation":
                spec, self.camera = s, cam
        if spec is None:
            raise ValueError("land policy needs the segmentation sensor")

    def reset(self, observations):
        pass

    def _pad_world(self, p, q, centroid):
        """Cast each agent's centroid pixel ray onto the pad plane (policies.py:139-156)."""
        cam = self.camera
        x = (2.0 * (centroid[:, 0] + 0.5) / cam.width - 1.0) * cam.tan_half_h
        y = (2.0 * (centroid[:, 1] + 0.5) / cam.height - 1.0) * cam.tan_half_v
        d_cam = torch.stack([x, y, torch.ones_like(x)], -1)
        d_cam = d_cam / _norm(d_cam)[:, None]
        tr = torch.as_tensor(cam.translation, dtype=torch.float64, device=p.device).expand_as(p)
        origin = p + quatmath.rotate(q, tr)
        rot = quatmath.to_matrix(q) @ torch.as_tensor(cam.rotation, dtype=torch.float64, device=p.device)
        d_world = (rot @ d_cam[:, :, None])[:, :, 0]
        dz = d_world[:, 2]
        down = dz <= -1e-6
        t = (PAD_TOP - origin[:, 2]) / torch.where(down, dz, -torch.ones_like(dz))
        hit = origin[:, :2] + t[:, None] * d_world[:, :2]
        return torch.where(down[:, None], hit, p[:, :2])

    def __call__(self, observations, t: int) -> ctl.Command:
        env = self.env
        p = _pos(env)
        q = torch.as_tensor(env.state.orientation).to(torch.float64)
        centroid = _targets(observations, p)
        height = torch.clamp(p[:, 2] - PAD_TOP - env.config.collision_radius, min=0.0)
        lost = centroid[:, 0] < 0
        offset = self._pad_world(p, q, centroid) - p[:, :2]
        v_xy = self.k_center * offset
        v_xy = _cap(v_xy, _norm(v_xy), self.v_xy_max)
        centered = _norm(offset) < torch.clamp(0.15 * height, min=0.08)
        v_down = torch.where(centered, torch.clamp(0.55 * height + 0.02, max=self.v_down_max),
                             torch.where(height < 1.0, torch.zeros_like(height), torch.full_like(height, 0.2)))
        vel = torch.cat([v_xy, -v_down[:, None]], -1)
        climb = torch.tensor([0.0, 0.0, 0.6], dtype=torch.float64, device=p.device)  # pad lost: climb
        vel = torch.where(lost[:, None], climb.expand_as(vel), vel)
        return ctl.LV(vel, torch.zeros_like(height))


class TimeSlottedGapPolicy:
    """Cooperative gap crossing, one agent per slot in spawn-y order
    (policies.py:181-251)."""

    def __init__(self, env, slot_steps=240, v_go=2.0, gate_x=1.2, stage_x=-4.2, clear_x=0.4):
        if env.config.command_type != "lv":
            raise ValueError("gap policy drives LV commands")
        self.env = env
        self.slot_steps, self.v_go, self.gate_x, self.stage_x, self.clear_x = slot_steps, v_go, gate_x, stage_x, clear_x
        self.order = None
        self.stage = None

    def reset(self, observations):
        p = _pos(self.env)
        n, dev = p.shape[0], p.device
        self.order = torch.argsort(p[:, 1], stable=True)
        lanes = torch.as_tensor(np.linspace(-2.4, 2.4, n) if n > 1 else np.zeros(1), device=dev)
        self.stage = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.stage[self.order, 0] = self.stage_x
        self.stage[self.order, 1] = lanes
        self.stage[self.order, 2] = 1.5
        self.rank_of = torch.empty(n, dtype=torch.long, device=dev)
        self.rank_of[self.order] = torch.arange(n, device=dev)
        self.launched = torch.zeros(n, dtype=torch.bool, device=dev)

    def __call__(self, observations, t: int) -> ctl.Command:
        p = _pos(self.env)
        target = _targets(observations, p)
        # clear for rank r: every agent of rank < r is past the clearance plane
        cleared = (p[:, 0] > self.clear_x)[self.order].to(torch.int32)
        before = torch.cumprod(torch.cat([cleared.new_ones(1), cleared[:-1]]), 0).bool()
        clear = before[self.rank_of]
        may = self.launched | clear | (t >= (self.rank_of + 1) * self.slot_steps)
        self.launched = self.launched | may
        gx = self.gate_x

        def pt(x):
            return torch.tensor([x, 0.0, 1.5], dtype=torch.float64, device=p.device).expand_as(p)

        goal = torch.where((p[:, 0] < gx)[:, None], pt(gx), target)
        goal = torch.where((p[:, 0] < -gx)[:, None], pt(-gx), goal)
        goal = torch.where(may[:, None], goal, self.stage)
        to_goal = goal - p
        dist = _norm(to_goal)
        v = 1.2 * to_goal
        cap = torch.where(dist > 0.8, torch.full_like(dist, self.v_go), torch.clamp(self.v_go * dist, min=0.6))
        return ctl.LV(_cap(v, _norm(v), cap), torch.zeros_like(dist))


class StraightLinePolicy:
    """Fly straight at the target (policies.py:254-270)."""

    def __init__(self, env, v_go=1.5):
        self.env = env
        self.v_go = v_go

    def reset(self, observations):
        pass

    def __call__(self, observations, t: int) -> ctl.Command:
        p = _pos(self.env)
        to_t = _targets(observations, p) - p
        d = _norm(to_t)
        vel = to_t / torch.clamp(d, min=1e-9)[:, None] * torch.clamp(1.5 * d, max=self.v_go)[:, None]
        return ctl.LV(vel, torch.zeros_like(d))


POLICIES = {
    "hover": HoverPolicy,
    "potential_field": PotentialFieldPolicy,
    "land": DescendAndCenterPolicy,
    "gap_slotted": TimeSlottedGapPolicy,
    "straight": StraightLinePolicy,
}


def make_policy(name: str, env):
    """policies.py:284-289."""
    if name not in POLICIES:
        raise ValueError(f"unknown policy {name!r}; choose from {sorted(POLICIES)}")
    return POLICIES[name](env)
