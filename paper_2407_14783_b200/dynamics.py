"""Batched vehicle state on the GPU and the dynamics step entry point.

`QuadState` keeps the reference's accessors (dynamics.py:29-92) but stores
the batch field-major, as one (17, N) tensor of planes in the order
p(3) v(3) q(4) omega(3) rotor(4) (dynamics.py:3-8): every per-env kernel
then reads each field with one coalesced 128 B transaction per warp, and
`position_w` / `orientation` / ... are zero-copy (N,k) views.

`step` is dynamics.step (dynamics.py:231-253) executed by the K1 kernel:
clamp commands, per substep exact rotor lag + Euler/RK4 + renormalisation,
finiteness mask -> NonFiniteState.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .errors import NonFiniteState
from .params import QuadParams, SimConfig, native_params

RIGID_DIM = 13
STATE_DIM = 17
_FIELDS = {"position_w": (0, 3), "velocity_w": (3, 6), "orientation": (6, 10), "angvel_b": (10, 13), "rotor_speeds": (13, 17)}


def _default_device():
    import torch

    nat.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


class QuadState:
    """Batched state; `planes` is a contiguous (17, N) CUDA tensor."""

    __slots__ = ("planes",)

    def __init__(self, planes):
        import torch

        if not isinstance(planes, torch.Tensor) or planes.dim() != 2 or planes.shape[0] != STATE_DIM:
            raise ValueError("QuadState expects a (17, N) tensor of planes")
        nat.require_cuda(planes)
        self.planes = planes.contiguous()

    # constructors --------------------------------------------------------
    @classmethod
    def from_vector(cls, vec, device=None, dtype=None) -> "QuadState":
        """(N,17) (numpy or torch) -> QuadState."""
        import torch

        t = torch.as_tensor(vec)
        t = torch.atleast_2d(t)
        dtype = dtype or (t.dtype if t.dtype in (torch.float32, torch.float64) else torch.float64)
        dev = device or (t.device if t.is_cuda else _default_device())
        return cls(t.to(device=dev, dtype=dtype).T.contiguous())

    @classmethod
    def hover(cls, n: int, params: QuadParams = None, position=None, device=None, dtype=None) -> "QuadState":
        import torch

        params = params or QuadParams()
        dev = device or _default_device()
        planes = torch.zeros((STATE_DIM, n), dtype=dtype or torch.float32, device=dev)
        if position is not None:
            planes[0:3] = torch.as_tensor(np.broadcast_to(np.asarray(position, float), (n, 3)).T.copy(), dtype=planes.dtype)
        planes[6] = 1.0
        planes[13:17] = params.hover_speed
        return cls(planes)

    # accessors ------------------------------------------------------------
    def _view(self, name):
        a, b = _FIELDS[name]
        return self.planes[a:b].T

    position_w = property(lambda s: s._view("position_w"))
    velocity_w = property(lambda s: s._view("velocity_w"))
    orientation = property(lambda s: s._view("orientation"))
    angvel_b = property(lambda s: s._view("angvel_b"))
    rotor_speeds = property(lambda s: s._view("rotor_speeds"))

    @property
    def batch_size(self) -> int:
        return self.planes.shape[1]

    @property
    def dtype(self):
        return self.planes.dtype

    @property
    def device(self):
        return self.planes.device

    def as_vector(self):
        """(N,17) in the reference order (a copy)."""
        return self.planes.T.contiguous()

    def numpy(self) -> np.ndarray:
        return self.as_vector().double().cpu().numpy()

    def copy(self) -> "QuadState":
        return QuadState(self.planes.clone())

    def select(self, idx) -> "QuadState":
        return QuadState(self.planes[:, idx : idx + 1].clone())

    def set_agent(self, idx: int, other: "QuadState", other_idx: int = 0):
        self.planes[:, idx] = other.planes[:, other_idx]

    def __repr__(self):
        return f"QuadState(N={self.batch_size}, dtype={self.dtype}, device={self.device})"


@dataclass
class Wrench:
    """Force and torque in the body frame, batched (dynamics.py:95-100)."""

    force_b: object
    torque_b: object


def rotor_thrusts(rotor_speeds, params: QuadParams):
    """dynamics.py:103-106: per-rotor thrust k2 w^2 + k1 w + k0 (elementwise,
    on the input's device; K1 evaluates it fused in the step)."""
    k2, k1, k0 = params.thrust_coeffs
    return k2 * rotor_speeds**2 + k1 * rotor_speeds + k0


def rotor_lag(current, desired, dt: float, params: QuadParams):
    """dynamics.py:109-114: first-order motor response over dt, clamped."""
    import math

    alpha = math.exp(-params.motor_decay * dt)
    out = desired + (current - desired) * alpha
    lo, hi = params.rotor_speed_limits
    return out.clip(lo, hi)


def drag_force(velocity_b, params: QuadParams):
    """dynamics.py:117-120: -c v |v| componentwise, c = 0.5 rho Cd s."""
    import torch

    c = 0.5 * params.air_density * np.asarray(params.drag_coeffs, float) * params.cross_area
    if isinstance(velocity_b, torch.Tensor):
        c = torch.as_tensor(c, dtype=velocity_b.dtype, device=velocity_b.device)
    return -c * velocity_b * abs(velocity_b)


def aggregate_wrench(thrusts, params: QuadParams) -> Wrench:
    """dynamics.py:123-140: collective force (body z) and torques sum_i t_i g_i."""
    import torch

    t = thrusts if thrusts.ndim == 2 else thrusts[None, :]
    g = np.asarray(params.torque_arms, float)
    if isinstance(t, torch.Tensor):
        g = torch.as_tensor(g, dtype=t.dtype, device=t.device)
        force = torch.zeros((t.shape[0], 3), dtype=t.dtype, device=t.device)
        stack = torch.stack
    else:
        force = np.zeros((t.shape[0], 3))
        stack = lambda xs, dim: np.stack(xs, axis=dim)  # noqa: E731
    force[:, 2] = t[:, 0] + t[:, 1] + t[:, 2] + t[:, 3]
    torque = stack([t[:, 0] * g[0, a] + t[:, 1] * g[1, a] + t[:, 2] * g[2, a] + t[:, 3] * g[3, a] for a in range(3)], 1)
    return Wrench(force, torque)


def step(state: QuadState, rotor_speed_commands, config: SimConfig = None, params: QuadParams = None, check: bool = True,
         out: QuadState = None) -> QuadState:
    """Advance every agent one control step on the GPU (dynamics.py:231-253).

    rotor_speed_commands: (N,4) desired rotor speeds.  Returns a new state
    (or writes `out`).  With check=True a host sync tests finiteness and
    raises NonFiniteState(state, mask) like the reference.
    """
    import torch

    nxt = out if out is not None else state.copy()
    if out is not None and out is not state:
        out.planes.copy_(state.planes)
    planes = nxt.planes
    n = planes.shape[1]
    cmd = torch.as_tensor(rotor_speed_commands, dtype=planes.dtype, device=planes.device).reshape(n, 4).contiguous()
    bad = torch.empty(n, dtype=torch.uint8, device=planes.device)
    P = native_params(params, config, None)
    code = nat.QB_F32 if planes.dtype == torch.float32 else nat.QB_F64
    with torch.cuda.device(planes.device):
        nat.check(nat.lib().qb_dynamics_step(P, nat.CMD["rotor"], code, n, planes.stride(0), nat.ptr(planes), nat.ptr(cmd),
                                             None, nat.ptr(bad), nat.stream_of()), "qb_dynamics_step")
    if check:
        mask = bad.bool()
        if bool(mask.any()):
            raise NonFiniteState(nxt, mask.cpu().numpy())
    return nxt


def control_step(state: QuadState, cmd, config: SimConfig = None, params: QuadParams = None, gains=None,
                 nonfinite=None) -> QuadState:
    """Fused controller + dynamics (one K1 launch), in place on `state`.

    Equivalent to step(state, command_to_rotor_speeds(cmd, state, ...)).
    """
    import torch

    from .control import command_kind

    planes = state.planes
    n = planes.shape[1]
    a = torch.as_tensor(cmd.as_array(), dtype=planes.dtype, device=planes.device).reshape(n, 4).contiguous()
    P = native_params(params, config, gains)
    code = nat.QB_F32 if planes.dtype == torch.float32 else nat.QB_F64
    with torch.cuda.device(planes.device):
        nat.check(nat.lib().qb_dynamics_step(P, nat.CMD[command_kind(cmd)], code, n, planes.stride(0), nat.ptr(planes),
                                             nat.ptr(a), None, nat.ptr(nonfinite), nat.stream_of()), "qb_dynamics_step")
    return state
