"""Command types and the cascaded controller entry point.

The four command dataclasses keep the reference's fields and flat layout
(control.py:26-92): SRT thrusts (N,4); CTBR [collective, rates(3)]; PS
[position(3), yaw]; LV [velocity(3), yaw].  Components may be numpy arrays
or CUDA tensors; `as_array()` returns the (N,4) batch in the same container
kind.  The controller itself (CTBR rate loop, LV/PS geometric attitude,
saturating mixer, thrust-curve inverse; control.py:101-252) runs inside the
K1 kernel -- `command_to_rotor_speeds` exposes it on its own.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .params import ControllerGains, QuadParams, SimConfig, native_params


def _cat(cols):
    try:
        import torch

        if any(isinstance(c, torch.Tensor) for c in cols):
            dev = next(c.device for c in cols if isinstance(c, torch.Tensor))
            cols = [torch.as_tensor(c, device=dev) for c in cols]
            dt = torch.float64 if any(c.dtype == torch.float64 for c in cols) else torch.float32
            return torch.cat([c.to(dt) for c in cols], dim=1)
    except ImportError:  # pragma: no cover
        pass
    return np.concatenate([np.asarray(c, dtype=float) for c in cols], axis=1)


def _col(x):
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return torch.atleast_1d(x).reshape(-1, 1)
    except ImportError:  # pragma: no cover
        pass
    return np.atleast_1d(np.asarray(x, dtype=float)).reshape(-1, 1)


def _mat(x, k):
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.reshape(-1, k)
    except ImportError:  # pragma: no cover
        pass
    return np.atleast_2d(np.asarray(x, dtype=float)).reshape(-1, k)


@dataclass
class SRT:
    """Per-rotor thrusts (N) -- (N,4)."""

    thrusts: object

    def as_array(self):
        return _mat(self.thrusts, 4)


@dataclass
class CTBR:
    """Mass-normalised collective thrust (m/s^2) + body rates (rad/s)."""

    collective: object
    body_rates: object

    def as_array(self):
        return _cat([_col(self.collective), _mat(self.body_rates, 3)])


@dataclass
class PS:
    """Position set-point (m, world) + yaw (rad)."""

    position: object
    yaw: object

    def as_array(self):
        return _cat([_mat(self.position, 3), _col(self.yaw)])


@dataclass
class LV:
    """Linear-velocity set-point (m/s, world) + yaw (rad)."""

    velocity: object
    yaw: object

    def as_array(self):
        return _cat([_mat(self.velocity, 3), _col(self.yaw)])


@dataclass
class RotorSpeeds:
    """Desired rotor speeds (rad/s), the action of gradients.step_jacobian."""

    speeds: object

    def as_array(self):
        return _mat(self.speeds, 4)


Command = SRT | CTBR | PS | LV
COMMAND_TYPES = {"srt": SRT, "ctbr": CTBR, "ps": PS, "lv": LV}
_KIND_OF = {SRT: "srt", CTBR: "ctbr", PS: "ps", LV: "lv", RotorSpeeds: "rotor"}


def command_kind(cmd) -> str:
    try:
        return _KIND_OF[type(cmd)]
    except KeyError:
        raise TypeError(f"unsupported command type {type(cmd).__name__}") from None


def command_from_array(kind: str, arr) -> Command:
    arr = _mat(arr, 4)
    kind = kind.lower()
    if kind == "srt":
        return SRT(arr[:, 0:4])
    if kind == "ctbr":
        return CTBR(arr[:, 0], arr[:, 1:4])
    if kind == "ps":
        return PS(arr[:, 0:3], arr[:, 3])
    if kind == "lv":
        return LV(arr[:, 0:3], arr[:, 3])
    if kind == "rotor":
        return RotorSpeeds(arr)
    raise ValueError(f"unknown command kind {kind!r}")


def command_to_rotor_speeds(cmd, state, gains: ControllerGains = None, params: QuadParams = None, sim: SimConfig = None):
    """Dispatch any command to desired rotor speeds (control.py:242-252), on the GPU.

    `state` is a dynamics.QuadState; returns an (N,4) tensor of its dtype
    (numpy in -> numpy out when the command components are numpy arrays).
    """
    import torch

    kind = command_kind(cmd)
    arr = cmd.as_array()
    host = isinstance(arr, np.ndarray)
    planes = state.planes
    a = torch.as_tensor(arr, dtype=planes.dtype, device=planes.device).contiguous()
    n = planes.shape[1]
    if a.shape[0] != n:
        raise ValueError(f"command batch {a.shape[0]} != state batch {n}")
    out = torch.empty((n, 4), dtype=planes.dtype, device=planes.device)
    P = native_params(params, sim, gains)
    code = nat.QB_F32 if planes.dtype == torch.float32 else nat.QB_F64
    with torch.cuda.device(planes.device):
        nat.check(nat.lib().qb_command_to_rotor_speeds(P, nat.CMD[kind], code, n, planes.stride(0), nat.ptr(planes),
                                                       nat.ptr(a), nat.ptr(out), nat.stream_of()), "command_to_rotor_speeds")
    return out.cpu().numpy() if host else out


# ---------------------------------------------------------------------------
# controller stages on their own (control.py:95-139), same kernels as K1


@dataclass
class MixerResult:
    thrusts: object  # (N, 4)
    saturated: object  # (N,) bool


def _stage(stage, rows, state, params, gains, dtype=None, device=None):
    import torch

    host = isinstance(rows, np.ndarray)
    if state is not None:
        planes = state.planes
        dtype, device = planes.dtype, planes.device
    else:
        planes = None
        dtype = dtype or (torch.float64 if host else rows.dtype)
        device = device or (torch.device("cuda", torch.cuda.current_device()) if host else rows.device)
    a = torch.as_tensor(rows, dtype=dtype, device=device).reshape(-1, 4).contiguous()
    n = a.shape[0]
    if planes is not None and planes.shape[1] != n:
        raise ValueError(f"command batch {n} != state batch {planes.shape[1]}")
    out = torch.empty((n, 4), dtype=dtype, device=device)
    flags = torch.empty(n, dtype=torch.uint8, device=device)
    code = nat.QB_F32 if dtype == torch.float32 else nat.QB_F64
    with torch.cuda.device(device):
        nat.check(nat.lib().qb_control_stage(native_params(params, None, gains), stage, code, n,
                                             planes.stride(0) if planes is not None else n, nat.ptr(planes), nat.ptr(a),
                                             nat.ptr(out), nat.ptr(flags), nat.stream_of()), "qb_control_stage")
    if host:
        return out.cpu().numpy(), flags.bool().cpu().numpy()
    return out, flags.bool()


def mixer(collective_force, torque_b, params: QuadParams = None) -> MixerResult:
    """Allocate (collective force, body torque) to per-rotor thrusts
    (control.py:101-130): collective clamped to the total-thrust range, the
    torque scaled down uniformly until every rotor fits its limits."""
    f, tq = _col(collective_force), _mat(torque_b, 3)
    thr, sat = _stage(0, _cat([f, tq]), None, params, None)
    return MixerResult(thr, sat)


def srt_to_rotor_speeds(cmd: SRT, params: QuadParams = None, state=None):
    """control.py:133-135 (clamp thrusts, invert the thrust curve)."""
    if state is None:
        from .dynamics import QuadState

        arr = cmd.as_array()
        state = QuadState.hover(arr.shape[0], params or QuadParams(),
                                dtype=_dtype_of(arr))
    return command_to_rotor_speeds(cmd, state, None, params)


def ctbr_to_rotor_speeds(cmd: CTBR, state, gains: ControllerGains = None, params: QuadParams = None):
    """control.py:138-158: body-rate P loop with gyroscopic feedforward, mixer, thrust inverse."""
    return command_to_rotor_speeds(cmd, state, gains, params)


def lv_to_ctbr(cmd: LV, state, gains: ControllerGains = None, params: QuadParams = None) -> CTBR:
    """control.py:161-223: velocity P loop, geometric attitude -> CTBR."""
    out, _ = _stage(1, cmd.as_array(), state, params, gains)
    return CTBR(out[:, 0], out[:, 1:4])


def ps_to_ctbr(cmd: PS, state, gains: ControllerGains = None, params: QuadParams = None) -> CTBR:
    """control.py:226-233: position PD to a speed-capped velocity, then the LV loop."""
    out, _ = _stage(2, cmd.as_array(), state, params, gains)
    return CTBR(out[:, 0], out[:, 1:4])


def _dtype_of(arr):
    import torch

    return arr.dtype if isinstance(arr, torch.Tensor) else torch.float64
