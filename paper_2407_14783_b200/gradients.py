"""Differentiable dynamics: the reference's gradient API (gradients.py) on the
K1 adjoint kernel, plus torch.autograd bindings for BPTT training.

Reference entry points kept (same arguments and return values):
  step_jacobian(state, action, config, params) -> StepJacobian   (:145-197)
  rollout(initial_state, actions, config, params) -> RolloutTape  (:200-215)
  rollout_grad(initial_state, actions, loss, config, params)
      -> (grad_actions, grad_initial_state, tape)                (:218-237)
but batched over envs and matrix-free: the tape holds only the states
((T+1) x 17 per env), and one backward launch sweeps the whole horizon
(lambda <- J^T lambda + g[t], grad_a[t] = Ja^T lambda) without ever forming J.
`step_jacobian` assembles the dense 17x17 / 17x4 matrices from 17 VJPs when a
caller wants them.

torch bindings: `DynamicsStep` (one step) and `Rollout` (a horizon) are
torch.autograd.Functions whose backward is the adjoint kernel, so a loss
built from their outputs trains with `loss.backward()`.

Action kinds: "rotor" (desired rotor speeds, the reference's action),
"ctbr" and "srt" (through the controller + mixer, beyond the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .dynamics import QuadState
from .params import ControllerGains, QuadParams, SimConfig, native_params

DIFFERENTIABLE_KINDS = ("rotor", "ctbr", "srt")


@dataclass
class StepJacobian:
    d_next_d_state: np.ndarray  # (13,13)
    d_next_d_action: np.ndarray  # (13,4)
    saturation_boundary: bool
    full_state_jacobian: np.ndarray  # (17,17)
    full_action_jacobian: np.ndarray  # (17,4)
    next_state: QuadState


@dataclass
class RolloutTape:
    """Saved forward pass: the states only (the adjoint recomputes the rest)."""

    states: object  # (T+1,17) for one agent (numpy), else (T+1,N,17)
    planes: object  # (T+1,17,N) device tensor
    actions: object  # (T,N,4) device tensor
    kind: str
    saturation_boundary: bool = False

    def __len__(self):
        return self.actions.shape[0]


def _code(dtype):
    import torch

    return nat.QB_F32 if dtype == torch.float32 else nat.QB_F64


def _check_kind(kind):
    if kind not in DIFFERENTIABLE_KINDS:
        raise ValueError(f"action kind {kind!r} is not differentiable; use one of {DIFFERENTIABLE_KINDS}")


def rollout_planes(P, kind, init_planes, actions):
    """Forward horizon: init (17,N), actions (T,N,4) -> tape (T+1,17,N)."""
    import torch

    T, n = actions.shape[0], actions.shape[1]
    tape = torch.empty((T + 1, 17, n), dtype=init_planes.dtype, device=init_planes.device)
    tape[0] = init_planes
    bad = torch.zeros(n, dtype=torch.uint8, device=init_planes.device)
    with torch.cuda.device(init_planes.device):
        nat.check(nat.lib().qb_rollout_forward(P, nat.CMD[kind], _code(init_planes.dtype), n, n, T, nat.ptr(tape),
                                               nat.ptr(actions.contiguous()), nat.ptr(bad), nat.stream_of()),
                  "qb_rollout_forward")
    return tape, bad


def backward_planes(P, kind, tape, actions, g_traj, action_grad_sum=None):
    """Reverse sweep: returns (grad_actions (T,N,4), grad_init (17,N), boundary (N,) uint8)."""
    import torch

    T, n = actions.shape[0], actions.shape[1]
    ga = torch.empty_like(actions)
    gi = torch.empty((17, n), dtype=tape.dtype, device=tape.device)
    bnd = torch.empty(n, dtype=torch.uint8, device=tape.device)
    with torch.cuda.device(tape.device):
        nat.check(nat.lib().qb_rollout_backward(P, nat.CMD[kind], _code(tape.dtype), n, n, T, nat.ptr(tape.contiguous()),
                                                nat.ptr(actions.contiguous()), nat.ptr(g_traj.contiguous()), nat.ptr(ga),
                                                nat.ptr(gi), nat.ptr(bnd), nat.ptr(action_grad_sum), nat.stream_of()),
                  "qb_rollout_backward")
    return ga, gi, bnd


def step_vjp(P, kind, planes, action, lam_next):
    """One-step VJP: (lam_prev (17,N), grad_action (N,4), boundary (N,))."""
    import torch

    n = planes.shape[1]
    lam_prev = torch.empty_like(planes)
    ga = torch.empty_like(action)
    bnd = torch.empty(n, dtype=torch.uint8, device=planes.device)
    with torch.cuda.device(planes.device):
        nat.check(nat.lib().qb_dynamics_vjp(P, nat.CMD[kind], _code(planes.dtype), n, n, nat.ptr(planes.contiguous()),
                                            nat.ptr(action.contiguous()), nat.ptr(lam_next.contiguous()), nat.ptr(lam_prev),
                                            nat.ptr(ga), nat.ptr(bnd), nat.stream_of()), "qb_dynamics_vjp")
    return lam_prev, ga, bnd


# ---------------------------------------------------------------------------
# reference-shaped API


def _state_planes(state, dtype):
    import torch

    if isinstance(state, QuadState):
        return state.planes.to(dtype)
    return QuadState.from_vector(np.atleast_2d(np.asarray(state, float)), dtype=dtype).planes


def step_jacobian(state, action, config: SimConfig = None, params: QuadParams = None, kind: str = "rotor",
                  gains: ControllerGains = None) -> StepJacobian:
    """Exact Jacobians of one step for a single agent (gradients.py:145-197),
    assembled from 17 adjoint sweeps in exact double."""
    import torch

    _check_kind(kind)
    P = native_params(params, config, gains)
    pl = _state_planes(state, torch.float64)
    if pl.shape[1] != 1:
        raise ValueError("step_jacobian operates on a single-agent state")
    a = torch.as_tensor(np.asarray(action, float).reshape(1, 4) if not isinstance(action, torch.Tensor) else action,
                        dtype=torch.float64, device=pl.device).reshape(1, 4)
    planes = pl.expand(17, 17).contiguous()
    acts = a.expand(17, 4).contiguous()
    eye = torch.eye(17, dtype=torch.float64, device=pl.device)  # lam_next column k = e_k
    lam_prev, ga, bnd = step_vjp(P, kind, planes, acts, eye)
    J = lam_prev.T.cpu().numpy()  # row k = e_k^T J
    Ja = ga.cpu().numpy()
    nxt = QuadState(pl.clone())
    nat.check(nat.lib().qb_dynamics_step(P, nat.CMD[kind], nat.QB_F64, 1, 1, nat.ptr(nxt.planes), nat.ptr(a.contiguous()),
                                         None, None, nat.stream_of()), "qb_dynamics_step")
    return StepJacobian(J[0:13, 0:13], Ja[0:13], bool(bnd[0].item()), J, Ja, nxt)


def rollout(initial_state, actions, config: SimConfig = None, params: QuadParams = None, kind: str = "rotor",
            gains: ControllerGains = None, dtype=None) -> RolloutTape:
    """Forward horizon saving the state tape (gradients.py:200-215).

    actions: (T,4) for one agent or (T,N,4); numpy in -> float64 (exact),
    tensors keep their dtype."""
    import torch

    _check_kind(kind)
    single = np.ndim(actions) == 2
    if dtype is None:
        dtype = actions.dtype if isinstance(actions, torch.Tensor) else torch.float64
    pl = _state_planes(initial_state, dtype)
    a = torch.as_tensor(actions, dtype=dtype, device=pl.device)
    a = a.reshape(a.shape[0], -1, 4).contiguous()
    P = native_params(params, config, gains)
    tape, _ = rollout_planes(P, kind, pl, a)
    states = tape.permute(0, 2, 1)
    host = states[:, 0, :].double().cpu().numpy() if single else states
    return RolloutTape(host, tape, a, kind)


def rollout_grad(initial_state, actions, loss, config: SimConfig = None, params: QuadParams = None, kind: str = "rotor",
                 gains: ControllerGains = None, dtype=None):
    """Reverse-accumulated gradients of a scalar rollout loss (gradients.py:218-237).

    `loss(states)` gets the trajectory ((T+1,17) numpy for one agent, as in
    the reference; (T+1,N,17) otherwise) and returns (value, d value /
    d trajectory) of the same shape.  Returns (grad_actions, grad_initial_state,
    tape) shaped like the reference for one agent ((T,4), (17,)), batched
    otherwise ((T,N,4), (N,17))."""
    import torch

    tape = rollout(initial_state, actions, config, params, kind, gains, dtype)
    _, g = loss(tape.states)
    single = isinstance(tape.states, np.ndarray)
    gt = torch.as_tensor(np.asarray(g, float) if single else g, dtype=tape.planes.dtype, device=tape.planes.device)
    if single:
        if tuple(gt.shape) != tuple(tape.states.shape):
            raise ValueError(f"loss gradient shape {tuple(gt.shape)} != trajectory shape {tape.states.shape}")
        gt = gt.reshape(gt.shape[0], 1, 17)
    g_planes = gt.permute(0, 2, 1).contiguous()
    P = native_params(params, config, gains)
    ga, gi, bnd = backward_planes(P, tape.kind, tape.planes, tape.actions, g_planes)
    tape.saturation_boundary = bool(bnd.any())
    if single:
        return ga[:, 0, :].double().cpu().numpy(), gi[:, 0].double().cpu().numpy(), tape
    return ga, gi.T, tape


# ---------------------------------------------------------------------------
# torch.autograd


def _autograd_classes():
    import torch

    class DynamicsStep(torch.autograd.Function):
        """next_planes = step(planes, action); backward = one adjoint sweep."""

        @staticmethod
        def forward(ctx, planes, action, P, kind):
            nxt = planes.detach().clone().contiguous()
            a = action.detach().contiguous()
            n = nxt.shape[1]
            nat.check(nat.lib().qb_dynamics_step(P, nat.CMD[kind], _code(nxt.dtype), n, n, nat.ptr(nxt), nat.ptr(a), None,
                                                 None, nat.stream_of()), "qb_dynamics_step")
            ctx.save_for_backward(planes.detach().contiguous(), a)
            ctx.P, ctx.kind = P, kind
            return nxt

        @staticmethod
        def backward(ctx, g):
            planes, a = ctx.saved_tensors
            lam_prev, ga, _ = step_vjp(ctx.P, ctx.kind, planes, a, g.contiguous())
            return lam_prev, ga, None, None

    class Rollout(torch.autograd.Function):
        """tape (T+1,17,N) = rollout(init (17,N), actions (T,N,4)); backward =
        one launch over the whole horizon."""

        @staticmethod
        def forward(ctx, init_planes, actions, P, kind):
            tape, _ = rollout_planes(P, kind, init_planes.detach().contiguous(), actions.detach().contiguous())
            ctx.save_for_backward(tape, actions.detach().contiguous())
            ctx.P, ctx.kind = P, kind
            return tape

        @staticmethod
        def backward(ctx, g):
            tape, actions = ctx.saved_tensors
            ga, gi, _ = backward_planes(ctx.P, ctx.kind, tape, actions, g.contiguous())
            return gi, ga, None, None

    return DynamicsStep, Rollout


_CLASSES = None


def _classes():
    global _CLASSES
    if _CLASSES is None:
        _CLASSES = _autograd_classes()
    return _CLASSES


def differentiable_step(planes, action, config: SimConfig = None, params: QuadParams = None, kind: str = "rotor",
                        gains: ControllerGains = None):
    """Autograd-aware dynamics step on (17,N) planes and (N,4) actions."""
    _check_kind(kind)
    return _classes()[0].apply(planes, action, native_params(params, config, gains), kind)


def differentiable_rollout(init_planes, actions, config: SimConfig = None, params: QuadParams = None, kind: str = "rotor",
                           gains: ControllerGains = None):
    """Autograd-aware horizon: (17,N), (T,N,4) -> tape (T+1,17,N)."""
    _check_kind(kind)
    return _classes()[1].apply(init_planes, actions, native_params(params, config, gains), kind)
