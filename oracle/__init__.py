"""CPU ORACLE for the VisFly/quadsim hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package; the product
(paper_2407_14783_b200) never does, and fails loudly when its CUDA library is
missing instead of falling back here.

Layout
  quadsim_oracle.c  FP64 C restatement of the reference kernels
                    (dynamics.py, control.py, gradients.py, geometry/bvh.py,
                    geometry/kernels.py), compiled to _build/liboracle.so
  __init__.py       ctypes bindings + host-side restatements that stay in
                    numpy (scene flattening shapes.py:139-212, camera pose
                    sensing.py:66-74, rollout_grad gradients.py:218-237)
  env.py            restatement of QuadEnvBase.step/reset + the tasks
                    (env/base.py, env/tasks.py) on top of the C kernels

Pinned by tests/test_oracle.py against tests/golden/*.npz, fixtures produced by
running the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

GRAVITY = 9.81
CMD_KINDS = {"srt": 0, "ctbr": 1, "ps": 2, "lv": 3, "rotor": 4}


def build(force: bool = False) -> str:
    """Compile the C restatement (make -C oracle)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.or_build_bvh.restype = ctypes.c_int64
        _lib.or_step_jacobian.restype = ctypes.c_int
    return _lib


class QbParams(ctypes.Structure):
    """Mirror of include/qb_params.h."""

    _fields_ = [
        ("mass", ctypes.c_double),
        ("inertia", ctypes.c_double * 3),
        ("gravity", ctypes.c_double * 3),
        ("torque_arms", (ctypes.c_double * 3) * 4),
        ("thrust_coeffs", ctypes.c_double * 3),
        ("drag_c", ctypes.c_double * 3),
        ("rotor_lo", ctypes.c_double),
        ("rotor_hi", ctypes.c_double),
        ("alloc_inv", (ctypes.c_double * 4) * 4),
        ("thrust_lo", ctypes.c_double),
        ("thrust_hi", ctypes.c_double),
        ("hover_speed", ctypes.c_double),
        ("physics_dt", ctypes.c_double),
        ("half_dt", ctypes.c_double),
        ("sixth_dt", ctypes.c_double),
        ("lag_alpha", ctypes.c_double),
        ("substeps", ctypes.c_int32),
        ("integrator", ctypes.c_int32),
        ("rate_p", ctypes.c_double * 3),
        ("attitude_p", ctypes.c_double * 3),
        ("vel_p", ctypes.c_double * 3),
        ("vel_d", ctypes.c_double * 3),
        ("pos_p", ctypes.c_double * 3),
        ("pos_d", ctypes.c_double * 3),
        ("max_speed", ctypes.c_double),
        ("max_tilt_accel", ctypes.c_double),
    ]


def pack_params(params, sim, gains) -> QbParams:
    """Derive the constants exactly as the reference evaluates them.

    Duck-typed over the reference dataclasses (params.py:45-178) or any object
    with the same fields.
    """
    p = QbParams()
    p.mass = float(params.mass)
    p.inertia[:] = [float(v) for v in np.asarray(params.inertia_diag, float)]
    p.gravity[:] = [float(v) for v in np.asarray(params.gravity, float)]
    z = np.array([0.0, 0.0, 1.0])  # params.py:82-88
    g = np.cross(np.asarray(params.arm_positions, float).reshape(4, 3), z)
    g = g + np.asarray(params.spin_directions, float)[:, None] * params.yaw_torque_coeff * z
    for i in range(4):
        p.torque_arms[i][:] = [float(v) for v in g[i]]
    k2, k1, k0 = (float(v) for v in params.thrust_coeffs)
    p.thrust_coeffs[:] = [k2, k1, k0]
    c = 0.5 * params.air_density * np.asarray(params.drag_coeffs, float) * np.asarray(params.cross_area, float)
    p.drag_c[:] = [float(v) for v in c]
    lo, hi = (float(v) for v in params.rotor_speed_limits)
    p.rotor_lo, p.rotor_hi = lo, hi
    a = np.empty((4, 4))  # params.py:90-100
    a[0, :] = 1.0
    a[1:4, :] = g.T
    minv = np.linalg.inv(a)
    for i in range(4):
        p.alloc_inv[i][:] = [float(v) for v in minv[i]]
    p.thrust_lo = float(k2 * lo**2 + k1 * lo + k0)
    p.thrust_hi = float(k2 * hi**2 + k1 * hi + k0)
    hover_thrust = params.mass * GRAVITY / 4.0
    arg = np.maximum(k1 * k1 + 4.0 * k2 * (hover_thrust - k0), 0.0)
    p.hover_speed = float(np.clip((-k1 + np.sqrt(arg)) / (2.0 * k2), lo, hi))
    h = sim.control_dt / sim.substeps
    p.physics_dt = h
    p.half_dt = 0.5 * h
    p.sixth_dt = h / 6.0
    p.lag_alpha = float(np.exp(-params.motor_decay * h))
    p.substeps = int(sim.substeps)
    integ = getattr(sim.integrator, "value", sim.integrator)
    p.integrator = 1 if str(integ).lower() == "rk4" else 0
    p.rate_p[:] = [float(v) for v in np.asarray(gains.rate_p, float)]
    p.attitude_p[:] = [float(v) for v in np.asarray(gains.attitude_p, float)]
    p.vel_p[:] = [float(v) for v in np.asarray(gains.velocity_pd[0], float)]
    p.vel_d[:] = [float(v) for v in np.asarray(gains.velocity_pd[1], float)]
    p.pos_p[:] = [float(v) for v in np.asarray(gains.position_pd[0], float)]
    p.pos_d[:] = [float(v) for v in np.asarray(gains.position_pd[1], float)]
    p.max_speed = float(gains.max_speed)
    p.max_tilt_accel = float(gains.max_tilt_accel)
    return p


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


# ---------------------------------------------------------------------------
# dynamics / control / gradients


def command_to_rotor_speeds(P: QbParams, kind: str, states, cmd) -> np.ndarray:
    """control.py:242-252 on AoS (N,17) states and an (N,4) command array."""
    states = _f64(states)
    n = states.shape[0]
    cmd = _f64(cmd, (n, 4))
    k = CMD_KINDS[kind]
    if k in (2, 3):  # yaw trig evaluated by numpy exactly as control.py:176
        cy = np.ascontiguousarray(np.cos(cmd[:, 3]))
        sy = np.ascontiguousarray(np.sin(cmd[:, 3]))
    else:
        cy = sy = np.zeros(n)
    out = np.empty((n, 4))
    lib().or_command_to_rotor_speeds(ctypes.byref(P), k, ctypes.c_int64(n), _ptr(states), _ptr(cmd), _ptr(cy), _ptr(sy), _ptr(out))
    return out


def command_mixer_info(P: QbParams, kind: str, states, cmd):
    """command_to_rotor_speeds plus, per agent, the mixer's torque scale and
    smallest clipped rotor thrust (test diagnostics).  Returns (speeds (N,4),
    scale (N,), min_thrust (N,))."""
    states = _f64(states)
    n = states.shape[0]
    cmd = _f64(cmd, (n, 4))
    cy = np.ascontiguousarray(np.cos(cmd[:, 3]))
    sy = np.ascontiguousarray(np.sin(cmd[:, 3]))
    out = np.empty((n, 4))
    info = np.empty((n, 2))
    lib().or_command_mixer_info(ctypes.byref(P), CMD_KINDS[kind], ctypes.c_int64(n), _ptr(states), _ptr(cmd), _ptr(cy),
                                _ptr(sy), _ptr(out), _ptr(info))
    return out, info[:, 0].copy(), info[:, 1].copy()


def dynamics_step(P: QbParams, states, rotor_cmds):
    """dynamics.py:231-253. Returns (next (N,17), nonfinite (N,) bool)."""
    x = _f64(states).copy()
    n = x.shape[0]
    cmd = _f64(rotor_cmds, (n, 4))
    bad = np.zeros(n, np.uint8)
    lib().or_dynamics_step(ctypes.byref(P), ctypes.c_int64(n), _ptr(x), _ptr(cmd), _ptr(bad))
    return x, bad.astype(bool)


def step_jacobian(P: QbParams, state, action):
    """gradients.py:145-197 -> (J (17,17), Ja (17,4), next (17,), flagged)."""
    s = _f64(state, (17,))
    a = _f64(action, (4,))
    J = np.empty((17, 17))
    Ja = np.empty((17, 4))
    nx = np.empty(17)
    f = lib().or_step_jacobian(ctypes.byref(P), _ptr(s), _ptr(a), _ptr(J), _ptr(Ja), _ptr(nx))
    return J, Ja, nx, bool(f)


def rollout_grad(P: QbParams, initial_state, actions, loss):
    """gradients.py:200-237 for one agent (T,4) actions.

    Returns (grad_actions (T,4), grad_initial (17,), states (T+1,17), flagged).
    """
    actions = np.atleast_2d(_f64(actions))
    T = actions.shape[0]
    states = np.empty((T + 1, 17))
    states[0] = _f64(initial_state, (17,))
    Js, Jas, flagged = [], [], False
    for t in range(T):
        J, Ja, nx, f = step_jacobian(P, states[t], actions[t])
        Js.append(J)
        Jas.append(Ja)
        flagged |= f
        states[t + 1] = nx
    _, g = loss(states)
    g = np.asarray(g, float)
    ga = np.zeros((T, 4))
    lam = g[T].copy()
    for t in range(T - 1, -1, -1):
        ga[t] = Jas[t].T @ lam
        lam = Js[t].T @ lam + g[t]
    return ga, lam, states, flagged


# ---------------------------------------------------------------------------
# geometry


PRIM_WIDTH = 16


def flatten_objects(objects):
    """shapes.py:139-212: objects -> (type, data(P,16), oid, lo(P,3), hi(P,3)).

    Duck-typed: each object has .id and .shape, the shape carrying
    center/radius (sphere), center/half_extents/rotation (box) or
    vertices/triangles (mesh).
    """
    types, datas, ids, los, his = [], [], [], [], []
    for obj in objects:
        s = obj.shape
        if hasattr(s, "radius"):
            row = np.zeros(PRIM_WIDTH)
            c = np.asarray(s.center, float)
            row[0:3] = c
            row[3] = s.radius
            types.append(0); datas.append(row[None]); ids.append(obj.id)
            los.append((c - s.radius)[None]); his.append((c + s.radius)[None])
        elif hasattr(s, "half_extents"):
            row = np.zeros(PRIM_WIDTH)
            c = np.asarray(s.center, float)
            h = np.asarray(s.half_extents, float)
            r = np.asarray(s.rotation, float).reshape(3, 3)
            row[0:3] = c; row[3:6] = h; row[6:15] = r.reshape(9)
            types.append(1); datas.append(row[None]); ids.append(obj.id)
            reach = np.abs(r) @ h
            los.append((c - reach)[None]); his.append((c + reach)[None])
        else:
            tris = np.asarray(s.vertices, float)[np.asarray(s.triangles, np.int64)]
            t = len(tris)
            rows = np.zeros((t, PRIM_WIDTH))
            rows[:, 0:9] = tris.reshape(t, 9)
            types.extend([2] * t); datas.append(rows); ids.extend([obj.id] * t)
            los.append(tris.min(axis=1)); his.append(tris.max(axis=1))
    return (
        np.asarray(types, np.int64),
        np.ascontiguousarray(np.concatenate(datas)),
        np.asarray(ids, np.int64),
        np.ascontiguousarray(np.concatenate(los)),
        np.ascontiguousarray(np.concatenate(his)),
    )


class OracleScene:
    """Flattened primitive table + the reference's median-split BVH."""

    def __init__(self, prim_type, prim_data, prim_oid, prim_lo, prim_hi):
        self.prim_type = np.ascontiguousarray(prim_type, np.int64)
        self.prim_data = np.ascontiguousarray(prim_data, np.float64)
        self.prim_oid = np.ascontiguousarray(prim_oid, np.int64)
        self.prim_lo = np.ascontiguousarray(prim_lo, np.float64)
        self.prim_hi = np.ascontiguousarray(prim_hi, np.float64)
        n = len(self.prim_type)
        m = max(2 * n, 1)
        self.node_lo = np.zeros((m, 3))
        self.node_hi = np.zeros((m, 3))
        self.node_first = np.zeros(m, np.int64)
        self.node_count = np.zeros(m, np.int64)
        self.prim_order = np.zeros(n, np.int64)
        nn = lib().or_build_bvh(ctypes.c_int64(n), _ptr(self.prim_lo), _ptr(self.prim_hi), _ptr(self.node_lo), _ptr(self.node_hi),
                                _ptr(self.node_first), _ptr(self.node_count), _ptr(self.prim_order))
        self.node_lo = np.ascontiguousarray(self.node_lo[:nn])
        self.node_hi = np.ascontiguousarray(self.node_hi[:nn])
        self.node_first = np.ascontiguousarray(self.node_first[:nn])
        self.node_count = np.ascontiguousarray(self.node_count[:nn])
        self._c = _CScene(_ptr(self.node_lo), _ptr(self.node_hi), _ptr(self.node_first), _ptr(self.node_count),
                          _ptr(self.prim_order), _ptr(self.prim_type), _ptr(self.prim_data), _ptr(self.prim_oid))
        self.bounds_lo = self.prim_lo.min(axis=0)  # shapes.py:214-217
        self.bounds_hi = self.prim_hi.max(axis=0)

    @classmethod
    def from_objects(cls, objects):
        return cls(*flatten_objects(objects))

    @property
    def num_prims(self):
        return len(self.prim_type)

    def nearest_point(self, q, brute: bool = False):
        """kernels.py:120-182 -> (point (N,3), distance (N,), object id (N,))."""
        q = _f64(q).reshape(-1, 3)
        n = len(q)
        pt = np.empty((n, 3)); d2 = np.empty(n); oid = np.empty(n, np.int64)
        if brute:
            lib().or_nearest_point_brute(ctypes.byref(self._c), ctypes.c_int64(self.num_prims), ctypes.c_int64(n), _ptr(q), _ptr(pt),
                                         _ptr(d2), _ptr(oid))
        else:
            lib().or_nearest_point(ctypes.byref(self._c), ctypes.c_int64(n), _ptr(q), _ptr(pt), _ptr(d2), _ptr(oid))
        return pt, np.sqrt(d2), oid

    def raycast(self, origins, dirs, tmax, tmin=0.0):
        """kernels.py:389-399 -> (t (N,) with -1 = miss, id (N,))."""
        o = _f64(origins).reshape(-1, 3)
        d = _f64(dirs).reshape(-1, 3)
        n = len(o)
        t = np.empty(n); oid = np.empty(n, np.int64)
        lib().or_raycast(ctypes.byref(self._c), ctypes.c_int64(n), _ptr(o), _ptr(d), ctypes.c_double(tmin), ctypes.c_double(tmax),
                         _ptr(t), _ptr(oid))
        return t, oid

    def render(self, origins, rotations, width, height, tan_half_h, tan_half_v, max_range, extra=None, extra_ids=None):
        """kernels.py:402-451 -> (depth (A,H,W) f64, ids (A,H,W) int64)."""
        o = _f64(origins).reshape(-1, 3)
        a = len(o)
        r = _f64(rotations).reshape(a, 3, 3)
        if extra is None:
            extra = np.zeros((a, 0, 4)); extra_ids = np.zeros((a, 0), np.int64)
        extra = _f64(extra)
        extra_ids = np.ascontiguousarray(extra_ids, np.int64)
        k = extra.shape[1]
        depth = np.empty((a, height, width)); ids = np.empty((a, height, width), np.int64)
        lib().or_render(ctypes.byref(self._c), ctypes.c_int64(a), _ptr(o), _ptr(r), ctypes.c_int64(width), ctypes.c_int64(height),
                        ctypes.c_double(tan_half_h), ctypes.c_double(tan_half_v), ctypes.c_double(max_range), ctypes.c_int64(k),
                        _ptr(extra), _ptr(extra_ids), _ptr(depth), _ptr(ids))
        return depth, ids


class _CScene(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("node_lo", "node_hi", "node_first", "node_count", "prim_order", "prim_type",
                                               "prim_data", "prim_oid")]


# ---------------------------------------------------------------------------
# camera (sensing.py)

FORWARD = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
DOWNWARD = np.array([[0.0, -1.0, 0.0], [-1.0, 0.0, 0.0], [0.0, 0.0, -1.0]])


def quat_rotate(q, v):
    """quatmath.py:39-55 (batched)."""
    w = q[..., 0]
    ux, uy, uz = q[..., 1], q[..., 2], q[..., 3]
    vx, vy, vz = v[..., 0], v[..., 1], v[..., 2]
    tx = uy * vz - uz * vy
    ty = uz * vx - ux * vz
    tz = ux * vy - uy * vx
    sx = uy * tz - uz * ty
    sy = uz * tx - ux * tz
    sz = ux * ty - uy * tx
    return np.stack([vx + 2.0 * (w * tx + sx), vy + 2.0 * (w * ty + sy), vz + 2.0 * (w * tz + sz)], axis=-1)


def quat_to_matrix(q):
    """quatmath.py:75-81 (batched)."""
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    row0 = np.stack([1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)], axis=-1)
    row1 = np.stack([2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)], axis=-1)
    row2 = np.stack([2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)], axis=-1)
    return np.stack([row0, row1, row2], axis=-2)


def camera_pose_world(pos, quat, cam_rotation, cam_translation):
    """sensing.py:66-74."""
    pos = np.atleast_2d(_f64(pos))
    quat = np.atleast_2d(_f64(quat))
    n = pos.shape[0]
    origins = pos + quat_rotate(quat, np.broadcast_to(np.asarray(cam_translation, float), (n, 3)))
    rot = np.einsum("nij,jk->nik", quat_to_matrix(quat), np.asarray(cam_rotation, float))
    return origins, np.ascontiguousarray(rot)


def render_frames(scene: OracleScene, pos, quat, width=64, height=64, vertical_fov=np.pi / 2, cam_rotation=FORWARD,
                  cam_translation=(0.0, 0.0, 0.0), max_range=10.0, extra=None, extra_ids=None):
    """sensing.py:77-100."""
    import math

    origins, rots = camera_pose_world(pos, quat, cam_rotation, cam_translation)
    tv = math.tan(vertical_fov / 2.0)
    th = tv * width / height
    return scene.render(origins, rots, width, height, th, tv, max_range, extra, extra_ids)
