"""Quaternion helpers with the reference's names and semantics
(quatmath.py:18-176), batched over leading axes.

Scalar-first [w, x, y, z], body -> world.  Every batched function accepts
numpy arrays or torch tensors (a CUDA tensor stays on its device) and keeps
the reference's operation order, so FP64 results are bit-identical to the
reference's on either.  The rotation is the polynomial v + 2 (w (u x v) +
u x (u x v)) that K1 integrates with (qb_dynamics.cuh `rotate`): it is a
rotation only for unit q and is used as the definition of the map between
renormalisations (quatmath.py:1-10).

These are host/boundary helpers for user code (policies, camera poses,
scene construction); the hot path evaluates the same polynomials inside the
kernels.
"""

from __future__ import annotations

import numpy as np

__all__ = ["normalize", "multiply", "rotate", "rotate_inv", "to_matrix", "from_matrix", "from_axis_angle", "yaw_of",
           "left_matrix", "right_matrix", "skew", "rotate_jacobian_q", "rotate_inv_jacobian_q"]


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _stack(parts, axis, like):
    if _is_torch(like):
        import torch

        return torch.stack(parts, dim=axis)
    return np.stack(parts, axis=axis)


def _sqrt(a):
    if _is_torch(a):
        import torch

        return torch.sqrt(a)
    return np.sqrt(a)


def _split(a, k):
    return tuple(a[..., i] for i in range(k))


def _cross(a, b):
    """a x b on component tuples, reference order (quatmath.py:45-52)."""
    (ax, ay, az), (bx, by, bz) = a, b
    return ay * bz - az * by, az * bx - ax * bz, ax * by - ay * bx


def normalize(q):
    """q / |q| along the last axis (quatmath.py:18-21)."""
    w, x, y, z = _split(q, 4)
    n = _sqrt(w ** 2 + x ** 2 + y ** 2 + z ** 2)
    return q / n[..., None]


def multiply(q, p):
    """Hamilton product q ⊗ p (quatmath.py:24-36)."""
    qw, qx, qy, qz = _split(q, 4)
    pw, px, py, pz = _split(p, 4)
    return _stack([
        qw * pw - qx * px - qy * py - qz * pz,
        qw * px + qx * pw + qy * pz - qz * py,
        qw * py - qx * pz + qy * pw + qz * px,
        qw * pz + qx * py - qy * px + qz * pw,
    ], -1, q)


def _rotate(w, u, v, like):
    t = _cross(u, v)
    s = _cross(u, t)
    return _stack([vc + 2.0 * (w * tc + sc) for vc, tc, sc in zip(v, t, s)], -1, like)


def rotate(q, v):
    """R(q) v, body -> world (quatmath.py:39-55)."""
    w, x, y, z = _split(q, 4)
    return _rotate(w, (x, y, z), _split(v, 3), q)


def rotate_inv(q, v):
    """R(q)^T v, world -> body: the polynomial with the conjugate (quatmath.py:58-72)."""
    w, x, y, z = _split(q, 4)
    return _rotate(w, (-x, -y, -z), _split(v, 3), q)


def to_matrix(q):
    """R(q) as (..., 3, 3) in the 1 - 2(y² + z²) form (quatmath.py:75-81)."""
    w, x, y, z = _split(q, 4)
    rows = [
        [1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)],
        [2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)],
        [2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)],
    ]
    return _stack([_stack(r, -1, q) for r in rows], -2, q)


def from_matrix(m) -> np.ndarray:
    """Unit quaternion of one 3x3 rotation matrix, Shepperd's branch on the
    largest of (trace, m00, m11, m22) (quatmath.py:84-100)."""
    m = np.asarray(m, dtype=float)
    tr = np.trace(m)
    if tr > 0.0:
        s = np.sqrt(tr + 1.0) * 2.0
        q = [0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s]
    elif m[0, 0] >= m[1, 1] and m[0, 0] >= m[2, 2]:
        s = np.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2.0
        q = [(m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s]
    elif m[1, 1] >= m[2, 2]:
        s = np.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2.0
        q = [(m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s]
    else:
        s = np.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2.0
        q = [(m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s]
    return normalize(np.array(q))


def from_axis_angle(axis, angle: float) -> np.ndarray:
    """Rotation of `angle` about a non-zero `axis` (quatmath.py:103-108)."""
    a = np.asarray(axis, dtype=float)
    a = a / np.linalg.norm(a)
    return np.concatenate([[np.cos(0.5 * angle)], np.sin(0.5 * angle) * a])


def yaw_of(q):
    """atan2 of the world xy-projection of the body x-axis (quatmath.py:111-114)."""
    w, x, y, z = _split(q, 4)
    if _is_torch(q):
        import torch

        zero, one = torch.zeros_like(w), torch.ones_like(w)
    else:
        zero, one = np.zeros_like(w), np.ones_like(w)
    xb = _rotate(w, (x, y, z), (one, zero, zero), q)
    if _is_torch(q):
        import torch

        return torch.atan2(xb[..., 1], xb[..., 0])
    return np.arctan2(xb[..., 1], xb[..., 0])


def left_matrix(q) -> np.ndarray:
    """L(q) with q ⊗ p = L(q) p, one quaternion (quatmath.py:117-127)."""
    w, x, y, z = q
    return np.array([[w, -x, -y, -z], [x, w, -z, y], [y, z, w, -x], [z, -y, x, w]])


def right_matrix(p) -> np.ndarray:
    """R(p) with q ⊗ p = R(p) q, one quaternion (quatmath.py:130-140)."""
    w, x, y, z = p
    return np.array([[w, -x, -y, -z], [x, w, z, -y], [y, -z, w, x], [z, y, -x, w]])


def skew(v) -> np.ndarray:
    """[v]x for one 3-vector (quatmath.py:143-151)."""
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def _rotate_jac(q, v, sign: float) -> np.ndarray:
    # d/dq of v + 2 (w (u' x v) + u' x (u' x v)) with u' = sign * u: the w column is
    # 2 u' x v; the u columns are sign * (-2 w [v]x - 2 [u' x v]x - 2 [u']x [v]x)
    q = np.asarray(q, dtype=float)
    v = np.asarray(v, dtype=float)
    w, u = q[0], sign * q[1:4]
    uxv = np.cross(u, v)
    J = np.empty((3, 4))
    J[:, 0] = 2.0 * uxv
    J[:, 1:4] = sign * (-2.0 * w * skew(v) - 2.0 * skew(uxv) - 2.0 * skew(u) @ skew(v))
    return J


def rotate_jacobian_q(q, v) -> np.ndarray:
    """d(R(q) v)/dq for fixed v, (3, 4) (quatmath.py:154-162)."""
    return _rotate_jac(q, v, 1.0)


def rotate_inv_jacobian_q(q, v) -> np.ndarray:
    """d(R(q)^T v)/dq for fixed v, (3, 4) (quatmath.py:165-173)."""
    return _rotate_jac(q, v, -1.0)
