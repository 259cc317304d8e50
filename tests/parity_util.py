"""Tolerances and the grazing-pixel analysis used by the GPU parity tests.

Tolerances (BASELINE.json north_star):
  states  |x_gpu - x_ref| <= 1e-5 * max(|x_ref|, s_f), s_f = 1 m, 1 m/s, 1,
          1 rad/s, 900 rad/s for p, v, q, omega, rotor speeds
  grads   same form with 1e-4
  depth   |d_gpu - d_ref| <= 1e-4 m on non-grazing pixels
  ids, collision / done / truncated flags: equal.
"""

import numpy as np

STATE_FLOOR = np.array([1.0] * 3 + [1.0] * 3 + [1.0] * 4 + [1.0] * 3 + [900.0] * 4)
DEPTH_TOL = 1e-4


def state_error(gpu, ref):
    """Per-element normalised error |gpu-ref| / max(|ref|, floor) for (..,17)."""
    gpu = np.asarray(gpu, float)
    ref = np.asarray(ref, float)
    return np.abs(gpu - ref) / np.maximum(np.abs(ref), STATE_FLOOR)


def summarize(err):
    e = np.asarray(err).ravel()
    return {"max": float(e.max()), "p99": float(np.percentile(e, 99)), "median": float(np.median(e))}


def _axis_rot(axis, ang):
    axis = np.asarray(axis, float)
    axis = axis / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K


def grazing_mask(scene, origins, rotations, width, height, th, tv, max_range, d_o=1e-5, d_r=3e-6):
    """Pixels whose oracle result is unstable under perturbations a few times
    larger than the FP32 error of the pose (~5e-7 m at 5 m) and of the ray
    direction (quaternion -> matrix -> pixel ray in FP32: up to ~8e-7 rad
    observed): silhouettes, edges, oblique incidence, near-tangent spheres
    (SURVEY.md 7.3-2).  A diagnostic set: parity asserts that every FP32
    mismatch lies inside it and that mismatches are rare.

    Returns (mask (A,H,W) bool, depth0, ids0)."""
    depth0, ids0 = scene.render(origins, rotations, width, height, th, tv, max_range)
    mask = np.zeros(depth0.shape, bool)
    perts = []
    for k in range(3):
        for s in (-1.0, 1.0):
            o = origins.copy()
            o[:, k] += s * d_o
            perts.append((o, rotations))
    for ax in ([1, 0, 0], [0, 1, 0], [0, 0, 1]):
        for s in (-1.0, 1.0):
            R = _axis_rot(ax, s * d_r)
            perts.append((origins, np.einsum("ij,njk->nik", R, rotations)))
    for o, r in perts:
        d, i = scene.render(o, r, width, height, th, tv, max_range)
        mask |= (i != ids0) | (np.abs(d - depth0) > DEPTH_TOL)
    return mask, depth0, ids0
