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


# one definition of the grazing set, shared with bench.py's parity leg
from oracle.parity import _axis_rot, grazing_mask  # noqa: E402,F401
