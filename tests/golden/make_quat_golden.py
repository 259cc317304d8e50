"""Golden vectors for quatmath (reference quatmath.py:18-176), made by RUNNING
THE REFERENCE in the build container:

    python tests/golden/make_quat_golden.py [/root/reference/pkg/src]

Writes tests/golden/quatmath.npz (inputs and the reference's outputs).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)
from quadsim import quatmath as qm  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "quatmath.npz")


def main():
    rng = np.random.default_rng(2407)
    n = 257
    q = rng.normal(size=(n, 4)) + np.array([0.5, 0.0, 0.0, 0.0])  # non-unit, as inside RK4 stages
    p = rng.normal(size=(n, 4))
    v = rng.normal(size=(n, 3)) * 3.0
    qu = qm.normalize(q)
    mats = qm.to_matrix(qu)
    # from_matrix on every Shepperd branch: random rotations + ones with a dominant diagonal entry
    fm_in = [mats[i] for i in range(16)]
    for ax in range(3):
        fm_in.append(qm.to_matrix(qm.from_axis_angle(np.eye(3)[ax], 3.0)))
    fm_in = np.array(fm_in)
    axes = rng.normal(size=(8, 3))
    angles = rng.uniform(-np.pi, np.pi, size=8)
    out = {
        "q": q, "p": p, "v": v,
        "normalize": qm.normalize(q),
        "multiply": qm.multiply(q, p),
        "rotate": qm.rotate(q, v),
        "rotate_inv": qm.rotate_inv(q, v),
        "to_matrix": qm.to_matrix(q),
        "yaw_of": qm.yaw_of(q),
        "fm_in": fm_in,
        "from_matrix": np.array([qm.from_matrix(m) for m in fm_in]),
        "axes": axes, "angles": angles,
        "from_axis_angle": np.array([qm.from_axis_angle(a, t) for a, t in zip(axes, angles)]),
        "left_matrix": np.array([qm.left_matrix(x) for x in q[:8]]),
        "right_matrix": np.array([qm.right_matrix(x) for x in p[:8]]),
        "skew": np.array([qm.skew(x) for x in v[:8]]),
        "rotate_jacobian_q": np.array([qm.rotate_jacobian_q(a, b) for a, b in zip(q[:16], v[:16])]),
        "rotate_inv_jacobian_q": np.array([qm.rotate_inv_jacobian_q(a, b) for a, b in zip(q[:16], v[:16])]),
    }
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, {k: a.shape for k, a in out.items()})


if __name__ == "__main__":
    main()
