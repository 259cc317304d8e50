"""quatmath (reference quatmath.py:18-176) against the reference's own
outputs (tests/golden/quatmath.npz, tests/golden/make_quat_golden.py): the
batched functions bit for bit on numpy arrays and on torch float64 tensors,
the single-sample helpers bit for bit on numpy."""

import os

import numpy as np
import pytest
import torch

from paper_2407_14783_b200 import quatmath as qm

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "quatmath.npz"))


@pytest.mark.parametrize("backend", ["numpy", "torch"])
def test_batched_bit_exact(backend):
    conv = (lambda a: a) if backend == "numpy" else (lambda a: torch.from_numpy(a))
    back = (lambda a: a) if backend == "numpy" else (lambda a: a.numpy())
    q, p, v = conv(G["q"]), conv(G["p"]), conv(G["v"])
    got = {
        "normalize": qm.normalize(q), "multiply": qm.multiply(q, p), "rotate": qm.rotate(q, v),
        "rotate_inv": qm.rotate_inv(q, v), "to_matrix": qm.to_matrix(q),
    }
    for k, a in got.items():
        np.testing.assert_array_equal(back(a), G[k], err_msg=k)
    # atan2: numpy and torch may differ in the last ulp of the libm call
    if backend == "numpy":
        np.testing.assert_array_equal(qm.yaw_of(q), G["yaw_of"])
    else:
        np.testing.assert_allclose(back(qm.yaw_of(q)), G["yaw_of"], rtol=0, atol=1e-15)


def test_single_sample_helpers_bit_exact():
    np.testing.assert_array_equal(np.array([qm.from_matrix(m) for m in G["fm_in"]]), G["from_matrix"])
    np.testing.assert_array_equal(
        np.array([qm.from_axis_angle(a, t) for a, t in zip(G["axes"], G["angles"])]), G["from_axis_angle"])
    np.testing.assert_array_equal(np.array([qm.left_matrix(x) for x in G["q"][:8]]), G["left_matrix"])
    np.testing.assert_array_equal(np.array([qm.right_matrix(x) for x in G["p"][:8]]), G["right_matrix"])
    np.testing.assert_array_equal(np.array([qm.skew(x) for x in G["v"][:8]]), G["skew"])
    for name, f in (("rotate_jacobian_q", qm.rotate_jacobian_q), ("rotate_inv_jacobian_q", qm.rotate_inv_jacobian_q)):
        got = np.array([f(a, b) for a, b in zip(G["q"][:16], G["v"][:16])])
        np.testing.assert_array_equal(got, G[name], err_msg=name)


def test_rotation_is_the_dynamics_polynomial():
    """rotate/rotate_inv are exact inverses for unit q and equal to_matrix there."""
    qu = qm.normalize(G["q"])
    v = G["v"]
    np.testing.assert_allclose(qm.rotate_inv(qu, qm.rotate(qu, v)), v, atol=1e-12)
    np.testing.assert_allclose(np.einsum("nij,nj->ni", qm.to_matrix(qu), v), qm.rotate(qu, v), atol=1e-12)
