"""The reference's flat-array geometry entry points (geometry/kernels.py,
SURVEY A19-A22) served by the device: bit-exact against the reference's own
outputs, with the reference's BVH arrays passed in and ignored."""

import numpy as np
import pytest

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2407_14783_b200.geometry import kernels  # noqa: E402
from paper_2407_14783_b200.sensing import DOWNWARD, FORWARD, CameraModel, camera_pose_world  # noqa: E402


def _args(g, name):
    return tuple(g[f"{name}_{k}"] for k in ("node_lo", "node_hi", "node_first", "node_count", "prim_order", "prim_type",
                                             "prim_data", "prim_oid"))


@pytest.mark.parametrize("name,cam", [("nav", "forward"), ("tess", "forward"), ("landing", "down")])
def test_render_batch_dropin_bit_exact(name, cam):
    g = golden("geometry")
    camera = CameraModel(rotation=FORWARD if cam == "forward" else DOWNWARD)
    o, r = camera_pose_world(g[f"{name}_render_pos"], g[f"{name}_render_quat"], camera)
    n = len(o)
    depth = np.empty((n, camera.height, camera.width))
    ids = np.empty((n, camera.height, camera.width), np.int64)
    kernels.render_batch(*_args(g, name), o, r, camera.width, camera.height, camera.tan_half_h, camera.tan_half_v,
                         camera.max_range, np.zeros((n, 0, 4)), np.zeros((n, 0), np.int64), depth, ids)
    assert np.array_equal(depth, g[f"{name}_render_depth"])
    assert np.array_equal(ids, g[f"{name}_render_ids"])


def test_render_batch_extra_spheres_match_oracle():
    """Swarm spheres (kernels.py:438-445) in the exact renderer == the oracle."""
    g = golden("geometry")
    camera = CameraModel(rotation=FORWARD, width=40, height=30)
    pos, quat = g["nav_render_pos"][:6], g["nav_render_quat"][:6]
    o, r = camera_pose_world(pos, quat, camera)
    n = len(o)
    rng = np.random.default_rng(4)
    fwd, right = r[:, :, 2], r[:, :, 0]  # camera axes in the world
    dist = rng.uniform(0.8, 3.0, (n, 5, 1))
    side = rng.uniform(-0.6, 0.6, (n, 5, 1))
    extra = np.concatenate([o[:, None, :] + dist * fwd[:, None, :] + side * dist * right[:, None, :],
                            np.full((n, 5, 1), 0.3)], axis=2)
    extra_ids = 60000 + np.tile(np.arange(5), (n, 1))
    depth = np.empty((n, camera.height, camera.width))
    ids = np.empty((n, camera.height, camera.width), np.int64)
    kernels.render_batch(*_args(g, "nav"), o, r, camera.width, camera.height, camera.tan_half_h, camera.tan_half_v,
                         camera.max_range, extra, extra_ids, depth, ids)
    s = oracle.OracleScene(g["nav_prim_type"], g["nav_prim_data"], g["nav_prim_oid"], g["nav_prim_lo"], g["nav_prim_hi"])
    d_ref, i_ref = s.render(o, r, camera.width, camera.height, camera.tan_half_h, camera.tan_half_v, camera.max_range,
                            extra, extra_ids)
    assert (ids >= 60000).any()
    assert np.array_equal(ids, i_ref)
    assert np.array_equal(depth, d_ref)


def test_point_and_ray_queries_dropin_bit_exact():
    g = golden("geometry")
    a = _args(g, "nav")
    for k in range(0, len(g["nav_np_q"]), 37):
        q = g["nav_np_q"][k]
        x, y, z, d2, oid = kernels.nearest_point_query(*a, *q)
        assert [x, y, z] == g["nav_np_pt"][k].tolist()
        assert np.sqrt(d2) == g["nav_np_d"][k] and oid == g["nav_np_id"][k]
    for k in range(0, len(g["nav_rc_o"]), 41):
        t, oid = kernels.raycast_query(*a, *g["nav_rc_o"][k], *g["nav_rc_d"][k], 0.0, 10.0)
        assert t == g["nav_rc_t"][k] and oid == g["nav_rc_id"][k]
