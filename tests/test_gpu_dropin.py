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


def test_render_frames_extra_spheres():
    """sensing.render_frames(..., extra_spheres, extra_ids) (sensing.py:77-100,
    kernels.py:438-445) through qb_render_poses: exact double == the oracle,
    FP32 ids equal and depth within 1e-4 m off the grazing set."""
    from parity_util import DEPTH_TOL, grazing_mask

    from paper_2407_14783_b200.sensing import render_frames

    g = golden("geometry")
    camera = CameraModel(rotation=FORWARD, width=48, height=32)
    pos, quat = g["nav_render_pos"][:8], g["nav_render_quat"][:8]
    o, r = camera_pose_world(pos, quat, camera)
    n = len(o)
    rng = np.random.default_rng(5)
    fwd, right = r[:, :, 2], r[:, :, 0]
    dist = rng.uniform(0.8, 3.0, (n, 4, 1))
    side = rng.uniform(-0.6, 0.6, (n, 4, 1))
    extra = np.concatenate([o[:, None, :] + dist * fwd[:, None, :] + side * dist * right[:, None, :],
                            np.full((n, 4, 1), 0.15)], axis=2)
    ids = 60000 + np.tile(np.arange(4), (n, 1))
    s = oracle.OracleScene(g["nav_prim_type"], g["nav_prim_data"], g["nav_prim_oid"], g["nav_prim_lo"], g["nav_prim_hi"])

    class _Carrier:  # the golden primitive table as a Scene-like object
        arrays = type("A", (), dict(prim_type=g["nav_prim_type"], prim_data=g["nav_prim_data"],
                                    prim_object_id=g["nav_prim_oid"], prim_aabb_lo=g["nav_prim_lo"],
                                    prim_aabb_hi=g["nav_prim_hi"], __len__=lambda a: len(g["nav_prim_type"])))()

    from paper_2407_14783_b200.geometry.device import DeviceScenes

    ds = DeviceScenes([_Carrier()], device="cuda")
    d64, i64 = render_frames(ds, pos, quat, camera, extra_spheres=extra, extra_ids=ids, dtype=torch.float64)
    d_ref, i_ref = s.render(o, r, camera.width, camera.height, camera.tan_half_h, camera.tan_half_v, camera.max_range,
                            extra, ids)
    assert (i_ref >= 60000).any()
    assert np.array_equal(i64, i_ref) and np.array_equal(d64, d_ref)
    d32, i32 = render_frames(ds, pos, quat, camera, extra_spheres=extra, extra_ids=ids)
    graz, _, _ = grazing_mask(s, o, r, camera.width, camera.height, camera.tan_half_h, camera.tan_half_v,
                              camera.max_range)
    # spheres are not in the scene the grazing mask perturbs: also tolerate their silhouettes
    sil = np.zeros_like(graz)
    sil[:, 1:, :] |= i_ref[:, 1:, :] != i_ref[:, :-1, :]
    sil[:, :, 1:] |= i_ref[:, :, 1:] != i_ref[:, :, :-1]
    bad = (i32 != i_ref) | (np.abs(d32 - d_ref) > DEPTH_TOL)
    assert not (bad & ~graz & ~sil).any()
    assert bad.mean() < 1e-2


def test_reference_loop_shape_fresh_results():
    """Code written against the reference keeps per-step results: a list of
    StepResults stored over a whole golden episode (respawns included) still
    holds every step's own rewards / flags / info afterwards, np.nonzero works
    on as_reference() flags, and a step's observations index correctly after
    the next step (double-buffered frames) but raise once overwritten
    (reference env/base.py:37-43, 186-210, 287-310)."""
    import dataclasses

    from paper_2407_14783_b200.control import command_from_array
    from paper_2407_14783_b200.env import StaleObservations, make_env, navigation_config

    g = golden("env_nav")
    cfg = dataclasses.replace(navigation_config(0, 12), episode_max_steps=int(g["max_steps"]))
    env = make_env(cfg, dtype=torch.float64)
    env.reset(seed=3)
    results = []
    T = g["actions"].shape[0]
    for t in range(T):
        res = env.step(command_from_array(cfg.command_type, g["actions"][t]))
        results.append(res)
        if t >= 1:  # the previous step's observations are still the previous step's
            prev = results[t - 1].observations
            # (LV yaw trig: CUDA libm vs numpy, <= 1e-6 over the episode -- test_gpu_env.py)
            np.testing.assert_allclose(prev[0]["state"], g["state"][t - 1][0], rtol=1e-6, atol=1e-9)
            if f"img_depth_{t - 1}" in g.files:
                assert np.abs(prev[3]["depth"] - g[f"img_depth_{t - 1}"][3]).max() < 1e-9
        if t >= 2:
            with pytest.raises(StaleObservations):
                results[t - 2].observations["depth"]
    for t, res in enumerate(results):  # every stored result is its own step's
        ref = res.as_reference()
        np.testing.assert_allclose(ref.reward, g["reward"][t], rtol=1e-6, atol=1e-6)  # reward is float32
        assert np.array_equal(ref.terminated, g["terminated"][t]) and np.array_equal(ref.truncated, g["truncated"][t])
        assert np.array_equal(np.nonzero(ref.terminated)[0], np.nonzero(g["terminated"][t])[0])
        for i in (0, 5, 11):
            info = res.info[i]
            assert info["collision"] == bool(g["collision"][t][i]) and info["step"] == int(g["step"][t][i])
            assert info["success"] == bool(g["success"][t][i])
            np.testing.assert_allclose(info["nearest_distance"], g["nearest_dist"][t][i], rtol=1e-9)
    assert int(g["terminated"].sum() + g["truncated"].sum()) > 0  # the episode crossed respawns
    # materialised observations never go stale
    last = results[-1].observations
    host = last.as_reference()
    env.step(command_from_array(cfg.command_type, g["actions"][0]))
    env.step(command_from_array(cfg.command_type, g["actions"][0]))
    assert np.array_equal(last[2]["state"], host[2]["state"])
    np.testing.assert_allclose(host[2]["state"], g["state"][T - 1][2], rtol=1e-6, atol=1e-9)
