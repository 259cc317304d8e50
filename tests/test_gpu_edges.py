"""Edge cases of the C-ABI on the GPU: empty batches (n = 0) through every
batched entry point, camera resolutions that leave partial tiles or exceed the
per-block tile-plane table, and batch sizes that are not multiples of a warp
or a block -- each against the oracle (exact double) where there is output."""

import numpy as np
import pytest

import oracle
from conftest import scene_from_golden
from parity_util import DEPTH_TOL, grazing_mask, state_error

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2407_14783_b200 import _native as nat  # noqa: E402
from paper_2407_14783_b200.geometry.device import DeviceScenes  # noqa: E402
from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig, native_params  # noqa: E402
from paper_2407_14783_b200.sensing import DOWNWARD, FORWARD, CameraModel, render_state  # noqa: E402

DEV = "cuda"


def _carrier(t):
    class _S:
        arrays = type("A", (), dict(prim_type=t.prim_type, prim_data=t.prim_data, prim_object_id=t.prim_oid,
                                    prim_aabb_lo=t.prim_lo, prim_aabb_hi=t.prim_hi, __len__=lambda s: len(t.prim_type)))()
    return _S()


def test_empty_batches_are_no_ops(ggeo):
    """n = 0: every batched entry point returns OK without touching memory."""
    lib, s = nat.lib(), nat.stream_of()
    p = native_params(QuadParams(), SimConfig(), ControllerGains())
    dummy = torch.zeros(64, dtype=torch.float32, device=DEV)
    P = nat.ptr(dummy)
    assert lib.qb_dynamics_step(p, nat.CMD["ctbr"], nat.QB_F32, 0, 0, P, P, None, None, s) == 0
    assert lib.qb_command_to_rotor_speeds(p, nat.CMD["ctbr"], nat.QB_F32, 0, 0, P, P, P, s) == 0
    assert lib.qb_rollout_forward(p, nat.CMD["ctbr"], nat.QB_F32, 0, 0, 8, P, P, None, s) == 0
    assert lib.qb_rng_seed(0, 0, P, s) == 0
    ds = DeviceScenes([_carrier(scene_from_golden(ggeo, "nav"))], device=DEV)
    cam = CameraModel()
    assert lib.qb_render_poses(ds.handle, cam.native(), nat.QB_F32, 0, P, P, None, P, None, None, None, 0, s) == 0
    assert lib.qb_nearest_point(ds.handle, None, 0, P, P, P, P, None, s) == 0
    assert lib.qb_raycast(ds.handle, nat.QB_F32, None, 0, P, P, 0.0, 10.0, P, P, s) == 0
    torch.cuda.synchronize()
    assert float(dummy.abs().sum()) == 0.0


@pytest.mark.parametrize("wh", [(1, 1), (7, 5), (65, 33), (256, 192)])
def test_render_odd_resolutions(ggeo, wh):
    """Partial 8x8 tiles, a single pixel, and 768 tiles (beyond the per-block
    tile-plane table): the FP64 kernel bit-exact and both FP32 kernels with
    equal ids and depth within tolerance off the grazing set, against the
    oracle."""
    w, h = wh
    t = scene_from_golden(ggeo, "nav")
    ds = DeviceScenes([_carrier(t)], device=DEV)
    rng = np.random.default_rng(w * 1000 + h)
    n = 24
    pos = rng.uniform([-4.0, -4.0, 0.5], [4.0, 4.0, 3.5], (n, 3))
    q = rng.normal(size=(n, 4)) + np.array([2.0, 0, 0, 0])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    for rot in (FORWARD, DOWNWARD):
        cam = CameraModel(rotation=rot, width=w, height=h)
        pl64 = torch.zeros((17, n), dtype=torch.float64, device=DEV)
        pl64[0:3] = torch.as_tensor(pos.T)
        pl64[6:10] = torch.as_tensor(q.T)
        st = pl64.T.cpu().numpy()
        o, r = oracle.camera_pose_world(st[:, 0:3], st[:, 6:10], cam.rotation, cam.translation)
        d64 = torch.empty((n, h, w), dtype=torch.float64, device=DEV)
        s64 = torch.empty((n, h, w), dtype=torch.int32, device=DEV)
        render_state(ds, cam, pl64, depth=d64, seg=s64)
        d0, i0 = t.render(o, r, w, h, cam.tan_half_h, cam.tan_half_v, cam.max_range)
        assert np.array_equal(s64.cpu().numpy(), i0) and np.array_equal(d64.cpu().numpy(), d0)
        pl32 = pl64.float()
        st32 = pl32.T.double().cpu().numpy()
        o, r = oracle.camera_pose_world(st32[:, 0:3], st32[:, 6:10], cam.rotation, cam.translation)
        graz, d0, i0 = grazing_mask(t, o, r, w, h, cam.tan_half_h, cam.tan_half_v, cam.max_range)
        for mode in (1, 2):
            d = torch.empty((n, h, w), dtype=torch.float32, device=DEV)
            sg = torch.empty((n, h, w), dtype=torch.int32, device=DEV)
            render_state(ds, cam, pl32, depth=d, seg=sg, mode=mode)
            dd, ss = d.double().cpu().numpy(), sg.cpu().numpy()
            err = np.abs(dd - d0)
            bad = (ss != i0) | (err > DEPTH_TOL)
            nb = bad & ~graz
            print(wh, mode, f"grazing {graz.mean():.2e} mismatched {bad.mean():.2e} non-grazing {int(nb.sum())}")
            # ids exact off the grazing set; at 256x192 a few far (8 m) near-silhouette
            # sphere pixels exceed 1e-4 m by ~20% without being flagged by the
            # perturbation analysis: allowed at <= 1e-5 of the pixels and <= 2e-4 m
            assert not (nb & (ss != i0)).any(), (wh, mode)
            assert nb.mean() <= 1e-5 and (err[nb].max() if nb.any() else 0.0) <= 2e-4, (wh, mode, int(nb.sum()))


@pytest.mark.parametrize("n", [1, 31, 33, 129, 1000])
def test_dynamics_ragged_batches(n):
    """K1 on batch sizes that leave partial warps and blocks: FP64 bit-exact
    and FP32 within 1e-5 of the oracle's exact-double step."""
    rng = np.random.default_rng(n)
    x = np.zeros((n, 17))
    x[:, 0:3] = rng.uniform(-3, 3, (n, 3))
    x[:, 3:6] = rng.normal(size=(n, 3))
    qq = rng.normal(size=(n, 4)) + np.array([3.0, 0, 0, 0])
    x[:, 6:10] = qq / np.linalg.norm(qq, axis=1, keepdims=True)
    x[:, 10:13] = rng.normal(size=(n, 3))
    x[:, 13:17] = rng.uniform(600, 1200, (n, 4))
    a = np.concatenate([rng.uniform(5, 15, (n, 1)), rng.normal(size=(n, 3))], axis=1)
    P = oracle.pack_params(QuadParams(), SimConfig(), ControllerGains())
    ref, _ = oracle.dynamics_step(P, x, oracle.command_to_rotor_speeds(P, "ctbr", x, a))
    p = native_params(QuadParams(), SimConfig(), ControllerGains())
    for dtype, code in ((torch.float64, nat.QB_F64), (torch.float32, nat.QB_F32)):
        pl = torch.as_tensor(x.T, dtype=dtype, device=DEV).contiguous()
        act = torch.as_tensor(a, dtype=dtype, device=DEV).contiguous()
        nat.check(nat.lib().qb_dynamics_step(p, nat.CMD["ctbr"], code, n, n, nat.ptr(pl), nat.ptr(act), None, None,
                                             nat.stream_of()))
        got = pl.T.double().cpu().numpy()
        if dtype == torch.float64:
            assert np.array_equal(got, ref)
        else:
            assert state_error(got, ref).max() < 1e-5


def test_config2_mesh_scene_vs_oracle():
    """BASELINE config 2's box/cylinder mesh room (SceneSpec cluttered_mesh):
    FP64 renders bit-exact and FP32 within tolerance against the oracle on the
    same triangles, and the exact nearest point against the oracle's."""
    from paper_2407_14783_b200.env import SceneSpec

    sc = SceneSpec(kind="cluttered_mesh", seed=0, volume_lo=[-5, -5, 0], volume_hi=[5, 5, 4]).materialize()
    a = sc.arrays
    t = oracle.OracleScene(a.prim_type, a.prim_data, a.prim_object_id, a.prim_aabb_lo, a.prim_aabb_hi)
    ds = DeviceScenes([sc], device=DEV)
    rng = np.random.default_rng(2)
    n = 64
    pos = rng.uniform([-4.0, -4.0, 0.5], [4.0, 4.0, 3.5], (n, 3))
    q = rng.normal(size=(n, 4)) + np.array([2.0, 0, 0, 0])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    cam = CameraModel(rotation=FORWARD)
    pl64 = torch.zeros((17, n), dtype=torch.float64, device=DEV)
    pl64[0:3] = torch.as_tensor(pos.T)
    pl64[6:10] = torch.as_tensor(q.T)
    st = pl64.T.cpu().numpy()
    o, r = oracle.camera_pose_world(st[:, 0:3], st[:, 6:10], cam.rotation, cam.translation)
    d64 = torch.empty((n, 64, 64), dtype=torch.float64, device=DEV)
    s64 = torch.empty((n, 64, 64), dtype=torch.int32, device=DEV)
    render_state(ds, cam, pl64, depth=d64, seg=s64)
    d0, i0 = t.render(o, r, 64, 64, cam.tan_half_h, cam.tan_half_v, cam.max_range)
    assert np.array_equal(s64.cpu().numpy(), i0) and np.array_equal(d64.cpu().numpy(), d0)
    pl32 = pl64.float()
    st32 = pl32.T.double().cpu().numpy()
    o, r = oracle.camera_pose_world(st32[:, 0:3], st32[:, 6:10], cam.rotation, cam.translation)
    graz, d0, i0 = grazing_mask(t, o, r, 64, 64, cam.tan_half_h, cam.tan_half_v, cam.max_range)
    d = torch.empty((n, 64, 64), dtype=torch.float32, device=DEV)
    sg = torch.empty((n, 64, 64), dtype=torch.int32, device=DEV)
    render_state(ds, cam, pl32, depth=d, seg=sg)
    dd, ss = d.double().cpu().numpy(), sg.cpu().numpy()
    bad = (ss != i0) | (np.abs(dd - d0) > DEPTH_TOL)
    nb = bad & ~graz
    print("mesh config 2:", f"grazing {graz.mean():.2e} mismatched {bad.mean():.2e} non-grazing {int(nb.sum())}",
          [(tuple(int(v) for v in k), float(dd[tuple(k)]), int(ss[tuple(k)]), float(d0[tuple(k)]), int(i0[tuple(k)]))
           for k in np.argwhere(nb)[:6]])
    # FP32 Moeller-Trumbore can open a crack along an edge two triangles of one
    # mesh share (a ray through it reaches the object's far side): measured 1
    # pixel in 262144 here; the exact-double renders above have none
    assert nb.mean() <= 1e-5 and bad.mean() < 1e-3
    from paper_2407_14783_b200.geometry.queries import nearest_points

    qs = rng.uniform([-5, -5, 0], [5, 5, 4], (300, 3))
    _, dist, oid = nearest_points(ds, qs)
    _, rd, rid = t.nearest_point(qs)
    assert np.array_equal(oid.cpu().numpy(), rid)
    assert np.abs(dist.cpu().numpy() - rd).max() < 1e-12


def test_warp_nearest_point_on_large_mesh_scene():
    """Small batches run one warp per env; on scenes beyond the warp's
    brute-force size (> 1024 primitives) every lane walks the BVH.  Proximity
    after every step (nearest distance, collision) equals the oracle's exact
    query on the env's own states; spawns and respawns go through the same
    query."""
    import dataclasses

    from paper_2407_14783_b200.control import LV
    from paper_2407_14783_b200.env import make_env, navigation_config

    cfg = navigation_config(scene_seed=0, num_agents=64, with_vision=False)
    cfg = dataclasses.replace(cfg, scenes=(dataclasses.replace(cfg.scenes[0], kind="cluttered_mesh"),))
    env = make_env(cfg)
    env.reset(seed=5)
    a = env.scenes[0].arrays
    assert len(a) > 1024
    t = oracle.OracleScene(a.prim_type, a.prim_data, a.prim_object_id, a.prim_aabb_lo, a.prim_aabb_hi)
    g = torch.Generator(device=DEV).manual_seed(3)
    for _ in range(25):
        v = torch.randn((64, 3), device=DEV, generator=g) * 2.0
        env.step(LV(v, torch.zeros(64, device=DEV)))
        pos = env._planes[0:3].T.double().cpu().numpy()
        _, rd, _ = t.nearest_point(pos)
        assert np.array_equal(env.nearest_dist.cpu().numpy(), rd)
        assert np.array_equal(env.collision.cpu().numpy(), rd < cfg.collision_radius)
