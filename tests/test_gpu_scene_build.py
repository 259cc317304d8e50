"""GPU scene ingestion: qb_scene_create_device -- the primitive
table expanded on the device and a linear BVH built there -- against the
host build (binned SAH, qb_scene_create).  Results are traversal-order
independent (nearest t / d^2, ties to the lower object id), so renders (FP32
BVH and culling kernels, FP64 exact) must be equal bit for bit and query
distances too (object ids up to the exact-tie caveat of _check_queries);
only the tree (and its traversal cost) differs."""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2407_14783_b200 import _native as nat  # noqa: E402
from paper_2407_14783_b200.geometry import Box, Scene, SceneObject, Sphere, TriMesh, indoor_mesh_scene  # noqa: E402
from paper_2407_14783_b200.geometry.device import DeviceScenes, flatten_on_device  # noqa: E402
from paper_2407_14783_b200.geometry.queries import nearest_points, raycasts  # noqa: E402
from paper_2407_14783_b200.sensing import DOWNWARD, FORWARD, CameraModel, render_state  # noqa: E402

DEV = "cuda"


def _nav():
    from paper_2407_14783_b200.env import navigation_config

    return navigation_config(scene_seed=0).scenes[0].materialize()


def _tiny(k):
    objs = [SceneObject(1 + j, Sphere(center=np.array([1.0 + 0.7 * j, 0.2 * j, 1.5]), radius=0.3)) for j in range(k)]
    return Scene(objs)


def _mixed():
    """Spheres, rotated boxes and a small mesh in one scene (all three prim types)."""
    rng = np.random.default_rng(3)
    objs = [SceneObject(1, Box(center=np.array([0.0, 0, -0.05]), half_extents=np.array([6.0, 6.0, 0.05]),
                               rotation=np.eye(3)))]
    for j in range(12):
        c = rng.uniform([-4, -4, 0.5], [4, 4, 3.5])
        if j % 2:
            objs.append(SceneObject(2 + j, Sphere(center=c, radius=float(rng.uniform(0.2, 0.6)))))
        else:
            a = rng.normal(size=3)
            a /= np.linalg.norm(a)
            th = rng.uniform(0, np.pi)
            K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
            R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
            objs.append(SceneObject(2 + j, Box(center=c, half_extents=rng.uniform(0.1, 0.5, 3), rotation=R)))
    v = rng.uniform([-2, -2, 1], [2, 2, 3], (40, 3))
    t = rng.integers(0, 40, (60, 3))
    objs.append(SceneObject(50, TriMesh(vertices=v, triangles=t)))
    return Scene(objs)


SCENES = {"nav": _nav, "mixed": _mixed, "tiny1": lambda: _tiny(1), "tiny3": lambda: _tiny(3), "tiny5": lambda: _tiny(5),
          "hall50k": lambda: indoor_mesh_scene(0, target_triangles=50_000)}


def _planes(n, seed, lo, hi, dtype):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(lo, hi, (n, 3))
    q = rng.normal(size=(n, 4)) + np.array([2.0, 0, 0, 0])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    pl = torch.zeros((17, n), dtype=dtype, device=DEV)
    pl[0:3] = torch.as_tensor(pos.T, dtype=dtype)
    pl[6:10] = torch.as_tensor(q.T, dtype=dtype)
    return pl


def _render(ds, cam, pl, mode, env_scene=None):
    n = pl.shape[1]
    d = torch.empty((n, cam.height, cam.width), dtype=pl.dtype, device=DEV)
    s = torch.empty((n, cam.height, cam.width), dtype=torch.int32, device=DEV)
    render_state(ds, cam, pl, env_scene=env_scene, depth=d, seg=s, mode=mode)
    return d.cpu().numpy(), s.cpu().numpy()


def _same(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("name", list(SCENES))
def test_device_build_equals_host_build(name):
    sc = SCENES[name]()
    host, dev = DeviceScenes([sc], device=DEV), DeviceScenes([sc], device=DEV, build="device")
    n_prims = len(sc.arrays)
    assert dev.n_prims == host.n_prims == n_prims
    assert dev.n_nodes == 2 * n_prims - 1 and 1 <= dev.max_depth <= 62
    assert np.array_equal(dev.bounds, host.bounds)
    lo, hi = host.bounds[0, :3], host.bounds[0, 3:]
    span = hi - lo
    for rot in (FORWARD, DOWNWARD):
        cam = CameraModel(rotation=rot, width=64, height=48)
        for dtype, modes in ((torch.float32, (1, 2) if n_prims <= 256 else (1,)), (torch.float64, (0,))):
            pl = _planes(96, 7, lo + 0.1 * span, hi - 0.1 * span, dtype)
            for mode in modes:
                assert _same(_render(host, cam, pl, mode), _render(dev, cam, pl, mode)), (name, dtype, mode)
    q = np.random.default_rng(1).uniform(lo - 1.0, hi + 1.0, (500, 3))
    dirs = np.random.default_rng(2).normal(size=(500, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    _check_queries(host, dev, q, dirs)


def _check_queries(host, dev, q, dirs, env_scene=None):
    """Nearest points and ray casts.  Distances / hit t must be equal; the
    object may differ only on exact ties between objects whose exact-double
    AABB test is an ulp less conservative than the primitive test (query
    points inside two overlapping boxes at a corner): there the reference's
    own answer depends on its tree too (kernels.py:150, 353 prune with the
    AABB bound before the id tie-break).  Mesh points of equal-distance
    triangles of one object may differ by an ulp (kernels.py:150)."""
    pa, da, ia = (x.cpu().numpy() for x in nearest_points(host, q, env_scene=env_scene))
    pb, db, ib = (x.cpu().numpy() for x in nearest_points(dev, q, env_scene=env_scene))
    assert np.array_equal(da, db)
    same = ia == ib
    assert same.mean() >= 0.99, np.nonzero(~same)
    assert np.abs(pa - pb)[same].max() < 1e-12
    for dt in (torch.float32, torch.float64):
        ta, ja = (x.cpu().numpy() for x in raycasts(host, q, dirs, 10.0, dtype=dt, env_scene=env_scene))
        tb, jb = (x.cpu().numpy() for x in raycasts(dev, q, dirs, 10.0, dtype=dt, env_scene=env_scene))
        assert np.array_equal(ta, tb), dt
        assert (ja == jb).mean() >= 0.99, (dt, np.nonzero(ja != jb))


def test_device_build_multi_scene_routing():
    scenes = [_nav(), _tiny(1), _mixed(), _tiny(5)]
    host, dev = DeviceScenes(scenes, device=DEV), DeviceScenes(scenes, device=DEV, build="device")
    assert np.array_equal(host.bounds, dev.bounds) and dev.n_scenes == 4
    n = 400
    which = torch.as_tensor(np.arange(n) % 4, dtype=torch.int32, device=DEV)
    cam = CameraModel(rotation=FORWARD, width=32, height=32)
    for dtype in (torch.float32, torch.float64):
        pl = _planes(n, 11, [-4, -4, 0.5], [4, 4, 3.5], dtype)
        assert _same(_render(host, cam, pl, 0, which), _render(dev, cam, pl, 0, which)), dtype
    q = np.random.default_rng(4).uniform([-5, -5, 0], [5, 5, 4], (n, 3))
    dirs = np.random.default_rng(5).normal(size=(n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    _check_queries(host, dev, q, dirs, env_scene=which)


def test_device_flatten_matches_host_rows():
    sc = _mixed()
    t = sc.arrays
    ptype, pdata, poid, plo, phi = (x.cpu().numpy() for x in flatten_on_device(sc, torch.device(DEV)))
    assert np.array_equal(ptype, t.prim_type) and np.array_equal(poid, t.prim_object_id)
    assert np.array_equal(pdata, t.prim_data)
    assert np.array_equal(plo, t.prim_aabb_lo) and np.array_equal(phi, t.prim_aabb_hi)


def test_device_build_env_equivalence():
    """An env whose scenes were built on the device steps exactly like one
    built on the host (renders, proximity, flags, rewards)."""
    from paper_2407_14783_b200.control import LV
    from paper_2407_14783_b200.env import make_env, navigation_config

    cfg = navigation_config(scene_seed=0, num_agents=256, with_segmentation=True)
    e_h, e_d = make_env(cfg), make_env(cfg, scene_build="device")
    o_h, o_d = e_h.reset(seed=3), e_d.reset(seed=3)
    assert torch.equal(o_h["depth"], o_d["depth"]) and torch.equal(o_h["segmentation"], o_d["segmentation"])
    g = torch.Generator(device=DEV).manual_seed(0)
    for _ in range(30):
        v = torch.randn((256, 3), device=DEV, generator=g) * 1.5
        yaw = torch.rand(256, device=DEV, generator=g) * 6.0 - 3.0
        r_h, r_d = e_h.step(LV(v, yaw)), e_d.step(LV(v, yaw))
        assert torch.equal(e_h._planes, e_d._planes)
        assert torch.equal(r_h.reward, r_d.reward) and torch.equal(r_h.terminated, r_d.terminated)
        assert torch.equal(r_h.observations["depth"], r_d.observations["depth"])
        assert torch.equal(r_h.observations["segmentation"], r_d.observations["segmentation"])


def test_device_build_validation():
    import ctypes

    sc = _tiny(3)
    ptype, pdata, poid, plo, phi = flatten_on_device(sc, torch.device(DEV))
    offs = np.array([0, 3], np.int64)
    h = ctypes.c_void_p()
    P = offs.ctypes.data_as(ctypes.c_void_p)
    lib = nat.lib()

    def create(t, o, lo, hi):
        return lib.qb_scene_create_device(1, P, t.data_ptr(), pdata.data_ptr(), o.data_ptr(), lo.data_ptr(),
                                          hi.data_ptr(), ctypes.byref(h), nat.stream_of())

    assert create(ptype, poid, plo, phi) == 0
    assert lib.qb_scene_destroy(h) == 0
    bad_oid = poid.clone()
    bad_oid[1] = 0
    assert create(ptype, bad_oid, plo, phi) != 0 and b"object ids" in lib.qb_last_error()
    bad_t = ptype.clone()
    bad_t[2] = 7
    assert create(bad_t, poid, plo, phi) != 0 and b"type" in lib.qb_last_error()
    assert create(ptype, poid, phi, plo) != 0 and b"bounds" in lib.qb_last_error()  # lo > hi
    empty = np.array([0, 0], np.int64)
    assert lib.qb_scene_create_device(1, empty.ctypes.data_as(ctypes.c_void_p), ptype.data_ptr(), pdata.data_ptr(),
                                      poid.data_ptr(), plo.data_ptr(), phi.data_ptr(), ctypes.byref(h),
                                      nat.stream_of()) != 0


def test_device_build_hall_500k():
    """Config 5's 5e5-triangle hall: device build time vs the host build, and
    equal renders of 128 down cameras (FP32 BVH kernel)."""
    sc = indoor_mesh_scene(0)
    sc.arrays  # host flatten outside the timing of either build
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host = DeviceScenes([sc], device=DEV)
    t1 = time.perf_counter()
    dev = DeviceScenes([sc], device=DEV, build="device")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"hall {dev.n_prims} tris: host SAH build {t1 - t0:.3f} s, device LBVH build {t2 - t1:.3f} s "
          f"(depth host {host.max_depth}, device {dev.max_depth})")
    cam = CameraModel(rotation=DOWNWARD)
    pl = _planes(128, 5, [-12, -12, 1.0], [12, 12, 4.5], torch.float32)
    pl[6:10] = 0
    pl[6] = 1.0  # level, looking down
    assert _same(_render(host, cam, pl, 1), _render(dev, cam, pl, 1))
    big = _planes(8192, 6, [-12, -12, 1.0], [12, 12, 4.5], torch.float32)
    big[6:10] = 0
    big[6] = 1.0
    for name, ds in (("host SAH", host), ("device LBVH", dev)):
        _render(ds, cam, big, 1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(3):
            _render(ds, cam, big, 1)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"  {name} tree: {3 * 8192 / ev[0].elapsed_time(ev[1]) * 1e3:.3g} frames/s (incl. D2H of the frames)")


@pytest.mark.parametrize("name", ["mixed", "hall500k"])
def test_device_build_renders_vs_oracle(name):
    """The device-built tree against the reference's algorithm directly (not
    only against the host build): 48 cameras rendered by the FP32 BVH kernel
    over the LBVH vs the oracle's restatement of render_batch
    (kernels.py:402-451) on the same poses -- ids equal and depth within
    1e-4 m on every pixel outside the oracle's grazing set, and the FP64
    kernel over the same LBVH bit-equal to the oracle."""
    import oracle
    from oracle.parity import DEPTH_TOL, grazing_mask

    sc = indoor_mesh_scene(0) if name == "hall500k" else _mixed()
    a = sc.arrays
    osc = oracle.OracleScene(a.prim_type, a.prim_data, a.prim_object_id, a.prim_aabb_lo, a.prim_aabb_hi)
    dev = DeviceScenes([sc], device=DEV, build="device")
    if name == "hall500k":
        cam = CameraModel(rotation=DOWNWARD)
        pl = _planes(48, 9, [-12, -12, 1.0], [12, 12, 4.5], torch.float32)
    else:
        cam = CameraModel(rotation=FORWARD)
        pl = _planes(48, 9, [-4, -4, 0.5], [4, 4, 3.5], torch.float32)
    d32, s32 = _render(dev, cam, pl, 1)
    st = pl.double().T.cpu().numpy()
    o, r = oracle.camera_pose_world(st[:, 0:3], st[:, 6:10], cam.rotation, cam.translation)
    graz, d0, i0 = grazing_mask(osc, o, r, cam.width, cam.height, cam.tan_half_h, cam.tan_half_v, cam.max_range,
                                cam_rot=cam.rotation)
    bad = (s32 != i0) | (np.abs(d32 - d0) > DEPTH_TOL)
    print(name, "mismatch", int(bad.sum()), "grazing", int(graz.sum()), "of", bad.size)
    assert not (bad & ~graz).any()
    assert bad.mean() < 1e-3
    d64, s64 = _render(dev, cam, pl.double(), 0)
    assert np.array_equal(s64, i0) and np.array_equal(d64, d0)
