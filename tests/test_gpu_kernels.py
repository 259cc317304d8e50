"""GPU parity of K1 (dynamics), K2 (render) and the spatial queries against
the oracle and the reference golden fixtures, through the C-ABI."""

import math

import numpy as np
import pytest

import oracle
from conftest import golden, scene_from_golden
from parity_util import DEPTH_TOL, grazing_mask, state_error, summarize

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2407_14783_b200 import _native as nat  # noqa: E402
from paper_2407_14783_b200.geometry import Scene  # noqa: E402
from paper_2407_14783_b200.geometry.device import DeviceScenes  # noqa: E402
from paper_2407_14783_b200.geometry.queries import nearest_points, raycasts  # noqa: E402
from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig, native_params  # noqa: E402
from paper_2407_14783_b200.sensing import DOWNWARD, FORWARD, CameraModel, camera_pose_world  # noqa: E402

DEV = "cuda"


def planes(x, dtype):
    return torch.as_tensor(np.asarray(x), dtype=dtype, device=DEV).T.contiguous()


def run_step(kind, x, cmd, dtype, sim=None):
    p = native_params(QuadParams(), sim or SimConfig(), ControllerGains())
    pl = planes(x, dtype)
    a = torch.as_tensor(np.asarray(cmd), dtype=dtype, device=DEV).contiguous()
    n = pl.shape[1]
    rot = torch.empty((n, 4), dtype=dtype, device=DEV)
    bad = torch.empty(n, dtype=torch.uint8, device=DEV)
    code = nat.QB_F32 if dtype == torch.float32 else nat.QB_F64
    nat.check(nat.lib().qb_dynamics_step(p, nat.CMD[kind], code, n, n, nat.ptr(pl), nat.ptr(a), nat.ptr(rot), nat.ptr(bad),
                                         nat.stream_of()))
    torch.cuda.synchronize()
    return pl.T.double().cpu().numpy(), rot.double().cpu().numpy(), bad.cpu().numpy()


@pytest.mark.parametrize("kind", ["srt", "ctbr", "rotor"])
@pytest.mark.parametrize("integ,sub", [("rk4", 2), ("euler", 4), ("rk4", 1)])
def test_k1_fp64_bit_exact(gdyn, kind, integ, sub):
    """Exact-double build == reference dynamics.step (+ controller) bit for bit."""
    x, rot, bad = run_step(kind, gdyn["state0"], gdyn[f"{kind}_cmd"], torch.float64, SimConfig(integrator=integ, substeps=sub))
    assert not bad.any()
    assert np.array_equal(rot, gdyn[f"{kind}_speeds"])
    assert np.array_equal(x, gdyn[f"{kind}_{integ}{sub}_next"])


@pytest.mark.parametrize("kind", ["ps", "lv"])
def test_k1_fp64_lv_ps(gdyn, kind):
    """LV/PS use cos/sin of the yaw set-point: libm vs numpy differ by <= 1 ulp."""
    x, rot, _ = run_step(kind, gdyn["state0"], gdyn[f"{kind}_cmd"], torch.float64)
    # near zero thrust sqrt(f/k2) turns a 1e-16 N difference into ~1e-5 rad/s
    np.testing.assert_allclose(rot, gdyn[f"{kind}_speeds"], rtol=1e-12, atol=1e-4)
    assert state_error(x, gdyn[f"{kind}_rk42_next"]).max() < 1e-8


@pytest.mark.parametrize("kind", ["srt", "ctbr", "ps", "lv", "rotor"])
def test_k1_fp32_one_step(gdyn, kind):
    x, rot, _ = run_step(kind, gdyn["state0"], gdyn[f"{kind}_cmd"], torch.float32)
    err = state_error(x, gdyn[f"{kind}_rk42_next"])
    assert err.max() < 1e-5, summarize(err)


def _gpu_trajectory(kind, x0, cmds):
    p = native_params(QuadParams(), SimConfig(), ControllerGains())
    pl = planes(x0, torch.float32)
    n = pl.shape[1]
    out = [pl.T.double().cpu().numpy()]
    for t in range(cmds.shape[0]):
        a = torch.as_tensor(cmds[t], dtype=torch.float32, device=DEV).contiguous()
        nat.check(nat.lib().qb_dynamics_step(p, nat.CMD[kind], nat.QB_F32, n, n, nat.ptr(pl), nat.ptr(a), None, None,
                                             nat.stream_of()))
        out.append(pl.T.double().cpu().numpy())
    return np.asarray(out)


def _check_100_steps(kind, x0, cmds, ref, label):
    """North star: FP32 states within 1e-5 (per-field floors) over 100 steps,
    on every env the reference itself can hold there.

    Closed loops through the saturating mixer (LV / PS) and tumbling open-loop
    SRT are ill-conditioned at FP32 precision: the FP64 oracle
    FED FP32-ROUNDED INPUTS (round to nearest, plus one-ulp perturbed replicas)
    already spends more than half of the 1e-5 budget on some envs.  Those envs
    are flagged by the oracle alone (oracle/parity.py fp32_conditioning) before
    the GPU result is looked at; every other env must meet 1e-5 exactly as the
    north star states.
    Reported: per-field max and p99, count over 1e-5, flagged count, and how
    many flagged envs start diverging at a mixer event (a rotor within 1e-3 N
    of the thrust floor, where sqrt(f/k2) amplifies rounding, or a torque
    scale s < 1)."""
    from oracle.parity import fp32_conditioning

    P = oracle.pack_params(QuadParams(), SimConfig(), ControllerGains())
    cond = fp32_conditioning(P, kind, x0, cmds, ref=ref)
    got = _gpu_trajectory(kind, x0, cmds)
    err = state_error(got, ref)  # (T+1, N, 17)
    env_err = err.max(axis=(0, 2))
    field_max = err.max(axis=(0, 1))
    field_p99 = np.percentile(err.max(axis=0), 99, axis=0)
    over = env_err > 1e-5
    fl = cond["flagged"]
    print(f"{label} {kind}: envs {len(env_err)}, GPU over 1e-5: {int(over.sum())}, oracle-flagged (FP32-rounded inputs "
          f"leave 1e-5): {int(fl.sum())}, flagged with a mixer event at onset: {int(cond['mixer_at_onset'].sum())}; "
          f"unflagged worst {env_err[~fl].max() if (~fl).any() else 0:.2e}")
    print("  per-field max", np.array2string(field_max, precision=1))
    print("  per-field p99", np.array2string(field_p99, precision=1))
    bad = over & ~fl
    assert not bad.any(), (f"{int(bad.sum())} unflagged envs over 1e-5", env_err[bad], cond["dev"][bad])
    if fl.any():  # flagged envs: the GPU drifts no further than a small multiple of the reference's own FP32-input drift
        ratio = env_err[fl] / cond["dev"][fl]
        print(f"  flagged: GPU err / oracle FP32-input drift: median {np.median(ratio):.2f}, max {ratio.max():.2f}")
        assert ratio.max() < 4.0, ratio.max()
    return over, fl


@pytest.mark.parametrize("kind", ["ctbr", "srt", "ps", "lv"])
def test_k1_fp32_100_steps(gdyn, kind):
    """The reference's own 100-step closed loops (golden, 16 envs)."""
    traj, cmds = gdyn[f"traj_{kind}"], gdyn[f"traj_{kind}_cmds"]
    over, fl = _check_100_steps(kind, traj[0], cmds, traj, "golden")
    if kind == "ctbr":  # well conditioned: every env within 1e-5
        assert not over.any()


@pytest.mark.parametrize("kind", ["ctbr", "srt", "ps", "lv"])
def test_k1_fp32_100_steps_parity_set(kind):
    """SURVEY 8-D parity set: 1024 seeded random envs x 100 steps with a fresh
    command every step, reference = the oracle (pinned bit-exact to the
    reference's goldens).  Fresh random commands every step make these loops
    strongly chaotic: for SRT / PS nearly every env is flagged, and the claim
    that carries is the ratio bound on flagged envs."""
    from oracle.parity import oracle_trajectory, parity_set

    P = oracle.pack_params(QuadParams(), SimConfig(), ControllerGains())
    x0, cmds = parity_set(kind, 1024, 100, seed=11)
    ref, _, _ = oracle_trajectory(P, kind, x0, cmds)
    _check_100_steps(kind, x0, cmds, ref, "parity-set")


def test_command_fp64_exact(gdyn):
    p = native_params()
    for kind in ("srt", "ctbr"):
        pl = planes(gdyn["state0"], torch.float64)
        a = torch.as_tensor(gdyn[f"{kind}_cmd"], dtype=torch.float64, device=DEV).contiguous()
        out = torch.empty_like(a)
        nat.check(nat.lib().qb_command_to_rotor_speeds(p, nat.CMD[kind], nat.QB_F64, a.shape[0], a.shape[0], nat.ptr(pl),
                                                       nat.ptr(a), nat.ptr(out), nat.stream_of()))
        assert np.array_equal(out.cpu().numpy(), gdyn[f"{kind}_speeds"])


def test_nonfinite_mask_gpu():
    x = np.zeros((5, 17)); x[:, 6] = 1.0; x[:, 13:] = 900.0
    x[2, 4] = np.nan
    for dt in (torch.float32, torch.float64):
        _, _, bad = run_step("rotor", x, np.full((5, 4), 900.0), dt)
        assert bad.tolist() == [0, 0, 1, 0, 0]


def _dev_scene(g, name):
    t = scene_from_golden(g, name)

    class _S:  # minimal Scene-like carrier of the golden primitive table
        arrays = type("A", (), dict(prim_type=t.prim_type, prim_data=t.prim_data, prim_object_id=t.prim_oid,
                                    prim_aabb_lo=t.prim_lo, prim_aabb_hi=t.prim_hi, __len__=lambda s: len(t.prim_type)))()

    return DeviceScenes([_S()], device=DEV), t


@pytest.mark.parametrize("name", ["nav", "tess"])
def test_nearest_point_exact(ggeo, name):
    ds, _ = _dev_scene(ggeo, name)
    pt, d, oid = nearest_points(ds, ggeo[f"{name}_np_q"])
    assert np.array_equal(oid.cpu().numpy(), ggeo[f"{name}_np_id"])
    if name == "nav":  # analytic primitives: one primitive per object -> bit-exact
        assert np.array_equal(pt.cpu().numpy(), ggeo[f"{name}_np_pt"])
        assert np.array_equal(d.cpu().numpy(), ggeo[f"{name}_np_d"])
    else:  # meshes: equal-distance triangles of ONE object tie; the reference keeps
        # whichever its traversal met first, so the point may differ by an ulp
        assert np.abs(pt.cpu().numpy() - ggeo[f"{name}_np_pt"]).max() < 1e-12
        assert np.abs(d.cpu().numpy() - ggeo[f"{name}_np_d"]).max() < 1e-12


@pytest.mark.parametrize("name", ["nav", "tess"])
def test_raycast(ggeo, name):
    ds, _ = _dev_scene(ggeo, name)
    t64, id64 = raycasts(ds, ggeo[f"{name}_rc_o"], ggeo[f"{name}_rc_d"], 10.0, dtype=torch.float64)
    assert np.array_equal(t64.cpu().numpy(), ggeo[f"{name}_rc_t"])
    assert np.array_equal(id64.cpu().numpy(), ggeo[f"{name}_rc_id"])
    t32, id32 = raycasts(ds, ggeo[f"{name}_rc_o"], ggeo[f"{name}_rc_d"], 10.0, dtype=torch.float32)
    ref_t, ref_id = ggeo[f"{name}_rc_t"], ggeo[f"{name}_rc_id"]
    same = id32.cpu().numpy() == ref_id
    assert same.mean() > 0.99
    hit = same & (ref_id >= 0)
    assert np.abs(t32.cpu().numpy()[hit] - ref_t[hit]).max() < 1e-4


def _render(ds, cam, pos, quat, dtype):
    o, r = camera_pose_world(pos, quat, cam)
    n = len(o)
    ot = torch.as_tensor(o, dtype=dtype, device=DEV).contiguous()
    rt = torch.as_tensor(r, dtype=dtype, device=DEV).contiguous()
    depth = torch.empty((n, cam.height, cam.width), dtype=dtype, device=DEV)
    seg = torch.empty((n, cam.height, cam.width), dtype=torch.int32, device=DEV)
    code = nat.QB_F32 if dtype == torch.float32 else nat.QB_F64
    nat.check(nat.lib().qb_render_poses(ds.handle, cam.native(), code, n, nat.ptr(ot), nat.ptr(rt), None, nat.ptr(depth),
                                        nat.ptr(seg), None, None, 0, nat.stream_of()))
    return depth.double().cpu().numpy(), seg.cpu().numpy(), o, r


@pytest.mark.parametrize("name,rot", [("nav", "fwd"), ("tess", "fwd"), ("landing", "down")])
def test_render_fp64_bit_exact(ggeo, name, rot):
    ds, _ = _dev_scene(ggeo, name)
    cam = CameraModel(rotation=FORWARD if rot == "fwd" else DOWNWARD)
    d, s, _, _ = _render(ds, cam, ggeo[f"{name}_render_pos"], ggeo[f"{name}_render_quat"], torch.float64)
    assert np.array_equal(s, ggeo[f"{name}_render_ids"])
    assert np.array_equal(d, ggeo[f"{name}_render_depth"])


@pytest.mark.parametrize("name,rot", [("nav", "fwd"), ("tess", "fwd"), ("landing", "down")])
def test_render_fp32_tolerance(ggeo, name, rot):
    ds, sc = _dev_scene(ggeo, name)
    cam = CameraModel(rotation=FORWARD if rot == "fwd" else DOWNWARD)
    d, s, o, r = _render(ds, cam, ggeo[f"{name}_render_pos"], ggeo[f"{name}_render_quat"], torch.float32)
    graz, d0, i0 = grazing_mask(sc, o, r, cam.width, cam.height, cam.tan_half_h, cam.tan_half_v, cam.max_range)
    bad = (s != i0) | (np.abs(d - d0) > DEPTH_TOL)
    print(f"{name}: grazing {graz.mean():.2e}, mismatched {bad.mean():.2e}, non-grazing mismatched {(bad & ~graz).sum()}")
    assert not (bad & ~graz).any()
    assert bad.mean() < 1e-3


def test_floor_kat(ggeo):
    """2 m above a floor looking down -> every pixel 2.0."""
    from paper_2407_14783_b200.geometry import floor_scene

    ds = DeviceScenes([floor_scene()], device=DEV)
    cam = CameraModel(rotation=DOWNWARD)
    for dt in (torch.float64, torch.float32):
        d, s, _, _ = _render(ds, cam, np.array([[0.0, 0, 2.0]]), np.array([[1.0, 0, 0, 0]]), dt)
        assert np.abs(d - 2.0).max() < (1e-15 if dt == torch.float64 else 1e-6)
        assert (s == 1).all()
    assert np.array_equal(_render(ds, cam, np.array([[0.0, 0, 2.0]]), np.array([[1.0, 0, 0, 0]]), torch.float64)[0],
                          ggeo["kat_floor_depth"])


def test_rng_seeding_matches_numpy():
    g = golden("rng")
    seeds = g["seeds"]
    for i, s in enumerate(seeds):
        out = torch.empty((1, 4), dtype=torch.int64, device=DEV)
        nat.check(nat.lib().qb_rng_seed(int(s), 1, nat.ptr(out), nat.stream_of()))
        words = out.cpu().numpy().view(np.uint64)[0]
        assert np.array_equal(words, g["pcg_state"][i])
        dbl = torch.empty((1, 8), dtype=torch.float64, device=DEV)
        nat.check(nat.lib().qb_rng_doubles(1, nat.ptr(out), 8, nat.ptr(dbl), nat.stream_of()))
        assert np.array_equal(dbl.cpu().numpy()[0], g["doubles"][i])


def test_multi_scene_set(ggeo):
    """Two scenes in one handle: per-env scene ids route queries correctly."""
    ds, _ = _dev_scene(ggeo, "nav")
    t1 = scene_from_golden(ggeo, "nav")
    t2 = scene_from_golden(ggeo, "landing")

    def carrier(t):
        class _S:
            arrays = type("A", (), dict(prim_type=t.prim_type, prim_data=t.prim_data, prim_object_id=t.prim_oid,
                                        prim_aabb_lo=t.prim_lo, prim_aabb_hi=t.prim_hi, __len__=lambda s: len(t.prim_type)))()
        return _S()

    both = DeviceScenes([carrier(t1), carrier(t2)], device=DEV)
    q = np.random.default_rng(0).uniform([-5, -5, 0], [5, 5, 4], (200, 3))
    which = torch.as_tensor(np.arange(200) % 2, dtype=torch.int32, device=DEV)
    pt, d, oid = nearest_points(both, q, env_scene=which)
    for k, t in enumerate((t1, t2)):
        rpt, rd, rid = t.nearest_point(q[k::2])
        assert np.array_equal(d.cpu().numpy()[k::2], rd) and np.array_equal(oid.cpu().numpy()[k::2], rid)


@pytest.mark.parametrize("name", ["nav", "tess", "landing"])
def test_culling_and_bvh_kernels_vs_oracle(ggeo, name):
    """Both FP32 render kernels (frustum-culling and BVH-packet) against the
    FP64 oracle on 256 random poses x 2 camera mounts: equal ids and depth
    within 1e-4 m on every non-grazing pixel."""
    from paper_2407_14783_b200.sensing import render_state

    ds, sc = _dev_scene(ggeo, name)
    rng = np.random.default_rng(5)
    n = 256
    pos = rng.uniform([-4.5, -4.5, 0.2], [4.5, 4.5, 3.8], (n, 3))
    q = rng.normal(size=(n, 4)) + np.array([2.0, 0, 0, 0])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    planes = torch.zeros((17, n), dtype=torch.float32, device=DEV)
    planes[0:3] = torch.as_tensor(pos.T, dtype=torch.float32)
    planes[6:10] = torch.as_tensor(q.T, dtype=torch.float32)
    st = planes.T.double().cpu().numpy()
    for rot in (FORWARD, DOWNWARD):
        cam = CameraModel(rotation=rot, width=64, height=48)
        o, r = oracle.camera_pose_world(st[:, 0:3], st[:, 6:10], cam.rotation, cam.translation)
        graz, d0, i0 = grazing_mask(sc, o, r, cam.width, cam.height, cam.tan_half_h, cam.tan_half_v, cam.max_range)
        for mode in (1, 2):
            d = torch.empty((n, 48, 64), dtype=torch.float32, device=DEV)
            sg = torch.empty((n, 48, 64), dtype=torch.int32, device=DEV)
            render_state(ds, cam, planes, depth=d, seg=sg, mode=mode)
            bad = (sg.cpu().numpy() != i0) | (np.abs(d.double().cpu().numpy() - d0) > DEPTH_TOL)
            print(name, "mode", mode, f"grazing {graz.mean():.2e} mismatched {bad.mean():.2e} "
                  f"non-grazing mismatched {(bad & ~graz).sum()}")
            for w in np.argwhere(bad & ~graz)[:3]:
                w = tuple(w)
                print("   pixel", w, "gpu", float(d.cpu().numpy()[w]), int(sg.cpu().numpy()[w]), "oracle", d0[w], i0[w],
                      "pos", st[w[0], 0:3], "q", st[w[0], 6:10])
            assert not (bad & ~graz).any()
            assert bad.mean() < 1e-3


def test_nan_action_flags_nonfinite():
    """A NaN command propagates to a non-finite state in the reference
    (np.clip keeps NaN); the FP32 build's single-instruction clamps must not
    hide it."""
    x = np.zeros((4, 17)); x[:, 6] = 1.0; x[:, 13:] = 900.0
    for kind, a in (("rotor", [900.0] * 4), ("ctbr", [9.81, 0, 0, 0]), ("lv", [0, 0, 0, 0])):
        acts = np.tile(np.asarray(a, float), (4, 1))
        acts[1, 0] = np.nan
        acts[3, 3] = np.nan
        for dt in (torch.float32, torch.float64):
            _, _, bad = run_step(kind, x, acts, dt)
            assert bad.tolist() == [0, 1, 0, 1], (kind, dt)


def test_controller_stages_fp64_match_reference():
    """control.mixer (thrusts + saturated), lv_to_ctbr, ps_to_ctbr, exact double."""
    from conftest import golden
    from paper_2407_14783_b200 import control as C
    from paper_2407_14783_b200.dynamics import QuadState

    g = golden("control")
    m = C.mixer(g["force"], g["torque"])
    assert np.array_equal(m.thrusts, g["thrusts"])
    assert np.array_equal(m.saturated, g["saturated"])
    st = QuadState(torch.as_tensor(g["states"].T.copy(), device="cuda"))
    lv = C.lv_to_ctbr(C.command_from_array("lv", g["lv"]), st).as_array()
    ps = C.ps_to_ctbr(C.command_from_array("ps", g["ps"]), st).as_array()
    # the attitude construction uses sin/cos of the yaw (CUDA libm vs numpy: <= 1 ulp)
    np.testing.assert_allclose(lv, g["lv_ctbr"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(ps, g["ps_ctbr"], rtol=1e-13, atol=1e-13)
