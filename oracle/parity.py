"""Oracle re-evaluation of one GPU env step -- TEST INFRASTRUCTURE ONLY.

Used by tests/test_gpu_scale.py (parity at the benchmark configs' launch
shapes) and by bench.py's parity leg (a checker run after the timed region,
never inside it).  Everything here compares the GPU's outputs with the CPU
oracle evaluated on the GPU's OWN pre- and post-step states:

  dynamics   oracle controller + dynamics.step (dynamics.py:231-253,
             control.py:242-252) from the post-respawn pre-step state
             (base.py:175), in FP64, vs the FP32 post-step state:
             per-field normalised error (SURVEY 8-D floors)
  proximity  nearest point / collision / out-of-bounds (base.py:214-224),
             success / reward (tasks.py:45-118), terminated / truncated
             (base.py:193-194): bit-exact by construction (K3 evaluates them
             in exact double from the stored state)
  render     depth / segmentation of a seeded camera sample (kernels.py:402-451)
             vs the oracle render of the same poses: ids equal and depth
             within 1e-4 m off the grazing set (tests/parity_util.py), the
             mismatch and grazing fractions reported (north_star)
  spawns     per-agent default_rng(seed + global index) streams (base.py:95,
             114-147) for a sample of agents, re-drawn at reset and at every
             respawn and compared with the GPU rows
"""

from __future__ import annotations

import dataclasses
import numpy as np

from . import OracleScene, camera_pose_world, command_to_rotor_speeds, dynamics_step
from .env import OracleEnv

STATE_FLOOR = np.array([1.0] * 3 + [1.0] * 3 + [1.0] * 4 + [1.0] * 3 + [900.0] * 4)
DEPTH_TOL = 1e-4
# a rotor commanded within 1e-3 N of the thrust floor: sqrt(f/k2) turns an FP32
# rounding of f (~1e-7 N at hover-scale thrusts) into > 1e-3 rad/s of speed
FLOOR_BAND = 1e-3


def oracle_scenes(cfg):
    out = []
    for spec in cfg.scenes:
        t = spec.materialize().arrays
        out.append(OracleScene(t.prim_type, t.prim_data, t.prim_object_id, t.prim_aabb_lo, t.prim_aabb_hi))
    return out


def _axis_rot(axis, ang):
    axis = np.asarray(axis, float)
    axis = axis / np.linalg.norm(axis)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K


def grazing_mask(scene, origins, rotations, width, height, th, tv, max_range, d_o=1e-5, d_r=3e-6, cam_rot=None,
                 d_q=4e-7):
    """Pixels whose oracle result is unstable under perturbations a few times
    larger than the FP32 error of the pose: origin shifts
    (d_o ~ 20x the FP32 rounding of a position at 5 m), rigid rotations of
    the ray bundle (d_r), and -- with cam_rot, the camera's body mount -- a
    change of the quaternion's norm by d_q (a few FP32 ulps of |q|^2).  The
    last one matters because the reference builds the camera rotation from a
    non-unit quaternion (quatmath.to_matrix: I + s^2 (R - I) for q = s q_hat)
    and its sphere test assumes a unit ray direction (kernels.py:185-201:
    disc = b^2 - c, no |d|^2 term): near a sphere's rim the depth moves by
    ~ (b^2 / sqrt(disc)) * (|q|^2 - 1), i.e. 1e-4 m for |q|^2 - 1 = 1e-7, the
    FP32 rounding level of the stored state.  Returns (mask, depth0, ids0)."""
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
    if cam_rot is not None:  # rotations = to_matrix(q) @ cam_rot: scale to_matrix(q) - I by (1 +- d_q)
        dev = rotations - np.asarray(cam_rot, float)[None]
        for s in (-1.0, 1.0):
            perts.append((origins, np.ascontiguousarray(rotations + s * d_q * dev)))
    for o, r in perts:
        d, i = scene.render(o, r, width, height, th, tv, max_range)
        mask |= (i != ids0) | (np.abs(d - depth0) > DEPTH_TOL)
    return mask, depth0, ids0


class SpawnTracker:
    """The reference's per-agent generators for a sample of agents.

    Agent i (GLOBAL index g = index_offset + i) draws from
    default_rng(seed + g) (base.py:95); every spawn continues that stream
    (base.py:114-147), so re-drawing reset + respawns in order reproduces
    the rows the device writes.  Single-scene parallel-mode configs."""

    def __init__(self, cfg, oscenes, P, seed, local_idx, index_offset=0):
        assert len(oscenes) == 1 and cfg.mode != "swarm"
        self.idx = np.asarray(local_idx)
        sub = dataclasses.replace(cfg, num_agents=len(self.idx))
        self.env = OracleEnv(sub, oscenes, *P)
        self.env.rngs = [np.random.default_rng(int(seed) + index_offset + int(i)) for i in self.idx]
        self.env.scene_perm = np.arange(1)
        self.env.reset_counts = np.zeros(len(self.idx), int)
        self.env.state[:, 6] = 1.0

    def spawn(self, which):
        """Spawn the sampled agents selected by the bool mask `which` (over the
        sample); returns their fresh (k,17) rows."""
        rows = []
        for k in np.nonzero(which)[0]:
            self.env._spawn(int(k))
            rows.append(self.env.state[k].copy())
        return np.asarray(rows).reshape(-1, 17)


def _gpu_commands(env, pre, act):
    """The product's FP32 controller (qb_command_to_rotor_speeds) on given
    pre-step states / commands: the rotor-speed commands K1 computes."""
    import torch

    from paper_2407_14783_b200 import _native as nat

    n = len(pre)
    pl = torch.as_tensor(pre.T.copy(), dtype=env.dtype, device=env.device).contiguous()
    a = torch.as_tensor(act, dtype=env.dtype, device=env.device).contiguous()
    out = torch.empty((n, 4), dtype=env.dtype, device=env.device)
    code = nat.QB_F32 if env.dtype.itemsize == 4 else nat.QB_F64
    nat.check(nat.lib().qb_command_to_rotor_speeds(env._P, env._kind, code, n, n, nat.ptr(pl), nat.ptr(a), nat.ptr(out),
                                                   nat.stream_of()))
    return out.double().cpu().numpy()


def _as_np(t, dtype=None):
    a = t.detach().cpu().numpy()
    return a.astype(dtype) if dtype is not None else a


def env_step_parity(env, cfg, obs, action, oscenes, P, sample, *, check_render=True, graze=True):
    """Oracle re-evaluation of the env step that just ran (see module doc).

    env      the GPU env right after `obs = env.step(action).observations`
    action   (N,4) array of the step's command (as_array()), any dtype
    sample   local env indices whose cameras are re-rendered by the oracle
    Returns a dict of findings; the caller asserts on it."""
    n = env.num_agents
    st = _as_np(env._planes.T, np.float64)
    pre = _as_np(env._prev.T, np.float64)
    act = np.asarray(action, np.float64).reshape(n, 4)
    if env.dtype.itemsize == 4:
        act = act.astype(np.float32).astype(np.float64)
    sub = dataclasses.replace(cfg, num_agents=n)
    oenv = OracleEnv(sub, oscenes, *P)
    out = {}
    # -- dynamics from the GPU's own pre-step state (after respawn, base.py:175)
    sp = command_to_rotor_speeds(oenv.P, cfg.command_type, pre, act)
    ref, bad = dynamics_step(oenv.P, pre, sp)
    ref[bad] = pre[bad]
    err = np.abs(st - ref) / np.maximum(np.abs(ref), STATE_FLOOR)
    env_err = err.max(axis=1)
    out["state_err_max"] = float(err.max())
    out["state_err_p99"] = float(np.percentile(env_err, 99))
    over = env_err > 1e-5
    out["envs_over_1e-5"] = int(over.sum())
    if over.any():  # attributable to the reference's own conditioning at FP32 precision?
        fl, dv = one_step_conditioning(oenv.P, cfg.command_type, pre[over], act[over], ref[over], return_dev=True)
        out["over_1e-5_flagged"] = int(fl.sum())
        out["over_1e-5_unflagged"] = int((~fl).sum())
        out["unflagged_err_max"] = float(env_err[over][~fl].max()) if (~fl).any() else 0.0
        # split the error: the GPU's own FP32 rotor-speed commands for these envs
        # (qb_command_to_rotor_speeds, the controller template K1 inlines) fed to
        # the oracle's dynamics.step -- the dynamics must then meet 1e-5; the
        # rest is the controller, whose sqrt(f / k2) thrust inverse
        # (params.py:106-111) amplifies FP32 rounding of f without bound as f -> 0
        from . import command_mixer_info

        ref_cmd, msc, mfmin = command_mixer_info(oenv.P, cfg.command_type, pre[over], act[over])
        gcmd = _gpu_commands(env, pre[over], act[over])
        nx2, bad2 = dynamics_step(oenv.P, pre[over], gcmd)
        nx2[bad2] = pre[over][bad2]
        dyn_err = (np.abs(st[over] - nx2) / np.maximum(np.abs(nx2), STATE_FLOOR)).max(axis=1)
        floor = mfmin < FLOOR_BAND
        out["over_1e-5_dynamics_err_max"] = float(dyn_err.max())
        out["over_1e-5_thrust_floor"] = int(floor.sum())
        out["over_1e-5_explained"] = int((fl | floor).sum())
        out["over_1e-5_unexplained"] = int((~(fl | floor)).sum())
        worst_field = err[over].argmax(axis=1)
        out["over_1e-5_detail"] = [
            {"err": float(a), "oracle_spread": float(b), "field": int(f), "min_thrust": float(m), "mixer_scale": float(c),
             "dynamics_err_given_gpu_cmds": float(d), "cmd_err": float(np.abs(g - r).max())}
            for a, b, f, m, c, d, g, r in list(zip(env_err[over], dv, worst_field, mfmin, msc, dyn_err, gcmd, ref_cmd))[:8]]
    else:
        out["over_1e-5_flagged"] = out["over_1e-5_unflagged"] = out["over_1e-5_unexplained"] = 0
        out["over_1e-5_thrust_floor"] = out["over_1e-5_explained"] = 0
        out["unflagged_err_max"] = out["over_1e-5_dynamics_err_max"] = 0.0
    out["nonfinite_equal"] = bool(np.array_equal(_as_np(env._nonfinite).astype(bool), bad))
    # -- proximity, task hooks and flags on the GPU's post-step state
    oenv.state = st.copy()
    oenv.prev_state = pre.copy()
    oenv.agent_scene = _as_np(env.agent_scene).astype(int)
    oenv.step_counts = _as_np(env.step_counts).astype(int)
    oenv._refresh_proximity()
    oenv.nonfinite = _as_np(env._nonfinite).astype(bool)
    succ = oenv.get_success()
    rew = oenv.get_reward().astype(np.float32)
    term = succ | oenv.collision | oenv.oob | oenv.nonfinite
    trunc = ~term & (oenv.step_counts >= cfg.episode_max_steps)
    g = {"collision": _as_np(env._collision).astype(bool), "out_of_bounds": _as_np(env._oob).astype(bool),
         "success": _as_np(env._success).astype(bool), "terminated": _as_np(env._terminated).astype(bool),
         "truncated": _as_np(env._truncated).astype(bool)}
    o = {"collision": oenv.collision, "out_of_bounds": oenv.oob, "success": succ, "terminated": term, "truncated": trunc}
    out["flag_mismatches"] = {k: int((g[k] != o[k]).sum()) for k in g}
    out["flags_equal"] = all(v == 0 for v in out["flag_mismatches"].values())
    gd, gp = _as_np(env.nearest_dist), _as_np(env.nearest_pt)
    out["nearest_equal"] = bool(np.array_equal(gd, oenv.nearest_dist) and np.array_equal(gp, oenv.nearest_pt))
    out["nearest_max_abs_err"] = float(max(np.abs(gd - oenv.nearest_dist).max(), np.abs(gp - oenv.nearest_pt).max())) if n else 0.0
    rg = _as_np(env._reward)
    out["reward_equal"] = bool(np.array_equal(rg, rew))
    out["reward_max_abs_err"] = float(np.abs(rg.astype(np.float64) - rew).max()) if n else 0.0
    out["counts"] = {"envs": n, "collision": int(o["collision"].sum()), "out_of_bounds": int(o["out_of_bounds"].sum()),
                     "success": int(succ.sum()), "terminated": int(term.sum()), "truncated": int(trunc.sum())}
    if not check_render:
        return out
    # -- renders of the sampled cameras, read from the step's observations
    sample = np.asarray(sample)
    n_pix = n_bad = n_graz = n_bad_ng = n_seg_bad = n_depth_bad = 0
    cent_checked = cent_bad = 0
    cams = {}
    for spec in cfg.sensors:
        if spec.kind in ("depth", "segmentation") and not spec.noise:
            cam = spec.camera()
            cams.setdefault((cam.width, cam.height, cam.vertical_fov, cam.rotation.tobytes(), tuple(cam.translation),
                             cam.max_range), []).append((spec, cam))
    assert len(oscenes) == 1, "render parity: single-scene configs"
    sc = oscenes[0]
    for specs in cams.values():
        cam = specs[0][1]
        o_, r_ = camera_pose_world(st[sample, 0:3], st[sample, 6:10], cam.rotation, cam.translation)
        if graze:
            graz, d0, i0 = grazing_mask(sc, o_, r_, cam.width, cam.height, cam.tan_half_h, cam.tan_half_v, cam.max_range,
                                        cam_rot=cam.rotation)
        else:
            d0, i0 = sc.render(o_, r_, cam.width, cam.height, cam.tan_half_h, cam.tan_half_v, cam.max_range)
            graz = np.zeros(d0.shape, bool)
        bad_any = np.zeros(d0.shape, bool)
        for spec, _ in specs:
            img = obs[spec.name]
            x = _as_np(img[torch_index(img, sample)])
            if spec.kind == "depth":
                bad = np.abs(x.astype(np.float64) - d0) > DEPTH_TOL
                n_depth_bad += int(bad.sum())
            else:
                bad = x != i0
                n_seg_bad += int(bad.sum())
            bad_any |= bad
        n_pix += bad_any.size
        n_bad += int(bad_any.sum())
        n_graz += int(graz.sum())
        ng = bad_any & ~graz
        n_bad_ng += int(ng.sum())
        if ng.any():
            lst = out.setdefault("non_grazing_detail", [])
            for k, i, j in np.argwhere(ng)[:max(0, 16 - len(lst))]:
                k, i, j = int(k), int(i), int(j)
                det = {"camera": int(sample[k]), "pixel": [i, j], "ref_depth": float(d0[k, i, j]),
                       "ref_id": int(i0[k, i, j]), "cam_pos": [float(x) for x in o_[k]]}
                for spec, _ in specs:
                    det[spec.name] = float(_as_np(obs[spec.name][int(sample[k]), i, j]))
                lst.append(det)
            out.setdefault("first_non_grazing", lst[0])
        if cfg.task == "landing" and "target" in obs:  # pad centroid target (tasks.py:121-128)
            tgt = _as_np(obs["target"][torch_index(obs["target"], sample)])
            for k in range(len(sample)):
                if bad_any[k].any():
                    continue
                rows, cols = np.nonzero(i0[k] == 9)
                refc = np.array([cols.mean(), rows.mean()]) if len(rows) else np.array([-1.0, -1.0])
                cent_checked += 1
                cent_bad += int(not np.array_equal(tgt[k], refc.astype(np.float32)))
    out["render"] = {"cameras": int(len(sample)), "pixels": n_pix, "mismatch": n_bad,
                     "mismatch_frac": n_bad / max(n_pix, 1), "grazing_frac": n_graz / max(n_pix, 1),
                     "non_grazing_mismatch": n_bad_ng, "depth_mismatch": n_depth_bad, "seg_mismatch": n_seg_bad}
    if cent_checked:
        out["render"]["centroid_checked"] = cent_checked
        out["render"]["centroid_mismatch"] = cent_bad
    return out


def torch_index(t, idx):
    import torch

    return torch.as_tensor(np.asarray(idx), dtype=torch.long, device=t.device)


# ----------------------------------------------------------------------------
# FP32 conditioning of closed-loop trajectories


def parity_set(kind, n, T, seed=0):
    """SURVEY 8-D C1 parity set: seeded random initial states (p ~ U(-3,3)^3,
    v ~ N(0,1)^3, q = normalise(N(0,1)^4 + (3,0,0,0)), omega ~ N(0,1)^3,
    rotors ~ U(600,1200)^4) and a fresh command per step of the given kind."""
    rng = np.random.default_rng(seed)
    x = np.zeros((n, 17))
    x[:, 0:3] = rng.uniform(-3, 3, (n, 3))
    x[:, 3:6] = rng.normal(size=(n, 3))
    q = rng.normal(size=(n, 4)) + [3.0, 0, 0, 0]
    x[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    x[:, 10:13] = rng.normal(size=(n, 3))
    x[:, 13:17] = rng.uniform(600, 1200, (n, 4))
    if kind == "ctbr":
        c = np.concatenate([rng.uniform(5, 15, (T, n, 1)), rng.normal(size=(T, n, 3))], 2)
    elif kind == "lv":
        c = np.concatenate([rng.normal(scale=1.5, size=(T, n, 3)), rng.uniform(-np.pi, np.pi, (T, n, 1))], 2)
    elif kind == "ps":
        c = np.concatenate([rng.uniform(-3, 3, (T, n, 3)), rng.uniform(-np.pi, np.pi, (T, n, 1))], 2)
    else:  # srt: per-rotor thrusts [N]
        c = rng.uniform(0.0, 3.0, (T, n, 4))
    return x, c


def oracle_trajectory(P, kind, x0, cmds, round32=False, perturb_seed=None):
    """The oracle's closed loop (controller + dynamics.step per step).

    round32: the FP64 oracle fed FP32-ROUNDED inputs -- state and command are
    rounded to float32 before every step, as the GPU holds them; with
    perturb_seed the rounded state is further moved by a random relative
    amount within one float32 ulp (2^-23), a stand-in for the rounding of the
    GPU's own FP32 intermediates.
    Returns (traj (T+1,N,17), mixer scale (T,N), smallest rotor thrust (T,N))."""
    from . import command_mixer_info

    pr = np.random.default_rng(perturb_seed) if perturb_seed is not None else None
    x = np.array(x0, np.float64)
    out, scale, fmin = [x.copy()], [], []
    for t in range(len(cmds)):
        c = np.asarray(cmds[t], np.float64)
        if round32:
            x = x.astype(np.float32).astype(np.float64)
            c = c.astype(np.float32).astype(np.float64)
        if pr is not None:
            x = x * (1.0 + pr.uniform(-2.0**-23, 2.0**-23, x.shape))
        sp, s, fm = command_mixer_info(P, kind, x, c)
        scale.append(s)
        fmin.append(fm)
        x, bad = dynamics_step(P, x, sp)
        out.append(x.copy())
    return np.asarray(out), np.asarray(scale), np.asarray(fmin)


def fp32_conditioning(P, kind, x0, cmds, ref=None, variants=8, tol=1e-5, budget=0.5):
    """Per env: how far the FP64 oracle fed FP32-rounded inputs (round to
    nearest + variants-1 one-ulp perturbed replicas) drifts from the FP64
    reference trajectory, and whether the divergence starts at a mixer event.

    Returns dict(ref=(T+1,N,17), dev=(N,) max normalised deviation, flagged=
    dev > budget * tol (the reference fed FP32-rounded inputs alone uses up
    more than `budget` of the error budget), mixer_at_onset=(N,) bool: at the step the drift first exceeds
    tol/10 the reference's mixer had a rotor within 1e-3 N of the thrust floor
    (sqrt(f/k2) amplifies without bound there, params.py:106-111) or a torque
    scale s < 1 (control.py:122-127))."""
    if ref is None:
        ref, scale, fmin = oracle_trajectory(P, kind, x0, cmds)
    else:
        _, scale, fmin = oracle_trajectory(P, kind, x0, cmds)
    devs = []
    for v in range(variants):
        r, _, _ = oracle_trajectory(P, kind, x0, cmds, round32=True, perturb_seed=None if v == 0 else 1000 + v)
        devs.append((np.abs(r - ref) / np.maximum(np.abs(ref), STATE_FLOOR)).max(axis=2))
    dv = np.max(devs, axis=0)  # (T+1, N)
    onset = np.argmax(dv > tol / 10, axis=0)
    band = (fmin < 1e-3) | (scale < 1.0)  # (T, N)
    n = dv.shape[1]
    at = np.array([band[max(int(onset[i]) - 1, 0), i] for i in range(n)])
    dev = dv.max(axis=0)
    flagged = dev > budget * tol
    return {"ref": ref, "dev": dev, "flagged": flagged, "mixer_at_onset": at & flagged}


def one_step_conditioning(P, kind, pre, act, ref, variants=8, tol=1e-5, budget=0.5, return_dev=False):
    """Envs whose one-step oracle result moves by more than budget * tol when
    its FP32 input state is perturbed within one float32 ulp (relative
    2^-23) -- the single-step form of fp32_conditioning."""
    dev = np.zeros(len(pre))
    for v in range(variants):
        pr = np.random.default_rng(2000 + v)
        x = pre * (1.0 + pr.uniform(-2.0**-23, 2.0**-23, pre.shape))
        sp = command_to_rotor_speeds(P, kind, x, act)
        nx, bad = dynamics_step(P, x, sp)
        nx[bad] = x[bad]
        dev = np.maximum(dev, (np.abs(nx - ref) / np.maximum(np.abs(ref), STATE_FLOOR)).max(axis=1))
    return (dev > budget * tol, dev) if return_dev else dev > budget * tol
