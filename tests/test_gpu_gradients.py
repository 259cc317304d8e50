"""K1 adjoint: parity of the matrix-free VJP with the reference's dense
step Jacobians and rollout_grad (golden fixtures), finite-difference checks
of the controller adjoint (beyond the reference), autograd plumbing."""

import numpy as np
import pytest

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2407_14783_b200 import gradients as G  # noqa: E402
from paper_2407_14783_b200.dynamics import QuadState  # noqa: E402
from paper_2407_14783_b200.params import ControllerGains, QuadParams, SimConfig, native_params  # noqa: E402

GRAD_FLOOR = np.array([1.0] * 13 + [900.0] * 4)


@pytest.mark.parametrize("name", ["rk4", "euler4"])
def test_step_jacobian_matches_reference(gjac, name):
    sim = SimConfig() if name == "rk4" else SimConfig(integrator="euler", substeps=4)
    for i in range(len(gjac[f"{name}_state"])):
        sj = G.step_jacobian(gjac[f"{name}_state"][i], gjac[f"{name}_action"][i], sim, QuadParams())
        np.testing.assert_allclose(sj.full_state_jacobian, gjac[f"{name}_J"][i], rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(sj.full_action_jacobian, gjac[f"{name}_Ja"][i], rtol=1e-9, atol=1e-13)
        assert sj.saturation_boundary == bool(gjac[f"{name}_flag"][i])
        assert np.array_equal(sj.next_state.numpy()[0], gjac[f"{name}_next"][i])


def _loss(target):
    def loss(traj):
        g = np.zeros_like(traj)
        d = traj[-1, 0:3] - target
        g[-1, 0:3] = 2.0 * d
        g[:, 3:6] = 0.02 * traj[:, 3:6]
        return float(d @ d + 0.01 * (traj[:, 3:6] ** 2).sum()), g

    return loss


def test_rollout_grad_matches_reference_fp64(gjac):
    loss = _loss(gjac["rg_target"])
    for i in range(len(gjac["rg_x0"])):
        ga, gi, tape = G.rollout_grad(QuadState.from_vector(gjac["rg_x0"][i]), gjac["rg_actions"][i], loss, SimConfig(),
                                      QuadParams())
        np.testing.assert_allclose(ga, gjac["rg_grad_actions"][i], rtol=1e-8, atol=1e-14)
        np.testing.assert_allclose(gi, gjac["rg_grad_init"][i], rtol=1e-8, atol=1e-12)


def test_rollout_grad_batched_fp32(gjac):
    """All reference agents in one batched FP32 launch: gradients within 1e-4
    (per-field floors, BASELINE north star)."""
    x0 = gjac["rg_x0"]
    acts = np.transpose(gjac["rg_actions"], (1, 0, 2))  # (T,N,4)
    target = gjac["rg_target"]

    def loss(states):  # (T+1,N,17) tensor
        g = torch.zeros_like(states)
        d = states[-1, :, 0:3] - torch.as_tensor(target, dtype=states.dtype, device=states.device)
        g[-1, :, 0:3] = 2.0 * d
        g[:, :, 3:6] = 0.02 * states[:, :, 3:6]
        return None, g

    ga, gi, _ = G.rollout_grad(QuadState.from_vector(x0, dtype=torch.float32), torch.as_tensor(acts, dtype=torch.float32,
                                                                                               device="cuda"), loss)
    ga = ga.double().cpu().numpy().transpose(1, 0, 2)
    gi = gi.double().cpu().numpy()
    ref_a, ref_i = gjac["rg_grad_actions"], gjac["rg_grad_init"]
    # north star 1e-4, norm-wise per agent (max abs error / max abs gradient)
    err_a = np.abs(ga - ref_a).max(axis=(1, 2)) / np.abs(ref_a).max(axis=(1, 2))
    err_i = np.abs(gi - ref_i).max(axis=1) / np.abs(ref_i).max(axis=1)
    print("golden rollout_grad FP32: action", err_a, "init", err_i)
    assert err_a.max() < 1e-4 and err_i.max() < 1e-4


def _fd_check(kind, acts_fn, n=6, T=5, seed=0):
    """Central finite differences of L = sum_t w . x_t (exact double) vs the adjoint."""
    rng = np.random.default_rng(seed)
    x0 = np.zeros((n, 17))
    x0[:, 0:3] = rng.uniform(-1, 1, (n, 3))
    x0[:, 3:6] = rng.normal(scale=0.5, size=(n, 3))
    q = rng.normal(size=(n, 4)) * 0.1 + [1, 0, 0, 0]
    x0[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    x0[:, 10:13] = rng.normal(scale=0.5, size=(n, 3))
    x0[:, 13:17] = rng.uniform(800, 1000, (n, 4))
    acts = acts_fn(rng, T, n)
    w = rng.normal(size=(T + 1, n, 17)) * np.concatenate([np.ones(13), np.full(4, 1e-3)])
    P = native_params()
    init = torch.as_tensor(x0.T.copy(), dtype=torch.float64, device="cuda")
    a = torch.as_tensor(acts, dtype=torch.float64, device="cuda")
    wt = torch.as_tensor(w.transpose(0, 2, 1).copy(), dtype=torch.float64, device="cuda")

    def L(aa):
        tape, _ = G.rollout_planes(P, kind, init, aa)
        return float((tape * wt).sum())

    tape, _ = G.rollout_planes(P, kind, init, a)
    ga, gi, _ = G.backward_planes(P, kind, tape, a, wt)
    ga = ga.cpu().numpy()
    errs = []
    for (t, i, k) in [(0, 0, 0), (1, 1, 1), (2, 2, 2), (3, 3, 3), (4, 4, 0), (0, 5, 3), (T - 1, 0, 2)]:
        h = 1e-6 * max(1.0, abs(acts[t, i, k]))
        ap, am = a.clone(), a.clone()
        ap[t, i, k] += h
        am[t, i, k] -= h
        fd = (L(ap) - L(am)) / (2 * h)
        errs.append(abs(fd - ga[t, i, k]) / max(abs(fd), 1e-3))
    return max(errs)


def test_ctbr_adjoint_finite_differences():
    def acts(rng, T, n):
        a = np.zeros((T, n, 4))
        a[..., 0] = rng.uniform(8.0, 12.0, (T, n))
        a[..., 1:] = rng.normal(scale=1.0, size=(T, n, 3))
        return a

    assert _fd_check("ctbr", acts) < 1e-4


def test_srt_adjoint_finite_differences():
    assert _fd_check("srt", lambda rng, T, n: rng.uniform(1.0, 3.0, (T, n, 4))) < 1e-4


def test_rotor_adjoint_finite_differences():
    assert _fd_check("rotor", lambda rng, T, n: rng.uniform(700, 1100, (T, n, 4))) < 1e-4


def test_autograd_gradcheck():
    n = 3
    rng = np.random.default_rng(1)
    x0 = np.zeros((17, n)); x0[6] = 1.0; x0[13:17] = 900.0
    x0[0:3] = rng.uniform(-1, 1, (3, n)); x0[3:6] = rng.normal(size=(3, n)) * 0.3
    planes = torch.as_tensor(x0, dtype=torch.float64, device="cuda").requires_grad_(True)
    act = torch.as_tensor(rng.uniform(800, 1000, (n, 4)), dtype=torch.float64, device="cuda").requires_grad_(True)
    f = lambda p, a: G.differentiable_step(p, a)  # noqa: E731
    assert torch.autograd.gradcheck(f, (planes, act), eps=1e-6, atol=1e-5, rtol=1e-4)
    acts = torch.as_tensor(rng.uniform(800, 1000, (4, n, 4)), dtype=torch.float64, device="cuda").requires_grad_(True)
    g = lambda p, a: G.differentiable_rollout(p, a)[-1]  # noqa: E731
    assert torch.autograd.gradcheck(g, (planes, acts), eps=1e-6, atol=1e-5, rtol=1e-4)


def test_action_grad_sum_is_env_sum():
    n, T = 300, 6
    rng = np.random.default_rng(2)
    x0 = np.zeros((17, n)); x0[6] = 1.0; x0[13:17] = 900.0
    P = native_params()
    init = torch.as_tensor(x0, dtype=torch.float32, device="cuda")
    a = torch.as_tensor(rng.uniform(800, 1000, (T, n, 4)), dtype=torch.float32, device="cuda")
    tape, _ = G.rollout_planes(P, "rotor", init, a)
    g = torch.zeros_like(tape)
    g[-1, 2] = 1.0
    s = torch.zeros(T * 4, dtype=torch.float64, device="cuda")
    ga, gi, _ = G.backward_planes(P, "rotor", tape, a, g, action_grad_sum=s)
    np.testing.assert_allclose(s.cpu().numpy().reshape(T, 4), ga.double().sum(1).cpu().numpy(), rtol=1e-5, atol=1e-8)


def test_c4_fp32_gradients_h64_vs_reference():
    """Config 4 shape: hover states + U(+-0.1) position,
    rotor-speed actions 900 + N(0, 20^2), H = 64, loss = mean_envs
    |p_T - (1,0,2)|^2 + 1e-6 sum |a - 900|^2.  The FP32 forward + adjoint
    against the reference's rollout_grad (gradients.py:218-237, the oracle's
    dense-Jacobian restatement pinned to the reference's goldens) on 64 envs:
    north star 1e-4, norm-wise per env (max |g_gpu - g_ref| / max |g_ref|
    over the env's (T, 4) action gradient, and over its 17-vector initial-state
    gradient)."""
    n, T = 64, 64
    rng = np.random.default_rng(64)
    x0 = np.zeros((n, 17))
    x0[:, 0:3] = rng.uniform(-0.1, 0.1, (n, 3))
    x0[:, 6] = 1.0
    x0[:, 13:17] = QuadParams().hover_speed  # hover states (rotors at hover speed)
    acts = 900.0 + rng.normal(scale=20.0, size=(T, n, 4))
    x0 = x0.astype(np.float32).astype(np.float64)  # the FP32 run's exact inputs
    acts = acts.astype(np.float32).astype(np.float64)
    target = np.array([1.0, 0.0, 2.0])
    P = native_params()
    init = torch.as_tensor(x0.T.copy(), dtype=torch.float32, device="cuda")
    a = torch.as_tensor(acts, dtype=torch.float32, device="cuda")
    tape, _ = G.rollout_planes(P, "rotor", init, a)
    gtraj = torch.zeros_like(tape)
    gtraj[-1, 0:3] = 2.0 * (tape[-1, 0:3] - torch.as_tensor(target, dtype=torch.float32, device="cuda")[:, None]) / n
    ga, gi, _ = G.backward_planes(P, "rotor", tape, a, gtraj)
    ga = ga.double().cpu().numpy() + 2e-6 * (acts - 900.0)  # + d/da of the action penalty
    gi = gi.double().cpu().numpy().T
    Po = oracle.pack_params(QuadParams(), SimConfig(), ControllerGains())
    err_a, err_i = [], []
    for i in range(n):
        def loss(tr):
            g = np.zeros_like(tr)
            g[-1, 0:3] = 2.0 * (tr[-1, 0:3] - target) / n
            return 0.0, g

        ra, ri, _, _ = oracle.rollout_grad(Po, x0[i], acts[:, i], loss)
        ra = ra + 2e-6 * (acts[:, i] - 900.0)
        err_a.append(np.abs(ga[:, i] - ra).max() / np.abs(ra).max())
        err_i.append(np.abs(gi[i] - ri).max() / np.abs(ri).max())
    err_a, err_i = np.array(err_a), np.array(err_i)
    print(f"C4 FP32 H=64, {n} envs: action grad norm-wise rel err max {err_a.max():.2e} p99 "
          f"{np.percentile(err_a, 99):.2e} median {np.median(err_a):.2e}; init grad max {err_i.max():.2e}")
    assert err_a.max() < 1e-4
    assert err_i.max() < 1e-4


@pytest.mark.parametrize("kind", ["rotor", "ctbr", "srt"])
def test_split_adjoint_fp32_vs_fp64(kind, monkeypatch):
    """The FP32 production adjoint (k_rollout_bwd_tr: one translational and one
    rotational warp per 32 envs) against the exact-double adjoint of the same
    FP32 forward tape, for every differentiable action kind, n not a multiple of 32,
    and the same check on the one-thread-per-env FP32 kernel (QB_ADJOINT_FUSED=1):
    both within 1e-4 norm-wise per env, and within 2e-5 of each other."""
    n, T = 777, 16
    rng = np.random.default_rng(5)
    x0 = np.zeros((n, 17))
    x0[:, 0:3] = rng.uniform(-1, 1, (n, 3))
    x0[:, 3:6] = rng.normal(scale=0.5, size=(n, 3))
    q = rng.normal(size=(n, 4)) * 0.1 + [1, 0, 0, 0]
    x0[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    x0[:, 10:13] = rng.normal(scale=0.5, size=(n, 3))
    x0[:, 13:17] = rng.uniform(800, 1000, (n, 4))
    if kind == "rotor":
        acts = rng.uniform(700, 1100, (T, n, 4))
    elif kind == "ctbr":  # mild rate commands: the mixer stays out of its torque-scale branch (below)
        acts = np.concatenate([rng.uniform(9, 11, (T, n, 1)), rng.normal(scale=0.1, size=(T, n, 3))], 2)
    else:
        acts = rng.uniform(1.0, 3.0, (T, n, 4))
    x0 = x0.astype(np.float32).astype(np.float64)
    acts = acts.astype(np.float32).astype(np.float64)
    w = rng.normal(size=(T + 1, 17, n)) * np.concatenate([np.ones(13), np.full(4, 1e-3)])[None, :, None]
    P = native_params()

    # one FP32 forward tape; the adjoints of that same tape in FP32 and in exact double
    init = torch.as_tensor(x0.T.copy(), dtype=torch.float32, device="cuda")
    a32 = torch.as_tensor(acts, dtype=torch.float32, device="cuda")
    tape32, _ = G.rollout_planes(P, kind, init, a32)

    def run(dtype):
        ga, gi, _ = G.backward_planes(P, kind, tape32.to(dtype), a32.to(dtype), torch.as_tensor(w, dtype=dtype, device="cuda"))
        return ga.double().cpu().numpy(), gi.double().cpu().numpy()

    ref_a, ref_i = run(torch.float64)
    split_a, split_i = run(torch.float32)
    monkeypatch.setenv("QB_ADJOINT_FUSED", "1")
    fused_a, fused_i = run(torch.float32)

    def err(x, r):  # per env, norm-wise
        return np.abs(x - r).max(axis=(0, 2)) / np.abs(r).max(axis=(0, 2))

    e_split, e_fused, e_sf = err(split_a, ref_a), err(fused_a, ref_a), err(split_a, fused_a)
    ei_split = np.abs(split_i - ref_i).max(axis=0) / np.abs(ref_i).max(axis=0)
    print(kind, "split max/p99", e_split.max(), np.percentile(e_split, 99), "init", ei_split.max(), "fused max/p99",
          e_fused.max(), np.percentile(e_fused, 99), "envs over 1e-4 split/fused", (e_split > 1e-4).sum(),
          (e_fused > 1e-4).sum())
    # (with saturating CTBR commands -- rates N(0, 1) rad/s -- the mixer's torque-scale branch,
    # scale = (bound - base_j) / tp_j (control.py:114-128), divides by tp_j: both FP32 kernels then differ
    # from the exact-double adjoint by up to 5e-3 on ~10% of envs, identically; the controller adjoint is
    # beyond the reference and FD-pinned in exact double by test_ctbr_adjoint_finite_differences)
    assert e_split.max() < 1e-4 and ei_split.max() < 1e-4 and e_fused.max() < 1e-4
    assert e_sf.max() < 2e-5
