// qb_adjoint.cuh -- K1 adjoint: matrix-free vector-Jacobian products of one
// control step, the BPTT factor of gradients.rollout_grad.
//
// The reference builds dense 17x17 / 17x4 Jacobians per substep
// (gradients.py:52-197: _dynamics_jacobian, the RK4 stage chain,
// _renorm_jacobian, clip masks) and multiplies them; here each env's thread
// recomputes the substep stages from the saved pre-step state and pushes the
// 17-vector lambda backwards through them: J^T lambda and Ja^T lambda without
// ever forming J.  Same derivative conventions as the reference:
//   clamps (commands, lag)     derivative 1 strictly inside AND on the bound,
//                              0 outside, boundary flagged (gradients.py:136-142)
//   renormalisation            exact projection (I - u u^T)/|q| (:130-133)
//   rotor lag memory           rotor speeds are state (17-dim chain, :161-186)
// plus, beyond the reference, the CTBR / SRT controller (control.py:101-158)
// so CTBR and SRT actions are differentiable too (pinned by finite differences).
#pragma once
#include "qb_dynamics.cuh"

#ifdef __CUDACC__

template <class R> QB_D R clip_mask(R v, R lo, R hi, bool &flag) {
    if (v == lo || v == hi) {
        flag = true;
        return R(1.0);
    }
    return (v > lo && v < hi) ? R(1.0) : R(0.0);
}

// VJP of the rotation polynomial out = M(q) v (SGN=+1) or M(q)^T v (SGN=-1)
// (quatmath.py:39-72): adds dL/dq to qb and dL/dv to vb for cotangent a.
template <class R, int SGN>
QB_D void q_rot_vjp(const R *q, R vx, R vy, R vz, R ax, R ay, R az, R *qb, R &vbx, R &vby, R &vbz) {
    R w = q[0];
    R ux = SGN > 0 ? q[1] : -q[1], uy = SGN > 0 ? q[2] : -q[2], uz = SGN > 0 ? q[3] : -q[3];
    // dL/dv = M^T a  (M^T for the polynomial with u, M for -u)
    R bx, by, bz;
    q_rot<R, -SGN>(q, ax, ay, az, bx, by, bz);
    vbx = vbx + bx;
    vby = vby + by;
    vbz = vbz + bz;
    // t = u x v ; a . (2 w t) -> dw = 2 a.(u x v), du = 2 w (v x a)
    R tx = uy * vz - uz * vy, ty = uz * vx - ux * vz, tz = ux * vy - uy * vx;
    qb[0] = qb[0] + R(2.0) * (ax * tx + ay * ty + az * tz);
    R vxa_x = vy * az - vz * ay, vxa_y = vz * ax - vx * az, vxa_z = vx * ay - vy * ax;
    // a . 2 u x (u x v): du = 2[(u.v) a + (u.a) v - 2 (v.a) u]
    R uv = ux * vx + uy * vy + uz * vz, ua = ux * ax + uy * ay + uz * az, va = vx * ax + vy * ay + vz * az;
    R gx = R(2.0) * (w * vxa_x + uv * ax + ua * vx - R(2.0) * va * ux);
    R gy = R(2.0) * (w * vxa_y + uv * ay + ua * vy - R(2.0) * va * uy);
    R gz = R(2.0) * (w * vxa_z + uv * az + ua * vz - R(2.0) * va * uz);
    if (SGN > 0) {
        qb[1] = qb[1] + gx; qb[2] = qb[2] + gy; qb[3] = qb[3] + gz;
    } else {  // the polynomial used -u
        qb[1] = qb[1] - gx; qb[2] = qb[2] - gy; qb[3] = qb[3] - gz;
    }
}

// VJP of ode_rhs (dynamics.py:154-200) at rigid state y with wrench W(w):
// given a = dL/d(dy) (13), adds dL/dy to yb (13) and dL/dthrust to fb (4).
template <class R>
QB_D void ode_rhs_vjp(const DynConsts<R> &C, const R *y, const Wrench<R> &W, const R *a, R *yb, R *fb) {
    const R *v = y + 3, *q = y + 6, *o = y + 10;
    // forward pieces
    R bx, by, bz;
    q_rot<R, -1>(q, v[0], v[1], v[2], bx, by, bz);
    R Fx = C.neg_drag[0] * bx * r_abs(bx);
    R Fy = C.neg_drag[1] * by * r_abs(by);
    R Fz = C.neg_drag[2] * bz * r_abs(bz) + W.fsum;
    // dp = v
    yb[3] = yb[3] + a[0];
    yb[4] = yb[4] + a[1];
    yb[5] = yb[5] + a[2];
    // dv = R(q) F / m + g
    R ax = a[3] * C.inv_mass, ay = a[4] * C.inv_mass, az = a[5] * C.inv_mass;
    R Fbx = R(0.0), Fby = R(0.0), Fbz = R(0.0);
    q_rot_vjp<R, 1>(q, Fx, Fy, Fz, ax, ay, az, yb + 6, Fbx, Fby, Fbz);
    fb[0] = fb[0] + Fbz; fb[1] = fb[1] + Fbz; fb[2] = fb[2] + Fbz; fb[3] = fb[3] + Fbz;
    // drag: F_k = -c_k vb_k |vb_k|  ->  dF/dvb = -2 c_k |vb_k|
    R gbx = Fbx * R(2.0) * C.neg_drag[0] * r_abs(bx);
    R gby = Fby * R(2.0) * C.neg_drag[1] * r_abs(by);
    R gbz = Fbz * R(2.0) * C.neg_drag[2] * r_abs(bz);
    q_rot_vjp<R, -1>(q, v[0], v[1], v[2], gbx, gby, gbz, yb + 6, yb[3], yb[4], yb[5]);
    // dq = 0.5 q (x) (0, omega)
    R qw = q[0], qx = q[1], qy = q[2], qz = q[3], ox = o[0], oy = o[1], oz = o[2];
    R a0 = R(0.5) * a[6], a1 = R(0.5) * a[7], a2 = R(0.5) * a[8], a3 = R(0.5) * a[9];
    yb[6] = yb[6] + (a1 * ox + a2 * oy + a3 * oz);
    yb[7] = yb[7] + (-a0 * ox - a2 * oz + a3 * oy);
    yb[8] = yb[8] + (-a0 * oy + a1 * oz - a3 * ox);
    yb[9] = yb[9] + (-a0 * oz - a1 * oy + a2 * ox);
    yb[10] = yb[10] + (-a0 * qx + a1 * qw + a2 * qz - a3 * qy);
    yb[11] = yb[11] + (-a0 * qy - a1 * qz + a2 * qw + a3 * qx);
    yb[12] = yb[12] + (-a0 * qz + a1 * qy - a2 * qx + a3 * qw);
    // domega = (tau - omega x J omega) / J
    R b0 = a[10] * C.invJ[0], b1 = a[11] * C.invJ[1], b2 = a[12] * C.invJ[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) fb[i] = fb[i] + C.arms[i][0] * b0 + C.arms[i][1] * b1 + C.arms[i][2] * b2;
    R jxz = C.J[0] - C.J[2], jyx = C.J[1] - C.J[0], jzy = C.J[2] - C.J[1];
    yb[10] = yb[10] - (b1 * jxz * oz + b2 * jyx * oy);
    yb[11] = yb[11] - (b0 * jzy * oz + b2 * jyx * ox);
    yb[12] = yb[12] - (b0 * jzy * oy + b1 * jxz * ox);
}

// RK4 (or Euler) stage states of one substep from its input y and wrench:
// y2, y3, y4 (RK4 stage arguments) and the raw (unnormalised) result
template <class R>
QB_D void substep_stages(const DynConsts<R> &C, const R *y, const Wrench<R> &Wr, R *y2, R *y3, R *y4, R *yraw) {
    R k[13];
    if (C.integrator == QB_RK4) {
        ode_rhs(C, y, Wr, k);
        R acc[13];
#pragma unroll
        for (int i = 0; i < 13; ++i) {
            acc[i] = k[i];
            y2[i] = y[i] + C.half_h * k[i];
        }
        ode_rhs(C, y2, Wr, k);
#pragma unroll
        for (int i = 0; i < 13; ++i) {
            acc[i] = acc[i] + R(2.0) * k[i];
            y3[i] = y[i] + C.half_h * k[i];
        }
        ode_rhs(C, y3, Wr, k);
#pragma unroll
        for (int i = 0; i < 13; ++i) {
            acc[i] = acc[i] + R(2.0) * k[i];
            y4[i] = y[i] + C.h * k[i];
        }
        ode_rhs(C, y4, Wr, k);
#pragma unroll
        for (int i = 0; i < 13; ++i) yraw[i] = y[i] + C.sixth_h * (acc[i] + k[i]);
    } else {
        ode_rhs(C, y, Wr, k);
#pragma unroll
        for (int i = 0; i < 13; ++i) yraw[i] = y[i] + C.h * k[i];
    }
}

// Stage cache: with SUB == 2 and a cache (per-thread column of 52 values
// with stride `cs`, in shared memory), the first substep's stages computed
// by the forward pass are kept instead of being recomputed in the reverse
// sweep (20 -> 16 RHS-level evaluations per control step).
template <class R> struct StageCache {
    R *p;
    int stride;
    QB_D R &at(int k) const { return p[k * stride]; }
};

// One control step: forward recomputation + reverse sweep.
// x: pre-step 17-state, cmd: desired rotor speeds (already from the
// controller), lam: dL/dnext (17, in-out -> dL/dx), cmd_bar: dL/dcmd (4,
// accumulated), boundary: clip-boundary flag.  Substep intermediates are
// recomputed per substep from the saved substep inputs (<= 8 substeps).
// SUB > 0: substep count known at compile time (== C.substeps): the substep
// inputs stay in registers instead of a local-memory array.
template <class R, int SUB = 0>
QB_D void dyn_step_vjp(const DynConsts<R> &C, const R *x_in, const R *cmd_in, R *lam, R *cmd_bar, bool &boundary,
                       StageCache<R> cache = StageCache<R>{nullptr, 0}) {
    constexpr int MAXS = SUB > 0 ? SUB : 8;
    R cmd[4], cmask[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        cmask[i] = clip_mask(cmd_in[i], C.rlo, C.rhi, boundary);
        cmd[i] = p_clip(cmd_in[i], C.rlo, C.rhi);
    }
    const int S = SUB > 0 ? SUB : (C.substeps < MAXS ? C.substeps : MAXS);
    const bool cached = SUB == 2 && cache.p != nullptr;
    // forward: keep each substep's input state (13 rigid + 4 rotors); the
    // last substep's output is not needed by the reverse sweep
    R xs[MAXS][17];
#pragma unroll
    for (int k = 0; k < 17; ++k) xs[0][k] = x_in[k];
#pragma unroll
    for (int s = 0; s + 1 < S; ++s) {
        R x[17];
#pragma unroll
        for (int k = 0; k < 17; ++k) x[k] = xs[s][k];
        R w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = p_clip(cmd[i] + (x[13 + i] - cmd[i]) * C.alpha, C.rlo, C.rhi);
        Wrench<R> Wr;
        make_wrench(C, w, Wr);
        if (cached && s == 0) {
            R y2[13], y3[13], y4[13], yraw[13];
            substep_stages(C, x, Wr, y2, y3, y4, yraw);
#pragma unroll
            for (int i = 0; i < 13; ++i) {
                cache.at(i) = y2[i];
                cache.at(13 + i) = y3[i];
                cache.at(26 + i) = y4[i];
                cache.at(39 + i) = yraw[i];
                x[i] = yraw[i];
            }
        } else {
            integrate_substep(C, x, Wr);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) x[13 + i] = w[i];
        q_normalize(x + 6);
#pragma unroll
        for (int k = 0; k < 17; ++k) xs[s + 1][k] = x[k];
    }
    R cb[4] = {R(0.0), R(0.0), R(0.0), R(0.0)};
#pragma unroll
    for (int s = S - 1; s >= 0; --s) {
        const R *x0 = xs[s];
        R raw[4], lm[4], w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            raw[i] = cmd[i] + (x0[13 + i] - cmd[i]) * C.alpha;
            lm[i] = clip_mask(raw[i], C.rlo, C.rhi, boundary);
            w[i] = p_clip(raw[i], C.rlo, C.rhi);
        }
        Wrench<R> Wr;
        make_wrench(C, w, Wr);
        // the stages of this substep (recomputed, or from the forward pass)
        R y[13], y2[13], y3[13], y4[13], yraw[13];
#pragma unroll
        for (int i = 0; i < 13; ++i) y[i] = x0[i];
        const bool rk4 = C.integrator == QB_RK4;
        if (cached && s == 0) {
#pragma unroll
            for (int i = 0; i < 13; ++i) {
                y2[i] = cache.at(i);
                y3[i] = cache.at(13 + i);
                y4[i] = cache.at(26 + i);
                yraw[i] = cache.at(39 + i);
            }
        } else {
            substep_stages(C, y, Wr, y2, y3, y4, yraw);
        }
        // renormalisation: q = q_raw / |q_raw|
        R yb_out[13];
#pragma unroll
        for (int i = 0; i < 13; ++i) yb_out[i] = lam[i];
        {
            const R *qr = yraw + 6;
            R n2 = qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3];
            R n = r_sqrt(n2);
            R u0 = qr[0] / n, u1 = qr[1] / n, u2 = qr[2] / n, u3 = qr[3] / n;
            R ul = u0 * lam[6] + u1 * lam[7] + u2 * lam[8] + u3 * lam[9];
            yb_out[6] = (lam[6] - u0 * ul) / n;
            yb_out[7] = (lam[7] - u1 * ul) / n;
            yb_out[8] = (lam[8] - u2 * ul) / n;
            yb_out[9] = (lam[9] - u3 * ul) / n;
        }
        // integrator VJP -> dL/dy (13), dL/dthrust (4)
        R yb[13], fb[4] = {R(0.0), R(0.0), R(0.0), R(0.0)};
#pragma unroll
        for (int i = 0; i < 13; ++i) yb[i] = yb_out[i];
        if (rk4) {
            R kb[13], sb[13];
#pragma unroll
            for (int i = 0; i < 13; ++i) kb[i] = C.sixth_h * yb_out[i];  // k4 cotangent
            // k4 = f(y4), y4 = y + h k3
#pragma unroll
            for (int i = 0; i < 13; ++i) sb[i] = R(0.0);
            ode_rhs_vjp(C, y4, Wr, kb, sb, fb);
#pragma unroll
            for (int i = 0; i < 13; ++i) {
                yb[i] = yb[i] + sb[i];
                kb[i] = R(2.0) * C.sixth_h * yb_out[i] + C.h * sb[i];  // k3 cotangent
                sb[i] = R(0.0);
            }
            ode_rhs_vjp(C, y3, Wr, kb, sb, fb);
#pragma unroll
            for (int i = 0; i < 13; ++i) {
                yb[i] = yb[i] + sb[i];
                kb[i] = R(2.0) * C.sixth_h * yb_out[i] + C.half_h * sb[i];  // k2 cotangent
                sb[i] = R(0.0);
            }
            ode_rhs_vjp(C, y2, Wr, kb, sb, fb);
#pragma unroll
            for (int i = 0; i < 13; ++i) {
                yb[i] = yb[i] + sb[i];
                kb[i] = C.sixth_h * yb_out[i] + C.half_h * sb[i];  // k1 cotangent
                sb[i] = R(0.0);
            }
            ode_rhs_vjp(C, y, Wr, kb, sb, fb);
#pragma unroll
            for (int i = 0; i < 13; ++i) yb[i] = yb[i] + sb[i];
        } else {
            R kb[13];
#pragma unroll
            for (int i = 0; i < 13; ++i) kb[i] = C.h * yb_out[i];
            ode_rhs_vjp(C, y, Wr, kb, yb, fb);
        }
        // thrust -> rotor speed of this substep; the post-substep rotor state is w itself
        R wb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            wb[i] = fb[i] * (R(2.0) * C.k2 * w[i] + C.k1) + lam[13 + i];
            R rb = lm[i] * wb[i];              // through clip(raw)
            lam[13 + i] = C.alpha * rb;        // d raw / d omega_prev
            cb[i] = cb[i] + (R(1.0) - C.alpha) * rb;  // d raw / d cmd
        }
#pragma unroll
        for (int i = 0; i < 13; ++i) lam[i] = yb[i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) cmd_bar[i] = cmd_bar[i] + cmask[i] * cb[i];
}

// ---- controller VJPs (beyond the reference, FD-pinned) ---------------------

// params.py:106-111 speed_of_thrust: d omega / d f (0 where clamped / at arg<=0)
template <class R> QB_D R speed_of_thrust_grad(const DynConsts<R> &C, R f) {
    R arg = C.k1sq + C.four_k2 * (f - C.k0);
    if (!(arg > R(0.0))) return R(0.0);
    R sq = r_sqrt(arg);
    R om = (C.neg_k1 + sq) * C.inv_two_k2;
    bool flag = false;
    R m = clip_mask(om, C.rlo, C.rhi, flag);
    return m / sq;  // d/df [(-k1 + sqrt(k1^2 + 4k2(f-k0))) / 2k2] = 1/sqrt(arg)
}

// control.py:138-158 + mixer :101-130.  speeds_bar: dL/d(rotor speed cmd);
// writes dL/d(collective, rates) to ab and adds dL/d omega to xb[10..12].
template <class R>
QB_D void ctbr_vjp(const DynConsts<R> &C, const R *x, R coll_in, R r0, R r1, R r2, const R *speeds_bar, R *ab, R *xb) {
    const R *om = x + 10;
    const bool coll_pos = coll_in > R(0.0);
    const R coll = p_max(coll_in, R(0.0));
    R err0 = r0 - om[0], err1 = r1 - om[1], err2 = r2 - om[2];
    R jo0 = C.J[0] * om[0], jo1 = C.J[1] * om[1], jo2 = C.J[2] * om[2];
    R tq[3] = {C.J[0] * (C.rate_p[0] * err0) + (om[1] * jo2 - om[2] * jo1),
               C.J[1] * (C.rate_p[1] * err1) + (om[2] * jo0 - om[0] * jo2),
               C.J[2] * (C.rate_p[2] * err2) + (om[0] * jo1 - om[1] * jo0)};
    // mixer forward
    R force = C.mass * coll;
    R fcl = p_clip(force, C.flo4, C.fhi4);
    bool fb_flag = false;
    R fmask = clip_mask(force, C.flo4, C.fhi4, fb_flag);
    R base[4], tp[4];
    R best = R(infinity_d());
    int arg = -1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        base[i] = C.minv[i][0] * fcl;
        tp[i] = C.minv[i][1] * tq[0] + C.minv[i][2] * tq[1] + C.minv[i][3] * tq[2];
        R up = tp[i] > R(0.0) ? (C.fhi - base[i]) / tp[i] : R(infinity_d());
        R dn = tp[i] < R(0.0) ? (C.flo - base[i]) / tp[i] : R(infinity_d());
        R b = up < dn ? up : dn;
        if (b < best) {
            best = b;
            arg = i;
        }
    }
    R scale = p_max(p_min(best, R(1.0)), R(0.0));
    const bool scale_active = best < R(1.0) && best > R(0.0) && arg >= 0;
    // backward
    R baseb[4], tpb[4], sb = R(0.0);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        R thr = base[i] + scale * tp[i];
        bool fl = false;
        R cm = clip_mask(thr, C.flo, C.fhi, fl);
        R thr_clamped = p_clip(thr, C.flo, C.fhi);
        R g = speeds_bar[i] * speed_of_thrust_grad(C, thr_clamped) * cm;
        baseb[i] = g;
        tpb[i] = scale * g;
        sb = sb + tp[i] * g;
    }
    if (scale_active) {  // scale = (bound - base_j) / tp_j for the limiting rotor j
        baseb[arg] = baseb[arg] - sb / tp[arg];
        tpb[arg] = tpb[arg] - sb * scale / tp[arg];
    }
    R fclb = R(0.0), tqb[3] = {R(0.0), R(0.0), R(0.0)};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        fclb = fclb + C.minv[i][0] * baseb[i];
        tqb[0] = tqb[0] + C.minv[i][1] * tpb[i];
        tqb[1] = tqb[1] + C.minv[i][2] * tpb[i];
        tqb[2] = tqb[2] + C.minv[i][3] * tpb[i];
    }
    ab[0] = coll_pos ? C.mass * fmask * fclb : R(0.0);
    R kr0 = C.J[0] * C.rate_p[0] * tqb[0], kr1 = C.J[1] * C.rate_p[1] * tqb[1], kr2 = C.J[2] * C.rate_p[2] * tqb[2];
    ab[1] = kr0;
    ab[2] = kr1;
    ab[3] = kr2;
    // d tau / d omega: -J k_p (rate loop) + d(omega x J omega)/d omega
    R jxz = C.J[0] - C.J[2], jyx = C.J[1] - C.J[0], jzy = C.J[2] - C.J[1];
    xb[10] = xb[10] - kr0 + (tqb[1] * jxz * om[2] + tqb[2] * jyx * om[1]);
    xb[11] = xb[11] - kr1 + (tqb[0] * jzy * om[2] + tqb[2] * jyx * om[0]);
    xb[12] = xb[12] - kr2 + (tqb[0] * jzy * om[1] + tqb[1] * jxz * om[0]);
}

#endif  // __CUDACC__
