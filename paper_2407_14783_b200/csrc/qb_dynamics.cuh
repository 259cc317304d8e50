// qb_dynamics.cuh -- K1 device math: controller -> mixer -> rotor lag ->
// Euler/RK4 rigid body -> renormalisation (forward), templated on the scalar
// policy (qb_real.cuh).  One env per thread, everything in registers.
//
// Reference map (all under /root/reference/pkg/src/quadsim):
//   rotate / rotate_inv / to_matrix / normalize  quatmath.py:18-81
//   thrusts, drag, wrench, rigid derivative      dynamics.py:103-200
//   integrate_substep, step                      dynamics.py:203-253
//   speed_of_thrust                              params.py:106-111
//   mixer, ctbr/lv/ps controllers                control.py:101-252
#pragma once
#include "../../include/qb_params.h"
#include "qb_real.cuh"

template <class R> struct DynConsts {
    R mass, inv_mass;
    R J[3], invJ[3];
    R g[3];
    R arms[4][3];
    R k2, k1, k0, k1sq, four_k2, two_k2, inv_two_k2, neg_k1;
    R neg_drag[3];  // -0.5*rho*Cd*s
    R ndm[3];       // neg_drag / mass                 (FP32 RHS folding)
    R cJ[3];        // (J[a+2] - J[a+1]) / J[a]: (w x Jw)_a / J_a = cJ[a] w_{a+1} w_{a+2}
    R rlo, rhi;
    R minv[4][4];
    R flo, fhi, flo4, fhi4;
    R h, half_h, sixth_h, alpha;
    R rate_p[3], neg_att_p[3], vel_p[3], pos_p[3], pos_d[3];
    R max_speed, max_tilt;
    R hover_speed;
    int substeps, integrator;
};

// host: fold qb_params into the policy's constants (exact same doubles; the
// float policy rounds them once)
template <class R> inline DynConsts<R> make_consts(const qb_params &p) {
    DynConsts<R> c;
    auto F = [](double x) { return from_dbl<R>(x); };
    c.mass = F(p.mass);
    c.inv_mass = F(1.0 / p.mass);
    for (int a = 0; a < 3; ++a) {
        c.J[a] = F(p.inertia[a]);
        c.invJ[a] = F(1.0 / p.inertia[a]);
        c.g[a] = F(p.gravity[a]);
        c.neg_drag[a] = F(-p.drag_c[a]);
        c.ndm[a] = F(-p.drag_c[a] / p.mass);
        c.cJ[a] = F((p.inertia[(a + 2) % 3] - p.inertia[(a + 1) % 3]) / p.inertia[a]);
        c.rate_p[a] = F(p.rate_p[a]);
        c.neg_att_p[a] = F(-p.attitude_p[a]);
        c.vel_p[a] = F(p.vel_p[a]);
        c.pos_p[a] = F(p.pos_p[a]);
        c.pos_d[a] = F(p.pos_d[a]);
    }
    for (int i = 0; i < 4; ++i) {
        for (int a = 0; a < 3; ++a) c.arms[i][a] = F(p.torque_arms[i][a]);
        for (int k = 0; k < 4; ++k) c.minv[i][k] = F(p.alloc_inv[i][k]);
    }
    double k2 = p.thrust_coeffs[0], k1 = p.thrust_coeffs[1], k0 = p.thrust_coeffs[2];
    c.k2 = F(k2); c.k1 = F(k1); c.k0 = F(k0);
    c.k1sq = F(k1 * k1);
    c.four_k2 = F(4.0 * k2);
    c.two_k2 = F(2.0 * k2);
    c.inv_two_k2 = F(1.0 / (2.0 * k2));
    c.neg_k1 = F(-k1);
    c.rlo = F(p.rotor_lo); c.rhi = F(p.rotor_hi);
    c.flo = F(p.thrust_lo); c.fhi = F(p.thrust_hi);
    c.flo4 = F(4.0 * p.thrust_lo); c.fhi4 = F(4.0 * p.thrust_hi);
    c.h = F(p.physics_dt); c.half_h = F(p.half_dt); c.sixth_h = F(p.sixth_dt);
    c.alpha = F(p.lag_alpha);
    c.max_speed = F(p.max_speed); c.max_tilt = F(p.max_tilt_accel);
    c.hover_speed = F(p.hover_speed);
    c.substeps = p.substeps;
    c.integrator = p.integrator;
    return c;
}

#ifdef __CUDACC__

// ---------------------------------------------------------------- quaternions
// quatmath.py:39-55: v + 2 (w (u x v) + u x (u x v)); sgn=-1 gives R(q)^T v
template <class R, int SGN>
QB_D void q_rot(const R *q, R vx, R vy, R vz, R &ox, R &oy, R &oz) {
    R w = q[0];
    R ux = SGN > 0 ? q[1] : -q[1], uy = SGN > 0 ? q[2] : -q[2], uz = SGN > 0 ? q[3] : -q[3];
    R tx = uy * vz - uz * vy;
    R ty = uz * vx - ux * vz;
    R tz = ux * vy - uy * vx;
    R sx = uy * tz - uz * ty;
    R sy = uz * tx - ux * tz;
    R sz = ux * ty - uy * tx;
    ox = vx + R(2.0) * (w * tx + sx);
    oy = vy + R(2.0) * (w * ty + sy);
    oz = vz + R(2.0) * (w * tz + sz);
}

// quatmath.py:75-81
template <class R> QB_D void q_matrix(const R *q, R m[3][3]) {
    R w = q[0], x = q[1], y = q[2], z = q[3];
    if constexpr (!is_exact<R>::value) {  // FP32: pre-doubled products, 24 ops
        const R x2 = x + x, y2 = y + y, z2 = z + z;
        const R xx = x * x2, yy = y * y2, zz = z * z2, xy = x * y2, xz = x * z2, yz = y * z2;
        const R wx = w * x2, wy = w * y2, wz = w * z2;
        m[0][0] = R(1.0) - (yy + zz); m[0][1] = xy - wz; m[0][2] = xz + wy;
        m[1][0] = xy + wz; m[1][1] = R(1.0) - (xx + zz); m[1][2] = yz - wx;
        m[2][0] = xz - wy; m[2][1] = yz + wx; m[2][2] = R(1.0) - (xx + yy);
        return;
    }
    m[0][0] = R(1.0) - R(2.0) * (y * y + z * z);
    m[0][1] = R(2.0) * (x * y - w * z);
    m[0][2] = R(2.0) * (x * z + w * y);
    m[1][0] = R(2.0) * (x * y + w * z);
    m[1][1] = R(1.0) - R(2.0) * (x * x + z * z);
    m[1][2] = R(2.0) * (y * z - w * x);
    m[2][0] = R(2.0) * (x * z - w * y);
    m[2][1] = R(2.0) * (y * z + w * x);
    m[2][2] = R(1.0) - R(2.0) * (x * x + y * y);
}

// quatmath.py:18-21
template <class R> QB_D void q_normalize(R *q) {
    R n2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    if constexpr (is_exact<R>::value) {
        R n = r_sqrt(n2);
        q[0] = q[0] / n; q[1] = q[1] / n; q[2] = q[2] / n; q[3] = q[3] / n;
    } else {
        R inv = rsqrtf(n2);
        q[0] *= inv; q[1] *= inv; q[2] *= inv; q[3] *= inv;
    }
}

// ---------------------------------------------------------------- dynamics
// Per-substep constants of the wrench: thrusts and torques depend only on the
// (held) rotor speeds (dynamics.py:203-207), so they are evaluated once per
// substep instead of once per RK4 stage -- same values, 4x fewer ops.
template <class R> struct Wrench {
    R f[4];
    R fsum;
    R tq[3];
    R fsum_m, tqJ[3];  // FP32 path: fsum / mass, tq / J
};

template <class R> QB_D void make_wrench(const DynConsts<R> &C, const R *w, Wrench<R> &W) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // dynamics.py:103-106
        if constexpr (is_exact<R>::value)
            W.f[i] = C.k2 * (w[i] * w[i]) + C.k1 * w[i] + C.k0;
        else  // Horner: two FMAs
            W.f[i] = (C.k2 * w[i] + C.k1) * w[i] + C.k0;
    }
    W.fsum = W.f[0] + W.f[1] + W.f[2] + W.f[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)  // dynamics.py:192-194
        W.tq[a] = W.f[0] * C.arms[0][a] + W.f[1] * C.arms[1][a] + W.f[2] * C.arms[2][a] + W.f[3] * C.arms[3][a];
    if constexpr (!is_exact<R>::value) {
        W.fsum_m = W.fsum * C.inv_mass;
#pragma unroll
        for (int a = 0; a < 3; ++a) W.tqJ[a] = W.tq[a] * C.invJ[a];
    }
}

// dynamics.py:154-200: 13 rigid rates at y = (p, v, q, omega)
template <class R> QB_D void ode_rhs(const DynConsts<R> &C, const R *y, const Wrench<R> &W, R *dy) {
    const R *v = y + 3, *q = y + 6, *o = y + 10;
    R bx, by, bz, fx, fy, fz, ax, ay, az;
    if constexpr (is_exact<R>::value) {  // reference operation order (quatmath.rotate / rotate_inv)
        q_rot<R, -1>(q, v[0], v[1], v[2], bx, by, bz);  // v_B = R^T v
        fx = C.neg_drag[0] * bx * r_abs(bx);            // dynamics.py:117-120
        fy = C.neg_drag[1] * by * r_abs(by);
        fz = C.neg_drag[2] * bz * r_abs(bz);
        fz = fz + W.f[0] + W.f[1] + W.f[2] + W.f[3];    // dynamics.py:190 evaluation order
        q_rot<R, 1>(q, fx, fy, fz, ax, ay, az);
    } else {  // same polynomial R(q) (== to_matrix, also for |q| != 1), built once per stage
        R m[3][3];
        q_matrix(q, m);
        bx = m[0][0] * v[0] + m[1][0] * v[1] + m[2][0] * v[2];
        by = m[0][1] * v[0] + m[1][1] * v[1] + m[2][1] * v[2];
        bz = m[0][2] * v[0] + m[1][2] * v[1] + m[2][2] * v[2];
        // body force / mass (drag coefficients and thrust pre-divided by m)
        fx = C.ndm[0] * bx * r_abs(bx);
        fy = C.ndm[1] * by * r_abs(by);
        fz = C.ndm[2] * bz * r_abs(bz) + W.fsum_m;
        ax = C.g[0] + m[0][0] * fx + m[0][1] * fy + m[0][2] * fz;
        ay = C.g[1] + m[1][0] * fx + m[1][1] * fy + m[1][2] * fz;
        az = C.g[2] + m[2][0] * fx + m[2][1] * fy + m[2][2] * fz;
    }
    dy[0] = v[0]; dy[1] = v[1]; dy[2] = v[2];
    if constexpr (is_exact<R>::value) {
        dy[3] = ax / C.mass + C.g[0];
        dy[4] = ay / C.mass + C.g[1];
        dy[5] = az / C.mass + C.g[2];
    } else {
        dy[3] = ax;
        dy[4] = ay;
        dy[5] = az;
    }
    R qw = q[0], qx = q[1], qy = q[2], qz = q[3], ox = o[0], oy = o[1], oz = o[2];
    dy[6] = R(0.5) * (-qx * ox - qy * oy - qz * oz);
    dy[7] = R(0.5) * (qw * ox + qy * oz - qz * oy);
    dy[8] = R(0.5) * (qw * oy - qx * oz + qz * ox);
    dy[9] = R(0.5) * (qw * oz + qx * oy - qy * ox);
    if constexpr (is_exact<R>::value) {
        R cx = oy * (C.J[2] * oz) - oz * (C.J[1] * oy);
        R cy = oz * (C.J[0] * ox) - ox * (C.J[2] * oz);
        R cz = ox * (C.J[1] * oy) - oy * (C.J[0] * ox);
        dy[10] = (W.tq[0] - cx) / C.J[0];
        dy[11] = (W.tq[1] - cy) / C.J[1];
        dy[12] = (W.tq[2] - cz) / C.J[2];
    } else {  // diagonal J: (w x Jw)_x / Jx = (Jz - Jy)/Jx * wy wz, two ops per axis
        dy[10] = W.tqJ[0] - C.cJ[0] * (oy * oz);
        dy[11] = W.tqJ[1] - C.cJ[1] * (oz * ox);
        dy[12] = W.tqJ[2] - C.cJ[2] * (ox * oy);
    }
}

// dynamics.py:203-228: raw substep in place (no renormalisation)
// out = y + c * k over the 13 rigid states; FP32: packed FFMA2 on component
// pairs (same per-lane rounding as the scalar FFMA, half the instructions)
template <class R, class K> QB_D void axpy13(R *out, const R *y, K c, const R *k) {
#pragma unroll
    for (int i = 0; i < 13; ++i) out[i] = y[i] + c * k[i];
}
QB_D void axpy13(float *out, const float *y, float c, const float *k) {
#pragma unroll
    for (int i = 0; i < 12; i += 2) {
        const float2 r = __ffma2_rn(make_float2(k[i], k[i + 1]), make_float2(c, c), make_float2(y[i], y[i + 1]));
        out[i] = r.x;
        out[i + 1] = r.y;
    }
    out[12] = fmaf(c, k[12], y[12]);
}

// dynamics.py:203-228: raw substep in place (no renormalisation)
template <class R> QB_D void integrate_substep(const DynConsts<R> &C, R *y, const Wrench<R> &W) {
    if (C.integrator == QB_EULER) {
        R d[13];
        ode_rhs(C, y, W, d);
        axpy13(y, y, C.h, d);
        return;
    }
    R k[13], acc[13], t[13];
    ode_rhs(C, y, W, k);  // k1
#pragma unroll
    for (int i = 0; i < 13; ++i) acc[i] = k[i];
    axpy13(t, y, C.half_h, k);
    ode_rhs(C, t, W, k);  // k2
    axpy13(acc, acc, R(2.0), k);
    axpy13(t, y, C.half_h, k);
    ode_rhs(C, t, W, k);  // k3
    axpy13(acc, acc, R(2.0), k);
    axpy13(t, y, C.h, k);
    ode_rhs(C, t, W, k);  // k4
#pragma unroll
    for (int i = 0; i < 13; ++i) acc[i] = acc[i] + k[i];
    axpy13(y, y, C.sixth_h, acc);
}

// dynamics.py:231-253 for one env. x = 17-state, cmd = desired rotor speeds.
// Returns false when any component is non-finite (NonFiniteState mask).
// SUB > 0: substep count known at compile time (loop unrolled; must equal C.substeps)
template <class R, int SUB = 0> QB_D bool dyn_step(const DynConsts<R> &C, R *x, const R *cmd_in) {
    R cmd[4];
    bool cmd_ok = true;  // FP32 clamps drop NaN: keep the reference's verdict (NaN command -> non-finite state)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        cmd_ok &= !r_isnan(cmd_in[i]);
        cmd[i] = p_clip(cmd_in[i], C.rlo, C.rhi);
    }
    const int nsub = SUB > 0 ? SUB : C.substeps;
#pragma unroll
    for (int s = 0; s < nsub; ++s) {
        R w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = p_clip(cmd[i] + (x[13 + i] - cmd[i]) * C.alpha, C.rlo, C.rhi);  // :109-114
        Wrench<R> W;
        make_wrench(C, w, W);
        integrate_substep(C, x, W);
#pragma unroll
        for (int i = 0; i < 4; ++i) x[13 + i] = w[i];
        q_normalize(x + 6);
    }
    bool ok = cmd_ok;
#pragma unroll
    for (int i = 0; i < 17; ++i) ok &= r_isfinite(x[i]);
    return ok;
}

// ---------------------------------------------------------------- controller
// params.py:106-111
template <class R> QB_D R speed_of_thrust(const DynConsts<R> &C, R f) {
    R arg = p_max(C.k1sq + C.four_k2 * (f - C.k0), R(0.0));
    R om;
    if constexpr (is_exact<R>::value)
        om = (C.neg_k1 + r_sqrt(arg)) / C.two_k2;
    else
        om = (C.neg_k1 + r_sqrt(arg)) * C.inv_two_k2;
    return p_clip(om, C.rlo, C.rhi);
}

// control.py:101-130
// saturated (optional): scale < 1 or the collective was clamped (control.py:130)
template <class R> QB_D void mixer(const DynConsts<R> &C, R force, const R *tq, R *thr, bool *saturated = nullptr) {
    R fcl = p_clip(force, C.flo4, C.fhi4);
    R base[4], tp[4];
    R scale;
    if constexpr (is_exact<R>::value) {
        R up_min = R(infinity_d()), dn_min = R(infinity_d());
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            base[i] = C.minv[i][0] * fcl;
            tp[i] = C.minv[i][1] * tq[0] + C.minv[i][2] * tq[1] + C.minv[i][3] * tq[2];
            R up = tp[i] > R(0.0) ? (C.fhi - base[i]) / tp[i] : R(infinity_d());
            R dn = tp[i] < R(0.0) ? (C.flo - base[i]) / tp[i] : R(infinity_d());
            up_min = p_min(up_min, up);
            dn_min = p_min(dn_min, dn);
        }
        scale = p_max(p_min(p_min(up_min, dn_min), R(1.0)), R(0.0));
    } else {  // only one of up / dn is finite per rotor: one (fast) division each
        R bmin = R(infinity_d());
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            base[i] = C.minv[i][0] * fcl;
            tp[i] = C.minv[i][1] * tq[0] + C.minv[i][2] * tq[1] + C.minv[i][3] * tq[2];
            R lim = tp[i] > R(0.0) ? C.fhi : C.flo;
            R b = tp[i] != R(0.0) ? __fdividef(lim - base[i], tp[i]) : R(infinity_d());
            bmin = fminf(bmin, b);
        }
        scale = fmaxf(fminf(bmin, R(1.0)), R(0.0));
    }
    if (saturated) *saturated = scale < R(1.0) || force != fcl;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        R f = base[i] + scale * tp[i];
        if constexpr (!is_exact<R>::value) {
            // A rotor the torque scale saturates lands on its thrust bound up to
            // the rounding of base + s*tp (~1e-7 N in FP32), and the thrust-curve
            // inverse sqrt(f/k2) turns that into ~0.2 rad/s near f_lo = 0.  Snap
            // values within a few ulps of the operands onto the bound: exact in
            // real arithmetic, and what FP64 rounding gives the reference.
            R tol = R(4e-7) * (r_abs(base[i]) + r_abs(scale * tp[i]));
            if (r_abs(f - C.flo) <= tol) f = C.flo;
            if (r_abs(f - C.fhi) <= tol) f = C.fhi;
        }
        thr[i] = p_clip(f, C.flo, C.fhi);
    }
}

// control.py:138-158
template <class R> QB_D void ctbr_speeds(const DynConsts<R> &C, const R *x, R coll, R r0, R r1, R r2, R *out) {
    const R *om = x + 10;
    coll = p_max(coll, R(0.0));
    R err0 = r0 - om[0], err1 = r1 - om[1], err2 = r2 - om[2];
    R jo0 = C.J[0] * om[0], jo1 = C.J[1] * om[1], jo2 = C.J[2] * om[2];
    R tq[3];
    tq[0] = C.J[0] * (C.rate_p[0] * err0) + (om[1] * jo2 - om[2] * jo1);
    tq[1] = C.J[1] * (C.rate_p[1] * err1) + (om[2] * jo0 - om[0] * jo2);
    tq[2] = C.J[2] * (C.rate_p[2] * err2) + (om[0] * jo1 - om[1] * jo0);
    R thr[4];
    mixer(C, C.mass * coll, tq, thr);
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = speed_of_thrust(C, thr[i]);
}

// control.py:236-239
template <class R> QB_D void clip_norm(R *v, R cap) {
    R n = r_sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    R s = n > cap ? cap / (n == R(0.0) ? R(1.0) : n) : R(1.0);
    v[0] = v[0] * s; v[1] = v[1] * s; v[2] = v[2] * s;
}

// control.py:161-213 (cy, sy) = (cos yaw, sin yaw)
template <class R>
QB_D void accel_to_ctbr(const DynConsts<R> &C, const R *x, const R *a_des, R cy, R sy, R &coll, R *rates) {
    R spec[3] = {a_des[0] - C.g[0], a_des[1] - C.g[1], a_des[2] - C.g[2]};
    R norm = r_sqrt(spec[0] * spec[0] + spec[1] * spec[1] + spec[2] * spec[2]);
    bool degenerate = norm < R(1e-8);
    R safe = degenerate ? R(1.0) : norm;
    R z0 = spec[0] / safe, z1 = spec[1] / safe, z2 = spec[2] / safe;
    R yx = z1 * R(0.0) - z2 * sy;
    R yy = z2 * cy - z0 * R(0.0);
    R yz = z0 * sy - z1 * cy;
    R yn = r_sqrt(yx * yx + yy * yy + yz * yz);
    R ys = yn < R(1e-8) ? R(1.0) : yn;
    yx = yx / ys; yy = yy / ys; yz = yz / ys;
    R xx = yy * z2 - yz * z1;
    R xy = yz * z0 - yx * z2;
    R xz = yx * z1 - yy * z0;
    R rot[3][3];
    q_matrix(x + 6, rot);
    // m[a][b] = sum_k rdes[k][a] rot[k][b]; columns of rdes: x_des, y_des, z_des
    R c0[3] = {xx, xy, xz}, c1[3] = {yx, yy, yz}, c2[3] = {z0, z1, z2};
    const R *col[3] = {c0, c1, c2};
    auto m = [&](int a, int b) { return col[a][0] * rot[0][b] + col[a][1] * rot[1][b] + col[a][2] * rot[2][b]; };
    R e0 = R(0.5) * (m(2, 1) - m(1, 2));
    R e1 = R(0.5) * (m(0, 2) - m(2, 0));
    R e2 = R(0.5) * (m(1, 0) - m(0, 1));
    rates[0] = C.neg_att_p[0] * e0;
    rates[1] = C.neg_att_p[1] * e1;
    rates[2] = C.neg_att_p[2] * e2;
    R c = p_max(spec[0] * rot[0][2] + spec[1] * rot[1][2] + spec[2] * rot[2][2], R(0.0));
    if (degenerate) {
        rates[0] = rates[1] = rates[2] = R(0.0);
        c = R(0.0);
    }
    coll = c;
}

template <class R> QB_D void sincos_r(R yaw, R &c, R &s) {
    if constexpr (is_exact<R>::value) {
        c = r_cos(yaw);
        s = r_sin(yaw);
    } else {
        sincosf(yaw, &s, &c);
    }
}

// control.py:122-139: LV / PS command -> CTBR (collective, body rates)
template <class R, int KIND> QB_D void to_ctbr(const DynConsts<R> &C, const R *x, const R *cmd, R &coll, R *rates) {
    R v_des[3];
    if constexpr (KIND == QB_CMD_PS) {  // control.py:226-233
#pragma unroll
        for (int a = 0; a < 3; ++a) v_des[a] = C.pos_p[a] * (cmd[a] - x[a]) - C.pos_d[a] * x[3 + a];
        clip_norm(v_des, C.max_speed);
    } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) v_des[a] = cmd[a];
    }
    R a_des[3];  // control.py:216-223
#pragma unroll
    for (int a = 0; a < 3; ++a) a_des[a] = C.vel_p[a] * (v_des[a] - x[3 + a]);
    clip_norm(a_des, C.max_tilt);
    R cy, sy;
    sincos_r(cmd[3], cy, sy);
    accel_to_ctbr(C, x, a_des, cy, sy, coll, rates);
}

// control.py:242-252: command (as_array layout) -> desired rotor speeds
template <class R, int KIND> QB_D void command_to_speeds(const DynConsts<R> &C, const R *x, const R *cmd, R *out) {
    if constexpr (KIND == QB_CMD_ROTOR) {
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = cmd[i];
    } else if constexpr (KIND == QB_CMD_SRT) {  // control.py:133-135
#pragma unroll
        for (int i = 0; i < 4; ++i) out[i] = speed_of_thrust(C, p_clip(cmd[i], C.flo, C.fhi));
    } else if constexpr (KIND == QB_CMD_CTBR) {
        ctbr_speeds(C, x, cmd[0], cmd[1], cmd[2], cmd[3], out);
    } else {
        R coll, rates[3];
        to_ctbr<R, KIND>(C, x, cmd, coll, rates);
        ctbr_speeds(C, x, coll, rates[0], rates[1], rates[2], out);
    }
}

#endif  // __CUDACC__
