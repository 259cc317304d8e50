/*
 * qb_params.h -- plain-old-data constants of one vehicle + integrator +
 * controller, shared by the sm_100a library (libquadb200.so) and the CPU
 * oracle (oracle/quadsim_oracle.c).
 *
 * Every field is a value the reference derives from its frozen dataclasses;
 * the host packs it once (paper_2407_14783_b200/params.py:pack_params) with
 * the SAME numpy expressions the reference evaluates per call, so the device
 * sees bit-identical constants:
 *
 *   mass, inertia, gravity ........ QuadParams            params.py:49-60
 *   torque_arms[4][3] ............. QuadParams.torque_arms params.py:82-88
 *   thrust_coeffs (k2,k1,k0) ...... params.py:55
 *   drag_c = 0.5*rho*Cd*s ......... dynamics.py:119 (drag_force)
 *   rotor_lo/hi ................... params.py:60
 *   alloc_inv[4][4] ............... np.linalg.inv(allocation_matrix) params.py:98-100
 *   thrust_lo/hi .................. QuadParams.thrust_limits params.py:113-116
 *   hover_speed ................... params.py:122-124
 *   physics_dt, lag_alpha ......... SimConfig.physics_dt params.py:147-149,
 *                                   exp(-c*h) dynamics.py:111 (np.exp on host)
 *   gains ......................... ControllerGains params.py:152-178
 */
#ifndef QB_PARAMS_H
#define QB_PARAMS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum qb_integrator { QB_EULER = 0, QB_RK4 = 1 };

/* command kinds (control.py:330 COMMAND_TYPES) */
enum qb_cmd_kind { QB_CMD_SRT = 0, QB_CMD_CTBR = 1, QB_CMD_PS = 2, QB_CMD_LV = 3, QB_CMD_ROTOR = 4 };

typedef struct qb_params {
    /* QuadParams */
    double mass;
    double inertia[3];
    double gravity[3];
    double torque_arms[4][3];
    double thrust_coeffs[3]; /* k2, k1, k0 */
    double drag_c[3];        /* 0.5*rho*Cd*s */
    double rotor_lo, rotor_hi;
    double alloc_inv[4][4];
    double thrust_lo, thrust_hi;
    double hover_speed;
    /* SimConfig */
    double physics_dt;  /* h = control_dt / substeps */
    double half_dt;     /* 0.5 * h   (dynamics.py:215, evaluated once as a scalar) */
    double sixth_dt;    /* h / 6.0   (dynamics.py:221) */
    double lag_alpha;   /* np.exp(-motor_decay * h) */
    int32_t substeps;
    int32_t integrator; /* qb_integrator */
    /* ControllerGains */
    double rate_p[3];
    double attitude_p[3];
    double vel_p[3];
    double vel_d[3];
    double pos_p[3];
    double pos_d[3];
    double max_speed;
    double max_tilt_accel;
} qb_params;

#ifdef __cplusplus
}
#endif

#endif /* QB_PARAMS_H */
