// qb_k_observe.cu -- the sensor half of QuadEnvBase.get_observation
// (env/base.py:287-305): ideal IMU readings (sensing.py:124-147) and the
// noise chains of sensing.py:195-235, one thread per env, sensors in config
// order, every draw taken from the env's PCG64 stream in numpy's order:
//   normal / speckle   rng.standard_normal(shape)       (ziggurat, qb_rng.cuh)
//   poisson            rng.poisson(max(v,0) * scaling)  (mult / PTRS)
//   saltpepper         rng.random(shape) twice          (corrupt, then salt)
//   redwood            rng.standard_normal(shape) in disparity space
// Values are processed in double like the reference (np.asarray(.., float));
// the FP32 build stores each pass in float32.
#include "qb_dynamics.cuh"
#include "qb_internal.h"
#include "qb_rng.cuh"

namespace {

struct ObsArgs {
    int n_sensors;
    qb_sensor_obs s[QB_MAX_SENSORS];
};

// one noise pass over an image of hw values: in (first pass: the rendered
// frame, int32 ids or S depth; later passes: the observation itself) -> out
template <class S>
__device__ void noise_pass(const qb_noise &nz, Pcg64 &r, const void *in_ptr, bool in_ids, S *out, long long hw) {
    auto in = [&](long long k) -> double {
        return in_ids ? (double)static_cast<const int32_t *>(in_ptr)[k] : (double)static_cast<const S *>(in_ptr)[k];
    };
    auto copy = [&]() {
        for (long long k = 0; k < hw; ++k) out[k] = (S)in(k);
    };
    switch (nz.kind) {
        case QB_NOISE_NORMAL:  // values + sigma * standard_normal
            if (nz.sigma == 0.0) return copy();
            for (long long k = 0; k < hw; ++k) out[k] = (S)__dadd_rn(in(k), __dmul_rn(nz.sigma, normal_draw(r)));
            return;
        case QB_NOISE_SPECKLE:  // values * (1 + sigma * standard_normal)
            if (nz.sigma == 0.0) return copy();
            for (long long k = 0; k < hw; ++k)
                out[k] = (S)__dmul_rn(in(k), __dadd_rn(1.0, __dmul_rn(nz.sigma, normal_draw(r))));
            return;
        case QB_NOISE_POISSON:  // poisson(maximum(values, 0) * scaling) / scaling
            for (long long k = 0; k < hw; ++k) {
                const double v = in(k);
                const double lam = __dmul_rn(isnan(v) ? v : fmax(v, 0.0), nz.scaling);
                out[k] = (S)__ddiv_rn((double)poisson_draw(r, lam), nz.scaling);
            }
            return;
        case QB_NOISE_SALTPEPPER: {
            if (nz.p == 0.0) return copy();
            double lo = in(0), hi = in(0);
            for (long long k = 1; k < hw; ++k) {
                lo = fmin(lo, in(k));
                hi = fmax(hi, in(k));
            }
            // corrupt = random(shape) < p, then salt = random(shape) < 0.5: the
            // second block of draws starts hw words later in the same stream
            Pcg64 rs = r;
            pcg64_advance(rs, (u128)hw);
            for (long long k = 0; k < hw; ++k) {
                const bool corrupt = pcg64_next_double(r) < nz.p;
                const bool salt = pcg64_next_double(rs) < 0.5;
                const double v = in(k);
                out[k] = (S)(corrupt ? (salt ? hi : lo) : v);
            }
            r = rs;
            return;
        }
        default: {  // QB_NOISE_REDWOOD (depth only)
            double vmax = in(0);
            for (long long k = 1; k < hw; ++k) vmax = fmax(vmax, in(k));
            const double floor_disp = hw > 0 ? __ddiv_rn(1.0, __dadd_rn(vmax, 1.0)) : 1e-6;
            for (long long k = 0; k < hw; ++k) {
                double d = __ddiv_rn(1.0, fmax(in(k), 1e-6));
                if (nz.sigma_disparity > 0.0) d = __dadd_rn(d, __dmul_rn(nz.sigma_disparity, normal_draw(r)));
                if (nz.quantization > 0.0) d = __dmul_rn(rint(__ddiv_rn(d, nz.quantization)), nz.quantization);
                out[k] = (S)__ddiv_rn(1.0, fmax(d, floor_disp));
            }
            return;
        }
    }
}

// sensing.py:124-147: body_wrench (thrusts from the rotor speeds, drag from
// v_B = R(q)^T v, force_z += t0 + t1 + t2 + t3) / mass and the body rates,
// in the reference's operation order (exact double)
template <class S> __device__ void imu_read(const DynConsts<xd> &C, const S *st, long long ld, long long i, double *o) {
    xd q[4], th[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        q[k] = xd((double)st[(6 + k) * ld + i]);
        const xd w((double)st[(13 + k) * ld + i]);
        th[k] = C.k2 * (w * w) + C.k1 * w + C.k0;
    }
    xd bx, by, bz;
    q_rot<xd, -1>(q, xd((double)st[3 * ld + i]), xd((double)st[4 * ld + i]), xd((double)st[5 * ld + i]), bx, by, bz);
    const xd fx = C.neg_drag[0] * bx * r_abs(bx), fy = C.neg_drag[1] * by * r_abs(by);
    const xd fz = C.neg_drag[2] * bz * r_abs(bz) + (th[0] + th[1] + th[2] + th[3]);
    o[0] = (fx / C.mass).v;
    o[1] = (fy / C.mass).v;
    o[2] = (fz / C.mass).v;
    for (int k = 0; k < 3; ++k) o[3 + k] = (double)st[(10 + k) * ld + i];
}

template <class S> __global__ void __launch_bounds__(128) k_env_observe(DynConsts<xd> C, qb_env_buffers B, ObsArgs O) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    Pcg64 r = pcg_load(B.rng + 4 * i);
    for (int s = 0; s < O.n_sensors; ++s) {
        const qb_sensor_obs &so = O.s[s];
        S *out = static_cast<S *>(so.out);
        if (so.kind == QB_SENSOR_IMU) {
            double v[6];
            imu_read<S>(C, static_cast<const S *>(B.state), B.ld, i, v);
            for (int m = 0; m < so.n_noise; ++m)  // IMU readings take Gaussian noise only
                if (so.noise[m].sigma != 0.0)
                    for (int k = 0; k < 6; ++k) v[k] = __dadd_rn(v[k], __dmul_rn(so.noise[m].sigma, normal_draw(r)));
            for (int k = 0; k < 6; ++k) out[6 * i + k] = (S)v[k];
            continue;
        }
        const long long hw = (long long)so.width * so.height;
        S *img = out + i * hw;
        const bool ids = so.kind == QB_SENSOR_SEGMENTATION;
        const void *src = ids ? (const void *)(static_cast<const int32_t *>(so.src) + i * hw)
                              : (const void *)(static_cast<const S *>(so.src) + i * hw);
        if (so.n_noise == 0) {
            for (long long k = 0; k < hw; ++k)
                img[k] = ids ? (S) static_cast<const int32_t *>(src)[k] : static_cast<const S *>(src)[k];
            continue;
        }
        for (int m = 0; m < so.n_noise; ++m) {
            if (m == 0)
                noise_pass<S>(so.noise[m], r, src, ids, img, hw);
            else
                noise_pass<S>(so.noise[m], r, img, false, img, hw);
        }
    }
    pcg_store(B.rng + 4 * i, r);
}

__global__ void k_rng_normals(long long n, uint64_t *rng, int k, double *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Pcg64 r = pcg_load(rng + 4 * i);
    for (int j = 0; j < k; ++j) out[i * k + j] = normal_draw(r);
    pcg_store(rng + 4 * i, r);
}

__global__ void k_rng_poissons(long long n, uint64_t *rng, int k, const double *lam, int64_t *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Pcg64 r = pcg_load(rng + 4 * i);
    for (int j = 0; j < k; ++j) out[i * k + j] = poisson_draw(r, lam[i * k + j]);
    pcg_store(rng + 4 * i, r);
}

}  // namespace

namespace qb {
int launch_observe(const qb_params *p, const qb_env_buffers *b, int n_sensors, const qb_sensor_obs *sensors,
                   cudaStream_t st) {
    if (n_sensors < 0 || n_sensors > QB_MAX_SENSORS) {
        set_error("env_observe: %d sensors (max %d)", n_sensors, QB_MAX_SENSORS);
        return QB_EINVAL;
    }
    ObsArgs O;
    O.n_sensors = n_sensors;
    for (int s = 0; s < n_sensors; ++s) {
        const qb_sensor_obs &so = sensors[s];
        if (so.kind < QB_SENSOR_DEPTH || so.kind > QB_SENSOR_IMU || so.n_noise < 0 || so.n_noise > QB_MAX_NOISE ||
            !so.out || (so.kind != QB_SENSOR_IMU && (!so.src || so.width < 1 || so.height < 1))) {
            set_error("env_observe: bad sensor %d", s);
            return QB_EINVAL;
        }
        for (int m = 0; m < so.n_noise; ++m) {
            const int k = so.noise[m].kind;
            const bool ok = so.kind == QB_SENSOR_IMU ? k == QB_NOISE_NORMAL
                                                     : (k >= QB_NOISE_NORMAL && k <= QB_NOISE_REDWOOD &&
                                                        (k != QB_NOISE_REDWOOD || so.kind == QB_SENSOR_DEPTH));
            if (!ok) {
                set_error("env_observe: noise kind %d is not defined for sensor kind %d", k, so.kind);
                return QB_EINVAL;
            }
        }
        O.s[s] = so;
    }
    if (b->n == 0 || n_sensors == 0) return QB_OK;
    DynConsts<xd> C = make_consts<xd>(*p);
    const int BS = 128;
    if (b->dtype == QB_F32)
        k_env_observe<float><<<env_grid(b->n, BS), BS, 0, st>>>(C, *b, O);
    else
        k_env_observe<double><<<env_grid(b->n, BS), BS, 0, st>>>(C, *b, O);
    return check_launch("env_observe");
}

int launch_rng_normals(long long n, uint64_t *rng, int k, double *out, cudaStream_t st) {
    if (n == 0) return QB_OK;
    k_rng_normals<<<env_grid(n, 128), 128, 0, st>>>(n, rng, k, out);
    return check_launch("rng_normals");
}

int launch_rng_poissons(long long n, uint64_t *rng, int k, const double *lam, int64_t *out, cudaStream_t st) {
    if (n == 0) return QB_OK;
    k_rng_poissons<<<env_grid(n, 128), 128, 0, st>>>(n, rng, k, lam, out);
    return check_launch("rng_poissons");
}
}  // namespace qb
