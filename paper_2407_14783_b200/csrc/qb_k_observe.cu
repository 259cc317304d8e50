// qb_k_observe.cu -- the sensor half of QuadEnvBase.get_observation
// (env/base.py:287-305): ideal IMU readings (sensing.py:124-147) and the
// noise chains of sensing.py:195-235, sensors in config order, every draw
// taken from the env's PCG64 stream in numpy's order:
//   normal / speckle   rng.standard_normal(shape)       (ziggurat, qb_rng.cuh)
//   poisson            rng.poisson(max(v,0) * scaling)  (mult / PTRS)
//   saltpepper         rng.random(shape) twice          (corrupt, then salt)
//   redwood            rng.standard_normal(shape) in disparity space
// Values are processed in double like the reference (np.asarray(.., float));
// the FP32 build stores each pass in float32.  Two kernels: warp per env with
// speculative stream reads (k_env_observe_warp, every chain without Poisson)
// and thread per env (k_env_observe, chains with Poisson noise, whose draw
// count per pixel depends on the value).
#include "qb_dynamics.cuh"
#include "qb_checks.cuh"
#include "qb_internal.h"
#include "qb_rng.cuh"

namespace {

struct ObsArgs {
    int n_sensors;
    qb_sensor_obs s[QB_MAX_SENSORS];
};

// Memory layout: one warp owns 32 consecutive envs; every pass walks the
// image in 32-pixel chunks, staged through a [32 envs][33] double tile in
// shared memory -- lane l loads / stores pixel l of each env's chunk (one
// coalesced 128 B line per env), while each thread runs its own env's chunk
// sequentially on its own generator (the numpy draw order).  Row stride 33
// keeps both access patterns bank-conflict free.
#ifndef QB_OBS_UNROLL
#define QB_OBS_UNROLL 8  // tile rows loaded per batch (loads in flight per lane)
#endif
#ifndef QB_OBS_MINB
#define QB_OBS_MINB 4  // measured: 4 blocks (128 regs) beats 3 (1.7x) and 6-8 (spills)
#endif
constexpr int kObsUnroll = QB_OBS_UNROLL;  // (pragma arguments are not macro-expanded)
// warps per block: two double-buffered tiles per warp stay under the 48 KB
// static shared-memory limit (FP64 validation build: 2 warps)
template <class S> struct ObsWarps {
    static constexpr int value = sizeof(S) == 8 ? 2 : 4;
};
constexpr int TILE_PX = 32;

// tile values are in the observation dtype: every pass rounds its output to
// S anyway, and the inputs (S depth, int32 ids < 2^24) are exact in S.  An
// id tile holds the raw int32 bits until read (cp.async copies bytes).
template <class S> struct Tile {
    S v[32][TILE_PX + 1];
};

template <class S> __device__ __forceinline__ S tile_val(const Tile<S> &t, int e, int k, bool ids) {
    return ids ? (S) * reinterpret_cast<const int32_t *>(&t.v[e][k]) : t.v[e][k];
}

// asynchronous warp-cooperative chunk load (cp.async, no registers held):
// tile.v[e][l] <- pixel c0 + l of env e0 + e; the caller commits / waits
template <class S>
__device__ __forceinline__ void tile_load_async(Tile<S> &t, const void *img, bool ids, long long e0, long long n,
                                                long long hw, long long c0, int lane) {
    const long long k = c0 + lane;
#pragma unroll 8
    for (int e = 0; e < 32; ++e) {
        S *dst = &t.v[e][lane];
        if (e0 + e < n && k < hw) {
            const long long off = (e0 + e) * hw + k;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
            if (ids)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(static_cast<const int32_t *>(img) + off));
            else if (sizeof(S) == 4)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(static_cast<const S *>(img) + off));
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(static_cast<const S *>(img) + off));
        } else {
            *dst = S(0);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

__device__ __forceinline__ void tile_wait_all_but_last() {
    asm volatile("cp.async.wait_group 1;\n" ::);
    __syncwarp();
}

template <class S>
__device__ __forceinline__ void tile_store(const Tile<S> &t, S *img, long long e0, long long n, long long hw, long long c0,
                                           int lane) {
    __syncwarp();
    const long long k = c0 + lane;
#pragma unroll kObsUnroll
    for (int e = 0; e < 32; ++e)
        if (e0 + e < n && k < hw) img[(e0 + e) * hw + k] = t.v[e][lane];
    __syncwarp();
}

// one noise pass over an image of hw values for the warp's 32 envs: in
// (first pass: the rendered frame, int32 ids or S depth; later passes: the
// observation itself) -> out.  `me` = this thread's env row in the tile.
// `range` holds the input's (min, max) when known (the previous pass tracks
// its output's range), else an extra read pass computes it; on return it
// holds this pass's output range.
template <class S>
__device__ void noise_pass(const qb_noise &nz, Pcg64 &r, bool live, const void *in, bool in_ids, S *out, Tile<S> *t,
                           long long e0, long long n, long long hw, int me, double2 &range, bool &have_range) {
    const int lane = me;
    const long long nchunk = (hw + TILE_PX - 1) / TILE_PX;
    // image reductions first (saltpepper: min / max, redwood: max)
    double lo = range.x, hi = range.y;
    const bool sp = nz.kind == QB_NOISE_SALTPEPPER && nz.p != 0.0, rw = nz.kind == QB_NOISE_REDWOOD;
    if ((sp || rw) && !have_range) {
        tile_load_async<S>(t[0], in, in_ids, e0, n, hw, 0, lane);
        for (long long c = 0; c < nchunk; ++c) {
            if (c + 1 < nchunk) tile_load_async<S>(t[(c + 1) & 1], in, in_ids, e0, n, hw, (c + 1) * TILE_PX, lane);
            else asm volatile("cp.async.commit_group;\n" ::);
            tile_wait_all_but_last();
            const Tile<S> &tc = t[c & 1];
            const int m = hw - c * TILE_PX < TILE_PX ? (int)(hw - c * TILE_PX) : TILE_PX;
            for (int k = 0; k < m; ++k) {
                const double v = (double)tile_val(tc, me, k, in_ids);
                lo = (c == 0 && k == 0) ? v : fmin(lo, v);
                hi = (c == 0 && k == 0) ? v : fmax(hi, v);
            }
            __syncwarp();
        }
    }
    Pcg64 rs = r;  // saltpepper: second block of draws, hw words later
    if (sp && live) pcg64_advance(rs, (u128)hw);
    const double floor_disp = hw > 0 ? __ddiv_rn(1.0, __dadd_rn(hi, 1.0)) : 1e-6;
    double olo = 0.0, ohi = 0.0;
    tile_load_async<S>(t[0], in, in_ids, e0, n, hw, 0, lane);
    for (long long c = 0; c < nchunk; ++c) {
        // prefetch the next chunk while this one is computed and stored
        if (c + 1 < nchunk) tile_load_async<S>(t[(c + 1) & 1], in, in_ids, e0, n, hw, (c + 1) * TILE_PX, lane);
        else asm volatile("cp.async.commit_group;\n" ::);
        tile_wait_all_but_last();
        Tile<S> &tc = t[c & 1];
        const long long c0 = c * TILE_PX;
        const int m = hw - c0 < TILE_PX ? (int)(hw - c0) : TILE_PX;
        if (live) {
            for (int k = 0; k < m; ++k) {
                const double v = (double)tile_val(tc, me, k, in_ids);
                double o = v;
                switch (nz.kind) {
                    case QB_NOISE_NORMAL:  // values + sigma * standard_normal
                        if (nz.sigma != 0.0) o = __dadd_rn(v, __dmul_rn(nz.sigma, normal_draw(r)));
                        break;
                    case QB_NOISE_SPECKLE:  // values * (1 + sigma * standard_normal)
                        if (nz.sigma != 0.0) o = __dmul_rn(v, __dadd_rn(1.0, __dmul_rn(nz.sigma, normal_draw(r))));
                        break;
                    case QB_NOISE_POISSON: {  // poisson(maximum(values, 0) * scaling) / scaling
                        const double lam = __dmul_rn(isnan(v) ? v : fmax(v, 0.0), nz.scaling);
                        o = __ddiv_rn((double)poisson_draw(r, lam), nz.scaling);
                        break;
                    }
                    case QB_NOISE_SALTPEPPER:  // random() < p corrupts, random() < 0.5 picks max
                        if (sp) {
                            const bool corrupt = pcg64_next_double(r) < nz.p;
                            const bool salt = pcg64_next_double(rs) < 0.5;
                            o = corrupt ? (salt ? hi : lo) : v;
                        }
                        break;
                    default: {  // QB_NOISE_REDWOOD (depth only)
                        double d = __ddiv_rn(1.0, fmax(v, 1e-6));
                        if (nz.sigma_disparity > 0.0) d = __dadd_rn(d, __dmul_rn(nz.sigma_disparity, normal_draw(r)));
                        if (nz.quantization > 0.0) d = __dmul_rn(rint(__ddiv_rn(d, nz.quantization)), nz.quantization);
                        o = __ddiv_rn(1.0, fmax(d, floor_disp));
                    }
                }
                const S so = (S)o;  // each pass stores in the observation dtype
                const double os = (double)so;
                tc.v[me][k] = so;
                olo = (c == 0 && k == 0) ? os : fmin(olo, os);
                ohi = (c == 0 && k == 0) ? os : fmax(ohi, os);
            }
        }  // (rows of envs beyond n are never stored)
        tile_store<S>(tc, out, e0, n, hw, c0, lane);
    }
    if (sp && live) r = rs;
    range = make_double2(olo, ohi);
    have_range = true;
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

template <class S>
__global__ void __launch_bounds__(ObsWarps<S>::value * 32, QB_OBS_MINB) k_env_observe(DynConsts<xd> C, qb_env_buffers B, ObsArgs O) {
    __shared__ Tile<S> tiles[ObsWarps<S>::value][2];
    Tile<S> *t = tiles[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long e0 = i - lane;  // first env of this warp
    if (e0 >= B.n) return;          // warp-uniform
    const bool live = i < B.n;
    Pcg64 r;
    if (live) r = pcg_load(B.rng + 4 * i);
    for (int s = 0; s < O.n_sensors; ++s) {
        const qb_sensor_obs &so = O.s[s];
        S *out = static_cast<S *>(so.out);
        if (so.kind == QB_SENSOR_IMU) {
            if (!live) continue;
            double v[6];
            imu_read<S>(C, static_cast<const S *>(B.state), B.ld, i, v);
            for (int m = 0; m < so.n_noise; ++m)  // IMU readings take Gaussian noise only
                if (so.noise[m].sigma != 0.0)
                    for (int k = 0; k < 6; ++k) v[k] = __dadd_rn(v[k], __dmul_rn(so.noise[m].sigma, normal_draw(r)));
            for (int k = 0; k < 6; ++k) out[6 * i + k] = (S)v[k];
            continue;
        }
        const long long hw = (long long)so.width * so.height;
        const bool ids = so.kind == QB_SENSOR_SEGMENTATION;
        if (so.n_noise == 0) {  // plain copy into the observation dtype
            for (long long c0 = 0; c0 < hw; c0 += TILE_PX) {
                tile_load_async<S>(t[0], so.src, ids, e0, B.n, hw, c0, lane);
                asm volatile("cp.async.wait_group 0;\n" ::);
                __syncwarp();
                if (ids) {
                    const int m = hw - c0 < TILE_PX ? (int)(hw - c0) : TILE_PX;
                    for (int k = 0; k < m; ++k) t[0].v[lane][k] = tile_val(t[0], lane, k, true);
                }
                tile_store<S>(t[0], out, e0, B.n, hw, c0, lane);
            }
            continue;
        }
        double2 range = make_double2(0.0, 0.0);
        bool have_range = false;
        for (int m = 0; m < so.n_noise; ++m) {
            if (m == 0)
                noise_pass<S>(so.noise[m], r, live, so.src, ids, out, t, e0, B.n, hw, lane, range, have_range);
            else
                noise_pass<S>(so.noise[m], r, live, out, false, out, t, e0, B.n, hw, lane, range, have_range);
        }
    }
    if (live) pcg_store(B.rng + 4 * i, r);
}

// ---- warp-per-env sensor pass -------------------------------------------
// One warp per env, 32 consecutive pixels per round.  The numpy draw order is
// kept by reading the env's stream speculatively: lane l evaluates word P+l+1
// (the LCG jump state -> A_{l+1} state + C_{l+1}, qb_rng.cuh) and the
// ziggurat fast test on it; the first lane whose word fails (~1.2% per draw)
// finishes its normal sequentially from there, the lanes before it keep
// theirs, and the next round starts after the words that draw consumed.
// Salt-and-pepper draws are fixed-count (corrupt block, then salt block), so
// every lane jumps straight to its words.  The reads and writes of a round
// are one coalesced 128 B line per env, and a 16384-env batch fills the GPU
// (the thread-per-env kernel above has 32x fewer warps).  Chains with
// Poisson noise (a data-dependent number of uniform draws) use that kernel.
struct WarpRng {
    u128 P, inc;    // the stream's state before the next draw (warp-uniform)
    u128 A, C;      // this lane's jump over lane+1 words
    u128 A32, C32;  // the jump over 32 words
};

__device__ __forceinline__ u128 shfl_u128(u128 v, int src) {
    const unsigned long long lo = __shfl_sync(0xffffffffu, (unsigned long long)v, src);
    const unsigned long long hi = __shfl_sync(0xffffffffu, (unsigned long long)(v >> 64), src);
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ double warp_fmin(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_fmax(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// pixel k of the input image in double: int32 ids through S (the tile rule
// above), S values as stored.  Plain loads: later passes read what the
// previous pass of this kernel wrote.
template <class S> __device__ __forceinline__ double px_in(const void *in, bool ids, long long k) {
    return ids ? (double)(S) static_cast<const int32_t *>(in)[k] : (double)static_cast<const S *>(in)[k];
}

__device__ __forceinline__ double draw_double(u128 state) {
    return (double)(pcg64_output(state) >> 11) * (1.0 / 9007199254740992.0);
}

// the per-pixel transform of the one-normal-per-pixel noises (x = the draw)
__device__ __forceinline__ double normal_noise(const qb_noise &nz, double v, double x, double floor_disp) {
    switch (nz.kind) {
        case QB_NOISE_NORMAL:
            return __dadd_rn(v, __dmul_rn(nz.sigma, x));
        case QB_NOISE_SPECKLE:
            return __dmul_rn(v, __dadd_rn(1.0, __dmul_rn(nz.sigma, x)));
        default: {  // redwood
            double d = __ddiv_rn(1.0, fmax(v, 1e-6));
            if (nz.sigma_disparity > 0.0) d = __dadd_rn(d, __dmul_rn(nz.sigma_disparity, x));
            if (nz.quantization > 0.0) d = __dmul_rn(rint(__ddiv_rn(d, nz.quantization)), nz.quantization);
            return __ddiv_rn(1.0, fmax(d, floor_disp));
        }
    }
}

// the input pixels of a round come from a two-line register window (32
// values per line, one per lane) so each load is issued a round before it
// is used; rounds start anywhere in the window and shuffle their values out.
template <class S> struct PxWindow {
    const void *in;
    bool ids;
    long long hw, base;  // base: pixel of cur's lane 0 (32-aligned)
    S cur, nxt;
    __device__ __forceinline__ S load(long long k) const {
        if (k >= hw) return S(0);
        return ids ? (S) static_cast<const int32_t *>(in)[k] : static_cast<const S *>(in)[k];
    }
    __device__ __forceinline__ void init(const void *in_, bool ids_, long long hw_, int lane) {
        in = in_;
        ids = ids_;
        hw = hw_;
        base = 0;
        cur = load(lane);
        nxt = load(32 + lane);
    }
    // pixel pk + lane (pk - base < 32)
    __device__ __forceinline__ S at(long long pk, int lane) const {
        const int src = (int)(pk - base) + lane;
        const S a = __shfl_sync(0xffffffffu, cur, src & 31), b = __shfl_sync(0xffffffffu, nxt, src & 31);
        return src < 32 ? a : b;
    }
    __device__ __forceinline__ void advance(long long pk, int lane) {
        if (pk - base >= 32) {  // warp-uniform
            base += 32;
            cur = nxt;
            nxt = load(base + 32 + lane);
        }
    }
};

// one noise pass over one env's image (in / out at the env's base); the
// range contract is noise_pass's, except that the output range is only
// tracked when the next pass reads it (need_range)
template <class S>
__device__ void warp_noise_pass(const qb_noise &nz, WarpRng &g, const void *in, bool in_ids, S *out, long long hw,
                                int lane, double2 &range, bool &have_range, bool need_range) {
    const bool sp = nz.kind == QB_NOISE_SALTPEPPER && nz.p != 0.0, rw = nz.kind == QB_NOISE_REDWOOD;
    double lo = range.x, hi = range.y;
    if ((sp || rw) && !have_range) {
        lo = hi = __longlong_as_double(0x7ff8000000000000LL);  // fmin / fmax skip NaN
        for (long long k = lane; k < hw; k += 32) {
            const double v = px_in<S>(in, in_ids, k);
            lo = fmin(lo, v);
            hi = fmax(hi, v);
        }
        lo = warp_fmin(lo);
        hi = warp_fmax(hi);
    }
    const double floor_disp = __ddiv_rn(1.0, __dadd_rn(hi, 1.0));
    S olo = S(__longlong_as_double(0x7ff8000000000000LL)), ohi = olo;  // (exact in S: outputs are S values)
    const bool draws = ((nz.kind == QB_NOISE_NORMAL || nz.kind == QB_NOISE_SPECKLE) && nz.sigma != 0.0) ||
                       (rw && nz.sigma_disparity > 0.0);
    if (draws) {
        PxWindow<S> win;
        win.init(in, in_ids, hw, lane);
        for (long long pk = 0; pk < hw;) {
            const int npx = hw - pk < 32 ? (int)(hw - pk) : 32;
            const double v = (double)win.at(pk, lane);
            u128 st = g.A * g.P + g.C;  // the state that yields word P + lane + 1
            const uint64_t w = pcg64_output(st);
            double x;
            const bool ok = normal_fast(w, x);
            const unsigned bad = __ballot_sync(0xffffffffu, lane < npx && !ok);
            int cnt = npx;
            if (bad) {
                const int f = __ffs(bad) - 1;
                cnt = f + 1;
                if (lane == f) {  // the slow continuation of this draw
                    Pcg64 rr;
                    rr.state = st;
                    rr.inc = g.inc;
                    x = normal_from(w, rr);
                    st = rr.state;
                }
            }
            if (lane < cnt) {
                const S so = (S)normal_noise(nz, v, x, floor_disp);
                out[pk + lane] = so;
                if (need_range) {
                    olo = fmin(olo, so);
                    ohi = fmax(ohi, so);
                }
            }
            g.P = shfl_u128(st, cnt - 1);
            pk += cnt;
            win.advance(pk, lane);
        }
    } else if (sp) {
        // corrupt = random(shape) < p over words P+1..P+hw, salt = random(shape)
        // < 0.5 over the next hw words
        const PcgJump jh = pcg64_jump(g.inc, (u128)hw);
        u128 sc = g.A * g.P + g.C, ss = jh.A * sc + jh.C;
        for (long long k0 = 0; k0 < hw; k0 += 32) {
            const long long k = k0 + lane;
            if (k < hw) {
                const double v = px_in<S>(in, in_ids, k);
                const bool corrupt = draw_double(sc) < nz.p;
                const bool salt = draw_double(ss) < 0.5;
                const S so = (S)(corrupt ? (salt ? hi : lo) : v);
                out[k] = so;
                if (need_range) {
                    olo = fmin(olo, so);
                    ohi = fmax(ohi, so);
                }
            }
            sc = g.A32 * sc + g.C32;
            ss = g.A32 * ss + g.C32;
        }
        g.P = jh.A * (jh.A * g.P + jh.C) + jh.C;
    } else {  // no draws: the deterministic part of the transform only
        for (long long k = lane; k < hw; k += 32) {
            const double v = px_in<S>(in, in_ids, k);
            const S so = (S)(rw ? normal_noise(nz, v, 0.0, floor_disp) : v);
            out[k] = so;
            if (need_range) {
                olo = fmin(olo, so);
                ohi = fmax(ohi, so);
            }
        }
    }
    __syncwarp();  // the next pass reads this one's output across lanes
    if (need_range) range = make_double2(warp_fmin((double)olo), warp_fmax((double)ohi));
    have_range = need_range;
}

#ifndef QB_OBSW_MINB
#define QB_OBSW_MINB 8  // measured: 64 regs, 8 blocks beat 80 regs (1.3x) and no cap (1.5x)
#endif
template <class S>
__global__ void __launch_bounds__(128, QB_OBSW_MINB) k_env_observe_warp(DynConsts<xd> C, qb_env_buffers B, ObsArgs O) {
    const int lane = threadIdx.x & 31;
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= B.n) return;  // warp-uniform
    WarpRng g;
    {
        const Pcg64 r = pcg_load(B.rng + 4 * i);
        g.P = r.state;
        g.inc = r.inc;
        const PcgJump j = pcg64_jump(r.inc, (u128)(lane + 1));
        g.A = j.A;
        g.C = j.C;
        g.A32 = shfl_u128(j.A, 31);
        g.C32 = shfl_u128(j.C, 31);
    }
    for (int s = 0; s < O.n_sensors; ++s) {
        const qb_sensor_obs &so = O.s[s];
        S *out = static_cast<S *>(so.out);
        if (so.kind == QB_SENSOR_IMU) {  // six readings: every lane runs the (uniform) sequential draws
            double v[6];
            imu_read<S>(C, static_cast<const S *>(B.state), B.ld, i, v);
            Pcg64 r;
            r.state = g.P;
            r.inc = g.inc;
            for (int m = 0; m < so.n_noise; ++m)
                if (so.noise[m].sigma != 0.0)
                    for (int k = 0; k < 6; ++k) v[k] = __dadd_rn(v[k], __dmul_rn(so.noise[m].sigma, normal_draw(r)));
            g.P = r.state;
            if (lane < 6) {
                double vk = v[0];
#pragma unroll
                for (int k = 1; k < 6; ++k)
                    if (lane == k) vk = v[k];
                out[6 * i + lane] = (S)vk;
            }
            continue;
        }
        const long long hw = (long long)so.width * so.height;
        const bool ids = so.kind == QB_SENSOR_SEGMENTATION;
        const void *src = ids ? (const void *)(static_cast<const int32_t *>(so.src) + i * hw)
                              : (const void *)(static_cast<const S *>(so.src) + i * hw);
        S *dst = out + i * hw;
        if (so.n_noise == 0) {  // plain copy into the observation dtype
            for (long long k = lane; k < hw; k += 32) dst[k] = (S)px_in<S>(src, ids, k);
            continue;
        }
        double2 range = make_double2(0.0, 0.0);
        bool have_range = false;
        for (int m = 0; m < so.n_noise; ++m) {
            const qb_noise *nx = m + 1 < so.n_noise ? &so.noise[m + 1] : nullptr;
            const bool need = nx && ((nx->kind == QB_NOISE_SALTPEPPER && nx->p != 0.0) || nx->kind == QB_NOISE_REDWOOD);
            if (m == 0)
                warp_noise_pass<S>(so.noise[m], g, src, ids, dst, hw, lane, range, have_range, need);
            else
                warp_noise_pass<S>(so.noise[m], g, dst, false, dst, hw, lane, range, have_range, need);
        }
    }
    if (lane == 0) {
        Pcg64 r;
        r.state = g.P;
        r.inc = g.inc;
        pcg_store(B.rng + 4 * i, r);
    }
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
    bool poisson = false;
    for (int s = 0; s < n_sensors; ++s)
        for (int m = 0; m < O.s[s].n_noise; ++m) poisson |= O.s[s].noise[m].kind == QB_NOISE_POISSON;
    if (!poisson) {  // warp per env (speculative stream reads)
        const int BS = 128;
        if (b->dtype == QB_F32)
            k_env_observe_warp<float><<<env_grid(b->n * 32, BS), BS, 0, st>>>(C, *b, O);
        else
            k_env_observe_warp<double><<<env_grid(b->n * 32, BS), BS, 0, st>>>(C, *b, O);
        return check_launch("env_observe");
    }
    if (b->dtype == QB_F32) {
        const int BS = ObsWarps<float>::value * 32;
        k_env_observe<float><<<env_grid(b->n, BS), BS, 0, st>>>(C, *b, O);
    } else {
        const int BS = ObsWarps<double>::value * 32;
        k_env_observe<double><<<env_grid(b->n, BS), BS, 0, st>>>(C, *b, O);
    }
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
