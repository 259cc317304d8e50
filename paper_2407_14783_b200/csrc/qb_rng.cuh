// qb_rng.cuh -- per-env numpy-compatible random streams.
//
// The reference gives agent i the generator np.random.default_rng(seed + i)
// (env/base.py:95): a PCG64 bit generator seeded through SeedSequence.  To
// keep spawns bit-identical without a host round trip per respawn, both the
// seeding (numpy/random/bit_generator.pyx SeedSequence.mix_entropy +
// generate_state, pcg64.c pcg64_set_seed) and the draws (pcg64 next64 ->
// next_double, distributions.c random_uniform) are restated here and run on
// the device, keyed by the GLOBAL env index so a shard of a multi-GPU run
// draws exactly what a single-GPU run draws for the same env.
#pragma once
#include <cstdint>

#include "qb_real.cuh"

typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state, inc;
};

namespace qbrng {
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;

QB_HD uint32_t hashmix(uint32_t value, uint32_t &hc) {
    value ^= hc;
    hc *= MULT_A;
    value *= hc;
    value ^= value >> 16;
    return value;
}

QB_HD uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
    r ^= r >> 16;
    return r;
}

QB_HD u128 pcg_mult() { return ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL; }

QB_HD void pcg_step(Pcg64 &r) { r.state = r.state * pcg_mult() + r.inc; }
}  // namespace qbrng

// np.random.default_rng(seed) for 0 <= seed < 2**64
QB_HD Pcg64 pcg64_from_seed(uint64_t seed) {
    using namespace qbrng;
    uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int n_ent = (seed >> 32) ? 2 : 1;  // _coerce_to_uint32_array: little-endian words, >= 1
    uint32_t pool[4];
    uint32_t hc = INIT_A;
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, hc);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    uint32_t words[8];
    uint32_t hb = INIT_B;
    for (int i = 0; i < 8; ++i) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> 16;
        words[i] = v;
    }
    uint64_t val[4];
    for (int i = 0; i < 4; ++i) val[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
    u128 initstate = ((u128)val[0] << 64) | val[1];
    u128 initseq = ((u128)val[2] << 64) | val[3];
    Pcg64 r;
    r.state = 0;
    r.inc = (initseq << 1) | 1u;
    pcg_step(r);
    r.state += initstate;
    pcg_step(r);
    return r;
}

QB_HD uint64_t pcg64_next64(Pcg64 &r) {
    qbrng::pcg_step(r);
    uint64_t hi = (uint64_t)(r.state >> 64), lo = (uint64_t)r.state;
    unsigned rot = (unsigned)(r.state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

// jump the stream ahead by delta draws (LCG power by squaring)
QB_HD void pcg64_advance(Pcg64 &r, u128 delta) {
    u128 cur_mult = qbrng::pcg_mult(), cur_plus = r.inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    r.state = acc_mult * r.state + acc_plus;
}

QB_HD double pcg64_next_double(Pcg64 &r) { return (double)(pcg64_next64(r) >> 11) * (1.0 / 9007199254740992.0); }

// storage: 4 x uint64 (state hi, state lo, inc hi, inc lo)
QB_HD Pcg64 pcg_load(const uint64_t *p) {
    Pcg64 r;
    r.state = ((u128)p[0] << 64) | p[1];
    r.inc = ((u128)p[2] << 64) | p[3];
    return r;
}
QB_HD void pcg_store(uint64_t *p, const Pcg64 &r) {
    p[0] = (uint64_t)(r.state >> 64);
    p[1] = (uint64_t)r.state;
    p[2] = (uint64_t)(r.inc >> 64);
    p[3] = (uint64_t)r.inc;
}

#ifdef __CUDACC__
// distributions.c random_uniform: lower + range * next_double, range = high - low
QB_D double uniform_draw(Pcg64 &r, double lo, double hi) {
    double range = __dsub_rn(hi, lo);
    return __dadd_rn(lo, __dmul_rn(range, pcg64_next_double(r)));
}

#define QB_ZIG_ATTR __device__
#include "qb_ziggurat.h"

// distributions.c random_standard_normal (numpy 2.3.5): 256-level ziggurat on
// 52-bit magnitudes; tables in qb_ziggurat.h (generated, pinned against
// numpy by tests/test_rng_restatement.py).  All arithmetic is the IEEE
// double op numpy's C performs (no contraction); log1p/exp are CUDA's libm
// (<= 1 ulp from glibc), which only matters on the ~1% wedge/tail draws.
// the draw that starts with word w (already taken from r); r continues after it
QB_D double normal_from(uint64_t w, Pcg64 &r) {
    for (;;) {
        const int idx = (int)(w & 0xff);
        w >>= 8;
        const uint64_t rabs = (w >> 1) & 0x000fffffffffffffULL;
        double x = __dmul_rn((double)rabs, __ldg(&qb_zig_wi[idx]));
        if (w & 0x1) x = -x;
        if (rabs < __ldg(&qb_zig_ki[idx])) return x;
        if (idx == 0) {
            for (;;) {
                const double xx = __dmul_rn(-(1.0 / QB_ZIG_R), log1p(-pcg64_next_double(r)));
                const double yy = -log1p(-pcg64_next_double(r));
                if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx))
                    return ((rabs >> 8) & 0x1) ? -__dadd_rn(QB_ZIG_R, xx) : __dadd_rn(QB_ZIG_R, xx);
            }
        }
        const double f0 = __ldg(&qb_zig_fi[idx - 1]), f1 = __ldg(&qb_zig_fi[idx]);
        const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(f0, f1), pcg64_next_double(r)), f1);
        const double arg = __dmul_rn(__dmul_rn(-0.5, x), x);  // in [-6.7, 0] on the wedges
        // decide with a float exp when lhs is clearly off it (|error| < 1e-6
        // relative here vs the 1e-5 margin); the double exp only near the edge
        const double ef = (double)__expf((float)arg);
        if (lhs < ef * (1.0 - 1e-5)) return x;
        if (!(lhs > ef * (1.0 + 1e-5)) && lhs < exp(arg)) return x;
        w = pcg64_next64(r);
    }
}

QB_D double normal_draw(Pcg64 &r) { return normal_from(pcg64_next64(r), r); }

// ---- warp-parallel stream access -----------------------------------------
// The LCG jump over d words as an affine map state -> A state + C (the
// advance algorithm above without applying it): lets 32 lanes produce 32
// consecutive words of one stream in parallel.
struct PcgJump {
    u128 A, C;
};
QB_HD PcgJump pcg64_jump(u128 inc, u128 delta) {
    u128 cur_mult = qbrng::pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return {acc_mult, acc_plus};
}
QB_HD uint64_t pcg64_output(u128 state) {
    uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    unsigned rot = (unsigned)(state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

// ziggurat fast path on one word (distributions.c random_standard_normal):
// true with x set when the word alone decides the draw (~98.8%)
QB_D bool normal_fast(uint64_t w, double &x) {
    const int idx = (int)(w & 0xff);
    w >>= 8;
    const uint64_t rabs = (w >> 1) & 0x000fffffffffffffULL;
    x = __dmul_rn((double)rabs, __ldg(&qb_zig_wi[idx]));
    if (w & 0x1) x = -x;
    return rabs < __ldg(&qb_zig_ki[idx]);
}

// distributions.c random_loggam
QB_D double loggam_np(double x) {
    const double a[10] = {8.333333333333333e-02, -2.777777777777778e-03, 7.936507936507937e-04,
                          -5.952380952380952e-04, 8.417508417508418e-04, -1.917526917526918e-03,
                          6.410256410256410e-03, -2.955065359477124e-02, 1.796443723688307e-01,
                          -1.39243221690590e+00};
    if (x == 1.0 || x == 2.0) return 0.0;
    const long long n = x < 7.0 ? (long long)(7 - x) : 0;
    double x0 = __dadd_rn(x, (double)n);
    const double ix = __ddiv_rn(1.0, x0), x2 = __dmul_rn(ix, ix);
    double gl0 = a[9];
    for (int k = 8; k >= 0; --k) gl0 = __dadd_rn(__dmul_rn(gl0, x2), a[k]);
    double gl = __dsub_rn(__dadd_rn(__dadd_rn(__ddiv_rn(gl0, x0), __dmul_rn(0.5, 1.8378770664093453e+00)),
                                    __dmul_rn(__dsub_rn(x0, 0.5), log(x0))),
                          x0);
    if (x < 7.0)
        for (long long k = 1; k <= n; ++k) {
            gl = __dsub_rn(gl, log(__dsub_rn(x0, 1.0)));
            x0 = __dsub_rn(x0, 1.0);
        }
    return gl;
}

// distributions.c random_poisson: multiplication method below 10, PTRS
// (Hoermann's transformed rejection) from 10 up
QB_D long long poisson_draw(Pcg64 &r, double lam) {
    if (lam >= 10) {
        const double slam = __dsqrt_rn(lam), loglam = log(lam);
        const double b = __dadd_rn(0.931, __dmul_rn(2.53, slam));
        const double a = __dadd_rn(-0.059, __dmul_rn(0.02483, b));
        const double invalpha = __dadd_rn(1.1239, __ddiv_rn(1.1328, __dsub_rn(b, 3.4)));
        const double vr = __dsub_rn(0.9277, __ddiv_rn(3.6224, __dsub_rn(b, 2.0)));
        for (;;) {
            const double U = __dsub_rn(pcg64_next_double(r), 0.5);
            const double V = pcg64_next_double(r);
            const double us = __dsub_rn(0.5, fabs(U));
            const long long k = (long long)floor(
                __dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(__ddiv_rn(__dmul_rn(2.0, a), us), b), U), lam), 0.43));
            if (us >= 0.07 && V <= vr) return k;
            if (k < 0 || (us < 0.013 && V > us)) continue;
            const double lhs = __dsub_rn(__dadd_rn(log(V), log(invalpha)),
                                         log(__dadd_rn(__ddiv_rn(a, __dmul_rn(us, us)), b)));
            const double rhs = __dsub_rn(__dadd_rn(-lam, __dmul_rn((double)k, loglam)), loggam_np((double)(k + 1)));
            if (lhs <= rhs) return k;
        }
    }
    if (lam == 0) return 0;
    const double enlam = exp(-lam);
    long long x = 0;
    double prod = 1.0;
    for (;;) {
        prod = __dmul_rn(prod, pcg64_next_double(r));
        if (prod > enlam)
            ++x;
        else
            return x;
    }
}
#endif
