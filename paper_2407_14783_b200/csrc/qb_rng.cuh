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

// Standard normal.  numpy's Generator uses a 256-level ziggurat whose
// tables are not exposed; this Marsaglia polar draw on the same stream is
// statistically (not bitwise) equivalent -- no BASELINE config spawns from a
// normal distribution.
QB_D double normal_draw(Pcg64 &r) {
    double u, v, s;
    do {
        u = 2.0 * pcg64_next_double(r) - 1.0;
        v = 2.0 * pcg64_next_double(r) - 1.0;
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    return u * sqrt(-2.0 * log(s) / s);
}
#endif
