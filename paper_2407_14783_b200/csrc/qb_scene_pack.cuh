// qb_scene_pack.cuh -- the per-node and per-primitive device records of a
// scene (DevScene, qb_geometry.cuh), shared by the host build (qb_abi.cu,
// binned SAH) and the device build (qb_k_scene.cu, LBVH) so both produce the
// same bits for the same input: every double op is an explicit
// round-to-nearest op on the device (no FMA contraction) and the plain
// operator on the host.
#pragma once
#include <cmath>
#include <cstring>

#include "qb_real.cuh"

namespace qbpack {

QB_HD double add(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
QB_HD double sub(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}
QB_HD double mul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
QB_HD double div(double a, double b) {
#ifdef __CUDA_ARCH__
    return __ddiv_rn(a, b);
#else
    return a / b;
#endif
}

// float node bounds rounded outward by 1e-6 relative (+ the float rounding),
// so the FP32 slab test never misses a box the exact one enters
QB_HD float f_down(double v) {
    const double m = sub(v, mul(1e-6, add(1.0, fabs(v))));
    float f = (float)m;
    if ((double)f > m) f = nextafterf(f, -INFINITY);
    return f;
}
QB_HD float f_up(double v) {
    const double m = add(v, mul(1e-6, add(1.0, fabs(v))));
    float f = (float)m;
    if ((double)f < m) f = nextafterf(f, INFINITY);
    return f;
}
QB_HD float i2f(int a) {
    float f;
    memcpy(&f, &a, 4);
    return f;
}

// conservative culling bounds of one primitive (see DevScene::primc)
QB_HD void cull_record(int type, const double *d, float4 *o) {
    for (int k = 0; k < 4; ++k) o[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    const double grow = 1.0 + 1e-6;
    if (type == 0) {  // sphere
        o[0] = make_float4((float)d[0], (float)d[1], (float)d[2], (float)mul(d[3], grow));
    } else if (type == 1) {  // box: column k of R scaled by h_k
        o[0] = make_float4((float)d[0], (float)d[1], (float)d[2], 0.0f);
        for (int k = 0; k < 3; ++k)
            o[1 + k] = make_float4((float)mul(mul(d[6 + k], d[3 + k]), grow), (float)mul(mul(d[9 + k], d[3 + k]), grow),
                                   (float)mul(mul(d[12 + k], d[3 + k]), grow), 0.0f);
    } else {  // triangle: bounding sphere about the centroid
        double c[3], r2 = 0.0;
        for (int a = 0; a < 3; ++a) c[a] = div(add(add(d[a], d[3 + a]), d[6 + a]), 3.0);
        for (int v = 0; v < 3; ++v) {
            double e = 0.0;
            for (int a = 0; a < 3; ++a) e = add(e, mul(sub(d[3 * v + a], c[a]), sub(d[3 * v + a], c[a])));
            r2 = fmax(r2, e);
        }
        o[0] = make_float4((float)c[0], (float)c[1], (float)c[2], (float)mul(sqrt(r2), grow));
    }
}

// FP32 traversal record of one primitive (ray_*_v in qb_geometry.cuh)
QB_HD void pack_prim(int type, const double *d, float4 *o) {
    for (int k = 0; k < 4; ++k) o[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (type == 0) {
        o[0] = make_float4((float)d[0], (float)d[1], (float)d[2], (float)d[3]);
        o[1] = make_float4((float)mul(d[3], d[3]), 0.f, 0.f, 0.f);
    } else if (type == 1) {
        o[0] = make_float4((float)d[0], (float)d[1], (float)d[2], (float)d[3]);
        o[1] = make_float4((float)d[4], (float)d[5], (float)d[6], (float)d[7]);
        o[2] = make_float4((float)d[8], (float)d[9], (float)d[10], (float)d[11]);
        // w: 1 when R is exactly the identity (+0 off the diagonal), which
        // lets the exact nearest-point scan skip the rotation products
        bool ident = true;
        for (int k = 0; k < 9; ++k) ident = ident && d[6 + k] == (k % 4 == 0 ? 1.0 : 0.0) && !signbit(d[6 + k]);
        o[3] = make_float4((float)d[12], (float)d[13], (float)d[14], ident ? 1.f : 0.f);
    } else {  // the vertices themselves: shared edges stay bit-identical (watertight test)
        o[0] = make_float4((float)d[0], (float)d[1], (float)d[2], (float)d[3]);
        o[1] = make_float4((float)d[4], (float)d[5], (float)d[6], (float)d[7]);
        o[2] = make_float4((float)d[8], 0.f, 0.f, 0.f);
    }
}

}  // namespace qbpack
