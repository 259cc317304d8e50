// qb_real.cuh -- scalar policies for the sm_100a kernels.
//
// Every device routine is a template over its arithmetic type R:
//   float  production path: FP32 CUDA-core math, FMA contraction allowed,
//          divisions by constants folded into reciprocals.
//   xd     "exact double": an FP64 value whose + - * / sqrt are the IEEE
//          round-to-nearest intrinsics (__dadd_rn, __dmul_rn, ...), which
//          ptxas never contracts into an FMA.  Evaluated in the reference's
//          operation order this reproduces numpy/numba (which never contract
//          either) bit for bit; it backs the FP64 validation build and the
//          collision/termination flags, which must be bit-exact.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define QB_HD __host__ __device__ __forceinline__
#define QB_D __device__ __forceinline__

struct xd {
    double v;
    xd() = default;
    QB_HD xd(double x) : v(x) {}
};

#ifdef __CUDACC__
QB_D xd operator+(xd a, xd b) { return xd(__dadd_rn(a.v, b.v)); }
QB_D xd operator-(xd a, xd b) { return xd(__dsub_rn(a.v, b.v)); }
QB_D xd operator*(xd a, xd b) { return xd(__dmul_rn(a.v, b.v)); }
QB_D xd operator/(xd a, xd b) { return xd(__ddiv_rn(a.v, b.v)); }
QB_D xd operator-(xd a) { return xd(-a.v); }
QB_D xd &operator+=(xd &a, xd b) { a = a + b; return a; }
QB_D xd &operator-=(xd &a, xd b) { a = a - b; return a; }
QB_D xd &operator*=(xd &a, xd b) { a = a * b; return a; }
QB_D bool operator<(xd a, xd b) { return a.v < b.v; }
QB_D bool operator>(xd a, xd b) { return a.v > b.v; }
QB_D bool operator<=(xd a, xd b) { return a.v <= b.v; }
QB_D bool operator>=(xd a, xd b) { return a.v >= b.v; }
QB_D bool operator==(xd a, xd b) { return a.v == b.v; }
QB_D bool operator!=(xd a, xd b) { return a.v != b.v; }

// math shims with one spelling for both policies
QB_D float r_sqrt(float x) { return sqrtf(x); }
QB_D xd r_sqrt(xd x) { return xd(__dsqrt_rn(x.v)); }
QB_D float r_abs(float x) { return fabsf(x); }
QB_D xd r_abs(xd x) { return xd(fabs(x.v)); }
QB_D float r_cos(float x) { return cosf(x); }
QB_D xd r_cos(xd x) { return xd(cos(x.v)); }
QB_D float r_sin(float x) { return sinf(x); }
QB_D xd r_sin(xd x) { return xd(sin(x.v)); }
QB_D float r_exp(float x) { return expf(x); }
QB_D xd r_exp(xd x) { return xd(exp(x.v)); }
QB_D bool r_isfinite(float x) { return isfinite(x); }
QB_D bool r_isfinite(xd x) { return isfinite(x.v); }
QB_D bool r_isnan(float x) { return isnan(x); }
QB_D bool r_isnan(xd x) { return isnan(x.v); }
QB_D double r_dbl(float x) { return (double)x; }
QB_D double r_dbl(xd x) { return x.v; }

// python builtin min/max semantics on two values (first argument wins ties)
template <class R> QB_D R py_max(R a, R b) { return b > a ? b : a; }
template <class R> QB_D R py_min(R a, R b) { return b < a ? b : a; }
// np.maximum / np.minimum (NaN propagating), np.clip
template <class R> QB_D R np_max(R a, R b) { return r_isnan(a) ? a : (r_isnan(b) ? b : (b > a ? b : a)); }
template <class R> QB_D R np_min(R a, R b) { return r_isnan(a) ? a : (r_isnan(b) ? b : (b < a ? b : a)); }
template <class R> QB_D R np_clip(R x, R lo, R hi) { return np_min(np_max(x, lo), hi); }

// policy clamps: the exact build keeps numpy's NaN propagation; the FP32
// build uses the single-instruction FMNMX forms (callers re-check finiteness
// of their inputs where NaN propagation is observable)
template <class R> QB_D R p_max(R a, R b) { return np_max(a, b); }
template <class R> QB_D R p_min(R a, R b) { return np_min(a, b); }
template <class R> QB_D R p_clip(R x, R lo, R hi) { return np_clip(x, lo, hi); }
template <> QB_D float p_max<float>(float a, float b) { return fmaxf(a, b); }
template <> QB_D float p_min<float>(float a, float b) { return fminf(a, b); }
template <> QB_D float p_clip<float>(float x, float lo, float hi) { return fminf(fmaxf(x, lo), hi); }
#endif

template <class R> struct is_exact { static constexpr bool value = false; };
template <> struct is_exact<xd> { static constexpr bool value = true; };

// storage type of an arithmetic policy
template <class R> struct storage_of { using type = R; };
template <> struct storage_of<xd> { using type = double; };

template <class R> QB_HD R from_dbl(double x) { return R(x); }
template <> QB_HD float from_dbl<float>(double x) { return (float)x; }

template <class R> QB_HD typename storage_of<R>::type to_store(R x) { return x; }
template <> QB_HD double to_store<xd>(xd x) { return x.v; }

QB_HD float infinity_f() { return __builtin_huge_valf(); }
QB_HD double infinity_d() { return __builtin_huge_val(); }
