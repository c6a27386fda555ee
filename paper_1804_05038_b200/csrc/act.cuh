// act.cuh -- fp64 exp / expm1 / sigmoid / tanh for the Tier-B activations
// (evaluate in fp64, round once to f32: layers.py:170-181, :225, :265).
//
// Table-free: t = k ln2 + r, |r| <= ln2/2, e^r - 1 by its Taylor series to
// degree 14 (truncation < 4e-19), coefficients in __constant__ memory so every
// DFMA reads them from the constant bank (no per-use 64-bit immediate moves).
// Quotients use the approximate fp64 reciprocal + two Newton steps + one
// residual correction, i.e. ~0.5 ulp like an IEEE division.
// benchmarks/act_err.cu compares these against the CUDA library versions
// exhaustively over every f32 input (profiles/r01_act_err.jsonl).
#pragma once
#include <cuda_runtime.h>

namespace qnmt {

// 1/14!, 1/13!, ..., 1/2!  (Horner order)
static __constant__ double c_expm1_poly[13] = {
    1.1470745597729725e-11, 1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
    2.755731922398589e-07,  2.7557319223985893e-06, 2.48015873015873e-05, 0.0001984126984126984,
    0.001388888888888889,   0.008333333333333333,   0.041666666666666664, 0.16666666666666666,
    0.5};

// e^r - 1 for |r| <= ln2/2 (~1 ulp)
__device__ __forceinline__ double expm1_core(double r) {
    double p = c_expm1_poly[0];
#pragma unroll
    for (int i = 1; i < 13; ++i) p = fma(p, r, c_expm1_poly[i]);
    return fma(r * r, p, r);
}

// t = k ln2 + r; returns r, sets k.  |t| <= 708.
__device__ __forceinline__ double exp_reduce(double t, int& k) {
    const double kd_m = fma(t, 1.4426950408889634, 6755399441055744.0);   // t / ln2 + 1.5 * 2^52
    k = __double2loint(kd_m);
    const double kd = kd_m - 6755399441055744.0;
    const double r = fma(kd, -0.6931471805599453, t);                      // ln2 rounded to f64
    return fma(kd, -2.3190468138462996e-17, r);                            // ln2 - the above
}

__device__ __forceinline__ double scale2k(double v, int k) {   // v * 2^k (result normal)
    return __hiloint2double(__double2hiint(v) + (k << 20), __double2loint(v));
}

// e^t, t in [-700, 700]
__device__ __forceinline__ double exp_f64(double t) {
    int k;
    const double r = exp_reduce(t, k);
    return scale2k(1.0 + expm1_core(r), k);
}

// e^t - 1, t in [-700, 700], relative accuracy near 0
__device__ __forceinline__ double expm1_f64(double t) {
    int k;
    const double r = exp_reduce(t, k);
    const double q = expm1_core(r);
    // branch-free: for k == 0, s = 1 and fma(1, q, 0) = q exactly (q is never -0: r = -0 gives +0)
    const double s = scale2k(1.0, k);
    return fma(s, q, s - 1.0);
}

// n / d for d in [1, 2]: approximate reciprocal, two Newton steps, residual correction
__device__ __forceinline__ double div12(double n, double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    r = fma(fma(-d, r, 1.0), r, r);
    r = fma(fma(-d, r, 1.0), r, r);
    const double q = n * r;
    return fma(fma(-d, q, n), r, q);
}

// fl32(tanh(x)) evaluated in fp64: tanh|x| = -expm1(-2|x|) / (2 + expm1(-2|x|))
__device__ __forceinline__ float tanh_b(float x) {
    const double a = fmin(fabs((double)x), 40.0);   // tanh(40) rounds to 1 in f64
    const double em = expm1_f64(-2.0 * a);
    const double t = div12(-em, 2.0 + em);
    return copysignf(__double2float_rn(t), x);   // odd, including tanh(-0) = -0
}

// fl32(sigmoid(x)) evaluated in fp64 as the reference: 1/(1+e^-x) (x >= 0), e^x/(1+e^x) (x < 0)
__device__ __forceinline__ float sigmoid_b(float x) {
    const double v = (double)x;
    const double t = -fabs(v);
    const double ex = exp_f64(t < -700.0 ? -700.0 : t);   // (branch-free: clamp, then select; NaN stays NaN)
    const double e = t < -700.0 ? 0.0 : ex;           // below: f32 result 0 either way
    const double d = 1.0 + e;
    return __double2float_rn(div12(v >= 0.0 ? 1.0 : e, d));
}

// the CUDA math library versions (reference for benchmarks/act_err.cu)
__device__ __forceinline__ float tanh_lib(float x) { return __double2float_rn(tanh((double)x)); }
__device__ __forceinline__ float sigmoid_lib(float x) {
    const double v = (double)x;
    if (v >= 0.0) return __double2float_rn(1.0 / (1.0 + exp(-v)));
    const double e = exp(v);
    return __double2float_rn(e / (1.0 + e));
}

// e^(2u) in f32 for |u| <= 20 (the one-MUFU attention scorer's E_u, attention.cu):
// x = 2u (exact), n = rint(x log2 e), r = x - n ln2 by two Cody-Waite FMAs
// (ln2_hi has 15 significant bits, so n * ln2_hi is exact for |n| <= 2^9), e^r
// by Taylor degree 7 on |r| <= 0.35 (truncation 5e-9 relative), 2^n added to the
// exponent.  No MUFU and no fp64.  Its relative error against e^(2u) is
// measured exhaustively over every f32 |u| <= 20 (benchmarks/att_exp_err.cu,
// profiles/r02_att_exp_err.json) and enters the scorer's rounding window.
__device__ __forceinline__ float exp2x_f32(float u) {
    const float x = 2.0f * u;
    const float n = rintf(x * 1.44269504088896341f);
    float r = fmaf(-n, 0.693145751953125f, x);        // ln2_hi = 0x3F317200
    r = fmaf(-n, 1.42860682030941723e-6f, r);         // ln2_lo
    float p = 1.98412698e-4f;                         // 1/7!
    p = fmaf(p, r, 1.38888889e-3f);
    p = fmaf(p, r, 8.33333333e-3f);
    p = fmaf(p, r, 4.16666667e-2f);
    p = fmaf(p, r, 1.66666667e-1f);
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    return __int_as_float(__float_as_int(p) + (int)((uint32_t)(int)n << 23));
}

}  // namespace qnmt
