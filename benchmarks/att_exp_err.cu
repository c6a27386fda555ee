// att_exp_err.cu -- error of the one-MUFU attention code fast path (attention.cu,
// k_att_score6), which evaluates
//     v_fast = fl(st - 2 st * rcp.approx(fl(E_ap * E_u + 1)))
// with E_ap = fl32(e^(2 ap)) (fp64 exp, rounded once) and E_u = exp2x_f32(u) (f32), against the
// reference's v = fl(fl32(tanh(fl32(ap + u))) * st)  (qmath.py:136-142, layers.py:225-226,
// Tier B: tanh in fp64 rounded once).
//
// (1) rcp.approx.ftz.f32: exhaustive relative error over every mantissa of [1, 2) at
//     several binades (the result's relative error only depends on the mantissa).
// (1b) exp2x_f32: exhaustive relative error against e^(2u) (fp64) over every f32 u with
//      |u| <= 20.
// (2) Monte-Carlo of |v_fast - v| over (ap, u, st) with |ap|, |u| <= 20 (the fast path's
//     eligibility bound), reported as the ratio to the analytic bound the kernel uses,
//     ATT_E_K1 * st + ATT_E_K2 (must stay < 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1804_05038_b200/csrc att_exp_err.cu -o att_exp_err
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "act.cuh"

using namespace qnmt;

__device__ __forceinline__ float rcpa(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void k_rcp(int binade, unsigned long long* out) {
    double m = 0;
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < (1u << 23); b += gridDim.x * blockDim.x) {
        const float d = __uint_as_float(((uint32_t)(127 + binade) << 23) | b);
        const double rel = fabs((double)rcpa(d) * (double)d - 1.0);
        m = fmax(m, rel);
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// every f32 bit pattern b in [lo, hi) (positive and negative), |u| <= 20
__global__ void k_exp2x(uint32_t lo, uint32_t hi, unsigned long long* out) {
    double m = 0;
    for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b < hi; b += gridDim.x * blockDim.x) {
        for (int sgn = 0; sgn < 2; ++sgn) {
            const float u = __uint_as_float(b | (sgn ? 0x80000000u : 0u));
            if (!(fabsf(u) <= 20.0f)) continue;
            const double ex = exp(2.0 * (double)u);
            m = fmax(m, fabs((double)exp2x_f32(u) / ex - 1.0));
        }
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ float unif(uint32_t h) { return (h >> 8) * (1.0f / 16777216.0f); }

// analytic bound used by the kernel (attention.cu, att_e_threshold): K1 * st + K2
constexpr double K1 = 5.5e-7, K2 = 9.5e-6;

__global__ void k_mc(uint64_t n, int dist, unsigned long long* out) {
    double worst = 0, worst_abs = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t h1 = hash32((uint32_t)i * 3u + 1u + (uint32_t)(i >> 32) * 0x9e3779b9u);
        const uint32_t h2 = hash32(h1 ^ 0x68bc21ebu), h3 = hash32(h2 ^ 0x02e5be93u), h4 = hash32(h3 + 77u);
        float ap, u;
        if (dist == 0) {          // uniform in [-20, 20]
            ap = 40.0f * unif(h1) - 20.0f;
            u = 40.0f * unif(h2) - 20.0f;
        } else if (dist == 1) {   // typical magnitudes (|x| ~ 0..4)
            ap = 8.0f * unif(h1) - 4.0f;
            u = 8.0f * unif(h2) - 4.0f;
        } else {                  // log-uniform magnitudes 2^-20 .. 20, random signs, near-cancelling pairs
            const float ma = exp2f(-20.0f + 24.3f * unif(h1));
            ap = (h3 & 1) ? ma : -ma;
            u = -ap + ((h3 & 2) ? 1.0f : -1.0f) * exp2f(-12.0f + 14.0f * unif(h2));
            u = fminf(fmaxf(u, -20.0f), 20.0f);
        }
        // st = 127 / tmax for tmax in (1e-4, 1]
        const float tmax = fmaxf(1e-4f, unif(h4));
        const float st = __fdiv_rn(127.0f, tmax);
        const float eap = __double2float_rn(exp_f64(2.0 * (double)ap));
        const float eu = exp2x_f32(u);
        const float r = rcpa(fmaf(eap, eu, 1.0f));
        const float vf = fmaf(-2.0f * st, r, st);
        const float t = tanh_b(__fadd_rn(ap, u));
        const float v = __fmul_rn(t, st);
        const double e = fabs((double)vf - (double)v);
        worst = fmax(worst, e / (K1 * st + K2));
        worst_abs = fmax(worst_abs, e);
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(worst));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(worst_abs));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    printf("{\"rcp_approx_ftz_f32_rel_err\": {");
    const int binades[] = {0, -60, -20, 20, 60};
    for (int k = 0; k < 5; ++k) {
        cudaMemset(d, 0, 8);
        k_rcp<<<148 * 8, 256>>>(binades[k], d);
        unsigned long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        double v;
        memcpy(&v, &h, 8);
        printf("%s\"2^%d\": %.6e", k ? ", " : "", binades[k], v);
    }
    {
        cudaMemset(d, 0, 8);
        k_exp2x<<<148 * 16, 256>>>(0u, 0x41a00001u, d);   // |u| <= 20 (0x41a00000 = 20.0f)
        unsigned long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        double v;
        memcpy(&v, &h, 8);
        printf("}, \"exp2x_f32_rel_err_exhaustive_abs_u_le_20\": %.6e", v);
    }
    printf(", \"fast_path_mc\": {\"bound\": \"%.3e * st + %.3e\"", K1, K2);
    const char* names[3] = {"uniform20", "uniform4", "cancelling_logmag"};
    for (int dist = 0; dist < 3; ++dist) {
        cudaMemset(d, 0, 16);
        const uint64_t n = 1ull << 33;
        k_mc<<<148 * 16, 256>>>(n, dist, d);
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        double w, wa;
        memcpy(&w, &h[0], 8);
        memcpy(&wa, &h[1], 8);
        printf(", \"%s\": {\"samples\": %llu, \"max_err_over_bound\": %.4f, \"max_abs_err\": %.4e}", names[dist],
               (unsigned long long)n, w, wa);
    }
    printf("}}\n");
    cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : 1;
}
