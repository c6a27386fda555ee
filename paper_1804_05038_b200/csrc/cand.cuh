// cand.cuh -- beam-candidate lists, block reductions and the fp64 exp used by
// the log-softmax / top-k kernels (output.cu, vocab_topk.cu).
#pragma once
#include <float.h>

#include "common.cuh"

namespace qnmt {

constexpr int LS_T = 512;   // threads of the per-row softmax / candidate kernels

struct Cand {
    double s;
    int t;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
    return a.s > b.s || (a.s == b.s && a.t < b.t);
}

// block-wide reductions (LS_T threads)
__device__ __forceinline__ float block_max_f(float v, float* red) {
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = threadIdx.x < LS_T / 32 ? red[threadIdx.x] : -FLT_MAX;
        t = warp_max(t);
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    float r = red[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ double block_sum_d(double v, double* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < LS_T / 32 ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    double r = red[0];
    __syncthreads();
    return r;
}

template <int KM>
__device__ __forceinline__ void insert(Cand (&L)[KM], Cand c) {
    if (!better(c, L[KM - 1])) return;
    L[KM - 1] = c;
#pragma unroll
    for (int i = KM - 1; i > 0; --i) {
        if (better(L[i], L[i - 1])) {
            Cand t = L[i];
            L[i] = L[i - 1];
            L[i - 1] = t;
        }
    }
}

// warp-cooperative k-way merge of 32 sorted per-lane lists; result in lane 0..k-1 order
template <int KM>
__device__ void warp_merge(Cand (&L)[KM], Cand* out, int k) {
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < k; ++r) {
        Cand b = L[0];
        int bl = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            double os = __shfl_xor_sync(0xffffffffu, b.s, o);
            int ot = __shfl_xor_sync(0xffffffffu, b.t, o);
            int ol = __shfl_xor_sync(0xffffffffu, bl, o);
            Cand oc{os, ot};
            if (better(oc, b) || (!better(b, oc) && ol < bl)) {
                b = oc;
                bl = ol;
            }
        }
        if (lane == 0) out[r] = b;
        if (lane == bl) {
#pragma unroll
            for (int i = 0; i < KM - 1; ++i) L[i] = L[i + 1];
            L[KM - 1] = Cand{-DBL_MAX, 0x7fffffff};
        }
    }
}

// exp(t) for t <= 0 in fp64 (~2 ulp): t = k*ln2/16 + r, |r| <= ln2/32,
// e^r by a degree-7 polynomial (truncation < 1.3e-18), 2^(k/16) = 2^(k>>4) * tab[k&15].
// The 16-entry f64 table is 128 B = all 32 smem banks, so lookups never
// conflict.  ~13 f64 ops instead of the general-purpose exp() (~27 DFMA slots).
__device__ __forceinline__ double exp_neg(double t, const double* __restrict__ tab) {
    t = fmax(t, -700.0);   // below: contributes < 1e-304 (branch-free range guard)
    // round(t * 16/ln2) without FRND/F2I: add 1.5*2^52 so the integer lands in the low word
    const double kd_m = fma(t, 23.083120654223414, 6755399441055744.0);
    const int k = __double2loint(kd_m);
    const double kd = kd_m - 6755399441055744.0;
    double r = fma(kd, -0.04332169878499658, t);             // ln2/16, rounded to f64
    r = fma(kd, -1.4494042586539372e-18, r);                 // ln2/16 - the above
    double p = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    double v = p * tab[k & 15];
    // multiply by 2^(k >> 4) through the exponent field (result stays normal for t >= -700)
    long long bits = __double_as_longlong(v) + ((long long)(k >> 4) << 52);
    return __longlong_as_double(bits);
}

// Same function with a 64-entry table (2^(j/64), 512 B of smem) and |r| <= ln2/128,
// so a degree-5 polynomial suffices (truncation < 3.5e-17): 12 f64 ops.  No range
// guard: the caller guarantees t >= -700 (result stays normal).
__device__ __forceinline__ double exp_neg64(double t, const double* __restrict__ tab64) {
    const double kd_m = fma(t, 92.33248261689366, 6755399441055744.0);    // t * 64/ln2 + 1.5*2^52
    const int k = __double2loint(kd_m);
    const double kd = kd_m - 6755399441055744.0;
    double r = fma(kd, -0.010830424696249145, t);                          // ln2/64, rounded to f64
    r = fma(kd, -3.623510646634843e-19, r);                                // ln2/64 - the above
    double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const double v = p * tab64[k & 63];
    // * 2^(k >> 6): shift then shift-add (SHF + LEA) rather than the compiler's
    // shift / mask / add form of (k >> 6) << 20
    int kk;
    asm("shr.s32 %0, %1, 6;" : "=r"(kk) : "r"(k));
    return __hiloint2double(__double2hiint(v) + kk * (1 << 20), __double2loint(v));
}

// acc + exp_neg64(t) with the 2^(k >> 6) scaling applied to the table entry (exact: a
// power of two, result normal for t >= -700) so the final multiply and the add fuse into
// one DFMA (one rounding instead of two)
__device__ __forceinline__ double exp_neg64_acc(double t, const double* __restrict__ tab64, double acc) {
    const double kd_m = fma(t, 92.33248261689366, 6755399441055744.0);    // t * 64/ln2 + 1.5*2^52
    const int k = __double2loint(kd_m);
    const double kd = kd_m - 6755399441055744.0;
    double r = fma(kd, -0.010830424696249145, t);
    r = fma(kd, -3.623510646634843e-19, r);
    double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const double tb = tab64[k & 63];
    int kk;
    asm("shr.s32 %0, %1, 6;" : "=r"(kk) : "r"(k));
    const double ts = __hiloint2double(__double2hiint(tb) + kk * (1 << 20), __double2loint(tb));
    return fma(p, ts, acc);
}

template <int KM>
__device__ void block_merge_cands(Cand (&L)[KM], Cand (*wl)[KM], Cand* out, int kk) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    warp_merge<KM>(L, wl[warp], kk);
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < KM; ++i) L[i] = (lane < LS_T / 32 && i < kk) ? wl[lane][i] : Cand{-DBL_MAX, 0x7fffffff};
        __syncwarp();
        Cand tmp[KM];
        warp_merge<KM>(L, tmp, kk);
        if (lane == 0)
            for (int i = 0; i < kk; ++i) out[i] = tmp[i];
    }
    __syncthreads();
}

}  // namespace qnmt
