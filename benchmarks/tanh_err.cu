// tanh_err.cu -- exhaustive error of the MUFU-based tanh variants used by the
// attention score kernel, over every f32 x with 2^-24 <= |x| < 64 (both signs).
// The attention fast path needs a proven bound on |t_fast - tanh(x)| to size
// its "unsafe" rounding window (attention.cu, att_code_fast).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tanh_err.cu -o tanh_err
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2a(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpa(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

// variant 0: |x| form, 1 - 2 r, copysign (round-1 kernel)
// variant 1: signed x, r = rcp(1 + 2^(2x log2 e)), t = 1 - 2 r (exact in fp64 for the test)
// variant 2: variant 1 + one Newton step on r, argument clamped at 64
__global__ void k_err(uint32_t lo, uint32_t hi, unsigned long long* out) {
    double m0 = 0, m1 = 0, m2 = 0;
    for (uint32_t b = lo + blockIdx.x * blockDim.x + threadIdx.x; b < hi; b += gridDim.x * blockDim.x) {
        for (int sgn = 0; sgn < 2; ++sgn) {
            const float x = __uint_as_float(b | (sgn ? 0x80000000u : 0u));
            const double ref = tanh((double)x);
            {
                const float e = ex2a(fabsf(x) * 2.8853900817779268f);
                const float r = rcpa(e + 1.0f);
                const double t = copysign(1.0 - 2.0 * (double)r, (double)x);
                m0 = fmax(m0, fabs(t - ref));
            }
            {
                const float e = ex2a(x * 2.8853900817779268f);
                const float r = rcpa(e + 1.0f);
                m1 = fmax(m1, fabs(1.0 - 2.0 * (double)r - ref));
            }
            {
                const float e = ex2a(fminf(x * 2.8853900817779268f, 64.0f));
                const float y = e + 1.0f;
                float r = rcpa(y);
                r = fmaf(r, fmaf(-y, r, 1.0f), r);
                m2 = fmax(m2, fabs(1.0 - 2.0 * (double)r - ref));
            }
        }
    }
    atomicMax(out + 0, (unsigned long long)__double_as_longlong(m0));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(m1));
    atomicMax(out + 2, (unsigned long long)__double_as_longlong(m2));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 24);
    cudaMemset(d, 0, 24);
    const uint32_t lo = 0x33800000u;   // 2^-24
    const uint32_t hi = 0x42800000u;   // 64
    k_err<<<148 * 8, 256>>>(lo, hi, d);
    unsigned long long h[3];
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    const char* names[3] = {"abs_form", "signed", "signed_newton"};
    for (int i = 0; i < 3; ++i) {
        double v;
        memcpy(&v, &h[i], 8);
        printf("{\"variant\": \"%s\", \"max_abs_err\": %.6e, \"range\": \"2^-24 <= |x| < 64, all f32\"}\n", names[i], v);
    }
    return 0;
}
