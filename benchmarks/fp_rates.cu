// fp_rates.cu -- measured arithmetic rates on this GPU (design input for the
// fp64 epilogues).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_ffma(float* out, int iters) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float b = 0.999999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
        a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_exp64(double* out, int iters) {
    double s = 0, x = -(threadIdx.x & 63) * 0.01;
    for (int i = 0; i < iters; ++i) { s += exp(x); x -= 1e-6; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_tanh64(double* out, int iters) {
    double s = 0, x = (threadIdx.x & 63) * 0.01;
    for (int i = 0; i < iters; ++i) { s += tanh(x); x += 1e-6; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_tanh32(float* out, int iters) {
    float s = 0, x = (threadIdx.x & 63) * 0.01f;
    for (int i = 0; i < iters; ++i) { s += tanhf(x); x += 1e-6f; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_cvt(double* out, int iters) {
    double s = 0;
    int a = threadIdx.x;
    for (int i = 0; i < iters; ++i) { s += (double)(a + i) * 1.0000001; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K, typename T>
void run(const char* name, K kern, T* buf, int iters, double ops_per_iter) {
    int blocks = 148 * 8, threads = 256;
    kern<<<blocks, threads>>>(buf, 16);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(buf, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double n = (double)blocks * threads * iters * ops_per_iter;
    printf("{\"op\": \"%s\", \"G_per_s\": %.1f, \"per_clk_per_sm_at_1.965GHz\": %.2f}\n", name, n / ms / 1e6,
           n / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
    double* d;
    float* f;
    cudaMalloc(&d, 148 * 8 * 256 * 8);
    cudaMalloc(&f, 148 * 8 * 256 * 4);
    run("dfma (fp64 FMA)", k_dfma, d, 4096, 8);
    run("ffma (fp32 FMA)", k_ffma, f, 4096, 8);
    run("exp(double)", k_exp64, d, 1024, 1);
    run("tanh(double)", k_tanh64, d, 1024, 1);
    run("tanhf(float)", k_tanh32, f, 1024, 1);
    run("i2f.f64 + dmul + dadd", k_cvt, d, 4096, 1);
    return 0;
}
