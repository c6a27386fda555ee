// act_err.cu -- exhaustive comparison of the fp64 activations in act.cuh
// (sigmoid_b, tanh_b) against the CUDA math library versions, over every
// finite f32 input: counts of differing f32 results and the first few inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../include act_err.cu -o act_err
#include <cstdio>
#include <cstdint>
#include <cstring>

#include "../paper_1804_05038_b200/csrc/act.cuh"

__global__ void k_cmp(unsigned long long* cnt, uint32_t* first) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (1ull << 32); b += stride) {
        const float x = __uint_as_float((uint32_t)b);
        if (!isfinite(x)) continue;
        atomicAdd(&cnt[2], 1ull);
        if (__float_as_uint(qnmt::sigmoid_b(x)) != __float_as_uint(qnmt::sigmoid_lib(x))) {
            const unsigned long long i = atomicAdd(&cnt[0], 1ull);
            if (i < 8) first[i] = (uint32_t)b;
        }
        if (__float_as_uint(qnmt::tanh_b(x)) != __float_as_uint(qnmt::tanh_lib(x))) {
            const unsigned long long i = atomicAdd(&cnt[1], 1ull);
            if (i < 8) first[8 + i] = (uint32_t)b;
        }
    }
}

int main() {
    unsigned long long* cnt;
    uint32_t* first;
    cudaMalloc(&cnt, 24);
    cudaMalloc(&first, 64);
    cudaMemset(cnt, 0, 24);
    cudaMemset(first, 0, 64);
    k_cmp<<<148 * 16, 256>>>(cnt, first);
    unsigned long long h[3];
    uint32_t f[16];
    cudaMemcpy(h, cnt, 24, cudaMemcpyDeviceToHost);
    printf("{\"evaluated_inputs\": %llu}\n", h[2]);
    cudaMemcpy(f, first, 64, cudaMemcpyDeviceToHost);
    const char* names[2] = {"sigmoid", "tanh"};
    for (int k = 0; k < 2; ++k) {
        printf("{\"function\": \"%s\", \"inputs\": \"all finite f32\", \"mismatches_vs_cuda_libm\": %llu, \"first\": [",
               names[k], h[k]);
        for (int i = 0; i < 8 && i < (int)h[k]; ++i) {
            float x;
            memcpy(&x, &f[8 * k + i], 4);
            printf("%s%.9g", i ? ", " : "", x);
        }
        printf("]}\n");
    }
    return 0;
}
