// gemm_f32.cu -- the fp32 precision path's products.
//
//   Y[n][m] = fl32( sum_k f64(W[m][k]) * f64(X[n][k]) )  (+ bias[m])  (+ Y[n][m])
//
// Replaces qmath.py:434-440 (gemm_f32, numpy/OpenBLAS sgemm) as called by the
// fp32 branch of LinearOp.apply (layers.py:138-145) and, for the scorer, by
// attend (layers.py:224-226).  Tier-B contract: the product is
// evaluated in fp64 and rounded once to f32 -- every f32 x f32 product is exact
// in fp64, so the result is the correctly rounded dot product up to the fp64
// summation error, independent of summation order except within ~1e-13
// relative of an f32 rounding midpoint.  Bias and accumulation are separate
// f32 additions in the reference's order.
//
//   k_gemv_f32<NC> : N <= 8 (latency path): one warp per weight row, 16-byte
//                    L1-bypassing weight loads, fp64 warp reduction.  HBM-bound
//                    (4 bytes per weight -- the paper's point against fp32).
//   k_gemm_f32     : N > 8: 128 x 64 CTA tiles, 8 x 8 fp64 register tiles per
//                    thread (the shared-memory read rate of 16 B per 4 DFMA is
//                    what lets the DFMA pipe run), operands widened to fp64
//                    once when staged into shared memory.
#include "common.cuh"

namespace qnmt {

struct F32Epi {
    const float* bias;
    float* Y;
    int64_t ldy;
    int accumulate;
};

__device__ __forceinline__ void f32_store(const F32Epi& e, int64_t m, int64_t n, double acc) {
    float y = __double2float_rn(acc);
    if (e.bias) y = __fadd_rn(y, e.bias[m]);
    float* dst = e.Y + n * e.ldy + m;
    if (e.accumulate) y = __fadd_rn(*dst, y);
    *dst = y;
}

template <int NC>
__global__ void __launch_bounds__(256)
k_gemv_f32(const float* __restrict__ W, int64_t M, int64_t K, int64_t ldw, const float* __restrict__ X,
           int64_t ldx, F32Epi e, int vec) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    const int64_t m = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (m >= M) return;
    const float* w = W + m * ldw;
    double acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = 0.0;
    if (vec) {   // K % 4 == 0, 16-byte aligned rows
        for (int64_t k = 4 * lane; k < K; k += 128) {
            const int4 wi = ld_stream16(w + k);
            const float4 wv = make_float4(__int_as_float(wi.x), __int_as_float(wi.y), __int_as_float(wi.z),
                                          __int_as_float(wi.w));
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const float4 xv = __ldg(reinterpret_cast<const float4*>(X + j * ldx + k));
                acc[j] = fma((double)wv.x, (double)xv.x, acc[j]);
                acc[j] = fma((double)wv.y, (double)xv.y, acc[j]);
                acc[j] = fma((double)wv.z, (double)xv.z, acc[j]);
                acc[j] = fma((double)wv.w, (double)xv.w, acc[j]);
            }
        }
    } else {
        for (int64_t k = lane; k < K; k += 32) {
            const double wv = (double)w[k];
#pragma unroll
            for (int j = 0; j < NC; ++j) acc[j] = fma(wv, (double)__ldg(X + j * ldx + k), acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = warp_sum(acc[j]);
    if (lane < NC) {
        double a = acc[0];
#pragma unroll
        for (int j = 1; j < NC; ++j)
            if (lane == j) a = acc[j];
        f32_store(e, m, lane, a);
    }
}

constexpr int FBM = 128, FBN = 64, FBK = 8, FT = 128;

// Thread (tm, tn) = (tid % 16, tid / 16) owns rows {32 r + 2 tm + {0,1}} and
// columns {16 c + 2 tn + {0,1}}, r, c in 0..3: every 16-byte shared load of a
// fragment is conflict-free and the f32 stores of a warp are 128-byte runs.
__global__ void __launch_bounds__(FT)
k_gemm_f32(const float* __restrict__ W, int64_t M, int64_t K, int64_t ldw, const float* __restrict__ X, int64_t N,
           int64_t ldx, F32Epi e) {
    pdl_entry();
    __shared__ __align__(16) double sW[2][FBK][FBM];
    __shared__ __align__(16) double sX[2][FBK][FBN];
    const int tid = threadIdx.x;
    const int tm = tid & 15, tn = tid >> 4;
    const int64_t m0 = (int64_t)blockIdx.x * FBM, n0 = (int64_t)blockIdx.y * FBN;
    // staging: thread t loads W row m0 + t (8 k-values) and half a row of X (4 k-values)
    const int64_t wm = m0 + tid;
    const int64_t xn = n0 + (tid >> 1);
    const int xk = (tid & 1) * 4;
    float wr[FBK], xr[4];
    auto load = [&](int64_t k0) {
#pragma unroll
        for (int i = 0; i < FBK; ++i) wr[i] = (wm < M && k0 + i < K) ? __ldg(W + wm * ldw + k0 + i) : 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) xr[i] = (xn < N && k0 + xk + i < K) ? __ldg(X + xn * ldx + k0 + xk + i) : 0.0f;
    };
    auto stage = [&](int b) {
#pragma unroll
        for (int i = 0; i < FBK; ++i) sW[b][i][tid] = (double)wr[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) sX[b][xk + i][tid >> 1] = (double)xr[i];
    };
    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    load(0);
    stage(0);
    __syncthreads();
    int b = 0;
    for (int64_t k0 = 0; k0 < K; k0 += FBK) {
        const bool more = k0 + FBK < K;
        if (more) load(k0 + FBK);
#pragma unroll
        for (int k = 0; k < FBK; ++k) {
            double a[8], x[8];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double2 v = *reinterpret_cast<const double2*>(&sW[b][k][32 * r + 2 * tm]);
                a[2 * r] = v.x;
                a[2 * r + 1] = v.y;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const double2 v = *reinterpret_cast<const double2*>(&sX[b][k][16 * c + 2 * tn]);
                x[2 * c] = v.x;
                x[2 * c + 1] = v.y;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fma(a[i], x[j], acc[i][j]);
        }
        if (more) {
            stage(b ^ 1);
            __syncthreads();
            b ^= 1;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t n = n0 + 16 * (j >> 1) + 2 * tn + (j & 1);
        if (n >= N) continue;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t m = m0 + 32 * (i >> 1) + 2 * tm + (i & 1);
            if (m < M) f32_store(e, m, n, acc[i][j]);
        }
    }
}

int gemm_f32_launch(const float* W, int64_t M, int64_t K, int64_t ldw, const float* X, int64_t N, int64_t ldx,
                    const float* bias, float* Y, int64_t ldy, int32_t flags, cudaStream_t st) {
    if (M <= 0 || N <= 0) return QNMT_OK;
    F32Epi e{bias, Y, ldy, (flags & QNMT_GEMM_ACCUMULATE) ? 1 : 0};
    if (N <= 8) {
        const int vec = (K % 4 == 0 && ldw % 4 == 0 && ldx % 4 == 0 && ((uintptr_t)W % 16) == 0 &&
                         ((uintptr_t)X % 16) == 0) ? 1 : 0;
        const unsigned grid = (unsigned)cdiv(M, 8);
        switch (N) {
#define QNMT_GEMV_F32(NC_) \
    case NC_: QNMT_LAUNCH(k_gemv_f32<NC_>, grid, 256, 0, st, W, M, K, ldw, X, ldx, e, vec); break;
            QNMT_GEMV_F32(1) QNMT_GEMV_F32(2) QNMT_GEMV_F32(3) QNMT_GEMV_F32(4)
            QNMT_GEMV_F32(5) QNMT_GEMV_F32(6) QNMT_GEMV_F32(7) QNMT_GEMV_F32(8)
#undef QNMT_GEMV_F32
        }
        QNMT_CHECK_LAUNCH("k_gemv_f32");
        return QNMT_OK;
    }
    const dim3 grid((unsigned)cdiv(M, FBM), (unsigned)cdiv(N, FBN));
    QNMT_LAUNCH(k_gemm_f32, grid, FT, 0, st, W, M, K, ldw, X, N, ldx, e);
    QNMT_CHECK_LAUNCH("k_gemm_f32");
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" int qnmt_gemm_f32(const float* W, int64_t M, int64_t K, int64_t ldw, const float* X, int64_t N,
                             int64_t ldx, const float* bias, float* Y, int64_t ldy, int32_t flags, void* stream) {
    if (M < 0 || N < 0 || K < 0 || ldw < K || ldx < K || ldy < M) {
        qnmt::set_error("qnmt_gemm_f32: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N, (long long)K);
        return QNMT_ERR_SHAPE;
    }
    return qnmt::gemm_f32_launch(W, M, K, ldw, X, N, ldx, bias, Y, ldy, flags, qnmt::as_stream(stream));
}
