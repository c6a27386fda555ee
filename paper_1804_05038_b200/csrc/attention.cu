// attention.cu -- Bahdanau attention step (layers.py:214-241).
//
// For query column n of sentence s (length l, encoder rows R = sent_row[s]):
//   x[a,i]   = fl32(att_proj[R+i][a] + u[n][a])                (f32 add, :225)
//   t        = tanh(x)  (fp64, rounded)                          (:225)
//   scale_n  = fl32(127 / max_{a,i} |t|)  -- ONE scale over the whole [A, l]
//              block of this hypothesis (LinearOp.apply on t, :226)
//   score_i  = fl32(f64(sum_a v_a * q(t[a,i])) / (f64 s_v * f64 scale_n))
//   alpha    = softmax_i(score) in fp64, rounded                 (:230)
//   ctx[c]   = fl32(sum_i f64(states[R+i][c]) * f64(alpha_i))    (:237)
//
// max|t| is obtained without evaluating tanh in the first pass: |tanh| is odd
// and monotone, and so is "evaluate in fp64 then round", hence
// max_{a,i} |fl32(tanh(x))| = fl32(tanh(max_{a,i} |x|)).  Pass 1 is thus a
// pure f32 add/abs/max sweep; only pass 2 evaluates the A*l tanh values.
#include "common.cuh"

namespace qnmt {

constexpr int ATT_PC = 4;     // positions per CTA in the max / score passes
constexpr int ATT_T = 256;

template <bool VEC>
__global__ void __launch_bounds__(ATT_T)
k_att_max(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ col_sent,
          const float* __restrict__ att_proj, const int64_t* __restrict__ sent_row,
          const int32_t* __restrict__ sent_len, int64_t A, uint32_t* maxbits, int32_t* err_flag,
          const int32_t* n_dev) {
    int64_t n = blockIdx.y;
    if (beyond(n_dev, n)) return;
    int s = col_sent[n];
    int l = sent_len[s];
    int i0 = blockIdx.x * ATT_PC;
    if (i0 >= l) return;
    int i1 = min(l, i0 + ATT_PC);
    const float* ap = att_proj + sent_row[s] * A;
    const float* un = u + n * ldu;
    uint32_t m = 0;
    for (int i = i0; i < i1; ++i) {
        const float* row = ap + (int64_t)i * A;
        if (VEC) {
            for (int64_t a = 4 * threadIdx.x; a < A; a += 4 * ATT_T) {
                float4 x = *reinterpret_cast<const float4*>(row + a);
                float4 y = *reinterpret_cast<const float4*>(un + a);
                m = max(m, __float_as_uint(__fadd_rn(x.x, y.x)) & 0x7fffffffu);
                m = max(m, __float_as_uint(__fadd_rn(x.y, y.y)) & 0x7fffffffu);
                m = max(m, __float_as_uint(__fadd_rn(x.z, y.z)) & 0x7fffffffu);
                m = max(m, __float_as_uint(__fadd_rn(x.w, y.w)) & 0x7fffffffu);
            }
        } else {
            for (int64_t a = threadIdx.x; a < A; a += ATT_T)
                m = max(m, __float_as_uint(__fadd_rn(row[a], un[a])) & 0x7fffffffu);
        }
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0 && m) {
        if (m >= 0x7f800000u) set_flag(err_flag, QNMT_FLAG_NUMERIC);
        atomicMax(maxbits + n, m);
    }
}

template <bool VEC>
__global__ void __launch_bounds__(ATT_T)
k_att_score(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ col_sent,
            const float* __restrict__ att_proj, const int64_t* __restrict__ sent_row,
            const int32_t* __restrict__ sent_len, int64_t A, const int8_t* __restrict__ v_codes,
            const float* __restrict__ v_scale, const uint32_t* __restrict__ maxbits,
            float* __restrict__ scores, int32_t max_len, const int32_t* n_dev) {
    int64_t n = blockIdx.y;
    if (beyond(n_dev, n)) return;
    int s = col_sent[n];
    int l = sent_len[s];
    int i0 = blockIdx.x * ATT_PC;
    if (i0 >= l) return;
    int i1 = min(l, i0 + ATT_PC);
    uint32_t mb = maxbits[n];
    if (mb >= 0x7f800000u) mb = 0;
    float tmax = tanh_b(__uint_as_float(mb));
    float st = (tmax == 0.0f) ? 1.0f : __fdiv_rn(127.0f, tmax);
    const float* ap = att_proj + sent_row[s] * A;
    const float* un = u + n * ldu;
    int acc[ATT_PC] = {};
    if (!VEC) {
        for (int64_t a = threadIdx.x; a < A; a += ATT_T) {
            float y = un[a];
            int v = v_codes[a];
#pragma unroll
            for (int p = 0; p < ATT_PC; ++p) {
                int i = i0 + p;
                if (i < i1) acc[p] += v * quant_code(tanh_b(__fadd_rn(ap[(int64_t)i * A + a], y)), st);
            }
        }
    }
    for (int64_t a = 4 * threadIdx.x; VEC && a < A; a += 4 * ATT_T) {
        float4 y = *reinterpret_cast<const float4*>(un + a);
        char4 v = *reinterpret_cast<const char4*>(v_codes + a);
#pragma unroll
        for (int p = 0; p < ATT_PC; ++p) {
            int i = i0 + p;
            if (i < i1) {
                float4 x = *reinterpret_cast<const float4*>(ap + (int64_t)i * A + a);
                int c0 = quant_code(tanh_b(__fadd_rn(x.x, y.x)), st);
                int c1 = quant_code(tanh_b(__fadd_rn(x.y, y.y)), st);
                int c2 = quant_code(tanh_b(__fadd_rn(x.z, y.z)), st);
                int c3 = quant_code(tanh_b(__fadd_rn(x.w, y.w)), st);
                acc[p] += c0 * (int)v.x + c1 * (int)v.y + c2 * (int)v.z + c3 * (int)v.w;
            }
        }
    }
    __shared__ int red[ATT_PC][ATT_T / 32];
#pragma unroll
    for (int p = 0; p < ATT_PC; ++p) {
        int t = warp_sum(acc[p]);
        if ((threadIdx.x & 31) == 0) red[p][threadIdx.x >> 5] = t;
    }
    __syncthreads();
    if (threadIdx.x < ATT_PC) {
        int p = threadIdx.x;
        int i = i0 + p;
        if (i < i1) {
            long long t = 0;
            for (int w = 0; w < ATT_T / 32; ++w) t += red[p][w];
            scores[n * max_len + i] = dequant(t, v_scale[0], st);
        }
    }
}

// softmax over the l scores of column n (fp64, fixed sequential sum order) and
// the context sum for a 256-wide slice of the 2H state features.
__global__ void __launch_bounds__(256)
k_att_context(const float* __restrict__ scores, int32_t max_len, const int32_t* __restrict__ col_sent,
              const float* __restrict__ states, const int64_t* __restrict__ sent_row,
              const int32_t* __restrict__ sent_len, int64_t H2, float* __restrict__ ctx, int64_t ldc,
              float* __restrict__ alpha, int64_t lda, int32_t* err_flag, const int32_t* n_dev) {
    extern __shared__ unsigned char smem_raw[];
    double* e = reinterpret_cast<double*>(smem_raw);          // [max_len]
    float* al = reinterpret_cast<float*>(e + max_len);         // [max_len]
    __shared__ double s_sum;
    __shared__ float s_max;
    int64_t n = blockIdx.y;
    if (beyond(n_dev, n)) return;
    int s = col_sent[n];
    int l = sent_len[s];
    const float* sc = scores + n * max_len;
    if (threadIdx.x == 0) {
        float m = sc[0];
        bool bad = !is_finite_f(m);
        for (int i = 1; i < l; ++i) {
            bad |= !is_finite_f(sc[i]);
            m = fmaxf(m, sc[i]);
        }
        if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
        s_max = m;
    }
    __syncthreads();
    double mx = (double)s_max;
    for (int i = threadIdx.x; i < l; i += blockDim.x) e[i] = exp((double)sc[i] - mx);
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < l; ++i) t += e[i];
        s_sum = t;
    }
    __syncthreads();
    double sum = s_sum;
    for (int i = threadIdx.x; i < l; i += blockDim.x) {
        float a = __double2float_rn(e[i] / sum);
        al[i] = a;
        if (alpha && blockIdx.x == 0) alpha[n * lda + i] = a;
    }
    __syncthreads();
    const float* st = states + sent_row[s] * H2;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < H2; c += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int i = 0; i < l; ++i) acc += (double)st[(int64_t)i * H2 + c] * (double)al[i];
        ctx[n * ldc + c] = __double2float_rn(acc);
    }
}

int attention_launch(const float* u, int64_t ldu, int64_t N, const int32_t* col_sent,
                     const float* att_proj, const float* states, const int64_t* sent_row,
                     const int32_t* sent_len, int32_t max_len, int64_t A, int64_t H2,
                     const int8_t* v_codes, const float* v_scale, float* ctx, int64_t ldc,
                     float* alpha, int64_t lda, void* scratch, int32_t* err_flag, cudaStream_t st) {
    if (N <= 0) return QNMT_OK;
    bool vec = (A % 4 == 0) && (ldu % 4 == 0) && ((uintptr_t)u % 16 == 0) &&
               ((uintptr_t)att_proj % 16 == 0) && ((uintptr_t)v_codes % 4 == 0);
    uint32_t* maxbits = reinterpret_cast<uint32_t*>(scratch);
    float* scores = reinterpret_cast<float*>(maxbits + ((N + 3) / 4) * 4);
    QNMT_CUDA(cudaMemsetAsync(maxbits, 0, sizeof(uint32_t) * (size_t)N, st));
    dim3 g1((unsigned)cdiv(max_len, ATT_PC), (unsigned)N);
    if (vec)
        k_att_max<true><<<g1, ATT_T, 0, st>>>(u, ldu, col_sent, att_proj, sent_row, sent_len, A, maxbits, err_flag, tl_ndev);
    else
        k_att_max<false><<<g1, ATT_T, 0, st>>>(u, ldu, col_sent, att_proj, sent_row, sent_len, A, maxbits, err_flag, tl_ndev);
    QNMT_CHECK_LAUNCH("k_att_max");
    if (vec)
        k_att_score<true><<<g1, ATT_T, 0, st>>>(u, ldu, col_sent, att_proj, sent_row, sent_len, A, v_codes,
                                               v_scale, maxbits, scores, max_len, tl_ndev);
    else
        k_att_score<false><<<g1, ATT_T, 0, st>>>(u, ldu, col_sent, att_proj, sent_row, sent_len, A, v_codes,
                                                v_scale, maxbits, scores, max_len, tl_ndev);
    QNMT_CHECK_LAUNCH("k_att_score");
    int64_t gx = cdiv(H2, 256);
    size_t smem = (size_t)max_len * (sizeof(double) + sizeof(float));
    if (smem > 48 * 1024) {
        QNMT_CUDA(cudaFuncSetAttribute(k_att_context, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    k_att_context<<<dim3((unsigned)gx, (unsigned)N), 256, smem, st>>>(
        scores, max_len, col_sent, states, sent_row, sent_len, H2, ctx, ldc, alpha, lda, err_flag, tl_ndev);
    QNMT_CHECK_LAUNCH("k_att_context");
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" int qnmt_attention(const float* u, int64_t ldu, int64_t N, const int32_t* col_sent,
                              const float* att_proj, const float* states, const int64_t* sent_row,
                              const int32_t* sent_len, int32_t max_len, int64_t A, int64_t H2,
                              const int8_t* v_codes, const float* v_scale, float* ctx, int64_t ldc,
                              float* alpha, int64_t lda, void* scratch, int32_t* err_flag,
                              void* stream) {
    return qnmt::attention_launch(u, ldu, N, col_sent, att_proj, states, sent_row, sent_len, max_len,
                                  A, H2, v_codes, v_scale, ctx, ldc, alpha, lda, scratch, err_flag,
                                  qnmt::as_stream(stream));
}
