// attention.cu -- Bahdanau attention step (layers.py:214-241), batched by sentence.
//
// For hypothesis column n of sentence s (length l, encoder rows R = sent_row[s]):
//   x[a,i]   = fl32(att_proj[R+i][a] + u[n][a])                (f32 add, :225)
//   t        = tanh(x)  (fp64-exact, rounded once)              (:225)
//   scale_n  = fl32(127 / max_{a,i} |t|)  -- ONE scale over the whole [A, l]
//              block of this hypothesis (LinearOp.apply on t, :226)
//   score_i  = fl32(f64(sum_a v_a * q(t[a,i])) / (f64 s_v * f64 scale_n))
//   alpha    = softmax_i(score) in fp64, rounded                 (:230)
//   ctx[c]   = fl32(sum_i f64(states[R+i][c]) * f64(alpha_i))    (:237)
//
// Layout for the batched decoder: the columns of sentence s are
// [sent_col_off[s], sent_col_off[s] + sent_ncols[s]).  Every CTA works on one
// sentence and ALL its live hypotheses, so att_proj and states rows are read
// once per sentence per step instead of once per hypothesis.
//
// max|t| needs no tanh: |tanh| is odd and monotone, and so is "evaluate in
// fp64, round once", hence max_{a,i} |fl32(tanh(x))| = fl32(tanh(max |x|)).
// Codes q(t) use an f32 fast path: tanhf (<= 2 ulp) gives v = t*scale within a
// few ulps of the exact product; the code floor(|v| + 1/2) can only differ if
// |v| is within ~2.5e-4 of a half-integer (>30 ulps of margin at |v| <= 127.5),
// and only those elements are recomputed with the fp64-exact tanh.
#include <algorithm>

#include "kernels.cuh"

#define TRY_LAUNCH(x) do { int _r = (x); if (_r != QNMT_OK) return _r; } while (0)

namespace qnmt {

constexpr int AT = 256;        // threads per CTA
constexpr int APC = 4;         // encoder positions per CTA (max / score passes)
constexpr int AMAXP = 16;      // max live hypotheses per sentence (beam <= 16)
constexpr int AKA = 8;         // a-elements per thread kept in registers (A <= AT * AKA)

// Fast code of t = tanh(x) at scale st.  Returns the code from tanhf (<= 2 ulp)
// and sets `unsafe` when fl(|v| + 1/2) is within 2.5e-4 of an integer, where
// the exact fp64 tanh could give a different floor (att_code_exact).
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// tanh with absolute error < ~1.2e-6 from two MUFU ops: 1 - 2 / (1 + e^{2|x|})
__device__ __forceinline__ float tanh_fast(float x) {
    const float e = ex2_approx(fabsf(x) * 2.8853900817779268f);   // 2 / ln 2
    const float r = rcp_approx(e + 1.0f);
    return copysignf(fmaf(-2.0f, r, 1.0f), x);
}

// win = max(4e-4, st * 2e-6) bounds |v_fast - v_exact| (+ rounding) with margin.
// No XU-pipe ops besides the two MUFU: floor(|v| + 1/2) equals round-to-nearest-
// even(|v|) except at exact ties |v| = k + 1/2, which lie inside the unsafe window
// (handled exactly); the rounding uses the 1.5*2^23 magic add, whose low mantissa
// bits are the integer code.
__device__ __forceinline__ int att_code_fast(float x, float st, float win, bool& unsafe) {
    const float v = __fmul_rn(tanh_fast(x), st);
    const float av = fminf(fabsf(v), 127.0f);
    const float m = __fadd_rn(av, 12582912.0f);            // 1.5 * 2^23
    const float d = __fsub_rn(av, __fsub_rn(m, 12582912.0f));   // av - rint(av), exact
    unsafe = fabsf(d) > 0.5f - win;
    const int q = __float_as_int(m) - 0x4B400000;
    return v < 0.0f ? -q : q;
}
__device__ __noinline__ int att_code_exact(float x, float st) { return quant_code(tanh_b(x), st); }

// load this thread's strided slice of APC att_proj rows (a = tid + AT*k)
__device__ __forceinline__ void load_ap(const float* __restrict__ ap, int64_t A, int i0, int i1,
                                        float (&apv)[APC][AKA]) {
#pragma unroll
    for (int p = 0; p < APC; ++p)
#pragma unroll
        for (int k = 0; k < AKA; ++k) {
            const int64_t a = threadIdx.x + (int64_t)AT * k;
            apv[p][k] = (i0 + p < i1 && a < A) ? ap[(int64_t)(i0 + p) * A + a] : 0.0f;
        }
}

// Per-sentence column extrema of att_proj: mm[s][0][a] = max_i, mm[s][1][a] = min_i.
// Since x -> |fl32(x + u)| restricted to a set of x is maximised at the set's
// max or min (f32 addition is monotone), the per-hypothesis scale needs only
// max_a max(|fl(mx_a + u_a)|, |fl(mn_a + u_a)|): 2*A adds instead of A*l.
__global__ void __launch_bounds__(AT)
k_att_minmax(const float* __restrict__ att_proj, const int64_t* __restrict__ sent_row,
             const int32_t* __restrict__ sent_len, int64_t A, float* __restrict__ mm) {
    const int s = blockIdx.y;
    const int64_t a = (int64_t)blockIdx.x * AT + threadIdx.x;
    if (a >= A) return;
    const int l = sent_len[s];
    const float* ap = att_proj + sent_row[s] * A + a;
    float mx = ap[0], mn = ap[0];
    for (int i = 1; i < l; ++i) {
        const float x = ap[(int64_t)i * A];
        mx = fmaxf(mx, x);
        mn = fminf(mn, x);
    }
    mm[((int64_t)s * 2) * A + a] = mx;
    mm[((int64_t)s * 2 + 1) * A + a] = mn;
}

int att_minmax_launch(const float* att_proj, const int64_t* sent_row, const int32_t* sent_len, int32_t n_sent,
                      int64_t A, float* mm, cudaStream_t st) {
    if (n_sent <= 0) return QNMT_OK;
    k_att_minmax<<<dim3((unsigned)cdiv(A, AT), (unsigned)n_sent), AT, 0, st>>>(att_proj, sent_row, sent_len, A, mm);
    QNMT_CHECK_LAUNCH("k_att_minmax");
    return QNMT_OK;
}

__global__ void __launch_bounds__(AT)
k_att_score3(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ sent_col_off,
             const int32_t* __restrict__ sent_ncols, const float* __restrict__ att_proj,
             const float* __restrict__ mm, const int64_t* __restrict__ sent_row,
             const int32_t* __restrict__ sent_len, int64_t A, const int8_t* __restrict__ v_codes,
             const float* __restrict__ v_scale, float* __restrict__ scores, int32_t max_len, int32_t* err_flag) {
    __shared__ int red[AMAXP][APC][AT / 32];
    __shared__ uint32_t mred[AMAXP][AT / 32];
    __shared__ float s_st[AMAXP];
    const int s = blockIdx.y;
    const int P = sent_ncols[s];
    const int l = sent_len[s];
    const int i0 = blockIdx.x * APC;
    if (P == 0 || i0 >= l) return;
    const int i1 = min(l, i0 + APC);
    const int c0 = sent_col_off[s];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per-hypothesis scale of the whole [A, l] block (layers.py:226) from the column extrema
    {
        float mxv[AKA], mnv[AKA];
#pragma unroll
        for (int k = 0; k < AKA; ++k) {
            const int64_t a = threadIdx.x + (int64_t)AT * k;
            mxv[k] = a < A ? mm[((int64_t)s * 2) * A + a] : 0.0f;
            mnv[k] = a < A ? mm[((int64_t)s * 2 + 1) * A + a] : 0.0f;
        }
        for (int j = 0; j < P; ++j) {
            const float* un = u + (int64_t)(c0 + j) * ldu;
            uint32_t m = 0;
#pragma unroll
            for (int k = 0; k < AKA; ++k) {
                const int64_t a = threadIdx.x + (int64_t)AT * k;
                if (a < A) {
                    const float uv = un[a];
                    m = max(m, __float_as_uint(__fadd_rn(mxv[k], uv)) & 0x7fffffffu);
                    m = max(m, __float_as_uint(__fadd_rn(mnv[k], uv)) & 0x7fffffffu);
                }
            }
            m = warp_max(m);
            if (lane == 0) mred[j][warp] = m;
        }
        __syncthreads();
        if (threadIdx.x < P) {
            uint32_t m = 0;
            for (int w = 0; w < AT / 32; ++w) m = max(m, mred[threadIdx.x][w]);
            if (m >= 0x7f800000u) {
                set_flag(err_flag, QNMT_FLAG_NUMERIC);
                m = 0;
            }
            const float tmax = tanh_b(__uint_as_float(m));
            s_st[threadIdx.x] = (tmax == 0.0f) ? 1.0f : __fdiv_rn(127.0f, tmax);
        }
        __syncthreads();
    }
    float apv[APC][AKA];
    load_ap(att_proj + sent_row[s] * A, A, i0, i1, apv);
    int vv[AKA];
#pragma unroll
    for (int k = 0; k < AKA; ++k) {
        const int64_t a = threadIdx.x + (int64_t)AT * k;
        vv[k] = a < A ? (int)v_codes[a] : 0;
    }
    for (int j = 0; j < P; ++j) {
        const float st = s_st[j];
        const float win = fmaxf(4e-4f, st * 2e-6f);
        const float* un = u + (int64_t)(c0 + j) * ldu;
        float uvv[AKA];
#pragma unroll
        for (int k = 0; k < AKA; ++k) {
            const int64_t a = threadIdx.x + (int64_t)AT * k;
            uvv[k] = a < A ? un[a] : 0.0f;
        }
        int acc[APC] = {};
        uint32_t unsafe = 0;   // bit p*AKA + k
#pragma unroll
        for (int p = 0; p < APC; ++p) {
            if (i0 + p >= i1) break;                       // block-uniform
#pragma unroll
            for (int k = 0; k < AKA; ++k) {
                bool uk;
                const int c = att_code_fast(__fadd_rn(apv[p][k], uvv[k]), st, win, uk);
                acc[p] += vv[k] * c;                        // vv = 0 for a >= A
                unsafe |= (uint32_t)uk << (p * AKA + k);
            }
        }
        if (__any_sync(0xffffffffu, unsafe != 0)) {       // rare: exact fp64 codes for flagged elements
            while (unsafe) {
                const int b = __ffs(unsafe) - 1;
                unsafe &= unsafe - 1;
                const int p = b / AKA, k = b % AKA;
                float xv = 0.0f;
#pragma unroll
                for (int pp = 0; pp < APC; ++pp)
#pragma unroll
                    for (int kk = 0; kk < AKA; ++kk)
                        if (pp * AKA + kk == b) xv = __fadd_rn(apv[pp][kk], uvv[kk]);
                bool dummy;
                const int fast = att_code_fast(xv, st, win, dummy);
                const int exact = att_code_exact(xv, st);
                int vk = 0;
#pragma unroll
                for (int kk = 0; kk < AKA; ++kk)
                    if (kk == k) vk = vv[kk];
#pragma unroll
                for (int pp = 0; pp < APC; ++pp)
                    if (pp == p) acc[pp] += vk * (exact - fast);
            }
        }
#pragma unroll
        for (int p = 0; p < APC; ++p) {
            const int t = warp_sum(acc[p]);
            if (lane == 0) red[j][p][warp] = t;
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < P * APC; idx += AT) {
        const int j = idx / APC, p = idx % APC;
        if (i0 + p >= i1) continue;
        long long t = 0;
        for (int w = 0; w < AT / 32; ++w) t += red[j][p][w];
        scores[(int64_t)(c0 + j) * max_len + i0 + p] = dequant(t, v_scale[0], s_st[j]);
    }
}

// softmax over the l scores of every hypothesis of sentence s (fp64, fixed
// sequential sum order) and the context sum for a 256-wide slice of 2H.
// alpha lives in smem position-major ([i][AMAXP]) so the context loop reads it
// with broadcast loads; P is a template parameter (exactly P fp64 FMAs per i).
template <int P>
__device__ __forceinline__ void att_context_body(const float* __restrict__ scores, int32_t max_len,
                                                 const int32_t* __restrict__ sent_col_off, const float* __restrict__ states,
                                                 const int64_t* __restrict__ sent_row, const int32_t* __restrict__ sent_len,
                                                 int64_t H2, float* __restrict__ ctx, int64_t ldc,
                                                 float* __restrict__ alpha, int64_t lda, int32_t* err_flag,
                                                 unsigned char* smem_raw, uint32_t* ctx_segmax) {
    double* ex = reinterpret_cast<double*>(smem_raw);                   // [AMAXP][max_len]
    float* al = reinterpret_cast<float*>(ex + AMAXP * max_len);         // [max_len][AMAXP]
    const int s = blockIdx.y;
    const int l = sent_len[s];
    const int c0 = sent_col_off[s];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < P; j += AT / 32) {
        const float* sc = scores + (int64_t)(c0 + j) * max_len;
        float m = -3.402823466e38f;
        bool bad = false;
        for (int i = lane; i < l; i += 32) {
            const float x = sc[i];
            bad |= !is_finite_f(x);
            m = fmaxf(m, x);
        }
        m = warp_max(m);
        if (__any_sync(0xffffffffu, bad) && lane == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);
        for (int i = lane; i < l; i += 32) ex[j * max_len + i] = exp((double)sc[i] - (double)m);
        __syncwarp();
        double sum = 0.0;
        if (lane == 0)
            for (int i = 0; i < l; ++i) sum += ex[j * max_len + i];
        sum = __shfl_sync(0xffffffffu, sum, 0);
        for (int i = lane; i < l; i += 32) {
            const float a = __double2float_rn(ex[j * max_len + i] / sum);
            al[i * AMAXP + j] = a;
            if (alpha && blockIdx.x == 0) alpha[(int64_t)(c0 + j) * lda + i] = a;
        }
    }
    __syncthreads();
    const int64_t c = (int64_t)blockIdx.x * AT + threadIdx.x;
    if (c >= H2) return;
    const float* st = states + sent_row[s] * H2 + c;
    double acc[P];
#pragma unroll
    for (int j = 0; j < P; ++j) acc[j] = 0.0;
    int i = 0;
    for (; i + 4 <= l; i += 4) {
        float sv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) sv[q] = st[(int64_t)(i + q) * H2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < P; ++j) acc[j] += (double)sv[q] * (double)al[(i + q) * AMAXP + j];
    }
    for (; i < l; ++i) {
        const double sv = (double)st[(int64_t)i * H2];
#pragma unroll
        for (int j = 0; j < P; ++j) acc[j] += sv * (double)al[i * AMAXP + j];
    }
    uint32_t mx = 0;
#pragma unroll
    for (int j = 0; j < P; ++j) {
        const float v = __double2float_rn(acc[j]);
        ctx[(int64_t)(c0 + j) * ldc + c] = v;
        mx = max(mx, __float_as_uint(v) & 0x7fffffffu);
    }
    if (ctx_segmax) {   // per-sentence max |ctx| for the next quantization (segment = sentence)
        const unsigned act = __activemask();   // threads with c >= H2 have returned
        mx = __reduce_max_sync(act, mx);
        if ((act & ((1u << lane) - 1u)) == 0 && mx) atomicMax(ctx_segmax + s, mx);
    }
}

__global__ void __launch_bounds__(AT)
k_att_context3(const float* __restrict__ scores, int32_t max_len, const int32_t* __restrict__ sent_col_off,
               const int32_t* __restrict__ sent_ncols, const float* __restrict__ states,
               const int64_t* __restrict__ sent_row, const int32_t* __restrict__ sent_len, int64_t H2,
               float* __restrict__ ctx, int64_t ldc, float* __restrict__ alpha, int64_t lda, int32_t* err_flag,
               uint32_t* ctx_segmax) {
    extern __shared__ unsigned char smem_raw[];
    const int P = sent_ncols[blockIdx.y];
#define QNMT_CTX_P(P_)                                                                                      \
    case P_:                                                                                               \
        att_context_body<P_>(scores, max_len, sent_col_off, states, sent_row, sent_len, H2, ctx, ldc, alpha, \
                             lda, err_flag, smem_raw, ctx_segmax);                                         \
        break;
    switch (P) {
        QNMT_CTX_P(1) QNMT_CTX_P(2) QNMT_CTX_P(3) QNMT_CTX_P(4) QNMT_CTX_P(5) QNMT_CTX_P(6) QNMT_CTX_P(7)
        QNMT_CTX_P(8) QNMT_CTX_P(9) QNMT_CTX_P(10) QNMT_CTX_P(11) QNMT_CTX_P(12) QNMT_CTX_P(13) QNMT_CTX_P(14)
        QNMT_CTX_P(15) QNMT_CTX_P(16)
        default: break;   // P == 0: sentence finished
    }
#undef QNMT_CTX_P
}

int attention_launch(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                     const int32_t* sent_ncols, int32_t n_sent, const float* att_proj, const float* att_minmax,
                     const float* states, const int64_t* sent_row, const int32_t* sent_len, int32_t max_len,
                     int64_t A, int64_t H2, const int8_t* v_codes, const float* v_scale, float* ctx, int64_t ldc,
                     float* alpha, int64_t lda, void* scratch, int32_t* err_flag, cudaStream_t st,
                     uint32_t* ctx_segmax) {
    if (N <= 0 || n_sent <= 0) return QNMT_OK;
    if (A > (int64_t)AT * AKA) {
        set_error("qnmt_attention: attention dim %lld > %d", (long long)A, AT * AKA);
        return QNMT_ERR_SHAPE;
    }
    float* scores = reinterpret_cast<float*>(scratch);
    if (!att_minmax) {   // extrema not supplied by the caller: compute them into scratch
        float* mm = scores + ((N * max_len + 63) / 64) * 64;
        TRY_LAUNCH(att_minmax_launch(att_proj, sent_row, sent_len, n_sent, A, mm, st));
        att_minmax = mm;
    }
    dim3 g1((unsigned)cdiv(max_len, APC), (unsigned)n_sent);
    k_att_score3<<<g1, AT, 0, st>>>(u, ldu, sent_col_off, sent_ncols, att_proj, att_minmax, sent_row, sent_len, A,
                                    v_codes, v_scale, scores, max_len, err_flag);
    QNMT_CHECK_LAUNCH("k_att_score3");
    const size_t smem = (size_t)AMAXP * max_len * (sizeof(float) + sizeof(double));
    const dim3 g2((unsigned)cdiv(H2, AT), (unsigned)n_sent);
if (smem > 48 * 1024)
        QNMT_CUDA(cudaFuncSetAttribute(k_att_context3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_att_context3<<<g2, AT, smem, st>>>(scores, max_len, sent_col_off, sent_ncols, states, sent_row, sent_len, H2,
                                          ctx, ldc, alpha, lda, err_flag, ctx_segmax);
    QNMT_CHECK_LAUNCH("k_att_context3");
    return QNMT_OK;
}

// column -> sentence ranges for callers that only have col_sent (columns grouped by sentence)
__global__ void k_col_ranges(const int32_t* __restrict__ col_sent, int64_t N, int32_t* off, int32_t* cnt) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int s = col_sent[n];
    atomicAdd(cnt + s, 1);
    atomicMin(off + s, (int)n);
}

int col_ranges_launch(const int32_t* col_sent, int64_t N, int32_t n_sent, int32_t* off, int32_t* cnt,
                      cudaStream_t st) {
    QNMT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)n_sent, st));
    QNMT_CUDA(cudaMemsetAsync(off, 0x7f, sizeof(int32_t) * (size_t)n_sent, st));
    if (N <= 0) return QNMT_OK;
    k_col_ranges<<<(unsigned)cdiv(N, 256), 256, 0, st>>>(col_sent, N, off, cnt);
    QNMT_CHECK_LAUNCH("k_col_ranges");
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" int qnmt_attention(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                              const int32_t* sent_ncols, int32_t n_sent, const float* att_proj,
                              const float* att_minmax, const float* states, const int64_t* sent_row, const int32_t* sent_len,
                              int32_t max_len, int64_t A, int64_t H2, const int8_t* v_codes,
                              const float* v_scale, float* ctx, int64_t ldc, float* alpha, int64_t lda,
                              void* scratch, int32_t* err_flag, void* stream) {
    return qnmt::attention_launch(u, ldu, N, sent_col_off, sent_ncols, n_sent, att_proj, att_minmax, states,
                                  sent_row,
                                  sent_len, max_len, A, H2, v_codes, v_scale, ctx, ldc, alpha, lda, scratch,
                                  err_flag, qnmt::as_stream(stream));
}

extern "C" int qnmt_attention_stats(const float* att_proj, const int64_t* sent_row, const int32_t* sent_len,
                                    int32_t n_sent, int64_t A, float* att_minmax, void* stream) {
    return qnmt::att_minmax_launch(att_proj, sent_row, sent_len, n_sent, A, att_minmax, qnmt::as_stream(stream));
}
