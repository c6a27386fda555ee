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
// Codes q(t) use an f32 fast path whose error against the reference's v = t*scale
// is bounded; the code floor(|v| + 1/2) can only differ if v is within that bound
// of a half-integer, and only those elements are recomputed with the fp64-exact
// tanh.  Two fast paths:
//   k_att_score6 (one MUFU per element): att_proj is fixed for the whole decode,
//     so E_ap = fl32(e^(2 ap)) is computed once per batch (k_att_exp) and
//     E_u = fl32(e^(2 u)) once per hypothesis and step (k_att_scale);
//     e^(2(ap+u)) = E_ap * E_u and t = 1 - 2 / (1 + E_ap E_u): one FFMA, one
//     MUFU.RCP, one FFMA per element (needs |ap|, |u| <= 20: no over/underflow);
//   k_att_score5 (two MUFU): t = 1 - 2 / (1 + 2^(2x log2 e)) from x = fl(ap + u).
#include <algorithm>

#include "kernels.cuh"
#include "tc_common.cuh"

#ifndef QNMT_APC
#define QNMT_APC 6
#endif
#define TRY_LAUNCH(x) do { int _r = (x); if (_r != QNMT_OK) return _r; } while (0)

namespace qnmt {

constexpr int AT = 256;        // threads per CTA
constexpr int APC = 4;         // encoder positions per CTA (max / score passes)
constexpr int AMAXP = 16;      // max live hypotheses per sentence (beam <= 16)
constexpr int AKA = 8;         // a-elements per thread kept in registers (A <= AT * AKA)
int g_att_ctx_staged = 1;      // context kernel: 0 context3, 1 context4, 2 context5 (A/B testing)

// Fast tanh from two MUFU ops, signed form: t = 1 - 2 / (1 + 2^(2x log2 e)).
// Exhaustive over every f32 x with 2^-24 <= |x| < 64 (benchmarks/tanh_err.cu,
// profiles/r01_tanh_err.jsonl): |t_fast - tanh(x)| <= 2.37e-7; outside that
// range t_fast is 0 / +-1 / within the same bound.
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

// Fast-path rounding window.  v_fast = fl(st - 2 st r) (one FFMA rounding,
// <= 3.8e-6 at |v| <= 128) differs from the reference's v = fl(fl32(tanh x) * st)
// by at most st * (2.37e-7 + 3e-8) + 7.6e-6 (2.37e-7: exhaustive max of
// |t_fast - tanh| over every f32 x, profiles/r01_tanh_err.jsonl); the window
// below is that bound plus ~9% / ~18% margin.  Where fl(v + 1.5*2^23) - 1.5*2^23
// (round-to-nearest-even, exact) is farther than the window from a
// half-integer, the reference's floor(|v| + 1/2) (qmath.py:136-142) gives the
// same integer; otherwise the element is recomputed with the fp64 tanh
// (att_code_exact).
__device__ __forceinline__ float att_threshold(float st) { return 0.5f - (st * 2.9e-7f + 9e-6f); }
constexpr float ATT_ST_FAST_MAX = 1.0e6f;   // above: window > 0.5, every element exact

__device__ __noinline__ int att_code_exact(float x, float st) { return quant_code(tanh_b(x), st); }

// One-MUFU fast path (k_att_score6/7): v_fast = fl(st - 2 st rcp.approx(fl(E_ap E_u + 1)))
// with E_ap = fl32(e^(2 ap)) (fp64 exp rounded once: rel. error d1 <= 2^-24) and
// E_u = exp2x_f32(u) (rel. error d2, measured exhaustively over every f32 |u| <= 20).
// With the FFMA's rounding d3 = 2^-24 and rcp.approx.ftz.f32's relative error
// d4 (<= 2^-23, exhaustive), r = 1/(1 + E)(1 + eta) with
// |eta| <= (E/(1+E))(d1 + d2) + d3 + d4, so |v_fast - st tanh(ap+u)| <=
// 2 st [r* E/(1+E) (d1+d2) + r* (d3+d4)] <= st [(d1+d2)/2 + 2(d3+d4)]
// (r* E/(1+E) = E/(1+E)^2 <= 1/4, r* <= 1), plus the FFMA's half ulp of v.  The
// reference's v carries one rounding of t (st 2^-25), one of the product (half
// an ulp), and tanh(fl(ap+u)) vs tanh(ap+u) (<= 0.45 * 2^-24 st).  With d2 <=
// With the measured d2 = 7.9e-8 and d4 = 9.83e-8 the total is <= 4.42e-7 st + 7.63e-6;
// the window below has 25% margin (profiles/r02_att_exp_err.json: the exhaustive d2
// and d4, and a Monte-Carlo of 2^33 draws per distribution of |v_fast - v| against the
// window).
__device__ __forceinline__ float att_e_threshold(float st) { return 0.5f - (st * 5.5e-7f + 9.5e-6f); }
constexpr int ATT_FIXCAP_MAX = 512;
constexpr float ATT_E_BOUND = 20.0f;   // |ap|, |u| <= 20: E_ap E_u in [1.8e-35, 5.5e34], no ftz / overflow
int g_att_score8 = 1;                  // two-MUFU scorer with the bulk-copied tile (k_att_score8)
#define A4_FITS(A) ((A) / 4 <= AQ5 * AT)
int g_att_fused_scale = 0;             // 1: two-MUFU scorer computes the scales itself (k_att_score5f; A/B: 125 vs 101 + 11 us)
int g_att_fixcap = ATT_FIXCAP_MAX;      // tests: 0 forces the queue-overflow rescan
int g_att_exp = 0;                      // scorer: 0 two-MUFU (score5/8), 1 one-MUFU (score6), 2 one-MUFU staged (score7)

// E_ap = fl32(e^(2 ap)) for n values of att_proj (fp64 exp, rounded once).  Values
// beyond the fast path's bound are clamped (their sentences take the two-MUFU path).
__global__ void k_att_exp(const float* __restrict__ ap, int64_t n, float* __restrict__ out) {
    pdl_entry();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = fmin(fmax((double)ap[i], -(double)ATT_E_BOUND), (double)ATT_E_BOUND);
        out[i] = __double2float_rn(exp_f64(2.0 * x));
    }
}

int att_exp_launch(const float* att_proj, int64_t n, float* out, cudaStream_t st) {
    if (n <= 0) return QNMT_OK;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 16);
    QNMT_LAUNCH(k_att_exp, grid, 256, 0, st, att_proj, n, out);
    QNMT_CHECK_LAUNCH("k_att_exp");
    return QNMT_OK;
}

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
    pdl_entry();
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
    QNMT_LAUNCH(k_att_minmax, dim3((unsigned)cdiv(A, AT), (unsigned)n_sent), AT, 0, st, att_proj, sent_row, sent_len, A, mm);
    QNMT_CHECK_LAUNCH("k_att_minmax");
    return QNMT_OK;
}

// Per-hypothesis scale of the whole [A, l] tanh block (layers.py:226) from the
// column extrema, and the fast-path thresholds:
//   st_thr[c] = {st, att_threshold(st), att_e_threshold(st), eligible for k_att_score6}.
// With eu != nullptr also E_u[c][a] = e^(2 u[c][a]) (exp2x_f32: f32, error measured exhaustively).
// Grid (n_sent, AMAXP): CTA (s, j) handles hypothesis j of sentence s.
__global__ void __launch_bounds__(AT)
k_att_scale(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ sent_col_off,
            const int32_t* __restrict__ sent_ncols, const float* __restrict__ mm, int64_t A,
            float4* __restrict__ st_thr, int32_t* err_flag, uint32_t* zero_seg, float* __restrict__ eu) {
    pdl_entry();
    __shared__ uint32_t mred[AT / 32], bred[AT / 32];
    const int s = blockIdx.x, j = blockIdx.y;
    // the context kernel of this step max-reduces |ctx| per sentence into zero_seg[s]
    // (replaces a memset node, which would break the programmatic-dependent-launch chain)
    if (zero_seg && j == 0 && threadIdx.x == 0) zero_seg[s] = 0u;
    if (j >= sent_ncols[s]) return;
    const int c = sent_col_off[s] + j;
    const float* un = u + (int64_t)c * ldu;
    const float* mx = mm + ((int64_t)s * 2) * A;
    const float* mn = mx + A;
    uint32_t m = 0, b = 0;   // b: max of |ap| extrema and |u| (fast-path eligibility)
    float uv[AKA];
#pragma unroll
    for (int k = 0; k < AKA; ++k) {   // A <= AT * AKA: all loads in flight at once
        const int64_t a = threadIdx.x + (int64_t)AT * k;
        uv[k] = 0.0f;
        if (a < A) {
            uv[k] = un[a];
            const float x0 = mx[a], x1 = mn[a];
            m = max(m, __float_as_uint(__fadd_rn(x0, uv[k])) & 0x7fffffffu);
            m = max(m, __float_as_uint(__fadd_rn(x1, uv[k])) & 0x7fffffffu);
            b = max(b, max(__float_as_uint(x0) & 0x7fffffffu, __float_as_uint(x1) & 0x7fffffffu));
            b = max(b, __float_as_uint(uv[k]) & 0x7fffffffu);
        }
    }
    if (eu) {
#pragma unroll
        for (int k = 0; k < AKA; ++k) {
            const int64_t a = threadIdx.x + (int64_t)AT * k;
            if (a < A) {
                eu[(int64_t)c * A + a] = exp2x_f32(fminf(fmaxf(uv[k], -ATT_E_BOUND), ATT_E_BOUND));
            }
        }
    }
    m = warp_max(m);
    b = warp_max(b);
    if ((threadIdx.x & 31) == 0) {
        mred[threadIdx.x >> 5] = m;
        bred[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < AT / 32; ++w) {
            m = max(m, mred[w]);
            b = max(b, bred[w]);
        }
        if (m >= 0x7f800000u) {
            set_flag(err_flag, QNMT_FLAG_NUMERIC);
            m = 0;
        }
        const float tmax = tanh_b(__uint_as_float(m));   // max |fl32(tanh)| = fl32(tanh(max |x|))
        const float st = (tmax == 0.0f) ? 1.0f : __fdiv_rn(127.0f, tmax);
        const bool elig = eu != nullptr && b <= __float_as_uint(ATT_E_BOUND) && st <= ATT_ST_FAST_MAX;
        st_thr[c] = make_float4(st, att_threshold(st), att_e_threshold(st), elig ? 1.0f : 0.0f);
    }
}

// scores for APC positions x all P hypotheses of one sentence.  Per element:
// FADD, FMUL, 2 MUFU, FADD, FFMA, 2 FADD + IADD (magic rounding), FADD, FMNMX,
// IMAD.  A thread whose max distance to a half-integer falls inside the window
// rescans its 32 elements and corrects the flagged ones exactly (rare).
__global__ void __launch_bounds__(AT, 2)
k_att_score4(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ sent_col_off,
             const int32_t* __restrict__ sent_ncols, const float* __restrict__ att_proj,
             const float4* __restrict__ st_thr, const int64_t* __restrict__ sent_row,
             const int32_t* __restrict__ sent_len, int64_t A, const int8_t* __restrict__ v_codes,
             const float* __restrict__ v_scale, float* __restrict__ scores, int32_t max_len) {
    pdl_entry();
    __shared__ int red[AMAXP][APC][AT / 32];
    const int s = blockIdx.y;
    const int P = sent_ncols[s];
    const int l = sent_len[s];
    const int i0 = blockIdx.x * APC;
    if (P == 0 || i0 >= l) return;
    const int i1 = min(l, i0 + APC);
    const int c0 = sent_col_off[s];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float apv[APC][AKA];
    load_ap(att_proj + sent_row[s] * A, A, i0, i1, apv);
    int vv[AKA];
    float uvv[AKA], unx[AKA];
#pragma unroll
    for (int k = 0; k < AKA; ++k) {
        const int64_t a = threadIdx.x + (int64_t)AT * k;
        vv[k] = a < A ? (int)v_codes[a] : 0;
        uvv[k] = a < A ? u[(int64_t)c0 * ldu + a] : 0.0f;
    }
    float4 sp = st_thr[c0];
    for (int j = 0; j < P; ++j) {
        float4 spx = sp;
        if (j + 1 < P) {   // prefetch the next hypothesis' query row and scale
            const float* un = u + (int64_t)(c0 + j + 1) * ldu;
#pragma unroll
            for (int k = 0; k < AKA; ++k) {
                const int64_t a = threadIdx.x + (int64_t)AT * k;
                unx[k] = a < A ? un[a] : 0.0f;
            }
            spx = st_thr[c0 + j + 1];
        }
        const float st = sp.x, thr = sp.y, m2st = -2.0f * st;
        int acc[APC] = {};
        if (st <= ATT_ST_FAST_MAX) {   // CTA-uniform
            float dmax = 0.0f;
#pragma unroll
            for (int p = 0; p < APC; ++p) {
                if (i0 + p >= i1) break;   // CTA-uniform
#pragma unroll
                for (int k = 0; k < AKA; ++k) {
                    const float x = __fadd_rn(apv[p][k], uvv[k]);
                    const float r = rcp_approx(__fadd_rn(ex2_approx(__fmul_rn(x, 2.8853900817779268f)), 1.0f));
                    const float v = fmaf(m2st, r, st);
                    const float mg = __fadd_rn(v, 12582912.0f);   // 1.5 * 2^23
                    dmax = fmaxf(dmax, fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))));
                    acc[p] += vv[k] * (__float_as_int(mg) - 0x4B400000);
                }
            }
            if (dmax > thr) {   // rare: some element within the window of a rounding boundary
#pragma unroll
                for (int p = 0; p < APC; ++p) {
                    if (i0 + p >= i1) break;
#pragma unroll
                    for (int k = 0; k < AKA; ++k) {
                        const float x = __fadd_rn(apv[p][k], uvv[k]);
                        const float r = rcp_approx(__fadd_rn(ex2_approx(__fmul_rn(x, 2.8853900817779268f)), 1.0f));
                        const float v = fmaf(m2st, r, st);
                        const float mg = __fadd_rn(v, 12582912.0f);
                        if (fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))) > thr && vv[k] != 0)
                            acc[p] += vv[k] * (att_code_exact(x, st) - (__float_as_int(mg) - 0x4B400000));
                    }
                }
            }
        } else {   // degenerate scale (max |tanh| < 1.3e-4): exact codes throughout
#pragma unroll
            for (int p = 0; p < APC; ++p) {
                if (i0 + p >= i1) break;
#pragma unroll
                for (int k = 0; k < AKA; ++k)
                    if (vv[k] != 0) acc[p] += vv[k] * att_code_exact(__fadd_rn(apv[p][k], uvv[k]), st);
            }
        }
#pragma unroll
        for (int p = 0; p < APC; ++p) {
            const int t = __reduce_add_sync(0xffffffffu, acc[p]);
            if (lane == 0) red[j][p][warp] = t;
        }
#pragma unroll
        for (int k = 0; k < AKA; ++k) uvv[k] = unx[k];
        sp = spx;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < P * APC; idx += AT) {
        const int j = idx / APC, p = idx % APC;
        if (i0 + p >= i1) continue;
        long long t = 0;
        for (int w = 0; w < AT / 32; ++w) t += red[j][p][w];
        scores[(int64_t)(c0 + j) * max_len + i0 + p] = dequant(t, v_scale[0], st_thr[c0 + j].x);
    }
}

// Attention dims beyond the register-resident kernels (A > AT * AKA = 2048): the same
// arithmetic with the a-loop strided over the CTA instead of unrolled into registers.
// k_att_scale_wide: per-hypothesis scale and thresholds, exactly as k_att_scale.
__global__ void __launch_bounds__(AT)
k_att_scale_wide(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ sent_col_off,
                 const int32_t* __restrict__ sent_ncols, const float* __restrict__ mm, int64_t A,
                 float4* __restrict__ st_thr, int32_t* err_flag, uint32_t* zero_seg) {
    pdl_entry();
    __shared__ uint32_t mred[AT / 32];
    const int s = blockIdx.x, j = blockIdx.y;
    if (zero_seg && j == 0 && threadIdx.x == 0) zero_seg[s] = 0u;
    if (j >= sent_ncols[s]) return;
    const int c = sent_col_off[s] + j;
    const float* un = u + (int64_t)c * ldu;
    const float* mx = mm + ((int64_t)s * 2) * A;
    const float* mn = mx + A;
    uint32_t m = 0;
    for (int64_t a = threadIdx.x; a < A; a += AT) {
        const float uv = un[a];
        m = max(m, __float_as_uint(__fadd_rn(mx[a], uv)) & 0x7fffffffu);
        m = max(m, __float_as_uint(__fadd_rn(mn[a], uv)) & 0x7fffffffu);
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) mred[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < AT / 32; ++w) m = max(m, mred[w]);
        if (m >= 0x7f800000u) {
            set_flag(err_flag, QNMT_FLAG_NUMERIC);
            m = 0;
        }
        const float tmax = tanh_b(__uint_as_float(m));
        const float st = (tmax == 0.0f) ? 1.0f : __fdiv_rn(127.0f, tmax);
        st_thr[c] = make_float4(st, att_threshold(st), att_e_threshold(st), 0.0f);
    }
}

// k_att_score_wide: scores for APC positions x all P hypotheses of one sentence, any A.
// Per element the two-MUFU fast path of k_att_score4 with the exact code taken at once
// for an element inside the rounding window (the same codes as every other scorer).
__global__ void __launch_bounds__(AT)
k_att_score_wide(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ sent_col_off,
                 const int32_t* __restrict__ sent_ncols, const float* __restrict__ att_proj,
                 const float4* __restrict__ st_thr, const int64_t* __restrict__ sent_row,
                 const int32_t* __restrict__ sent_len, int64_t A, const int8_t* __restrict__ v_codes,
                 const float* __restrict__ v_scale, float* __restrict__ scores, int32_t max_len) {
    pdl_entry();
    __shared__ long long red[APC][AT / 32];
    const int s = blockIdx.y;
    const int P = sent_ncols[s];
    const int l = sent_len[s];
    const int i0 = blockIdx.x * APC;
    if (P == 0 || i0 >= l) return;
    const int np = min(l - i0, APC);
    const int c0 = sent_col_off[s];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* ap = att_proj + (sent_row[s] + i0) * A;
    for (int j = 0; j < P; ++j) {
        const float* un = u + (int64_t)(c0 + j) * ldu;
        const float4 sp = st_thr[c0 + j];
        const float st = sp.x, thr = sp.y, m2st = -2.0f * st;
        const bool fast = st <= ATT_ST_FAST_MAX;
        long long acc[APC] = {};
        for (int64_t a = threadIdx.x; a < A; a += AT) {
            const int vk = (int)v_codes[a];
            const float uv = un[a];
            if (vk == 0) continue;
#pragma unroll
            for (int p = 0; p < APC; ++p) {
                if (p >= np) break;
                const float x = __fadd_rn(ap[(int64_t)p * A + a], uv);
                int code;
                if (fast) {
                    const float r = rcp_approx(__fadd_rn(ex2_approx(__fmul_rn(x, 2.8853900817779268f)), 1.0f));
                    const float v = fmaf(m2st, r, st);
                    const float mg = __fadd_rn(v, 12582912.0f);   // 1.5 * 2^23
                    code = __float_as_int(mg) - 0x4B400000;
                    if (fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))) > thr) code = att_code_exact(x, st);
                } else {
                    code = att_code_exact(x, st);
                }
                acc[p] += (long long)(vk * code);
            }
        }
        __syncthreads();   // red of the previous hypothesis consumed
#pragma unroll
        for (int p = 0; p < APC; ++p) {
            long long t = acc[p];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) red[p][warp] = t;
        }
        __syncthreads();
        if (threadIdx.x < np) {
            long long t = 0;
            for (int w = 0; w < AT / 32; ++w) t += red[threadIdx.x][w];
            scores[(int64_t)(c0 + j) * max_len + i0 + threadIdx.x] = dequant(t, v_scale[0], st);
        }
    }
}

// Same scores with each thread's slice of the tile parked in shared memory
// (APC5 positions x its a-quads; a thread only ever reads its own slots, so no
// barrier), registers holding just the query slice, codes and accumulators:
// 4 CTAs / SM to hide the MUFU / FMA latency.  Thread t owns a-quads
// 4t + 4*AT*k; quads past A are zero (no bounds checks in the hot loop).  Warps
// store their per-position sums in shared memory and the last warp to finish
// writes the scores (no end-of-CTA barrier wait).
//   EXPM = false (k_att_score5): tile = att_proj, query = u, two MUFU per element;
//   EXPM = true  (k_att_score6, sentences whose hypotheses are all eligible):
//     tile = E_ap, query = E_u, one MUFU per element; elements in the rounding
//     window are recomputed exactly from att_proj / u in global memory.
constexpr int APC5 = QNMT_APC;   // positions per CTA (6: 48 KB of tile slices, 4 CTAs / SM)
constexpr int AQ5 = 2;         // a-quads per thread (A <= 4 * AT * AQ5 = 2048)

struct ScoreArgs {
    const float* u;
    int64_t ldu;
    const int32_t* sent_col_off;
    const int32_t* sent_ncols;
    const float* att_proj;
    const float* att_exp;      // E_ap [rows][A] (score6)
    const float* eu;           // E_u [N][A] (score6)
    const float4* st_thr;
    const int64_t* sent_row;
    const int32_t* sent_len;
    int64_t A;
    const int8_t* v_codes;
    const float* v_scale;
    float* scores;
    int32_t max_len;
    int32_t fixcap;            // deferred fixup queue length used (<= ATT_FIXCAP; tests lower it)
};

constexpr int ATT_FIXCAP = ATT_FIXCAP_MAX;   // deferred fixup slots per CTA (score6); beyond: the last warp rescans all

// A deferred fixup entry j | p << 4 | t << 7 names thread t's slots of position p
// for hypothesis j, which hold an element inside the rounding window.  Returns
// sum over those slots' flagged elements of va * (exact code - fast code).
__device__ __forceinline__ int att_fix_slot(const float4* __restrict__ sap, const float* __restrict__ ap_row0,
                                            int64_t A, const float* __restrict__ u_c0, int64_t ldu,
                                            const float* __restrict__ eu_c0, const int8_t* __restrict__ v_codes,
                                            int ent, float st, float thr) {
    const int j = ent & 15, p = (ent >> 4) & 7, t = ent >> 7;
    const float m2st = -2.0f * st;
    const int64_t A4 = A / 4;
    int d = 0;
    for (int k = 0; k < AQ5; ++k) {
        const int64_t q = t + (int64_t)AT * k;
        if (q >= A4) break;
        const float4 apq = sap[(p * AQ5 + k) * AT + t];
        const float4 euq = reinterpret_cast<const float4*>(eu_c0 + (int64_t)j * A)[q];
        for (int e = 0; e < 4; ++e) {
            const int64_t a = 4 * q + e;
            const int va = v_codes[a];
            const float v = fmaf(m2st, rcp_approx(fmaf((&apq.x)[e], (&euq.x)[e], 1.0f)), st);
            const float mg = __fadd_rn(v, 12582912.0f);
            if (fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))) > thr && va != 0) {
                const float x = __fadd_rn(ap_row0[p * A + a], u_c0[(int64_t)j * ldu + a]);
                d += va * (att_code_exact(x, st) - (__float_as_int(mg) - 0x4B400000));
            }
        }
    }
    return d;
}

template <bool EXPM>
__device__ __forceinline__ void att_score_body(const ScoreArgs& g, float4* sap, int (*red5)[APC5][AT / 32],
                                               int* s_done, int s, int P, int l, int i0,
                                               int* fixl = nullptr, int* s_nfix = nullptr,
                                               const float4* stv = nullptr) {
    const int i1 = min(l, i0 + APC5);
    const int np = i1 - i0;
    const int c0 = g.sent_col_off[s];
    const int lane = threadIdx.x & 31;
    const int64_t A = g.A, A4 = A / 4;
    const int64_t row0 = g.sent_row[s] + i0;
    const float4* sv = stv ? stv : g.st_thr + g.sent_col_off[s];   // per-hypothesis {st, thresholds} of the sentence
    if (threadIdx.x == 0) {
        *s_done = 0;
        if (EXPM) *s_nfix = 0;
    }
    {   // this thread's slots of the tile (positions past i1 and quads past A are zero)
        const float4* src = reinterpret_cast<const float4*>((EXPM ? g.att_exp : g.att_proj) + row0 * A);
#pragma unroll
        for (int p = 0; p < APC5; ++p)
#pragma unroll
            for (int k = 0; k < AQ5; ++k) {
                const int64_t q = threadIdx.x + (int64_t)AT * k;
                sap[(p * AQ5 + k) * AT + threadIdx.x] =
                    (p < np && q < A4) ? src[p * A4 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
    }
    const float* qsrc = EXPM ? g.eu : g.u;   // query side: E_u [N][A] or u [N][ldu]
    const int64_t ldq = EXPM ? A : g.ldu;
    int vv[AQ5][4];
    float4 uq[AQ5], ux[AQ5];
#pragma unroll
    for (int k = 0; k < AQ5; ++k) {
        const int64_t q = threadIdx.x + (int64_t)AT * k;
        const bool ok = q < A4;
        const char4 c = ok ? reinterpret_cast<const char4*>(g.v_codes)[q] : make_char4(0, 0, 0, 0);
        vv[k][0] = c.x; vv[k][1] = c.y; vv[k][2] = c.z; vv[k][3] = c.w;
        uq[k] = ok ? reinterpret_cast<const float4*>(qsrc + (int64_t)c0 * ldq)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4 sp = sv[0];
    int vsum = 0;
#pragma unroll
    for (int k = 0; k < AQ5; ++k) vsum += vv[k][0] + vv[k][1] + vv[k][2] + vv[k][3];
    const int vsum_off = (int)((unsigned)vsum * 0x4B400000u);
    __syncthreads();   // s_done initialised
    for (int j = 0; j < P; ++j) {
        float4 spx = sp;
        if (j + 1 < P) {   // prefetch the next hypothesis' query slice and scale
#pragma unroll
            for (int k = 0; k < AQ5; ++k) {
                const int64_t q = threadIdx.x + (int64_t)AT * k;
                ux[k] = q < A4 ? reinterpret_cast<const float4*>(qsrc + (int64_t)(c0 + j + 1) * ldq)[q]
                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            spx = sv[j + 1];
        }
        const float st = sp.x, thr = EXPM ? sp.z : sp.y, m2st = -2.0f * st;
        int acc[APC5];
#pragma unroll
        for (int p = 0; p < APC5; ++p) acc[p] = 0;
        // v for element e of quad k at position p (the fast path)
        auto fast_v = [&](const float4& apq, int k, int e) -> float {
            const float a4[4] = {apq.x, apq.y, apq.z, apq.w};
            const float u4[4] = {uq[k].x, uq[k].y, uq[k].z, uq[k].w};
            float r;
            if (EXPM) {
                r = rcp_approx(fmaf(a4[e], u4[e], 1.0f));
            } else {
                const float x = __fadd_rn(a4[e], u4[e]);
                r = rcp_approx(__fadd_rn(ex2_approx(__fmul_rn(x, 2.8853900817779268f)), 1.0f));
            }
            return fmaf(m2st, r, st);
        };
        if (EXPM || st <= ATT_ST_FAST_MAX) {   // CTA-uniform
            float dmx[APC5];   // per position: max distance of v to its rounding integer
#pragma unroll
            for (int p = 0; p < APC5; ++p) {
                dmx[p] = 0.0f;
                if (p >= np) break;   // CTA-uniform
#pragma unroll
                for (int k = 0; k < AQ5; ++k) {
                    const float4 apq = sap[(p * AQ5 + k) * AT + threadIdx.x];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float v = fast_v(apq, k, e);
                        const float mg = __fadd_rn(v, 12582912.0f);   // 1.5 * 2^23
                        dmx[p] = fmaxf(dmx[p], fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))));
                        // code = bits - 0x4B400000: the offset is removed once per position below
                        acc[p] = (int)((unsigned)acc[p] + (unsigned)vv[k][e] * (unsigned)__float_as_int(mg));
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < APC5; ++p)   // sum_a v_a * code_a = sum_a v_a * bits_a - 0x4B400000 * sum_a v_a (mod 2^32)
                if (p < np) acc[p] = (int)((unsigned)acc[p] - (unsigned)vsum_off);
            // rare: a position with an element within the window of a rounding boundary.
            // Two-MUFU mode: recompute it now, flagged elements exactly (fp64 tanh of
            // x = fl(ap + u)).  E mode: att_proj / u must come from global memory, so the
            // slots are queued and the CTA's last warp resolves the queue with all loads in
            // flight at once (att_fix_slot).
#pragma unroll
            for (int p = 0; p < APC5; ++p) {
                if (p >= np) break;
                if (dmx[p] <= thr) continue;
                if (EXPM) {
                    const int slot = atomicAdd(s_nfix, 1);
                    if (slot < g.fixcap) fixl[slot] = j | (p << 4) | ((int)threadIdx.x << 7);
                    continue;
                }
                int d = 0;
#pragma unroll
                for (int k = 0; k < AQ5; ++k) {
                    const float4 apq = sap[(p * AQ5 + k) * AT + threadIdx.x];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float v = fast_v(apq, k, e);
                        const float mg = __fadd_rn(v, 12582912.0f);
                        if (fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))) > thr && vv[k][e] != 0) {
                            const float x = __fadd_rn((&apq.x)[e], (&uq[k].x)[e]);
                            d += vv[k][e] * (att_code_exact(x, st) - (__float_as_int(mg) - 0x4B400000));
                        }
                    }
                }
                acc[p] += d;
            }
        } else {   // degenerate scale (max |tanh| < 1.3e-4): exact codes throughout (two-MUFU mode only)
            for (int p = 0; p < np; ++p) {
                int a_sum = 0;
#pragma unroll
                for (int k = 0; k < AQ5; ++k) {
                    const float4 apq = sap[(p * AQ5 + k) * AT + threadIdx.x];
                    const float ap4[4] = {apq.x, apq.y, apq.z, apq.w};
                    const float u4[4] = {uq[k].x, uq[k].y, uq[k].z, uq[k].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (vv[k][e] != 0) a_sum += vv[k][e] * att_code_exact(__fadd_rn(ap4[e], u4[e]), st);
                }
#pragma unroll
                for (int pp = 0; pp < APC5; ++pp)
                    if (pp == p) acc[pp] += a_sum;
            }
        }
#pragma unroll
        for (int p = 0; p < APC5; ++p) {
            const int t = __reduce_add_sync(0xffffffffu, acc[p]);
            if (lane == 0) red5[j][p][threadIdx.x >> 5] = t;
        }
#pragma unroll
        for (int k = 0; k < AQ5; ++k) uq[k] = ux[k];
        sp = spx;
    }
    // the last warp to finish writes the scores
    int last = 0;
    if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(s_done, 1) == AT / 32 - 1;
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence_block();
    if (EXPM) {   // deferred exact codes of the queued slots (queue overflow: every slot of the CTA)
        const bool all = *s_nfix > g.fixcap;
        const int nf = all ? P * np * AT : *s_nfix;
        for (int f = lane; f < nf; f += 32) {
            const int e = all ? (f / (np * AT)) | (((f / AT) % np) << 4) | ((f % AT) << 7) : fixl[f];
            const float4 sp = sv[e & 15];
            const int d = att_fix_slot(sap, g.att_proj + row0 * A, A, g.u + (int64_t)c0 * g.ldu, g.ldu,
                                       g.eu + (int64_t)c0 * A, g.v_codes, e, sp.x, sp.z);
            if (d) atomicAdd(&red5[e & 15][(e >> 4) & 7][0], d);
        }
        __syncwarp();
    }
    for (int idx = lane; idx < P * np; idx += 32) {
        const int j = idx / np, p = idx % np;
        int t = 0;
#pragma unroll
        for (int w = 0; w < AT / 32; ++w) t += red5[j][p][w];
        g.scores[(int64_t)(c0 + j) * g.max_len + i0 + p] = dequant(t, g.v_scale[0], sv[j].x);
    }
}

// two-MUFU scorer for every sentence
__global__ void __launch_bounds__(AT, 4)
k_att_score5(ScoreArgs g) {
    pdl_entry();
    extern __shared__ float4 sap[];   // [APC5][AQ5][AT]
    __shared__ int red5[AMAXP][APC5][AT / 32];
    __shared__ int s_done;
    const int s = blockIdx.y;
    const int P = g.sent_ncols[s], l = g.sent_len[s], i0 = blockIdx.x * APC5;
    if (P == 0 || i0 >= l) return;
    att_score_body<false>(g, sap, red5, &s_done, s, P, l, i0);
}

// two-MUFU scorer with the per-hypothesis scale computed in the CTA (no k_att_scale
// launch): every CTA of sentence s reduces max_a max(|fl(mx_a + u_a)|, |fl(mn_a + u_a)|)
// for each of the sentence's hypotheses from its own quads (a warp max, a shared-memory
// atomicMax), then thread j evaluates fl32(tanh) of the max and the scale (identical to
// k_att_scale: the same operations, so every CTA of the sentence gets the same st).
// The CTA with blockIdx.x == 0 also zeroes the context kernel's per-sentence max.
__global__ void __launch_bounds__(AT, 4)
k_att_score5f(ScoreArgs g, const float* __restrict__ mm, int32_t* err_flag, uint32_t* zero_seg) {
    pdl_entry();
    extern __shared__ float4 sap[];   // [APC5][AQ5][AT]
    __shared__ int red5[AMAXP][APC5][AT / 32];
    __shared__ int s_done;
    __shared__ uint32_t s_m[AMAXP];
    __shared__ float4 s_st[AMAXP];
    const int s = blockIdx.y;
    if (zero_seg && blockIdx.x == 0 && threadIdx.x == 0) zero_seg[s] = 0u;
    const int P = g.sent_ncols[s], l = g.sent_len[s], i0 = blockIdx.x * APC5;
    if (P == 0 || i0 >= l) return;
    const int c0 = g.sent_col_off[s];
    const int64_t A = g.A, A4 = A / 4;
    if (threadIdx.x < AMAXP) s_m[threadIdx.x] = 0u;
    float4 mxq[AQ5], mnq[AQ5];
#pragma unroll
    for (int k = 0; k < AQ5; ++k) {
        const int64_t q = threadIdx.x + (int64_t)AT * k;
        const bool ok = q < A4;
        mxq[k] = ok ? reinterpret_cast<const float4*>(mm + (int64_t)s * 2 * A)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
        mnq[k] = ok ? reinterpret_cast<const float4*>(mm + (int64_t)s * 2 * A + A)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();   // s_m initialised
    for (int j = 0; j < P; ++j) {
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < AQ5; ++k) {
            const int64_t q = threadIdx.x + (int64_t)AT * k;
            if (q < A4) {
                const float4 uv = reinterpret_cast<const float4*>(g.u + (int64_t)(c0 + j) * g.ldu)[q];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    m = max(m, __float_as_uint(__fadd_rn((&mxq[k].x)[e], (&uv.x)[e])) & 0x7fffffffu);
                    m = max(m, __float_as_uint(__fadd_rn((&mnq[k].x)[e], (&uv.x)[e])) & 0x7fffffffu);
                }
            }
        }
        m = __reduce_max_sync(0xffffffffu, m);
        if ((threadIdx.x & 31) == 0) atomicMax(&s_m[j], m);
    }
    __syncthreads();
    if (threadIdx.x < P) {
        uint32_t m = s_m[threadIdx.x];
        if (m >= 0x7f800000u) {
            if (blockIdx.x == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);
            m = 0;
        }
        const float tmax = tanh_b(__uint_as_float(m));   // max |fl32(tanh)| = fl32(tanh(max |x|))
        const float st = (tmax == 0.0f) ? 1.0f : __fdiv_rn(127.0f, tmax);
        s_st[threadIdx.x] = make_float4(st, att_threshold(st), att_e_threshold(st), 0.0f);
    }
    __syncthreads();
    att_score_body<false>(g, sap, red5, &s_done, s, P, l, i0, nullptr, nullptr, s_st);
}

// one-MUFU scorer where every live hypothesis of the sentence is eligible, else two-MUFU
__global__ void __launch_bounds__(AT, 4)
k_att_score6(ScoreArgs g) {
    pdl_entry();
    extern __shared__ float4 sap[];   // [APC5][AQ5][AT]
    __shared__ int red5[AMAXP][APC5][AT / 32];
    __shared__ int s_done;
    const int s = blockIdx.y;
    const int P = g.sent_ncols[s], l = g.sent_len[s], i0 = blockIdx.x * APC5;
    if (P == 0 || i0 >= l) return;
    __shared__ int fixl[ATT_FIXCAP];
    __shared__ int s_nfix;
    const int c0 = g.sent_col_off[s];
    bool elig = true;
    for (int j = 0; j < P; ++j) elig &= g.st_thr[c0 + j].w != 0.0f;
    if (elig)
        att_score_body<true>(g, sap, red5, &s_done, s, P, l, i0, fixl, &s_nfix);
    else
        att_score_body<false>(g, sap, red5, &s_done, s, P, l, i0);
}

// ---------------------------------------------------------------------------
// k_att_score7: the one-MUFU scorer, restructured for latency hiding.
//   * The CTA's tile (E_ap rows i0 .. i0+np of the sentence: contiguous in HBM)
//     arrives by ONE cp.async.bulk, issued before the programmatic-dependent-
//     launch wait: E_ap is fixed for the whole batch, so the copy overlaps the
//     predecessor kernel's tail and no registers stage it.
//   * The smem layout [p][A/4] float4 gives thread t quads t + AT*k of every
//     row (the same slots score5/6 use).  The element loop runs all APC7
//     positions unconditionally (rows past np hold stale data whose sums are
//     discarded), so the compiler interleaves 48 independent elements per
//     hypothesis: per element FFMA, MUFU.RCP, FFMA, 3 FADD, 1/2 FMNMX3, IMAD.
//   * Elements inside the rounding window are queued (thread, position,
//     hypothesis) and resolved exactly by the CTA's last warp (att_fix_slot).
// Needs A == 4*AT*AQ5 (2048) or smaller with A % 4 == 0, and every hypothesis
// of the sentence eligible (|att_proj|, |u| <= 20); k_att_score7 falls back to
// the two-MUFU body for the others (as score6).
constexpr int APC7 = APC5;
static_assert(APC7 == APC5, "score7 falls back to the score5 body on the same position chunks");

// 1-D TMA bulk copy global -> shared, completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(tc::smem_u32(dst)), "l"(src), "r"(bytes), "r"(tc::smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(AT, 4)
k_att_score7(ScoreArgs g) {
    extern __shared__ __align__(128) float4 sap7[];   // [APC7][AQ5 * AT]
    __shared__ __align__(8) uint64_t bar;
    __shared__ int red7[AMAXP][APC7][AT / 32];
    __shared__ int s_done, s_nfix;
    __shared__ int fixl[ATT_FIXCAP];
    const int s = blockIdx.y;
    const int i0 = blockIdx.x * APC7;
    // per-batch constants (encoder layout, E_ap): safe before the PDL wait
    const int l = g.sent_len[s];
    if (i0 >= l) {
        pdl_entry();
        return;
    }
    const int np = min(l - i0, APC7);
    const int64_t A = g.A, A4 = A / 4;
    const int64_t row0 = g.sent_row[s] + i0;
    const bool tma = g.att_exp != nullptr && A4 <= AQ5 * AT;
    if (threadIdx.x == 0 && tma) {   // one row per copy: smem rows have the fixed stride AQ5 * AT quads
        tc::mbar_init(&bar, 1);
        tc::fence_mbar_init();
        tc::mbar_arrive_expect_tx(&bar, (uint32_t)(np * A * 4));
        for (int p = 0; p < np; ++p)
            bulk_g2s(sap7 + p * (AQ5 * AT), g.att_exp + (row0 + p) * A, (uint32_t)(A * 4), &bar);
    }
    pdl_entry();
    const int P = g.sent_ncols[s];
    const int c0 = g.sent_col_off[s];
    bool elig = tma && P > 0;
    for (int j = 0; j < P; ++j) elig &= g.st_thr[c0 + j].w != 0.0f;
    if (!elig) {
        if (tma) {   // the copy must land before the CTA's shared memory is reused
            __syncthreads();
            tc::mbar_wait(&bar, 0);
        }
        if (P == 0) return;
        __syncthreads();   // everyone is past the wait before the tile is overwritten
        att_score_body<false>(g, sap7, red7, &s_done, s, P, l, i0);
        return;
    }
    if (threadIdx.x == 0) {
        s_done = 0;
        s_nfix = 0;
    }
    const int lane = threadIdx.x & 31;
    int vv4[AQ5];      // the thread's v codes, four int8 per register (dp4a operand)
    float4 uq[AQ5], ux[AQ5];
#pragma unroll
    for (int k = 0; k < AQ5; ++k) {
        const int64_t q = threadIdx.x + (int64_t)AT * k;
        const bool ok = q < A4;
        vv4[k] = ok ? reinterpret_cast<const int*>(g.v_codes)[q] : 0;
        uq[k] = ok ? reinterpret_cast<const float4*>(g.eu + (int64_t)c0 * A)[q] : make_float4(1.f, 1.f, 1.f, 1.f);
    }
    float4 sp = g.st_thr[c0];
    __syncthreads();   // s_done / s_nfix initialised
    tc::mbar_wait(&bar, 0);
    for (int j = 0; j < P; ++j) {
        float4 spx = sp;
        if (j + 1 < P) {   // prefetch the next hypothesis' E_u slice and scale
#pragma unroll
            for (int k = 0; k < AQ5; ++k) {
                const int64_t q = threadIdx.x + (int64_t)AT * k;
                ux[k] = q < A4 ? reinterpret_cast<const float4*>(g.eu + (int64_t)(c0 + j + 1) * A)[q]
                               : make_float4(1.f, 1.f, 1.f, 1.f);
            }
            spx = g.st_thr[c0 + j + 1];
        }
        const float st = sp.x, thr = sp.z, m2st = -2.0f * st;
        int acc[APC7];
        float dmx[APC7];
#pragma unroll
        for (int p = 0; p < APC7; ++p) {
            acc[p] = 0;
            dmx[p] = 0.0f;
#pragma unroll
            for (int k = 0; k < AQ5; ++k) {
                const float4 e4 = sap7[p * (AQ5 * AT) + k * AT + threadIdx.x];
                uint32_t mb[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float r = rcp_approx(fmaf((&e4.x)[e], (&uq[k].x)[e], 1.0f));
                    const float v = fmaf(m2st, r, st);
                    const float mg = __fadd_rn(v, 12582912.0f);   // 1.5 * 2^23: round to integer
                    dmx[p] = fmaxf(dmx[p], fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))));
                    mb[e] = __float_as_uint(mg);   // low byte = the code (two's complement, |code| <= 127)
                }
                // pack the four codes' low bytes (PRMT) and dot them with four v codes (IDP4A)
                const uint32_t lo = __byte_perm(mb[0], mb[1], 0x0040), hi = __byte_perm(mb[2], mb[3], 0x0040);
                acc[p] = __dp4a((int)__byte_perm(lo, hi, 0x5410), vv4[k], acc[p]);
            }
        }
#pragma unroll
        for (int p = 0; p < APC7; ++p) {
            if (p < np && dmx[p] > thr) {   // rare: queue the slot for the exact pass
                const int slot = atomicAdd(&s_nfix, 1);
                if (slot < g.fixcap) fixl[slot] = j | (p << 4) | ((int)threadIdx.x << 7);
            }
            const int t = __reduce_add_sync(0xffffffffu, acc[p]);
            if (lane == 0) red7[j][p][threadIdx.x >> 5] = t;
        }
#pragma unroll
        for (int k = 0; k < AQ5; ++k) uq[k] = ux[k];
        sp = spx;
    }
    int last = 0;
    if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&s_done, 1) == AT / 32 - 1;
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence_block();
    {   // deferred exact codes of the queued slots (queue overflow: every slot of the CTA)
        const bool all = s_nfix > g.fixcap;
        const int nf = all ? P * np * AT : s_nfix;
        for (int f = lane; f < nf; f += 32) {
            const int e = all ? (f / (np * AT)) | (((f / AT) % np) << 4) | ((f % AT) << 7) : fixl[f];
            const float4 spj = g.st_thr[c0 + (e & 15)];
            const int d = att_fix_slot(sap7, g.att_proj + row0 * A, A, g.u + (int64_t)c0 * g.ldu, g.ldu,
                                       g.eu + (int64_t)c0 * A, g.v_codes, e, spj.x, spj.z);
            if (d) atomicAdd(&red7[e & 15][(e >> 4) & 7][0], d);
        }
        __syncwarp();
    }
    for (int idx = lane; idx < P * np; idx += 32) {
        const int j = idx / np, p = idx % np;
        int t = 0;
#pragma unroll
        for (int w = 0; w < AT / 32; ++w) t += red7[j][p][w];
        g.scores[(int64_t)(c0 + j) * g.max_len + i0 + p] = dequant(t, g.v_scale[0], g.st_thr[c0 + j].x);
    }
}

// ---------------------------------------------------------------------------
// k_att_score8: the two-MUFU scorer (codes identical to score5) restructured like
// score7: the CTA's att_proj tile (rows i0 .. i0+np, contiguous) arrives by one
// cp.async.bulk issued before the PDL wait (att_proj is fixed for the batch), so
// no registers or instructions stage it; the 6-position element loop runs
// unconditionally (stale rows are discarded) and the codes are summed by dp4a.
// A position with an element inside the rounding window is rescanned inline from
// the tile in shared memory (x = fl(ap + u) needs no global access), flagged
// elements with the fp64 tanh.  Sentences with a degenerate scale (some
// hypothesis' max |tanh| < 1.3e-4) take the score5 body.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(AT, 4)
k_att_score8(ScoreArgs g) {
    extern __shared__ __align__(128) float4 sap8[];   // [APC7][AQ5 * AT] = [p][A/4]
    __shared__ __align__(8) uint64_t bar;
    __shared__ int red8[AMAXP][APC7][AT / 32];
    __shared__ int s_done;
    const int s = blockIdx.y;
    const int i0 = blockIdx.x * APC7;
    const int l = g.sent_len[s];   // per-batch constants: safe before the PDL wait
    if (i0 >= l) {
        pdl_entry();
        return;
    }
    const int np = min(l - i0, APC7);
    const int64_t A = g.A, A4 = A / 4;
    const int64_t row0 = g.sent_row[s] + i0;
    if (threadIdx.x == 0) {   // one row per copy: smem rows have the fixed stride AQ5 * AT quads
        tc::mbar_init(&bar, 1);
        tc::fence_mbar_init();
        tc::mbar_arrive_expect_tx(&bar, (uint32_t)(np * A * 4));
        for (int p = 0; p < np; ++p)
            bulk_g2s(sap8 + p * (AQ5 * AT), g.att_proj + (row0 + p) * A, (uint32_t)(A * 4), &bar);
    }
    pdl_entry();
    const int P = g.sent_ncols[s];
    const int c0 = g.sent_col_off[s];
    bool fast = P > 0;
    for (int j = 0; j < P; ++j) fast &= g.st_thr[c0 + j].x <= ATT_ST_FAST_MAX;
    if (!fast) {
        __syncthreads();
        tc::mbar_wait(&bar, 0);   // the copy lands before the tile is restaged / the CTA exits
        if (P == 0) return;
        __syncthreads();
        att_score_body<false>(g, sap8, red8, &s_done, s, P, l, i0);
        return;
    }
    if (threadIdx.x == 0) s_done = 0;
    const int lane = threadIdx.x & 31;
    int vv4[AQ5];   // four int8 v codes per register (dp4a operand)
    float4 uq[AQ5], ux[AQ5];
#pragma unroll
    for (int k = 0; k < AQ5; ++k) {
        const int64_t q = threadIdx.x + (int64_t)AT * k;
        const bool ok = q < A4;
        vv4[k] = ok ? reinterpret_cast<const int*>(g.v_codes)[q] : 0;
        uq[k] = ok ? reinterpret_cast<const float4*>(g.u + (int64_t)c0 * g.ldu)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4 sp = g.st_thr[c0];
    __syncthreads();   // s_done initialised
    tc::mbar_wait(&bar, 0);
    for (int j = 0; j < P; ++j) {
        float4 spx = sp;
        if (j + 1 < P) {   // prefetch the next hypothesis' query slice and scale
#pragma unroll
            for (int k = 0; k < AQ5; ++k) {
                const int64_t q = threadIdx.x + (int64_t)AT * k;
                ux[k] = q < A4 ? reinterpret_cast<const float4*>(g.u + (int64_t)(c0 + j + 1) * g.ldu)[q]
                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            spx = g.st_thr[c0 + j + 1];
        }
        const float st = sp.x, thr = sp.y, m2st = -2.0f * st;
        int acc[APC7];
        float dmx[APC7];
#pragma unroll
        for (int p = 0; p < APC7; ++p) {
            acc[p] = 0;
            dmx[p] = 0.0f;
#pragma unroll
            for (int k = 0; k < AQ5; ++k) {
                const float4 a4 = sap8[p * (AQ5 * AT) + k * AT + threadIdx.x];
                uint32_t mb[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float x = __fadd_rn((&a4.x)[e], (&uq[k].x)[e]);
                    const float r = rcp_approx(__fadd_rn(ex2_approx(__fmul_rn(x, 2.8853900817779268f)), 1.0f));
                    const float v = fmaf(m2st, r, st);
                    const float mg = __fadd_rn(v, 12582912.0f);   // 1.5 * 2^23: round to integer
                    dmx[p] = fmaxf(dmx[p], fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))));
                    mb[e] = __float_as_uint(mg);   // low byte = the code
                }
                const uint32_t lo = __byte_perm(mb[0], mb[1], 0x0040), hi = __byte_perm(mb[2], mb[3], 0x0040);
                acc[p] = __dp4a((int)__byte_perm(lo, hi, 0x5410), vv4[k], acc[p]);
            }
        }
#pragma unroll
        for (int p = 0; p < APC7; ++p) {
            if (p < np && dmx[p] > thr) {   // rare: exact codes of this position's window elements
                int d = 0;
#pragma unroll
                for (int k = 0; k < AQ5; ++k) {
                    const float4 a4 = sap8[p * (AQ5 * AT) + k * AT + threadIdx.x];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float x = __fadd_rn((&a4.x)[e], (&uq[k].x)[e]);
                        const float r = rcp_approx(__fadd_rn(ex2_approx(__fmul_rn(x, 2.8853900817779268f)), 1.0f));
                        const float v = fmaf(m2st, r, st);
                        const float mg = __fadd_rn(v, 12582912.0f);
                        const int va = (int)(int8_t)(vv4[k] >> (8 * e));
                        if (fabsf(__fsub_rn(v, __fsub_rn(mg, 12582912.0f))) > thr && va != 0)
                            d += va * (att_code_exact(x, st) - (int)(int8_t)(__float_as_uint(mg) & 0xffu));
                    }
                }
                acc[p] += d;
            }
            const int t = __reduce_add_sync(0xffffffffu, acc[p]);
            if (lane == 0) red8[j][p][threadIdx.x >> 5] = t;
        }
#pragma unroll
        for (int k = 0; k < AQ5; ++k) uq[k] = ux[k];
        sp = spx;
    }
    int last = 0;
    if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&s_done, 1) == AT / 32 - 1;
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence_block();
    for (int idx = lane; idx < P * np; idx += 32) {
        const int j = idx / np, p = idx % np;
        int t = 0;
#pragma unroll
        for (int w = 0; w < AT / 32; ++w) t += red8[j][p][w];
        g.scores[(int64_t)(c0 + j) * g.max_len + i0 + p] = dequant(t, g.v_scale[0], g.st_thr[c0 + j].x);
    }
}

// softmax over the l scores of every hypothesis of sentence s (fp64, fixed
// sequential sum order) into smem alpha, position-major ([i][AMAXP]) so the
// context loop reads it with broadcast loads, widened to f64 once.
__device__ __forceinline__ void att_softmax(const float* __restrict__ scores, int32_t max_len, int P, int l, int c0,
                                            double* ex, double* al, float* __restrict__ alpha, int64_t lda,
                                            int32_t* err_flag, int pst = AMAXP) {
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
        for (int i = lane; i < l; i += 32) {   // exp below e^-700 contributes nothing (sum >= 1)
            const double t = (double)sc[i] - (double)m;
            ex[j * max_len + i] = t < -700.0 ? 0.0 : exp_f64(t);
        }
        __syncwarp();
        double sum = 0.0;
        if (lane == 0)
            for (int i = 0; i < l; ++i) sum += ex[j * max_len + i];
        sum = __shfl_sync(0xffffffffu, sum, 0);
        for (int i = lane; i < l; i += 32) {
            const float a = __double2float_rn(ex[j * max_len + i] / sum);
            al[i * pst + j] = (double)a;
            if (alpha && blockIdx.x == 0) alpha[(int64_t)(c0 + j) * lda + i] = a;
        }
    }
}

// ctx[c] = fl32(sum_i f64(states[R+i][c]) * f64(alpha_i)) for the features of
// this thread: 4 consecutive (V4, float4 loads) or one; P fp64 FMAs per value.
template <int P, bool V4>
__device__ __forceinline__ uint32_t att_context_acc(const float* __restrict__ st_row0, int64_t H2, int l,
                                                    const double* al, int64_t c, float* __restrict__ ctx,
                                                    int64_t ldc, int c0) {
    constexpr int W = V4 ? 4 : 1;
    uint32_t mx = 0;
    if (c >= H2) return 0;
    const float* st = st_row0 + c;
    double acc[P][W];
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
        for (int e = 0; e < W; ++e) acc[j][e] = 0.0;
    auto load = [&](int i, float (&d)[W]) {   // widened to f64 at use
        if (V4) {
            const float4 q = *reinterpret_cast<const float4*>(st + (int64_t)i * H2);
            d[0] = q.x;
            if (W > 1) { d[W > 1 ? 1 : 0] = q.y; d[W > 2 ? 2 : 0] = q.z; d[W > 3 ? 3 : 0] = q.w; }
        } else {
            d[0] = st[(int64_t)i * H2];
        }
    };
    int i = 0;
    for (; i + 4 <= l; i += 4) {
        float d[4][W];
#pragma unroll
        for (int q = 0; q < 4; ++q) load(i + q, d[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const double aj = al[(i + q) * AMAXP + j];
#pragma unroll
                for (int e = 0; e < W; ++e) acc[j][e] += (double)d[q][e] * aj;
            }
    }
    for (; i < l; ++i) {
        float d[W];
        load(i, d);
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const double aj = al[i * AMAXP + j];
#pragma unroll
            for (int e = 0; e < W; ++e) acc[j][e] += (double)d[e] * aj;
        }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) {
        float v[W];
#pragma unroll
        for (int e = 0; e < W; ++e) {
            v[e] = __double2float_rn(acc[j][e]);
            mx = max(mx, __float_as_uint(v[e]) & 0x7fffffffu);
        }
        float* dst = ctx + (int64_t)(c0 + j) * ldc + c;
        if (V4)
            *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[W > 1 ? 1 : 0], v[W > 2 ? 2 : 0], v[W > 3 ? 3 : 0]);
        else
            dst[0] = v[0];
    }
    return mx;
}

// Grid (features / (V4 ? 4 AT : AT), sentences).  V4 CTAs of sentences with more
// than 6 live hypotheses run the scalar accumulation 4 times (register bound).
__global__ void __launch_bounds__(AT)
k_att_context3(const float* __restrict__ scores, int32_t max_len, const int32_t* __restrict__ sent_col_off,
               const int32_t* __restrict__ sent_ncols, const float* __restrict__ states,
               const int64_t* __restrict__ sent_row, const int32_t* __restrict__ sent_len, int64_t H2,
               float* __restrict__ ctx, int64_t ldc, float* __restrict__ alpha, int64_t lda, int32_t* err_flag,
               uint32_t* ctx_segmax, int v4) {
    pdl_entry();
    extern __shared__ unsigned char smem_raw[];
    const int s = blockIdx.y;
    const int P = sent_ncols[s];
    if (P == 0) return;   // sentence finished
    const int l = sent_len[s];
    const int c0 = sent_col_off[s];
    double* ex = reinterpret_cast<double*>(smem_raw);   // [AMAXP][max_len]
    double* al = ex + AMAXP * max_len;                 // [max_len][AMAXP]
    att_softmax(scores, max_len, P, l, c0, ex, al, alpha, lda, err_flag);
    __syncthreads();
    const float* st0 = states + sent_row[s] * H2;
    uint32_t mx = 0;
#define QNMT_CTX_P(P_, V4_, C_) \
    case P_: mx = max(mx, att_context_acc<P_, V4_>(st0, H2, l, al, (C_), ctx, ldc, c0)); break;
    if (v4 && P <= 6) {
        const int64_t c = ((int64_t)blockIdx.x * AT + threadIdx.x) * 4;
        switch (P) {
            QNMT_CTX_P(1, true, c) QNMT_CTX_P(2, true, c) QNMT_CTX_P(3, true, c) QNMT_CTX_P(4, true, c)
            QNMT_CTX_P(5, true, c) QNMT_CTX_P(6, true, c)
            default: break;
        }
    } else {
        const int reps = v4 ? 4 : 1;
        for (int r = 0; r < reps; ++r) {
            const int64_t c = (int64_t)blockIdx.x * AT * reps + (int64_t)r * AT + threadIdx.x;
            switch (P) {
                QNMT_CTX_P(1, false, c) QNMT_CTX_P(2, false, c) QNMT_CTX_P(3, false, c) QNMT_CTX_P(4, false, c)
                QNMT_CTX_P(5, false, c) QNMT_CTX_P(6, false, c) QNMT_CTX_P(7, false, c) QNMT_CTX_P(8, false, c)
                QNMT_CTX_P(9, false, c) QNMT_CTX_P(10, false, c) QNMT_CTX_P(11, false, c) QNMT_CTX_P(12, false, c)
                QNMT_CTX_P(13, false, c) QNMT_CTX_P(14, false, c) QNMT_CTX_P(15, false, c) QNMT_CTX_P(16, false, c)
                default: break;
            }
        }
    }
#undef QNMT_CTX_P
    if (ctx_segmax) {   // per-sentence max |ctx| for the next quantization (segment = sentence)
        mx = __reduce_max_sync(0xffffffffu, mx);
        if ((threadIdx.x & 31) == 0 && mx) atomicMax(ctx_segmax + s, mx);
    }
}

// ---------------------------------------------------------------------------
// k_att_context4: the context sum with the encoder states staged by TMA bulk
// copies (cp.async.bulk, one 4 KB row slice per position) into a 5-stage
// shared-memory ring of 4 positions each, so HBM streams at full depth
// instead of a few float4 loads per thread in flight.  The states do not
// depend on the predecessor kernel (they are the batch's encoder output), so
// the first stages are issued before the programmatic-dependent-launch wait
// and overlap the scorer's tail.  Same arithmetic and summation order as
// k_att_context3 (sequential over positions, fp64 FMAs).  Sentences with more
// than 8 live hypotheses (register bound) drain the ring and use the direct
// loads of k_att_context3.
// ---------------------------------------------------------------------------
constexpr int ACF = 4 * AT;   // features per CTA (one float4 per thread)
constexpr int ACH = 4;        // positions per stage
constexpr int ACS = 5;        // stages (80 KB ring + softmax arrays: 2 CTAs / SM)
constexpr int ACP_MAX = 8;    // hypotheses per sentence supported by context4


template <int P>
__device__ __forceinline__ uint32_t att_context_staged(const float* buf, uint64_t* full, const float* src0,
                                                       int64_t H2, uint32_t row_bytes, int l, const double* al,
                                                       int64_t c, bool cok, float* __restrict__ ctx, int64_t ldc,
                                                       int c0) {
    double acc[P][4];
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] = 0.0;
    const int nst = (l + ACH - 1) / ACH;
    for (int k = 0; k < nst; ++k) {
        const int b = k % ACS;
        tc::mbar_wait(&full[b], (uint32_t)(k / ACS) & 1u);
        const int np = min(ACH, l - k * ACH);
        const float4* bp = reinterpret_cast<const float4*>(buf + (size_t)b * ACH * ACF) + threadIdx.x;
#pragma unroll 4
        for (int p = 0; p < np; ++p) {
            const float4 q = bp[p * (ACF / 4)];
            const double d[4] = {(double)q.x, (double)q.y, (double)q.z, (double)q.w};
            const double* ap = al + (k * ACH + p) * AMAXP;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const double aj = ap[j];
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[j][e] += d[e] * aj;
            }
        }
        __syncthreads();   // every thread is done with buffer b
        if (threadIdx.x == 0 && k + ACS < nst) {
            const int k2 = k + ACS, n2 = min(ACH, l - k2 * ACH);
            tc::mbar_arrive_expect_tx(&full[b], (uint32_t)n2 * row_bytes);
            for (int p = 0; p < n2; ++p)
                bulk_g2s(const_cast<float*>(buf) + ((size_t)b * ACH + p) * ACF, src0 + (int64_t)(k2 * ACH + p) * H2,
                         row_bytes, &full[b]);
        }
    }
    uint32_t mx = 0;
    if (!cok) return 0;
#pragma unroll
    for (int j = 0; j < P; ++j) {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            v[e] = __double2float_rn(acc[j][e]);
            mx = max(mx, __float_as_uint(v[e]) & 0x7fffffffu);
        }
        *reinterpret_cast<float4*>(ctx + (int64_t)(c0 + j) * ldc + c) = make_float4(v[0], v[1], v[2], v[3]);
    }
    return mx;
}

// Grid (ceil(H2 / ACF), sentences).  Requires H2 % 4 == 0, 16-byte aligned states/ctx rows.
__global__ void __launch_bounds__(AT, 2)
k_att_context4(const float* __restrict__ scores, int32_t max_len, const int32_t* __restrict__ sent_col_off,
               const int32_t* __restrict__ sent_ncols, const float* __restrict__ states,
               const int64_t* __restrict__ sent_row, const int32_t* __restrict__ sent_len, int64_t H2,
               float* __restrict__ ctx, int64_t ldc, float* __restrict__ alpha, int64_t lda, int32_t* err_flag,
               uint32_t* ctx_segmax) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[ACS];
    float* buf = reinterpret_cast<float*>(smem_raw);                      // [ACS][ACH][ACF]
    double* ex = reinterpret_cast<double*>(buf + (size_t)ACS * ACH * ACF);  // [AMAXP][max_len]
    double* al = ex + AMAXP * max_len;                                    // [max_len][AMAXP]
    const int s = blockIdx.y;
    // sentence metadata and states were written >= 2 kernels ago (the scorer waits for its own
    // predecessor before triggering us): safe to read before the PDL wait
    const int P = sent_ncols[s];
    const int l = sent_len[s];
    const int64_t cb = (int64_t)blockIdx.x * ACF;
    const int64_t nfeat = min((int64_t)ACF, H2 - cb);
    const uint32_t row_bytes = (uint32_t)(nfeat * 4);
    const float* src0 = states + sent_row[s] * H2 + cb;
    const int nst = (l + ACH - 1) / ACH;
    if (P > 0 && threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < ACS; ++b) tc::mbar_init(&full[b], 1);
        tc::fence_mbar_init();
        for (int k = 0; k < min(ACS, nst); ++k) {
            const int np = min(ACH, l - k * ACH);
            tc::mbar_arrive_expect_tx(&full[k], (uint32_t)np * row_bytes);
            for (int p = 0; p < np; ++p)
                bulk_g2s(buf + ((size_t)k * ACH + p) * ACF, src0 + (int64_t)(k * ACH + p) * H2, row_bytes, &full[k]);
        }
    }
    pdl_entry();
    if (P == 0) return;   // sentence finished
    const int c0 = sent_col_off[s];
    att_softmax(scores, max_len, P, l, c0, ex, al, alpha, lda, err_flag);
    __syncthreads();   // al ready; barriers initialised
    const int64_t c = cb + 4 * threadIdx.x;
    const bool cok = 4 * threadIdx.x < nfeat;
    uint32_t mx = 0;
#define QNMT_CTX4(P_) \
    case P_: mx = att_context_staged<P_>(buf, full, src0, H2, row_bytes, l, al, c, cok, ctx, ldc, c0); break;
    switch (P) {
        QNMT_CTX4(1) QNMT_CTX4(2) QNMT_CTX4(3) QNMT_CTX4(4) QNMT_CTX4(5) QNMT_CTX4(6) QNMT_CTX4(7) QNMT_CTX4(8)
        default: break;
    }
#undef QNMT_CTX4
    if (P > ACP_MAX) {   // wide beams (register bound): drain the staged copies, read states directly
        for (int k = 0; k < min(ACS, nst); ++k) tc::mbar_wait(&full[k], 0);
        const float* st0 = states + sent_row[s] * H2;
        for (int r = 0; r < 4; ++r) {
            const int64_t cc = cb + (int64_t)r * AT + threadIdx.x;
            if (cc >= cb + nfeat) break;
            switch (P) {
#define QNMT_CTX4W(P_) case P_: mx = max(mx, att_context_acc<P_, false>(st0, H2, l, al, cc, ctx, ldc, c0)); break;
                QNMT_CTX4W(9) QNMT_CTX4W(10) QNMT_CTX4W(11) QNMT_CTX4W(12) QNMT_CTX4W(13) QNMT_CTX4W(14)
                QNMT_CTX4W(15) QNMT_CTX4W(16)
#undef QNMT_CTX4W
                default: break;
            }
        }
    }
    if (ctx_segmax) {
        mx = __reduce_max_sync(0xffffffffu, mx);
        if ((threadIdx.x & 31) == 0 && mx) atomicMax(ctx_segmax + s, mx);
    }
}

// k_att_context5: k_att_context4 with half the features per CTA (one float2 per
// thread, 512 features: 4 CTAs per sentence at 2H = 2048) and the softmax arrays
// sized by the batch's hypothesis bound pst instead of 16: ~48 KB of shared
// memory and 2 x P doubles of accumulators per thread, so 4 CTAs / SM stream
// twice as many sentences' states at once (context4: 2 CTAs / SM, 25-45% of
// HBM bandwidth at N = 1280).  Same arithmetic and summation order.
constexpr int AC5F = 2 * AT;   // features per CTA
constexpr int AC5S = 5;        // ring stages of ACH positions (40 KB)

template <int P>
__device__ __forceinline__ uint32_t att_context_staged2(const float* buf, uint64_t* full, const float* src0,
                                                        int64_t H2, uint32_t row_bytes, int l, const double* al,
                                                        int pst, int64_t c, bool cok, float* __restrict__ ctx,
                                                        int64_t ldc, int c0) {
    double acc[P][2];
#pragma unroll
    for (int j = 0; j < P; ++j) acc[j][0] = acc[j][1] = 0.0;
    const int nst = (l + ACH - 1) / ACH;
    for (int k = 0; k < nst; ++k) {
        const int b = k % AC5S;
        tc::mbar_wait(&full[b], (uint32_t)(k / AC5S) & 1u);
        const int np = min(ACH, l - k * ACH);
        const float2* bp = reinterpret_cast<const float2*>(buf + (size_t)b * ACH * AC5F) + threadIdx.x;
#pragma unroll 4
        for (int p = 0; p < np; ++p) {
            const float2 q = bp[p * (AC5F / 2)];
            const double d0 = (double)q.x, d1 = (double)q.y;
            const double* ap = al + (k * ACH + p) * pst;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const double aj = ap[j];
                acc[j][0] += d0 * aj;
                acc[j][1] += d1 * aj;
            }
        }
        __syncthreads();   // every thread is done with buffer b
        if (threadIdx.x == 0 && k + AC5S < nst) {
            const int k2 = k + AC5S, n2 = min(ACH, l - k2 * ACH);
            tc::mbar_arrive_expect_tx(&full[b], (uint32_t)n2 * row_bytes);
            for (int p = 0; p < n2; ++p)
                bulk_g2s(const_cast<float*>(buf) + ((size_t)b * ACH + p) * AC5F,
                         src0 + (int64_t)(k2 * ACH + p) * H2, row_bytes, &full[b]);
        }
    }
    uint32_t mx = 0;
    if (!cok) return 0;
#pragma unroll
    for (int j = 0; j < P; ++j) {
        const float v0 = __double2float_rn(acc[j][0]), v1 = __double2float_rn(acc[j][1]);
        mx = max(mx, max(__float_as_uint(v0) & 0x7fffffffu, __float_as_uint(v1) & 0x7fffffffu));
        *reinterpret_cast<float2*>(ctx + (int64_t)(c0 + j) * ldc + c) = make_float2(v0, v1);
    }
    return mx;
}

// Grid (ceil(H2 / AC5F), sentences).  Requires H2 % 2 == 0, 8-byte aligned states/ctx
// rows, and every sentence's live hypotheses <= pst <= ACP_MAX.
__global__ void __launch_bounds__(AT, 4)
k_att_context5(const float* __restrict__ scores, int32_t max_len, const int32_t* __restrict__ sent_col_off,
               const int32_t* __restrict__ sent_ncols, const float* __restrict__ states,
               const int64_t* __restrict__ sent_row, const int32_t* __restrict__ sent_len, int64_t H2,
               float* __restrict__ ctx, int64_t ldc, float* __restrict__ alpha, int64_t lda, int32_t* err_flag,
               uint32_t* ctx_segmax, int pst) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[AC5S];
    float* buf = reinterpret_cast<float*>(smem_raw);                         // [AC5S][ACH][AC5F]
    double* ex = reinterpret_cast<double*>(buf + (size_t)AC5S * ACH * AC5F);  // [pst][max_len]
    double* al = ex + (size_t)pst * max_len;                                 // [max_len][pst]
    const int s = blockIdx.y;
    // as context4: sentence metadata and states are >= 2 kernels old, safe before the PDL wait
    const int P = sent_ncols[s];
    const int l = sent_len[s];
    const int64_t cb = (int64_t)blockIdx.x * AC5F;
    const int64_t nfeat = min((int64_t)AC5F, H2 - cb);
    const uint32_t row_bytes = (uint32_t)(nfeat * 4);
    const float* src0 = states + sent_row[s] * H2 + cb;
    const int nst = (l + ACH - 1) / ACH;
    const bool run = P > 0 && P <= pst;
    if (run && threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < AC5S; ++b) tc::mbar_init(&full[b], 1);
        tc::fence_mbar_init();
        for (int k = 0; k < min(AC5S, nst); ++k) {
            const int np = min(ACH, l - k * ACH);
            tc::mbar_arrive_expect_tx(&full[k], (uint32_t)np * row_bytes);
            for (int p = 0; p < np; ++p)
                bulk_g2s(buf + ((size_t)k * ACH + p) * AC5F, src0 + (int64_t)(k * ACH + p) * H2, row_bytes, &full[k]);
        }
    }
    pdl_entry();
    if (!run) {
        if (P > pst && threadIdx.x == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);   // host bound violated
        return;
    }
    const int c0 = sent_col_off[s];
    att_softmax(scores, max_len, P, l, c0, ex, al, alpha, lda, err_flag, pst);
    __syncthreads();   // al ready; barriers initialised
    const int64_t c = cb + 2 * threadIdx.x;
    const bool cok = 2 * threadIdx.x < nfeat;
    uint32_t mx = 0;
#define QNMT_CTX5(P_) \
    case P_: mx = att_context_staged2<P_>(buf, full, src0, H2, row_bytes, l, al, pst, c, cok, ctx, ldc, c0); break;
    switch (P) {
        QNMT_CTX5(1) QNMT_CTX5(2) QNMT_CTX5(3) QNMT_CTX5(4) QNMT_CTX5(5) QNMT_CTX5(6) QNMT_CTX5(7) QNMT_CTX5(8)
        default: break;
    }
#undef QNMT_CTX5
    if (ctx_segmax) {
        mx = __reduce_max_sync(0xffffffffu, mx);
        if ((threadIdx.x & 31) == 0 && mx) atomicMax(ctx_segmax + s, mx);
    }
}

int attention_launch(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                     const int32_t* sent_ncols, int32_t n_sent, const float* att_proj, const float* att_minmax,
                     const float* states, const int64_t* sent_row, const int32_t* sent_len, int32_t max_len,
                     int64_t A, int64_t H2, const int8_t* v_codes, const float* v_scale, float* ctx, int64_t ldc,
                     float* alpha, int64_t lda, void* scratch, int32_t* err_flag, cudaStream_t st,
                     uint32_t* ctx_segmax, int max_p, const float* att_exp) {
    if (N <= 0 || n_sent <= 0) return QNMT_OK;
    const bool wide = A > (int64_t)AT * AKA;   // beyond the register-resident kernels: strided a-loops
    // scratch: scores [N][max_len] | st_thr [N] float4 | (column extrema [n_sent][2][A]) | (E_u [N][A])
    float* scores = reinterpret_cast<float*>(scratch);
    float4* st_thr = reinterpret_cast<float4*>(scores + ((N * max_len + 63) / 64) * 64);
    float* tail = reinterpret_cast<float*>(st_thr) + ((4 * N + 63) / 64) * 64;
    if (!att_minmax) {   // extrema not supplied by the caller: compute them into scratch
        float* mm = tail;
        tail += ((2 * (int64_t)n_sent * A + 63) / 64) * 64;
        TRY_LAUNCH(att_minmax_launch(att_proj, sent_row, sent_len, n_sent, A, mm, st));
        att_minmax = mm;
    }
    const bool quads = !wide && A % 4 == 0 && ldu % 4 == 0 && A <= 4 * AT * AQ5 && ((uintptr_t)u % 16) == 0 &&
                       ((uintptr_t)att_proj % 16) == 0 && ((uintptr_t)v_codes % 4) == 0;
    const bool expm = quads && att_exp != nullptr && g_att_exp && ((uintptr_t)att_exp % 16) == 0;
    const bool fused_scale = quads && !expm && g_att_fused_scale && ((uintptr_t)att_minmax % 16) == 0;
    float* eu = expm ? tail : nullptr;
    if (fused_scale) {   // k_att_score5f computes the scales itself
        const size_t smem5 = (size_t)APC5 * AQ5 * AT * sizeof(float4);
        static size_t done5f = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_att_score5f, smem5, done5f));
        ScoreArgs ga{u, ldu, sent_col_off, sent_ncols, att_proj, att_exp, nullptr, st_thr, sent_row, sent_len, A,
                     v_codes, v_scale, scores, max_len, 0};
        dim3 g5((unsigned)cdiv(max_len, APC5), (unsigned)n_sent);
        QNMT_LAUNCH(k_att_score5f, g5, AT, smem5, st, ga, att_minmax, err_flag, ctx_segmax);
        QNMT_CHECK_LAUNCH("k_att_score5f");
    } else if (wide) {
        QNMT_LAUNCH(k_att_scale_wide, dim3((unsigned)n_sent, AMAXP), AT, 0, st, u, ldu, sent_col_off, sent_ncols,
                    att_minmax, A, st_thr, err_flag, ctx_segmax);
        QNMT_CHECK_LAUNCH("k_att_scale_wide");
        dim3 gw((unsigned)cdiv(max_len, APC), (unsigned)n_sent);
        QNMT_LAUNCH(k_att_score_wide, gw, AT, 0, st, u, ldu, sent_col_off, sent_ncols, att_proj, st_thr, sent_row,
                    sent_len, A, v_codes, v_scale, scores, max_len);
        QNMT_CHECK_LAUNCH("k_att_score_wide");
    } else {
    QNMT_LAUNCH(k_att_scale, dim3((unsigned)n_sent, AMAXP), AT, 0, st, u, ldu, sent_col_off, sent_ncols, att_minmax, A,
                st_thr, err_flag, ctx_segmax, eu);
    QNMT_CHECK_LAUNCH("k_att_scale");
    if (quads) {   // smem-staged tile, 4 CTAs / SM
        const size_t smem5 = (size_t)APC5 * AQ5 * AT * sizeof(float4);
        static size_t done5 = 0, done6 = 0;   // (dynamic + static > 48 KB needs the opt-in)
        ScoreArgs ga{u, ldu, sent_col_off, sent_ncols, att_proj, att_exp, eu, st_thr, sent_row, sent_len, A,
                     v_codes, v_scale, scores, max_len, std::min(g_att_fixcap, ATT_FIXCAP_MAX)};
        dim3 g5((unsigned)cdiv(max_len, APC5), (unsigned)n_sent);
        if (expm && g_att_exp == 2) {
            static size_t done7 = 0;
            QNMT_CUDA(raise_smem_limit((const void*)k_att_score7, smem5, done7));
            QNMT_LAUNCH(k_att_score7, g5, AT, smem5, st, ga);
            QNMT_CHECK_LAUNCH("k_att_score7");
        } else if (expm) {
            QNMT_CUDA(raise_smem_limit((const void*)k_att_score6, smem5, done6));
            QNMT_LAUNCH(k_att_score6, g5, AT, smem5, st, ga);
            QNMT_CHECK_LAUNCH("k_att_score6");
        } else if (g_att_score8 && A4_FITS(A)) {
            static size_t done8 = 0;
            QNMT_CUDA(raise_smem_limit((const void*)k_att_score8, smem5, done8));
            QNMT_LAUNCH(k_att_score8, g5, AT, smem5, st, ga);
            QNMT_CHECK_LAUNCH("k_att_score8");
        } else {
            QNMT_CUDA(raise_smem_limit((const void*)k_att_score5, smem5, done5));
            QNMT_LAUNCH(k_att_score5, g5, AT, smem5, st, ga);
            QNMT_CHECK_LAUNCH("k_att_score5");
        }
    } else {
        dim3 g1((unsigned)cdiv(max_len, APC), (unsigned)n_sent);
        QNMT_LAUNCH(k_att_score4, g1, AT, 0, st, u, ldu, sent_col_off, sent_ncols, att_proj, st_thr, sent_row, sent_len, A,
                                        v_codes, v_scale, scores, max_len);
        QNMT_CHECK_LAUNCH("k_att_score4");
    }
    }   // !fused_scale
    const size_t smem = (size_t)AMAXP * max_len * 2 * sizeof(double);
    const bool v4 = H2 % 4 == 0 && ldc % 4 == 0 && ((uintptr_t)states % 16) == 0 && ((uintptr_t)ctx % 16) == 0;
    const dim3 g2((unsigned)cdiv(H2, v4 ? 4 * AT : AT), (unsigned)n_sent);
    const size_t smem4 = (size_t)ACS * ACH * ACF * sizeof(float) + smem;
    const int pst = std::max(1, max_p);
    const size_t smem5c = (size_t)AC5S * ACH * AC5F * sizeof(float) + (size_t)pst * max_len * 2 * sizeof(double);
    if (g_att_ctx_staged == 2 && pst <= ACP_MAX && H2 % 2 == 0 && ldc % 2 == 0 && ((uintptr_t)states % 8) == 0 &&
        ((uintptr_t)ctx % 8) == 0 && smem5c <= 200 * 1024) {
        static size_t done5c = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_att_context5, smem5c, done5c));
        const dim3 g5c((unsigned)cdiv(H2, AC5F), (unsigned)n_sent);
        QNMT_LAUNCH(k_att_context5, g5c, AT, smem5c, st, scores, max_len, sent_col_off, sent_ncols, states, sent_row,
                    sent_len, H2, ctx, ldc, alpha, lda, err_flag, ctx_segmax, pst);
        QNMT_CHECK_LAUNCH("k_att_context5");
        return QNMT_OK;
    }
    if (v4 && g_att_ctx_staged && smem4 <= 200 * 1024) {
        static size_t done4 = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_att_context4, smem4, done4));
        QNMT_LAUNCH(k_att_context4, g2, AT, smem4, st, scores, max_len, sent_col_off, sent_ncols, states, sent_row,
                    sent_len, H2, ctx, ldc, alpha, lda, err_flag, ctx_segmax);
        QNMT_CHECK_LAUNCH("k_att_context4");
        return QNMT_OK;
    }
    if (smem > 48 * 1024) {
        static size_t done = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_att_context3, smem, done));
    }
    QNMT_LAUNCH(k_att_context3, g2, AT, smem, st, scores, max_len, sent_col_off, sent_ncols, states, sent_row, sent_len, H2,
                                          ctx, ldc, alpha, lda, err_flag, ctx_segmax, v4 ? 1 : 0);
    QNMT_CHECK_LAUNCH("k_att_context3");
    return QNMT_OK;
}

// column -> sentence ranges for callers that only have col_sent (columns grouped by sentence)
// ---------------------------------------------------------------------------
// fp32 precision path: the scorer is a float LinearOp, so
//   score_i = fl32(sum_a f64(v_a) * f64(fl32(tanh(fl32(att_proj[R+i][a] + u[n][a])))))
// (gemm_f32 of layers.py:226 under the Tier-B fp64 contract), then the same
// softmax + context kernel as the int8 path.  One warp per (position, sentence)
// covers every live hypothesis of the sentence, so att_proj is read once.
// ---------------------------------------------------------------------------
constexpr int AFW = 8;   // warps (positions) per CTA

__global__ void __launch_bounds__(AFW * 32)
k_att_score_f32(const float* __restrict__ u, int64_t ldu, const int32_t* __restrict__ sent_col_off,
                const int32_t* __restrict__ sent_ncols, const float* __restrict__ att_proj,
                const int64_t* __restrict__ sent_row, const int32_t* __restrict__ sent_len, int64_t A,
                const float* __restrict__ v, float* __restrict__ scores, int32_t max_len, int32_t* err_flag) {
    pdl_entry();
    const int s = blockIdx.y;
    const int i = blockIdx.x * AFW + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int P = sent_ncols[s];
    if (P == 0 || i >= sent_len[s]) return;
    const int c0 = sent_col_off[s];
    const float* ap = att_proj + (sent_row[s] + i) * A;
    double acc[AMAXP];
#pragma unroll
    for (int j = 0; j < AMAXP; ++j) acc[j] = 0.0;
    bool bad = false;
    for (int64_t a = lane; a < A; a += 32) {
        const float at = ap[a];
        const double va = (double)v[a];
#pragma unroll
        for (int j = 0; j < AMAXP; ++j) {
            if (j < P) {
                const float x = __fadd_rn(at, u[(int64_t)(c0 + j) * ldu + a]);
                bad |= !is_finite_f(x);
                acc[j] = fma(va, (double)tanh_b(x), acc[j]);
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);
#pragma unroll
    for (int j = 0; j < AMAXP; ++j) {
        if (j < P) {
            const double t = warp_sum(acc[j]);
            if (lane == 0) scores[(int64_t)(c0 + j) * max_len + i] = __double2float_rn(t);
        }
    }
}

int attention_f32_launch(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                         const int32_t* sent_ncols, int32_t n_sent, const float* att_proj, const float* states,
                         const int64_t* sent_row, const int32_t* sent_len, int32_t max_len, int64_t A, int64_t H2,
                         const float* v, float* ctx, int64_t ldc, float* alpha, int64_t lda, void* scratch,
                         int32_t* err_flag, cudaStream_t st) {
    if (N <= 0 || n_sent <= 0) return QNMT_OK;
    float* scores = reinterpret_cast<float*>(scratch);   // [N][max_len]
    const dim3 g1((unsigned)cdiv(max_len, AFW), (unsigned)n_sent);
    QNMT_LAUNCH(k_att_score_f32, g1, AFW * 32, 0, st, u, ldu, sent_col_off, sent_ncols, att_proj, sent_row, sent_len,
                A, v, scores, max_len, err_flag);
    QNMT_CHECK_LAUNCH("k_att_score_f32");
    const size_t smem = (size_t)AMAXP * max_len * 2 * sizeof(double);
    const bool v4 = H2 % 4 == 0 && ldc % 4 == 0 && ((uintptr_t)states % 16) == 0 && ((uintptr_t)ctx % 16) == 0;
    const dim3 g2((unsigned)cdiv(H2, v4 ? 4 * AT : AT), (unsigned)n_sent);
    if (smem > 48 * 1024) {
        static size_t done = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_att_context3, smem, done));
    }
    QNMT_LAUNCH(k_att_context3, g2, AT, smem, st, scores, max_len, sent_col_off, sent_ncols, states, sent_row, sent_len,
                H2, ctx, ldc, alpha, lda, err_flag, (uint32_t*)nullptr, v4 ? 1 : 0);
    QNMT_CHECK_LAUNCH("k_att_context3");
    return QNMT_OK;
}

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
                              const float* att_minmax, const float* att_exp, const float* states,
                              const int64_t* sent_row, const int32_t* sent_len,
                              int32_t max_len, int64_t A, int64_t H2, const int8_t* v_codes,
                              const float* v_scale, float* ctx, int64_t ldc, float* alpha, int64_t lda,
                              void* scratch, int32_t* err_flag, void* stream) {
    return qnmt::attention_launch(u, ldu, N, sent_col_off, sent_ncols, n_sent, att_proj, att_minmax, states,
                                  sent_row,
                                  sent_len, max_len, A, H2, v_codes, v_scale, ctx, ldc, alpha, lda, scratch,
                                  err_flag, qnmt::as_stream(stream), nullptr, 16, att_exp);
}

extern "C" int qnmt_attention_exp(const float* att_proj, int64_t n, float* att_exp, void* stream) {
    return qnmt::att_exp_launch(att_proj, n, att_exp, qnmt::as_stream(stream));
}

extern "C" int qnmt_set_att_score8(int32_t enable) {
    const int old = qnmt::g_att_score8;
    qnmt::g_att_score8 = enable ? 1 : 0;
    return old;
}

extern "C" int qnmt_set_att_fused_scale(int32_t enable) {
    const int old = qnmt::g_att_fused_scale;
    qnmt::g_att_fused_scale = enable ? 1 : 0;
    return old;
}

extern "C" int qnmt_set_att_ctx(int32_t mode) {
    const int old = qnmt::g_att_ctx_staged;
    qnmt::g_att_ctx_staged = mode < 0 ? 0 : (mode > 2 ? 2 : mode);
    return old;
}

extern "C" int qnmt_set_att_fixcap(int32_t cap) {
    const int old = qnmt::g_att_fixcap;
    qnmt::g_att_fixcap = std::max(0, std::min((int)cap, qnmt::ATT_FIXCAP_MAX));
    return old;
}

extern "C" int qnmt_set_att_exp(int32_t enable) {
    const int old = qnmt::g_att_exp;
    qnmt::g_att_exp = enable < 0 ? 0 : (enable > 2 ? 2 : enable);
    return old;
}

extern "C" int qnmt_attention_stats(const float* att_proj, const int64_t* sent_row, const int32_t* sent_len,
                                    int32_t n_sent, int64_t A, float* att_minmax, void* stream) {
    return qnmt::att_minmax_launch(att_proj, sent_row, sent_len, n_sent, A, att_minmax, qnmt::as_stream(stream));
}

extern "C" int qnmt_attention_f32(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                                  const int32_t* sent_ncols, int32_t n_sent, const float* att_proj,
                                  const float* states, const int64_t* sent_row, const int32_t* sent_len,
                                  int32_t max_len, int64_t A, int64_t H2, const float* v, float* ctx, int64_t ldc,
                                  float* alpha, int64_t lda, void* scratch, int32_t* err_flag, void* stream) {
    return qnmt::attention_f32_launch(u, ldu, N, sent_col_off, sent_ncols, n_sent, att_proj, states, sent_row,
                                      sent_len, max_len, A, H2, v, ctx, ldc, alpha, lda, scratch, err_flag,
                                      qnmt::as_stream(stream));
}
