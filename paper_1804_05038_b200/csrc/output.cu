// output.cu -- column log-softmax over the target vocabulary and the beam
// candidates of each hypothesis.
//
// layers.py:60-67 (_log_softmax_cols), evaluated in fp64 and rounded once:
//   t_v = f64(logit_v) - f64(max), lse = log(sum_v exp(t_v)), lp_v = fl32(t_v - lse)
// decoder.py:125 + :74-85: score = live + f64(lp); candidates ordered by
//   (score desc, token asc).  For one parent the global order restricted to
//   that parent is exactly this order, so the global top-`beam` over the
//   parent-major [P*V] flat array is contained in the union of every parent's
//   top-`beam` list (selection is finished by search.cu).
#include <float.h>

#include "common.cuh"

namespace qnmt {

constexpr int LS_T = 512;

struct Cand {
    double s;
    int t;
};

__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
    return a.s > b.s || (a.s == b.s && a.t < b.t);
}

// block-wide reductions (LS_T threads)
__device__ float block_max_f(float v, float* red) {
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

__device__ double block_sum_d(double v, double* red) {
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

// max and lse of one column; non-finite logits poison both (flag raised).
__device__ void column_stats(const float* __restrict__ row, int64_t V, float* redf, double* redd,
                             float& mx_out, double& lse_out, int32_t* err_flag) {
    float m = -FLT_MAX;
    bool bad = false;
    for (int64_t v = threadIdx.x; v < V; v += LS_T) {
        float x = row[v];
        bad |= !is_finite_f(x);
        m = fmaxf(m, x);
    }
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    }
    float mx = block_max_f(m, redf);
    double dm = (double)mx;
    double s = 0.0;
    for (int64_t v = threadIdx.x; v < V; v += LS_T) s += exp((double)row[v] - dm);
    double tot = block_sum_d(s, redd);
    mx_out = mx;
    lse_out = log(tot);
}

__global__ void __launch_bounds__(LS_T)
k_log_softmax(const float* __restrict__ logits, int64_t V, int64_t ld, float* __restrict__ lp,
              int64_t ldlp, int32_t* err_flag) {
    __shared__ float redf[32];
    __shared__ double redd[32];
    int64_t n = blockIdx.x;
    const float* row = logits + n * ld;
    float mx;
    double lse;
    column_stats(row, V, redf, redd, mx, lse, err_flag);
    double dm = (double)mx;
    for (int64_t v = threadIdx.x; v < V; v += LS_T)
        lp[n * ldlp + v] = __double2float_rn(((double)row[v] - dm) - lse);
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

template <int KM>
__global__ void __launch_bounds__(LS_T)
k_topk(const float* __restrict__ logits, int64_t V, int64_t ld, const double* __restrict__ live,
       int k, double* __restrict__ cand_score, int32_t* __restrict__ cand_tok, int32_t* err_flag) {
    __shared__ float redf[32];
    __shared__ double redd[32];
    __shared__ Cand wl[LS_T / 32][KM];
    int64_t n = blockIdx.x;
    const float* row = logits + n * ld;
    float mx;
    double lse;
    column_stats(row, V, redf, redd, mx, lse, err_flag);
    double dm = (double)mx;
    double base = live ? live[n] : 0.0;
    Cand L[KM];
#pragma unroll
    for (int i = 0; i < KM; ++i) L[i] = Cand{-DBL_MAX, 0x7fffffff};
    for (int64_t v = threadIdx.x; v < V; v += LS_T) {
        float lp = __double2float_rn(((double)row[v] - dm) - lse);
        insert<KM>(L, Cand{base + (double)lp, (int)v});
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    warp_merge<KM>(L, wl[warp], k);
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < KM; ++i) L[i] = (lane < LS_T / 32 && i < k) ? wl[lane][i] : Cand{-DBL_MAX, 0x7fffffff};
        Cand* res = wl[0];   // reuse; lane 0 writes sequentially after reading
        __syncwarp();
        Cand outv[KM];
        warp_merge<KM>(L, outv, k);
        if (lane == 0) {
            for (int i = 0; i < k; ++i) {
                cand_score[n * k + i] = outv[i].s;
                cand_tok[n * k + i] = outv[i].t;
            }
        }
        (void)res;
    }
}

int log_softmax_launch(const float* logits, int64_t N, int64_t V, int64_t ld, float* lp, int64_t ldlp,
                       int32_t* err_flag, cudaStream_t st) {
    if (N <= 0) return QNMT_OK;
    k_log_softmax<<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, lp, ldlp, err_flag);
    QNMT_CHECK_LAUNCH("k_log_softmax");
    return QNMT_OK;
}

int topk_launch(const float* logits, int64_t N, int64_t V, int64_t ld, const double* live, int32_t k,
                double* cand_score, int32_t* cand_tok, int32_t* err_flag, cudaStream_t st) {
    if (N <= 0) return QNMT_OK;
    if (k < 1 || k > 16 || k > V) {
        set_error("qnmt_topk_candidates: k=%d outside [1, min(16, V)]", k);
        return QNMT_ERR_CONFIG;
    }
    if (k <= 4)
        k_topk<4><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag);
    else if (k <= 8)
        k_topk<8><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag);
    else
        k_topk<16><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag);
    QNMT_CHECK_LAUNCH("k_topk");
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" {

int qnmt_log_softmax(const float* logits, int64_t N, int64_t V, int64_t ld, float* lp, int64_t ldlp,
                     int32_t* err_flag, void* stream) {
    return qnmt::log_softmax_launch(logits, N, V, ld, lp, ldlp, err_flag, qnmt::as_stream(stream));
}

int qnmt_topk_candidates(const float* logits, int64_t N, int64_t V, int64_t ld,
                         const double* live_scores, int32_t k, double* cand_score, int32_t* cand_tok,
                         int32_t* err_flag, void* stream) {
    return qnmt::topk_launch(logits, N, V, ld, live_scores, k, cand_score, cand_tok, err_flag,
                             qnmt::as_stream(stream));
}

}  // extern "C"
