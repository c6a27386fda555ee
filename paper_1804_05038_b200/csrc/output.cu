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

#include "cand.cuh"
#include "kernels.cuh"

namespace qnmt {

int g_topk_exact = 0;   // 1: use the three-pass reference kernel (testing)

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

struct LCand {
    float x;
    int t;
};
__device__ __forceinline__ bool lbetter(const LCand& a, const LCand& b) {
    return a.x > b.x || (a.x == b.x && a.t < b.t);
}
template <int KM>
__device__ __forceinline__ void linsert(LCand (&L)[KM], LCand c) {
    if (!lbetter(c, L[KM - 1])) return;
    L[KM - 1] = c;
#pragma unroll
    for (int i = KM - 1; i > 0; --i) {
        if (lbetter(L[i], L[i - 1])) {
            LCand t = L[i];
            L[i] = L[i - 1];
            L[i - 1] = t;
        }
    }
}

// ---------------------------------------------------------------------------
// Single-pass candidates (the production path).
//
// One read of the logits row: per thread an online (max, sum exp) in f64 and a
// top-KM list by (logit desc, token asc).  lp = fl32((x - M) - lse) is monotone
// non-decreasing in the logit x, so every token outside the KM-list has a
// score <= the KM-th list entry's score.  After computing exact scores for the
// KM entries and sorting by (score desc, token asc), the first k are the exact
// answer whenever the k-th score is STRICTLY greater than the KM-th entry's
// score (or the list covers the whole vocabulary).  Otherwise (an f32 rounding
// tie across the boundary -- practically never) the CTA rescans the column
// exactly with the three-pass method of k_topk.
// ---------------------------------------------------------------------------
template <int KM>
__global__ void __launch_bounds__(LS_T, 2)
k_topk1(const float* __restrict__ logits, int64_t V, int64_t ld, const double* __restrict__ live, int k,
        double* __restrict__ cand_score, int32_t* __restrict__ cand_tok, int32_t* err_flag,
        const int32_t* n_dev) {
    __shared__ float redf[32];
    __shared__ double redd[32];
    __shared__ Cand wl[LS_T / 32][KM];
    __shared__ Cand lst[KM];
    __shared__ int s_ok;
    const int64_t n = blockIdx.x;
    if (beyond(n_dev, n)) return;
    __shared__ double tab[16];
    if (threadIdx.x < 16) tab[threadIdx.x] = exp2((double)threadIdx.x / 16.0);
    __syncthreads();
    const float* row = logits + n * ld;
    float m = -FLT_MAX;
    double s = 0.0;
    bool bad = false;
    // per-thread top-3 by (logit desc, token asc), branch-free: elements arrive in
    // increasing token order, so strict '>' keeps the smaller token on ties
    float a1 = -FLT_MAX, a2 = -FLT_MAX, a3 = -FLT_MAX;
    int i1 = 0x7fffffff, i2 = 0x7fffffff, i3 = 0x7fffffff;
    auto top3 = [&](float x, int v) {
        const bool g1 = x > a1, g2 = x > a2, g3 = x > a3;
        a3 = g2 ? a2 : (g3 ? x : a3);
        i3 = g2 ? i2 : (g3 ? v : i3);
        a2 = g1 ? a1 : (g2 ? x : a2);
        i2 = g1 ? i1 : (g2 ? v : i2);
        a1 = g1 ? x : a1;
        i1 = g1 ? v : i1;
    };
    const bool vec = (V % 4 == 0) && (ld % 4 == 0) && (((uintptr_t)logits & 15) == 0);
    if (vec) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        const int64_t Q = V / 4;
        constexpr int U = 4;   // float4 loads in flight per thread
        for (int64_t q0 = threadIdx.x; q0 < Q; q0 += U * LS_T) {
            float4 xs[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t q = q0 + (int64_t)u * LS_T;
                xs[u] = q < Q ? __ldg(r4 + q) : make_float4(-FLT_MAX, -FLT_MAX, -FLT_MAX, -FLT_MAX);
            }
            float cm = -FLT_MAX;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float4 x = xs[u];
                bad |= !(is_finite_f(x.x) && is_finite_f(x.y) && is_finite_f(x.z) && is_finite_f(x.w));
                cm = fmaxf(cm, fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w)));
            }
            if (cm > m) {   // rare after the first chunks: rescale the running sum once
                s = (m == -FLT_MAX) ? 0.0 : s * exp_neg((double)m - (double)cm, tab);
                m = cm;
            }
            const double dm = (double)m;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t q = q0 + (int64_t)u * LS_T;
                if (q >= Q) break;
                const float4 x = xs[u];
                const int v = (int)(4 * q);
                const double e0 = exp_neg((double)x.x - dm, tab), e1 = exp_neg((double)x.y - dm, tab);
                const double e2 = exp_neg((double)x.z - dm, tab), e3 = exp_neg((double)x.w - dm, tab);
                s += (e0 + e1) + (e2 + e3);
                const float gm = fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w));
                if (__any_sync(__activemask(), gm > a3)) {   // warp-uniform; rare after the first groups
                    top3(x.x, v);
                    top3(x.y, v + 1);
                    top3(x.z, v + 2);
                    top3(x.w, v + 3);
                }
            }
        }
    } else {
        for (int64_t v = threadIdx.x; v < V; v += LS_T) {
            const float x = row[v];
            bad |= !is_finite_f(x);
            if (x > m) {
                s = (m == -FLT_MAX) ? 0.0 : s * exp_neg((double)m - (double)x, tab);
                m = x;
            }
            s += exp_neg((double)x - (double)m, tab);
            top3(x, (int)v);
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    const float M = block_max_f(m, redf);
    const double dM = (double)M;
    const double S = block_sum_d(m == -FLT_MAX ? 0.0 : s * exp_neg((double)m - dM, tab), redd);
    const double lse = log(S);
    const int kk = (int)(V < KM ? V : KM);
    {
        Cand Lc[KM];
#pragma unroll
        for (int i = 0; i < KM; ++i) Lc[i] = Cand{-DBL_MAX, 0x7fffffff};
        if (i1 != 0x7fffffff) Lc[0] = Cand{(double)a1, i1};
        if (i2 != 0x7fffffff) Lc[1] = Cand{(double)a2, i2};
        if (i3 != 0x7fffffff) Lc[2] = Cand{(double)a3, i3};
        block_merge_cands<KM>(Lc, wl, lst, kk);
    }
    // The merged list is the exact top-KM unless some thread may hold a 4th element
    // that belongs to it, i.e. its 3rd entry still reaches the KM-th value: then rescan.
    {
        const Cand thr = lst[kk - 1];
        const bool maybe_more = (i3 != 0x7fffffff) && !better(thr, Cand{(double)a3, i3});
        if (__syncthreads_or(maybe_more)) {
            Cand L[KM];
#pragma unroll
            for (int i = 0; i < KM; ++i) L[i] = Cand{-DBL_MAX, 0x7fffffff};
            for (int64_t v = threadIdx.x; v < V; v += LS_T) {
                const float x = row[v];
                if ((double)x >= thr.s) insert<KM>(L, Cand{(double)x, (int)v});
            }
            block_merge_cands<KM>(L, wl, lst, kk);
        }
    }
    const double base = live ? live[n] : 0.0;
    if (threadIdx.x == 0) {
        // exact scores for the KM logit-candidates, then order by (score desc, token asc)
        Cand c[KM];
        for (int i = 0; i < kk; ++i) {
            float lp = __double2float_rn((lst[i].s - dM) - lse);
            c[i] = Cand{base + (double)lp, lst[i].t};
        }
        const double s_last = c[kk - 1].s;
        for (int i = 1; i < kk; ++i) {
            Cand t = c[i];
            int j = i - 1;
            while (j >= 0 && better(t, c[j])) { c[j + 1] = c[j]; --j; }
            c[j + 1] = t;
        }
        const bool ok = (V <= KM) || (c[k - 1].s > s_last);
        if (ok)
            for (int i = 0; i < k; ++i) {
                cand_score[n * k + i] = c[i].s;
                cand_tok[n * k + i] = c[i].t;
            }
        s_ok = ok;
    }
    __syncthreads();
    if (s_ok) return;
    // ---- exact fallback: rescan with final lp values (three-pass method) ----
    Cand L2[KM];
#pragma unroll
    for (int i = 0; i < KM; ++i) L2[i] = Cand{-DBL_MAX, 0x7fffffff};
    for (int64_t v = threadIdx.x; v < V; v += LS_T) {
        float lp = __double2float_rn(((double)row[v] - dM) - lse);
        insert<KM>(L2, Cand{base + (double)lp, (int)v});
    }
    block_merge_cands<KM>(L2, wl, lst, k);
    if (threadIdx.x == 0)
        for (int i = 0; i < k; ++i) {
            cand_score[n * k + i] = lst[i].s;
            cand_tok[n * k + i] = lst[i].t;
        }
}

// ---------------------------------------------------------------------------
// Ensemble candidates (decoder.py:115-120 + :125): every member's column
// log-softmax (fp64, rounded once, as k_log_softmax), summed in member order in
// f32, divided by f32(#members), then score = live + f64(lp) and the top-k by
// (score desc, token asc).  One CTA per hypothesis column; members' logits are
// read once for the statistics and once for the candidates.
// ---------------------------------------------------------------------------
template <int KM>
__global__ void __launch_bounds__(LS_T)
k_ens_topk(EnsRows rows, int nm, int64_t V, int64_t ld, const double* __restrict__ live, int k,
           double* __restrict__ cand_score, int32_t* __restrict__ cand_tok, int32_t* err_flag) {
    __shared__ float redf[32];
    __shared__ double redd[32];
    __shared__ Cand wl[LS_T / 32][KM];
    __shared__ Cand lst[KM];
    const int64_t n = blockIdx.x;
    double dm[QNMT_ENS_MAX], lse[QNMT_ENS_MAX];
#pragma unroll
    for (int i = 0; i < QNMT_ENS_MAX; ++i) {
        dm[i] = 0.0;
        lse[i] = 0.0;
        if (i < nm) {
            float mx;
            column_stats(rows.p[i] + n * ld, V, redf, redd, mx, lse[i], err_flag);
            dm[i] = (double)mx;
        }
    }
    const float fn = (float)nm;
    const double base = live ? live[n] : 0.0;
    Cand L[KM];
#pragma unroll
    for (int i = 0; i < KM; ++i) L[i] = Cand{-DBL_MAX, 0x7fffffff};
    for (int64_t v = threadIdx.x; v < V; v += LS_T) {
        float acc = __double2float_rn(((double)rows.p[0][n * ld + v] - dm[0]) - lse[0]);
#pragma unroll
        for (int i = 1; i < QNMT_ENS_MAX; ++i)
            if (i < nm) acc = __fadd_rn(acc, __double2float_rn(((double)rows.p[i][n * ld + v] - dm[i]) - lse[i]));
        acc = __fdiv_rn(acc, fn);
        insert<KM>(L, Cand{base + (double)acc, (int)v});
    }
    block_merge_cands<KM>(L, wl, lst, k);
    if (threadIdx.x == 0)
        for (int i = 0; i < k; ++i) {
            cand_score[n * k + i] = lst[i].s;
            cand_tok[n * k + i] = lst[i].t;
        }
}

int ens_topk_launch(const EnsRows& rows, int nm, int64_t N, int64_t V, int64_t ld, const double* live, int32_t k,
                    double* cand_score, int32_t* cand_tok, int32_t* err_flag, cudaStream_t st) {
    if (N <= 0) return QNMT_OK;
    if (nm < 2 || nm > QNMT_ENS_MAX) {
        set_error("ensemble of %d members outside [2, %d]", nm, QNMT_ENS_MAX);
        return QNMT_ERR_CONFIG;
    }
    if (k < 1 || k > 16 || k > V) {
        set_error("ensemble candidates: k=%d outside [1, min(16, V)]", k);
        return QNMT_ERR_CONFIG;
    }
    if (k <= 8)
        k_ens_topk<8><<<(unsigned)N, LS_T, 0, st>>>(rows, nm, V, ld, live, k, cand_score, cand_tok, err_flag);
    else
        k_ens_topk<16><<<(unsigned)N, LS_T, 0, st>>>(rows, nm, V, ld, live, k, cand_score, cand_tok, err_flag);
    QNMT_CHECK_LAUNCH("k_ens_topk");
    return QNMT_OK;
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
    if (g_topk_exact) {   // reference three-pass kernel (A/B testing)
        if (k <= 4)
            k_topk<4><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag);
        else if (k <= 8)
            k_topk<8><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag);
        else
            k_topk<16><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag);
        QNMT_CHECK_LAUNCH("k_topk");
        return QNMT_OK;
    }
    if (k <= 6)
        k_topk1<8><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag, tl_ndev);
    else if (k <= 13)
        k_topk1<16><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag, tl_ndev);
    else
        k_topk1<32><<<(unsigned)N, LS_T, 0, st>>>(logits, V, ld, live, k, cand_score, cand_tok, err_flag, tl_ndev);
    QNMT_CHECK_LAUNCH("k_topk1");
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

extern "C" int qnmt_set_topk_exact(int exact) {
    int old = qnmt::g_topk_exact;
    qnmt::g_topk_exact = exact;
    return old;
}
