// search.cu -- device-resident beam bookkeeping for a batch of sentences.
//
// One iteration of decoder.py:112-155 for every live sentence of the batch:
//   chosen  = top-`beam` of the parent-major candidates under
//             (score desc, token asc, parent asc)            (_select_candidates :74-85)
//   EOS candidates -> finished list; others -> next live set  (:127-141)
//   no live candidate -> stop                                 (:143-144)
//   best finished >= best live -> stop (survivors dropped)    (:150-151)
//   last allowed step -> survivors frozen into finished       (:152-155, for-else)
// Per-column inputs come from output.cu's per-parent candidate lists (each
// sorted by (score desc, token asc)); a P-way merge over them is exact.
// History (token, parent slot) per step lets the host rebuild token lists for
// the final min-by-(-logp, tokens) selection (:157).
#include <float.h>

#include <algorithm>

#include "common.cuh"
#include "search.cuh"

namespace qnmt {

constexpr int SEARCH_T = 1024;
constexpr int EOS = 2;   // model.py:33

__device__ __forceinline__ bool cand_better(double sa, int ta, int pa, double sb, int tb, int pb) {
    if (sa != sb) return sa > sb;
    if (ta != tb) return ta < tb;
    return pa < pb;
}

// Two kernels per step.
//  k_search_select (one warp per sentence, many CTAs): the sentence's P * kt
//    candidates (kt = min(k_list, beam) per parent list, each sorted by (score
//    desc, token asc)) are spread over the lanes; a candidate's rank under
//    (score desc, token asc, parent asc) is the number of better candidates, so
//    the selection is ranks < beam -- the same set and order as the P-way merge
//    of decoder.py:74-85.  Lane 0 applies the finished / live rules in rank order
//    and parks the live selections (token | parent << 26, score) in the
//    sentence's consumed candidate slots (P * k_list >= selections).
//  k_search_layout (one CTA): prefix sum of the live counts over sentences and
//    the next step's column layout from the parked selections.
constexpr int SEL_WARPS = 8;
constexpr int SLOTS = 8;   // candidates per lane (P * kt <= 16 * 16 = 256)

__global__ void __launch_bounds__(32 * SEL_WARPS)
k_search_select(SearchState ss, int step, int n_sent, int beam, int k_list) {
    pdl_entry();
    __shared__ double sel_sc[SEL_WARPS][16];
    __shared__ int sel_tok[SEL_WARPS][16], sel_par[SEL_WARPS][16];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = blockIdx.x * SEL_WARPS + warp;
    if (s >= n_sent) return;   // warp-uniform
    if (ss.step_dev) step = *ss.step_dev;   // graph-captured loop: step counter lives on the device
    if (ss.done[s]) {
        if (lane == 0) ss.np_tmp[s] = 0;
        return;
    }
    const int kt = min(k_list, beam);
    const int P = ss.P[s];
    const int off = ss.col_off[s];
    const int C = P * kt;
    const int nslot = (C + 31) >> 5;   // warp-uniform
    double cs[SLOTS];
    int ct[SLOTS], cp[SLOTS], rk[SLOTS];
#pragma unroll
    for (int q = 0; q < SLOTS; ++q) {
        const int c = q * 32 + lane;
        rk[q] = 0;
        if (q < nslot && c < C) {
            const int p = c / kt, r = c - p * kt;
            const int64_t idx = (int64_t)(off + p) * k_list + r;
            cs[q] = ss.cand_score[idx];
            ct[q] = ss.cand_tok[idx];
            cp[q] = p;
        } else {
            cs[q] = -DBL_MAX;
            ct[q] = 0x7fffffff;
            cp[q] = 0x7fffffff;
        }
    }
#pragma unroll
    for (int q2 = 0; q2 < SLOTS; ++q2) {
        if (q2 >= nslot) break;
        const int nsrc = min(32, C - q2 * 32);   // warp-uniform
        for (int src = 0; src < nsrc; ++src) {
            const double os = __shfl_sync(0xffffffffu, cs[q2], src);
            const int ot = __shfl_sync(0xffffffffu, ct[q2], src);
            const int op = __shfl_sync(0xffffffffu, cp[q2], src);
#pragma unroll
            for (int q = 0; q < SLOTS; ++q)
                if (q < nslot) rk[q] += cand_better(os, ot, op, cs[q], ct[q], cp[q]) ? 1 : 0;
        }
    }
    const int nsel = min(beam, C);
#pragma unroll
    for (int q = 0; q < SLOTS; ++q) {
        const int c = q * 32 + lane;
        if (q < nslot && c < C && rk[q] < beam) {
            sel_sc[warp][rk[q]] = cs[q];
            sel_tok[warp][rk[q]] = ct[q];
            sel_par[warp][rk[q]] = cp[q];
        }
    }
    __syncwarp();
    if (lane != 0) return;
    // finished / live split (decoder.py:127-141), in selection order
    double best_live = -DBL_MAX;
    int new_p = 0;
    const int64_t hbase = ((int64_t)s * ss.max_steps_cap + step) * ss.beam_cap;
    int fin = ss.fin_cnt[s];
    double fbest = ss.fin_best[s];
    for (int i = 0; i < nsel; ++i) {
        const double sc = sel_sc[warp][i];
        const int tok = sel_tok[warp][i], par = sel_par[warp][i];
        if (tok == EOS) {
            const int64_t fb = (int64_t)s * ss.fin_cap + fin;
            ss.fin_score[fb] = sc;
            ss.fin_step[fb] = step;
            ss.fin_slot[fb] = par;
            ss.fin_eos[fb] = 1;
            if (fin == 0 || sc > fbest) fbest = sc;
            ++fin;
        } else {
            ss.hist_tok[hbase + new_p] = tok;
            ss.hist_par[hbase + new_p] = par;
            if (sc > best_live) best_live = sc;
            const int64_t idx = (int64_t)off * k_list + new_p;
            ss.cand_score[idx] = sc;
            ss.cand_tok[idx] = tok | (par << 26);
            ++new_p;
        }
    }
    bool stop = false;
    if (new_p == 0) {
        stop = true;                                   // :143-144
    } else if (fin > 0 && fbest >= best_live) {
        stop = true;                                   // :150-151
    } else if (step == ss.max_steps[s] - 1) {
        for (int j = 0; j < new_p; ++j) {              // :152-155
            const int64_t fb = (int64_t)s * ss.fin_cap + fin;
            ss.fin_score[fb] = ss.cand_score[(int64_t)off * k_list + j];
            ss.fin_step[fb] = step;
            ss.fin_slot[fb] = j;
            ss.fin_eos[fb] = 0;
            ++fin;
        }
        stop = true;
    }
    ss.fin_cnt[s] = fin;
    ss.fin_best[s] = fbest;
    ss.steps_run[s] = step + 1;
    if (stop) {
        ss.done[s] = 1;
        new_p = 0;
    }
    ss.np_tmp[s] = new_p;
}

__global__ void __launch_bounds__(SEARCH_T)
k_search_layout(SearchState ss, int step, int n_sent, int k_list) {
    pdl_entry();
    __shared__ int wsum[SEARCH_T / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    if (ss.step_dev) step = *ss.step_dev;
    const int s = tid;
    const int new_p = s < n_sent ? ss.np_tmp[s] : 0;
    // exclusive prefix sum of new_p over sentences: warp scans, then a scan of the warp sums
    int incl = new_p;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nwarps ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        if (lane < nwarps) wsum[lane] = w;
    }
    __syncthreads();
    incl += warp > 0 ? wsum[warp - 1] : 0;
    const int new_off = incl - new_p;
    if (tid == (int)blockDim.x - 1) *ss.n_live = incl;
    if (s < n_sent) {   // only this thread touches col_off[s] / P[s]; only cand_* slots of s are read
        const int old_off = ss.col_off[s];
        for (int j = 0; j < new_p; ++j) {
            const int64_t idx = (int64_t)old_off * k_list + j;
            const int v = ss.cand_tok[idx];
            const int n = new_off + j;
            ss.col_sent_next[n] = s;
            ss.parent_col[n] = old_off + (v >> 26);
            ss.y_next[n] = v & ((1 << 26) - 1);
            ss.live_next[n] = ss.cand_score[idx];
        }
        ss.P[s] = new_p;
        ss.col_off[s] = new_off;
    }
    if (ss.step_dev) {
        __syncthreads();
        if (tid == 0) *ss.step_dev = step + 1;
    }
}

// next-step state columns: dst[n] = src[parent_col[n]] for the state tensors,
// plus (optionally) the per-segment max-abs bits the next step's quantization needs
__global__ void k_gather_rows(const float* __restrict__ a, const float* __restrict__ b,
                              const int32_t* __restrict__ parent, int64_t H,
                              float* __restrict__ a_out, float* __restrict__ b_out, const int32_t* n_dev,
                              uint32_t* a_max, uint32_t* b_max, const int32_t* __restrict__ col_seg) {
    pdl_entry();
    int64_t n = blockIdx.x;
    if (beyond(n_dev, n)) return;
    int64_t p = parent[n];
    uint32_t ma = 0, mb = 0;
    for (int64_t j = threadIdx.x; j < H; j += blockDim.x) {
        const float va = a[p * H + j];
        a_out[n * H + j] = va;
        ma = max(ma, __float_as_uint(va) & 0x7fffffffu);
        if (b) {
            const float vb = b[p * H + j];
            b_out[n * H + j] = vb;
            mb = max(mb, __float_as_uint(vb) & 0x7fffffffu);
        }
    }
    if (a_max) {
        const int seg = col_seg[n];
        ma = warp_max(ma);
        mb = warp_max(mb);
        if ((threadIdx.x & 31) == 0) {
            if (ma) atomicMax(a_max + seg, ma);
            if (b_max && mb) atomicMax(b_max + seg, mb);
        }
    }
}

// ---------------------------------------------------------------------------
// Final selection on the device (decoder.py:157-160): the answer is the
// finished hypothesis minimising (-log_prob, token list), EOS stripped.  One
// warp per sentence: the lanes stage the sentence's (token, parent) history
// in shared memory (coalesced) and find the best score; lane 0 backtracks the
// hypotheses holding that score (Python's list order breaks exact ties) and
// writes one packed row [len, logp lo, logp hi, tokens...] per sentence, so
// the host copies n * (Tmax + 3) words instead of the whole history block.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int fin_backtrack(const int32_t* ht, const int32_t* hp, int B, int step, int slot, int eos,
                                             int32_t* out) {
    // tokens 0..t of the hypothesis ending in `slot` at step t (t = step - 1 for an EOS entry)
    const int t = eos ? step - 1 : step;
    int j = slot;
    for (int tt = t; tt >= 0; --tt) {
        out[tt] = ht[tt * B + j];
        j = hp[tt * B + j];
    }
    if (eos) out[t + 1] = EOS;
    return t + 2 - (eos ? 0 : 1);   // EOS entries: t + 2 tokens incl. the EOS; survivors: t + 1
}

__global__ void __launch_bounds__(32)
k_finalize(FinalizeArgs a) {
    extern __shared__ int32_t fsm[];
    const int s = blockIdx.x, lane = threadIdx.x;
    const int B = a.B, T = a.T;
    const int64_t hb = (int64_t)s * T * B;
    const int fc = a.fin_cnt[s];
    const int64_t fb = (int64_t)s * a.fin_cap;
    int rows = 0;   // history rows any finished hypothesis reaches
    for (int f = lane; f < fc; f += 32) rows = max(rows, a.fin_step[fb + f] + 1);
#pragma unroll
    for (int o = 16; o; o >>= 1) rows = max(rows, __shfl_xor_sync(0xffffffffu, rows, o));
    rows = min(rows, T);
    const int32_t* ht = a.hist_tok + hb;
    const int32_t* hp = a.hist_par + hb;
    int32_t* bufA = fsm;
    int32_t* bufB = fsm + (T + 2);
    if (a.stage) {   // generic pointers: the backtrack reads shared memory when the history fits
        int32_t* st = fsm + 2 * (T + 2);
        for (int i = lane; i < rows * B; i += 32) {
            st[i] = ht[i];
            st[T * B + i] = hp[i];
        }
        __syncwarp();
        ht = st;
        hp = st + T * B;
    } else {
        bufA = a.scratch + (int64_t)s * 2 * (T + 2);
        bufB = bufA + (T + 2);
    }
    double best = -DBL_MAX;
    for (int f = lane; f < fc; f += 32) best = fmax(best, a.fin_score[fb + f]);
#pragma unroll
    for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane != 0) return;
    int32_t* row = a.res + (int64_t)s * a.res_stride;
    int la = -1, fa = -1;
    for (int f = 0; f < fc; ++f) {
        if (a.fin_score[fb + f] != best) continue;
        const int st_ = a.fin_step[fb + f], sl = a.fin_slot[fb + f], eo = a.fin_eos[fb + f];
        if (la < 0) {
            la = fin_backtrack(ht, hp, B, st_, sl, eo, bufA);
            fa = f;
            continue;
        }
        const int lb = fin_backtrack(ht, hp, B, st_, sl, eo, bufB);
        int i = 0;
        while (i < la && i < lb && bufA[i] == bufB[i]) ++i;
        const bool less = (i < la && i < lb) ? bufB[i] < bufA[i] : lb < la;
        if (less) {
            int32_t* t = bufA; bufA = bufB; bufB = t;
            la = lb;
            fa = f;
        }
    }
    int len = 0;
    double lp = 0.0;
    if (fa >= 0) {
        len = (la > 0 && bufA[la - 1] == EOS) ? la - 1 : la;   // decoder.py:158
        lp = best;
    }
    row[0] = len;
    const long long bits = __double_as_longlong(lp);
    row[1] = (int32_t)(bits & 0xffffffffll);
    row[2] = (int32_t)(bits >> 32);
    for (int i = 0; i < len; ++i) row[3 + i] = bufA[i];
}

int finalize_launch(const FinalizeArgs& a, int n, cudaStream_t st) {
    if (n <= 0) return QNMT_OK;
    FinalizeArgs b = a;
    const size_t bufs = (size_t)2 * (a.T + 2) * 4, hist = (size_t)2 * a.T * a.B * 4;
    b.stage = bufs + hist <= 48 * 1024 ? 1 : 0;
    if (!b.stage && !a.scratch) { set_error("finalize: no global scratch for a %d-step history", a.T); return QNMT_ERR_CONFIG; }
    const size_t smem = b.stage ? bufs + hist : 0;
    k_finalize<<<(unsigned)n, 32, smem, st>>>(b);
    QNMT_CHECK_LAUNCH("k_finalize");
    return QNMT_OK;
}

int search_step_launch(const SearchState& ss, int step, int n_sent, int beam, int k_list,
                       cudaStream_t st) {
    if (n_sent > SEARCH_T || beam > 16 || k_list > 16) {
        set_error("search: n_sent=%d beam=%d exceed limits (%d, 16)", n_sent, beam, SEARCH_T);
        return QNMT_ERR_CONFIG;
    }
    if (!ss.np_tmp) { set_error("search: no per-sentence scratch"); return QNMT_ERR_CONFIG; }
    QNMT_LAUNCH(k_search_select, (unsigned)cdiv(n_sent, SEL_WARPS), 32 * SEL_WARPS, 0, st, ss, step, n_sent, beam,
                k_list);
    QNMT_CHECK_LAUNCH("k_search_select");
    const int threads = (int)std::min<int64_t>(SEARCH_T, std::max<int64_t>(32, cdiv(n_sent, 32) * 32));
    QNMT_LAUNCH(k_search_layout, 1, threads, 0, st, ss, step, n_sent, k_list);
    QNMT_CHECK_LAUNCH("k_search_layout");
    return QNMT_OK;
}

int search_select_launch(const SearchState& ss, int step, int n_sent, int beam, int k_list, cudaStream_t st) {
    if (n_sent > SEARCH_T || beam > 16 || k_list > 16) {
        set_error("search: n_sent=%d beam=%d exceed limits (%d, 16)", n_sent, beam, SEARCH_T);
        return QNMT_ERR_CONFIG;
    }
    if (!ss.np_tmp) { set_error("search: no per-sentence scratch"); return QNMT_ERR_CONFIG; }
    QNMT_LAUNCH(k_search_select, (unsigned)cdiv(n_sent, SEL_WARPS), 32 * SEL_WARPS, 0, st, ss, step, n_sent, beam,
                k_list);
    QNMT_CHECK_LAUNCH("k_search_select");
    return QNMT_OK;
}

int gather_rows_launch(const float* a, const float* b, const int32_t* parent, int64_t N, int64_t H,
                       float* a_out, float* b_out, cudaStream_t st, uint32_t* a_max, uint32_t* b_max,
                       const int32_t* col_seg) {
    if (N <= 0) return QNMT_OK;
    QNMT_LAUNCH(k_gather_rows, (unsigned)N, 256, 0, st, a, b, parent, H, a_out, b_out, tl_ndev, a_max, b_max, col_seg);
    QNMT_CHECK_LAUNCH("k_gather_rows");
    return QNMT_OK;
}

}  // namespace qnmt
