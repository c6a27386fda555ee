// search.cu -- device-resident beam bookkeeping for a batch of sentences.
//
// One thread per sentence executes one iteration of decoder.py:112-155:
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

__global__ void __launch_bounds__(SEARCH_T)
k_search_step(SearchState ss, int step, int n_sent, int beam, int k_list) {
    pdl_entry();
    __shared__ int wsum[SEARCH_T / 32];
    const int tid = threadIdx.x;
    if (ss.step_dev) step = *ss.step_dev;   // graph-captured loop: step counter lives on the device
    int new_p = 0;
    // per-thread selection results
    int sel_tok[16], sel_par[16];
    double sel_sc[16];
    int nsel = 0;
    const int s = tid;
    if (s < n_sent && !ss.done[s]) {
        const int P = ss.P[s];
        const int off = ss.col_off[s];
        // merge with each parent's current head kept in registers: one dependent load per round
        const int kt = min(k_list, beam);
        double hs[16];
        int ht[16], ptr[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            ptr[p] = 0;
            if (p < P) {
                const int64_t idx = (int64_t)(off + p) * k_list;
                hs[p] = ss.cand_score[idx];
                ht[p] = ss.cand_tok[idx];
            }
        }
        for (int r = 0; r < beam; ++r) {
            int bp = -1;
            double bs = 0.0;
            int bt = 0;
#pragma unroll
            for (int p = 0; p < 16; ++p) {
                if (p >= P || ptr[p] >= kt) continue;
                if (bp < 0 || cand_better(hs[p], ht[p], p, bs, bt, bp)) {
                    bp = p;
                    bs = hs[p];
                    bt = ht[p];
                }
            }
            if (bp < 0) break;
            sel_tok[nsel] = bt;
            sel_par[nsel] = bp;
            sel_sc[nsel] = bs;
            nsel++;
#pragma unroll
            for (int p = 0; p < 16; ++p)
                if (p == bp) {
                    ptr[p]++;
                    if (ptr[p] < kt) {
                        const int64_t idx = (int64_t)(off + p) * k_list + ptr[p];
                        hs[p] = ss.cand_score[idx];
                        ht[p] = ss.cand_tok[idx];
                    }
                }
        }
        // split into finished / live
        double best_live = -DBL_MAX;
        int64_t hbase = ((int64_t)s * ss.max_steps_cap + step) * ss.beam_cap;
        for (int i = 0; i < nsel; ++i) {
            if (sel_tok[i] == EOS) {
                int f = ss.fin_cnt[s]++;
                int64_t fb = (int64_t)s * ss.fin_cap + f;
                ss.fin_score[fb] = sel_sc[i];
                ss.fin_step[fb] = step;
                ss.fin_slot[fb] = sel_par[i];
                ss.fin_eos[fb] = 1;
                if (f == 0 || sel_sc[i] > ss.fin_best[s]) ss.fin_best[s] = sel_sc[i];
            } else {
                ss.hist_tok[hbase + new_p] = sel_tok[i];
                ss.hist_par[hbase + new_p] = sel_par[i];
                if (sel_sc[i] > best_live) best_live = sel_sc[i];
                sel_tok[new_p] = sel_tok[i];
                sel_par[new_p] = sel_par[i];
                sel_sc[new_p] = sel_sc[i];
                new_p++;
            }
        }
        bool stop = false;
        if (new_p == 0) {
            stop = true;                                   // :143-144
        } else if (ss.fin_cnt[s] > 0 && ss.fin_best[s] >= best_live) {
            stop = true;                                   // :150-151
        } else if (step == ss.max_steps[s] - 1) {
            for (int j = 0; j < new_p; ++j) {              // :152-155
                int f = ss.fin_cnt[s]++;
                int64_t fb = (int64_t)s * ss.fin_cap + f;
                ss.fin_score[fb] = sel_sc[j];
                ss.fin_step[fb] = step;
                ss.fin_slot[fb] = j;
                ss.fin_eos[fb] = 0;
            }
            stop = true;
        }
        ss.steps_run[s] = step + 1;
        if (stop) {
            ss.done[s] = 1;
            new_p = 0;
        }
    }
    // exclusive prefix sum of new_p over sentences: warp scans, then a scan of the warp sums
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
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
    if (s < n_sent) {
        const int old_off = ss.col_off[s];
        for (int j = 0; j < new_p; ++j) {
            int n = new_off + j;
            ss.col_sent_next[n] = s;
            ss.parent_col[n] = old_off + sel_par[j];
            ss.y_next[n] = sel_tok[j];
            ss.live_next[n] = sel_sc[j];
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

int search_step_launch(const SearchState& ss, int step, int n_sent, int beam, int k_list,
                       cudaStream_t st) {
    if (n_sent > SEARCH_T || beam > 16) {
        set_error("search: n_sent=%d beam=%d exceed limits (%d, 16)", n_sent, beam, SEARCH_T);
        return QNMT_ERR_CONFIG;
    }
    const int threads = (int)std::min<int64_t>(SEARCH_T, std::max<int64_t>(32, cdiv(n_sent, 32) * 32));
    QNMT_LAUNCH(k_search_step, 1, threads, 0, st, ss, step, n_sent, beam, k_list);
    QNMT_CHECK_LAUNCH("k_search_step");
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
