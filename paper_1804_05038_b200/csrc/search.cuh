// search.cuh -- device state of the batched beam search (search.cu).
#pragma once
#include "common.cuh"

namespace qnmt {

struct SearchState {
    // per sentence
    int32_t* P;            // live columns this step
    int32_t* col_off;      // offset of the sentence's columns
    int32_t* done;
    int32_t* max_steps;    // ceil(max_ratio * l) + 1   (decoder.py:103)
    int32_t* steps_run;
    int32_t* fin_cnt;
    double* fin_best;
    double* fin_score;     // [S][fin_cap]
    int32_t* fin_step;
    int32_t* fin_slot;     // parent slot (EOS) or own slot (frozen survivor)
    int32_t* fin_eos;
    int32_t* hist_tok;     // [S][max_steps_cap][beam_cap]
    int32_t* hist_par;
    int32_t fin_cap, max_steps_cap, beam_cap;
    // per column (current step); the search parks its selections in the consumed slots
    double* cand_score;    // [N][k_list]
    int32_t* cand_tok;
    // per column (next step)
    int32_t* col_sent_next;
    int32_t* parent_col;
    int32_t* y_next;
    double* live_next;
    int32_t* n_live;       // device scalar: columns of the next step
    int32_t* step_dev;     // device step counter (graph mode) or nullptr (host passes step)
    int32_t* np_tmp = nullptr;   // [S] live selections per sentence (select -> layout)
};

// device-side final selection (decoder.py:157-160), one packed row per sentence
struct FinalizeArgs {
    const int32_t* fin_cnt;
    const double* fin_score;
    const int32_t* fin_step;
    const int32_t* fin_slot;
    const int32_t* fin_eos;
    const int32_t* hist_tok;   // [S][T][B]
    const int32_t* hist_par;
    int32_t fin_cap, T, B;
    int32_t* res;              // [n][res_stride]: len, logp (2 words), tokens
    int32_t res_stride;
    int32_t* scratch;          // [n][2][T + 2] when the history does not fit in shared memory
    int32_t stage;             // set by finalize_launch
};
int finalize_launch(const FinalizeArgs& a, int n, cudaStream_t st);

int search_step_launch(const SearchState& ss, int step, int n_sent, int beam, int k_list,
                       cudaStream_t st);
// the selection alone (k_search_select); the layout then comes from layout_gather_q_launch
int search_select_launch(const SearchState& ss, int step, int n_sent, int beam, int k_list, cudaStream_t st);
// k_search_layout + k_gather_q in one launch (graph-captured steps: step counter on the device)
int layout_gather_q_launch(const SearchState& ss, int n_sent, int beam, int k_list, const float* a, const float* b,
                           int64_t H, float* a_out, float* b_out, int8_t* qa, float* sca, int8_t* qb, float* scb,
                           int32_t* err_flag, cudaStream_t st);
// optional a_max/b_max: per-segment max |a_out| / |b_out| (segment = col_seg[n]) for the next step
int gather_rows_launch(const float* a, const float* b, const int32_t* parent, int64_t N, int64_t H,
                       float* a_out, float* b_out, cudaStream_t st, uint32_t* a_max = nullptr,
                       uint32_t* b_max = nullptr, const int32_t* col_seg = nullptr);

}  // namespace qnmt
