// kernels.cuh -- internal launch helpers shared by the C ABI wrappers and the engine.
// Optional trailing `segmax`/`col_seg`: fused per-segment max-abs of the output
// (u32 bits, atomicMax) for the next quantization (see elementwise.cu).
#pragma once
#include "common.cuh"

namespace qnmt {

int gru_gates_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* gh,
                     int64_t ldgh, const float* h, int64_t ldh, int64_t N, int64_t H, float* z,
                     float* rh, int32_t* err_flag, cudaStream_t st, uint32_t* segmax = nullptr,
                     const int32_t* col_seg = nullptr);
int gru_combine_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* ghc,
                       int64_t ldghc, const float* z, const float* h, int64_t ldh, int64_t N,
                       int64_t H, float* h_out, int64_t ldo, float* out2, int64_t ld2,
                       const int32_t* out2_row, int32_t* err_flag, cudaStream_t st,
                       uint32_t* segmax = nullptr, const int32_t* col_seg = nullptr);
int tanh_launch(const float* x, int64_t N, int64_t D, int64_t ldx, float* y, int64_t ldy,
                int32_t* err_flag, cudaStream_t st, uint32_t* segmax = nullptr,
                const int32_t* col_seg = nullptr);
int embed_gather_launch(const float* table, int64_t rows, int64_t E, const int32_t* ids, int64_t n,
                        float* out, int64_t ldo, int32_t* err_flag, cudaStream_t st,
                        uint32_t* segmax = nullptr, const int32_t* col_seg = nullptr);
int attention_launch(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                     const int32_t* sent_ncols, int32_t n_sent, const float* att_proj, const float* att_minmax,
                     const float* states, const int64_t* sent_row, const int32_t* sent_len, int32_t max_len,
                     int64_t A, int64_t H2, const int8_t* v_codes, const float* v_scale, float* ctx, int64_t ldc,
                     float* alpha, int64_t lda, void* scratch, int32_t* err_flag, cudaStream_t st,
                     uint32_t* ctx_segmax = nullptr, int max_p = 16, const float* att_exp = nullptr);
// E_ap = fl32(e^(2 att_proj)) for the one-MUFU attention scorer (n values)
int att_exp_launch(const float* att_proj, int64_t n, float* out, cudaStream_t st);
int att_minmax_launch(const float* att_proj, const int64_t* sent_row, const int32_t* sent_len, int32_t n_sent,
                      int64_t A, float* mm, cudaStream_t st);
int col_ranges_launch(const int32_t* col_sent, int64_t N, int32_t n_sent, int32_t* off, int32_t* cnt,
                      cudaStream_t st);
int gemm_f32_launch(const float* W, int64_t M, int64_t K, int64_t ldw, const float* X, int64_t N, int64_t ldx,
                    const float* bias, float* Y, int64_t ldy, int32_t flags, cudaStream_t st);
int attention_f32_launch(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                         const int32_t* sent_ncols, int32_t n_sent, const float* att_proj, const float* states,
                         const int64_t* sent_row, const int32_t* sent_len, int32_t max_len, int64_t A, int64_t H2,
                         const float* v, float* ctx, int64_t ldc, float* alpha, int64_t lda, void* scratch,
                         int32_t* err_flag, cudaStream_t st);
struct EnsRows {
    const float* p[QNMT_ENS_MAX];   // member logits [N][ld], same layout
};
int ens_topk_launch(const EnsRows& rows, int nm, int64_t N, int64_t V, int64_t ld, const double* live, int32_t k,
                    double* cand_score, int32_t* cand_tok, int32_t* err_flag, cudaStream_t st);
int topk_launch(const float* logits, int64_t N, int64_t V, int64_t ld, const double* live, int32_t k,
                double* cand_score, int32_t* cand_tok, int32_t* err_flag, cudaStream_t st);
// encode pass only: seg_maxbits already holds the per-segment max-abs bits
int quantize_encode_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                           int8_t* q, int64_t ldq, float* scales, const uint32_t* seg_maxbits, int32_t mode,
                           int32_t* err_flag, cudaStream_t st);
// max-abs pass only, accumulating into (already zeroed) seg_maxbits
int quantize_max_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                        uint32_t* seg_maxbits, cudaStream_t st);

// fused vocab projection + log-softmax statistics + beam candidates (vocab_topk.cu)
struct VocabTopk {
    const int8_t* X;          // [N][ldx] readout codes (K-major)
    int64_t N, ldx;
    const float* x_scales;
    const int32_t* row_seg;
    const int8_t* W;          // [V][ldw] vocabulary codes
    int64_t V, K, ldw;
    const float* w_scales;
    int64_t w_rows_per_scale;
    const float* bias;
    const double* live;       // [N] running hypothesis scores
    int32_t k;
    void* part;               // vocab_topk_part_bytes(N, V)
    double* cand_score;       // [N][k]
    int32_t* cand_tok;
    int32_t* err_flag;
};
extern int g_vocab_fused;
bool vocab_topk_eligible(int64_t K, int64_t ldx, int64_t ldw, const void* X, const void* W, int k);
size_t vocab_topk_part_bytes(int64_t rows, int64_t V);
int vocab_stats_launch(const VocabTopk& p, cudaStream_t st);
int vocab_merge_launch(const VocabTopk& p, cudaStream_t st);

// decoder elementwise ops fused with the quantization of their output, one CTA per
// sentence segment [off[s], off[s] + cnt[s]) (fused_q.cu); max_cols bounds cnt[s]
constexpr size_t FQ_SMEM_MAX = 227 * 1024;
int gates_q_launch(const float* gx, int64_t ldgx, const float* gh, int64_t ldgh, const float* h, int64_t ldh,
                   int64_t H, const int32_t* off, const int32_t* cnt, int n_seg, int max_cols, float* z,
                   int8_t* q_rh, float* sc_rh, int32_t* err_flag, cudaStream_t st);
int combine_q_launch(const float* gxc, int64_t ldgx, const float* ghc, int64_t ldghc, const float* z,
                     const float* h, int64_t ldh, int64_t H, const int32_t* off, const int32_t* cnt, int n_seg,
                     int max_cols, float* h_out, int64_t ldo, int8_t* q_out, float* sc_out, int32_t* err_flag,
                     cudaStream_t st);
// encoder steps: one CTA per (sentence, direction) column -- GRU phase + quantization of its output
int enc_gates_q_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* gh, int64_t ldgh,
                       const float* h, int64_t ldh, int64_t ncols, int64_t H, float* z, int8_t* q_rh, float* sc_rh,
                       int32_t* err_flag, cudaStream_t st);
int enc_combine_q_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* ghc, int64_t ldghc,
                         const float* z, float* h, int64_t ldh, int64_t ncols, int64_t H, float* states, int64_t lds,
                         const int32_t* out_row, int8_t* q_h, float* sc_h, int32_t* err_flag, cudaStream_t st);
int embed_q_launch(const float* table, int64_t rows, int64_t E, const int32_t* ids, const int32_t* off,
                   const int32_t* cnt, int n_seg, int max_cols, int8_t* q_out, float* sc_out, int32_t* err_flag,
                   cudaStream_t st, uint32_t* zero4 = nullptr, int zstride = 0);
int tanh_q_launch(const float* x, int64_t ldx, int64_t D, const int32_t* off, const int32_t* cnt, int n_seg,
                  int max_cols, int8_t* q_out, float* sc_out, int32_t* err_flag, cudaStream_t st,
                  const float* a1 = nullptr, int64_t ld1 = 0, const float* a2 = nullptr, int64_t ld2 = 0);
int gather_q_launch(const float* a, const float* b, const int32_t* parent, int64_t H, const int32_t* off,
                    const int32_t* cnt, int n_seg, int max_cols, float* a_out, float* b_out, int8_t* qa,
                    float* sca, int8_t* qb, float* scb, int32_t* err_flag, cudaStream_t st);

}  // namespace qnmt
