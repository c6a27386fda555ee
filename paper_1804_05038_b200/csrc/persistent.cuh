// persistent.cuh -- arguments of the persistent batch-1 greedy decode kernel (persistent.cu).
#pragma once
#include "common.cuh"

namespace qnmt {

// control words of the persistent kernels: [0..4] y, best token, done, barrier top
// counter, barrier generation; [32 + 32 g] barrier group counters (persistent.cu gsync)
constexpr int PK_CTL_INTS = 32 + 32 * 16;

struct PkArgs {
    int E, H, A, R, V;
    const float* tgt_embed;
    const int8_t* w2x; const float* w2x_s; const float* b2x;   // [3H+R][E] = [W_x2; W_e], per-row scales, [b_x2; 0]
    const int8_t* uzr2; const float* uzr2_s;                   // [2H][H], 2 block scales
    const int8_t* uc2; const float* uc2_s;
    const int8_t* wuq; const float* wuq_s;                     // [A+2H][H] = [U_att; U_zr3], per-row scales
    const int8_t* w3x; const float* w3x_s; const float* b3x;   // [3H+R][2H] = [W_x3; W_c]
    const int8_t* uc3; const float* uc3_s;
    const int8_t* v; const float* v_s;                         // [A]
    const int8_t* w_state; const float* w_state_s; const float* b_r;
    const int8_t* w_vocab; const float* w_vocab_s; const float* b_vocab;
    const float* states;   // [l][2H] encoder states of the sentence
    const float* att;      // [l][A] att_proj
    const float* att_mm;   // [2][A] column max / min of att_proj
    int l;
    int max_steps;
    // scratch written and read inside the kernel (loads bypass L1)
    float* s;        // [H] state (s0 on entry)
    float* sp;       // [H] s'
    float* gxr;      // [3H+R]
    float* gh;       // [2H]
    float* ghc;      // [H]
    float* uq;       // [A+2H]
    float* scores;   // [l]
    float* ctx;      // [2H]
    float* gxq;      // [3H+R]
    float* ro;       // [R]
    float* logits;   // [V]
    double* part;    // [grid][2]
    int32_t* ctl;    // [0] y, [1] best token, [2] done, [3..4] grid barrier
    // search outputs (engine layout, sentence 0)
    int32_t* hist_tok; int32_t* hist_par; int hist_stride;
    double* fin_score; int32_t* fin_step; int32_t* fin_slot; int32_t* fin_eos; int32_t* fin_cnt;
    int32_t* err;
    long long* stamps;   // nullable: %globaltimer after each barrier of each step ([t][11], CTA 0)
    int32_t* step_dev;   // nullable: steps run (for qnmt_engine_stamps_read)
};

int greedy1_launch(const PkArgs& a, cudaStream_t st);
extern int g_greedy1;

// batch-1 bidirectional GRU recurrence (layers.py:331-340) as one persistent kernel
struct PeArgs {
    int H, l;
    const float* gx;            // [l][2][3H]: W_x q(emb_i) + b_x per position and direction
    const int8_t* uzr[2]; const float* uzr_s[2];   // per direction (0 fwd, 1 bwd): [2H][H], 2 block scales
    const int8_t* uc[2]; const float* uc_s[2];
    float* gh;       // [2][2H] scratch
    float* ghc;      // [2][H] scratch
    float* states;   // [l][2H] output, backward half first (layers.py:342)
    float* h2;       // [2][H] final states (fwd, bwd)
    int32_t* ctl;    // [3..4] grid barrier
    int32_t* err;
};
int enc1_launch(const PeArgs& a, cudaStream_t st);
extern int g_enc1;

}  // namespace qnmt
