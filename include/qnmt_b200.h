/*
 * qnmt_b200.h -- C ABI of the B200-native int8 NMT decode path.
 *
 * The reference (arXiv 1804.05038's engine, Python package ``qnmt`` under
 * /root/reference/pkg/src/qnmt) has no FFI: its drop-in surface is the Python
 * API.  Each entry point below replaces the arithmetic behind one reference
 * function; the Python package ``paper_1804_05038_b200`` binds them with
 * ctypes and mirrors the reference names, argument meaning and exceptions.
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers unless a parameter says "host".
 *    Callers own every buffer (the library never frees caller memory); the
 *    engine handle owns only its scratch.
 *  - Activations are stored column-major w.r.t. the reference's ``[features, P]``
 *    convention (layers.py:9-11): one contiguous row of ``features`` values per
 *    column, i.e. a ``[N][K]`` array with row stride ``ld``.  Weights are the
 *    reference's ``[out][in]`` row-major int8 codes (qmath.py:63).
 *  - ``stream`` is a ``cudaStream_t`` (NULL = legacy default stream).
 *  - Return value: QNMT_OK or an error code; codes map 1:1 onto the reference
 *    exceptions (errors.py:4-47).  ``qnmt_last_error()`` gives a message.
 *  - Device-side numeric checks (non-finite activations, out-of-range ids)
 *    set bits in a caller-provided sticky ``err_flag`` (int32, device); the
 *    caller maps them with QNMT_FLAG_* after synchronising.
 */
#ifndef QNMT_B200_H
#define QNMT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define QNMT_ABI_VERSION 1

enum {
    QNMT_OK = 0,
    QNMT_ERR_SHAPE = 1,          /* errors.py:12  ShapeError        */
    QNMT_ERR_INVALID_INPUT = 2,  /* errors.py:8   InvalidInputError */
    QNMT_ERR_NUMERIC = 3,        /* errors.py:45  NumericError      */
    QNMT_ERR_VOCAB = 4,          /* errors.py:29  VocabError        */
    QNMT_ERR_CONFIG = 5,         /* errors.py:37  ConfigError       */
    QNMT_ERR_EMPTY = 6,          /* errors.py:33  EmptyInputError   */
    QNMT_ERR_CUDA = 7            /* device / launch failure          */
};

/* sticky device error-flag bits */
#define QNMT_FLAG_NUMERIC 1   /* non-finite activation (qmath.py:180, layers.py:30/65) */
#define QNMT_FLAG_INVALID 2   /* non-finite weight (qmath.py:152)                        */
#define QNMT_FLAG_VOCAB 4     /* token id outside the vocabulary (layers.py:318, :366)    */
#define QNMT_FLAG_SHARD_TIE 8 /* K7 combine: a row's top-k may hold a token outside the
                                 shards' lists (f32 score tie); recompute it unsharded   */

/* qmath.py:41 -- int32 accumulation is safe up to this K */
#define QNMT_INT32_SAFE_K 131000

int qnmt_abi_version(void);
const char* qnmt_last_error(void);
int qnmt_device_sync(void);

/* ---------------------------------------------------------------------------
 * K1 quantize  (replaces qmath.quantize :145-154, quantize_activations
 * :172-182, _max_abs_scan :157-169, _encode :136-142, _encode_i8 :119-133)
 *
 * x: [ncols][K] f32, row stride ldx.  Column c belongs to segment
 * col_seg[c] (col_seg == NULL: every column is segment 0).  One scale per
 * segment: s = fl32(127 / max|x_seg|) (1.0 when the max is 0); codes are
 * sign(v)*floor(fl32(|v|+0.5)), v = fl32(x*s), clamped to +-127.
 * q: [ncols][ldq] int8; scales: [nseg] f32; seg_maxbits: [nseg] u32 scratch.
 * mode 0 = weights (non-finite -> QNMT_FLAG_INVALID),
 * mode 1 = activations (non-finite -> QNMT_FLAG_NUMERIC).
 * ------------------------------------------------------------------------- */
int qnmt_quantize(const float* x, int64_t ncols, int64_t K, int64_t ldx,
                  const int32_t* col_seg, int32_t nseg,
                  int8_t* q, int64_t ldq, float* scales, uint32_t* seg_maxbits,
                  int32_t mode, int32_t* err_flag, void* stream);

/* LinearOp.apply of the int8 path (layers.py:124-146): y = W q(x) (+ bias) with
 * one activation scale over the whole input (quantize_activations,
 * qmath.py:172-182) and the exact dequant of qnmt_gemm_i8.  X: f32 K-major
 * [N][ldx]; codes_out [N][ldc] and scale_out[1] receive q(x) and its scale;
 * maxbits: 1 word of device scratch (general shapes).  N <= 8 (the batch-1
 * latency path, cfg1) runs as ONE kernel: every CTA quantizes the input into
 * its shared memory and streams its weight rows (weights prefetched before
 * the PDL wait with QNMT_GEMM_W_STATIC); larger N: quantize kernels + GEMM.
 * Non-finite x sets QNMT_FLAG_NUMERIC. */
int qnmt_linear_i8(const int8_t* W, int64_t M, int64_t K, int64_t ldw, const float* w_scales,
                   int64_t w_rows_per_scale, const float* X, int64_t N, int64_t ldx, const float* bias,
                   float* Y, int64_t ldy, int8_t* codes_out, int64_t ldc, float* scale_out,
                   uint32_t* maxbits, int32_t flags, int32_t* err_flag, void* stream);

/* dequantize (qmath.py:185-187): y = f32(code) / scale, scale a host float */
int qnmt_dequantize(const int8_t* q, int64_t n, float scale, float* y, void* stream);

/* ---------------------------------------------------------------------------
 * K2/K3 int8 GEMM with fused dequant epilogue  (replaces qgemm :384-397,
 * qgemm_panel :400-427, _scale_output :379-381, and LinearOp.apply's bias
 * add layers.py:144-145)
 *
 *   acc[n][m] = sum_k W[m][k] * X[n][k]              (exact; int64 if K > SAFE_K)
 *   y = fl32( f64(acc) / (f64(w_scales[m / w_rows_per_scale]) * f64(x_scales[seg(n)])) )
 *   if bias:            y = fl32(y + bias[m])
 *   if ACCUMULATE:      y = fl32(Y[n][m] + y)
 *   Y[n][m] = y           (Y: [N][ldy] f32; may be NULL if acc_out given)
 *   acc_out (nullable): [N][M] int64 raw accumulators
 * seg(n) = col_seg[n] (col_seg NULL -> 0).  Scales are device f32 arrays.
 * ------------------------------------------------------------------------- */
#define QNMT_GEMM_ACCUMULATE 1
/* W is not written by the kernels immediately preceding this call on the stream
 * (model weights): the CUDA-core GEMV may stream W before its programmatic-
 * dependent-launch wait, overlapping the predecessor kernel. */
#define QNMT_GEMM_W_STATIC 2
int qnmt_gemm_i8(const int8_t* W, int64_t M, int64_t K, int64_t ldw,
                 const float* w_scales, int64_t w_rows_per_scale,
                 const int8_t* X, int64_t N, int64_t ldx,
                 const float* x_scales, const int32_t* col_seg,
                 const float* bias, float* Y, int64_t ldy,
                 int64_t* acc_out, int32_t flags, void* stream);

/* GEMM implementation selector (testing / A-B measurement): 0 = auto
 * (tcgen05 for N > 8, dp4a GEMV otherwise), 1 = CUDA-core dp4a only,
 * 2 = tcgen05 whenever the shape is eligible.  Returns the previous value. */
int qnmt_set_gemm_impl(int impl);
/* 1 (default): products with at least one wave of 256 x 256 tiles use the
 * CTA-pair tcgen05 kernel (cta_group::2, M = 256); 0: single-CTA tiles only.
 * Results are identical.  Returns the old value. */
int qnmt_set_tc_pair(int enable);
/* 1 (default): translations of one sentence at beam 1 run the persistent
 * batch-1 decode kernel (one cooperative launch for all steps); 0: the step
 * graphs.  Results are identical.  Returns the old value. */
int qnmt_set_greedy1(int enable);

/* fp32 precision path: replaces qmath.py:434-440
 * (gemm_f32) in LinearOp's float branch (layers.py:138-145).
 *   Y[n][m] = fl32(sum_k f64(W[m][k]) f64(X[n][k])) (+ bias[m]) (+ Y[n][m] if
 *   flags & QNMT_GEMM_ACCUMULATE); W [M][ldw] f32, X K-major [N][ldx] f32. */
int qnmt_gemm_f32(const float* W, int64_t M, int64_t K, int64_t ldw, const float* X, int64_t N,
                  int64_t ldx, const float* bias, float* Y, int64_t ldy, int32_t flags, void* stream);

/* ---------------------------------------------------------------------------
 * GRU gate arithmetic (layers.py:170-181), f32 ops in the reference's
 * association order, sigmoid/tanh evaluated in fp64 and rounded once.
 *   gx : [*][3H] x-side pre-activations (Wz x+bz | Wr x+br | Wc x+bc), row of
 *        column n is gx_row[n] (NULL -> n), stride ldgx
 *   gh : [N][2H] state-side products (Uz h | Ur h), stride ldgh
 *   z  = sigmoid(gx_z + gh_z), r = sigmoid(gx_r + gh_r), rh = r * h
 * qnmt_gru_combine:  cand = tanh(gx_c + ghc); h_out = (1 - z) * h + z * cand
 *   h_out row n also copied to out2 row out2_row[n] (if out2 != NULL).
 * ------------------------------------------------------------------------- */
int qnmt_gru_gates(const float* gx, int64_t ldgx, const int32_t* gx_row,
                   const float* gh, int64_t ldgh, const float* h, int64_t ldh,
                   int64_t N, int64_t H, float* z, float* rh, int32_t* err_flag, void* stream);
int qnmt_gru_combine(const float* gx, int64_t ldgx, const int32_t* gx_row,
                     const float* ghc, int64_t ldghc, const float* z, const float* h, int64_t ldh,
                     int64_t N, int64_t H, float* h_out, int64_t ldo,
                     float* out2, int64_t ld2, const int32_t* out2_row,
                     int32_t* err_flag, void* stream);

/* y = tanh(x) elementwise (fp64-evaluated, rounded once), [N][D] rows */
int qnmt_tanh(const float* x, int64_t N, int64_t D, int64_t ldx, float* y, int64_t ldy,
              int32_t* err_flag, void* stream);

/* ---------------------------------------------------------------------------
 * Attention (layers.py:214-241) for N query columns.
 *   sentence s (< n_sent) owns columns [sent_col_off[s], +sent_ncols[s]) (at
 *   most 16), has length sent_len[s], and its att_proj / states rows start at
 *   row sent_row[s] of att_proj [*][A] and states [*][2H] (position-major);
 *   A <= 2048.
 *   u = state_proj(query) : [N][A] (stride ldu), v: [A] int8 codes, v_scale
 *   device f32[1].
 *   scores[n][i] = v . q(tanh(att_proj_i + u_n)) with ONE scale per column
 *   over its whole [A, l] block (layers.py:224-226);
 *   alpha = softmax_i(scores) (fp64, rounded); ctx = sum_i alpha_i states_i
 *   (fp64, rounded).
 *   att_minmax (nullable): [n_sent][2][A] per-sentence column max / min of
 *   att_proj (qnmt_attention_stats); computed into scratch when NULL.
 *   att_exp (nullable): fl32(e^(2 att_proj)) in att_proj's layout
 *   (qnmt_attention_exp, once per encoder output): enables the one-MUFU
 *   scorer (same results; sentences with |att_proj| or |u| > 20 use the
 *   two-MUFU one).
 *   ctx: [N][2H] (ldc); alpha (nullable): [N][lda];
 *   scratch: >= 4*(N*max_len + 4*N + 192 + 2*n_sent*A + N*A) bytes
 * ------------------------------------------------------------------------- */
/* fp32 attend (layers.py:214-241 with float LinearOps): scores
 * fl32(sum_a f64(v_a) f64(tanh(att_proj + u))) then the same softmax/context as
 * qnmt_attention.  v: f32 [A]; scratch >= 4*N*max_len bytes. */
int qnmt_attention_f32(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                       const int32_t* sent_ncols, int32_t n_sent, const float* att_proj,
                       const float* states, const int64_t* sent_row, const int32_t* sent_len,
                       int32_t max_len, int64_t A, int64_t H2, const float* v, float* ctx, int64_t ldc,
                       float* alpha, int64_t lda, void* scratch, int32_t* err_flag, void* stream);
int qnmt_attention_stats(const float* att_proj, const int64_t* sent_row, const int32_t* sent_len,
                         int32_t n_sent, int64_t A, float* att_minmax, void* stream);
/* att_exp[i] = fl32(e^(2 att_proj[i])) (fp64 exp, rounded once) for n values
 * (values beyond +-20 clamped: their sentences take the two-MUFU scorer). */
int qnmt_attention_exp(const float* att_proj, int64_t n, float* att_exp, void* stream);
/* Scorer variant when att_exp is supplied (A/B testing; results identical):
 * 0 two-MUFU (k_att_score5), 1 one-MUFU (k_att_score6), 2 one-MUFU with the
 * tile staged by a bulk copy (k_att_score7).  Returns the previous value. */
int qnmt_set_att_exp(int32_t enable);
/* Testing knob of the one-MUFU scorer: length of its per-CTA deferred fixup queue
 * (0..512, default 512; 0 sends every window hit through the overflow rescan).
 * Returns the previous value. */
int qnmt_set_att_fixcap(int32_t cap);
/* Context kernel variant (A/B testing; results identical): 0 direct loads,
 * 1 bulk-copy ring with 1024 features per CTA, 2 bulk-copy ring with 512
 * features per CTA (used when the batch's hypotheses per sentence are <= 8).
 * Returns the previous value. */
int qnmt_set_att_ctx(int32_t mode);
/* 1: the two-MUFU scorer computes the per-hypothesis scales in its own CTAs
 * (k_att_score5f, no k_att_scale launch); 0 (default): separate scale kernel
 * (A/B testing; results identical).  Returns the previous value. */
int qnmt_set_att_fused_scale(int32_t enable);
/* 1 (default): the two-MUFU scorer stages its tile with one bulk copy before
 * the PDL wait (k_att_score8); 0: register-staged k_att_score5 (A/B testing;
 * results identical).  Returns the previous value. */
int qnmt_set_att_score8(int32_t enable);
/* 1: tile-starved tcgen05 products (fewer output tiles than half the SMs)
 * split K over more CTAs, exact int32 partial sums added in a per-stream
 * workspace; 0 (default, measured faster at cfg1 B=64): never split (A/B
 * testing; results identical).  Returns the previous value. */
int qnmt_set_tc_split(int enable);
/* 1: in batched decode steps (more than 8 columns) the GRU gate
 * nonlinearities run in the tcgen05 GEMM epilogues -- z = sigmoid(W_z x + U_z h)
 * and r*h on the accumulators of the cell's input GEMM, h' = (1-z) h + z tanh(..)
 * on those of the candidate GEMM (layers.py:170-181) -- with the per-sentence
 * max |.| for the next quantization reduced there too; 0 (default, measured
 * faster on the cfg5 decode): the separate fused elementwise + quantize kernels.
 * Results are identical.  Returns the old value. */
int qnmt_set_gate_epi(int enable);
/* Tile widths (64..256, multiple of 32; 0 = the general rule) of the two GRU-epilogue
 * GEMMs (tuning knob; results identical).  Returns the old gates width. */
int qnmt_set_gru_epi_bn(int gates_bn, int combine_bn);
int qnmt_attention(const float* u, int64_t ldu, int64_t N, const int32_t* sent_col_off,
                   const int32_t* sent_ncols, int32_t n_sent,
                   const float* att_proj, const float* att_minmax, const float* att_exp,
                   const float* states,
                   const int64_t* sent_row,
                   const int32_t* sent_len, int32_t max_len, int64_t A, int64_t H2,
                   const int8_t* v_codes, const float* v_scale,
                   float* ctx, int64_t ldc, float* alpha, int64_t lda,
                   void* scratch, int32_t* err_flag, void* stream);

/* ---------------------------------------------------------------------------
 * Output softmax (layers.py:60-67) and beam candidates (decoder.py:74-85,
 * :125).  logits: [N][V] f32 (ld).
 *   lp = fl32( (f64 v - f64 max) - log(sum exp(f64 v - f64 max)) )
 * qnmt_log_softmax writes lp [N][ldlp].
 * qnmt_topk_candidates: per column n, the k best (score desc, token asc) with
 *   score = live_scores[n] + f64(lp); cand_score [N][k] f64, cand_tok [N][k].
 * ------------------------------------------------------------------------- */
int qnmt_log_softmax(const float* logits, int64_t N, int64_t V, int64_t ld,
                     float* lp, int64_t ldlp, int32_t* err_flag, void* stream);
int qnmt_topk_candidates(const float* logits, int64_t N, int64_t V, int64_t ld,
                         const double* live_scores, int32_t k,
                         double* cand_score, int32_t* cand_tok, int32_t* err_flag, void* stream);

/* 1 = use the three-pass reference candidate kernel instead of the single-pass
 * one (A/B testing; results are identical by construction).  Returns old. */
int qnmt_set_topk_exact(int exact);

/* 1 (default) = the engine's decode loop runs the vocabulary projection fused
 * with the log-softmax statistics and the candidate selection (the [N][V]
 * logits never reach HBM); 0 = vocab GEMM + qnmt_topk_candidates (A/B
 * testing; results are identical by construction).  Returns old. */
int qnmt_set_vocab_fused(int enable);

/* Fused vocabulary projection + log-softmax statistics + beam candidates
 * (vocab_topk.cu): the same candidates as qnmt_gemm_i8 (bias) followed by
 * qnmt_topk_candidates, without materialising the [N][V] logits.
 *   X: [N][ldx] readout codes, x_scales[row_seg[n]]; W: [V][ldw] vocabulary
 *   codes, w_scales[v / w_rows_per_scale]; bias: [V] or NULL; live: [N] or NULL.
 *   K % 16 == 0, ldx/ldw % 16 == 0, 16-byte aligned X/W, 1 <= k <= min(16, V).
 *   scratch: qnmt_vocab_candidates_scratch(N, V) bytes of device memory. */
int qnmt_vocab_candidates(const int8_t* X, int64_t N, int64_t ldx, const float* x_scales,
                          const int32_t* row_seg, const int8_t* W, int64_t V, int64_t K, int64_t ldw,
                          const float* w_scales, int64_t w_rows_per_scale, const float* bias,
                          const double* live_scores, int32_t k, void* scratch, double* cand_score,
                          int32_t* cand_tok, int32_t* err_flag, void* stream);
int64_t qnmt_vocab_candidates_scratch(int64_t N, int64_t V);

/* ---------------------------------------------------------------------------
 * K7: vocabulary-sharded output projection (the optional NCCL
 * variant of layers.py:266 + :60-67 + decoder.py:74-85).  A shard owns W_vocab
 * rows [tok_off, tok_off + V_shard) (W, bias and the scale pointer passed at
 * that offset).
 *   qnmt_vocab_shard_partials: per hypothesis row n, parts[n] = the shard's
 *     max logit M, S = sum exp(x - M) (fp64) and its top-8 logits by (logit
 *     desc, token asc) with global token ids (qnmt_vocab_shard_part_bytes()
 *     bytes per row; scratch: qnmt_vocab_candidates_scratch(N, V_shard)).
 *   qnmt_vocab_shard_combine: parts = [G][N] (the shards' partials, e.g. after
 *     an all-gather) -> cand_score/cand_tok [N][k] exactly as
 *     qnmt_vocab_candidates over the whole vocabulary, unless a row sets
 *     QNMT_FLAG_SHARD_TIE (then recompute that step unsharded).  G, k <= 16.
 * ------------------------------------------------------------------------- */
int64_t qnmt_vocab_shard_part_bytes(void);
int qnmt_vocab_shard_partials(const int8_t* X, int64_t N, int64_t ldx, const float* x_scales,
                              const int32_t* row_seg, const int8_t* W, int64_t V_shard, int64_t K, int64_t ldw,
                              const float* w_scales, int64_t w_rows_per_scale, const float* bias, int64_t tok_off,
                              void* scratch, void* parts, int32_t* err_flag, void* stream);
int qnmt_vocab_shard_combine(const void* parts, int32_t G, int64_t N, const double* live_scores, int32_t k,
                             double* cand_score, int32_t* cand_tok, int32_t* err_flag, void* stream);

/* Embedding gather (layers.py:324, :367): out[n] = table[ids[n]] ([rows][E]);
 * ids outside [0, rows) raise QNMT_FLAG_VOCAB and yield zeros. */
int qnmt_embed_gather(const float* table, int64_t rows, int64_t E, const int32_t* ids,
                      int64_t n, float* out, int64_t ldo, int32_t* err_flag, void* stream);

/* ---------------------------------------------------------------------------
 * Model + batched translation engine (decoder.py:88-160 translate,
 * layers.py:313-384 encode / decoder_step, bench.py:126-132 corpus loop).
 *
 * qnmt_model_create takes device pointers in the order of QNMT_T_* below
 * (the per-cell weights are the reference's per-gate tensors stacked:
 * WX = [wz; wr; wc] with 3 scales, UZR = [uz; ur] with 2 scales, UC = uc).
 * ------------------------------------------------------------------------- */
enum {
    QNMT_T_SRC_EMBED = 0, QNMT_T_TGT_EMBED = 1,
    /* cell c in {0 enc_fwd, 1 enc_bwd, 2 dec_r, 3 dec_q}: base = 2 + 7*c */
    QNMT_T_CELL_WX = 0, QNMT_T_CELL_WX_SCALES = 1, QNMT_T_CELL_BX = 2,
    QNMT_T_CELL_UZR = 3, QNMT_T_CELL_UZR_SCALES = 4, QNMT_T_CELL_UC = 5,
    QNMT_T_CELL_UC_SCALE = 6,
    QNMT_T_ATT_WENC = 30, QNMT_T_ATT_WENC_SCALE = 31, QNMT_T_ATT_BENC = 32,
    QNMT_T_ATT_USTATE = 33, QNMT_T_ATT_USTATE_SCALE = 34,
    QNMT_T_ATT_V = 35, QNMT_T_ATT_V_SCALE = 36,
    QNMT_T_OUT_WSTATE = 37, QNMT_T_OUT_WSTATE_SCALE = 38, QNMT_T_OUT_BREADOUT = 39,
    QNMT_T_OUT_WEMBED = 40, QNMT_T_OUT_WEMBED_SCALE = 41,
    QNMT_T_OUT_WCTX = 42, QNMT_T_OUT_WCTX_SCALE = 43,
    QNMT_T_OUT_WVOCAB = 44, QNMT_T_OUT_WVOCAB_SCALE = 45, QNMT_T_OUT_BVOCAB = 46,
    QNMT_T_S0_W = 47, QNMT_T_S0_W_SCALE = 48, QNMT_T_S0_B = 49,
    QNMT_T_COUNT = 50
};

/* dims: {src_vocab, tgt_vocab, embed, hidden, attn, readout, s0_mode(0 transform,
 *        1 zero), attention_query(0 current, 1 previous)} */
typedef struct qnmt_model qnmt_model;
typedef struct qnmt_engine qnmt_engine;

int qnmt_model_create(const int32_t* dims, const void* const* tensors, int32_t ntensors,
                      qnmt_model** out);
/* fp32 model (same tensor table; weight slots hold f32 matrices, scale slots
 * are ignored): engines built on it decode with the fp32 path. */
int qnmt_model_create_f32(const int32_t* dims, const void* const* tensors, int32_t ntensors,
                          qnmt_model** out);
int qnmt_model_destroy(qnmt_model* m);

/* Engine: scratch for up to max_sentences sentences of length <= max_src_len
 * at beam width <= max_beam. */
int qnmt_engine_create(const qnmt_model* m, int32_t max_sentences, int32_t max_src_len,
                       int32_t max_beam, qnmt_engine** out);
int qnmt_engine_destroy(qnmt_engine* e);

/* Translate n_sent sentences (each exactly as decoder.translate with one
 * model and the given beam / max_ratio).
 *   src_ids (host): concatenated source ids; src_len (host): lengths.
 *   out_tokens (host): [n_sent][out_stride] target ids without the final EOS
 *   out_len (host), out_logp (host): length and total log-prob per sentence.
 *   out_stride must be >= ceil(max_ratio * max_len) + 1.
 * Returns QNMT_ERR_EMPTY / _VOCAB / _NUMERIC / _CONFIG like translate. */
int qnmt_translate_batch(qnmt_engine* e, const int32_t* src_ids, const int32_t* src_len,
                         int32_t n_sent, int32_t beam, double max_ratio,
                         int32_t* out_tokens, int32_t out_stride, int32_t* out_len,
                         double* out_logp, void* stream);

/* Ensemble translation (decoder.py:88-160 with several models, :115-120):
 * per step every member runs its own decoder step on its own states; the
 * per-column log-probs are summed in member order in f32 and divided by
 * f32(n_members); search state lives in engines[0].  Every engine must come
 * from a model with the same target vocabulary size and have the same
 * capacity.  src_ids holds n_members x sum(src_len) ids, member-major (each
 * member maps the tokens with its own source vocabulary, decoder.py:99).
 * 1 <= n_members <= QNMT_ENS_MAX (1 = qnmt_translate_batch).  Same outputs as
 * qnmt_translate_batch (replaces decoder.py:115-120 for ensembles). */
#define QNMT_ENS_MAX 8
int qnmt_translate_ensemble(qnmt_engine* const* engines, int32_t n_members, const int32_t* src_ids,
                            const int32_t* src_len, int32_t n_sent, int32_t beam, double max_ratio,
                            int32_t* out_tokens, int32_t out_stride, int32_t* out_len,
                            double* out_logp, void* stream);

/* Encoder only (layers.py:313-348) for a batch, device in/out:
 *   src_ids (device) concatenated, sent_row (host) row offsets, src_len (host).
 *   states [sum_l][2H] (backward half first, layers.py:342), att_proj [sum_l][A],
 *   s0 [n_sent][H]. */
int qnmt_encode_batch(qnmt_engine* e, const int32_t* src_ids_dev, const int32_t* src_len,
                      int32_t n_sent, float* states, float* att_proj, float* s0,
                      void* stream);

/* One decoder step (layers.py:356-384) for N hypothesis columns of n_sent
 * sentences, all buffers on device:
 *   col_sent [N] sentence of each column (activation scales are per sentence,
 *   i.e. per reference decoder_step call); y [N] previous tokens; s, sp [N][H]
 *   state and previous intermediate state; states/att_proj from
 *   qnmt_encode_batch with sent_row [n_sent] (int64) / sent_len [n_sent];
 *   outputs s_int, s_new [N][H], logits [N][V] (log_softmax is separate),
 *   alpha [N][lda] (nullable). */
int qnmt_decoder_step(qnmt_engine* e, int64_t N, const int32_t* col_sent, int32_t n_sent,
                      const int32_t* y, const float* s, const float* sp, const float* states,
                      const float* att_proj, const int64_t* sent_row, const int32_t* sent_len,
                      int32_t max_len, float* s_int, float* s_new, float* logits, float* alpha,
                      int64_t lda, void* stream);

/* Device-resident variant for benchmarking / pipelines: src_ids already on the
 * device, results kept in the engine until qnmt_fetch_results (the final
 * min-by-(-logp, tokens) selection of decoder.py:157 runs on the device, then
 * one D2H of n * (max_steps + 3) words). */
int qnmt_decode_batch_device(qnmt_engine* e, const int32_t* src_ids_dev, const int32_t* src_len,
                             int32_t n_sent, int32_t beam, double max_ratio, void* stream);
int qnmt_fetch_results(qnmt_engine* e, int32_t* out_tokens, int32_t out_stride, int32_t* out_len,
                       double* out_logp, void* stream);
/* bytes copied device->host by the last fetch */
int64_t qnmt_last_d2h_bytes(const qnmt_engine* e);
/* bytes copied host->device by the last decode call (ids, lengths, batch plan, search init) */
int64_t qnmt_last_h2d_bytes(const qnmt_engine* e);
/* kernels launched by this library since load (process-wide counter) */
int64_t qnmt_kernel_launches(void);

/* 1 (default): decode steps run as captured CUDA graphs with a device-side
 * live-column count (host polls it every 16 steps); 0: eager per-step loop
 * with one host sync per step.  Results are identical.  Returns old value. */
int qnmt_engine_set_graphs(qnmt_engine* e, int enable);

/* Device-clock stamps (%globaltimer) inside the captured decode steps, for
 * live per-kernel timing in graph mode.  After a decode, _read copies one row
 * of QNMT_STAMP_COLS int64 per executed step: [step start, attention start,
 * attention end, candidate merge start, candidate merge end, vocab projection
 * start, vocab projection end, (unused), live columns N, sum of source lengths
 * of live sentences, sum over sentences of live hypotheses x source length];
 * returns the number of rows.  With the fused vocabulary path the projection
 * interval is k_vocab_stats and the merge interval k_vocab_merge; otherwise
 * the vocab GEMM and qnmt_topk_candidates. */
#define QNMT_STAMP_COLS 11
int qnmt_engine_stamps(qnmt_engine* e, int enable);
int qnmt_engine_stamps_read(qnmt_engine* e, int64_t* out, int32_t max_rows, void* stream);

/* Phase profiler (forces the eager loop while enabled): CUDA events on the engine stream around the kernel groups
 * of a decode (0 encoder, 1 embed, 2 quantize, 3 decoder GEMMs, 4 GRU gates,
 * 5 attention, 6 vocab GEMM, 7 top-k, 8 search, 9 gather, 10 misc).
 * qnmt_engine_profile(e, 1) resets and enables; _read fills [16] arrays with
 * elapsed ms, launches, algorithmic int-ops and algorithmic bytes per group. */
int qnmt_engine_profile(qnmt_engine* e, int enable);
int qnmt_engine_profile_read(const qnmt_engine* e, double* ms, double* calls, double* ops, double* bytes);

/* device bytes held by the engine (scratch + history) */
size_t qnmt_engine_bytes(const qnmt_engine* e);
/* Checked mode (QNMT_CANARY=1 in the environment when the engine is created):
 * every device buffer of the engine is followed by a 256-byte guard band of
 * 0xA5.  Returns the number of guard bytes that changed (0: no out-of-bounds
 * write into a neighbouring buffer so far), -1 if the engine is not in checked
 * mode.  Synchronises the stream. */
int64_t qnmt_engine_check_canaries(qnmt_engine* e, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* QNMT_B200_H */
