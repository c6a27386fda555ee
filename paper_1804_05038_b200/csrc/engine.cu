// engine.cu -- model handle and the batched translation engine.
//
// Batched form of decoder.translate (decoder.py:88-160) over many sentences
// at once, bit-identical to running translate sentence by sentence:
//  * every activation quantization keeps the reference's granularity
//    (one scale per LinearOp.apply call) via per-segment
//    scales: segment = sentence (decoder), = (sentence, direction) (encoder
//    state side), = position (encoder input side), = sentence (att_proj, s0);
//  * the search runs on device (search.cu) one thread per sentence;
//  * the host only reads back the live-column count once per step and the
//    finished lists / history once per batch.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <numeric>
#include <mutex>
#include <shared_mutex>
#include <vector>

#include "gemm.cuh"
#include "kernels.cuh"
#include "persistent.cuh"
#include "search.cuh"

namespace qnmt {


struct Cell {
    const int8_t* wx;
    const float* wx_s;
    const float* bx;
    const int8_t* uzr;
    const float* uzr_s;
    const int8_t* uc;
    const float* uc_s;
    int in;
};

}  // namespace qnmt

struct qnmt_model {
    int Vs, Vt, E, H, A, R, s0_mode, aq;
    const float* src_embed;
    const float* tgt_embed;
    qnmt::Cell cell[4];
    const int8_t* w_enc; const float* w_enc_s; const float* b_enc;
    const int8_t* u_att; const float* u_att_s;
    const int8_t* v; const float* v_s;
    const int8_t* w_state; const float* w_state_s; const float* b_r;
    const int8_t* w_embed; const float* w_embed_s;
    const int8_t* w_ctx; const float* w_ctx_s;
    const int8_t* w_vocab; const float* w_vocab_s; const float* b_vocab;
    const int8_t* s0_w; const float* s0_s; const float* s0_b;
    int fp32 = 0;   // 1: the fp32 precision path -- every weight pointer above holds f32 values, no scales
};

namespace qnmt {

// simple bump allocator over one cudaMalloc block
// Bump allocator of an engine's device block.  Checked mode (QNMT_CANARY=1 in the
// environment when the engine is created): every buffer is followed by a 256-byte
// guard band filled with 0xA5; qnmt_engine_check_canaries counts guard bytes that
// changed -- an out-of-bounds write into a neighbouring buffer (the memcheck class
// of bug) shows up there.  (compute-sanitizer is not available on the GPU pool.)
constexpr size_t ARENA_GUARD = 256;
struct Arena {
    char* base = nullptr;
    size_t cap = 0, used = 0;
    bool guard = false;
    std::vector<size_t>* guards = nullptr;   // guard band offsets (checked mode)
    template <typename T>
    T* take(size_t n) {
        size_t bytes = (n * sizeof(T) + 255) & ~(size_t)255;
        T* p = reinterpret_cast<T*>(base + used);
        used += bytes;
        if (guard) {
            if (guards) guards->push_back(used);
            used += ARENA_GUARD;
        }
        return p;
    }
};

__global__ void k_check_guards(const unsigned char* base, const size_t* offs, int n, unsigned long long* bad) {
    for (int g = blockIdx.x; g < n; g += gridDim.x) {
        const unsigned char* p = base + offs[g];
        int c = 0;
        for (int i = threadIdx.x; i < (int)ARENA_GUARD; i += blockDim.x) c += p[i] != 0xA5;
        c = __reduce_add_sync(0xffffffffu, c);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, (unsigned long long)c);
    }
}

}  // namespace qnmt

struct qnmt_engine {
    const qnmt_model* m;
    int S, L, B;       // max sentences, max source length, max beam
    int64_t NMAX;      // S * B
    int64_t PMAX;      // S * L
    char* block = nullptr;
    size_t block_bytes = 0;
    bool guard = false;              // checked mode: guard bands after every device buffer
    std::vector<size_t> guards;      // their offsets in block
    size_t* guards_dev = nullptr;
    // shared
    int32_t* err;            // device sticky flag
    uint32_t* seg_bits;      // [max(PMAX, 2S, S)]
    int32_t* iota;           // [max(PMAX, 2S)] identity
    int32_t* even;           // [S] 0,2,4..
    int32_t* odd;            // [S] 1,3,5..
    // encoder
    int32_t* src_ids;        // [PMAX]
    float* emb_src;          // [PMAX][E]
    int8_t* q_emb_src;       // [PMAX][E]
    float* sc_pos;           // [PMAX]
    float* gx_enc;           // [PMAX][2][3H]
    float* h2;               // [S][2][H]
    int8_t* q_h2;            // [S][2][H]
    float* sc_h2;            // [2S]
    float* gh2;              // [S][2][2H]
    float* z2;               // [2S][H]
    float* rh2;              // [2S][H]
    int8_t* q_rh2;           // [2S][H]
    float* sc_rh2;           // [2S]
    float* ghc2;             // [S][2][H]
    int32_t* enc_rows;       // [L][2S] gx rows per step
    int32_t* enc_out_rows;   // [L][2S] states half-rows per step
    uint32_t* enc_qm;        // [L+1][2][2S] fused max-abs bits of h2 (slot 0) / rh2 (slot 1) per step
    int8_t* q_states;        // [PMAX][2H]
    float* sc_sent;          // [S]
    int32_t* pos_sent;       // [PMAX] sentence of each position
    float* s0tmp;            // [S][H]
    int32_t* s0_dst;         // [S] original index of sorted slot
    float* enc_states;       // [PMAX][2H]  (engine-owned encoder output for translate)
    float* enc_att;          // [PMAX][A]
    float* enc_attx;         // [PMAX][A] fl32(e^(2 att_proj)) for the one-MUFU attention scorer
    float* enc_s0;           // [S][H]
    int64_t* sent_row;       // [S]
    int32_t* sent_len;       // [S]
    // decoder (NMAX columns)
    float* emb;              // [N][E]
    int8_t* q_emb;           // [N][E]
    float* sc_emb;           // [S]
    int8_t* q_s;             // [N][H]
    float* sc_s;
    float* gx;               // [N][3H]
    float* gh;               // [N][2H]
    float* z;                // [N][H]
    float* rh;               // [N][H]
    int8_t* q_rh;
    float* sc_rh;
    float* ghc;              // [N][H]
    int8_t* q_q;             // query codes [N][H]
    float* sc_q;
    float* u;                // [N][A]
    float* ctx;              // [N][2H]
    int8_t* q_ctx;
    float* sc_ctx;
    int8_t* q_si;            // s_int codes (when query != s_int)
    float* sc_si;
    int8_t* q_sn;
    float* sc_sn;
    float* ro;               // [N][R]
    int8_t* q_ro;
    float* sc_ro;
    float* logits;           // [N][V]
    void* vocab_part;        // fused vocab projection partials (vocab_topk_part_bytes(N, V))
    void* att_scratch;
    float* att_mm;           // [S][2][A] per-sentence column max / min of att_proj
    uint32_t* ctx_max;       // [S] max |ctx| bits per sentence (attention context -> its quantization)
    uint32_t* gmax = nullptr; // [4][S] max |r*h| / |h'| bits per sentence of the two decoder cells (GRU epilogues)
    bool gate_epi = false;   // GRU gates / combine run in the tcgen05 GEMM epilogues (gemm.cuh GruEpi)
    bool fq_ok = false;      // per-sentence fused op + quantize kernels fit in shared memory (fused_q.cu)
    // Stacked weights (copied at engine creation) for GEMMs that share an input:
    //   w2x = [cell2 W_x; W_e] x q(emb), w3x = [cell3 W_x; W_c] x q(ctx): the readout terms
    //   W_e e and W_c c come out of the cells' input GEMMs and are added in the W_s epilogue;
    //   wuq = [U_att; cell3 U_zr] x q(s') (current-state query only).  Per-row scales.
    bool stack_ok = false, stack_u = false;
    int8_t* w2x = nullptr; float* w2x_s = nullptr; float* b2x = nullptr;
    int8_t* w3x = nullptr; float* w3x_s = nullptr; float* b3x = nullptr;
    int8_t* wuq = nullptr; float* wuq_s = nullptr;
    float* gxr = nullptr;    // [N][3H+R] cell2 input side + W_e e
    float* gxq = nullptr;    // [N][3H+R] cell3 input side + W_c c
    float* uq = nullptr;     // [N][A+2H] U_att q + cell3 U_zr s'
    // translate loop state
    float* st_s[2];          // [N][H] s
    float* st_sp[2];         // [N][H] s_prime
    float* s_int;            // [N][H]
    float* s_new;            // [N][H]
    int32_t* y[2];
    int32_t* col_sent[2];
    double* live[2];
    int32_t* parent_col;
    double* cand_score;      // [N][B]
    int32_t* cand_tok;
    int32_t* n_live;
    int32_t* P; int32_t* col_off; int32_t* done; int32_t* max_steps; int32_t* steps_run; int32_t* np_tmp;
    int32_t* pk_ctl;         // [8] persistent greedy kernel: y, best token, done, grid barrier
    int32_t* fin_cnt; double* fin_best;
    // history/finished (grown on demand)
    char* hblock = nullptr;
    size_t hblock_bytes = 0;
    int hist_steps = 0;
    double* fin_score; int32_t* fin_step; int32_t* fin_slot; int32_t* fin_eos;
    int32_t* hist_tok; int32_t* hist_par;
    int32_t* h_pinned = nullptr;   // host pinned scalar
    int32_t* res_dev = nullptr;    // [S][hist_steps + 3] packed results (k_finalize)
    int32_t* fin_scratch = nullptr;
    int32_t* res_host = nullptr;   // pinned staging of res_dev
    int last_n = 0, last_tmax = 0;
    int64_t d2h_bytes = 0;         // last batch: result bytes copied device -> host
    int64_t h2d_bytes = 0;         // last batch: host -> device bytes (ids, lengths, batch plan, search init)
    // phase profiler (CUDA events on the engine stream; off by default)
    bool prof_on = false;
    int prof_group = -1;
    cudaEvent_t prof_start = nullptr;
    std::vector<cudaEvent_t> ev_pool, ev_used;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_open;
    double prof_ms[16] = {}, prof_calls[16] = {}, prof_ops[16] = {}, prof_bytes[16] = {};
    // graph-captured decode steps (device-side live count and step counter)
    bool use_graphs = true;
    int32_t* d_N = nullptr;      // [2] live columns, ping-pong
    int32_t* rng_off = nullptr;  // [S] column ranges for qnmt_decoder_step callers
    int32_t* rng_cnt = nullptr;
    int32_t* d_step = nullptr;
    int graph_kernels = 1;        // kernel nodes in one captured step graph
    bool stamp_on = false;        // device-clock stamps in captured steps (qnmt_engine_stamps)
    long long* stamps = nullptr;  // [hist_steps][ST_COLS]
    cudaStream_t cap_stream = nullptr;
    std::vector<std::pair<std::pair<int, int>, std::pair<cudaGraphExec_t, cudaGraphExec_t>>> graphs;
};

namespace qnmt {

enum { PG_ENCODER = 0, PG_EMBED, PG_QUANT, PG_GEMM, PG_GRU, PG_ATT, PG_GEMM_VOCAB, PG_TOPK, PG_SEARCH,
       PG_GATHER, PG_MISC, PG_COUNT };

static cudaEvent_t prof_event(qnmt_engine* e) {
    cudaEvent_t ev;
    if (!e->ev_pool.empty()) {
        ev = e->ev_pool.back();
        e->ev_pool.pop_back();
    } else {
        cudaEventCreate(&ev);
    }
    e->ev_used.push_back(ev);
    return ev;
}

// close the open region (if any) and open one for group g (g < 0: just close)
static void prof_mark(qnmt_engine* e, int g, cudaStream_t st, double ops = 0, double bytes = 0) {
    if (!e->prof_on) return;
    cudaEvent_t ev = prof_event(e);
    cudaEventRecord(ev, st);
    if (e->prof_group >= 0) e->ev_open.push_back({e->prof_group, {e->prof_start, ev}});
    e->prof_group = g;
    e->prof_start = ev;
    if (g >= 0) {
        e->prof_calls[g] += 1;
        e->prof_ops[g] += ops;
        e->prof_bytes[g] += bytes;
    }
}

// after a stream sync: fold finished regions into the totals and recycle events
static void prof_collect(qnmt_engine* e) {
    if (!e->prof_on) return;
    for (auto& r : e->ev_open) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.second.first, r.second.second) == cudaSuccess) e->prof_ms[r.first] += ms;
    }
    e->ev_open.clear();
    for (auto ev : e->ev_used)
        if (ev != e->prof_start) e->ev_pool.push_back(ev);
    e->ev_used.clear();
    if (e->prof_group >= 0) e->ev_used.push_back(e->prof_start);
}

static int check_flag(qnmt_engine* e, cudaStream_t st) {
    int32_t f = 0;
    QNMT_CUDA(cudaMemcpyAsync(&f, e->err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    QNMT_CUDA(cudaStreamSynchronize(st));
    if (f & QNMT_FLAG_VOCAB) { set_error("token id outside the vocabulary"); return QNMT_ERR_VOCAB; }
    if (f & QNMT_FLAG_NUMERIC) { set_error("activations contain non-finite values"); return QNMT_ERR_NUMERIC; }
    if (f & QNMT_FLAG_INVALID) { set_error("invalid input (non-finite weight, or more than 16 hypotheses of one sentence in a step)"); return QNMT_ERR_INVALID_INPUT; }
    return QNMT_OK;
}

#define TRY(x) do { int _r = (x); if (_r != QNMT_OK) return _r; } while (0)

// host -> device copy of per-batch inputs, counted for the e2e traffic report
static cudaError_t h2d(qnmt_engine* e, void* dst, const void* src, size_t bytes, cudaStream_t st) {
    e->h2d_bytes += (int64_t)bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
}

static int gemm(const int8_t* W, int64_t M, int64_t K, const float* ws, int64_t rps, const int8_t* X,
                int64_t N, int64_t ldx, const float* xs, const int32_t* seg, const float* bias, float* Y,
                int64_t ldy, int32_t flags, cudaStream_t st, const float* add1 = nullptr, int64_t ld1 = 0,
                const float* add2 = nullptr, int64_t ld2 = 0, const GruEpi* gru = nullptr) {
    GemmArgs g{W, M, K, K, ws, rps, X, N, ldx, xs, seg, bias, Y, ldy, nullptr, flags | QNMT_GEMM_W_STATIC};
    if (gru) g.gru = *gru;
    g.add1 = add1;
    g.ld1 = ld1;
    g.add2 = add2;
    g.ld2 = ld2;
    return gemm_i8_launch(g, st);
}

// graph-captured steps: k_search_layout + k_gather_q as one launch (QNMT_LAYOUT_GATHER=0 for A/B runs)
static const int g_layout_gather = [] {
    const char* v = getenv("QNMT_LAYOUT_GATHER");
    return v ? atoi(v) : 1;
}();

// encoder steps with the per-column fused phase + quantize kernels (QNMT_ENC_FQ=0 for A/B runs)
static const int g_enc_fq = [] {
    const char* v = getenv("QNMT_ENC_FQ");
    return v ? atoi(v) : 1;
}();

// the two directions' products of an encoder step (same shape): one launch when the tcgen05
// path takes them, else one after the other
static int gemm_pair(const int8_t* W0, const float* ws0, const int8_t* W1, const float* ws1, int64_t M, int64_t K,
                     int64_t rps, const int8_t* X0, const int8_t* X1, int64_t N, int64_t ldx, const float* xs,
                     const int32_t* seg0, const int32_t* seg1, float* Y0, float* Y1, int64_t ldy, cudaStream_t st) {
    GemmArgs g0{W0, M, K, K, ws0, rps, X0, N, ldx, xs, seg0, nullptr, Y0, ldy, nullptr, QNMT_GEMM_W_STATIC};
    GemmArgs g1{W1, M, K, K, ws1, rps, X1, N, ldx, xs, seg1, nullptr, Y1, ldy, nullptr, QNMT_GEMM_W_STATIC};
    if (g_gemm_impl != 1 && (N > 8 || tl_ndev) && gemm_tc_dual_eligible(g0, g1)) return gemm_tc_dual_launch(g0, g1, st);
    const int rc = gemm_i8_launch(g0, st);
    return rc != QNMT_OK ? rc : gemm_i8_launch(g1, st);
}

static int encode_core_f32(qnmt_engine* e, const int32_t* ids_dev, const int32_t* len, int n, int Lmax, int64_t P,
                           const std::vector<int>& perm, float* states, float* att_proj, float* s0,
                           cudaStream_t st);

// ---------------------------------------------------------------------------
// encoder (layers.py:313-348) for n sentences in arbitrary order.
//   ids: device, concatenated; len/row: host.  Outputs at caller pointers.
// ---------------------------------------------------------------------------
static int encode_core(qnmt_engine* e, const int32_t* ids_dev, const int32_t* len, const int64_t* row,
                       int n, float* states, float* att_proj, float* s0, cudaStream_t st) {
    const qnmt_model* m = e->m;
    const int64_t E = m->E, H = m->H, A = m->A;
    int64_t P = 0;
    int Lmax = 0;
    for (int i = 0; i < n; ++i) {
        if (len[i] < 1) { set_error("cannot encode an empty sentence"); return QNMT_ERR_EMPTY; }
        if (len[i] > e->L) { set_error("sentence length %d exceeds engine max %d", len[i], e->L); return QNMT_ERR_CONFIG; }
        P = std::max<int64_t>(P, row[i] + len[i]);
        Lmax = std::max(Lmax, len[i]);
    }
    if (n > e->S || P > e->PMAX) { set_error("batch exceeds engine capacity"); return QNMT_ERR_CONFIG; }
    // sorted slots: longest first (stable) -> active sentences are a prefix
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return len[a] > len[b]; });
    std::vector<int32_t> rows((size_t)Lmax * 2 * n), orows((size_t)Lmax * 2 * n), pos_sent(P, 0);
    for (int t = 0; t < Lmax; ++t) {
        for (int k = 0; k < n; ++k) {
            int s = perm[k];
            if (len[s] <= t) continue;
            int64_t pf = row[s] + t, pb = row[s] + len[s] - 1 - t;
            rows[(size_t)t * 2 * n + 2 * k] = (int32_t)(2 * pf + 0);
            rows[(size_t)t * 2 * n + 2 * k + 1] = (int32_t)(2 * pb + 1);
            orows[(size_t)t * 2 * n + 2 * k] = (int32_t)(2 * pf + 1);      // fwd half = upper
            orows[(size_t)t * 2 * n + 2 * k + 1] = (int32_t)(2 * pb + 0);  // bwd half = lower
        }
    }
    for (int s = 0; s < n; ++s)
        for (int i = 0; i < len[s]; ++i) pos_sent[row[s] + i] = s;
    std::vector<int32_t> s0dst(n);   // slot of each sentence (inverse permutation)
    for (int k = 0; k < n; ++k) s0dst[perm[k]] = k;
    QNMT_CUDA(h2d(e, e->enc_rows, rows.data(), rows.size() * 4, st));
    QNMT_CUDA(h2d(e, e->enc_out_rows, orows.data(), orows.size() * 4, st));
    QNMT_CUDA(h2d(e, e->pos_sent, pos_sent.data(), (size_t)P * 4, st));
    QNMT_CUDA(h2d(e, e->s0_dst, s0dst.data(), (size_t)n * 4, st));

    if (m->fp32) return encode_core_f32(e, ids_dev, len, n, Lmax, P, perm, states, att_proj, s0, st);
    // input side for every position at once (per-position scales; one GEMM per direction)
    TRY(embed_gather_launch(m->src_embed, m->Vs, E, ids_dev, P, e->emb_src, E, e->err, st));
    TRY(quantize_launch(e->emb_src, P, E, E, e->iota, (int32_t)P, e->q_emb_src, E, e->sc_pos,
                        e->seg_bits, 1, e->err, st));
    for (int d = 0; d < 2; ++d) {
        const Cell& c = m->cell[d];
        TRY(gemm(c.wx, 3 * H, E, c.wx_s, H, e->q_emb_src, P, E, e->sc_pos, e->iota, c.bx,
                 e->gx_enc + d * 3 * H, 6 * H, 0, st));
    }
    if (n == 1 && g_enc1 && H % 16 == 0 && 2 * H <= 4096 && !e->prof_on) {
        // one sentence: the recurrence as one persistent kernel (persistent.cu)
        PeArgs pa{};
        pa.H = (int)H;
        pa.l = len[0];
        pa.gx = e->gx_enc;
        for (int d = 0; d < 2; ++d) {
            pa.uzr[d] = m->cell[d].uzr; pa.uzr_s[d] = m->cell[d].uzr_s;
            pa.uc[d] = m->cell[d].uc; pa.uc_s[d] = m->cell[d].uc_s;
        }
        pa.gh = e->gh2; pa.ghc = e->ghc2;
        pa.states = states + row[0] * 2 * H;
        pa.h2 = e->h2;
        pa.ctl = e->pk_ctl;
        pa.err = e->err;
        QNMT_CUDA(cudaMemsetAsync(e->pk_ctl, 0, PK_CTL_INTS * sizeof(int32_t), st));
        TRY(enc1_launch(pa, st));
    } else {
    QNMT_CUDA(cudaMemsetAsync(e->h2, 0, sizeof(float) * (size_t)n * 2 * H, st));
    // per-step max-abs bits (column c = its own segment): the gates kernel of step t
    // produces rh2's, the combine kernel of step t the next step's h2's
    QNMT_CUDA(cudaMemsetAsync(e->enc_qm, 0, sizeof(uint32_t) * (size_t)(Lmax + 1) * 4 * n, st));
    for (int t = 0; t < Lmax; ++t) {
        int na = 0;
        while (na < n && len[perm[na]] > t) ++na;
        int64_t N2 = 2 * (int64_t)na;
        const int32_t* gxr = e->enc_rows + (size_t)t * 2 * n;
        const int32_t* outr = e->enc_out_rows + (size_t)t * 2 * n;
        uint32_t* qm_h = e->enc_qm + (size_t)t * 4 * n;
        uint32_t* qm_rh = qm_h + 2 * n;
        uint32_t* qm_hn = qm_h + 4 * n;
        if (e->fq_ok && g_enc_fq) {
            // one CTA per (sentence, direction) column: GRU phase + the codes the next product reads
            if (t == 0)   // h = 0: codes 0, scale of a zero segment
                TRY(quantize_encode_launch(e->h2, N2, H, H, e->iota, e->q_h2, H, e->sc_h2, qm_h, 1, e->err, st));
            TRY(gemm_pair(m->cell[0].uzr, m->cell[0].uzr_s, m->cell[1].uzr, m->cell[1].uzr_s, 2 * H, H, H, e->q_h2,
                          e->q_h2 + H, na, 2 * H, e->sc_h2, e->even, e->odd, e->gh2, e->gh2 + 2 * H, 4 * H, st));
            TRY(enc_gates_q_launch(e->gx_enc, 3 * H, gxr, e->gh2, 2 * H, e->h2, H, N2, H, e->z2, e->q_rh2, e->sc_rh2,
                                   e->err, st));
            TRY(gemm_pair(m->cell[0].uc, m->cell[0].uc_s, m->cell[1].uc, m->cell[1].uc_s, H, H, H, e->q_rh2,
                          e->q_rh2 + H, na, 2 * H, e->sc_rh2, e->even, e->odd, e->ghc2, e->ghc2 + H, 2 * H, st));
            TRY(enc_combine_q_launch(e->gx_enc, 3 * H, gxr, e->ghc2, H, e->z2, e->h2, H, N2, H, states, H, outr,
                                     e->q_h2, e->sc_h2, e->err, st));
            continue;
        }
        TRY(quantize_encode_launch(e->h2, N2, H, H, e->iota, e->q_h2, H, e->sc_h2, qm_h, 1, e->err, st));
        TRY(gemm_pair(m->cell[0].uzr, m->cell[0].uzr_s, m->cell[1].uzr, m->cell[1].uzr_s, 2 * H, H, H, e->q_h2,
                      e->q_h2 + H, na, 2 * H, e->sc_h2, e->even, e->odd, e->gh2, e->gh2 + 2 * H, 4 * H, st));
        TRY(gru_gates_launch(e->gx_enc, 3 * H, gxr, e->gh2, 2 * H, e->h2, H, N2, H, e->z2, e->rh2, e->err, st,
                             qm_rh, nullptr));
        TRY(quantize_encode_launch(e->rh2, N2, H, H, e->iota, e->q_rh2, H, e->sc_rh2, qm_rh, 1, e->err, st));
        TRY(gemm_pair(m->cell[0].uc, m->cell[0].uc_s, m->cell[1].uc, m->cell[1].uc_s, H, H, H, e->q_rh2,
                      e->q_rh2 + H, na, 2 * H, e->sc_rh2, e->even, e->odd, e->ghc2, e->ghc2 + H, 2 * H, st));
        TRY(gru_combine_launch(e->gx_enc, 3 * H, gxr, e->ghc2, H, e->z2, e->h2, H, N2, H, e->h2, H,
                               states, H, outr, e->err, st, qm_hn, nullptr));
    }
    }   // per-step kernels
    // att_proj = enc_proj(states) with one scale per sentence over [2H, l] (layers.py:343)
    TRY(quantize_launch(states, P, 2 * H, 2 * H, e->pos_sent, n, e->q_states, 2 * H, e->sc_sent,
                        e->seg_bits, 1, e->err, st));
    TRY(gemm(m->w_enc, A, 2 * H, m->w_enc_s, A, e->q_states, P, 2 * H, e->sc_sent, e->pos_sent, m->b_enc,
             att_proj, A, 0, st));
    // s0 = tanh(W_s0 . q(bwd[:, 0]) + b) (layers.py:347); bwd final states are odd rows of h2
    if (m->s0_mode == 1) {
        QNMT_CUDA(cudaMemsetAsync(s0, 0, sizeof(float) * (size_t)n * H, st));
    } else {
        TRY(quantize_launch(e->h2, 2 * (int64_t)n, H, H, e->iota, 2 * n, e->q_h2, H, e->sc_h2,
                            e->seg_bits, 1, e->err, st));
        TRY(gemm(m->s0_w, H, H, m->s0_s, H, e->q_h2 + H, n, 2 * H, e->sc_h2, e->odd, m->s0_b,
                 e->s0tmp, H, 0, st));
        // tanh, then rows back to the caller's sentence order: s0[s] = s0tmp[slot_of[s]]
        TRY(tanh_launch(e->s0tmp, n, H, H, e->s0tmp, H, e->err, st));
        TRY(gather_rows_launch(e->s0tmp, nullptr, e->s0_dst, n, H, s0, nullptr, st));
    }
    return QNMT_OK;
}

// ---------------------------------------------------------------------------
// one decoder step (layers.py:356-384) for N columns; logits [N][V] out.
// ---------------------------------------------------------------------------
struct StepIO {
    int64_t N;
    int nseg;
    const int32_t* col_sent;
    const int32_t* y;
    const float* s;
    const float* sp;
    const float* states;
    const float* att_proj;
    const int64_t* sent_row;
    const int32_t* sent_len;
    int max_len;
    float* s_int;
    float* s_new;
    float* logits;
    float* alpha;
    int64_t lda;
    const int32_t* sent_col_off;   // [nseg] first column of each sentence (columns grouped by sentence)
    const int32_t* sent_ncols;     // [nseg] live columns of each sentence
    const float* att_minmax;       // [nseg][2][A] column extrema of att_proj (nullable)
    const float* att_exp;          // fl32(e^(2 att_proj)) rows (nullable: two-MUFU scorer)
    int max_cols;                  // bound on columns per sentence (fused quantize smem)
    bool codes_ready;              // q_s (and q_q for the previous-state query) hold this step's state codes
    bool fuse_vocab;               // skip the vocab GEMM: the caller runs cands_launch (vocab_topk.cu)
};

// ---------------------------------------------------------------------------
// Device-clock stamps inside captured decode steps (for live per-kernel timing
// in graph mode, where host events cannot bracket single kernels).  Row t of
// e->stamps holds %globaltimer at ST_* points of step t, the live column count
// and the sum of source lengths of live sentences (algorithmic-work accounting).
// ---------------------------------------------------------------------------
enum { ST_STEP0 = 0, ST_ATT0, ST_ATT1, ST_TOPK0, ST_TOPK1, ST_VOC0, ST_VOC1, ST_STEP1, ST_N, ST_SUML, ST_SUMPL,
       ST_COLS };
static_assert(ST_COLS == QNMT_STAMP_COLS, "stamp row layout");

__global__ void k_stamp(long long* stamps, const int32_t* step_dev, int slot, int slot2, const int32_t* n_dev,
                        const int32_t* P, const int32_t* len, int n_sent) {
    pdl_entry();
    const int t = *step_dev;
    long long* row = stamps + (int64_t)t * ST_COLS;
    if (slot == ST_ATT0) {   // also record the work descriptors of this step
        __shared__ int red[2][32];
        int sl = 0, spl = 0;
        for (int s = threadIdx.x; s < n_sent; s += blockDim.x) {
            sl += P[s] > 0 ? len[s] : 0;
            spl += P[s] * len[s];
        }
        sl = warp_sum(sl);
        spl = warp_sum(spl);
        if ((threadIdx.x & 31) == 0) {
            red[0][threadIdx.x >> 5] = sl;
            red[1][threadIdx.x >> 5] = spl;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long tot = 0, totp = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                tot += red[0][w];
                totp += red[1][w];
            }
            row[ST_SUML] = tot;
            row[ST_SUMPL] = totp;
            row[ST_N] = *n_dev;
        }
    }
    if (threadIdx.x == 0) {
        long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        row[slot] = g;
        if (slot2 >= 0) row[slot2] = g;
    }
}

static int stamp(qnmt_engine* e, int slot, const StepIO& io, cudaStream_t st, int slot2 = -1) {
    if (!e->stamp_on || !tl_ndev || !e->stamps) return QNMT_OK;   // graph-captured steps only
    QNMT_LAUNCH(k_stamp, 1, 256, 0, st, e->stamps, e->d_step, slot, slot2, tl_ndev, io.sent_ncols, io.sent_len, io.nseg);
    QNMT_CHECK_LAUNCH("k_stamp");
    return QNMT_OK;
}

// one GRU cell (layers.py:170-181) over the step's columns; h_out's codes -> q_out / sc_out.
// fq: gates and combine are the per-sentence fused op+quantize kernels (fused_q.cu);
// otherwise elementwise kernels followed by the two-pass quantization.
// Optional stacking (see qnmt_engine::w2x): xs = {W, per-row scales, bias, rows, out, ld} replaces the
// cell's own W_x GEMM; gh_pre (ld ldgh_pre) is a U_zr product already computed by a stacked GEMM.
// GRU gates / combine in the tcgen05 epilogues (qnmt_set_gate_epi; QNMT_GATE_EPI=0/1 for A/B runs).
// Off by default: measured slower than the separate fused kernels on the cfg5 decode (the fp64
// sigmoid / tanh chains run on the 8 epilogue warps of a CTA that owns its SM; K3g).
int g_gate_epi = [] {
    const char* v = getenv("QNMT_GATE_EPI");
    return v ? atoi(v) != 0 : 0;
}();

struct XSide {
    const int8_t* w;
    const float* ws;
    const float* b;
    int64_t rows;
    float* out;
    int64_t ld;
};

static int gru_cell(qnmt_engine* e, const Cell& c, const StepIO& io, const int8_t* qx, const float* sx,
                    const int8_t* qh, const float* sh, const float* h, float* h_out, int8_t* q_out, float* sc_out,
                    cudaStream_t st, const XSide* xs = nullptr, const float* gh_pre = nullptr,
                    int64_t ldgh_pre = 0, int cell_slot = 0) {
    const int64_t H = e->m->H, N = io.N;
    // GRU elementwise phases inside the tcgen05 epilogues (N > 8: those GEMMs take the tcgen05 path)
    const bool ge = e->gate_epi && g_gate_epi && g_gemm_impl != 1 && N > 8;
    uint32_t* mx_rh = e->gmax + (size_t)(2 * cell_slot) * e->S;
    uint32_t* mx_h = e->gmax + (size_t)(2 * cell_slot + 1) * e->S;
    const int32_t* seg = io.col_sent;
    const int ns = io.nseg;
    float* gx = xs ? xs->out : e->gx;
    const int64_t ldgx = xs ? xs->ld : 3 * H;
    const float* gh = gh_pre ? gh_pre : e->gh;
    const int64_t ldgh = gh_pre ? ldgh_pre : 2 * H;
    prof_mark(e, PG_GEMM, st, 2.0 * N * (3 * H * c.in + 2 * H * H), 3.0 * H * c.in + 2.0 * H * H);
    if (ge) {
        // U_zr h first; the W_x GEMM's epilogue then computes z and r*h from both products
        if (!gh_pre) TRY(gemm(c.uzr, 2 * H, H, c.uzr_s, H, qh, N, H, sh, seg, nullptr, e->gh, 2 * H, 0, st));
        GruEpi ga;
        ga.mode = 1; ga.H = H; ga.g = gh; ga.ldg = ldgh; ga.h = h; ga.ldh = H; ga.z = e->z; ga.out = e->rh;
        ga.ldo = H; ga.segmax = mx_rh; ga.err_flag = e->err;
        if (xs)
            TRY(gemm(xs->w, xs->rows, c.in, xs->ws, 1, qx, N, c.in, sx, seg, xs->b, gx, ldgx, 0, st, nullptr, 0,
                     nullptr, 0, &ga));
        else
            TRY(gemm(c.wx, 3 * H, c.in, c.wx_s, H, qx, N, c.in, sx, seg, c.bx, gx, ldgx, 0, st, nullptr, 0, nullptr,
                     0, &ga));
        prof_mark(e, PG_QUANT, st);
        TRY(quantize_encode_launch(e->rh, N, H, H, seg, e->q_rh, H, e->sc_rh, mx_rh, 1, e->err, st));
        prof_mark(e, PG_GEMM, st, 2.0 * N * H * H, (double)H * H);
        GruEpi gc;
        gc.mode = 2; gc.H = H; gc.g = gx + 2 * H; gc.ldg = ldgx; gc.h = h; gc.ldh = H; gc.z = e->z; gc.out = h_out;
        gc.ldo = H; gc.segmax = mx_h; gc.err_flag = e->err;
        TRY(gemm(c.uc, H, H, c.uc_s, H, e->q_rh, N, H, e->sc_rh, seg, nullptr, nullptr, H, 0, st, nullptr, 0, nullptr,
                 0, &gc));
        prof_mark(e, PG_QUANT, st);
        TRY(quantize_encode_launch(h_out, N, H, H, seg, q_out, H, sc_out, mx_h, 1, e->err, st));
        return QNMT_OK;
    }
    if (xs)
        TRY(gemm(xs->w, xs->rows, c.in, xs->ws, 1, qx, N, c.in, sx, seg, xs->b, gx, ldgx, 0, st));
    else
        TRY(gemm(c.wx, 3 * H, c.in, c.wx_s, H, qx, N, c.in, sx, seg, c.bx, gx, ldgx, 0, st));
    if (!gh_pre) TRY(gemm(c.uzr, 2 * H, H, c.uzr_s, H, qh, N, H, sh, seg, nullptr, e->gh, 2 * H, 0, st));
    prof_mark(e, PG_GRU, st);
    if (e->fq_ok) {
        TRY(gates_q_launch(gx, ldgx, gh, ldgh, h, H, H, io.sent_col_off, io.sent_ncols, ns, io.max_cols,
                           e->z, e->q_rh, e->sc_rh, e->err, st));
    } else {
        TRY(gru_gates_launch(gx, ldgx, nullptr, gh, ldgh, h, H, N, H, e->z, e->rh, e->err, st));
        TRY(quantize_launch(e->rh, N, H, H, seg, ns, e->q_rh, H, e->sc_rh, e->seg_bits, 1, e->err, st));
    }
    prof_mark(e, PG_GEMM, st, 2.0 * N * H * H, (double)H * H);
    TRY(gemm(c.uc, H, H, c.uc_s, H, e->q_rh, N, H, e->sc_rh, seg, nullptr, e->ghc, H, 0, st));
    prof_mark(e, PG_GRU, st);
    if (e->fq_ok) {
        TRY(combine_q_launch(gx + 2 * H, ldgx, e->ghc, H, e->z, h, H, H, io.sent_col_off, io.sent_ncols, ns,
                             io.max_cols, h_out, H, q_out, sc_out, e->err, st));
    } else {
        TRY(gru_combine_launch(gx, ldgx, nullptr, e->ghc, H, e->z, h, H, N, H, h_out, H, nullptr, 0,
                               nullptr, e->err, st));
        TRY(quantize_launch(h_out, N, H, H, seg, ns, q_out, H, sc_out, e->seg_bits, 1, e->err, st));
    }
    return QNMT_OK;
}

// ---------------------------------------------------------------------------
// fp32 precision path (LinearOp's float branch,
// layers.py:138-145): the same network with every LinearOp an f32 product
// (gemm_f32.cu, fp64-evaluated and rounded once) and no quantization.
// ---------------------------------------------------------------------------
static inline const float* F(const int8_t* p) { return reinterpret_cast<const float*>(p); }

static int gemm32(const int8_t* W, int64_t M, int64_t K, const float* X, int64_t N, int64_t ldx, const float* bias,
                  float* Y, int64_t ldy, int32_t flags, cudaStream_t st) {
    return gemm_f32_launch(F(W), M, K, K, X, N, ldx, bias, Y, ldy, flags, st);
}

static int encode_core_f32(qnmt_engine* e, const int32_t* ids_dev, const int32_t* len, int n, int Lmax, int64_t P,
                           const std::vector<int>& perm, float* states, float* att_proj, float* s0,
                           cudaStream_t st) {
    const qnmt_model* m = e->m;
    const int64_t E = m->E, H = m->H, A = m->A;
    TRY(embed_gather_launch(m->src_embed, m->Vs, E, ids_dev, P, e->emb_src, E, e->err, st));
    for (int d = 0; d < 2; ++d) {
        const Cell& c = m->cell[d];
        TRY(gemm32(c.wx, 3 * H, E, e->emb_src, P, E, c.bx, e->gx_enc + d * 3 * H, 6 * H, 0, st));
    }
    QNMT_CUDA(cudaMemsetAsync(e->h2, 0, sizeof(float) * (size_t)n * 2 * H, st));
    for (int t = 0; t < Lmax; ++t) {
        int na = 0;
        while (na < n && len[perm[na]] > t) ++na;
        const int64_t N2 = 2 * (int64_t)na;
        const int32_t* gxr = e->enc_rows + (size_t)t * 2 * n;
        const int32_t* outr = e->enc_out_rows + (size_t)t * 2 * n;
        for (int d = 0; d < 2; ++d)   // rows of direction d: h2 + d*H with stride 2H
            TRY(gemm32(m->cell[d].uzr, 2 * H, H, e->h2 + d * H, na, 2 * H, nullptr, e->gh2 + d * 2 * H, 4 * H, 0, st));
        TRY(gru_gates_launch(e->gx_enc, 3 * H, gxr, e->gh2, 2 * H, e->h2, H, N2, H, e->z2, e->rh2, e->err, st));
        for (int d = 0; d < 2; ++d)
            TRY(gemm32(m->cell[d].uc, H, H, e->rh2 + d * H, na, 2 * H, nullptr, e->ghc2 + d * H, 2 * H, 0, st));
        TRY(gru_combine_launch(e->gx_enc, 3 * H, gxr, e->ghc2, H, e->z2, e->h2, H, N2, H, e->h2, H, states, H, outr,
                               e->err, st));
    }
    TRY(gemm32(m->w_enc, A, 2 * H, states, P, 2 * H, m->b_enc, att_proj, A, 0, st));   // layers.py:343
    if (m->s0_mode == 1) {
        QNMT_CUDA(cudaMemsetAsync(s0, 0, sizeof(float) * (size_t)n * H, st));
    } else {   // s0 = tanh(W_s0 bwd[:, 0] + b): bwd final states are the odd rows of h2 (layers.py:347)
        TRY(gemm32(m->s0_w, H, H, e->h2 + H, n, 2 * H, m->s0_b, e->s0tmp, H, 0, st));
        TRY(tanh_launch(e->s0tmp, n, H, H, e->s0tmp, H, e->err, st));
        TRY(gather_rows_launch(e->s0tmp, nullptr, e->s0_dst, n, H, s0, nullptr, st));
    }
    return QNMT_OK;
}

static int gru_cell_f32(qnmt_engine* e, const Cell& c, const StepIO& io, const float* x, const float* h, float* h_out,
                        cudaStream_t st) {
    const int64_t H = e->m->H, N = io.N;
    TRY(gemm32(c.wx, 3 * H, c.in, x, N, c.in, c.bx, e->gx, 3 * H, 0, st));
    TRY(gemm32(c.uzr, 2 * H, H, h, N, H, nullptr, e->gh, 2 * H, 0, st));
    TRY(gru_gates_launch(e->gx, 3 * H, nullptr, e->gh, 2 * H, h, H, N, H, e->z, e->rh, e->err, st));
    TRY(gemm32(c.uc, H, H, e->rh, N, H, nullptr, e->ghc, H, 0, st));
    return gru_combine_launch(e->gx, 3 * H, nullptr, e->ghc, H, e->z, h, H, N, H, h_out, H, nullptr, 0, nullptr,
                              e->err, st);
}

static int step_core_f32(qnmt_engine* e, const StepIO& io, cudaStream_t st) {
    const qnmt_model* m = e->m;
    const int64_t N = io.N, E = m->E, H = m->H, A = m->A, R = m->R, V = m->Vt;
    TRY(embed_gather_launch(m->tgt_embed, V, E, io.y, N, e->emb, E, e->err, st));
    TRY(gru_cell_f32(e, m->cell[2], io, e->emb, io.s, io.s_int, st));                  // s' (layers.py:372)
    const float* query = m->aq == 1 ? io.sp : io.s_int;                                  // layers.py:373
    TRY(gemm32(m->u_att, A, H, query, N, H, nullptr, e->u, A, 0, st));
    TRY(attention_f32_launch(e->u, A, N, io.sent_col_off, io.sent_ncols, io.nseg, io.att_proj, io.states, io.sent_row,
                             io.sent_len, io.max_len, A, 2 * H, F(m->v), e->ctx, 2 * H, io.alpha, io.lda,
                             e->att_scratch, e->err, st));
    TRY(gru_cell_f32(e, m->cell[3], io, e->ctx, io.s_int, io.s_new, st));                // s (layers.py:375)
    // readout = tanh(((W_s s + b_r) + W_e emb) + W_c ctx), logits = W_v readout + b_v (layers.py:255-266)
    TRY(gemm32(m->w_state, R, H, io.s_new, N, H, m->b_r, e->ro, R, 0, st));
    TRY(gemm32(m->w_embed, R, E, e->emb, N, E, nullptr, e->ro, R, QNMT_GEMM_ACCUMULATE, st));
    TRY(gemm32(m->w_ctx, R, 2 * H, e->ctx, N, 2 * H, nullptr, e->ro, R, QNMT_GEMM_ACCUMULATE, st));
    TRY(tanh_launch(e->ro, N, R, R, e->ro, R, e->err, st));
    return gemm32(m->w_vocab, V, R, e->ro, N, R, m->b_vocab, io.logits, V, 0, st);
}

static int step_core(qnmt_engine* e, const StepIO& io, cudaStream_t st) {
    const qnmt_model* m = e->m;
    if (m->fp32) return io.N > 0 ? step_core_f32(e, io, st) : QNMT_OK;
    const int64_t N = io.N, E = m->E, H = m->H, A = m->A, R = m->R, V = m->Vt;
    const int32_t* seg = io.col_sent;
    const int ns = io.nseg;
    if (N <= 0) return QNMT_OK;
    const bool fq = e->fq_ok;
    // codes of the state (and, for the previous-state query, of s') when not produced by gather_q
    if (!io.codes_ready) {
        prof_mark(e, PG_QUANT, st);
        TRY(quantize_launch(io.s, N, H, H, seg, ns, e->q_s, H, e->sc_s, e->seg_bits, 1, e->err, st));
        if (m->aq == 1) TRY(quantize_launch(io.sp, N, H, H, seg, ns, e->q_q, H, e->sc_q, e->seg_bits, 1, e->err, st));
    }
    prof_mark(e, PG_EMBED, st);
    if (fq) {
        TRY(embed_q_launch(m->tgt_embed, V, E, io.y, io.sent_col_off, io.sent_ncols, ns, io.max_cols, e->q_emb,
                           e->sc_emb, e->err, st, e->gate_epi ? e->gmax : nullptr, e->S));
    } else {
        TRY(embed_gather_launch(m->tgt_embed, V, E, io.y, N, e->emb, E, e->err, st));
        TRY(quantize_launch(e->emb, N, E, E, seg, ns, e->q_emb, E, e->sc_emb, e->seg_bits, 1, e->err, st));
    }
    // stacked GEMMs (fq + tcgen05 only): W_e e / W_c c ride on the cells' W_x GEMMs, U_att on U_zr
    const bool stk = fq && e->stack_ok && g_gemm_impl != 1;
    const bool stk_u = stk && e->stack_u;
    const int64_t LX = 3 * H + R, LU = A + 2 * H;
    const XSide xs2{e->w2x, e->w2x_s, e->b2x, LX, e->gxr, LX};
    const XSide xs3{e->w3x, e->w3x_s, e->b3x, LX, e->gxq, LX};
    // s' = GRU_r(emb, s) (layers.py:372); the query (layers.py:373) is s' or the previous s'
    int8_t* q_si = m->aq == 1 ? e->q_si : e->q_q;
    float* sc_si = m->aq == 1 ? e->sc_si : e->sc_q;
    TRY(gru_cell(e, m->cell[2], io, e->q_emb, e->sc_emb, e->q_s, e->sc_s, io.s, io.s_int, q_si, sc_si, st,
                 stk ? &xs2 : nullptr, nullptr, 0, 0));
    prof_mark(e, PG_GEMM, st, 2.0 * N * A * H, (double)A * H);
    const float* u = e->u;
    int64_t ldu = A;
    if (stk_u) {
        TRY(gemm(e->wuq, LU, H, e->wuq_s, 1, e->q_q, N, H, e->sc_q, seg, nullptr, e->uq, LU, 0, st));
        u = e->uq;
        ldu = LU;
    } else {
        TRY(gemm(m->u_att, A, H, m->u_att_s, A, e->q_q, N, H, e->sc_q, seg, nullptr, e->u, A, 0, st));
    }
    prof_mark(e, PG_ATT, st);
    TRY(stamp(e, ST_ATT0, io, st));
    // (ctx_max is zeroed by the attention scale kernel)
    TRY(attention_launch(u, ldu, N, io.sent_col_off, io.sent_ncols, io.nseg, io.att_proj, io.att_minmax, io.states,
                         io.sent_row, io.sent_len, io.max_len, A, 2 * H, m->v, m->v_s, e->ctx, 2 * H,
                         io.alpha, io.lda, e->att_scratch, e->err, st, fq ? e->ctx_max : nullptr, io.max_cols,
                         io.att_exp));
    TRY(stamp(e, ST_ATT1, io, st));
    prof_mark(e, PG_QUANT, st);
    if (fq) {
        TRY(quantize_encode_launch(e->ctx, N, 2 * H, 2 * H, seg, e->q_ctx, 2 * H, e->sc_ctx, e->ctx_max, 1, e->err,
                                   st));
    } else {
        TRY(quantize_launch(e->ctx, N, 2 * H, 2 * H, seg, ns, e->q_ctx, 2 * H, e->sc_ctx, e->seg_bits, 1, e->err,
                            st));
    }
    // s = GRU_q(ctx, s')                                        (layers.py:375)
    TRY(gru_cell(e, m->cell[3], io, e->q_ctx, e->sc_ctx, q_si, sc_si, io.s_int, io.s_new, e->q_sn, e->sc_sn, st,
                 stk ? &xs3 : nullptr, stk_u ? e->uq + A : nullptr, LU, 1));
    // readout = tanh(((W_s s + b_r) + W_e emb) + W_c ctx)       (layers.py:255-265)
    prof_mark(e, PG_GEMM, st, 2.0 * N * R * (H + E + 2 * H), (double)R * (H + E + 2 * H));
    if (stk) {   // W_e emb and W_c ctx were computed with the cells' input GEMMs; added in tanh_q below
        TRY(gemm(m->w_state, R, H, m->w_state_s, R, e->q_sn, N, H, e->sc_sn, seg, m->b_r, e->ro, R, 0, st));
    } else {
        TRY(gemm(m->w_state, R, H, m->w_state_s, R, e->q_sn, N, H, e->sc_sn, seg, m->b_r, e->ro, R, 0, st));
        TRY(gemm(m->w_embed, R, E, m->w_embed_s, R, e->q_emb, N, E, e->sc_emb, seg, nullptr, e->ro, R,
                 QNMT_GEMM_ACCUMULATE, st));
        TRY(gemm(m->w_ctx, R, 2 * H, m->w_ctx_s, R, e->q_ctx, N, 2 * H, e->sc_ctx, seg, nullptr, e->ro, R,
                 QNMT_GEMM_ACCUMULATE, st));
    }
    prof_mark(e, PG_MISC, st);
    if (fq) {
        TRY(tanh_q_launch(e->ro, R, R, io.sent_col_off, io.sent_ncols, ns, io.max_cols, e->q_ro, e->sc_ro, e->err,
                          st, stk ? e->gxr + 3 * H : nullptr, LX, stk ? e->gxq + 3 * H : nullptr, LX));
    } else {
        TRY(tanh_launch(e->ro, N, R, R, e->ro, R, e->err, st));
        TRY(quantize_launch(e->ro, N, R, R, seg, ns, e->q_ro, R, e->sc_ro, e->seg_bits, 1, e->err, st));
    }
    if (io.fuse_vocab) return QNMT_OK;
    prof_mark(e, PG_GEMM_VOCAB, st, 2.0 * N * V * R, (double)V * R + (double)N * R + 4.0 * N * V);
    TRY(stamp(e, ST_VOC0, io, st));
    TRY(gemm(m->w_vocab, V, R, m->w_vocab_s, V, e->q_ro, N, R, e->sc_ro, seg, m->b_vocab, io.logits, V,
             0, st));
    TRY(stamp(e, ST_VOC1, io, st));
    return QNMT_OK;
}

// next-step state columns by parent (decoder.py:131-140) and, with fq, their codes
// (srch: the engine holding the search state -- e itself, or an ensemble's lead engine)
static int gather_next(qnmt_engine* e, int cur, int64_t N2, int n, int beam, cudaStream_t st,
                       const qnmt_engine* srch = nullptr) {
    const qnmt_model* m = e->m;
    const int64_t H = m->H;
    if (!srch) srch = e;
    if (e->fq_ok)
        return gather_q_launch(e->s_new, m->aq == 1 ? e->s_int : nullptr, srch->parent_col, H, srch->col_off, srch->P,
                               n, beam, e->st_s[cur ^ 1], e->st_sp[cur ^ 1], e->q_s, e->sc_s,
                               m->aq == 1 ? e->q_q : nullptr, m->aq == 1 ? e->sc_q : nullptr, e->err, st);
    return gather_rows_launch(e->s_new, e->s_int, srch->parent_col, N2, H, e->st_s[cur ^ 1], e->st_sp[cur ^ 1], st);
}

static bool vocab_fusable(const qnmt_engine* e, int k) {
    const qnmt_model* m = e->m;
    return !m->fp32 && g_vocab_fused && g_gemm_impl != 1 && vocab_topk_eligible(m->R, m->R, m->R, e->q_ro, m->w_vocab, k);
}

// beam candidates of the step: fused vocab projection + statistics + merge, or
// the plain vocab GEMM (inside step_core) followed by the candidate kernel
static int cands_launch(qnmt_engine* e, const StepIO& io, const double* live, int k, cudaStream_t st) {
    const qnmt_model* m = e->m;
    const int64_t N = io.N, V = m->Vt, R = m->R;
    if (io.fuse_vocab) {
        VocabTopk p{e->q_ro, N, R, e->sc_ro, io.col_sent, m->w_vocab, V, R, R, m->w_vocab_s, V, m->b_vocab,
                    live, k, e->vocab_part, e->cand_score, e->cand_tok, e->err};
        prof_mark(e, PG_GEMM_VOCAB, st, 2.0 * N * V * R, (double)V * R + (double)N * R);
        TRY(stamp(e, ST_VOC0, io, st));
        TRY(vocab_stats_launch(p, st));
        TRY(stamp(e, ST_VOC1, io, st, ST_TOPK0));
        prof_mark(e, PG_TOPK, st);
        TRY(vocab_merge_launch(p, st));
        return stamp(e, ST_TOPK1, io, st);
    }
    TRY(stamp(e, ST_TOPK0, io, st));
    prof_mark(e, PG_TOPK, st, 0, 4.0 * N * V);
    TRY(topk_launch(io.logits, N, V, V, live, k, e->cand_score, e->cand_tok, e->err, st));
    return stamp(e, ST_TOPK1, io, st);
}

static int grow_history(qnmt_engine* e, int steps) {
    if (steps <= e->hist_steps) return QNMT_OK;
    // captured step graphs point into the old history block
    for (auto& kv : e->graphs) {
        cudaGraphExecDestroy(kv.second.first);
        cudaGraphExecDestroy(kv.second.second);
    }
    e->graphs.clear();
    std::unique_lock<std::shared_mutex> gate(g_capture_gate);   // cudaFree synchronises the device
    if (e->hblock) cudaFree(e->hblock);
    size_t S = e->S, B = e->B, T = steps;
    size_t fin_cap = (T + 1) * B;
    size_t res_w = T + 3;   // packed result row: len, logp (2 words), up to T tokens
    size_t bytes = S * fin_cap * (8 + 4 + 4 + 4) + 2 * S * T * B * 4 + (T + 1) * ST_COLS * 8 +
                   S * res_w * 4 + S * 2 * (T + 2) * 4 + 8192;
    QNMT_CUDA(cudaMalloc(&e->hblock, bytes));
    if (e->res_host) cudaFreeHost(e->res_host);
    e->res_host = nullptr;
    QNMT_CUDA(cudaMallocHost(&e->res_host, S * res_w * 4));
    e->hblock_bytes = bytes;
    Arena a{e->hblock, bytes, 0};
    e->stamps = a.take<long long>((T + 1) * ST_COLS);
    e->fin_score = a.take<double>(S * fin_cap);
    e->fin_step = a.take<int32_t>(S * fin_cap);
    e->fin_slot = a.take<int32_t>(S * fin_cap);
    e->fin_eos = a.take<int32_t>(S * fin_cap);
    e->hist_tok = a.take<int32_t>(S * T * B);
    e->hist_par = a.take<int32_t>(S * T * B);
    e->res_dev = a.take<int32_t>(S * res_w);
    e->fin_scratch = a.take<int32_t>(S * 2 * (T + 2));
    e->hist_steps = steps;
    return QNMT_OK;
}

}  // namespace qnmt

using namespace qnmt;

extern "C" {

int qnmt_model_create(const int32_t* dims, const void* const* t, int32_t nt, qnmt_model** out) {
    if (nt != QNMT_T_COUNT) { set_error("expected %d tensors, got %d", QNMT_T_COUNT, nt); return QNMT_ERR_CONFIG; }
    qnmt_model* m = new qnmt_model();
    m->Vs = dims[0]; m->Vt = dims[1]; m->E = dims[2]; m->H = dims[3]; m->A = dims[4]; m->R = dims[5];
    m->s0_mode = dims[6]; m->aq = dims[7];
    m->src_embed = (const float*)t[QNMT_T_SRC_EMBED];
    m->tgt_embed = (const float*)t[QNMT_T_TGT_EMBED];
    for (int c = 0; c < 4; ++c) {
        int b = 2 + 7 * c;
        Cell& k = m->cell[c];
        k.wx = (const int8_t*)t[b + QNMT_T_CELL_WX];
        k.wx_s = (const float*)t[b + QNMT_T_CELL_WX_SCALES];
        k.bx = (const float*)t[b + QNMT_T_CELL_BX];
        k.uzr = (const int8_t*)t[b + QNMT_T_CELL_UZR];
        k.uzr_s = (const float*)t[b + QNMT_T_CELL_UZR_SCALES];
        k.uc = (const int8_t*)t[b + QNMT_T_CELL_UC];
        k.uc_s = (const float*)t[b + QNMT_T_CELL_UC_SCALE];
        k.in = (c == 3) ? 2 * m->H : m->E;
    }
    m->w_enc = (const int8_t*)t[QNMT_T_ATT_WENC]; m->w_enc_s = (const float*)t[QNMT_T_ATT_WENC_SCALE];
    m->b_enc = (const float*)t[QNMT_T_ATT_BENC];
    m->u_att = (const int8_t*)t[QNMT_T_ATT_USTATE]; m->u_att_s = (const float*)t[QNMT_T_ATT_USTATE_SCALE];
    m->v = (const int8_t*)t[QNMT_T_ATT_V]; m->v_s = (const float*)t[QNMT_T_ATT_V_SCALE];
    m->w_state = (const int8_t*)t[QNMT_T_OUT_WSTATE]; m->w_state_s = (const float*)t[QNMT_T_OUT_WSTATE_SCALE];
    m->b_r = (const float*)t[QNMT_T_OUT_BREADOUT];
    m->w_embed = (const int8_t*)t[QNMT_T_OUT_WEMBED]; m->w_embed_s = (const float*)t[QNMT_T_OUT_WEMBED_SCALE];
    m->w_ctx = (const int8_t*)t[QNMT_T_OUT_WCTX]; m->w_ctx_s = (const float*)t[QNMT_T_OUT_WCTX_SCALE];
    m->w_vocab = (const int8_t*)t[QNMT_T_OUT_WVOCAB]; m->w_vocab_s = (const float*)t[QNMT_T_OUT_WVOCAB_SCALE];
    m->b_vocab = (const float*)t[QNMT_T_OUT_BVOCAB];
    m->s0_w = (const int8_t*)t[QNMT_T_S0_W]; m->s0_s = (const float*)t[QNMT_T_S0_W_SCALE];
    m->s0_b = (const float*)t[QNMT_T_S0_B];
    *out = m;
    return QNMT_OK;
}

int qnmt_model_create_f32(const int32_t* dims, const void* const* t, int32_t nt, qnmt_model** out) {
    TRY(qnmt_model_create(dims, t, nt, out));
    (*out)->fp32 = 1;
    return QNMT_OK;
}

int qnmt_model_destroy(qnmt_model* m) {
    delete m;
    return QNMT_OK;
}

int qnmt_engine_create(const qnmt_model* m, int32_t max_sentences, int32_t max_src_len,
                       int32_t max_beam, qnmt_engine** out) {
    if (max_sentences < 1 || max_sentences > 1024 || max_src_len < 1 || max_beam < 1 || max_beam > 16) {
        set_error("engine limits: 1<=sentences<=1024, len>=1, 1<=beam<=16");
        return QNMT_ERR_CONFIG;
    }
    qnmt_engine* e = new qnmt_engine();
    e->m = m;
    e->S = max_sentences; e->L = max_src_len; e->B = max_beam;
    const size_t S = e->S, L = e->L, B = e->B;
    const size_t E = m->E, H = m->H, A = m->A, R = m->R, V = m->Vt;
    const size_t N = S * B, P = S * L;
    e->NMAX = N; e->PMAX = P;
    const size_t idx = std::max(P, std::max(2 * S, N));
    size_t bytes = 0;
    {
        const char* cv = getenv("QNMT_CANARY");
        e->guard = cv && cv[0] == '1';
    }
    // size pass then carve pass
    for (int pass = 0; pass < 2; ++pass) {
        Arena a{e->block, pass ? e->block_bytes : 0, 0, e->guard, pass ? &e->guards : nullptr};
        e->err = a.take<int32_t>(4);
        e->seg_bits = a.take<uint32_t>(idx);
        e->iota = a.take<int32_t>(idx);
        e->even = a.take<int32_t>(S);
        e->odd = a.take<int32_t>(S);
        e->src_ids = a.take<int32_t>(P);
        e->emb_src = a.take<float>(P * E);
        e->q_emb_src = a.take<int8_t>(P * E);
        e->sc_pos = a.take<float>(P);
        e->gx_enc = a.take<float>(P * 6 * H);
        e->h2 = a.take<float>(2 * S * H);
        e->q_h2 = a.take<int8_t>(2 * S * H);
        e->sc_h2 = a.take<float>(2 * S);
        e->gh2 = a.take<float>(4 * S * H);
        e->z2 = a.take<float>(2 * S * H);
        e->rh2 = a.take<float>(2 * S * H);
        e->q_rh2 = a.take<int8_t>(2 * S * H);
        e->sc_rh2 = a.take<float>(2 * S);
        e->ghc2 = a.take<float>(2 * S * H);
        e->enc_rows = a.take<int32_t>(L * 2 * S);
        e->enc_out_rows = a.take<int32_t>(L * 2 * S);
        e->enc_qm = a.take<uint32_t>((L + 1) * 4 * S);
        e->q_states = a.take<int8_t>(P * 2 * H);
        e->sc_sent = a.take<float>(S);
        e->pos_sent = a.take<int32_t>(P);
        e->s0tmp = a.take<float>(S * H);
        e->s0_dst = a.take<int32_t>(S);
        e->enc_states = a.take<float>(P * 2 * H);
        e->enc_att = a.take<float>(P * A);
        e->enc_attx = a.take<float>(P * A);
        e->enc_s0 = a.take<float>(S * H);
        e->sent_row = a.take<int64_t>(S);
        e->sent_len = a.take<int32_t>(S);
        e->emb = a.take<float>(N * E);
        e->q_emb = a.take<int8_t>(N * E);
        e->sc_emb = a.take<float>(S);
        e->q_s = a.take<int8_t>(N * H);
        e->sc_s = a.take<float>(S);
        e->gx = a.take<float>(N * 3 * H);
        e->gh = a.take<float>(N * 2 * H);
        e->z = a.take<float>(N * H);
        e->rh = a.take<float>(N * H);
        e->q_rh = a.take<int8_t>(N * H);
        e->sc_rh = a.take<float>(S);
        e->ghc = a.take<float>(N * H);
        e->q_q = a.take<int8_t>(N * H);
        e->sc_q = a.take<float>(S);
        e->u = a.take<float>(N * A);
        e->ctx = a.take<float>(N * 2 * H);
        e->q_ctx = a.take<int8_t>(N * 2 * H);
        e->sc_ctx = a.take<float>(S);
        e->q_si = a.take<int8_t>(N * H);
        e->sc_si = a.take<float>(S);
        e->q_sn = a.take<int8_t>(N * H);
        e->sc_sn = a.take<float>(S);
        e->ro = a.take<float>(N * R);
        e->q_ro = a.take<int8_t>(N * R);
        e->sc_ro = a.take<float>(S);
        e->logits = a.take<float>(N * V);
        // (also the persistent greedy kernel's per-CTA (max, sum) partials: 2 doubles per CTA, up to
        // 256 CTAs -- more than the fused kernel's partials of one row of a small vocabulary)
        e->vocab_part = a.take<char>(std::max<size_t>(vocab_topk_part_bytes((int64_t)N, (int64_t)V), 256 * 2 * sizeof(double)));
        e->att_scratch = a.take<char>(N * (L + 4) * 4 + 2 * S * A * 4 + N * A * 4 + 1024);
        e->att_mm = a.take<float>(2 * S * A);
        e->ctx_max = a.take<uint32_t>(S);
        e->gmax = a.take<uint32_t>(4 * S);
        e->w2x = a.take<int8_t>((3 * H + R) * E);
        e->w2x_s = a.take<float>(3 * H + R);
        e->b2x = a.take<float>(3 * H + R);
        e->w3x = a.take<int8_t>((3 * H + R) * 2 * H);
        e->w3x_s = a.take<float>(3 * H + R);
        e->b3x = a.take<float>(3 * H + R);
        e->wuq = a.take<int8_t>((A + 2 * H) * H);
        e->wuq_s = a.take<float>(A + 2 * H);
        e->gxr = a.take<float>(N * (3 * H + R));
        e->gxq = a.take<float>(N * (3 * H + R));
        e->uq = a.take<float>(N * (A + 2 * H));
        for (int i = 0; i < 2; ++i) {
            e->st_s[i] = a.take<float>(N * H);
            e->st_sp[i] = a.take<float>(N * H);
            e->y[i] = a.take<int32_t>(N);
            e->col_sent[i] = a.take<int32_t>(N);
            e->live[i] = a.take<double>(N);
        }
        e->s_int = a.take<float>(N * H);
        e->s_new = a.take<float>(N * H);
        e->parent_col = a.take<int32_t>(N);
        e->cand_score = a.take<double>(N * B);
        e->cand_tok = a.take<int32_t>(N * B);
        e->n_live = a.take<int32_t>(4);
        e->d_N = a.take<int32_t>(4);
        e->rng_off = a.take<int32_t>(S);
        e->rng_cnt = a.take<int32_t>(S);
        e->d_step = a.take<int32_t>(4);
        e->P = a.take<int32_t>(S);
        e->col_off = a.take<int32_t>(S);
        e->done = a.take<int32_t>(S);
        e->max_steps = a.take<int32_t>(S);
        e->steps_run = a.take<int32_t>(S);
        e->np_tmp = a.take<int32_t>(S);
        e->pk_ctl = a.take<int32_t>(PK_CTL_INTS);
        e->fin_cnt = a.take<int32_t>(S);
        e->fin_best = a.take<double>(S);
        if (pass == 0) {
            bytes = a.used;
            e->block_bytes = bytes;
            cudaError_t ce = cudaMalloc(&e->block, bytes);
            if (ce != cudaSuccess) { delete e; return cuda_status(ce, "engine cudaMalloc"); }
        }
    }
    if (e->guard) {   // fill the guard bands; their offsets to the device for the checker
        for (size_t o : e->guards) cudaMemset(e->block + o, 0xA5, ARENA_GUARD);
        cudaMalloc(&e->guards_dev, std::max<size_t>(1, e->guards.size()) * sizeof(size_t));
        cudaMemcpy(e->guards_dev, e->guards.data(), e->guards.size() * sizeof(size_t), cudaMemcpyHostToDevice);
    }
    std::vector<int32_t> io(idx), ev(S), od(S);
    for (size_t i = 0; i < idx; ++i) io[i] = (int32_t)i;
    for (size_t i = 0; i < S; ++i) { ev[i] = (int32_t)(2 * i); od[i] = (int32_t)(2 * i + 1); }
    cudaMemcpy(e->iota, io.data(), idx * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(e->even, ev.data(), S * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(e->odd, od.data(), S * 4, cudaMemcpyHostToDevice);
    cudaMemset(e->err, 0, 16);
    {   // per-sentence fused op + quantize: [16 columns][max(E, H, R)] values, gather [2][B][H]
        const size_t d = std::max(E, std::max(H, R));
        e->fq_ok = !m->fp32 && 16 * d * 4 <= FQ_SMEM_MAX && 2 * B * H * 4 <= FQ_SMEM_MAX && E % 4 == 0 && H % 4 == 0 &&
                   R % 4 == 0 && ((uintptr_t)m->tgt_embed % 16) == 0;   // float4 groups (fused_q.cu)
    }
    if (!m->fp32 && E % 16 == 0 && H % 16 == 0 && A % 16 == 0 && R % 16 == 0) {   // stacked weights (tcgen05 path)
        auto host_scale = [](const float* d) { float v = 0; cudaMemcpy(&v, d, 4, cudaMemcpyDeviceToHost); return v; };
        std::vector<float> sc;
        auto stack = [&](int8_t* dst, const int8_t* a0, size_t rows0, const int8_t* a1, size_t rows1, size_t K) {
            cudaMemcpy(dst, a0, rows0 * K, cudaMemcpyDeviceToDevice);
            cudaMemcpy(dst + rows0 * K, a1, rows1 * K, cudaMemcpyDeviceToDevice);
        };
        const qnmt::Cell& c2 = m->cell[2];
        const qnmt::Cell& c3 = m->cell[3];
        // [cell W_x (3 row-block scales); readout W (one scale)], bias [b_x; 0]
        auto stack_x = [&](const qnmt::Cell& c, const int8_t* wr, const float* wr_s, size_t K, int8_t* w, float* ws,
                           float* b) {
            stack(w, c.wx, 3 * H, wr, R, K);
            sc.assign(3 * H + R, 0.0f);
            for (size_t g = 0; g < 3; ++g) {
                const float v = host_scale(c.wx_s + g);
                for (size_t i = 0; i < H; ++i) sc[g * H + i] = v;
            }
            const float vr = host_scale(wr_s);
            for (size_t i = 0; i < R; ++i) sc[3 * H + i] = vr;
            cudaMemcpy(ws, sc.data(), (3 * H + R) * 4, cudaMemcpyHostToDevice);
            cudaMemset(b, 0, (3 * H + R) * 4);
            cudaMemcpy(b, c.bx, 3 * H * 4, cudaMemcpyDeviceToDevice);
        };
        stack_x(c2, m->w_embed, m->w_embed_s, E, e->w2x, e->w2x_s, e->b2x);
        stack_x(c3, m->w_ctx, m->w_ctx_s, 2 * H, e->w3x, e->w3x_s, e->b3x);
        // [U_att (one scale); cell3 U_zr (z, r scales)]
        stack(e->wuq, m->u_att, A, c3.uzr, 2 * H, H);
        sc.assign(A + 2 * H, 0.0f);
        const float va = host_scale(m->u_att_s);
        for (size_t i = 0; i < A; ++i) sc[i] = va;
        for (size_t g = 0; g < 2; ++g) {
            const float v = host_scale(c3.uzr_s + g);
            for (size_t i = 0; i < H; ++i) sc[A + g * H + i] = v;
        }
        cudaMemcpy(e->wuq_s, sc.data(), (A + 2 * H) * 4, cudaMemcpyHostToDevice);
        e->stack_ok = true;
        e->stack_u = m->aq == 0;
    }
    cudaMemset(e->gmax, 0, 4 * S * sizeof(uint32_t));
    e->gate_epi = e->fq_ok && H % 32 == 0 && E % 16 == 0 && H % 16 == 0;
    cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking);
    cudaError_t ce = cudaMallocHost(&e->h_pinned, 64);
    if (ce != cudaSuccess) { cudaFree(e->block); delete e; return cuda_status(ce, "cudaMallocHost"); }
    *out = e;
    return QNMT_OK;
}

int qnmt_engine_destroy(qnmt_engine* e) {
    if (!e) return QNMT_OK;
    std::unique_lock<std::shared_mutex> gate(g_capture_gate);   // not while another thread captures a step
    cudaDeviceSynchronize();
    if (e->block) cudaFree(e->block);
    if (e->guards_dev) cudaFree(e->guards_dev);
    if (e->hblock) cudaFree(e->hblock);
    if (e->h_pinned) cudaFreeHost(e->h_pinned);
    if (e->res_host) cudaFreeHost(e->res_host);
    for (auto& kv : e->graphs) {
        cudaGraphExecDestroy(kv.second.first);
        cudaGraphExecDestroy(kv.second.second);
    }
    if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
    delete e;
    return QNMT_OK;
}

int qnmt_engine_stamps(qnmt_engine* e, int enable) {
    int old = e->stamp_on ? 1 : 0;
    e->stamp_on = enable != 0;
    return old;
}

int qnmt_engine_stamps_read(qnmt_engine* e, int64_t* out, int32_t max_rows, void* stream) {
    cudaStream_t st = as_stream(stream);
    int32_t steps = 0;
    QNMT_CUDA(cudaMemcpyAsync(&steps, e->d_step, 4, cudaMemcpyDeviceToHost, st));
    QNMT_CUDA(cudaStreamSynchronize(st));
    int rows = std::min(std::min(steps, max_rows), e->hist_steps);
    if (rows > 0) {
        QNMT_CUDA(cudaMemcpyAsync(out, e->stamps, (size_t)rows * ST_COLS * 8, cudaMemcpyDeviceToHost, st));
        QNMT_CUDA(cudaStreamSynchronize(st));
    }
    return rows;
}

int qnmt_engine_set_graphs(qnmt_engine* e, int enable) {
    int old = e->use_graphs ? 1 : 0;
    e->use_graphs = enable != 0;
    return old;
}

int qnmt_engine_profile(qnmt_engine* e, int enable) {
    {
        std::unique_lock<std::shared_mutex> gate(g_capture_gate);
        cudaDeviceSynchronize();
    }
    prof_collect(e);
    e->prof_on = enable != 0;
    e->prof_group = -1;
    for (int i = 0; i < 16; ++i) e->prof_ms[i] = e->prof_calls[i] = e->prof_ops[i] = e->prof_bytes[i] = 0;
    return QNMT_OK;
}

int qnmt_engine_profile_read(const qnmt_engine* e, double* ms, double* calls, double* ops, double* bytes) {
    for (int i = 0; i < 16; ++i) {
        ms[i] = e->prof_ms[i];
        calls[i] = e->prof_calls[i];
        ops[i] = e->prof_ops[i];
        bytes[i] = e->prof_bytes[i];
    }
    return PG_COUNT;
}

size_t qnmt_engine_bytes(const qnmt_engine* e) { return e ? e->block_bytes + e->hblock_bytes : 0; }

int64_t qnmt_engine_check_canaries(qnmt_engine* e, void* stream) {
    if (!e || !e->guard) return -1;
    cudaStream_t st = qnmt::as_stream(stream);
    unsigned long long* bad = nullptr;
    if (cudaMalloc(&bad, sizeof(unsigned long long)) != cudaSuccess) return -2;
    cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st);
    if (!e->guards.empty())
        qnmt::k_check_guards<<<std::min<size_t>(e->guards.size(), 1024), 256, 0, st>>>(
            reinterpret_cast<const unsigned char*>(e->block), e->guards_dev, (int)e->guards.size(), bad);
    unsigned long long h = 0;
    cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(bad);
    return (int64_t)h;
}

int qnmt_encode_batch(qnmt_engine* e, const int32_t* src_ids_dev, const int32_t* src_len, int32_t n,
                      float* states, float* att_proj, float* s0, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (n < 1) { set_error("no sentences"); return QNMT_ERR_EMPTY; }
    std::vector<int64_t> row(n);
    int64_t acc = 0;
    for (int i = 0; i < n; ++i) { row[i] = acc; acc += src_len[i]; }
    QNMT_CUDA(cudaMemsetAsync(e->err, 0, 4, st));
    TRY(encode_core(e, src_ids_dev, src_len, row.data(), n, states, att_proj, s0, st));
    return check_flag(e, st);
}

int qnmt_decoder_step(qnmt_engine* e, int64_t N, const int32_t* col_sent, int32_t n_sent,
                      const int32_t* y, const float* s, const float* sp, const float* states,
                      const float* att_proj, const int64_t* sent_row, const int32_t* sent_len,
                      int32_t max_len, float* s_int, float* s_new, float* logits, float* alpha,
                      int64_t lda, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (N > e->NMAX || n_sent > e->S || max_len > e->L) { set_error("step exceeds engine capacity"); return QNMT_ERR_CONFIG; }
    QNMT_CUDA(cudaMemsetAsync(e->err, 0, 4, st));
    TRY(col_ranges_launch(col_sent, N, n_sent, e->rng_off, e->rng_cnt, st));
    StepIO io{N, n_sent, col_sent, y, s, sp, states, att_proj, sent_row, sent_len, max_len,
              s_int, s_new, logits, alpha, lda, e->rng_off, e->rng_cnt, nullptr, nullptr, 16, false, false};
    TRY(step_core(e, io, st));
    return check_flag(e, st);
}

// ---------------------------------------------------------------------------
// CUDA-graph decode step.  Every kernel of a step reads the live column count
// from d_N[cur] (grids are sized for n*beam); the search kernel writes
// d_N[cur^1] and advances d_step.  Two graphs (cur = 0, 1) cover the
// ping-pong state buffers; they are captured once per (n_sent, beam).
// ---------------------------------------------------------------------------
static bool graph_eligible(const qnmt_engine* e) {
    const qnmt_model* m = e->m;
    return e->use_graphs && !e->prof_on && !m->fp32 && g_gemm_impl != 1 && m->E % 16 == 0 && m->H % 16 == 0 &&
           m->A % 16 == 0 && m->R % 16 == 0;
}

static int capture_step(qnmt_engine* e, int cur, int n, int beam, int k_list, cudaGraphExec_t* out) {
    const qnmt_model* m = e->m;
    const int64_t H = m->H, V = m->Vt;
    const int64_t NM = (int64_t)n * beam;
    cudaStream_t cs = e->cap_stream;
    std::shared_lock<std::shared_mutex> gate(g_capture_gate);   // no device-wide sync / free meanwhile
    QNMT_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    int rc = QNMT_OK;
    bool fused_gather = false;
    {
        NdevScope nd(e->d_N + cur);
        StepIO io{NM, n, e->col_sent[cur], e->y[cur], e->st_s[cur], e->st_sp[cur], e->enc_states, e->enc_att,
                  e->sent_row, e->sent_len, e->L, e->s_int, e->s_new, e->logits, nullptr, 0,
                  e->col_off, e->P, e->att_mm, e->enc_attx, beam, e->fq_ok, vocab_fusable(e, k_list)};
        rc = stamp(e, ST_STEP0, io, cs);
        if (rc == QNMT_OK) rc = step_core(e, io, cs);
        if (rc == QNMT_OK) rc = cands_launch(e, io, e->live[cur], k_list, cs);
        if (rc == QNMT_OK) {
            SearchState ss{e->P, e->col_off, e->done, e->max_steps, e->steps_run, e->fin_cnt, e->fin_best,
                           e->fin_score, e->fin_step, e->fin_slot, e->fin_eos, e->hist_tok, e->hist_par,
                           (e->hist_steps + 1) * e->B, e->hist_steps, e->B, e->cand_score, e->cand_tok,
                           e->col_sent[cur ^ 1], e->parent_col, e->y[cur ^ 1], e->live[cur ^ 1],
                           e->d_N + (cur ^ 1), e->d_step};
            ss.np_tmp = e->np_tmp;
            if (e->fq_ok && g_layout_gather) {   // selection, then layout + state gather in one launch
                rc = search_select_launch(ss, 0, n, beam, k_list, cs);
                if (rc == QNMT_OK)
                    rc = layout_gather_q_launch(ss, n, beam, k_list, e->s_new, m->aq == 1 ? e->s_int : nullptr, H,
                                                e->st_s[cur ^ 1], e->st_sp[cur ^ 1], e->q_s, e->sc_s,
                                                m->aq == 1 ? e->q_q : nullptr, m->aq == 1 ? e->sc_q : nullptr, e->err,
                                                cs);
                fused_gather = true;
            } else {
                rc = search_step_launch(ss, 0, n, beam, k_list, cs);
            }
        }
    }
    if (rc == QNMT_OK && !fused_gather) {
        NdevScope nd(e->d_N + (cur ^ 1));
        rc = gather_next(e, cur, NM, n, beam, cs);
    }
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(cs, &g);
    if (rc != QNMT_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (ce != cudaSuccess) return cuda_status(ce, "cudaStreamEndCapture");
    {   // kernel nodes per step graph (for the launch counter: one graph launch runs all of them)
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) cudaGraphGetNodes(g, nodes.data(), &nn);
        int kn = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) ++kn;
        }
        e->graph_kernels = kn;
    }
    ce = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return cuda_status(ce, "cudaGraphInstantiate");
    return QNMT_OK;
}

static int get_step_graphs(qnmt_engine* e, int n, int beam, int k_list, cudaGraphExec_t* g) {
    // history buffers may have been re-allocated: graphs are keyed on the history capacity too
    const int key2 = ((beam * 100000 + e->hist_steps) * 2 + (e->stamp_on ? 1 : 0)) * 2 + (vocab_fusable(e, k_list) ? 1 : 0);
    for (auto& kv : e->graphs)
        if (kv.first.first == n && kv.first.second == key2) {
            g[0] = kv.second.first;
            g[1] = kv.second.second;
            return QNMT_OK;
        }
    TRY(capture_step(e, 0, n, beam, k_list, &g[0]));
    TRY(capture_step(e, 1, n, beam, k_list, &g[1]));
    e->graphs.push_back({{n, key2}, {g[0], g[1]}});
    return QNMT_OK;
}

static void drop_graphs(qnmt_engine* e) {
    for (auto& kv : e->graphs) {
        cudaGraphExecDestroy(kv.second.first);
        cudaGraphExecDestroy(kv.second.second);
    }
    e->graphs.clear();
}

// host-side batch layout: row offsets, per-sentence step caps (decoder.py:103)
struct BatchPlan {
    std::vector<int64_t> row;
    std::vector<int32_t> msteps;
    int64_t P = 0;
    int Lmax = 0, Tmax = 0;
};

static int plan_batch(const qnmt_engine* e, const int32_t* src_ids, bool ids_on_device, const int32_t* src_len,
                      int32_t n, int32_t beam, double max_ratio, BatchPlan& b) {
    const qnmt_model* m = e->m;
    if (n < 1) { set_error("no sentences"); return QNMT_ERR_EMPTY; }
    if (beam < 1 || beam > e->B || !(max_ratio > 0)) { set_error("bad beam/max_ratio"); return QNMT_ERR_CONFIG; }
    if (n > e->S) { set_error("batch of %d exceeds engine capacity %d", n, e->S); return QNMT_ERR_CONFIG; }
    b.row.resize(n);
    b.msteps.resize(n);
    for (int i = 0; i < n; ++i) {
        if (src_len[i] < 1) { set_error("cannot translate an empty sentence"); return QNMT_ERR_EMPTY; }
        if (src_len[i] > e->L) { set_error("sentence of length %d exceeds engine capacity %d", src_len[i], e->L); return QNMT_ERR_CONFIG; }
        b.row[i] = b.P;
        b.P += src_len[i];
        b.Lmax = std::max(b.Lmax, src_len[i]);
        b.msteps[i] = (int32_t)ceil(max_ratio * (double)src_len[i]) + 1;   // decoder.py:103
        b.Tmax = std::max(b.Tmax, b.msteps[i]);
    }
    if (!ids_on_device)
        for (int64_t i = 0; i < b.P; ++i)
            if (src_ids[i] < 0 || src_ids[i] >= m->Vs) { set_error("source id outside [0, %d)", m->Vs); return QNMT_ERR_VOCAB; }
    return QNMT_OK;
}

// encoder + per-model decoder state for a batch: s = s' = s0 and the first step's state codes
static int init_member(qnmt_engine* e, const int32_t* src_ids, bool ids_on_device, const int32_t* src_len,
                       const BatchPlan& b, int32_t n, cudaStream_t st) {
    const qnmt_model* m = e->m;
    const int64_t H = m->H;
    QNMT_CUDA(cudaMemsetAsync(e->err, 0, 4, st));
    if (ids_on_device)
        QNMT_CUDA(cudaMemcpyAsync(e->src_ids, src_ids, (size_t)b.P * 4, cudaMemcpyDeviceToDevice, st));
    else
        QNMT_CUDA(h2d(e, e->src_ids, src_ids, (size_t)b.P * 4, st));
    prof_mark(e, PG_ENCODER, st);
    TRY(encode_core(e, e->src_ids, src_len, b.row.data(), n, e->enc_states, e->enc_att, e->enc_s0, st));
    prof_mark(e, PG_MISC, st);
    QNMT_CUDA(h2d(e, e->sent_row, b.row.data(), (size_t)n * 8, st));
    QNMT_CUDA(h2d(e, e->sent_len, src_len, (size_t)n * 4, st));
    TRY(att_minmax_launch(e->enc_att, e->sent_row, e->sent_len, n, m->A, e->att_mm, st));
    if (!m->fp32) TRY(att_exp_launch(e->enc_att, b.P * m->A, e->enc_attx, st));
    QNMT_CUDA(cudaMemcpyAsync(e->st_s[0], e->enc_s0, (size_t)n * H * 4, cudaMemcpyDeviceToDevice, st));
    QNMT_CUDA(cudaMemcpyAsync(e->st_sp[0], e->enc_s0, (size_t)n * H * 4, cudaMemcpyDeviceToDevice, st));
    if (e->fq_ok) {   // first step's state codes (later steps get them from gather_q); column n = sentence n
        TRY(quantize_launch(e->enc_s0, n, H, H, e->iota, n, e->q_s, H, e->sc_s, e->seg_bits, 1, e->err, st));
        if (m->aq == 1)
            TRY(quantize_launch(e->enc_s0, n, H, H, e->iota, n, e->q_q, H, e->sc_q, e->seg_bits, 1, e->err, st));
    }
    return QNMT_OK;
}

// search state: one column per sentence, y = EOS (BOS), live score 0 (decoder.py:105-110)
static int init_search(qnmt_engine* e, const BatchPlan& b, int32_t n, cudaStream_t st) {
    {
        // Size the history for the longest sentence this engine can hold at this batch's length
        // ratio, not for this batch: regrowing drops the captured step graphs (they point into
        // the old block), and an engine of a pool that meets a slightly longer batch than before
        // paid a re-capture (~0.1-0.25 s) in the middle of a corpus (seen as e2e outlier steps).
        int want = b.Tmax;
        if (b.Tmax > e->hist_steps && b.Lmax > 0) {
            const long long cap = ((long long)b.Tmax * e->L + b.Lmax - 1) / b.Lmax + 1;
            want = (int)std::min<long long>(std::max<long long>(cap, b.Tmax), std::max(4096, b.Tmax));
            if ((size_t)e->S * e->B * (size_t)want * 28 > ((size_t)256 << 20)) want = b.Tmax;   // (huge engines: exact fit)
        }
        TRY(grow_history(e, want));
    }
    e->last_n = n;
    e->last_tmax = b.Tmax;
    std::vector<int32_t> iota_n(n), y0(n, 2), ones(n, 1);
    std::iota(iota_n.begin(), iota_n.end(), 0);
    std::vector<double> dz(n, 0.0);
    QNMT_CUDA(h2d(e, e->max_steps, b.msteps.data(), (size_t)n * 4, st));
    QNMT_CUDA(h2d(e, e->P, ones.data(), (size_t)n * 4, st));
    QNMT_CUDA(h2d(e, e->col_off, iota_n.data(), (size_t)n * 4, st));
    QNMT_CUDA(h2d(e, e->col_sent[0], iota_n.data(), (size_t)n * 4, st));
    QNMT_CUDA(h2d(e, e->y[0], y0.data(), (size_t)n * 4, st));
    QNMT_CUDA(h2d(e, e->live[0], dz.data(), (size_t)n * 8, st));
    QNMT_CUDA(cudaMemsetAsync(e->done, 0, (size_t)n * 4, st));
    QNMT_CUDA(cudaMemsetAsync(e->fin_cnt, 0, (size_t)n * 4, st));
    QNMT_CUDA(cudaMemsetAsync(e->steps_run, 0, (size_t)n * 4, st));
    return QNMT_OK;   // (pageable H2D copies are staged before cudaMemcpyAsync returns)
}

static SearchState search_state(qnmt_engine* e, int cur, int32_t* n_out) {
    SearchState ss{e->P, e->col_off, e->done, e->max_steps, e->steps_run, e->fin_cnt, e->fin_best,
                   e->fin_score, e->fin_step, e->fin_slot, e->fin_eos, e->hist_tok, e->hist_par,
                   (e->hist_steps + 1) * e->B, e->hist_steps, e->B, e->cand_score, e->cand_tok,
                   e->col_sent[cur ^ 1], e->parent_col, e->y[cur ^ 1], e->live[cur ^ 1], n_out};
    ss.np_tmp = e->np_tmp;
    return ss;
}

// Batch-1 greedy translation as one persistent kernel (persistent.cu): the
// latency path of BASELINE cfg3.  Needs the stacked decoder weights (current-
// state query) and vectors of at most 2048 values per quantization.
static bool greedy1_eligible(const qnmt_engine* e) {
    const qnmt_model* m = e->m;
    return g_greedy1 && !m->fp32 && m->aq == 0 && e->stack_ok && e->stack_u && e->fq_ok && !e->prof_on &&
           m->E % 16 == 0 && m->H % 16 == 0 && m->A % 16 == 0 && m->R % 16 == 0 && 2 * m->H <= 2048 &&
           m->A <= 2048 && m->E <= 2048 && m->R <= 2048 && e->L * 8 <= 96 * 1024;
}

static int decode_greedy1(qnmt_engine* e, const BatchPlan& b, cudaStream_t st) {
    const qnmt_model* m = e->m;
    const int H = m->H;
    const Cell& c2 = m->cell[2];
    const Cell& c3 = m->cell[3];
    PkArgs a{};
    a.E = m->E; a.H = H; a.A = m->A; a.R = m->R; a.V = m->Vt;
    a.tgt_embed = m->tgt_embed;
    a.w2x = e->w2x; a.w2x_s = e->w2x_s; a.b2x = e->b2x;
    a.uzr2 = c2.uzr; a.uzr2_s = c2.uzr_s; a.uc2 = c2.uc; a.uc2_s = c2.uc_s;
    a.wuq = e->wuq; a.wuq_s = e->wuq_s;
    a.w3x = e->w3x; a.w3x_s = e->w3x_s; a.b3x = e->b3x;
    a.uc3 = c3.uc; a.uc3_s = c3.uc_s;
    a.v = m->v; a.v_s = m->v_s;
    a.w_state = m->w_state; a.w_state_s = m->w_state_s; a.b_r = m->b_r;
    a.w_vocab = m->w_vocab; a.w_vocab_s = m->w_vocab_s; a.b_vocab = m->b_vocab;
    a.states = e->enc_states; a.att = e->enc_att; a.att_mm = e->att_mm;
    a.l = (int)b.P;
    a.max_steps = b.msteps[0];
    a.s = e->st_s[0]; a.sp = e->st_sp[0];
    a.gxr = e->gxr; a.gh = e->gh; a.ghc = e->ghc; a.uq = e->uq;
    a.scores = reinterpret_cast<float*>(e->att_scratch);
    a.ctx = e->ctx; a.gxq = e->gxq; a.ro = e->ro; a.logits = e->logits;
    a.part = reinterpret_cast<double*>(e->vocab_part);
    a.ctl = e->pk_ctl;
    a.hist_tok = e->hist_tok; a.hist_par = e->hist_par; a.hist_stride = e->B;
    a.fin_score = e->fin_score; a.fin_step = e->fin_step; a.fin_slot = e->fin_slot; a.fin_eos = e->fin_eos;
    a.fin_cnt = e->fin_cnt;
    a.err = e->err;
    a.stamps = e->stamp_on ? e->stamps : nullptr;
    a.step_dev = e->d_step;
    int32_t* ctl0 = e->h_pinned + 4;   // host staging of the control words
    ctl0[0] = 2; ctl0[1] = 0x7fffffff; ctl0[2] = 0; ctl0[3] = 0; ctl0[4] = 0;
    QNMT_CUDA(cudaMemsetAsync(e->pk_ctl, 0, PK_CTL_INTS * sizeof(int32_t), st));   // barrier counters
    QNMT_CUDA(h2d(e, e->pk_ctl, ctl0, 5 * sizeof(int32_t), st));
    TRY(greedy1_launch(a, st));
    return check_flag(e, st);
}

// device-resident decode of one batch; results stay in the engine until finalize.
static int decode_core(qnmt_engine* e, const int32_t* src_ids, bool ids_on_device, const int32_t* src_len,
                       int32_t n, int32_t beam, double max_ratio, cudaStream_t st) {
    const qnmt_model* m = e->m;
    const int64_t V = m->Vt;
    BatchPlan b;
    e->h2d_bytes = 0;
    TRY(plan_batch(e, src_ids, ids_on_device, src_len, n, beam, max_ratio, b));
    TRY(init_search(e, b, n, st));
    TRY(init_member(e, src_ids, ids_on_device, src_len, b, n, st));
    const int Tmax = b.Tmax, Lmax = b.Lmax;
    const int k_list = (int)std::min<int64_t>(beam, V);
    if (n == 1 && beam == 1 && greedy1_eligible(e)) return decode_greedy1(e, b, st);
    if (graph_eligible(e)) {
        // device-resident loop: one graph launch per step, live count polled every POLL steps
        cudaGraphExec_t g[2];
        TRY(get_step_graphs(e, n, beam, k_list, g));
        e->h_pinned[1] = n;
        QNMT_CUDA(h2d(e, e->d_N, e->h_pinned + 1, 4, st));
        QNMT_CUDA(cudaMemsetAsync(e->d_step, 0, 4, st));
        constexpr int POLL = 16;
        for (int t = 0; t < Tmax; ++t) {
            QNMT_CUDA(cudaGraphLaunch(g[t & 1], st));
            for (int q = 0; q < e->graph_kernels; ++q) count_launch();
            if ((t + 1) % POLL == 0 && t + 1 < Tmax) {
                QNMT_CUDA(cudaMemcpyAsync(e->h_pinned, e->d_N + ((t + 1) & 1), 4, cudaMemcpyDeviceToHost, st));
                QNMT_CUDA(cudaStreamSynchronize(st));
                if (e->h_pinned[0] == 0) break;
            }
        }
        return check_flag(e, st);
    }
    int64_t N = n;
    int cur = 0;
    for (int t = 0; t < Tmax && N > 0; ++t) {
        StepIO io{N, n, e->col_sent[cur], e->y[cur], e->st_s[cur], e->st_sp[cur], e->enc_states,
                  e->enc_att, e->sent_row, e->sent_len, Lmax, e->s_int, e->s_new, e->logits, nullptr, 0,
                  e->col_off, e->P, e->att_mm, e->enc_attx, beam, e->fq_ok, vocab_fusable(e, k_list)};
        TRY(step_core(e, io, st));
        TRY(cands_launch(e, io, e->live[cur], k_list, st));
        prof_mark(e, PG_SEARCH, st);
        TRY(search_step_launch(search_state(e, cur, e->n_live), t, n, beam, k_list, st));
        QNMT_CUDA(cudaMemcpyAsync(e->h_pinned, e->n_live, 4, cudaMemcpyDeviceToHost, st));
        QNMT_CUDA(cudaStreamSynchronize(st));
        prof_collect(e);
        int64_t N2 = e->h_pinned[0];
        prof_mark(e, PG_GATHER, st);
        TRY(gather_next(e, cur, N2, n, beam, st));
        N = N2;
        cur ^= 1;
    }
    prof_mark(e, -1, st);
    int rc = check_flag(e, st);
    prof_collect(e);
    return rc;
}

// Ensemble decode (decoder.py:88-160 with several members): eager steps, one host
// sync per step.  es[0] holds the search state; every member steps its own
// states against the shared column layout, tokens and parents.
static int decode_ensemble(qnmt_engine* const* es, int nm, const int32_t* src_ids, const int32_t* src_len, int32_t n,
                           int32_t beam, double max_ratio, cudaStream_t st) {
    qnmt_engine* lead = es[0];
    const int64_t V = lead->m->Vt;
    if (nm < 2 || nm > QNMT_ENS_MAX) { set_error("ensemble of %d members outside [2, %d]", nm, QNMT_ENS_MAX); return QNMT_ERR_CONFIG; }
    for (int i = 1; i < nm; ++i) {
        if (es[i]->m->Vt != V) { set_error("ensemble members must share the target vocabulary"); return QNMT_ERR_CONFIG; }
        if (es[i]->S != lead->S || es[i]->L != lead->L || es[i]->B != lead->B) {
            set_error("ensemble engines must have the same capacity");
            return QNMT_ERR_CONFIG;
        }
        for (int j = 0; j < i; ++j)
            if (es[j] == es[i]) { set_error("ensemble members need distinct engines"); return QNMT_ERR_CONFIG; }
    }
    // members map the tokens with their own source vocabularies (decoder.py:99): ids are member-major
    BatchPlan b;
    TRY(plan_batch(lead, src_ids, false, src_len, n, beam, max_ratio, b));
    for (int i = 1; i < nm; ++i) {
        BatchPlan bi;
        TRY(plan_batch(es[i], src_ids + (size_t)i * b.P, false, src_len, n, beam, max_ratio, bi));
    }
    for (int i = 0; i < nm; ++i) es[i]->h2d_bytes = 0;
    TRY(init_search(lead, b, n, st));
    for (int i = 0; i < nm; ++i) TRY(init_member(es[i], src_ids + (size_t)i * b.P, false, src_len, b, n, st));
    const int k_list = (int)std::min<int64_t>(beam, V);
    EnsRows rows{};
    for (int i = 0; i < nm; ++i) rows.p[i] = es[i]->logits;
    int64_t N = n;
    int cur = 0;
    for (int t = 0; t < b.Tmax && N > 0; ++t) {
        for (int i = 0; i < nm; ++i) {
            qnmt_engine* e = es[i];
            StepIO io{N, n, lead->col_sent[cur], lead->y[cur], e->st_s[cur], e->st_sp[cur], e->enc_states,
                      e->enc_att, e->sent_row, e->sent_len, b.Lmax, e->s_int, e->s_new, e->logits, nullptr, 0,
                      lead->col_off, lead->P, e->att_mm, e->enc_attx, beam, e->fq_ok, false};
            TRY(step_core(e, io, st));
        }
        TRY(ens_topk_launch(rows, nm, N, V, V, lead->live[cur], k_list, lead->cand_score, lead->cand_tok, lead->err,
                            st));
        TRY(search_step_launch(search_state(lead, cur, lead->n_live), t, n, beam, k_list, st));
        QNMT_CUDA(cudaMemcpyAsync(lead->h_pinned, lead->n_live, 4, cudaMemcpyDeviceToHost, st));
        QNMT_CUDA(cudaStreamSynchronize(st));
        const int64_t N2 = lead->h_pinned[0];
        for (int i = 0; i < nm; ++i) TRY(gather_next(es[i], cur, N2, n, beam, st, lead));
        N = N2;
        cur ^= 1;
    }
    for (int i = 0; i < nm; ++i) TRY(check_flag(es[i], st));
    return QNMT_OK;
}

// min by (-logp, tokens) on the device (k_finalize, decoder.py:157-160), then one
// D2H of the packed rows [len, logp, tokens] -- n * (Tmax + 3) words per batch
static int finalize(qnmt_engine* e, int32_t* out_tokens, int32_t out_stride, int32_t* out_len,
                    double* out_logp, cudaStream_t st) {
    const int n = e->last_n;
    if (out_stride < e->last_tmax) { set_error("out_stride %d < max steps %d", out_stride, e->last_tmax); return QNMT_ERR_CONFIG; }
    if (n <= 0) return QNMT_OK;
    const int T = e->hist_steps, W = T + 3, Wc = e->last_tmax + 3;
    FinalizeArgs a{e->fin_cnt, e->fin_score, e->fin_step, e->fin_slot, e->fin_eos, e->hist_tok, e->hist_par,
                   (T + 1) * e->B, T, e->B, e->res_dev, W, e->fin_scratch, 0};
    TRY(finalize_launch(a, n, st));
    QNMT_CUDA(cudaMemcpy2DAsync(e->res_host, (size_t)Wc * 4, e->res_dev, (size_t)W * 4, (size_t)Wc * 4, n,
                                cudaMemcpyDeviceToHost, st));
    QNMT_CUDA(cudaStreamSynchronize(st));
    e->d2h_bytes = (int64_t)n * Wc * 4;
    for (int s = 0; s < n; ++s) {
        const int32_t* row = e->res_host + (size_t)s * Wc;
        const int len = row[0];
        out_len[s] = len;
        const uint64_t bits = (uint64_t)(uint32_t)row[1] | ((uint64_t)(uint32_t)row[2] << 32);
        memcpy(&out_logp[s], &bits, 8);
        memcpy(out_tokens + (size_t)s * out_stride, row + 3, (size_t)len * 4);
    }
    return QNMT_OK;
}

int qnmt_translate_batch(qnmt_engine* e, const int32_t* src_ids, const int32_t* src_len, int32_t n,
                         int32_t beam, double max_ratio, int32_t* out_tokens, int32_t out_stride,
                         int32_t* out_len, double* out_logp, void* stream) {
    cudaStream_t st = as_stream(stream);
    TRY(decode_core(e, src_ids, false, src_len, n, beam, max_ratio, st));
    return finalize(e, out_tokens, out_stride, out_len, out_logp, st);
}

int qnmt_translate_ensemble(qnmt_engine* const* engines, int32_t n_members, const int32_t* src_ids,
                            const int32_t* src_len, int32_t n, int32_t beam, double max_ratio, int32_t* out_tokens,
                            int32_t out_stride, int32_t* out_len, double* out_logp, void* stream) {
    if (n_members == 1) return qnmt_translate_batch(engines[0], src_ids, src_len, n, beam, max_ratio, out_tokens,
                                                    out_stride, out_len, out_logp, stream);
    cudaStream_t st = as_stream(stream);
    TRY(decode_ensemble(engines, n_members, src_ids, src_len, n, beam, max_ratio, st));
    return finalize(engines[0], out_tokens, out_stride, out_len, out_logp, st);
}

int qnmt_decode_batch_device(qnmt_engine* e, const int32_t* src_ids_dev, const int32_t* src_len,
                             int32_t n, int32_t beam, double max_ratio, void* stream) {
    return decode_core(e, src_ids_dev, true, src_len, n, beam, max_ratio, as_stream(stream));
}

int qnmt_fetch_results(qnmt_engine* e, int32_t* out_tokens, int32_t out_stride, int32_t* out_len,
                       double* out_logp, void* stream) {
    return finalize(e, out_tokens, out_stride, out_len, out_logp, as_stream(stream));
}

int64_t qnmt_last_d2h_bytes(const qnmt_engine* e) { return e ? e->d2h_bytes : 0; }

int64_t qnmt_last_h2d_bytes(const qnmt_engine* e) { return e ? e->h2d_bytes : 0; }

}  // extern "C"

extern "C" int qnmt_set_gate_epi(int enable) {
    const int old = qnmt::g_gate_epi;
    qnmt::g_gate_epi = enable ? 1 : 0;
    return old;
}
