// persistent.cu -- the batch-1 greedy latency path (BASELINE cfg3) as ONE
// persistent kernel: every decoder step of decoder.translate(beam=1) for one
// sentence, on a cooperative grid of one CTA per SM with grid-wide barriers
// between the dependent phases of a step, instead of ~16 kernel launches per
// step.  Per step (layers.py:356-384 + decoder.py:112-155 at P = 1):
//
//   P0  q(emb[y]), q(s)                 (every CTA, redundantly: <= 2H values)
//       GEMV  [W_x2; W_e] q(emb) + b, U_zr2 q(s)            rows over all warps
//   P1  z, q(r * s)  ->  GEMV U_c2                          (cell dec_r)
//   P2  s' = (1-z) s + z tanh(.)  ->  q(s')  ->  GEMV [U_att; U_zr3] q(s')
//   P3  attention scale; scores of the positions (one CTA per position)
//   P4  softmax (every CTA); context features over all threads
//   P5  q(ctx)  ->  GEMV [W_x3; W_c] q(ctx) + b
//   P6  z, q(r * s')  ->  GEMV U_c3                         (cell dec_q)
//   P7  s_new  ->  q(s_new)  ->  GEMV W_s q(s_new) + b_r
//   P8  readout tanh(((.) + W_e e) + W_c c)  ->  q  ->  vocab GEMV (logits)
//   P9  per-CTA (max, sum exp) of its token range
//   P10 lse; every CTA finds the smallest token whose log-prob equals the best
//       one (so the next step needs no further barrier)
//   P11 CTA 0: search bookkeeping (EOS -> finished, length cap -> frozen)
//
// Numerics are those of the batched engine (Tier B): the same quantization,
// exact integer dot products, exact dequantization (dequant: __ddiv_rn), fp64
// sigmoid / tanh rounded once, fp64 softmax and context in position order,
// attention codes from the fp64 tanh (the engine's fast path + exact fallback
// produces exactly these codes).  Only fp64 summation orders of the vocabulary
// log-sum-exp differ (as between any two correct implementations).  Results go
// to the engine's history / finished arrays, so finalize() is unchanged.
// Weights stay L2-resident across the steps of the one launch (34 MB at cfg3).
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "persistent.cuh"
#include "search.cuh"

namespace qnmt {

#ifndef QNMT_PK_T
#define QNMT_PK_T 256
#endif
constexpr int PK_T = QNMT_PK_T;        // threads per CTA (8 warps)
constexpr int PK_W = PK_T / 32;
constexpr int PK_MAXD = 2048;          // longest vector quantized per CTA (2H, A <= 2048)



__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }

// grid-wide barrier; every CTA is resident (cooperative launch).  One monotonically
// increasing arrival counter (zeroed by the host before the launch): barrier number b is
// passed when the counter reaches b * gridDim.x, so an arrival is ONE fire-and-forget
// red.release (no returned value, no reset, no separate generation word) and the wait is
// an acquire load of the same word -- the last arriver's critical path is one L2 hop
// instead of four dependent round trips (load generation, add, exchange, add generation).
// `epoch` is the caller's running target (uniform across the grid).
// (A two-level variant -- groups of 16 CTAs on their own counters -- measured slower:
// cfg3 74.3 vs 67.6 us per decoder step; the second hop costs more latency than the
// 148-way contention on one counter.)
__device__ __forceinline__ void gsync(int32_t* ctl, unsigned& epoch) {
    __syncthreads();
    epoch += gridDim.x;
    if (threadIdx.x == 0) {
        unsigned* count = reinterpret_cast<unsigned*>(ctl + 3);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        unsigned cur;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(count) : "memory");
        } while ((int)(cur - epoch) < 0);
    }
    __syncthreads();
}

// block max of |x| bits
__device__ __forceinline__ uint32_t block_max_u(uint32_t m, uint32_t* red) {
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    uint32_t r = red[0];
#pragma unroll
    for (int w = 1; w < PK_W; ++w) r = max(r, red[w]);
    __syncthreads();
    return r;
}

// quantize vals[0..D) (smem f32) into q (smem int8) with the segment scale rule
// (qmath.py:119-142 / fused_q.cu seg_scale: a non-finite max raises the flag, scale 1)
__device__ float quantize_vec(const float* vals, int D, int8_t* q, uint32_t* red, int32_t* err) {
    uint32_t m = 0;
    for (int j = threadIdx.x; j < D; j += PK_T) m = max(m, __float_as_uint(vals[j]) & 0x7fffffffu);
    uint32_t mm = block_max_u(m, red);
    if (mm >= 0x7f800000u) {
        if (threadIdx.x == 0 && blockIdx.x == 0) set_flag(err, QNMT_FLAG_NUMERIC);
        mm = 0;
    }
    const float sc = scale_from_maxbits(mm);
    for (int j = threadIdx.x; j < D; j += PK_T) q[j] = (int8_t)quant_code(vals[j], sc);
    __syncthreads();
    return sc;
}

// one weight row . q (int8, K % 16 == 0) by a warp: 16-byte chunks per lane, dp4a, REDUX
__device__ __forceinline__ int row_dot(const int8_t* __restrict__ w, const int8_t* q, int K) {
    const int lane = threadIdx.x & 31;
    int acc = 0;
    for (int k = lane * 16; k < K; k += 512) {
        const int4 a = __ldg(reinterpret_cast<const int4*>(w + k));
        const int4 b = *reinterpret_cast<const int4*>(q + k);
        acc = __dp4a(a.x, b.x, acc);
        acc = __dp4a(a.y, b.y, acc);
        acc = __dp4a(a.z, b.z, acc);
        acc = __dp4a(a.w, b.w, acc);
    }
    return __reduce_add_sync(0xffffffffu, acc);
}

// rows [0, M) of W (row stride K) against q: out[m] = fl32(acc / (sw * sx)) (+ bias[m]);
// scale of row m: ws[m / rps].  Each warp owns a contiguous block of rows and keeps
// PK_RB rows' weight loads in flight; lane r dequantizes row r of each group.
constexpr int PK_RB = 8;
__device__ __forceinline__ void gemv(const int8_t* __restrict__ W, int M, int K, const float* ws, int rps,
                                     const int8_t* q, float sx, const float* bias, float* out, int row0, int gw,
                                     int nw) {
    const int lane = threadIdx.x & 31;
    const int rpw = (M + nw - 1) / nw;
    const int m0 = gw * rpw, m1 = min(M, m0 + rpw);
    for (int mb = m0; mb < m1; mb += PK_RB) {
        int acc[PK_RB];
#pragma unroll
        for (int r = 0; r < PK_RB; ++r) acc[r] = 0;
#pragma unroll 2   // K <= 1024: every chunk's loads issued together (one L2 round trip)
        for (int k = lane * 16; k < K; k += 512) {
            const int4 b = *reinterpret_cast<const int4*>(q + k);
            int4 wv[PK_RB];
#pragma unroll
            for (int r = 0; r < PK_RB; ++r)
                wv[r] = (mb + r < m1) ? __ldg(reinterpret_cast<const int4*>(W + (int64_t)(mb + r) * K + k))
                                      : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int r = 0; r < PK_RB; ++r) {
                acc[r] = __dp4a(wv[r].x, b.x, acc[r]);
                acc[r] = __dp4a(wv[r].y, b.y, acc[r]);
                acc[r] = __dp4a(wv[r].z, b.z, acc[r]);
                acc[r] = __dp4a(wv[r].w, b.w, acc[r]);
            }
        }
        int mine = 0;
#pragma unroll
        for (int r = 0; r < PK_RB; ++r) {
            const int tot = __reduce_add_sync(0xffffffffu, acc[r]);
            if (lane == r) mine = tot;
        }
        const int m = mb + lane;
        if (lane < PK_RB && m < m1) {
            const float sw = ws[m / rps];
            float y = dequant_rcp(mine, (1.0 / (double)sw) * (1.0 / (double)sx), sw, sx);   // == dequant()
            if (bias) y = __fadd_rn(y, bias[m]);
            out[row0 + m] = y;
        }
    }
}

// L1 prefetch of the weight rows this warp's gemv() will read in the next phase
// (same row distribution), issued before the grid barrier so the L2 latency of the
// first loads overlaps the barrier wait.
__device__ __forceinline__ void prefetch_rows(const int8_t* __restrict__ W, int M, int K, int gw, int nw) {
    const int lane = threadIdx.x & 31;
    const int rpw = (M + nw - 1) / nw;
    const int m0 = gw * rpw, m1 = min(M, m0 + rpw);
    if (m0 >= m1) return;
    const int64_t bytes = (int64_t)(m1 - m0) * K;
    const int8_t* base = W + (int64_t)m0 * K;
    for (int64_t o = (int64_t)lane * 128; o < bytes; o += 32 * 128)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(base + o));
}

#define PK_STAMP(k)                                                                 \
    if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) {                          \
        long long g_;                                                               \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                      \
        if ((k) < 11) a.stamps[(int64_t)t * 11 + (k)] = g_;                          \
    }

__global__ void __launch_bounds__(PK_T, 1) k_greedy1(PkArgs a) {
    unsigned gs_epoch = 0;   // grid-barrier target (gsync)
    extern __shared__ __align__(16) unsigned char pk_smem[];
    __shared__ __align__(16) int8_t q[PK_MAXD];
    __shared__ __align__(16) float vals[PK_MAXD];
    __shared__ uint32_t red[PK_W];
    __shared__ double dred[PK_W];
    __shared__ int sh_done;
    double* al = reinterpret_cast<double*>(pk_smem);   // [l] softmax weights
    const int E = a.E, H = a.H, A = a.A, R = a.R, V = a.V, LX = 3 * H + R;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * PK_W + warp, nw = gridDim.x * PK_W;
    double score = 0.0;   // live log-prob (CTA 0, thread 0)
    int y = 2;            // BOS = EOS (decoder.py:109); afterwards the token every CTA selected
    for (int t = 0; t < a.max_steps; ++t) {
        // ---- P0: q(emb[y]), q(s); GEMV [W_x2; W_e] and U_zr2 ----
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < E; j += PK_T) vals[j] = a.tgt_embed[(int64_t)y * E + j];
        __syncthreads();
        const float se = quantize_vec(vals, E, q, red, a.err);
        gemv(a.w2x, LX, E, a.w2x_s, 1, q, se, a.b2x, a.gxr, 0, gw, nw);
        __syncthreads();
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < H; j += PK_T) vals[j] = ldcg(a.s + j);
        __syncthreads();
        const float ss = quantize_vec(vals, H, q, red, a.err);
        gemv(a.uzr2, 2 * H, H, a.uzr2_s, H, q, ss, nullptr, a.gh, 0, gw, nw);
        prefetch_rows(a.uc2, H, H, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(0);
        // ---- P1: gates of dec_r -> q(r * s); GEMV U_c2 ----
        bool bad = false;
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < H; j += PK_T) {
            const float pz = __fadd_rn(ldcg(a.gxr + j), ldcg(a.gh + j));
            const float pr = __fadd_rn(ldcg(a.gxr + H + j), ldcg(a.gh + H + j));
            bad |= !(is_finite_f(pz) && is_finite_f(pr));
            vals[j] = __fmul_rn(sigmoid_b(pr), ldcg(a.s + j));
        }
        if (bad && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
        __syncthreads();
        const float srh = quantize_vec(vals, H, q, red, a.err);
        gemv(a.uc2, H, H, a.uc2_s, H, q, srh, nullptr, a.ghc, 0, gw, nw);
        prefetch_rows(a.wuq, A + 2 * H, H, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(1);
        // ---- P2: combine of dec_r -> s', q(s'); GEMV [U_att; U_zr3] ----
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < H; j += PK_T) {
            const float z = sigmoid_b(__fadd_rn(ldcg(a.gxr + j), ldcg(a.gh + j)));
            const float pc = __fadd_rn(ldcg(a.gxr + 2 * H + j), ldcg(a.ghc + j));
            if (!is_finite_f(pc) && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
            const float h = ldcg(a.s + j);
            const float v = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, z), h), __fmul_rn(z, tanh_b(pc)));
            vals[j] = v;
            if (blockIdx.x == 0) a.sp[j] = v;
        }
        __syncthreads();
        const float ssp = quantize_vec(vals, H, q, red, a.err);
        gemv(a.wuq, A + 2 * H, H, a.wuq_s, 1, q, ssp, nullptr, a.uq, 0, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(2);
        // ---- P3: attention scale (every CTA) and scores (one CTA per position) ----
        float st;
        {
            uint32_t m = 0;
            #pragma unroll 4   // independent iterations: their L2 loads in flight together
            for (int k = threadIdx.x; k < A; k += PK_T) {
                const float u = ldcg(a.uq + k);
                m = max(m, __float_as_uint(__fadd_rn(a.att_mm[k], u)) & 0x7fffffffu);
                m = max(m, __float_as_uint(__fadd_rn(a.att_mm[A + k], u)) & 0x7fffffffu);
            }
            m = block_max_u(m, red);
            if (m >= 0x7f800000u) {
                if (threadIdx.x == 0 && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
                m = 0;
            }
            const float tmax = tanh_b(__uint_as_float(m));
            st = (tmax == 0.0f) ? 1.0f : __fdiv_rn(127.0f, tmax);
        }
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int k = threadIdx.x; k < A; k += PK_T) vals[k] = ldcg(a.uq + k);
        __syncthreads();
        for (int i = blockIdx.x; i < a.l; i += gridDim.x) {
            int acc = 0;
            const float* ap = a.att + (int64_t)i * A;
            #pragma unroll 4   // independent iterations: their L2 loads in flight together
            for (int k = threadIdx.x; k < A; k += PK_T)
                acc += (int)a.v[k] * quant_code(tanh_b(__fadd_rn(ap[k], vals[k])), st);
            acc = warp_sum(acc);
            __shared__ int ired[PK_W];
            if (lane == 0) ired[warp] = acc;
            __syncthreads();
            if (threadIdx.x == 0) {
                int tot = 0;
                for (int w = 0; w < PK_W; ++w) tot += ired[w];
                a.scores[i] = dequant(tot, a.v_s[0], st);
            }
            __syncthreads();
        }
        gsync(a.ctl, gs_epoch);
        PK_STAMP(3);
        // ---- P4: softmax (every CTA, fp64, sequential sum) and context features ----
        {
            float m = -3.402823466e38f;
            bool bad4 = false;
            for (int i = threadIdx.x; i < a.l; i += PK_T) {
                const float x = ldcg(a.scores + i);
                bad4 |= !is_finite_f(x);
                m = fmaxf(m, x);
            }
            if (bad4 && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
            m = warp_max(m);
            if (lane == 0) vals[warp] = m;
            __syncthreads();
            float mm = vals[0];
            for (int w = 1; w < PK_W; ++w) mm = fmaxf(mm, vals[w]);
            for (int i = threadIdx.x; i < a.l; i += PK_T) {
                const double tt = (double)ldcg(a.scores + i) - (double)mm;
                al[i] = tt < -700.0 ? 0.0 : exp_f64(tt);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                double sum = 0.0;
                for (int i = 0; i < a.l; ++i) sum += al[i];
                dred[0] = sum;
            }
            __syncthreads();
            const double sum = dred[0];
            for (int i = threadIdx.x; i < a.l; i += PK_T) al[i] = (double)__double2float_rn(al[i] / sum);
            __syncthreads();
            // features spread over the CTAs (feature c: CTA c % grid); positions in order, 8 loads in flight
            for (int c = blockIdx.x + gridDim.x * threadIdx.x; c < 2 * H; c += gridDim.x * PK_T) {
                double acc = 0.0;
                const float* sp = a.states + c;
                int i = 0;
                for (; i + 8 <= a.l; i += 8) {
                    float d[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) d[u] = sp[(int64_t)(i + u) * 2 * H];
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc = fma((double)d[u], al[i + u], acc);
                }
                for (; i < a.l; ++i) acc = fma((double)sp[(int64_t)i * 2 * H], al[i], acc);
                a.ctx[c] = __double2float_rn(acc);
            }
        }
        prefetch_rows(a.w3x, LX, 2 * H, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(4);
        // ---- P5: q(ctx); GEMV [W_x3; W_c] ----
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < 2 * H; j += PK_T) vals[j] = ldcg(a.ctx + j);
        __syncthreads();
        const float sctx = quantize_vec(vals, 2 * H, q, red, a.err);
        gemv(a.w3x, LX, 2 * H, a.w3x_s, 1, q, sctx, a.b3x, a.gxq, 0, gw, nw);
        prefetch_rows(a.uc3, H, H, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(5);
        // ---- P6: gates of dec_q (h = s') -> q(r * s'); GEMV U_c3 ----
        bad = false;
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < H; j += PK_T) {
            const float pz = __fadd_rn(ldcg(a.gxq + j), ldcg(a.uq + A + j));
            const float pr = __fadd_rn(ldcg(a.gxq + H + j), ldcg(a.uq + A + H + j));
            bad |= !(is_finite_f(pz) && is_finite_f(pr));
            vals[j] = __fmul_rn(sigmoid_b(pr), ldcg(a.sp + j));
        }
        if (bad && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
        __syncthreads();
        const float srh3 = quantize_vec(vals, H, q, red, a.err);
        gemv(a.uc3, H, H, a.uc3_s, H, q, srh3, nullptr, a.ghc, 0, gw, nw);
        prefetch_rows(a.w_state, R, H, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(6);
        // ---- P7: combine of dec_q -> s_new (next state), q(s_new); GEMV W_s + b_r ----
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < H; j += PK_T) {
            const float z = sigmoid_b(__fadd_rn(ldcg(a.gxq + j), ldcg(a.uq + A + j)));
            const float pc = __fadd_rn(ldcg(a.gxq + 2 * H + j), ldcg(a.ghc + j));
            if (!is_finite_f(pc) && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
            const float h = ldcg(a.sp + j);
            const float v = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, z), h), __fmul_rn(z, tanh_b(pc)));
            vals[j] = v;
            if (blockIdx.x == 0) a.s[j] = v;   // every CTA read s for this step before the last barrier
        }
        __syncthreads();
        const float ssn = quantize_vec(vals, H, q, red, a.err);
        gemv(a.w_state, R, H, a.w_state_s, R, q, ssn, a.b_r, a.ro, 0, gw, nw);
        prefetch_rows(a.w_vocab, V, R, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(7);
        // ---- P8: readout tanh -> q; vocabulary GEMV (logits) ----
        #pragma unroll 4   // independent iterations: their L2 loads in flight together
        for (int j = threadIdx.x; j < R; j += PK_T) {
            const float x = __fadd_rn(__fadd_rn(ldcg(a.ro + j), ldcg(a.gxr + 3 * H + j)), ldcg(a.gxq + 3 * H + j));
            if (!is_finite_f(x) && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
            vals[j] = tanh_b(x);
        }
        __syncthreads();
        const float sro = quantize_vec(vals, R, q, red, a.err);
        gemv(a.w_vocab, V, R, a.w_vocab_s, V, q, sro, a.b_vocab, a.logits, 0, gw, nw);
        __threadfence_block();
        __syncthreads();   // P9 reads only the logits this CTA's warps just wrote: no grid barrier
        PK_STAMP(8);
        // ---- P9: per-CTA (max, sum exp(x - max)) over the CTA's own vocabulary GEMV rows ----
        const int per = PK_W * ((V + nw - 1) / nw);
        const int v0 = blockIdx.x * per, v1 = min(V, v0 + per);
        {
            float m = -3.402823466e38f;
            #pragma unroll 4   // independent iterations: their L2 loads in flight together
            for (int v = v0 + threadIdx.x; v < v1; v += PK_T) m = fmaxf(m, ldcg(a.logits + v));
            m = warp_max(m);
            if (lane == 0) vals[warp] = m;
            __syncthreads();
            float mm = vals[0];
            for (int w = 1; w < PK_W; ++w) mm = fmaxf(mm, vals[w]);
            double sacc = 0.0;
            #pragma unroll 4   // independent iterations: their L2 loads in flight together
            for (int v = v0 + threadIdx.x; v < v1; v += PK_T) {
                const float x = ldcg(a.logits + v);
                if (!is_finite_f(x)) set_flag(a.err, QNMT_FLAG_NUMERIC);
                const double tt = (double)x - (double)mm;
                sacc += tt < -700.0 ? 0.0 : exp_f64(tt);
            }
            sacc = warp_sum(sacc);
            if (lane == 0) dred[warp] = sacc;
            __syncthreads();
            if (threadIdx.x == 0) {
                double tot = 0.0;
                for (int w = 0; w < PK_W; ++w) tot += dred[w];
                a.part[2 * blockIdx.x] = v0 < v1 ? (double)mm : -1.0e308;
                a.part[2 * blockIdx.x + 1] = v0 < v1 ? tot : 0.0;
            }
        }
        prefetch_rows(a.w2x, LX, E, gw, nw);   // the next step's P0 (after P10 / P11, no barrier between)
        prefetch_rows(a.uzr2, 2 * H, H, gw, nw);
        gsync(a.ctl, gs_epoch);
        PK_STAMP(9);
        // ---- P10: lse (every CTA, same order); smallest token with the best log-prob ----
        // (thread c reads partial c; block tree reductions in a fixed order: every CTA gets the
        // same M and lse)
        double mc = -1.0e308, scv = 0.0;
        if (threadIdx.x < (int)gridDim.x) {
            mc = __ldcg(a.part + 2 * threadIdx.x);
            scv = __ldcg(a.part + 2 * threadIdx.x + 1);
        }
        double dM = mc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dM = fmax(dM, __shfl_xor_sync(0xffffffffu, dM, o));
        if (lane == 0) dred[warp] = dM;
        __syncthreads();
        dM = dred[0];
#pragma unroll
        for (int w = 1; w < PK_W; ++w) dM = fmax(dM, dred[w]);
        __syncthreads();
        double S = mc > -1.0e308 ? scv * exp_f64(mc - dM) : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
        if (lane == 0) dred[warp] = S;
        __syncthreads();
        S = dred[0];
#pragma unroll
        for (int w = 1; w < PK_W; ++w) S += dred[w];
        __syncthreads();
        const double lse = log(S);
        const float lp_best = __double2float_rn((dM - dM) - lse);
        // every CTA scans the whole vocabulary for the smallest token whose log-prob equals the best
        // one (logits more than 1.0 below the max cannot round to it): the next y is known everywhere
        // without another grid barrier
        {
            // a token whose log-prob rounds to the best one has a logit within 4 f32-ulps of lp_best
            // below M (as k_vocab_merge's tie rescan): only those CTAs' token ranges are scanned
            const int lex = (int)((__float_as_uint(lp_best) >> 23) & 0xffu);
            const double delta = ldexp(1.0, max(lex, 1) - 150 + 2);
            __shared__ int cand_cta[PK_T];
            __shared__ int ncand;
            if (threadIdx.x == 0) ncand = 0;
            __syncthreads();
            if (threadIdx.x < (int)gridDim.x && mc > -1.0e308 && mc >= dM - delta) cand_cta[atomicAdd(&ncand, 1)] = threadIdx.x;
            __syncthreads();
            int best = 0x7fffffff;
            for (int ci = 0; ci < ncand; ++ci) {
                const int c = cand_cta[ci];
                const int u0 = c * per, u1 = min(V, u0 + per);
                for (int v = u0 + threadIdx.x; v < u1; v += PK_T) {
                    const float x = ldcg(a.logits + v);
                    if ((double)x >= dM - delta && v < best && __double2float_rn(((double)x - dM) - lse) == lp_best)
                        best = v;
                }
            }
            best = __reduce_min_sync(0xffffffffu, best);
            if (lane == 0) red[warp] = (uint32_t)best;
            __syncthreads();
            best = (int)red[0];
#pragma unroll
            for (int w = 1; w < PK_W; ++w) best = min(best, (int)red[w]);
            __syncthreads();
            if (threadIdx.x == 0) sh_done = best;   // (reused as the CTA's token slot)
        }
        __syncthreads();
        const int tok = sh_done;
        __syncthreads();
        PK_STAMP(10);
        // ---- P11: search bookkeeping (decoder.py:112-155 at beam 1); every CTA knows tok ----
        const bool done = tok == 2 || t == a.max_steps - 1;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            score += (double)lp_best;
            if (tok == 2) {   // EOS: the only candidate goes to the finished list, no live hypothesis left
                a.fin_score[0] = score;
                a.fin_step[0] = t;
                a.fin_slot[0] = 0;
                a.fin_eos[0] = 1;
                *a.fin_cnt = 1;
            } else {
                a.hist_tok[(int64_t)t * a.hist_stride] = tok;
                a.hist_par[(int64_t)t * a.hist_stride] = 0;
                if (t == a.max_steps - 1) {   // length cap: the survivor is frozen (for-else)
                    a.fin_score[0] = score;
                    a.fin_step[0] = t;
                    a.fin_slot[0] = 0;
                    a.fin_eos[0] = 0;
                    *a.fin_cnt = 1;
                }
            }
        }
        y = tok;
        if (done) {
            if (a.step_dev && blockIdx.x == 0 && threadIdx.x == 0) *a.step_dev = t + 1;
            break;
        }
    }
}

int g_greedy1 = 1;

int greedy1_launch(const PkArgs& a, cudaStream_t st) {
    static int grid = 0;
    const size_t smem = (size_t)a.l * sizeof(double);
    if (smem > 48 * 1024) {
        static size_t done = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_greedy1, smem, done));
    }
    if (!grid) {
        int dev = 0, sms = 0, per_sm = 0;
        QNMT_CUDA(cudaGetDevice(&dev));
        QNMT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        QNMT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_greedy1, PK_T, smem));
        if (per_sm < 1) { set_error("greedy1: kernel does not fit on an SM"); return QNMT_ERR_CUDA; }
        grid = sms < PK_T ? sms : PK_T;   // P10 reads one vocabulary partial per thread
    }
    PkArgs args = a;
    void* params[] = {&args};
    QNMT_CUDA(cudaLaunchCooperativeKernel((const void*)k_greedy1, dim3(grid), dim3(PK_T), params, smem, st));
    count_launch();
    QNMT_CUDA(cudaGetLastError());
    return QNMT_OK;
}

// ---------------------------------------------------------------------------
// Batch-1 encoder recurrence: both directions advance together, one step per
// iteration: S1 q(h_d) -> GEMV U_zr_d; barrier; S2 gates -> q(r * h_d) -> GEMV
// U_c_d; barrier; S3 combine (every CTA keeps both h_d in shared memory, so the
// next step needs no barrier).  Same arithmetic as encode_core's per-step
// kernels (k_gru_gates / k_gru_combine, per-(sentence, direction) scales).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PK_T, 1) k_enc1(PeArgs a) {
    unsigned gs_epoch = 0;   // grid-barrier target (gsync)
    extern __shared__ __align__(16) unsigned char pe_smem[];
    const int H = a.H;
    float* h = reinterpret_cast<float*>(pe_smem);   // [2][H]
    float* zb = h + 2 * H;                          // [2][H]
    float* vals = zb + 2 * H;                       // [H]
    int8_t* q = reinterpret_cast<int8_t*>(vals + H);   // [2][H]
    __shared__ uint32_t red[PK_W];
    const int warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * PK_W + warp, nw = gridDim.x * PK_W;
    for (int j = threadIdx.x; j < 2 * H; j += PK_T) h[j] = 0.0f;   // layers.py:330
    __syncthreads();
    for (int t = 0; t < a.l; ++t) {
        const int pos[2] = {t, a.l - 1 - t};
        // S1: q(h_d) and U_zr_d q(h_d)
        float sh[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) sh[d] = quantize_vec(h + d * H, H, q + d * H, red, a.err);
#pragma unroll
        for (int d = 0; d < 2; ++d)
            gemv(a.uzr[d], 2 * H, H, a.uzr_s[d], H, q + d * H, sh[d], nullptr, a.gh + d * 2 * H, 0, gw, nw);
        gsync(a.ctl, gs_epoch);
        // S2: gates -> q(r * h_d) -> U_c_d
        float srh[2];
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            const float* gx = a.gx + ((int64_t)pos[d] * 2 + d) * 3 * H;
            bool bad = false;
            #pragma unroll 4   // independent iterations: their L2 loads in flight together
            for (int j = threadIdx.x; j < H; j += PK_T) {
                const float pz = __fadd_rn(gx[j], ldcg(a.gh + d * 2 * H + j));
                const float pr = __fadd_rn(gx[H + j], ldcg(a.gh + d * 2 * H + H + j));
                bad |= !(is_finite_f(pz) && is_finite_f(pr));
                zb[d * H + j] = sigmoid_b(pz);
                vals[j] = __fmul_rn(sigmoid_b(pr), h[d * H + j]);
            }
            if (bad && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
            __syncthreads();
            srh[d] = quantize_vec(vals, H, q + d * H, red, a.err);
        }
#pragma unroll
        for (int d = 0; d < 2; ++d)
            gemv(a.uc[d], H, H, a.uc_s[d], H, q + d * H, srh[d], nullptr, a.ghc + d * H, 0, gw, nw);
        gsync(a.ctl, gs_epoch);
        // S3: combine; the new states stay in this CTA's shared memory
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            const float* gx = a.gx + ((int64_t)pos[d] * 2 + d) * 3 * H + 2 * H;
            #pragma unroll 4   // independent iterations: their L2 loads in flight together
            for (int j = threadIdx.x; j < H; j += PK_T) {
                const float pc = __fadd_rn(gx[j], ldcg(a.ghc + d * H + j));
                if (!is_finite_f(pc) && blockIdx.x == 0) set_flag(a.err, QNMT_FLAG_NUMERIC);
                const float z = zb[d * H + j];
                const float v = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, z), h[d * H + j]), __fmul_rn(z, tanh_b(pc)));
                h[d * H + j] = v;
                if (blockIdx.x == 0) a.states[(int64_t)pos[d] * 2 * H + (d == 0 ? H : 0) + j] = v;
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0)
        for (int j = threadIdx.x; j < 2 * H; j += PK_T) a.h2[j] = h[j];
}

// ---------------------------------------------------------------------------
// k_enc1c: the batch-1 bidirectional recurrence with the recurrent weights
// RESIDENT IN SHARED MEMORY of one 16-CTA cluster per direction.  U_zr and U_c of
// one direction are 3 H^2 bytes (3 MB at H = 1024): 16 CTAs x 192 KB hold them,
// so a position costs two cluster barriers and two all-gathers of H floats
// through distributed shared memory, instead of two grid-wide barriers over all
// SMs plus 6 MB of L2 reads per position (k_enc1: ~19 us per position).
//
//   CTA r of direction d owns the hidden indices J = [r H/16, (r+1) H/16): the
//   z rows J and the r rows H + J of U_zr, the rows J of U_c (loaded once),
//   and a full copy of the state h.
//   S1  q(h) (every CTA); its 2|J| rows of U_zr q(h); z_J; v_J = r_J * h_J;
//       v_J stored into every CTA's `vals` (st.shared::cluster); cluster barrier
//   S2  q(v) (every CTA); its |J| rows of U_c q(v); h'_J = (1-z) h + z tanh(.);
//       h'_J stored into every CTA's h and the output; cluster barrier
//
// Same arithmetic as k_enc1 (quantize_vec, exact integer dots, dequant_rcp ==
// dequant, fp64 sigmoid / tanh rounded once), so the states are bit-identical.
// ---------------------------------------------------------------------------
constexpr int EC_CL = 16;    // CTAs per cluster
#ifndef QNMT_EC_T
#define QNMT_EC_T 512
#endif
constexpr int EC_T = QNMT_EC_T;    // threads per CTA
constexpr int EC_W = EC_T / 32;

__device__ __forceinline__ void ec_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ec_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// store v at the same shared-memory offset as `local` in every CTA of the cluster
__device__ __forceinline__ void ec_bcast(float* local, float v) {
    const uint32_t la = (uint32_t)__cvta_generic_to_shared(local);
#pragma unroll
    for (uint32_t c = 0; c < EC_CL; ++c) {
        uint32_t ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(c));
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
    }
}

// block max / quantization with EC_T threads (quantize_vec's arithmetic)
__device__ float ec_quantize(const float* vals, int D, int8_t* q, uint32_t* red, int32_t* err, bool lead) {
    uint32_t m = 0;
    for (int j = threadIdx.x; j < D; j += EC_T) m = max(m, __float_as_uint(vals[j]) & 0x7fffffffu);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    uint32_t mm = red[0];
#pragma unroll
    for (int w = 1; w < EC_W; ++w) mm = max(mm, red[w]);
    if (mm >= 0x7f800000u) {
        if (threadIdx.x == 0 && lead) set_flag(err, QNMT_FLAG_NUMERIC);
        mm = 0;
    }
    const float sc = scale_from_maxbits(mm);
    for (int j = threadIdx.x; j < D; j += EC_T) q[j] = (int8_t)quant_code(vals[j], sc);
    __syncthreads();
    return sc;
}

// rows [0, M) of a shared-memory weight block (row stride K) against q: out[m] =
// dequant(acc, ws[m / rows_per_scale], sx).  Warp w takes rows w, w + EC_W, ... in groups of 8.
__device__ __forceinline__ void ec_gemv(const int8_t* W, int M, int K, const float* ws, int rows_per_scale,
                                        const int8_t* q, float sx, float* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int mb = warp * 8; mb < M; mb += EC_W * 8) {
        int acc[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r] = 0;
        for (int k = lane * 16; k < K; k += 512) {
            const int4 b = *reinterpret_cast<const int4*>(q + k);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int4 wv = (mb + r < M) ? *reinterpret_cast<const int4*>(W + (size_t)(mb + r) * K + k)
                                             : make_int4(0, 0, 0, 0);
                acc[r] = __dp4a(wv.x, b.x, acc[r]);
                acc[r] = __dp4a(wv.y, b.y, acc[r]);
                acc[r] = __dp4a(wv.z, b.z, acc[r]);
                acc[r] = __dp4a(wv.w, b.w, acc[r]);
            }
        }
        int mine = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int tot = __reduce_add_sync(0xffffffffu, acc[r]);
            if (lane == r) mine = tot;
        }
        const int m = mb + lane;
        if (lane < 8 && m < M) {
            const float sw = ws[m / rows_per_scale];
            out[m] = dequant_rcp(mine, (1.0 / (double)sw) * (1.0 / (double)sx), sw, sx);   // == dequant()
        }
    }
}

__global__ void __launch_bounds__(EC_T, 1) k_enc1c(PeArgs a) {
    extern __shared__ __align__(16) unsigned char ec_smem[];
    const int H = a.H, J = H / EC_CL;
    const int d = blockIdx.x / EC_CL;           // cluster = direction
    const int r = (int)ec_rank();
    const int j0 = r * J;
    int8_t* wzr = reinterpret_cast<int8_t*>(ec_smem);       // [2J][H]: z rows J, then r rows J
    int8_t* wc = wzr + (size_t)2 * J * H;                   // [J][H]
    float* h = reinterpret_cast<float*>(wc + (size_t)J * H);   // [H] state (full copy)
    float* vals = h + H;                                    // [H] r * h (all-gathered)
    float* gloc = vals + H;                                 // [2J] this CTA's U_zr / U_c products
    float* zloc = gloc + 2 * J;                             // [J]
    int8_t* q = reinterpret_cast<int8_t*>(zloc + J);        // [H]
    __shared__ uint32_t red[EC_W];
    __shared__ float wsc[3];                                // z, r, c block scales of this direction
    // resident weights: this CTA's rows (16-byte chunks; H % 16 == 0)
    {
        const int cpr = H / 16;   // chunks per row
        const int4* gz = reinterpret_cast<const int4*>(a.uzr[d] + (size_t)j0 * H);
        const int4* gr = reinterpret_cast<const int4*>(a.uzr[d] + (size_t)(H + j0) * H);
        const int4* gc = reinterpret_cast<const int4*>(a.uc[d] + (size_t)j0 * H);
        int4* sz = reinterpret_cast<int4*>(wzr);
        int4* sr = reinterpret_cast<int4*>(wzr + (size_t)J * H);
        int4* sc = reinterpret_cast<int4*>(wc);
        for (int i = threadIdx.x; i < J * cpr; i += EC_T) {
            sz[i] = __ldg(gz + i);
            sr[i] = __ldg(gr + i);
            sc[i] = __ldg(gc + i);
        }
        if (threadIdx.x == 0) {
            wsc[0] = a.uzr_s[d][0];
            wsc[1] = a.uzr_s[d][1];
            wsc[2] = a.uc_s[d][0];
        }
    }
    for (int j = threadIdx.x; j < H; j += EC_T) h[j] = 0.0f;   // layers.py:330
    __syncthreads();
    ec_cluster_sync();   // every CTA's buffers exist before any remote store
    for (int t = 0; t < a.l; ++t) {
        const int pos = d == 0 ? t : a.l - 1 - t;
        const float* gx = a.gx + ((int64_t)pos * 2 + d) * 3 * H;
        // this position's input-side terms: requested first, consumed after the products (the L2
        // round trip overlaps the quantization and the dot products)
        float gx_zr = 0.0f, gx_c = 0.0f;
        if (threadIdx.x < 2 * J) gx_zr = threadIdx.x < J ? gx[j0 + threadIdx.x] : gx[H + j0 + threadIdx.x - J];
        if (threadIdx.x < J) gx_c = gx[2 * H + j0 + threadIdx.x];
        // S1: q(h), this CTA's rows of U_zr, gates of its indices
        const float sh = ec_quantize(h, H, q, red, a.err, r == 0);
        ec_gemv(wzr, 2 * J, H, wsc, J, q, sh, gloc);   // rows [0, J): z scale, [J, 2J): r scale
        __syncthreads();
        if (threadIdx.x < 2 * J) {   // one fp64 sigmoid chain per thread: z by threads [0, J), r by [J, 2J)
            const bool is_r = threadIdx.x >= J;
            const int jj = is_r ? threadIdx.x - J : threadIdx.x;
            const float p = __fadd_rn(gx_zr, gloc[threadIdx.x]);
            if (!is_finite_f(p)) set_flag(a.err, QNMT_FLAG_NUMERIC);
            const float sg = sigmoid_b(p);
            if (is_r)
                ec_bcast(vals + j0 + jj, __fmul_rn(sg, h[j0 + jj]));
            else
                zloc[jj] = sg;
        }
        ec_cluster_sync();   // vals complete in every CTA
        // S2: q(r * h), this CTA's rows of U_c, new state of its indices
        const float srh = ec_quantize(vals, H, q, red, a.err, r == 0);
        ec_gemv(wc, J, H, wsc + 2, J, q, srh, gloc);
        __syncthreads();
        if (threadIdx.x < J) {
            const int j = j0 + threadIdx.x;
            const float pc = __fadd_rn(gx_c, gloc[threadIdx.x]);
            if (!is_finite_f(pc)) set_flag(a.err, QNMT_FLAG_NUMERIC);
            const float z = zloc[threadIdx.x];
            const float v = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, z), h[j]), __fmul_rn(z, tanh_b(pc)));
            a.states[(int64_t)pos * 2 * H + (d == 0 ? H : 0) + j] = v;
            ec_bcast(h + j, v);   // peers read only their own slice of h after the S1 barrier
        }
        ec_cluster_sync();   // h complete in every CTA
    }
    if (threadIdx.x < J) a.h2[d * H + j0 + threadIdx.x] = h[j0 + threadIdx.x];
}

static size_t enc1c_smem(int H) {
    const size_t J = (size_t)H / EC_CL;
    return 3 * J * H + sizeof(float) * (2 * (size_t)H + 3 * J) + (size_t)H + 64;
}

// launches k_enc1c when the shape fits and two 16-CTA clusters can be resident; false = not used
static bool enc1c_try(const PeArgs& a, cudaStream_t st, int& rc) {
    rc = QNMT_OK;
    static const int enabled = [] {
        const char* v = getenv("QNMT_ENC1C");
        return v ? atoi(v) : 1;
    }();
    const int H = a.H;
    if (!enabled || H % 64 != 0 || 2 * (H / EC_CL) > EC_T) return false;   // J = H/16 rows per CTA, 16-byte aligned buffers
    const size_t smem = enc1c_smem(H);
    if (smem > 227 * 1024) return false;
    static int ready = 0;   // 0 unknown, 1 usable, -1 not usable
    static size_t smem_set = 0;
    if (ready < 0) return false;
    if (cudaFuncSetAttribute((const void*)k_enc1c, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        (smem > smem_set &&
         cudaFuncSetAttribute((const void*)k_enc1c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
             cudaSuccess)) {
        cudaGetLastError();
        ready = -1;
        return false;
    }
    smem_set = smem > smem_set ? smem : smem_set;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * EC_CL);
    cfg.blockDim = dim3(EC_T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = EC_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (ready == 0) {
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)k_enc1c, &cfg) != cudaSuccess || ncl < 2) {
            cudaGetLastError();
            ready = -1;
            return false;
        }
        ready = 1;
    }
    const cudaError_t le = cudaLaunchKernelEx(&cfg, k_enc1c, a);
    if (le != cudaSuccess) {
        rc = cuda_status(le, "k_enc1c");
        return true;
    }
    count_launch();
    return true;
}

int g_enc1 = 1;

int enc1_launch(const PeArgs& a, cudaStream_t st) {
    {   // preferred: weights resident in the shared memory of one cluster per direction
        int rc;
        if (enc1c_try(a, st, rc)) return rc;
    }
    const size_t smem = (size_t)a.H * (2 + 2 + 1) * sizeof(float) + 2 * (size_t)a.H;
    if (smem > 48 * 1024) {
        static size_t done = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_enc1, smem, done));
    }
    int dev = 0, sms = 0;
    QNMT_CUDA(cudaGetDevice(&dev));
    QNMT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PeArgs args = a;
    void* params[] = {&args};
    QNMT_CUDA(cudaLaunchCooperativeKernel((const void*)k_enc1, dim3(sms), dim3(PK_T), params, smem, st));
    count_launch();
    QNMT_CUDA(cudaGetLastError());
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" int qnmt_set_greedy1(int enable) {
    const int old = qnmt::g_greedy1;
    qnmt::g_greedy1 = enable;
    qnmt::g_enc1 = enable;
    return old;
}
