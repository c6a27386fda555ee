// fused_q.cu -- decoder elementwise ops fused with the quantization of their
// output, one CTA per quantization segment.
//
// In the batched decoder a quantization segment is one sentence: the columns
// [off[s], off[s] + cnt[s]) of all its live hypotheses (LinearOp.apply on the
// sentence's [features, P] block, layers.py:118-146).  A CTA that owns the whole
// segment can compute the op, reduce max|v| (qmath.py:157-169), derive the scale
// (qmath.py:136-142) and write the int8 codes (qmath.py:119-133) in one launch,
// instead of op + max-abs pass + encode pass.  Values wait in shared memory
// ([cnt][D] f32) between the reduction and the encode.
//
//   k_gates_q    z, q(r*h)        GRU first phase      (layers.py:170-176)
//   k_combine_q  h', q(h')        GRU second phase     (layers.py:177-181)
//   k_embed_q    q(E[y])          target embedding     (layers.py:367)
//   k_tanh_q     q(tanh(x))       readout activation   (layers.py:265)
//   k_gather_q   s, s', q(s), q(s') next-step states by parent column (decoder.py:131-140)
#include "kernels.cuh"
#include "search.cuh"

namespace qnmt {

constexpr int FQ_T = 640;    // threads per segment CTA: 5 x 1024 / 4 = 1280 float4 groups -> 2 per thread at beam 5, 2 CTAs / SM

// block max of |v| bits -> scale of the segment (non-finite: flag, scale 1 as k_encode)
__device__ __forceinline__ float seg_scale(uint32_t m, uint32_t* red, int32_t* err_flag, float* sc_out) {
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    uint32_t mm = 0;
#pragma unroll
    for (int w = 0; w < FQ_T / 32; ++w) mm = max(mm, red[w]);
    if (mm >= 0x7f800000u) {
        if (threadIdx.x == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);
        mm = 0;
    }
    const float sc = scale_from_maxbits(mm);
    if (threadIdx.x == 0 && sc_out) *sc_out = sc;
    return sc;
}

__device__ __forceinline__ uint32_t absbits(float v) { return __float_as_uint(v) & 0x7fffffffu; }

// Elements are processed in groups of 4 consecutive features of one column
// (D % 4 == 0 and 16-byte aligned rows, checked by the engine): group g of the
// flattened [P][D] segment is column (4g) / D, features 4g % D .. +3.
__device__ __forceinline__ void seg_encode(const float* vals, int P, int64_t D, int c0, float sc, int8_t* q,
                                           int64_t ldq) {
    const int64_t G = (int64_t)P * D / 4;
#pragma unroll 4
    for (int64_t g = threadIdx.x; g < G; g += FQ_T) {
        const int64_t c = (4 * g) / D, j = 4 * g - c * D;
        const float4 v = *reinterpret_cast<const float4*>(vals + 4 * g);
        const uint32_t packed = (uint32_t)(quant_code(v.x, sc) & 0xff) | ((uint32_t)(quant_code(v.y, sc) & 0xff) << 8) |
                                ((uint32_t)(quant_code(v.z, sc) & 0xff) << 16) |
                                ((uint32_t)(quant_code(v.w, sc) & 0xff) << 24);
        *reinterpret_cast<uint32_t*>(q + (int64_t)(c0 + c) * ldq + j) = packed;
    }
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ uint32_t max4(uint32_t m, float4 v) {
    return max(max(m, max(absbits(v.x), absbits(v.y))), max(absbits(v.z), absbits(v.w)));
}
__device__ __forceinline__ bool fin4(float4 v) {
    return is_finite_f(v.x) && is_finite_f(v.y) && is_finite_f(v.z) && is_finite_f(v.w);
}

#define FQ_SEG_PROLOGUE                                                  \
    extern __shared__ float vals[];                                      \
    __shared__ uint32_t red[FQ_T / 32];                                  \
    const int s = blockIdx.x;                                            \
    const int P = cnt[s];                                                \
    if (P == 0) return;                                                  \
    if (P > max_cols) { /* more columns than smem was sized for */       \
        if (threadIdx.x == 0) set_flag(err_flag, QNMT_FLAG_INVALID);     \
        return;                                                          \
    }                                                                    \
    const int c0 = off[s];

__global__ void __launch_bounds__(FQ_T, 2)
k_gates_q(const float* __restrict__ gx, int64_t ldgx, const float* __restrict__ gh, int64_t ldgh,
          const float* __restrict__ h, int64_t ldh, int64_t H, const int32_t* __restrict__ off,
          const int32_t* __restrict__ cnt, float* __restrict__ z, int8_t* __restrict__ q_rh, float* sc_rh,
          int32_t* err_flag, int max_cols) {
    pdl_entry();
    FQ_SEG_PROLOGUE
    uint32_t m = 0;
    bool bad = false;
    const int64_t G = (int64_t)P * H / 4;
#pragma unroll 2
    for (int64_t g = threadIdx.x; g < G; g += FQ_T) {
        const int64_t c = (4 * g) / H, j = 4 * g - c * H, n = c0 + c;
        const float4 xz = ld4(gx + n * ldgx + j), xr = ld4(gx + n * ldgx + H + j);
        const float4 hz = ld4(gh + n * ldgh + j), hr = ld4(gh + n * ldgh + H + j);
        const float4 hh = ld4(h + n * ldh + j);
        const float4 pz = make_float4(__fadd_rn(xz.x, hz.x), __fadd_rn(xz.y, hz.y), __fadd_rn(xz.z, hz.z),
                                      __fadd_rn(xz.w, hz.w));
        const float4 pr = make_float4(__fadd_rn(xr.x, hr.x), __fadd_rn(xr.y, hr.y), __fadd_rn(xr.z, hr.z),
                                      __fadd_rn(xr.w, hr.w));
        bad |= !fin4(pz) || !fin4(pr);
        st4(z + n * H + j, make_float4(sigmoid_b(pz.x), sigmoid_b(pz.y), sigmoid_b(pz.z), sigmoid_b(pz.w)));
        const float4 v = make_float4(__fmul_rn(sigmoid_b(pr.x), hh.x), __fmul_rn(sigmoid_b(pr.y), hh.y),
                                     __fmul_rn(sigmoid_b(pr.z), hh.z), __fmul_rn(sigmoid_b(pr.w), hh.w));
        st4(vals + 4 * g, v);
        m = max4(m, v);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    const float sc = seg_scale(m, red, err_flag, sc_rh + s);
    seg_encode(vals, P, H, c0, sc, q_rh, H);
}

__global__ void __launch_bounds__(FQ_T, 2)
k_combine_q(const float* __restrict__ gxc, int64_t ldgx, const float* __restrict__ ghc, int64_t ldghc,
            const float* __restrict__ z, const float* __restrict__ h, int64_t ldh, int64_t H,
            const int32_t* __restrict__ off, const int32_t* __restrict__ cnt, float* __restrict__ h_out,
            int64_t ldo, int8_t* __restrict__ q_out, float* sc_out, int32_t* err_flag, int max_cols) {
    pdl_entry();
    FQ_SEG_PROLOGUE
    uint32_t m = 0;
    bool bad = false;
    const int64_t G = (int64_t)P * H / 4;
#pragma unroll 2
    for (int64_t g = threadIdx.x; g < G; g += FQ_T) {
        const int64_t c = (4 * g) / H, j = 4 * g - c * H, n = c0 + c;
        const float4 xc = ld4(gxc + n * ldgx + j), hc = ld4(ghc + n * ldghc + j);
        const float4 zz = ld4(z + n * H + j), hh = ld4(h + n * ldh + j);
        const float4 pc = make_float4(__fadd_rn(xc.x, hc.x), __fadd_rn(xc.y, hc.y), __fadd_rn(xc.z, hc.z),
                                      __fadd_rn(xc.w, hc.w));
        bad |= !fin4(pc);
        float4 v;
        v.x = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.x), hh.x), __fmul_rn(zz.x, tanh_b(pc.x)));
        v.y = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.y), hh.y), __fmul_rn(zz.y, tanh_b(pc.y)));
        v.z = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.z), hh.z), __fmul_rn(zz.z, tanh_b(pc.z)));
        v.w = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.w), hh.w), __fmul_rn(zz.w, tanh_b(pc.w)));
        st4(h_out + n * ldo + j, v);
        st4(vals + 4 * g, v);
        m = max4(m, v);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    const float sc = seg_scale(m, red, err_flag, sc_out + s);
    seg_encode(vals, P, H, c0, sc, q_out, H);
}

__global__ void __launch_bounds__(FQ_T, 2)
k_embed_q(const float* __restrict__ table, int64_t rows, int64_t E, const int32_t* __restrict__ ids,
          const int32_t* __restrict__ off, const int32_t* __restrict__ cnt, int8_t* __restrict__ q_out,
          float* sc_out, int32_t* err_flag, int max_cols, uint32_t* zero4, int zstride) {
    pdl_entry();
    // first kernel of a decoder step: clear this sentence's four GRU-epilogue maxima (engine.cu gmax)
    if (zero4 && threadIdx.x < 4) zero4[(size_t)threadIdx.x * zstride + blockIdx.x] = 0u;
    FQ_SEG_PROLOGUE
    uint32_t m = 0;
    const int64_t G = (int64_t)P * E / 4;
#pragma unroll 2
    for (int64_t g = threadIdx.x; g < G; g += FQ_T) {
        const int64_t c = (4 * g) / E, j = 4 * g - c * E;
        const int32_t id = ids[c0 + c];
        const bool ok = id >= 0 && id < rows;
        if (!ok && j == 0) set_flag(err_flag, QNMT_FLAG_VOCAB);
        const float4 v = ok ? ld4(table + (int64_t)id * E + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        st4(vals + 4 * g, v);
        m = max4(m, v);
    }
    const float sc = seg_scale(m, red, err_flag, sc_out + s);
    seg_encode(vals, P, E, c0, sc, q_out, E);
}

__global__ void __launch_bounds__(FQ_T, 2)
k_tanh_q(const float* __restrict__ x, int64_t ldx, int64_t D, const int32_t* __restrict__ off,
         const int32_t* __restrict__ cnt, int8_t* __restrict__ q_out, float* sc_out, int32_t* err_flag,
         int max_cols, const float* __restrict__ a1, int64_t ld1, const float* __restrict__ a2, int64_t ld2) {
    pdl_entry();
    FQ_SEG_PROLOGUE
    uint32_t m = 0;
    bool bad = false;
    const int64_t G = (int64_t)P * D / 4;
#pragma unroll 2
    for (int64_t g = threadIdx.x; g < G; g += FQ_T) {
        const int64_t c = (4 * g) / D, j = 4 * g - c * D;
        float4 xv = ld4(x + (int64_t)(c0 + c) * ldx + j);
        if (a1) {   // readout terms of stacked GEMMs: ((W_s s + b_r) + W_e e) + W_c c (layers.py:255-265)
            const float4 u = ld4(a1 + (int64_t)(c0 + c) * ld1 + j), w = ld4(a2 + (int64_t)(c0 + c) * ld2 + j);
            xv = make_float4(__fadd_rn(__fadd_rn(xv.x, u.x), w.x), __fadd_rn(__fadd_rn(xv.y, u.y), w.y),
                             __fadd_rn(__fadd_rn(xv.z, u.z), w.z), __fadd_rn(__fadd_rn(xv.w, u.w), w.w));
        }
        bad |= !fin4(xv);
        const float4 v = make_float4(tanh_b(xv.x), tanh_b(xv.y), tanh_b(xv.z), tanh_b(xv.w));
        st4(vals + 4 * g, v);
        m = max4(m, v);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    const float sc = seg_scale(m, red, err_flag, sc_out + s);
    seg_encode(vals, P, D, c0, sc, q_out, D);
}

// a_out[n] = a[parent[n]] (+ codes qa); optionally the same for b (second state)
__global__ void __launch_bounds__(FQ_T, 2)
k_gather_q(const float* __restrict__ a, const float* __restrict__ b, const int32_t* __restrict__ parent,
           int64_t H, const int32_t* __restrict__ off, const int32_t* __restrict__ cnt, float* __restrict__ a_out,
           float* __restrict__ b_out, int8_t* __restrict__ qa, float* sca, int8_t* __restrict__ qb, float* scb,
           int32_t* err_flag, int max_cols) {
    pdl_entry();
    FQ_SEG_PROLOGUE
    float* va = vals;                    // [P][H]
    float* vb = vals + (int64_t)P * H;   // [P][H]
    uint32_t ma = 0, mb = 0;
    const int64_t G = (int64_t)P * H / 4;
#pragma unroll 2
    for (int64_t g = threadIdx.x; g < G; g += FQ_T) {
        const int64_t c = (4 * g) / H, j = 4 * g - c * H, n = c0 + c;
        const int64_t p = parent[n];
        const float4 xa = ld4(a + p * H + j);
        st4(a_out + n * H + j, xa);
        st4(va + 4 * g, xa);
        ma = max4(ma, xa);
        if (b) {
            const float4 xb = ld4(b + p * H + j);
            st4(b_out + n * H + j, xb);
            st4(vb + 4 * g, xb);
            mb = max4(mb, xb);
        }
    }
    const float sa = seg_scale(ma, red, err_flag, sca + s);
    seg_encode(va, P, H, c0, sa, qa, H);
    if (qb) {
        __syncthreads();   // red reused
        const float sb = seg_scale(mb, red, err_flag, scb + s);
        seg_encode(vb, P, H, c0, sb, qb, H);
    }
}


// ---------------------------------------------------------------------------
// Encoder steps (layers.py:331-340, batched over sentences and directions): a
// quantization segment is ONE column (sentence, direction), so one CTA per
// column computes the GRU phase, reduces max |v| and writes the codes the next
// product reads -- instead of the phase kernel, an atomicMax pass and an encode
// launch.  gx rows go through the per-step row map (position of the column's
// sentence at this step); combine also scatters the new state to `states`.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(FQ_T, 2)
k_enc_gates_q(const float* __restrict__ gx, int64_t ldgx, const int32_t* __restrict__ gx_row,
              const float* __restrict__ gh, int64_t ldgh, const float* __restrict__ h, int64_t ldh, int64_t H,
              float* __restrict__ z, int8_t* __restrict__ q_rh, float* sc_rh, int32_t* err_flag) {
    pdl_entry();
    extern __shared__ float vals[];
    __shared__ uint32_t red[FQ_T / 32];
    const int64_t n = blockIdx.x;
    const float* gxr = gx + (int64_t)gx_row[n] * ldgx;
    uint32_t m = 0;
    bool bad = false;
    for (int64_t g = threadIdx.x; g < H / 4; g += FQ_T) {
        const int64_t j = 4 * g;
        const float4 xz = ld4(gxr + j), xr = ld4(gxr + H + j);
        const float4 hz = ld4(gh + n * ldgh + j), hr = ld4(gh + n * ldgh + H + j);
        const float4 hh = ld4(h + n * ldh + j);
        const float4 pz = make_float4(__fadd_rn(xz.x, hz.x), __fadd_rn(xz.y, hz.y), __fadd_rn(xz.z, hz.z),
                                      __fadd_rn(xz.w, hz.w));
        const float4 pr = make_float4(__fadd_rn(xr.x, hr.x), __fadd_rn(xr.y, hr.y), __fadd_rn(xr.z, hr.z),
                                      __fadd_rn(xr.w, hr.w));
        bad |= !fin4(pz) || !fin4(pr);
        st4(z + n * H + j, make_float4(sigmoid_b(pz.x), sigmoid_b(pz.y), sigmoid_b(pz.z), sigmoid_b(pz.w)));
        const float4 v = make_float4(__fmul_rn(sigmoid_b(pr.x), hh.x), __fmul_rn(sigmoid_b(pr.y), hh.y),
                                     __fmul_rn(sigmoid_b(pr.z), hh.z), __fmul_rn(sigmoid_b(pr.w), hh.w));
        st4(vals + j, v);
        m = max4(m, v);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    const float sc = seg_scale(m, red, err_flag, sc_rh + n);
    seg_encode(vals, 1, H, (int)n, sc, q_rh, H);
}

__global__ void __launch_bounds__(FQ_T, 2)
k_enc_combine_q(const float* __restrict__ gx, int64_t ldgx, const int32_t* __restrict__ gx_row,
                const float* __restrict__ ghc, int64_t ldghc, const float* __restrict__ z, float* __restrict__ h,
                int64_t ldh, int64_t H, float* __restrict__ states, int64_t lds, const int32_t* __restrict__ out_row,
                int8_t* __restrict__ q_h, float* sc_h, int32_t* err_flag) {
    pdl_entry();
    extern __shared__ float vals[];
    __shared__ uint32_t red[FQ_T / 32];
    const int64_t n = blockIdx.x;
    const float* gxc = gx + (int64_t)gx_row[n] * ldgx + 2 * H;
    float* so = states + (int64_t)out_row[n] * lds;
    uint32_t m = 0;
    bool bad = false;
    for (int64_t g = threadIdx.x; g < H / 4; g += FQ_T) {
        const int64_t j = 4 * g;
        const float4 xc = ld4(gxc + j), hc = ld4(ghc + n * ldghc + j);
        const float4 zz = ld4(z + n * H + j), hh = ld4(h + n * ldh + j);
        const float4 pc = make_float4(__fadd_rn(xc.x, hc.x), __fadd_rn(xc.y, hc.y), __fadd_rn(xc.z, hc.z),
                                      __fadd_rn(xc.w, hc.w));
        bad |= !fin4(pc);
        float4 v;
        v.x = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.x), hh.x), __fmul_rn(zz.x, tanh_b(pc.x)));
        v.y = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.y), hh.y), __fmul_rn(zz.y, tanh_b(pc.y)));
        v.z = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.z), hh.z), __fmul_rn(zz.z, tanh_b(pc.z)));
        v.w = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz.w), hh.w), __fmul_rn(zz.w, tanh_b(pc.w)));
        st4(h + n * ldh + j, v);   // (this thread read these four before)
        st4(so + j, v);
        st4(vals + j, v);
        m = max4(m, v);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    const float sc = seg_scale(m, red, err_flag, sc_h + n);
    seg_encode(vals, 1, H, (int)n, sc, q_h, H);
}

// ---------------------------------------------------------------------------
// k_layout_gather_q: k_search_layout (search.cu) + k_gather_q in one launch, one
// CTA per sentence.  The next step's column offset of sentence s is the sum of
// the live selections of the sentences before it -- every CTA sums the
// per-sentence counts itself (<= 1024 ints) instead of waiting for a one-CTA
// prefix-sum kernel; it then writes the layout of its own columns (sentence,
// parent column, token, live score) and gathers / quantizes their states by
// parent.  CTA 0 publishes the live column count and advances the step counter.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(FQ_T, 2)
k_layout_gather_q(SearchState ss, int step, int n_sent, int k_list, const float* __restrict__ a,
                  const float* __restrict__ b, int64_t H, float* __restrict__ a_out, float* __restrict__ b_out,
                  int8_t* __restrict__ qa, float* sca, int8_t* __restrict__ qb, float* scb, int32_t* err_flag,
                  int max_cols) {
    pdl_entry();
    extern __shared__ float vals[];
    __shared__ uint32_t red[FQ_T / 32];
    __shared__ int psum[2][FQ_T / 32];
    __shared__ int s_parent[16];
    const int s = blockIdx.x;
    int before = 0, total = 0;
    for (int i = threadIdx.x; i < n_sent; i += FQ_T) {
        const int v = ss.np_tmp[i];
        total += v;
        before += i < s ? v : 0;
    }
    before = __reduce_add_sync(0xffffffffu, before);
    total = __reduce_add_sync(0xffffffffu, total);
    if ((threadIdx.x & 31) == 0) {
        psum[0][threadIdx.x >> 5] = before;
        psum[1][threadIdx.x >> 5] = total;
    }
    __syncthreads();
    before = total = 0;
#pragma unroll
    for (int w = 0; w < FQ_T / 32; ++w) {
        before += psum[0][w];
        total += psum[1][w];
    }
    const int P = ss.np_tmp[s];
    const int c0 = before;
    const int old_off = ss.col_off[s];
    if (threadIdx.x < P && threadIdx.x < 16) {   // layout of this sentence's next-step columns
        const int64_t idx = (int64_t)old_off * k_list + threadIdx.x;
        const int v = ss.cand_tok[idx];
        const int n = c0 + threadIdx.x;
        const int pc = old_off + (v >> 26);
        ss.col_sent_next[n] = s;
        ss.parent_col[n] = pc;
        s_parent[threadIdx.x] = pc;
        ss.y_next[n] = v & ((1 << 26) - 1);
        ss.live_next[n] = ss.cand_score[idx];
    }
    __syncthreads();   // old_off read by every thread; s_parent visible
    if (threadIdx.x == 0) {
        ss.P[s] = P;
        ss.col_off[s] = c0;
        if (s == 0) {
            *ss.n_live = total;
            if (ss.step_dev) *ss.step_dev = *ss.step_dev + 1;
        }
    }
    if (P == 0) return;
    if (P > max_cols) {
        if (threadIdx.x == 0) set_flag(err_flag, QNMT_FLAG_INVALID);
        return;
    }
    float* va = vals;                    // [P][H]
    float* vb = vals + (int64_t)P * H;   // [P][H]
    uint32_t ma = 0, mb = 0;
    const int64_t G = (int64_t)P * H / 4;
#pragma unroll 2
    for (int64_t g = threadIdx.x; g < G; g += FQ_T) {
        const int64_t c = (4 * g) / H, j = 4 * g - c * H, n = c0 + c;
        const int64_t p = s_parent[c];
        const float4 xa = ld4(a + p * H + j);
        st4(a_out + n * H + j, xa);
        st4(va + 4 * g, xa);
        ma = max4(ma, xa);
        if (b) {
            const float4 xb = ld4(b + p * H + j);
            st4(b_out + n * H + j, xb);
            st4(vb + 4 * g, xb);
            mb = max4(mb, xb);
        }
    }
    const float sa = seg_scale(ma, red, err_flag, sca + s);
    seg_encode(va, P, H, c0, sa, qa, H);
    if (qb) {
        __syncthreads();   // red reused
        const float sb = seg_scale(mb, red, err_flag, scb + s);
        seg_encode(vb, P, H, c0, sb, qb, H);
    }
}

static int set_smem(const void* fn, size_t bytes, size_t& done) {
    if (bytes > FQ_SMEM_MAX) {
        set_error("fused quantize: %zu bytes of segment values exceed shared memory", bytes);
        return QNMT_ERR_CONFIG;
    }
    if (bytes > 48 * 1024) QNMT_CUDA(raise_smem_limit(fn, bytes, done));
    return QNMT_OK;
}

#define FQ_TRY(x) do { int _r = (x); if (_r != QNMT_OK) return _r; } while (0)

int gates_q_launch(const float* gx, int64_t ldgx, const float* gh, int64_t ldgh, const float* h, int64_t ldh,
                   int64_t H, const int32_t* off, const int32_t* cnt, int n_seg, int max_cols, float* z,
                   int8_t* q_rh, float* sc_rh, int32_t* err_flag, cudaStream_t st) {
    if (n_seg <= 0) return QNMT_OK;
    const size_t smem = (size_t)max_cols * H * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_gates_q, smem, done));
    QNMT_LAUNCH(k_gates_q, (unsigned)n_seg, FQ_T, smem, st, gx, ldgx, gh, ldgh, h, ldh, H, off, cnt, z, q_rh, sc_rh,
                                                    err_flag, max_cols);
    QNMT_CHECK_LAUNCH("k_gates_q");
    return QNMT_OK;
}

int combine_q_launch(const float* gxc, int64_t ldgx, const float* ghc, int64_t ldghc, const float* z,
                     const float* h, int64_t ldh, int64_t H, const int32_t* off, const int32_t* cnt, int n_seg,
                     int max_cols, float* h_out, int64_t ldo, int8_t* q_out, float* sc_out, int32_t* err_flag,
                     cudaStream_t st) {
    if (n_seg <= 0) return QNMT_OK;
    const size_t smem = (size_t)max_cols * H * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_combine_q, smem, done));
    QNMT_LAUNCH(k_combine_q, (unsigned)n_seg, FQ_T, smem, st, gxc, ldgx, ghc, ldghc, z, h, ldh, H, off, cnt, h_out, ldo,
                                                      q_out, sc_out, err_flag, max_cols);
    QNMT_CHECK_LAUNCH("k_combine_q");
    return QNMT_OK;
}

int enc_gates_q_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* gh, int64_t ldgh,
                       const float* h, int64_t ldh, int64_t ncols, int64_t H, float* z, int8_t* q_rh, float* sc_rh,
                       int32_t* err_flag, cudaStream_t st) {
    if (ncols <= 0) return QNMT_OK;
    const size_t smem = (size_t)H * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_enc_gates_q, smem, done));
    QNMT_LAUNCH(k_enc_gates_q, (unsigned)ncols, FQ_T, smem, st, gx, ldgx, gx_row, gh, ldgh, h, ldh, H, z, q_rh, sc_rh,
                err_flag);
    QNMT_CHECK_LAUNCH("k_enc_gates_q");
    return QNMT_OK;
}

int enc_combine_q_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* ghc, int64_t ldghc,
                         const float* z, float* h, int64_t ldh, int64_t ncols, int64_t H, float* states, int64_t lds,
                         const int32_t* out_row, int8_t* q_h, float* sc_h, int32_t* err_flag, cudaStream_t st) {
    if (ncols <= 0) return QNMT_OK;
    const size_t smem = (size_t)H * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_enc_combine_q, smem, done));
    QNMT_LAUNCH(k_enc_combine_q, (unsigned)ncols, FQ_T, smem, st, gx, ldgx, gx_row, ghc, ldghc, z, h, ldh, H, states,
                lds, out_row, q_h, sc_h, err_flag);
    QNMT_CHECK_LAUNCH("k_enc_combine_q");
    return QNMT_OK;
}

int layout_gather_q_launch(const SearchState& ss, int n_sent, int beam, int k_list, const float* a, const float* b,
                           int64_t H, float* a_out, float* b_out, int8_t* qa, float* sca, int8_t* qb, float* scb,
                           int32_t* err_flag, cudaStream_t st) {
    if (n_sent <= 0) return QNMT_OK;
    if (!ss.np_tmp || !ss.step_dev || beam > 16 || k_list > 16) {
        set_error("layout_gather_q: needs the graph-mode search state (np_tmp, step_dev), beam <= 16");
        return QNMT_ERR_CONFIG;
    }
    const size_t smem = (size_t)2 * beam * H * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_layout_gather_q, smem, done));
    QNMT_LAUNCH(k_layout_gather_q, (unsigned)n_sent, FQ_T, smem, st, ss, 0, n_sent, k_list, a, b, H, a_out, b_out, qa,
                sca, qb, scb, err_flag, beam);
    QNMT_CHECK_LAUNCH("k_layout_gather_q");
    return QNMT_OK;
}

int embed_q_launch(const float* table, int64_t rows, int64_t E, const int32_t* ids, const int32_t* off,
                   const int32_t* cnt, int n_seg, int max_cols, int8_t* q_out, float* sc_out, int32_t* err_flag,
                   cudaStream_t st, uint32_t* zero4, int zstride) {
    if (n_seg <= 0) return QNMT_OK;
    const size_t smem = (size_t)max_cols * E * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_embed_q, smem, done));
    QNMT_LAUNCH(k_embed_q, (unsigned)n_seg, FQ_T, smem, st, table, rows, E, ids, off, cnt, q_out, sc_out, err_flag, max_cols,
                zero4, zstride);
    QNMT_CHECK_LAUNCH("k_embed_q");
    return QNMT_OK;
}

int tanh_q_launch(const float* x, int64_t ldx, int64_t D, const int32_t* off, const int32_t* cnt, int n_seg,
                  int max_cols, int8_t* q_out, float* sc_out, int32_t* err_flag, cudaStream_t st, const float* a1,
                  int64_t ld1, const float* a2, int64_t ld2) {
    if (n_seg <= 0) return QNMT_OK;
    const size_t smem = (size_t)max_cols * D * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_tanh_q, smem, done));
    QNMT_LAUNCH(k_tanh_q, (unsigned)n_seg, FQ_T, smem, st, x, ldx, D, off, cnt, q_out, sc_out, err_flag, max_cols, a1,
                ld1, a2, ld2);
    QNMT_CHECK_LAUNCH("k_tanh_q");
    return QNMT_OK;
}

int gather_q_launch(const float* a, const float* b, const int32_t* parent, int64_t H, const int32_t* off,
                    const int32_t* cnt, int n_seg, int max_cols, float* a_out, float* b_out, int8_t* qa,
                    float* sca, int8_t* qb, float* scb, int32_t* err_flag, cudaStream_t st) {
    if (n_seg <= 0) return QNMT_OK;
    const size_t smem = (size_t)2 * max_cols * H * sizeof(float);
    static size_t done = 0;
    FQ_TRY(set_smem((const void*)k_gather_q, smem, done));
    QNMT_LAUNCH(k_gather_q, (unsigned)n_seg, FQ_T, smem, st, a, b, parent, H, off, cnt, a_out, b_out, qa, sca, qb, scb,
                                                     err_flag, max_cols);
    QNMT_CHECK_LAUNCH("k_gather_q");
    return QNMT_OK;
}

}  // namespace qnmt
