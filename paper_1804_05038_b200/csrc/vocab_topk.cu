// vocab_topk.cu -- vocabulary projection fused with the log-softmax statistics
// and the beam candidates: the [N][V] logits never touch HBM.
//
// Same numbers as gemm (layers.py:266, W_vocab . q(readout) + b) followed by
// topk_launch (output.cu: layers.py:60-67 + decoder.py:125/:74-85):
//   x[n][v]  = fl32(fl32(acc / (s_w * s_x)) + b[v])             exact dequant
//   lp[n][v] = fl32((f64 x - f64 max_n) - log(sum_v exp(f64 x - f64 max_n)))
//   cand     = top-k of (live[n] + f64 lp, token asc)
//
// K5a k_vocab_stats: the tcgen05 main loop (tc_mainloop.cuh) with the roles
//   swapped -- A = activations (TMEM lane = hypothesis row), B = W_vocab (TMEM
//   column = token) -- so every epilogue thread owns one hypothesis row and a
//   128-token half-tile.  Per (row, tile, half) it keeps an online (max, sum
//   exp) in fp64, the token of the max (smallest on ties) and the runner-up
//   value, and writes one 24-byte partial.  Traffic: 24 B per 128 logits
//   instead of 512 B written + 512 B re-read.
// K5b k_vocab_merge: one warp per row combines the partials into (max, lse) and
//   the top-KM of the half-tile maxima.  That is the exact top-KM unless some
//   half-tile's runner-up reaches the KM-th value (~C(KM,2)/#half-tiles of the
//   rows); those half-tiles are recomputed exactly (dp4a over K) and merged in
//   full.  Exact scores, ordering and the f32 tie check then follow k_topk1
//   (output.cu); a tie across the KM boundary recomputes the whole row (never
//   seen outside constructed tie tests).
#include "cand.cuh"
#include "kernels.cuh"
#include "tc_mainloop.cuh"

namespace qnmt {

#ifndef QNMT_VT_BN      // (A/B builds: 256 tokens per tile with 16 epilogue warps)
#define QNMT_VT_BN 192
#endif
#ifndef QNMT_VT_EPI_WARPS
#define QNMT_VT_EPI_WARPS 12
#endif
constexpr int VT_BN = QNMT_VT_BN;          // tokens per tile (UMMA N); 2 accumulators in a 512-column TMEM slot
constexpr int VT_EPI_WARPS = QNMT_VT_EPI_WARPS;   // 3 per TMEM lane group (64 tokens each): latency hiding for the fp64 epilogue
constexpr int VT_THREADS = 64 + 32 * VT_EPI_WARPS;
#ifndef QNMT_VT_STAGES
#define QNMT_VT_STAGES 4
#endif
using VtRing = TcRing<VT_BN, QNMT_VT_STAGES>;
constexpr int VT_SPLIT = VT_EPI_WARPS / 4;   // token groups per tile (one per warp of a lane group)
constexpr int VT_HALF = VT_BN / VT_SPLIT;    // tokens per partial
constexpr int VT_RESCAN_MAX = 64;    // flagged half-tiles handled per row before a full row rescan

struct VtPart {
    double s;       // sum exp(x - m) over the half-tile
    float m;        // max logit (-FLT_MAX: empty)
    float a2;       // second-largest logit (may equal m; -FLT_MAX: fewer than 2 tokens)
    int32_t i1;     // smallest token with logit m (INT_MAX: empty)
    int32_t pad;    // row's first partial, after the merge: path taken (diagnostics, see k_vocab_merge)
};

// K7 vocabulary-shard partial of one hypothesis row (qnmt_vocab_shard_partials): the
// shard's max logit M, S = sum over its tokens of exp(x - M) (fp64), and its top-VS_KR
// logits by (logit desc, token asc) with global token ids.
constexpr int VS_KR = 8;
struct VsPart {
    double S;
    float M;
    int32_t n;               // candidates held (min(VS_KR, shard rows))
    float x[VS_KR];
    int32_t t[VS_KR];
};
static_assert(sizeof(VsPart) == 80, "VsPart layout is part of the C ABI");

struct VtArgs {
    const float* x_scales;    // activation scale per segment
    const int32_t* row_seg;   // segment of each hypothesis row
    const float* w_scales;    // weight scale per w_rows_per_scale vocabulary rows
    int64_t w_rows_per_scale;
    const float* bias;        // [V]
    VtPart* part;             // [rows][2 * n_blocks]
    int32_t* err_flag;
};

#ifdef QNMT_VT_MAXREG   // (A/B builds: cap registers so another stream's CTAs fit beside this one)
#define VT_BOUNDS __maxnreg__(QNMT_VT_MAXREG)
#else
#define VT_BOUNDS __launch_bounds__(VT_THREADS, 1)
#endif
__global__ void VT_BOUNDS
k_vocab_stats(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int M, int V,
              int K, VtArgs e, const int32_t* n_dev) {
    using C = VtRing;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const TcBars<C> bars(smem);
    // per epilogue warp: bias (and weight scale, 1/scale) of its 64-token group of the current
    // tile -- warp-private, so __syncwarp orders the writes and reads (no barrier across warps)
    __shared__ double col_isw[VT_EPI_WARPS][VT_HALF];
    __shared__ float col_sw[VT_EPI_WARPS][VT_HALF];
    __shared__ __align__(16) float col_b[VT_EPI_WARPS][VT_HALF];
    __shared__ double tab[16];
    __shared__ double tab64[64];
    // per epilogue thread: the 16 logits of the chunk holding its group's running max
    // ([slot][thread]: consecutive lanes hit consecutive 16-byte words)
    __shared__ float4 xbest[4][VT_EPI_WARPS * 32];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 16) tab[threadIdx.x] = exp2((double)threadIdx.x / 16.0);
    if (threadIdx.x < 64) tab64[threadIdx.x] = exp2((double)threadIdx.x / 64.0);
    pdl_trigger();
    const uint32_t tmem_base = tc_setup<C>(&tmX, &tmW, bars, VT_EPI_WARPS);   // includes __syncthreads
    pdl_wait();   // everything above overlaps the predecessor kernel (PDL)
    if (n_dev) M = min(M, *n_dev);
    const int m_blocks = (M + TC_BM - 1) / TC_BM;
    const int n_blocks = (V + VT_BN - 1) / VT_BN;
    const int tiles = m_blocks * n_blocks;
    // contiguous tile range per CTA (row block changes at most a few times per CTA, and the
    // next tile's bias is known one tile ahead); equal shares +-1 tile
    const int t_begin = (int)((int64_t)blockIdx.x * tiles / gridDim.x);
    const int t_end = (int)((int64_t)(blockIdx.x + 1) * tiles / gridDim.x);
    const int k_blocks = (K + TC_BK - 1) / TC_BK;

    if (warp == 0) {
        tc_produce<C, VT_BN>(&tmX, &tmW, smem, bars, t_end, n_blocks, k_blocks, t_begin, 1);
    } else if (warp == 1) {
        tc_issue<C, VT_BN>(smem, bars, tmem_base, t_end, k_blocks, t_begin, 1);
    } else {
        const int ew = warp - 2;
        const int lg = warp & 3;     // TMEM lane group
        const int half = ew >> 2;    // token group of the tile
        const int np = VT_SPLIT * n_blocks;
        const bool one_scale = e.w_rows_per_scale >= V;   // kernel-uniform
        const float sw0 = e.w_scales[0];
        const double isw0 = 1.0 / (double)sw0;
        bool bad = false;
        int it = 0;
        // the row's activation scale and multipliers depend only on the m-block: computed when it
        // changes (at most a few times in a CTA's contiguous tile range), not per tile
        int cur_mb = -1;
        float sx = 1.0f;
        double isx = 1.0, rs0 = isw0;
        int mb = t_begin / n_blocks, nb = t_begin % n_blocks;
        // this tile's bias for tokens lane and lane + 32 of the group (loaded one tile ahead)
        float bp0 = 0.0f, bp1 = 0.0f;
        if (t_begin < t_end && e.bias) {
            const int v = nb * VT_BN + half * VT_HALF + lane;
            if (v < V) bp0 = e.bias[v];
            if (v + 32 < V) bp1 = e.bias[v + 32];
        }
        for (int tile = t_begin; tile < t_end; ++tile, ++it) {
            const int buf = it & 1;
            const uint32_t use = (uint32_t)(it >> 1) & 1u;
            float bmx;   // max |bias| over the group
            {   // this warp's group: bias (and per-token weight scale) -> its smem slice
                const int vg = nb * VT_BN + half * VT_HALF;
                const float b0 = bp0, b1 = bp1;
                {   // prefetch the next tile's
                    const int vn = (nb + 1 == n_blocks ? 0 : nb + 1) * VT_BN + half * VT_HALF + lane;
                    const bool more = tile + 1 < t_end && e.bias;
                    bp0 = (more && vn < V) ? e.bias[vn] : 0.0f;
                    bp1 = (more && vn + 32 < V) ? e.bias[vn + 32] : 0.0f;
                }
                __syncwarp();   // the previous tile's reads of the slice are done
                if (!one_scale) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int v = vg + lane + 32 * h;
                        const float sw = v < V ? e.w_scales[v / e.w_rows_per_scale] : 1.0f;
                        col_sw[ew][lane + 32 * h] = sw;
                        col_isw[ew][lane + 32 * h] = 1.0 / (double)sw;
                    }
                }
                col_b[ew][lane] = b0;
                col_b[ew][lane + 32] = b1;
                bmx = warp_max(fmaxf(fabsf(b0), fabsf(b1)));
                bad |= !(is_finite_f(b0) && is_finite_f(b1));
                __syncwarp();
            }
            const int row = mb * TC_BM + lg * 32 + lane;
            const bool rok = row < M;
            if (mb != cur_mb) {
                sx = rok ? e.x_scales[e.row_seg ? e.row_seg[row] : 0] : 1.0f;
                isx = 1.0 / (double)sx;
                rs0 = isx * isw0;   // acc -> logit multiplier when W has one scale
                cur_mb = mb;
            }
            tc::mbar_wait(&bars.tfull[buf], use);
            tc::tc_fence_after();
            // fast-path preconditions, per thread and tile: one weight scale, and every
            // nonzero |q| = |acc| * rs in [2^-124, 2^127) (f32 normal range for |acc| < 2^31)
            const bool fast_row = one_scale && rs0 >= 0x1p-124 && rs0 * 2147483648.0 < 0x1p127;
            // every logit of the tile lies in [-340, 340] when K * 127^2 * rs + max|b| < 340
            // (|acc| <= K * 127^2; roundings add < 2^-22 relative), so no x - m falls below
            // -700: the chunk minimum (the exp range guard) is then skipped
            bool narrow = false;
            if (__all_sync(0xffffffffu, fast_row))
                narrow = __all_sync(0xffffffffu, (double)K * 16129.0 * rs0 + (double)bmx < 340.0);
            // top-1 (value, smallest token) and runner-up value from chunk maxima: the chunk that
            // raised the running max is parked in shared memory; after the group, its token and
            // the runner-up (its own second value vs the other chunks' maxima) are resolved
            const int et = ew * 32 + lane;
            float om = -FLT_MAX;   // max of the chunk maxima other than the best chunk's
            int bc0 = -1;          // first token of the best chunk (-1: none)
            float m = -FLT_MAX;   // running max of the half-tile (the exp reference)
            double e4[4] = {0.0, 0.0, 0.0, 0.0};   // sum exp(x - m) as 4 interleaved chains over the group
#pragma unroll 1
            for (int c0 = half * VT_HALF; c0 < (half + 1) * VT_HALF; c0 += 16) {
                uint32_t r[16];
                tc::tmem_ld16(tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * VT_BN + c0), r);
                const int vbase = nb * VT_BN + c0;
                const int ncols = min(16, V - vbase);   // warp-uniform
                tc::tmem_ld_wait();
                if (ncols <= 0) continue;
                float x[16];
                if (__all_sync(0xffffffffu, fast_row) && ncols == 16) {
                    // exact dequant fl32(acc * rs): safe unless q's bits below f32 precision lie
                    // within 64 f64-ulps of the rounding midpoint (0x10000000)
                    // (int32 -> f64 through the exponent field on the fp64 pipe instead of the XU
                    // conversion: 2^52 + (acc + 2^31) - (2^52 + 2^31), exact; |d| <= 64 test as one
                    // wrapped unsigned range check)
                    uint32_t dmin = 0xffffffffu;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const double av = __hiloint2double(0x43300000, (int)(r[j] ^ 0x80000000u)) - 4503601774854144.0;
                        const double q = av * rs0;
                        x[j] = __double2float_rn(q);
                        // (low 29 bits of q + 64 - 2^28, times 8 so the wrap is the u32 one: one IMAD)
                        dmin = min(dmin, (uint32_t)__double2loint(q) * 8u + (64u - 0x10000000u) * 8u);
                    }
                    if (__any_sync(0xffffffffu, dmin <= 1024u)) {   // rare: exact division where needed
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const double q = (double)(int)r[j] * rs0;
                            if ((((uint32_t)__double2loint(q) + (64u - 0x10000000u)) & 0x1fffffffu) <= 128u)
                                x[j] = dequant((int)r[j], sw0, sx);   // (fast path: one scale)
                        }
                    }
                    const float4* b4 = reinterpret_cast<const float4*>(&col_b[ew][c0 - half * VT_HALF]);
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        const float4 bb = b4[q4];
                        x[4 * q4 + 0] = __fadd_rn(x[4 * q4 + 0], bb.x);
                        x[4 * q4 + 1] = __fadd_rn(x[4 * q4 + 1], bb.y);
                        x[4 * q4 + 2] = __fadd_rn(x[4 * q4 + 2], bb.z);
                        x[4 * q4 + 3] = __fadd_rn(x[4 * q4 + 3], bb.w);
                    }
                } else {   // vocabulary tail, per-row weight scales or extreme scales
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (j < ncols) {
                            const double isw = one_scale ? isw0 : col_isw[ew][c0 - half * VT_HALF + j];
                            const float swj = one_scale ? sw0 : col_sw[ew][c0 - half * VT_HALF + j];
                            const double q = (double)(int)r[j] * (isx * isw);
                            x[j] = dequant_rcp_safe(q) ? __double2float_rn(q) : dequant((int)r[j], swj, sx);
                            x[j] = __fadd_rn(x[j], col_b[ew][c0 - half * VT_HALF + j]);
                        } else {
                            x[j] = -FLT_MAX;   // excluded below (exp skipped, never above a real logit)
                        }
                    }
                }
                float cm, cn = 0.0f;
                {   // chunk max / min as shallow trees (invalid tail tokens are -FLT_MAX: a tail chunk's
                    // min is then -FLT_MAX, harmless: tail chunks take the range-guarded exp anyway)
                    float t[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) t[j] = fmaxf(x[2 * j], x[2 * j + 1]);
                    cm = fmaxf(fmaxf(fmaxf(t[0], t[1]), fmaxf(t[2], t[3])), fmaxf(fmaxf(t[4], t[5]), fmaxf(t[6], t[7])));
                    if (!narrow) {   // warp-uniform
                        float u[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) u[j] = fminf(x[2 * j], x[2 * j + 1]);
                        cn = fminf(fminf(fminf(u[0], u[1]), fminf(u[2], u[3])), fminf(fminf(u[4], u[5]), fminf(u[6], u[7])));
                    }
                }
                // +-inf (NaN only from non-finite bias); a narrow tile's logits are finite by its bound
                bad |= !(is_finite_f(cm) && is_finite_f(cn));
                {   // strict '>': on equal maxima the earlier chunk (smaller tokens) stays best
                    const bool nbst = cm > m;
                    om = fmaxf(om, nbst ? m : cm);
                    if (nbst) {
                        bc0 = vbase;
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4)
                            xbest[q4][et] = make_float4(x[4 * q4], x[4 * q4 + 1], x[4 * q4 + 2], x[4 * q4 + 3]);
                    }
                }
                if (cm > m) {   // rescale the running sum (first chunk, then rare)
                    const double f = (m == -FLT_MAX) ? 0.0 : exp_neg((double)m - (double)cm, tab);
#pragma unroll
                    for (int q = 0; q < 4; ++q) e4[q] *= f;
                    m = cm;
                }
                const double dm = (double)m;
                if (ncols == 16 && (narrow || !__any_sync(0xffffffffu, (double)cn - dm < -700.0))) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) e4[j & 3] = exp_neg64_acc((double)x[j] - dm, tab64, e4[j & 3]);
                } else {   // vocabulary tail or a logit range beyond 700 (range-guarded exp)
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < ncols) e4[j & 3] += exp_neg((double)x[j] - dm, tab);
                }
            }
            float a2 = om;
            int i1 = 0x7fffffff;
            if (bc0 >= 0) {   // first token of the best chunk equal to m; the chunk's second value
                float xb[16];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                    const float4 v4 = xbest[q4][et];
                    xb[4 * q4] = v4.x;
                    xb[4 * q4 + 1] = v4.y;
                    xb[4 * q4 + 2] = v4.z;
                    xb[4 * q4 + 3] = v4.w;
                }
                int idx = 15;
#pragma unroll
                for (int j = 14; j >= 0; --j) idx = xb[j] == m ? j : idx;
                float sm = -FLT_MAX;
#pragma unroll
                for (int j = 0; j < 16; ++j) sm = fmaxf(sm, j == idx ? -FLT_MAX : xb[j]);
                a2 = fmaxf(a2, sm);
                i1 = bc0 + idx;
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&bars.tempty[buf]);
            if (rok) {
                VtPart p;
                p.s = (e4[0] + e4[1]) + (e4[2] + e4[3]);
                p.m = m;
                p.a2 = a2;
                p.i1 = i1;
                p.pad = 0;
                e.part[(int64_t)row * np + nb * VT_SPLIT + half] = p;
            }
            if (++nb == n_blocks) {
                nb = 0;
                ++mb;
            }
        }
        if (bad) set_flag(e.err_flag, QNMT_FLAG_NUMERIC);
    }
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}

struct VtMergeArgs {
    const int8_t* X;
    int64_t ldx;
    const int8_t* W;
    int64_t ldw;
    int K, V, n_blocks;
    const float* x_scales;
    const int32_t* row_seg;
    const float* w_scales;
    int64_t w_rows_per_scale;
    const float* bias;
    VtPart* part;
    const double* live;
    int k;
    double* cand_score;
    int32_t* cand_tok;
    VsPart* raw;        // vocabulary shard mode (K7): per-row (M, S, top-KR logits) instead of candidates
    int32_t tok_off;    // shard mode: global token id of the shard's first row
};

// Warp-cooperative exact logits of tokens v0 .. v0+31 for one row: lane j returns
// the logit of token v0 + j (-FLT_MAX past the vocabulary).  Every token's K
// codes are read as one coalesced 512-byte row slice (16 B per lane), dot
// products by dp4a, reduced with one REDUX each; 8 tokens' loads in flight.
__device__ __forceinline__ float vt_logits32(const VtMergeArgs& a, const int8_t* __restrict__ xr, int v0, float sx) {
    const int lane = threadIdx.x & 31;
    int mytot = 0;
#pragma unroll 1
    for (int t0 = 0; t0 < 32; t0 += 16) {
        int part[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) part[u] = 0;
        for (int k = lane * 16; k < a.K; k += 512) {
            const int4 xa = *reinterpret_cast<const int4*>(xr + k);
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int v = min(v0 + t0 + u, a.V - 1);   // clamped tokens are discarded below
                const int4 wa = *reinterpret_cast<const int4*>(a.W + (int64_t)v * a.ldw + k);
                part[u] = __dp4a(xa.x, wa.x, part[u]);
                part[u] = __dp4a(xa.y, wa.y, part[u]);
                part[u] = __dp4a(xa.z, wa.z, part[u]);
                part[u] = __dp4a(xa.w, wa.w, part[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int tot = __reduce_add_sync(0xffffffffu, part[u]);
            if (lane == t0 + u) mytot = tot;
        }
    }
    const int v = v0 + lane;   // one exact dequant per lane, in parallel
    if (v >= a.V) return -FLT_MAX;
    return __fadd_rn(dequant(mytot, a.w_scales[v / a.w_rows_per_scale], sx), a.bias ? a.bias[v] : 0.0f);
}

constexpr int VM_WARPS = 4;   // rows per merge CTA (one warp per row)

#ifdef QNMT_VM_PROF   // (benchmarks/build_variant.sh + benchmarks/vm_prof.py: per-row phase clocks of k_vocab_merge)
__device__ long long g_vm_prof[8 * 2048];
#define VM_STAMP(k) do { if (lane == 0 && n < 2048) g_vm_prof[n * 8 + (k)] = clock64(); } while (0)
#else
#define VM_STAMP(k) do { } while (0)
#endif

// (logit desc, token asc) as one descending u64 key: order-preserving f32 bits, then ~token
__device__ __forceinline__ uint64_t cand_key(float x, int tok) {
    const uint32_t b = __float_as_uint(x);
    const uint32_t sb = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((uint64_t)sb << 32) | (uint32_t)~(uint32_t)tok;
}
__device__ __forceinline__ Cand key_cand(uint64_t k) {
    const uint32_t sb = (uint32_t)(k >> 32);
    const uint32_t b = (sb & 0x80000000u) ? (sb & 0x7fffffffu) : ~sb;
    return k == 0 ? Cand{-DBL_MAX, 0x7fffffff} : Cand{(double)__uint_as_float(b), (int)~(uint32_t)k};
}
// bitonic sort of one key per lane, descending (lane 0 = largest); 15 compare-exchange stages
__device__ __forceinline__ uint64_t warp_sort_desc(uint64_t key) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, key, j);
            const bool desc = (lane & k) == 0 || k == 32;
            const bool take_max = ((lane & j) == 0) == desc;
            key = take_max ? (key > other ? key : other) : (key < other ? key : other);
        }
    return key;
}

template <int KM, bool RAW = false>
__global__ void __launch_bounds__(32 * VM_WARPS)
k_vocab_merge(VtMergeArgs a, int64_t N, const int32_t* n_dev) {
    pdl_entry();
    __shared__ double tab[16];
    __shared__ Cand lst[VM_WARPS][KM];
    __shared__ int flagged[VM_WARPS][VT_RESCAN_MAX];
    __shared__ uint64_t clist[VM_WARPS][32];
    __shared__ int ncand[VM_WARPS];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 16) tab[threadIdx.x] = exp2((double)threadIdx.x / 16.0);
    __syncthreads();
    const int64_t n = (int64_t)blockIdx.x * VM_WARPS + wib;
    if (n >= N || beyond(n_dev, n)) return;   // warp-uniform
    const int np = VT_SPLIT * a.n_blocks;
    VtPart* pr = a.part + n * np;
    VM_STAMP(0);
    // pass 1: online (max, sum exp), each lane's best (max, token) and largest runner-up
    const int kk = a.V < KM ? a.V : KM;
    Cand* out = lst[wib];
    float ml = -FLT_MAX, a2l = -FLT_MAX;
    int tl = 0x7fffffff;   // token of the lane's best max (smallest on ties)
    double sl = 0.0;
    constexpr int PB = 8;   // partials per lane in flight
    for (int b0 = lane; b0 < np; b0 += 32 * PB) {
        VtPart p[PB];
#pragma unroll
        for (int i = 0; i < PB; ++i) {
            const int b = b0 + 32 * i;
            if (b < np) {
                p[i] = pr[b];
            } else {
                p[i].m = -FLT_MAX;
                p[i].a2 = -FLT_MAX;
                p[i].i1 = 0x7fffffff;
            }
        }
        float cmx = ml;
#pragma unroll
        for (int i = 0; i < PB; ++i) {
            cmx = fmaxf(cmx, p[i].m);
            a2l = fmaxf(a2l, p[i].a2);
        }
        if (cmx > ml) {
            sl = (ml == -FLT_MAX) ? 0.0 : sl * exp_neg((double)ml - (double)cmx, tab);
            ml = cmx;
            tl = 0x7fffffff;
        }
#pragma unroll
        for (int i = 0; i < PB; ++i) {
            if (p[i].i1 != 0x7fffffff) {
                sl += p[i].s * exp_neg((double)p[i].m - (double)ml, tab);
                if (p[i].m == ml && p[i].i1 < tl) tl = p[i].i1;
            }
        }
    }
    const float M = warp_max(ml);
    const double dM = (double)M;
    const double ssum = warp_sum(ml == -FLT_MAX ? 0.0 : sl * exp_neg((double)ml - dM, tab));
    const double lse = log(ssum);
    VM_STAMP(1);
    // tau = kk-th best of the 32 lane maxima (bitonic sort of (logit, token) keys): at least kk
    // group maxima are >= tau, so every member of the top-kk is too
    const uint64_t tau_key = __shfl_sync(0xffffffffu,
                                         warp_sort_desc(ml == -FLT_MAX ? 0ull : cand_key(ml, tl)), kk - 1);
    // pass 2 (L1-resident): the few group maxima with key >= tau -> a per-warp list
    if (lane == 0) ncand[wib] = 0;
    __syncwarp();
    for (int b = lane; b < np; b += 32) {
        const float pm = pr[b].m;
        if (pm != -FLT_MAX) {
            const uint64_t k = cand_key(pm, pr[b].i1);
            if (k >= tau_key) {
                const int slot = atomicAdd(&ncand[wib], 1);
                if (slot < 32) clist[wib][slot] = k;
            }
        }
    }
    __syncwarp();
    const int nc = ncand[wib];
    if (nc <= 32) {   // sort the list across the warp: lanes 0..kk-1 hold the top-kk
        const uint64_t k = warp_sort_desc(lane < nc ? clist[wib][lane] : 0ull);
        if (lane < kk) out[lane] = key_cand(k);
    } else {          // many equal logits: per-lane lists and a k-way merge
        Cand L0[KM];
#pragma unroll
        for (int i = 0; i < KM; ++i) L0[i] = Cand{-DBL_MAX, 0x7fffffff};
        for (int b = lane; b < np; b += 32) {
            const float pm = pr[b].m;
            if (pm != -FLT_MAX && cand_key(pm, pr[b].i1) >= tau_key) insert<KM>(L0, Cand{(double)pm, pr[b].i1});
        }
        warp_merge<KM>(L0, out, kk);
    }
    __syncwarp();
    VM_STAMP(2);
    const Cand tau = key_cand(tau_key);
    Cand L[KM];
    // half-tiles whose runner-up reaches the KM-th value may hold more of the top-KM
    const Cand thr = out[kk - 1];
    int nf = 0;
    if (__any_sync(0xffffffffu, a2l != -FLT_MAX && (double)a2l >= thr.s))   // rare: find the half-tiles
    for (int b0 = 0; b0 < np; b0 += 32) {
        const int b = b0 + lane;
        const bool f = b < np && pr[b].a2 != -FLT_MAX && (double)pr[b].a2 >= thr.s;
        const unsigned mask = __ballot_sync(0xffffffffu, f);
        const int slot = nf + __popc(mask & ((1u << lane) - 1u));
        if (f && slot < VT_RESCAN_MAX) flagged[wib][slot] = b;
        nf += __popc(mask);
    }
    __syncwarp();
    const int8_t* xr = a.X + n * a.ldx;
    const float sx = a.x_scales[a.row_seg ? a.row_seg[n] : 0];
    if (nf > 0 && nf <= VT_RESCAN_MAX) {
        // rebuild: unflagged partials' entries + every token of the flagged half-tiles
#pragma unroll
        for (int i = 0; i < KM; ++i) L[i] = Cand{-DBL_MAX, 0x7fffffff};
        // (only candidates not worse than tau can be in the top-kk)
        for (int b = lane; b < np; b += 32) {
            const float pm = pr[b].m;
            if ((double)pm < tau.s || pm == -FLT_MAX) continue;
            bool fl = false;
            for (int f = 0; f < nf; ++f) fl |= flagged[wib][f] == b;
            const Cand c{(double)pm, pr[b].i1};
            if (!fl && !better(tau, c)) insert<KM>(L, c);
        }
        for (int f = 0; f < nf; ++f) {
            const int b = flagged[wib][f];
            const int vb = (b / VT_SPLIT) * VT_BN + (b % VT_SPLIT) * VT_HALF;
            for (int g = 0; g < VT_HALF; g += 32) {
                const float x = vt_logits32(a, xr, vb + g, sx);
                const Cand c{(double)x, vb + g + lane};
                if (vb + g + lane < a.V && !better(tau, c)) insert<KM>(L, c);
            }
        }
        __syncwarp();
        warp_merge<KM>(L, out, kk);
        __syncwarp();
    }
    if (RAW) {   // vocabulary shard (K7): the shard's (max, sum exp(x - max)) and exact top-KR logits
        if (nf > VT_RESCAN_MAX) {   // too many flagged half-tiles: the shard's whole row, by logit
#pragma unroll
            for (int i = 0; i < KM; ++i) L[i] = Cand{-DBL_MAX, 0x7fffffff};
            for (int v0 = 0; v0 < a.V; v0 += 32) {
                const float x = vt_logits32(a, xr, v0, sx);
                if (v0 + lane < a.V) insert<KM>(L, Cand{(double)x, v0 + lane});
            }
            __syncwarp();
            warp_merge<KM>(L, out, kk);
            __syncwarp();
        }
        VsPart* r = a.raw + n;
        const int nr = kk < VS_KR ? kk : VS_KR;
        if (lane == 0) {
            r->S = ssum;
            r->M = M;
            r->n = nr;
        }
        if (lane < VS_KR) {
            r->x[lane] = lane < nr ? (float)out[lane].s : -FLT_MAX;
            r->t[lane] = lane < nr ? out[lane].t + a.tok_off : 0x7fffffff;
        }
        return;
    }
    VM_STAMP(3);
    const double base = a.live ? a.live[n] : 0.0;
    int ok = 0;
    if (nf <= VT_RESCAN_MAX) {
        // exact scores of the KM logit-candidates (lane i: candidate i), then each lane's rank
        // in (score desc, token asc) order; exact unless the k-th score ties the KM-th
        Cand c{-DBL_MAX, 0x7fffffff};
        if (lane < kk) c = Cand{base + (double)__double2float_rn((out[lane].s - dM) - lse), out[lane].t};
        const double s_last = __shfl_sync(0xffffffffu, c.s, kk - 1);
        int rank = 0;
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const double os = __shfl_sync(0xffffffffu, c.s, j);
            const int ot = __shfl_sync(0xffffffffu, c.t, j);
            rank += (j < kk && j != lane && better(Cand{os, ot}, c)) ? 1 : 0;
        }
        const unsigned at_k = __ballot_sync(0xffffffffu, lane < kk && rank == a.k - 1);
        const double sk = __shfl_sync(0xffffffffu, c.s, at_k ? __ffs(at_k) - 1 : 0);
        ok = (a.V <= KM) || (sk > s_last);
        if (ok && lane < kk && rank < a.k) {
            a.cand_score[n * a.k + rank] = c.s;
            a.cand_tok[n * a.k + rank] = c.t;
        }
    }
    // diagnostics: pad of the row's first partial = flagged half-tiles (phase 1) + 1000 * path
    // (0 merged, 1 boundary-tie rescan, 2 whole row)
    if (ok) {
        if (lane == 0) pr[0].pad = nf;
        VM_STAMP(4);
        return;
    }
#pragma unroll
    for (int i = 0; i < KM; ++i) L[i] = Cand{-DBL_MAX, 0x7fffffff};
    // f32 tie across the KM boundary: tokens outside the list whose log-prob rounds to the KM-th
    // candidate's have logits within a few f32 ulps of lp below x_KM.  Every other token scores
    // strictly lower, so the exact answer is the top-k of the exact scores of all tokens in the
    // half-tiles that may hold a logit >= x_KM - 4 ulp(lp_KM) (max or runner-up reaching it).
    int nf2 = VT_RESCAN_MAX + 1;
    if (nf <= VT_RESCAN_MAX) {
        const float lpk = __double2float_rn((out[kk - 1].s - dM) - lse);
        const int ex = (int)((__float_as_uint(lpk) >> 23) & 0xffu);
        const double tau2 = out[kk - 1].s - ldexp(1.0, max(ex, 1) - 150 + 2);
        nf2 = 0;
        for (int b0 = 0; b0 < np; b0 += 32) {
            const int b = b0 + lane;
            const bool f = b < np && ((pr[b].i1 != 0x7fffffff && (double)pr[b].m >= tau2) ||
                                      (pr[b].a2 != -FLT_MAX && (double)pr[b].a2 >= tau2));
            const unsigned mask = __ballot_sync(0xffffffffu, f);
            const int slot = nf2 + __popc(mask & ((1u << lane) - 1u));
            if (f && slot < VT_RESCAN_MAX) flagged[wib][slot] = b;
            nf2 += __popc(mask);
        }
        __syncwarp();
        if (nf2 <= VT_RESCAN_MAX) {
            for (int f = 0; f < nf2; ++f) {
                const int b = flagged[wib][f];
                const int vb = (b / VT_SPLIT) * VT_BN + (b % VT_SPLIT) * VT_HALF;
                for (int g = 0; g < VT_HALF; g += 32) {
                    const float x = vt_logits32(a, xr, vb + g, sx);
                    if (vb + g + lane < a.V)
                        insert<KM>(L, Cand{base + (double)__double2float_rn(((double)x - dM) - lse), vb + g + lane});
                }
            }
        }
    }
    if (lane == 0) pr[0].pad = nf + (nf2 > VT_RESCAN_MAX ? 2000 : 1000) + 10000 * min(nf2, 99);
    if (nf2 > VT_RESCAN_MAX) {   // pathological ties (e.g. repeated vocabulary rows): the whole row
#pragma unroll
        for (int i = 0; i < KM; ++i) L[i] = Cand{-DBL_MAX, 0x7fffffff};
        for (int v0 = 0; v0 < a.V; v0 += 32) {
            const float x = vt_logits32(a, xr, v0, sx);
            if (v0 + lane < a.V)
                insert<KM>(L, Cand{base + (double)__double2float_rn(((double)x - dM) - lse), v0 + lane});
        }
    }
    __syncwarp();
    warp_merge<KM>(L, out, a.k);
    __syncwarp();
    if (lane == 0)
        for (int i = 0; i < a.k; ++i) {
            a.cand_score[n * a.k + i] = out[i].s;
            a.cand_tok[n * a.k + i] = out[i].t;
        }
}

#ifdef QNMT_VM_PROF
}  // namespace qnmt
extern "C" __attribute__((visibility("default"))) int qnmt_debug_vm_prof(long long* out, int rows) {
    return (int)cudaMemcpyFromSymbol(out, qnmt::g_vm_prof, sizeof(long long) * 8 * (size_t)rows);
}
namespace qnmt {
#endif

bool vocab_topk_eligible(int64_t K, int64_t ldx, int64_t ldw, const void* X, const void* W, int k) {
    return K % 16 == 0 && K > 0 && K <= QNMT_INT32_SAFE_K && ldx % 16 == 0 && ldw % 16 == 0 &&
           ((uintptr_t)X % 16 == 0) && ((uintptr_t)W % 16 == 0) && k >= 1 && k <= 16;
}

size_t vocab_topk_part_bytes(int64_t rows, int64_t V) {
    return (size_t)rows * VT_SPLIT * (size_t)cdiv(V, VT_BN) * sizeof(VtPart);
}

int g_vocab_fused = 1;

int vocab_stats_launch(const VocabTopk& p, cudaStream_t st) {
    const int8_t* X = p.X;
    const int64_t N = p.N, ldx = p.ldx, V = p.V, K = p.K, ldw = p.ldw;
    const int8_t* W = p.W;
    const int k = p.k;
    if (N <= 0) return QNMT_OK;
    if (!vocab_topk_eligible(K, ldx, ldw, X, W, k) || k > V) {
        set_error("vocab_topk: ineligible shape K=%lld k=%d V=%lld", (long long)K, k, (long long)V);
        return QNMT_ERR_CONFIG;
    }
    static size_t attr_done = 0;
    QNMT_CUDA(raise_smem_limit((const void*)k_vocab_stats, VtRing::SMEM, attr_done));
    CUtensorMap tx, tw;
    int rc = tc_get_map(X, N, K, ldx, TC_BM, &tx);
    if (rc) return rc;
    rc = tc_get_map(W, V, K, ldw, VT_BN, &tw);
    if (rc) return rc;
    VtArgs e{p.x_scales, p.row_seg, p.w_scales, p.w_rows_per_scale, p.bias, reinterpret_cast<VtPart*>(p.part),
             p.err_flag};
    const int n_blocks = (int)cdiv(V, VT_BN);
    const int tiles = (int)(cdiv(N, TC_BM) * n_blocks);
    const int grid = tiles < tc_sm_count() ? tiles : tc_sm_count();
    QNMT_LAUNCH(k_vocab_stats, grid, VT_THREADS, VtRing::SMEM, st, tx, tw, (int)N, (int)V, (int)K, e, tl_ndev);
    QNMT_CHECK_LAUNCH("k_vocab_stats");
    return QNMT_OK;
}

int vocab_merge_launch(const VocabTopk& p, cudaStream_t st) {
    const int64_t N = p.N;
    const int k = p.k;
    if (N <= 0) return QNMT_OK;
    VtMergeArgs ma{p.X, p.ldx, p.W, p.ldw, (int)p.K, (int)p.V, (int)cdiv(p.V, VT_BN), p.x_scales, p.row_seg,
                   p.w_scales, p.w_rows_per_scale, p.bias, reinterpret_cast<VtPart*>(p.part), p.live, k,
                   p.cand_score, p.cand_tok, nullptr, 0};
    const unsigned g = (unsigned)cdiv(N, VM_WARPS);
    auto kfn = k <= 6 ? k_vocab_merge<8> : k <= 13 ? k_vocab_merge<16> : k_vocab_merge<32>;
    QNMT_LAUNCH(kfn, g, 32 * VM_WARPS, 0, st, ma, N, tl_ndev);
    QNMT_CHECK_LAUNCH("k_vocab_merge");
    return QNMT_OK;
}

// K7 combine: one warp per row merges the G shards' partials into the step's
// candidates, exactly as k_vocab_merge scores them:
//   M = max_g M_g, lse = log(sum_g S_g e^(M_g - M)) (fp64, shard order),
//   score = live + fl32((x - M) - lse) for the union of the shards' top-VS_KR
//   logits, ranked by (score desc, token asc).
// The union holds the global top-k unless a shard with a full list has its
// VS_KR-th candidate scoring >= the k-th best (a token outside its list could
// then tie into the top-k): those rows set QNMT_FLAG_SHARD_TIE and the caller
// recomputes them unsharded.
__global__ void __launch_bounds__(32 * VM_WARPS)
k_vocab_shard_combine(const VsPart* __restrict__ parts, int G, int64_t N, const double* __restrict__ live, int k,
                      double* __restrict__ cand_score, int32_t* __restrict__ cand_tok, int32_t* err_flag) {
    pdl_entry();
    const int lane = threadIdx.x & 31;
    const int64_t n = (int64_t)blockIdx.x * VM_WARPS + (threadIdx.x >> 5);
    if (n >= N) return;
    float M = -FLT_MAX;
    for (int g = 0; g < G; ++g) M = fmaxf(M, parts[(int64_t)g * N + n].M);
    const double dM = (double)M;
    double S = 0.0;
    for (int g = 0; g < G; ++g) {   // fixed shard order (every rank computes the same sum)
        const VsPart& p = parts[(int64_t)g * N + n];
        if (p.n > 0) S += p.S * exp_f64((double)p.M - dM);
    }
    const double lse = log(S);
    const double base = live ? live[n] : 0.0;
    // candidates: lane owns entries lane, lane + 32, ... of the G x VS_KR union
    constexpr int PER = 4;   // G <= 16
    Cand c[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int e = lane + 32 * q;
        const int g = e / VS_KR, i = e % VS_KR;
        c[q] = Cand{-DBL_MAX, 0x7fffffff};
        if (g < G) {
            const VsPart& p = parts[(int64_t)g * N + n];
            if (i < p.n) c[q] = Cand{base + (double)__double2float_rn(((double)p.x[i] - dM) - lse), p.t[i]};
        }
    }
    // top-k by repeated warp argmax (k <= 16); lane 0 writes each as it is found
    Cand kth{-DBL_MAX, 0x7fffffff};
    for (int r = 0; r < k; ++r) {
        Cand w = c[0];
#pragma unroll
        for (int q = 1; q < PER; ++q) if (better(c[q], w)) w = c[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const Cand x{__shfl_xor_sync(0xffffffffu, w.s, o), __shfl_xor_sync(0xffffffffu, w.t, o)};
            if (better(x, w)) w = x;
        }
        if (lane == 0) {
            cand_score[n * k + r] = w.s;
            cand_tok[n * k + r] = w.t;
        }
        kth = w;
#pragma unroll
        for (int q = 0; q < PER; ++q) if (c[q].t == w.t && c[q].s == w.s) c[q] = Cand{-DBL_MAX, 0x7fffffff};
    }
    // exactness: every full shard's last candidate must score strictly below the k-th
    bool tie = false;
    if (lane < G) {
        const VsPart& p = parts[(int64_t)lane * N + n];
        if (p.n == VS_KR) {
            const double sl = base + (double)__double2float_rn(((double)p.x[VS_KR - 1] - dM) - lse);
            tie = !(sl < kth.s);
        }
    }
    if (__any_sync(0xffffffffu, tie) && lane == 0) set_flag(err_flag, QNMT_FLAG_SHARD_TIE);
}

int vocab_shard_partials_launch(const VocabTopk& p, int32_t tok_off, void* raw, cudaStream_t st) {
    int rc = vocab_stats_launch(p, st);
    if (rc != QNMT_OK || p.N <= 0) return rc;
    VtMergeArgs ma{p.X, p.ldx, p.W, p.ldw, (int)p.K, (int)p.V, (int)cdiv(p.V, VT_BN), p.x_scales, p.row_seg,
                   p.w_scales, p.w_rows_per_scale, p.bias, reinterpret_cast<VtPart*>(p.part), nullptr, 1,
                   nullptr, nullptr, reinterpret_cast<VsPart*>(raw), tok_off};
    const unsigned g = (unsigned)cdiv(p.N, VM_WARPS);
    QNMT_LAUNCH((k_vocab_merge<VS_KR, true>), g, 32 * VM_WARPS, 0, st, ma, p.N, tl_ndev);
    QNMT_CHECK_LAUNCH("k_vocab_merge (shard)");
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" int qnmt_set_vocab_fused(int enable) {
    const int old = qnmt::g_vocab_fused;
    qnmt::g_vocab_fused = enable;
    return old;
}

extern "C" int qnmt_vocab_candidates(const int8_t* X, int64_t N, int64_t ldx, const float* x_scales,
                                     const int32_t* row_seg, const int8_t* W, int64_t V, int64_t K, int64_t ldw,
                                     const float* w_scales, int64_t w_rows_per_scale, const float* bias,
                                     const double* live_scores, int32_t k, void* scratch, double* cand_score,
                                     int32_t* cand_tok, int32_t* err_flag, void* stream) {
    if (N < 0 || V < 1 || w_rows_per_scale < 1) {
        qnmt::set_error("qnmt_vocab_candidates: bad shape N=%lld V=%lld", (long long)N, (long long)V);
        return QNMT_ERR_SHAPE;
    }
    const qnmt::VocabTopk p{X, N, ldx, x_scales, row_seg, W, V, K, ldw, w_scales, w_rows_per_scale, bias,
                            live_scores, k, scratch, cand_score, cand_tok, err_flag};
    const cudaStream_t st = qnmt::as_stream(stream);
    int rc = qnmt::vocab_stats_launch(p, st);
    if (rc != QNMT_OK) return rc;
    return qnmt::vocab_merge_launch(p, st);
}

extern "C" int64_t qnmt_vocab_candidates_scratch(int64_t N, int64_t V) {
    return (int64_t)qnmt::vocab_topk_part_bytes(N, V);
}

extern "C" int64_t qnmt_vocab_shard_part_bytes(void) { return (int64_t)sizeof(qnmt::VsPart); }

extern "C" int qnmt_vocab_shard_partials(const int8_t* X, int64_t N, int64_t ldx, const float* x_scales,
                                         const int32_t* row_seg, const int8_t* W, int64_t V_shard, int64_t K,
                                         int64_t ldw, const float* w_scales, int64_t w_rows_per_scale,
                                         const float* bias, int64_t tok_off, void* scratch, void* parts,
                                         int32_t* err_flag, void* stream) {
    if (N < 0 || V_shard < 1 || w_rows_per_scale < 1 || tok_off < 0) {
        qnmt::set_error("qnmt_vocab_shard_partials: bad shape N=%lld V_shard=%lld", (long long)N, (long long)V_shard);
        return QNMT_ERR_SHAPE;
    }
    const qnmt::VocabTopk p{X, N, ldx, x_scales, row_seg, W, V_shard, K, ldw, w_scales, w_rows_per_scale, bias,
                            nullptr, 1, scratch, nullptr, nullptr, err_flag};
    return qnmt::vocab_shard_partials_launch(p, (int32_t)tok_off, parts, qnmt::as_stream(stream));
}

extern "C" int qnmt_vocab_shard_combine(const void* parts, int32_t G, int64_t N, const double* live_scores,
                                        int32_t k, double* cand_score, int32_t* cand_tok, int32_t* err_flag,
                                        void* stream) {
    if (G < 1 || G > 16 || k < 1 || k > 16 || N < 0) {
        qnmt::set_error("qnmt_vocab_shard_combine: G=%d k=%d (1..16)", G, k);
        return QNMT_ERR_CONFIG;
    }
    if (N == 0) return QNMT_OK;
    const unsigned g = (unsigned)qnmt::cdiv(N, qnmt::VM_WARPS);
    QNMT_LAUNCH(qnmt::k_vocab_shard_combine, g, 32 * qnmt::VM_WARPS, 0, qnmt::as_stream(stream),
                reinterpret_cast<const qnmt::VsPart*>(parts), (int)G, N, live_scores, (int)k, cand_score, cand_tok,
                err_flag);
    QNMT_CHECK_LAUNCH("k_vocab_shard_combine");
    return QNMT_OK;
}
