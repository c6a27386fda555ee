// gemm_tcgen05.cu -- K3: int8 GEMM on the 5th-generation tensor cores.
//
//   D[m][n] = sum_k W[m][k] * X[n][k]    (both operands K-major int8)
//
// Replaces qmath.py:400-427 (qgemm_panel) for wide panels (batched decode:
// N = live hypotheses of many sentences; encoder input side: N = positions).
//
// Persistent, warp-specialised CTA (one per SM):
//   warp 0      TMA producer: W tile [128 x 128B] and X tile [BN x 128B] per
//               k-block into a STAGES-deep ring (SWIZZLE_128B), mbarrier
//               complete_tx signalling.
//   warp 1      TMEM allocator + single-thread MMA issuer:
//               tcgen05.mma.cta_group::1.kind::i8, M=128, N=BN, K=32 x4 per
//               k-block, int32 accumulators in TMEM (2 buffers -> the epilogue
//               of tile i overlaps the MMAs of tile i+1); tcgen05.commit frees
//               ring slots and publishes finished accumulators.
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x16 -> exact dequant
//               fl32(acc / (sw*sx)) (reciprocal fast path, __ddiv_rn near f32
//               midpoints) -> +bias -> (+Y) -> coalesced f32 stores of Y[n][m].
// Tiles are visited n-fastest so consecutive CTAs share the W block in L2.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "act.cuh"
#include "gemm.cuh"
#include "tc_mainloop.cuh"

namespace qnmt {

constexpr int TC_EPI_WARPS = 8;
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;

// ring depth: as many stages as fit ~200 KB of smem, at most 8
// (QNMT_TC_SMEM_KB: A/B builds with a shallower ring that leaves shared memory to other streams' CTAs)
#ifndef QNMT_TC_SMEM_KB
#define QNMT_TC_SMEM_KB 200
#endif
template <int BN>
using TcCfg = TcRing<BN, (QNMT_TC_SMEM_KB * 1024 / (TC_BM * TC_BK + BN * TC_BK)) < 8
                             ? (QNMT_TC_SMEM_KB * 1024 / (TC_BM * TC_BK + BN * TC_BK))
                             : 8>;

struct TcEpi {
    const float* w_scales;
    int64_t w_rows_per_scale;
    const float* x_scales;
    const int32_t* col_seg;
    const float* bias;
    float* Y;
    int64_t ldy;
    int64_t* acc_out;
    int32_t flags;
    const float* add1;
    int64_t ld1;
    const float* add2;
    int64_t ld2;
    GruEpi gru;
};

// EPI_ADD2: two precomputed f32 terms added in order after the bias (the readout's
// ((W_s s + b_r) + W_e e) + W_c c with W_e e and W_c c from stacked GEMMs)
// EPI_GATES / EPI_COMBINE: the GRU elementwise phases on the accumulators (GruEpi, gemm.cuh)
enum { EPI_BIAS = 1, EPI_ACCUMULATE = 2, EPI_RAW = 4, EPI_ADD2 = 8, EPI_GATES = 16, EPI_COMBINE = 32 };

// per-column max over the warp's 32 rows of |out| bits -> segmax[col_seg[n]]
__device__ __forceinline__ void gru_segmax(const TcEpi& e, const uint32_t (&mb)[16], int nbase, int ncols, int lane) {
    uint32_t mine = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t r = __reduce_max_sync(0xffffffffu, mb[j]);
        if (lane == j) mine = r;
    }
    if (lane < ncols && mine) atomicMax(e.gru.segmax + (e.col_seg ? e.col_seg[nbase + lane] : 0), mine);
}

// Epilogue warps (2..9) of one CTA: every tile of the persistent schedule
// (tile0, tile0 + tstep, ...) -> TMEM accumulator rows m_tile * mb + m_off + [0, 128)
// -> exact dequant (+ bias / + Y / + addends) -> f32 stores.  Shared by the
// 1-CTA kernel and the CTA-pair kernel (tempty_remote: shared::cluster address
// of the leader CTA's tempty barriers, 0 = local).
// Tile t -> (m-block, n-block).  group_m == 0: n fastest (consecutive CTAs share the
// weight block).  group_m > 0: bands of group_m m-blocks with the m-block fastest, so
// the tiles in flight at once touch ~group_m A blocks and ~(grid / group_m) B blocks
// -- an L2-resident working set for large products instead of one B block per tile.
__device__ __forceinline__ void tile_coords(int tile, int m_blocks, int n_blocks, int group_m, int& mb, int& nb) {
    if (group_m <= 0) {
        mb = tile / n_blocks;
        nb = tile % n_blocks;
        return;
    }
    const int band_tiles = group_m * n_blocks;
    const int band = tile / band_tiles;
    const int r = tile - band * band_tiles;
    const int m_base = band * group_m;
    const int gm = min(group_m, m_blocks - m_base);
    mb = m_base + r % gm;
    nb = r / gm;
}

// Split-K (k_gemm_tc with ksplit > 1): each split adds its int32 partial tile into the
// per-stream workspace ws[n][m] (RED.ADD, exact and order-free), then counts itself in
// cnt[tile]; the split that arrives last re-reads the complete sums, runs the normal
// dequant epilogue, and leaves ws and cnt zeroed for the next product.
struct TcSplit {
    int ksplit;
    int32_t* ws;
    int32_t* cnt;
};

// one 16-column chunk of the dequant epilogue from int32 accumulators already in registers
template <int EPI>
__device__ __forceinline__ void tc_epi_chunk(const TcEpi& e, const uint32_t (&r)[16], int m, bool mok, int nbase,
                                             int ncols, int M, float sw, float bias, double isw, const float* csx,
                                             const double* cisx) {
    float* yrow = e.Y + (int64_t)nbase * e.ldy + m;
    if (EPI & EPI_RAW) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (mok && j < ncols) e.acc_out[(int64_t)(nbase + j) * M + m] = (int)r[j];
        if (e.Y == nullptr) return;
    }
    uint32_t unsafe = 0;
    float yd[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const double q = i2d_exact((int)r[j]) * (isw * cisx[j]);
        yd[j] = __double2float_rn(q);
        unsafe |= (uint32_t)(!dequant_rcp_safe(q)) << j;
    }
    if (__any_sync(0xffffffffu, unsafe != 0)) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if ((unsafe >> j) & 1u) yd[j] = dequant((int)r[j], sw, csx[j]);
    }
    if (!mok) return;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j >= ncols) break;
        float y = yd[j];
        if (EPI & EPI_BIAS) y = __fadd_rn(y, bias);
        if (EPI & EPI_ACCUMULATE) y = __fadd_rn(yrow[(int64_t)j * e.ldy], y);
        if (EPI & EPI_ADD2)
            y = __fadd_rn(__fadd_rn(y, e.add1[(int64_t)(nbase + j) * e.ld1 + m]), e.add2[(int64_t)(nbase + j) * e.ld2 + m]);
        yrow[(int64_t)j * e.ldy] = y;
    }
}

template <int BN, int EPI>
__device__ __forceinline__ void tc_epilogue(const TcEpi& e, uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty,
                                            uint32_t tempty_remote, int tile0, int tstep, int tiles, int n_blocks,
                                            int m_tile, int m_off, int M, int N, float (*col_sx)[256],
                                            double (*col_isx)[256], int m_blocks = 0, int group_m = 0,
                                            TcSplit sk = TcSplit{1, nullptr, nullptr}, int* s_last = nullptr) {
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int ew = warp - 2;                 // 0..7
        const int lg = warp & 3;                 // TMEM lane group this warp may access
        const int half = ew >> 2;                // column half of the tile
        constexpr int COLS = BN / 2;
        int it = 0;
        for (int tile = tile0; tile < tiles; tile += tstep, ++it) {
            int mb, nb;
            const int mnt = sk.ksplit > 1 ? tile / sk.ksplit : tile;
            tile_coords(mnt, m_blocks, n_blocks, group_m, mb, nb);
            const int buf = it & 1;
            const uint32_t use = (uint32_t)(it >> 1) & 1u;
            // Column scales of this tile -> smem (x scale and its f64 reciprocal), row scale and
            // bias -> registers; all loads are issued before waiting for the accumulator.
            {
                const int c = ew * 32 + lane;    // 8 warps x 32 lanes cover BN <= 256 columns
                if (c < BN) {
                    const int n = nb * BN + c;
                    float sx = 1.0f;
                    if (n < N) sx = e.x_scales[e.col_seg ? e.col_seg[n] : 0];
                    col_sx[buf][c] = sx;
                    col_isx[buf][c] = 1.0 / (double)sx;
                }
            }
            const int m = mb * m_tile + m_off + lg * 32 + lane;
            const bool mok = m < M;
            float sw = 1.0f, bias = 0.0f;
            if (mok) {
                sw = e.w_scales[m / e.w_rows_per_scale];
                if (e.bias) bias = e.bias[m];
            }
            const double isw = 1.0 / (double)sw;
            asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI_WARPS));   // epilogue warps only
            tc::mbar_wait(&tfull[buf], use);
            tc::tc_fence_after();
            if (sk.ksplit > 1) {   // split-K: add the partial tile into the workspace
#pragma unroll 1
                for (int c0 = half * COLS; c0 < (half + 1) * COLS; c0 += 16) {
                    uint32_t r[16];
                    tc::tmem_ld16(tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * BN + c0), r);
                    const int nbase = nb * BN + c0;
                    const int ncols = min(16, N - nbase);
                    tc::tmem_ld_wait();
                    if (mok)
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (j < ncols) atomicAdd(&sk.ws[(int64_t)(nbase + j) * M + m], (int)r[j]);
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[buf]);   // TMEM buffer free for the next tile
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI_WARPS));
                if (ew == 0 && lane == 0) {
                    const int old = atomicAdd(&sk.cnt[mnt], 1);
                    *s_last = old == sk.ksplit - 1;
                    if (*s_last) sk.cnt[mnt] = 0;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(32 * TC_EPI_WARPS));
                if (!*s_last) continue;
                __threadfence();
#pragma unroll 1
                for (int c0 = half * COLS; c0 < (half + 1) * COLS; c0 += 16) {
                    const int nbase = nb * BN + c0;
                    const int ncols = min(16, N - nbase);
                    if (ncols <= 0) continue;
                    uint32_t r[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        r[j] = 0u;
                        if (mok && j < ncols) {
                            int32_t* w = &sk.ws[(int64_t)(nbase + j) * M + m];
                            r[j] = (uint32_t)__ldcg(w);
                            *w = 0;
                        }
                    }
                    tc_epi_chunk<EPI>(e, r, m, mok, nbase, ncols, M, sw, bias, isw, &col_sx[buf][c0],
                                      &col_isx[buf][c0]);
                }
                continue;
            }
#pragma unroll 1
            for (int c0 = half * COLS; c0 < (half + 1) * COLS; c0 += 16) {
                uint32_t r[16];
                const uint32_t ta = tmem_base + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * BN + c0);
                tc::tmem_ld16(ta, r);
                const int nbase = nb * BN + c0;
                const int ncols = min(16, N - nbase);          // warp-uniform
                if (ncols <= 0) {
                    tc::tmem_ld_wait();
                    continue;
                }
                float* yrow = e.Y + (int64_t)nbase * e.ldy + m;
                float yv[16], a1v[16], a2v[16];
                // GRU epilogues: addend g, previous state h and (combine) z of this thread's row
                float gv[16], hv[16], zv[16];
                const int64_t gH = e.gru.H;
                const bool g_row = (EPI & EPI_COMBINE) || ((EPI & EPI_GATES) && m < 2 * gH);   // row gets the GRU op
                const bool g_rrow = (EPI & EPI_GATES) && m >= gH && m < 2 * gH;               // reset-gate row
                if (EPI & (EPI_GATES | EPI_COMBINE)) {
                    const int64_t hm = (EPI & EPI_COMBINE) ? m : m - gH;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const bool ok = mok && j < ncols;
                        gv[j] = (ok && g_row) ? e.gru.g[(int64_t)(nbase + j) * e.gru.ldg + m] : 0.0f;
                        hv[j] = (ok && ((EPI & EPI_COMBINE) || g_rrow)) ? e.gru.h[(int64_t)(nbase + j) * e.gru.ldh + hm] : 0.0f;
                        if (EPI & EPI_COMBINE) zv[j] = ok ? e.gru.z[(int64_t)(nbase + j) * gH + m] : 0.0f;
                    }
                }
                if (EPI & EPI_ACCUMULATE) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) yv[j] = (mok && j < ncols) ? yrow[(int64_t)j * e.ldy] : 0.0f;
                }
                if (EPI & EPI_ADD2) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        a1v[j] = (mok && j < ncols) ? e.add1[(int64_t)(nbase + j) * e.ld1 + m] : 0.0f;
                        a2v[j] = (mok && j < ncols) ? e.add2[(int64_t)(nbase + j) * e.ld2 + m] : 0.0f;
                    }
                }
                tc::tmem_ld_wait();
                if (EPI & EPI_RAW) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (mok && j < ncols) e.acc_out[(int64_t)(nbase + j) * M + m] = (int)r[j];
                    if (e.Y == nullptr) continue;
                }
                // branch-free fast dequant; lanes flag elements near an f32 rounding midpoint
                uint32_t unsafe = 0;
                float yd[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const double q = i2d_exact((int)r[j]) * (isw * col_isx[buf][c0 + j]);
                    yd[j] = __double2float_rn(q);
                    unsafe |= (uint32_t)(!dequant_rcp_safe(q)) << j;
                }
                if (__any_sync(0xffffffffu, unsafe != 0)) {   // rare: exact division for flagged elements
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if ((unsafe >> j) & 1u) yd[j] = dequant((int)r[j], sw, col_sx[buf][c0 + j]);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float y = yd[j];
                    if (EPI & EPI_BIAS) y = __fadd_rn(y, bias);
                    if (EPI & EPI_ACCUMULATE) y = __fadd_rn(yv[j], y);
                    if (EPI & EPI_ADD2) y = __fadd_rn(__fadd_rn(y, a1v[j]), a2v[j]);
                    yd[j] = y;
                }
                if (EPI & (EPI_GATES | EPI_COMBINE)) {
                    // a warp's 32 rows lie on one side of the H / 2H boundaries (H % 32 == 0, checked by the host)
                    const bool wg = __any_sync(0xffffffffu, g_row);
                    if (wg) {
                        uint32_t mb_[16];
                        bool bad = false;
                        float vo[16], sg[16];
                        // arithmetic first (branch-free, 16 independent fp64 chains), stores after
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const float p = __fadd_rn(gv[j], yd[j]);   // fadd is commutative: (x + h) as fused_q.cu
                            bad |= mok && j < ncols && g_row && !is_finite_f(p);
                            if (EPI & EPI_COMBINE) {
                                vo[j] = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zv[j]), hv[j]), __fmul_rn(zv[j], tanh_b(p)));
                            } else {
                                sg[j] = sigmoid_b(p);
                                vo[j] = __fmul_rn(sg[j], hv[j]);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const bool ok = mok && j < ncols && g_row;
                            if (EPI & EPI_COMBINE) {
                                if (ok) e.gru.out[(int64_t)(nbase + j) * e.gru.ldo + m] = vo[j];
                            } else {
                                if (ok && !g_rrow) e.gru.z[(int64_t)(nbase + j) * gH + m] = sg[j];
                                if (ok && g_rrow) e.gru.out[(int64_t)(nbase + j) * e.gru.ldo + (m - gH)] = vo[j];
                            }
                            mb_[j] = (ok && ((EPI & EPI_COMBINE) || g_rrow)) ? (__float_as_uint(vo[j]) & 0x7fffffffu) : 0u;
                        }
                        if (bad) set_flag(e.gru.err_flag, QNMT_FLAG_NUMERIC);
                        gru_segmax(e, mb_, nbase, ncols, lane);
                    }
                    if ((EPI & EPI_COMBINE) || wg) continue;   // no plain store for GRU rows
                }
                if (mok && ncols == 16) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) yrow[(int64_t)j * e.ldy] = yd[j];
                } else if (mok) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < ncols) yrow[(int64_t)j * e.ldy] = yd[j];
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (tempty_remote)   // 2-CTA pair: the leader's MMA warp waits for both CTAs' epilogues
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tempty_remote + 8u * buf)
                                 : "memory");
                else
                    tc::mbar_arrive(&tempty[buf]);
            }
        }
    }

template <int BN, int EPI>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
          TcEpi e, const int32_t* n_dev, TcSplit sk, int pre) {
    using C = TcCfg<BN>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const TcBars<C> bars(smem);
    __shared__ float col_sx[2][256];      // per-column activation scale (double-buffered by tile)
    __shared__ double col_isx[2][256];    // and its f64 reciprocal

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    pdl_trigger();
    const uint32_t tmem_base = tc_setup<C>(&tmA, &tmB, bars, TC_EPI_WARPS);
    // static weights, host-known N: the first tile's weight blocks stream while the predecessor runs
    if (pre > 0 && warp == 0 && lane == 0) tc_prefetch_a<C>(&tmA, smem, bars, (N + BN - 1) / BN, pre);
    pdl_wait();   // everything above overlaps the predecessor kernel (PDL)
    if (n_dev) N = min(N, *n_dev);   // graph mode: live columns from the device
    const int m_blocks = (M + TC_BM - 1) / TC_BM;
    const int n_blocks = (N + BN - 1) / BN;
    const int tiles = m_blocks * n_blocks * sk.ksplit;
    const int k_blocks = (K + TC_BK - 1) / TC_BK;
    __shared__ int s_last;

    if (warp == 0) {
        tc_produce<C, BN>(&tmA, &tmB, smem, bars, tiles, n_blocks, k_blocks, -1, 0, sk.ksplit, pre);
    } else if (warp == 1) {
        tc_issue<C, BN>(smem, bars, tmem_base, tiles, k_blocks, -1, 0, sk.ksplit);
    } else {
        tc_epilogue<BN, EPI>(e, tmem_base, bars.tfull, bars.tempty, 0u, blockIdx.x, gridDim.x, tiles, n_blocks,
                             TC_BM, 0, M, N, col_sx, col_isx, 0, 0, sk, &s_last);
    }
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}


// ---------------------------------------------------------------------------
// Two products of one shape in ONE launch (the encoder's per-direction U_zr h and
// U_c (r*h): same M, N, K, different weights / activations / outputs).  At decode
// sizes a tcgen05 product is ~8 us of prologue, pipeline fill and epilogue for
// well under 1 us of MMA; the two directions' CTAs run side by side instead
// of back to back.  CTAs [0, per) take product 0, [per, 2 per) product 1, each
// with k_gemm_tc's persistent tile loop over its own product.
// ---------------------------------------------------------------------------
template <int BN, int EPI>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_gemm_tc_dual(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
               const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1, int M, int N, int K,
               const __grid_constant__ TcEpi e0, const __grid_constant__ TcEpi e1, const int32_t* n_dev, int per) {
    using C = TcCfg<BN>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const TcBars<C> bars(smem);
    __shared__ float col_sx[2][256];
    __shared__ double col_isx[2][256];
    const int warp = threadIdx.x >> 5;
    const bool second = (int)blockIdx.x >= per;
    const int local = (int)blockIdx.x - (second ? per : 0);
    const CUtensorMap* tmA = second ? &tmA1 : &tmA0;
    const CUtensorMap* tmB = second ? &tmB1 : &tmB0;
    const TcEpi& e = second ? e1 : e0;
    pdl_trigger();
    const uint32_t tmem_base = tc_setup<C>(tmA, tmB, bars, TC_EPI_WARPS);
    pdl_wait();
    if (n_dev) N = min(N, *n_dev);
    const int m_blocks = (M + TC_BM - 1) / TC_BM;
    const int n_blocks = (N + BN - 1) / BN;
    const int tiles = m_blocks * n_blocks;
    const int k_blocks = (K + TC_BK - 1) / TC_BK;
    if (warp == 0) {
        tc_produce<C, BN>(tmA, tmB, smem, bars, tiles, n_blocks, k_blocks, local, per);
    } else if (warp == 1) {
        tc_issue<C, BN>(smem, bars, tmem_base, tiles, k_blocks, local, per);
    } else {
        tc_epilogue<BN, EPI>(e, tmem_base, bars.tfull, bars.tempty, 0u, local, per, tiles, n_blocks, TC_BM, 0, M, N,
                             col_sx, col_isx);
    }
    __syncthreads();
    if (warp == 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc<C::TMEM_COLS>(tmem_base);
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant for large products (tcgen05.mma.cta_group::2, M = 256).
// A cluster of two CTAs on one TPC computes a 256 x BN tile: CTA r loads A rows
// [256 mb + 128 r, +128) and B rows [BN nb + BN/2 r, +BN/2) into its own
// shared memory; the leader (rank 0) issues the M = 256 MMAs, which read A and
// B from both CTAs and accumulate rows 128 r .. of the tile in CTA r's TMEM.
// Per CTA the ring carries 32 KB per k-block instead of 48 KB for the same MMA
// work (BN = 256), which is what lets the tensor pipe run at the int8 rate
// (single-CTA M = 128 tiles are shared-memory-bandwidth bound).  TMA loads of
// both CTAs complete on the leader's full barrier (cta_group::2 TMA); MMA
// commits multicast to both CTAs' empty / tmem-full barriers; both CTAs'
// epilogues release a TMEM buffer on the leader's tmem-empty barrier.
// ---------------------------------------------------------------------------
constexpr int TC2_GROUP_M = 16;  // tile rasterization band of the pair kernel (see tile_coords; swept 0..32)

template <int BN>
struct Tc2Ring {
    static constexpr int A_BYTES = TC_BM * TC_BK;
    static constexpr int B_BYTES = (BN / 2) * TC_BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024 / STAGE_BYTES) < 8 ? (200 * 1024 / STAGE_BYTES) : 8;
    static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_in_rank(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tc::smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(tc::smem_u32(dst)), "l"(map), "r"(leader_bar), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {   // arrive on bar in both CTAs
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(tc::smem_u32(bar)), "h"((uint16_t)3)
                 : "memory");
}

template <int BN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
k_gemm_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
           TcEpi e, int group_m) {
    using C = Tc2Ring<BN>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const TcBars<C> bars(smem);
    __shared__ float col_sx[2][256];
    __shared__ double col_isx[2][256];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    pdl_trigger();
    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&tmA);
        tc::prefetch_tmap(&tmB);
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&bars.full[s], 1);
            tc::mbar_init(&bars.empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&bars.tfull[i], 1);
            tc::mbar_init(&bars.tempty[i], 2 * TC_EPI_WARPS);
        }
        tc::fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tc::smem_u32(bars.tmem_slot)), "n"(C::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc::tc_fence_before();
    cluster_sync_all();
    tc::tc_fence_after();
    const uint32_t tmem_base = *bars.tmem_slot;
    pdl_wait();
    const int m_blocks = (M + 2 * TC_BM - 1) / (2 * TC_BM);
    const int n_blocks = (N + BN - 1) / BN;
    const int tiles = m_blocks * n_blocks;
    const int k_blocks = (K + TC_BK - 1) / TC_BK;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    if (warp == 0) {
        if (lane == 0) {
            const uint32_t full0 = smem_in_rank(bars.full, 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = cid; tile < tiles; tile += ncl) {
                int mb, nb;
                tile_coords(tile, m_blocks, n_blocks, group_m, mb, nb);
                for (int kb = 0; kb < k_blocks; ++kb) {
                    tc::mbar_wait(&bars.empty[stage], phase ^ 1);
                    unsigned char* sa = smem + stage * C::STAGE_BYTES;
                    unsigned char* sb = sa + C::A_BYTES;
                    if (rank == 0) tc::mbar_arrive_expect_tx(&bars.full[stage], 2 * C::STAGE_BYTES);
                    tma_load_2d_pair(sa, &tmA, full0 + 8u * stage, kb * TC_BK, mb * 2 * TC_BM + (int)rank * TC_BM);
                    tma_load_2d_pair(sb, &tmB, full0 + 8u * stage, kb * TC_BK, nb * BN + (int)rank * (BN / 2));
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            constexpr uint32_t IDESC = tc::idesc_i8(2 * TC_BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = cid; tile < tiles; tile += ncl, ++it) {
                const int buf = it & 1;
                const uint32_t use = (uint32_t)(it >> 1) & 1u;
                tc::mbar_wait(&bars.tempty[buf], use ^ 1);
                tc::tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(buf * BN);
                for (int kb = 0; kb < k_blocks; ++kb) {
                    tc::mbar_wait(&bars.full[stage], phase);
                    tc::tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = tc::smem_u32(smem + stage * C::STAGE_BYTES);
                        const uint32_t b0 = a0 + C::A_BYTES;
#pragma unroll
                        for (int k = 0; k < TC_BK / 32; ++k)
                            mma_i8_pair(d, tc::sw128_kmajor_desc(a0 + 32 * k), tc::sw128_kmajor_desc(b0 + 32 * k),
                                        IDESC, (kb | k) != 0);
                        mma_commit_pair(&bars.empty[stage]);
                        if (kb == k_blocks - 1) mma_commit_pair(&bars.tfull[buf]);
                    }
                    __syncwarp();
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else {
        tc_epilogue<BN, EPI>(e, tmem_base, bars.tfull, bars.tempty, rank ? smem_in_rank(bars.tempty, 0) : 0u, cid, ncl,
                             tiles, n_blocks, 2 * TC_BM, (int)rank * TC_BM, M, N, col_sx, col_isx, m_blocks,
                             group_m);
    }
    tc::tc_fence_before();
    cluster_sync_all();   // both CTAs finished: no MMA writes or remote arrivals pending
    if (warp == 1) {
        tc::tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(C::TMEM_COLS)
                     : "memory");
    }
}

// ---------------------------------------------------------------------------
// host side: tensor maps (cached per (pointer, shape)) and launch
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

struct MapKey {
    const void* p;
    int64_t rows, cols, ld;
    int box_rows;
    bool operator==(const MapKey& o) const {
        return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        return std::hash<const void*>()(k.p) ^ (size_t)(k.rows * 1315423911u) ^ (size_t)(k.cols << 20) ^
               (size_t)(k.ld * 2654435761u) ^ (size_t)k.box_rows;
    }
};

int tc_get_map(const int8_t* p, int64_t rows, int64_t cols, int64_t ld, int box_rows, CUtensorMap* out) {
    static std::mutex mu;
    static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    MapKey key{p, rows, cols, ld, box_rows};
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return QNMT_OK;
    }
    EncodeTiledFn fn = encode_fn();
    if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return QNMT_ERR_CUDA; }
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)p, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return QNMT_ERR_CUDA; }
    if (cache.size() > 4096) cache.clear();
    cache[key] = m;
    *out = m;
    return QNMT_OK;
}

int tc_sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// ---------------------------------------------------------------------------
// split-K workspace: one zeroed int32 [N][M] buffer + tile counters per stream
// (kernels on one stream run in order; engines own their streams).  Grown only
// outside stream capture; a captured product that finds it too small runs
// without splitting.  tc_split_reserve lets an engine size it before capture.
// ---------------------------------------------------------------------------
struct SplitWs {
    int32_t* ws = nullptr;
    size_t ws_elems = 0;
    int32_t* cnt = nullptr;
    size_t cnt_elems = 0;
};
static std::mutex g_ws_mu;
static std::unordered_map<cudaStream_t, SplitWs> g_ws;
int g_tc_split = 0;   // 1: split K for tile-starved products (A/B: cfg1 B=64 21.4 vs 14.4 us, off)

static bool split_ws(cudaStream_t st, size_t ws_elems, size_t cnt_elems, TcSplit& sk) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    SplitWs& w = g_ws[st];
    if (w.ws_elems < ws_elems || w.cnt_elems < cnt_elems) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
        if (cudaStreamSynchronize(st) != cudaSuccess) return false;   // the old buffers may be in use
        std::unique_lock<std::shared_mutex> gate(g_capture_gate);     // cudaFree synchronises the device
        cudaFree(w.ws);
        cudaFree(w.cnt);
        w = SplitWs{};
        const size_t we = std::max(ws_elems, (size_t)1 << 20), ce = std::max(cnt_elems, (size_t)4096);
        if (cudaMalloc(&w.ws, we * sizeof(int32_t)) != cudaSuccess) return false;
        if (cudaMalloc(&w.cnt, ce * sizeof(int32_t)) != cudaSuccess) {
            cudaFree(w.ws);
            w = SplitWs{};
            return false;
        }
        if (cudaMemsetAsync(w.ws, 0, we * sizeof(int32_t), st) != cudaSuccess ||
            cudaMemsetAsync(w.cnt, 0, ce * sizeof(int32_t), st) != cudaSuccess)
            return false;
        w.ws_elems = we;
        w.cnt_elems = ce;
    }
    sk.ws = w.ws;
    sk.cnt = w.cnt;
    return true;
}

int tc_split_reserve(cudaStream_t st, int64_t ws_elems, int64_t tiles) {
    TcSplit sk{1, nullptr, nullptr};
    return split_ws(st, (size_t)ws_elems, (size_t)tiles, sk) ? QNMT_OK : QNMT_ERR_CUDA;
}

// K splits for a product of `tiles` output tiles and k_blocks k-blocks: enough CTAs to
// cover half the SMs or more, >= 2 k-blocks per split... but never past one wave
static int choose_ksplit(int64_t tiles, int64_t k_blocks, int sms) {
    if (!g_tc_split || tiles * 2 > sms || k_blocks < 2) return 1;
    const int64_t req = std::min<int64_t>({k_blocks, sms / tiles, 16});
    if (req < 2) return 1;
    const int64_t kpb = cdiv(k_blocks, req);
    return (int)cdiv(k_blocks, kpb);
}

// static weight blocks requested before the PDL wait (QNMT_TC_PREFETCH_W=0 for A/B runs)
static const int g_tc_prefetch_w = [] {
    const char* v = getenv("QNMT_TC_PREFETCH_W");
    return v ? atoi(v) : 1;
}();

template <int BN, int EPI>
static int launch_tc(const GemmArgs& g, cudaStream_t st) {
    using C = TcCfg<BN>;
    static size_t attr_done = 0;
    QNMT_CUDA(raise_smem_limit((const void*)k_gemm_tc<BN, EPI>, C::SMEM, attr_done));
    CUtensorMap ta, tb;
    int rc = tc_get_map(g.W, g.M, g.K, g.ldw, TC_BM, &ta);
    if (rc) return rc;
    rc = tc_get_map(g.X, g.N, g.K, g.ldx, BN, &tb);
    if (rc) return rc;
    TcEpi e{g.w_scales, g.w_rows_per_scale, g.x_scales, g.col_seg, g.bias, g.Y, g.ldy, g.acc_out, g.flags,
            g.add1, g.ld1, g.add2, g.ld2, g.gru};
    int tiles = (int)(cdiv(g.M, TC_BM) * cdiv(g.N, BN));
    TcSplit sk{(EPI & (EPI_GATES | EPI_COMBINE)) ? 1 : choose_ksplit(tiles, cdiv(g.K, TC_BK), tc_sm_count()), nullptr,
               nullptr};
    if (sk.ksplit > 1 && !split_ws(st, (size_t)g.M * g.N, (size_t)tiles, sk)) sk.ksplit = 1;
    tiles *= sk.ksplit;
    int grid = tiles < tc_sm_count() ? tiles : tc_sm_count();
    auto kfn = k_gemm_tc<BN, EPI>;
    // weights flagged static (not written by the predecessor kernel): request the first tile's
    // A blocks before the PDL wait (not in graph-captured steps: N is device-side there)
    const int kb_all = (int)cdiv(g.K, TC_BK);
    const int pre = ((g.flags & QNMT_GEMM_W_STATIC) && !tl_ndev && sk.ksplit == 1 && g_tc_prefetch_w)
                        ? (kb_all < C::STAGES ? kb_all : C::STAGES) : 0;
    QNMT_LAUNCH(kfn, grid, TC_THREADS, C::SMEM, st, ta, tb, (int)g.M, (int)g.N, (int)g.K, e, tl_ndev, sk, pre);
    QNMT_CHECK_LAUNCH("k_gemm_tc");
    return QNMT_OK;
}

int g_tc_pair = 1;   // 0: never use the CTA-pair kernel (A/B testing)
// tile width of the GRU-epilogue GEMMs ([0] gates, [1] combine); 0 = the general rule
int g_gru_bn[2] = {0, 0};
static const int g_gru_bn_env = [] {   // QNMT_GRU_BN="gates,combine" (A/B runs)
    const char* v = getenv("QNMT_GRU_BN");
    if (v) sscanf(v, "%d,%d", &g_gru_bn[0], &g_gru_bn[1]);
    return 0;
}();

template <int EPI>
static int launch_tc2(const GemmArgs& g, cudaStream_t st) {
    constexpr int BN = 256;
    using C = Tc2Ring<BN>;
    static size_t attr_done = 0;
    QNMT_CUDA(raise_smem_limit((const void*)k_gemm_tc2<BN, EPI>, C::SMEM, attr_done));
    CUtensorMap ta, tb;
    int rc = tc_get_map(g.W, g.M, g.K, g.ldw, TC_BM, &ta);
    if (rc) return rc;
    rc = tc_get_map(g.X, g.N, g.K, g.ldx, BN / 2, &tb);
    if (rc) return rc;
    TcEpi e{g.w_scales, g.w_rows_per_scale, g.x_scales, g.col_seg, g.bias, g.Y, g.ldy, g.acc_out, g.flags,
            g.add1, g.ld1, g.add2, g.ld2, GruEpi{}};
    const int tiles = (int)(cdiv(g.M, 2 * TC_BM) * cdiv(g.N, BN));
    const int pairs = tc_sm_count() / 2;
    const int grid = 2 * (tiles < pairs ? tiles : pairs);
    static const int group_m = [] {
        const char* v = getenv("QNMT_TC2_GROUP_M");   // (tuning knob; default TC2_GROUP_M)
        return v ? atoi(v) : TC2_GROUP_M;
    }();
    QNMT_LAUNCH(k_gemm_tc2<BN, EPI>, grid, TC_THREADS, C::SMEM, st, ta, tb, (int)g.M, (int)g.N, (int)g.K, e, group_m);
    QNMT_CHECK_LAUNCH("k_gemm_tc2");
    return QNMT_OK;
}


template <int BN>
static int launch_tc_dual(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t st) {
    using C = TcCfg<BN>;
    static size_t attr_done = 0;
    QNMT_CUDA(raise_smem_limit((const void*)k_gemm_tc_dual<BN, 0>, C::SMEM, attr_done));
    CUtensorMap ta0, tb0, ta1, tb1;
    int rc = tc_get_map(g0.W, g0.M, g0.K, g0.ldw, TC_BM, &ta0);
    if (!rc) rc = tc_get_map(g0.X, g0.N, g0.K, g0.ldx, BN, &tb0);
    if (!rc) rc = tc_get_map(g1.W, g1.M, g1.K, g1.ldw, TC_BM, &ta1);
    if (!rc) rc = tc_get_map(g1.X, g1.N, g1.K, g1.ldx, BN, &tb1);
    if (rc) return rc;
    const TcEpi e0{g0.w_scales, g0.w_rows_per_scale, g0.x_scales, g0.col_seg, g0.bias, g0.Y, g0.ldy, nullptr, g0.flags,
                   nullptr, 0, nullptr, 0, GruEpi{}};
    const TcEpi e1{g1.w_scales, g1.w_rows_per_scale, g1.x_scales, g1.col_seg, g1.bias, g1.Y, g1.ldy, nullptr, g1.flags,
                   nullptr, 0, nullptr, 0, GruEpi{}};
    const int tiles = (int)(cdiv(g0.M, TC_BM) * cdiv(g0.N, BN));
    const int half = tc_sm_count() / 2;
    const int per = tiles < half ? tiles : half;
    auto kfn = k_gemm_tc_dual<BN, 0>;
    QNMT_LAUNCH(kfn, 2 * per, TC_THREADS, C::SMEM, st, ta0, tb0, ta1, tb1, (int)g0.M, (int)g0.N, (int)g0.K, e0, e1,
                tl_ndev, per);
    QNMT_CHECK_LAUNCH("k_gemm_tc_dual");
    return QNMT_OK;
}

// two plain products (no bias / accumulate / addends) of one shape in one launch; false = not eligible
bool gemm_tc_dual_eligible(const GemmArgs& g0, const GemmArgs& g1) {
    static const int enabled = [] {
        const char* v = getenv("QNMT_TC_DUAL");   // (A/B runs)
        return v ? atoi(v) : 1;
    }();
    return enabled && g0.M == g1.M && g0.N == g1.N && g0.K == g1.K && g0.N > 8 && !g0.bias && !g1.bias &&
           !g0.acc_out && !g1.acc_out && !g0.add1 && !g1.add1 && !g0.gru.mode && !g1.gru.mode &&
           !(g0.flags & QNMT_GEMM_ACCUMULATE) && !(g1.flags & QNMT_GEMM_ACCUMULATE) && tc_eligible(g0) &&
           tc_eligible(g1) && g_gemm_impl != 1;
}

int gemm_tc_dual_launch(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t st) {
    const int64_t mb = cdiv(g0.M, TC_BM);
    const int half = tc_sm_count() / 2;
    static const int cand[] = {64, 96, 128, 160, 192, 224, 256};
    int bn = 256;
    int64_t best = INT64_MAX;
    for (int b : cand) {   // fewest waves over half the SMs, then the narrowest tile
        const int64_t waves = cdiv(mb * cdiv(g0.N, b), half);
        if (waves < best) {
            best = waves;
            bn = b;
        }
    }
    switch (bn) {
        case 64: return launch_tc_dual<64>(g0, g1, st);
        case 96: return launch_tc_dual<96>(g0, g1, st);
        case 128: return launch_tc_dual<128>(g0, g1, st);
        case 160: return launch_tc_dual<160>(g0, g1, st);
        case 192: return launch_tc_dual<192>(g0, g1, st);
        case 224: return launch_tc_dual<224>(g0, g1, st);
        default: return launch_tc_dual<256>(g0, g1, st);
    }
}

bool tc_eligible(const GemmArgs& g) {
    return g.K % 16 == 0 && g.ldw % 16 == 0 && g.ldx % 16 == 0 && ((uintptr_t)g.W % 16 == 0) &&
           ((uintptr_t)g.X % 16 == 0) && g.K <= QNMT_INT32_SAFE_K && g.K > 0 && g.M < (1 << 30) &&
           g.N < (1 << 30);
}

int gemm_tc_launch(const GemmArgs& g, cudaStream_t st) {
    const int64_t mb = cdiv(g.M, TC_BM);
    const int sms = tc_sm_count();
    const int epi = (g.bias ? EPI_BIAS : 0) | ((g.flags & QNMT_GEMM_ACCUMULATE) ? EPI_ACCUMULATE : 0) |
                    (g.acc_out ? EPI_RAW : 0) | (g.add1 ? EPI_ADD2 : 0) | (g.gru.mode == 1 ? EPI_GATES : 0) |
                    (g.gru.mode == 2 ? EPI_COMBINE : 0);
    if (g.gru.mode) {
        if (g.gru.H % 32 != 0 || !g.gru.g || !g.gru.h || !g.gru.z || !g.gru.out || !g.gru.segmax ||
            (g.gru.mode == 1 && (epi != (EPI_BIAS | EPI_GATES) || g.M < 2 * g.gru.H)) ||
            (g.gru.mode == 2 && (epi != EPI_COMBINE || g.M != g.gru.H))) {
            set_error("gemm_tc: bad GRU epilogue arguments (mode %d epi %d M %lld H %lld)", g.gru.mode, epi,
                      (long long)g.M, (long long)g.gru.H);
            return QNMT_ERR_CONFIG;
        }
    }
    // large products (at least two waves of 256 x 256 pair tiles, not graph-captured): CTA pairs
    if (g_tc_pair && !tl_ndev && !(epi & (EPI_ADD2 | EPI_GATES | EPI_COMBINE)) && g.M >= 2 * TC_BM && g.N >= 256 &&
        cdiv(g.M, 2 * TC_BM) * cdiv(g.N, 256) >= sms) {
        switch (epi) {
            case 0: return launch_tc2<0>(g, st);
            case 1: return launch_tc2<1>(g, st);
            case 2: return launch_tc2<2>(g, st);
            case 3: return launch_tc2<3>(g, st);
            case 4: return launch_tc2<4>(g, st);
            case 5: return launch_tc2<5>(g, st);
            case 6: return launch_tc2<6>(g, st);
            case 7: return launch_tc2<7>(g, st);
            default: break;
        }
    }
    int bn;
    if (epi & EPI_RAW) {   // op-API accumulator export: three tile widths
        bn = (g.N > 128 && mb * cdiv(g.N, 256) >= sms) ? 256 : (g.N > 64 && mb * cdiv(g.N, 128) >= sms / 2) ? 128 : 64;
    } else {
        // fewest waves of tiles over the SMs, then the narrowest tile (less B data and epilogue
        // per tile, more CTAs): e.g. N = 1280 -> M 2048: 160 (128 tiles), M 3072: 256, M 1024: 96
        static const int cand[] = {64, 96, 128, 160, 192, 224, 256};
        static const int forced = [] {   // (tuning knob: QNMT_TC_BN forces one tile width)
            const char* v = getenv("QNMT_TC_BN");
            return v ? atoi(v) : 0;
        }();
        bn = 256;
        int64_t best = INT64_MAX;
        for (int b : cand) {
            const int64_t waves = cdiv(mb * cdiv(g.N, b), sms);
            if (waves < best) {
                best = waves;
                bn = b;
            }
        }
        if (forced) bn = forced;
        if (g.gru.mode && g_gru_bn[g.gru.mode - 1]) bn = g_gru_bn[g.gru.mode - 1];
    }
#define QNMT_TC_CASE(BN_, E_) \
    if (bn == BN_ && epi == E_) return launch_tc<BN_, E_>(g, st);
#define QNMT_TC_BN4(BN_) QNMT_TC_CASE(BN_, 0) QNMT_TC_CASE(BN_, 1) QNMT_TC_CASE(BN_, 2) QNMT_TC_CASE(BN_, 3)
#define QNMT_TC_BN8(BN_) QNMT_TC_BN4(BN_) QNMT_TC_CASE(BN_, 4) QNMT_TC_CASE(BN_, 5) QNMT_TC_CASE(BN_, 6) QNMT_TC_CASE(BN_, 7)
    QNMT_TC_BN8(256) QNMT_TC_BN8(128) QNMT_TC_BN8(64)
    QNMT_TC_BN4(96) QNMT_TC_BN4(160) QNMT_TC_BN4(192) QNMT_TC_BN4(224)
    QNMT_TC_CASE(64, 9) QNMT_TC_CASE(96, 9) QNMT_TC_CASE(128, 9) QNMT_TC_CASE(160, 9) QNMT_TC_CASE(192, 9)
    QNMT_TC_CASE(224, 9) QNMT_TC_CASE(256, 9)
#define QNMT_TC_GRU(BN_) QNMT_TC_CASE(BN_, 17) QNMT_TC_CASE(BN_, 32)
    QNMT_TC_GRU(64) QNMT_TC_GRU(96) QNMT_TC_GRU(128) QNMT_TC_GRU(160) QNMT_TC_GRU(192) QNMT_TC_GRU(224) QNMT_TC_GRU(256)
#undef QNMT_TC_GRU
#undef QNMT_TC_BN4
#undef QNMT_TC_BN8
#undef QNMT_TC_CASE
    set_error("gemm_tc: no kernel for bn=%d epi=%d", bn, epi);
    return QNMT_ERR_CONFIG;
}

}  // namespace qnmt

extern "C" int qnmt_set_tc_split(int enable) {
    const int old = qnmt::g_tc_split;
    qnmt::g_tc_split = enable;
    return old;
}

// tile widths of the GRU-epilogue GEMMs (0 = general rule); returns the old gates width
extern "C" int qnmt_set_gru_epi_bn(int gates_bn, int combine_bn) {
    const int old = qnmt::g_gru_bn[0];
    auto okbn = [](int b) { return b == 0 || (b >= 64 && b <= 256 && b % 32 == 0); };
    if (okbn(gates_bn)) qnmt::g_gru_bn[0] = gates_bn;
    if (okbn(combine_bn)) qnmt::g_gru_bn[1] = combine_bn;
    return old;
}

extern "C" int qnmt_set_tc_pair(int enable) {
    const int old = qnmt::g_tc_pair;
    qnmt::g_tc_pair = enable;
    return old;
}
