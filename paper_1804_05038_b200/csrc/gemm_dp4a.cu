// gemm_dp4a.cu -- int8 x int8 -> int32 products on CUDA cores with the fused
// dequant / bias / accumulate epilogue.
//
// Replaces qmath.py:400-427 (qgemm_panel), :302-328 (_panel_vnni), :243-299
// (_vnni_dot64), :331-360 (_panel_maddw), :205-228 (naive kernels), and the
// epilogue of :379-381 + layers.py:144-145.
//
//   k_gemv<ROWS, NC>  : N <= 8 columns (beam-sized panels, batch-1 latency path).
//                       Each warp streams ROWS weight rows with 16-byte
//                       L1-bypassing loads (every weight byte read once), the
//                       NC activation columns come through the read-only path
//                       (L1 hits shared by all warps), dp4a, warp butterfly sum.
//   k_gemm_tile       : N > 8, 64x64x64 smem-tiled dp4a (interim bulk path;
//                       the tcgen05 kernel in gemm_tcgen05.cu supersedes it
//                       where it applies).
//   k_gemm_generic    : any alignment, int64 accumulation for K > INT32_SAFE_K.
#include "common.cuh"
#include "gemm.cuh"

namespace qnmt {

struct EpiArgs {
    const float* w_scales;
    int64_t w_rows_per_scale;
    const float* x_scales;
    const int32_t* col_seg;
    const float* bias;
    float* Y;
    int64_t ldy;
    int64_t* acc_out;
    int64_t M;
    int32_t flags;
    const float* add1 = nullptr;   // y = ((dq + bias) + add1[n][m]) + add2[n][m] (stacked readout terms)
    int64_t ld1 = 0;
    const float* add2 = nullptr;
    int64_t ld2 = 0;
};

__device__ __forceinline__ void epilogue(const EpiArgs& e, int64_t m, int64_t n, long long acc) {
    if (e.acc_out) e.acc_out[n * e.M + m] = acc;
    if (!e.Y) return;
    float sw = e.w_scales[m / e.w_rows_per_scale];
    float sx = e.x_scales[e.col_seg ? e.col_seg[n] : 0];
    float y = dequant_rcp(acc, (1.0 / (double)sw) * (1.0 / (double)sx), sw, sx);
    if (e.bias) y = __fadd_rn(y, e.bias[m]);
    float* dst = e.Y + n * e.ldy + m;
    if (e.flags & QNMT_GEMM_ACCUMULATE) y = __fadd_rn(*dst, y);
    if (e.add1) y = __fadd_rn(__fadd_rn(y, e.add1[n * e.ld1 + m]), e.add2[n * e.ld2 + m]);
    *dst = y;
}

__device__ __forceinline__ int dp4a16(int acc, const int4& a, const int4& b) {
    acc = __dp4a(a.x, b.x, acc);
    acc = __dp4a(a.y, b.y, acc);
    acc = __dp4a(a.z, b.z, acc);
    acc = __dp4a(a.w, b.w, acc);
    return acc;
}

// ---------------------------------------------------------------------------
// GEMV-class kernel: N <= 8
// ---------------------------------------------------------------------------
template <int ROWS, int NC, int U = 2>
__global__ void __launch_bounds__(256)
k_gemv(const int8_t* __restrict__ W, int64_t M, int64_t K, int64_t ldw,
       const int8_t* __restrict__ X, int64_t ldx, EpiArgs e, int w_static, const int32_t* n_dev) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t row0 = ((int64_t)blockIdx.x * 8 + warp) * ROWS;
    const int64_t nch = K >> 4;   // 16-byte chunks per row (U chunk-iterations' loads issued together)
    int4 w[U][ROWS];
    auto load_w = [&](int64_t c0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + 32 * u;
#pragma unroll
            for (int r = 0; r < ROWS; ++r) {
                if (c < nch && row0 + r < M)
                    w[u][r] = ld_stream16(W + (row0 + r) * ldw + (c << 4));
                else
                    w[u][r] = make_int4(0, 0, 0, 0);
            }
        }
    };
    // PDL: model weights (w_static) do not depend on the predecessor kernel, so the
    // first weight chunks stream from HBM while the predecessor drains; X and the
    // epilogue operands are touched only after griddepcontrol.wait.  The early trigger
    // lets a following GEMV start its own weight stream in turn (its wait still
    // orders it after this grid's completion).
    pdl_trigger();
    if (w_static) {
        load_w(lane);
        pdl_wait();
    } else {
        pdl_wait();
        load_w(lane);
    }
    if (row0 >= M) return;
    // graph-captured decode step: NC is the host-side maximum, the live column count is on the device
    const int nlive = n_dev ? min(NC, *n_dev) : NC;
    int acc[ROWS][NC];
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[r][j] = 0;

    for (int64_t c0 = lane; c0 < nch; c0 += 32 * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + 32 * u;
            if (c < nch) {
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    int4 xv = __ldg(reinterpret_cast<const int4*>(X + j * ldx + (c << 4)));
#pragma unroll
                    for (int r = 0; r < ROWS; ++r) acc[r][j] = dp4a16(acc[r][j], w[u][r], xv);
                }
            }
        }
        if (c0 + 32 * U < nch) load_w(c0 + 32 * U);
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[r][j] = warp_sum(acc[r][j]);
#pragma unroll
    for (int t = 0; t < ROWS * NC; ++t) {
        if ((t & 31) == lane) {
            int r = t / NC, j = t % NC;
            if (row0 + r < M && j < nlive) epilogue(e, row0 + r, j, (long long)acc[r][j]);
        }
    }
}

// ---------------------------------------------------------------------------
// LinearOp.apply for the batch-1 latency path (layers.py:124-146: quantize_activations,
// qgemm_panel, + bias) as ONE kernel for N <= 8 columns: every CTA reduces max|x| over
// the [N][K] f32 input itself (N*K*4 bytes, L2-resident: 4 KB at batch 1), derives the
// per-call scale (qmath.py:172-182: s = fl32(127 / max), 1 when max = 0), encodes its own
// copy of the codes into shared memory (qmath.py:119-133), and streams its weight rows
// exactly as k_gemv (rows prefetched before the PDL wait).  CTA 0 also writes the codes
// and the scale.  One launch instead of three (max scan, encode, GEMV).
// ---------------------------------------------------------------------------
template <int ROWS, int NC, int U>
__global__ void __launch_bounds__(256)
k_linear_gemv(const int8_t* __restrict__ W, int64_t M, int64_t K, int64_t ldw, const float* __restrict__ Xf,
              int64_t ldxf, int N, EpiArgs e, int w_static, int8_t* __restrict__ codes_out, int64_t ldc,
              float* __restrict__ scale_out, int32_t* err_flag) {
    extern __shared__ __align__(16) int8_t xq[];   // [NC][K] codes
    __shared__ uint32_t s_red[8];
    __shared__ float s_scale;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t row0 = ((int64_t)blockIdx.x * 8 + warp) * ROWS;
    const int64_t nch = K >> 4;
    int4 w[U][ROWS];
    auto load_w = [&](int64_t c0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + 32 * u;
#pragma unroll
            for (int r = 0; r < ROWS; ++r)
                w[u][r] = (c < nch && row0 + r < M) ? ld_stream16(W + (row0 + r) * ldw + (c << 4))
                                                    : make_int4(0, 0, 0, 0);
        }
    };
    pdl_trigger();
    if (w_static) {
        load_w(lane);
        pdl_wait();
    } else {
        pdl_wait();
        load_w(lane);
    }
    // max |x| over the N x K input (float4 rows: K % 16 == 0, ldxf % 4 == 0)
    const int64_t K4 = K >> 2;
    uint32_t mb = 0;
    for (int64_t i = threadIdx.x; i < (int64_t)N * K4; i += 256) {
        const int64_t n = i / K4, k4 = i - n * K4;
        const float4 v = reinterpret_cast<const float4*>(Xf + n * ldxf)[k4];
        mb = max(mb, max(max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu),
                         max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu)));
    }
    mb = __reduce_max_sync(0xffffffffu, mb);
    if (lane == 0) s_red[warp] = mb;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        for (int i = 0; i < 8; ++i) m = max(m, s_red[i]);
        if (m >= 0x7f800000u) {   // non-finite activation (qmath.py:180)
            if (blockIdx.x == 0) set_flag(err_flag, QNMT_FLAG_NUMERIC);
            m = 0;
        }
        s_scale = scale_from_maxbits(m);
        if (blockIdx.x == 0 && scale_out) *scale_out = s_scale;
    }
    __syncthreads();
    const float sx = s_scale;
    for (int64_t i = threadIdx.x; i < (int64_t)N * K4; i += 256) {
        const int64_t n = i / K4, k4 = i - n * K4;
        const float4 v = reinterpret_cast<const float4*>(Xf + n * ldxf)[k4];
        const char4 c = make_char4((signed char)quant_code(v.x, sx), (signed char)quant_code(v.y, sx),
                                   (signed char)quant_code(v.z, sx), (signed char)quant_code(v.w, sx));
        reinterpret_cast<char4*>(xq + n * K)[k4] = c;
        if (blockIdx.x == 0 && codes_out) reinterpret_cast<char4*>(codes_out + n * ldc)[k4] = c;
    }
    __syncthreads();
    if (row0 >= M) return;
    int acc[ROWS][NC];
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[r][j] = 0;
    for (int64_t c0 = lane; c0 < nch; c0 += 32 * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + 32 * u;
            if (c < nch) {
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    const int4 xv = *reinterpret_cast<const int4*>(xq + j * K + (c << 4));
#pragma unroll
                    for (int r = 0; r < ROWS; ++r) acc[r][j] = dp4a16(acc[r][j], w[u][r], xv);
                }
            }
        }
        if (c0 + 32 * U < nch) load_w(c0 + 32 * U);
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[r][j] = warp_sum(acc[r][j]);
    e.x_scales = &s_scale;   // the epilogue's activation scale: this CTA's (identical in every CTA)
    e.col_seg = nullptr;
#pragma unroll
    for (int t = 0; t < ROWS * NC; ++t) {
        if ((t & 31) == lane) {
            const int r = t / NC, j = t % NC;
            if (row0 + r < M && j < N) epilogue(e, row0 + r, j, (long long)acc[r][j]);
        }
    }
}

template <int ROWS, int NC>
static int launch_linear(const int8_t* W, int64_t M, int64_t K, int64_t ldw, const float* Xf, int64_t ldxf, int N,
                         const EpiArgs& e, int8_t* codes, int64_t ldc, float* scale, int32_t* err, cudaStream_t st) {
    const unsigned grid = (unsigned)cdiv(M, 8 * ROWS);
    const int w_static = (e.flags & QNMT_GEMM_W_STATIC) ? 1 : 0;
    const size_t smem = (size_t)NC * K;
    if (K >= 2048 && NC <= 2) {
        static size_t done = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_linear_gemv<ROWS, NC, 4>, smem, done));
        QNMT_LAUNCH((k_linear_gemv<ROWS, NC, 4>), grid, 256, smem, st, W, M, K, ldw, Xf, ldxf, N, e, w_static,
                    codes, ldc, scale, err);
    } else {
        static size_t done = 0;
        QNMT_CUDA(raise_smem_limit((const void*)k_linear_gemv<ROWS, NC, 2>, smem, done));
        QNMT_LAUNCH((k_linear_gemv<ROWS, NC, 2>), grid, 256, smem, st, W, M, K, ldw, Xf, ldxf, N, e, w_static,
                    codes, ldc, scale, err);
    }
    QNMT_CHECK_LAUNCH("k_linear_gemv");
    return QNMT_OK;
}

template <int ROWS>
static int dispatch_linear(const int8_t* W, int64_t M, int64_t K, int64_t ldw, const float* Xf, int64_t ldxf, int N,
                           const EpiArgs& e, int8_t* codes, int64_t ldc, float* scale, int32_t* err, cudaStream_t st) {
#define QNMT_LIN(NC_) \
    case NC_: return launch_linear<ROWS, NC_>(W, M, K, ldw, Xf, ldxf, N, e, codes, ldc, scale, err, st);
    switch (N) {
        QNMT_LIN(1) QNMT_LIN(2) QNMT_LIN(3) QNMT_LIN(4) QNMT_LIN(5) QNMT_LIN(6) QNMT_LIN(7) QNMT_LIN(8)
        default: break;
    }
#undef QNMT_LIN
    set_error("linear: N=%d > 8", N);
    return QNMT_ERR_CONFIG;
}

// ---------------------------------------------------------------------------
// Tiled dp4a GEMM: 64(M) x 64(N) x 64(K) tiles, 256 threads, 4x4 per thread
// ---------------------------------------------------------------------------
constexpr int TBM = 64, TBN = 64, TBK = 64;
constexpr int TSTR = 17;   // smem row stride in 32-bit words (conflict-free reads)

__global__ void __launch_bounds__(256)
k_gemm_tile(const int8_t* __restrict__ W, int64_t M, int64_t K, int64_t ldw,
            const int8_t* __restrict__ X, int64_t N, int64_t ldx, EpiArgs e) {
    __shared__ int sA[TBM * TSTR];
    __shared__ int sB[TBN * TSTR];
    const int tid = threadIdx.x;
    const int tx = tid & 15;   // M direction
    const int ty = tid >> 4;   // N direction
    const int64_t m0 = (int64_t)blockIdx.x * TBM;
    const int64_t n0 = (int64_t)blockIdx.y * TBN;
    int acc[4][4] = {};
    // loader mapping: 256 threads x 16 bytes = 64 rows x 64 bytes
    const int lrow = tid >> 2, lcol = (tid & 3) * 4;   // lcol in words
    for (int64_t k0 = 0; k0 < K; k0 += TBK) {
        int4 a = make_int4(0, 0, 0, 0), b = make_int4(0, 0, 0, 0);
        if (m0 + lrow < M) a = ld_stream16(W + (m0 + lrow) * ldw + k0 + lcol * 4);
        if (n0 + lrow < N) b = __ldg(reinterpret_cast<const int4*>(X + (n0 + lrow) * ldx + k0 + lcol * 4));
        __syncthreads();
        int* pa = sA + lrow * TSTR + lcol;
        pa[0] = a.x; pa[1] = a.y; pa[2] = a.z; pa[3] = a.w;
        int* pb = sB + lrow * TSTR + lcol;
        pb[0] = b.x; pb[1] = b.y; pb[2] = b.z; pb[3] = b.w;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < TBK / 4; ++w) {
            int av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = sA[(tx + 16 * i) * TSTR + w];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = sB[(ty + 16 * j) * TSTR + w];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __dp4a(av[i], bv[j], acc[i][j]);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int64_t n = n0 + ty + 16 * j;
        if (n >= N) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int64_t m = m0 + tx + 16 * i;
            if (m < M) epilogue(e, m, n, (long long)acc[i][j]);
        }
    }
}

// ---------------------------------------------------------------------------
// Generic: one block per output element, int64 partial sums.
// ---------------------------------------------------------------------------
__global__ void k_gemm_generic(const int8_t* __restrict__ W, int64_t M, int64_t K, int64_t ldw,
                               const int8_t* __restrict__ X, int64_t N, int64_t ldx, EpiArgs e) {
    int64_t idx = blockIdx.x;
    int64_t m = idx % M, n = idx / M;
    const int8_t* a = W + m * ldw;
    const int8_t* b = X + n * ldx;
    long long s = 0;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) s += (int)a[k] * (int)b[k];
    s = warp_sum(s);
    __shared__ long long part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        epilogue(e, m, n, t);
    }
}

template <int ROWS, int NC>
static int launch_gemv(const int8_t* W, int64_t M, int64_t K, int64_t ldw, const int8_t* X,
                       int64_t ldx, const EpiArgs& e, cudaStream_t st) {
    unsigned grid = (unsigned)cdiv(M, 8 * ROWS);
    const int w_static = (e.flags & QNMT_GEMM_W_STATIC) ? 1 : 0;
    if (K >= 2048 && NC <= 2)   // long rows: four 16-byte chunks per lane and row in flight
        QNMT_LAUNCH((k_gemv<ROWS, NC, 4>), grid, 256, 0, st, W, M, K, ldw, X, ldx, e, w_static, tl_ndev);
    else
        QNMT_LAUNCH((k_gemv<ROWS, NC, 2>), grid, 256, 0, st, W, M, K, ldw, X, ldx, e, w_static, tl_ndev);
    return QNMT_OK;
}

template <int ROWS>
static int dispatch_gemv(int64_t N, const int8_t* W, int64_t M, int64_t K, int64_t ldw,
                         const int8_t* X, int64_t ldx, const EpiArgs& e, cudaStream_t st) {
    switch (N) {
        case 1: return launch_gemv<ROWS, 1>(W, M, K, ldw, X, ldx, e, st);
        case 2: return launch_gemv<ROWS, 2>(W, M, K, ldw, X, ldx, e, st);
        case 3: return launch_gemv<ROWS, 3>(W, M, K, ldw, X, ldx, e, st);
        case 4: return launch_gemv<ROWS, 4>(W, M, K, ldw, X, ldx, e, st);
        case 5: return launch_gemv<ROWS, 5>(W, M, K, ldw, X, ldx, e, st);
        case 6: return launch_gemv<ROWS, 6>(W, M, K, ldw, X, ldx, e, st);
        case 7: return launch_gemv<ROWS, 7>(W, M, K, ldw, X, ldx, e, st);
        default: return launch_gemv<ROWS, 8>(W, M, K, ldw, X, ldx, e, st);
    }
}

int g_gemm_impl = 0;

int gemm_i8_launch(const GemmArgs& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return QNMT_OK;
    EpiArgs e{g.w_scales, g.w_rows_per_scale, g.x_scales, g.col_seg, g.bias, g.Y, g.ldy,
              g.acc_out, g.M, g.flags, g.add1, g.ld1, g.add2, g.ld2};
    bool aligned = (g.K % 16 == 0) && (g.ldw % 16 == 0) && (g.ldx % 16 == 0) &&
                   ((uintptr_t)g.W % 16 == 0) && ((uintptr_t)g.X % 16 == 0);
    // batch-sized panels (latency path, N <= 8 incl. graph-captured steps with a device-side N):
    // the HBM-streaming GEMV, weights prefetched before the PDL wait
    // (in graph mode only for N <= 2: at beam-size N the tcgen05 tile is faster, measured cfg3 beam 5)
    const bool gemv_ok = g_gemm_impl != 2 && g.N <= (tl_ndev ? 2 : 8) && aligned && g.K <= QNMT_INT32_SAFE_K &&
                         g.K > 0;
    if (g.gru.mode) {   // GRU elementwise phase in the epilogue: tcgen05 kernels only
        if (!tc_eligible(g)) { set_error("gemm: the GRU epilogue needs the tcgen05 path"); return QNMT_ERR_CONFIG; }
        return gemm_tc_launch(g, st);
    }
    if (g.add1 && !gemv_ok) {
        if (!tc_eligible(g)) { set_error("gemm: epilogue addends need the tcgen05 path"); return QNMT_ERR_CONFIG; }
        return gemm_tc_launch(g, st);
    }
    if (tl_ndev && !gemv_ok) {   // graph-captured step: device-side N (tcgen05 or GEMV kernels)
        if (!tc_eligible(g)) { set_error("graph mode needs tcgen05-eligible GEMM shapes"); return QNMT_ERR_CONFIG; }
        return gemm_tc_launch(g, st);
    }
    if (g_gemm_impl != 1 && tc_eligible(g) && (g.N > 8 || g_gemm_impl == 2)) return gemm_tc_launch(g, st);
    if (g.K > QNMT_INT32_SAFE_K || !aligned || g.K == 0) {
        k_gemm_generic<<<(unsigned)(g.M * g.N), 128, 0, st>>>(g.W, g.M, g.K, g.ldw, g.X, g.N, g.ldx, e);
        QNMT_CHECK_LAUNCH("k_gemm_generic");
        return QNMT_OK;
    }
    if (g.N <= 8) {
        int rc = g.K <= 512 ? dispatch_gemv<4>(g.N, g.W, g.M, g.K, g.ldw, g.X, g.ldx, e, st)
                            : dispatch_gemv<2>(g.N, g.W, g.M, g.K, g.ldw, g.X, g.ldx, e, st);
        if (rc != QNMT_OK) return rc;
        QNMT_CHECK_LAUNCH("k_gemv");
        return QNMT_OK;
    }
    if (g.K % TBK == 0) {
        dim3 grid((unsigned)cdiv(g.M, TBM), (unsigned)cdiv(g.N, TBN));
        k_gemm_tile<<<grid, 256, 0, st>>>(g.W, g.M, g.K, g.ldw, g.X, g.N, g.ldx, e);
        QNMT_CHECK_LAUNCH("k_gemm_tile");
        return QNMT_OK;
    }
    // K multiple of 16 but not of 64: process N in panels of 8 with the GEMV kernel
    for (int64_t n0 = 0; n0 < g.N; n0 += 8) {
        EpiArgs e2 = e;
        int64_t nn = g.N - n0 < 8 ? g.N - n0 : 8;
        if (e2.Y) e2.Y += n0 * g.ldy;
        if (e2.acc_out) e2.acc_out += n0 * g.M;
        if (e2.col_seg) e2.col_seg += n0;
        const int rc = dispatch_gemv<2>(nn, g.W, g.M, g.K, g.ldw, g.X + n0 * g.ldx, g.ldx, e2, st);
        if (rc != QNMT_OK) return rc;
        QNMT_CHECK_LAUNCH("k_gemv(panel)");
    }
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" int qnmt_set_gemm_impl(int impl) {
    int old = qnmt::g_gemm_impl;
    qnmt::g_gemm_impl = impl;
    return old;
}

extern "C" int qnmt_gemm_i8(const int8_t* W, int64_t M, int64_t K, int64_t ldw,
                            const float* w_scales, int64_t w_rows_per_scale, const int8_t* X,
                            int64_t N, int64_t ldx, const float* x_scales, const int32_t* col_seg,
                            const float* bias, float* Y, int64_t ldy, int64_t* acc_out,
                            int32_t flags, void* stream) {
    if (M < 0 || N < 0 || K < 0 || ldw < K || ldx < K || (Y && ldy < M) || w_rows_per_scale < 1) {
        qnmt::set_error("qnmt_gemm_i8: bad shape M=%lld N=%lld K=%lld", (long long)M,
                        (long long)N, (long long)K);
        return QNMT_ERR_SHAPE;
    }
    qnmt::GemmArgs g{W, M, K, ldw, w_scales, w_rows_per_scale, X, N, ldx, x_scales, col_seg,
                     bias, Y, ldy, acc_out, flags};
    return qnmt::gemm_i8_launch(g, qnmt::as_stream(stream));
}

extern "C" int qnmt_linear_i8(const int8_t* W, int64_t M, int64_t K, int64_t ldw, const float* w_scales,
                              int64_t w_rows_per_scale, const float* X, int64_t N, int64_t ldx, const float* bias,
                              float* Y, int64_t ldy, int8_t* codes_out, int64_t ldc, float* scale_out,
                              uint32_t* maxbits, int32_t flags, int32_t* err_flag, void* stream) {
    if (M < 0 || N < 0 || K < 1 || ldw < K || ldx < K || ldc < K || (Y && ldy < M) || w_rows_per_scale < 1) {
        qnmt::set_error("qnmt_linear_i8: bad shape M=%lld N=%lld K=%lld", (long long)M, (long long)N, (long long)K);
        return QNMT_ERR_SHAPE;
    }
    if (M == 0 || N == 0) return QNMT_OK;
    const cudaStream_t st = qnmt::as_stream(stream);
    const bool fused = N <= 8 && K % 16 == 0 && ldw % 16 == 0 && ldx % 4 == 0 && ldc % 4 == 0 &&
                       (uintptr_t)W % 16 == 0 && (uintptr_t)X % 16 == 0 && (uintptr_t)codes_out % 4 == 0 &&
                       N * K <= 96 * 1024 && K <= QNMT_INT32_SAFE_K && codes_out != nullptr && scale_out != nullptr;
    if (fused) {
        qnmt::EpiArgs e{w_scales, w_rows_per_scale, nullptr, nullptr, bias, Y, ldy, nullptr, M, flags,
                        nullptr, 0, nullptr, 0};
        return K <= 512 ? qnmt::dispatch_linear<4>(W, M, K, ldw, X, ldx, (int)N, e, codes_out, ldc, scale_out,
                                                  err_flag, st)
                        : qnmt::dispatch_linear<2>(W, M, K, ldw, X, ldx, (int)N, e, codes_out, ldc, scale_out,
                                                  err_flag, st);
    }
    // general shapes: the activation quantize kernels, then the product
    if (!codes_out || !scale_out || !maxbits) {
        qnmt::set_error("qnmt_linear_i8: codes_out, scale_out and maxbits are required");
        return QNMT_ERR_CONFIG;
    }
    int rc = qnmt_quantize(X, N, K, ldx, nullptr, 1, codes_out, ldc, scale_out, maxbits, 1, err_flag, stream);
    if (rc != QNMT_OK) return rc;
    qnmt::GemmArgs g{W, M, K, ldw, w_scales, w_rows_per_scale, codes_out, N, ldc, scale_out, nullptr,
                     bias, Y, ldy, nullptr, flags};
    return qnmt::gemm_i8_launch(g, st);
}
