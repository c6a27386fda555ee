// elementwise.cu -- GRU gate arithmetic, tanh, embedding gather.
//
// GRU (layers.py:170-181):
//   z  = sigmoid((Wz x + bz) + Uz h)            -- f32 add, fp64 sigmoid, round
//   r  = sigmoid((Wr x + br) + Ur h)
//   rh = r * h                                  -- f32 mul (feeds the 2nd phase)
//   h~ = tanh((Wc x + bc) + Uc (r*h))
//   h' = (1 - z) * h + z * h~                   -- four separate f32 ops
// Every f32 op is an explicit __f*_rn intrinsic, so no FMA contraction can
// change the association the reference's numpy expression fixes.
//
// Fused quantization statistics: when `segmax` is given, each kernel also
// atomically maxes |output| (as u32 bits) into segmax[col_seg[n]] -- the
// per-segment max-abs that the next quantization (qmath.py:157-169) needs --
// so the consumer only runs the encode pass.
#include "kernels.cuh"

namespace qnmt {

__device__ __forceinline__ void warp_seg_max(uint32_t m, uint32_t* segmax, int seg) {
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(segmax + seg, m);
}

__global__ void k_gru_gates(const float* __restrict__ gx, int64_t ldgx, const int32_t* __restrict__ gx_row,
                            const float* __restrict__ gh, int64_t ldgh, const float* __restrict__ h,
                            int64_t ldh, int64_t N, int64_t H, float* __restrict__ z,
                            float* __restrict__ rh, int32_t* err_flag, const int32_t* n_dev,
                            uint32_t* segmax, const int32_t* __restrict__ col_seg) {
    pdl_entry();
    int64_t n = blockIdx.y;
    if (beyond(n_dev, n)) return;
    int64_t rowx = gx_row ? gx_row[n] : n;
    const float* gxr = gx + rowx * ldgx;
    const float* ghr = gh + n * ldgh;
    bool bad = false;
    uint32_t m = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < H; j += (int64_t)gridDim.x * blockDim.x) {
        float pz = __fadd_rn(gxr[j], ghr[j]);
        float pr = __fadd_rn(gxr[H + j], ghr[H + j]);
        bad |= !is_finite_f(pz) || !is_finite_f(pr);
        float zz = sigmoid_b(pz);
        float rr = sigmoid_b(pr);
        z[n * H + j] = zz;
        const float v = __fmul_rn(rr, h[n * ldh + j]);
        rh[n * H + j] = v;
        m = max(m, __float_as_uint(v) & 0x7fffffffu);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    if (segmax) warp_seg_max(m, segmax, col_seg ? col_seg[n] : (int)n);
}

__global__ void k_gru_combine(const float* __restrict__ gx, int64_t ldgx, const int32_t* __restrict__ gx_row,
                              const float* __restrict__ ghc, int64_t ldghc, const float* __restrict__ z,
                              const float* __restrict__ h, int64_t ldh, int64_t N, int64_t H,
                              float* __restrict__ h_out, int64_t ldo, float* __restrict__ out2,
                              int64_t ld2, const int32_t* __restrict__ out2_row, int32_t* err_flag,
                              const int32_t* n_dev, uint32_t* segmax, const int32_t* __restrict__ col_seg) {
    pdl_entry();
    int64_t n = blockIdx.y;
    if (beyond(n_dev, n)) return;
    int64_t rowx = gx_row ? gx_row[n] : n;
    const float* gxr = gx + rowx * ldgx + 2 * H;
    bool bad = false;
    uint32_t m = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < H; j += (int64_t)gridDim.x * blockDim.x) {
        float pc = __fadd_rn(gxr[j], ghc[n * ldghc + j]);
        bad |= !is_finite_f(pc);
        float c = tanh_b(pc);
        float zz = z[n * H + j];
        float hh = h[n * ldh + j];
        float v = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zz), hh), __fmul_rn(zz, c));
        h_out[n * ldo + j] = v;
        if (out2) out2[(int64_t)out2_row[n] * ld2 + j] = v;
        m = max(m, __float_as_uint(v) & 0x7fffffffu);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    if (segmax) warp_seg_max(m, segmax, col_seg ? col_seg[n] : (int)n);
}

__global__ void k_tanh(const float* __restrict__ x, int64_t N, int64_t D, int64_t ldx,
                       float* __restrict__ y, int64_t ldy, int32_t* err_flag, const int32_t* n_dev,
                       uint32_t* segmax, const int32_t* __restrict__ col_seg) {
    pdl_entry();
    int64_t n = blockIdx.y;
    if (beyond(n_dev, n)) return;
    bool bad = false;
    uint32_t m = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < D; j += (int64_t)gridDim.x * blockDim.x) {
        float v = x[n * ldx + j];
        bad |= !is_finite_f(v);
        const float t = tanh_b(v);
        y[n * ldy + j] = t;
        m = max(m, __float_as_uint(t) & 0x7fffffffu);
    }
    if (bad) set_flag(err_flag, QNMT_FLAG_NUMERIC);
    if (segmax) warp_seg_max(m, segmax, col_seg ? col_seg[n] : (int)n);
}

__global__ void k_embed_gather(const float* __restrict__ table, int64_t rows, int64_t E,
                               const int32_t* __restrict__ ids, float* __restrict__ out,
                               int64_t ldo, int32_t* err_flag, const int32_t* n_dev,
                               uint32_t* segmax, const int32_t* __restrict__ col_seg) {
    pdl_entry();
    int64_t n = blockIdx.x;
    if (beyond(n_dev, n)) return;
    int32_t id = ids[n];
    bool ok = id >= 0 && id < rows;
    if (!ok && threadIdx.x == 0) set_flag(err_flag, QNMT_FLAG_VOCAB);
    uint32_t m = 0;
    for (int64_t j = threadIdx.x; j < E; j += blockDim.x) {
        const float v = ok ? table[(int64_t)id * E + j] : 0.0f;
        out[n * ldo + j] = v;
        m = max(m, __float_as_uint(v) & 0x7fffffffu);
    }
    if (segmax) warp_seg_max(m, segmax, col_seg ? col_seg[n] : (int)n);
}

static inline dim3 rows_grid(int64_t N, int64_t D, int threads) {
    int64_t bx = cdiv(D, threads);
    if (bx > 64) bx = 64;
    return dim3((unsigned)bx, (unsigned)N);
}

int gru_gates_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* gh,
                     int64_t ldgh, const float* h, int64_t ldh, int64_t N, int64_t H, float* z,
                     float* rh, int32_t* err_flag, cudaStream_t st, uint32_t* segmax,
                     const int32_t* col_seg) {
    if (N <= 0) return QNMT_OK;
    QNMT_LAUNCH(k_gru_gates, rows_grid(N, H, 256), 256, 0, st, gx, ldgx, gx_row, gh, ldgh, h, ldh, N, H, z, rh, err_flag,
                                                     tl_ndev, segmax, col_seg);
    QNMT_CHECK_LAUNCH("k_gru_gates");
    return QNMT_OK;
}

int gru_combine_launch(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* ghc,
                       int64_t ldghc, const float* z, const float* h, int64_t ldh, int64_t N,
                       int64_t H, float* h_out, int64_t ldo, float* out2, int64_t ld2,
                       const int32_t* out2_row, int32_t* err_flag, cudaStream_t st,
                       uint32_t* segmax, const int32_t* col_seg) {
    if (N <= 0) return QNMT_OK;
    QNMT_LAUNCH(k_gru_combine, rows_grid(N, H, 256), 256, 0, st, gx, ldgx, gx_row, ghc, ldghc, z, h, ldh, N, H,
                                                        h_out, ldo, out2, ld2, out2_row, err_flag, tl_ndev,
                                                        segmax, col_seg);
    QNMT_CHECK_LAUNCH("k_gru_combine");
    return QNMT_OK;
}

int tanh_launch(const float* x, int64_t N, int64_t D, int64_t ldx, float* y, int64_t ldy,
                int32_t* err_flag, cudaStream_t st, uint32_t* segmax,
                const int32_t* col_seg) {
    if (N <= 0) return QNMT_OK;
    QNMT_LAUNCH(k_tanh, rows_grid(N, D, 256), 256, 0, st, x, N, D, ldx, y, ldy, err_flag, tl_ndev, segmax, col_seg);
    QNMT_CHECK_LAUNCH("k_tanh");
    return QNMT_OK;
}

int embed_gather_launch(const float* table, int64_t rows, int64_t E, const int32_t* ids, int64_t n,
                        float* out, int64_t ldo, int32_t* err_flag, cudaStream_t st,
                        uint32_t* segmax, const int32_t* col_seg) {
    if (n <= 0) return QNMT_OK;
    QNMT_LAUNCH(k_embed_gather, (unsigned)n, 128, 0, st, table, rows, E, ids, out, ldo, err_flag, tl_ndev, segmax,
                                                col_seg);
    QNMT_CHECK_LAUNCH("k_embed_gather");
    return QNMT_OK;
}

}  // namespace qnmt

extern "C" {

int qnmt_gru_gates(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* gh,
                   int64_t ldgh, const float* h, int64_t ldh, int64_t N, int64_t H, float* z,
                   float* rh, int32_t* err_flag, void* stream) {
    return qnmt::gru_gates_launch(gx, ldgx, gx_row, gh, ldgh, h, ldh, N, H, z, rh, err_flag,
                                  qnmt::as_stream(stream));
}

int qnmt_gru_combine(const float* gx, int64_t ldgx, const int32_t* gx_row, const float* ghc,
                     int64_t ldghc, const float* z, const float* h, int64_t ldh, int64_t N,
                     int64_t H, float* h_out, int64_t ldo, float* out2, int64_t ld2,
                     const int32_t* out2_row, int32_t* err_flag, void* stream) {
    return qnmt::gru_combine_launch(gx, ldgx, gx_row, ghc, ldghc, z, h, ldh, N, H, h_out, ldo, out2,
                                    ld2, out2_row, err_flag, qnmt::as_stream(stream));
}

int qnmt_tanh(const float* x, int64_t N, int64_t D, int64_t ldx, float* y, int64_t ldy,
              int32_t* err_flag, void* stream) {
    return qnmt::tanh_launch(x, N, D, ldx, y, ldy, err_flag, qnmt::as_stream(stream));
}

int qnmt_embed_gather(const float* table, int64_t rows, int64_t E, const int32_t* ids, int64_t n,
                      float* out, int64_t ldo, int32_t* err_flag, void* stream) {
    return qnmt::embed_gather_launch(table, rows, E, ids, n, out, ldo, err_flag,
                                     qnmt::as_stream(stream));
}

}  // extern "C"
