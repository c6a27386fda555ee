// quantize.cu -- K1: segmented max-abs -> scale -> int8 codes.
//
// Replaces qmath.py:157-169 (_max_abs_scan), :136-142 (_encode), :119-133
// (_encode_i8), :145-154 (quantize) and :172-182 (quantize_activations).
//
// Pass 1 (k_seg_maxabs): warp-shuffle max of |x| per (column chunk), one
//   atomicMax on the u32 bit pattern per warp into the segment's slot.  For
//   non-negative floats the u32 order equals the float order, and any NaN/Inf
//   has bits >= 0x7f800000, so the same max doubles as the finiteness probe.
// Pass 2 (k_encode): scale = fl32(127/max) per segment, 128-bit loads of x,
//   32-bit packed stores of 4 codes.
#include "kernels.cuh"

namespace qnmt {

constexpr int QT = 256;   // threads per block

__global__ void k_seg_maxabs(const float* __restrict__ x, int64_t ncols, int64_t K, int64_t ldx,
                             int chunks_per_col, int64_t chunk_elems,
                             const int32_t* __restrict__ col_seg, uint32_t* seg_maxbits,
                             bool vec4, const int32_t* n_dev) {
    pdl_entry();
    int64_t b = blockIdx.x;
    int64_t col = b / chunks_per_col;
    int64_t chunk = b % chunks_per_col;
    if (col >= ncols || beyond(n_dev, col)) return;
    const float* row = x + col * ldx;
    int64_t k0 = chunk * chunk_elems;
    int64_t k1 = min(K, k0 + chunk_elems);
    uint32_t m = 0;
    if (vec4) {
        for (int64_t k = k0 + 4 * threadIdx.x; k < k1; k += 4 * QT) {
            float4 v = *reinterpret_cast<const float4*>(row + k);
            m = max(m, __float_as_uint(v.x) & 0x7fffffffu);
            m = max(m, __float_as_uint(v.y) & 0x7fffffffu);
            m = max(m, __float_as_uint(v.z) & 0x7fffffffu);
            m = max(m, __float_as_uint(v.w) & 0x7fffffffu);
        }
    } else {
        for (int64_t k = k0 + threadIdx.x; k < k1; k += QT)
            m = max(m, __float_as_uint(row[k]) & 0x7fffffffu);
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0 && m) {
        int seg = col_seg ? col_seg[col] : 0;
        atomicMax(seg_maxbits + seg, m);
    }
}

__global__ void k_encode(const float* __restrict__ x, int64_t ncols, int64_t K, int64_t ldx,
                         int chunks_per_col, int64_t chunk_elems,
                         const int32_t* __restrict__ col_seg, const uint32_t* __restrict__ seg_maxbits,
                         int8_t* __restrict__ q, int64_t ldq, float* __restrict__ scales,
                         int32_t mode, int32_t* err_flag, bool vec4, const int32_t* n_dev) {
    pdl_entry();
    int64_t b = blockIdx.x;
    int64_t col = b / chunks_per_col;
    int64_t chunk = b % chunks_per_col;
    if (col >= ncols || beyond(n_dev, col)) return;
    int seg = col_seg ? col_seg[col] : 0;
    uint32_t bits = seg_maxbits[seg];
    if (bits >= 0x7f800000u) {   // non-finite somewhere in the segment
        if (threadIdx.x == 0) set_flag(err_flag, mode == 0 ? QNMT_FLAG_INVALID : QNMT_FLAG_NUMERIC);
        bits = 0;                // codes of a failed call are zeros
    }
    float s = scale_from_maxbits(bits);
    if (chunk == 0 && threadIdx.x == 0 && scales) scales[seg] = s;
    const float* row = x + col * ldx;
    int8_t* qrow = q + col * ldq;
    int64_t k0 = chunk * chunk_elems;
    int64_t k1 = min(K, k0 + chunk_elems);
    if (vec4) {
        for (int64_t k = k0 + 4 * threadIdx.x; k < k1; k += 4 * QT) {
            float4 v = *reinterpret_cast<const float4*>(row + k);
            uint32_t packed = (uint32_t)(quant_code(v.x, s) & 0xff) |
                              ((uint32_t)(quant_code(v.y, s) & 0xff) << 8) |
                              ((uint32_t)(quant_code(v.z, s) & 0xff) << 16) |
                              ((uint32_t)(quant_code(v.w, s) & 0xff) << 24);
            *reinterpret_cast<uint32_t*>(qrow + k) = packed;
        }
    } else {
        for (int64_t k = k0 + threadIdx.x; k < k1; k += QT) qrow[k] = (int8_t)quant_code(row[k], s);
    }
}

int quantize_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                    int32_t nseg, int8_t* q, int64_t ldq, float* scales, uint32_t* seg_maxbits,
                    int32_t mode, int32_t* err_flag, cudaStream_t st) {
    if (ncols <= 0 || K <= 0) return QNMT_OK;
    QNMT_CUDA(cudaMemsetAsync(seg_maxbits, 0, sizeof(uint32_t) * (size_t)nseg, st));
    bool vec4 = (K % 4 == 0) && (ldx % 4 == 0) && (ldq % 4 == 0) &&
                ((uintptr_t)x % 16 == 0) && ((uintptr_t)q % 4 == 0);
    int64_t chunk_elems = 4096;
    int chunks = (int)cdiv(K, chunk_elems);
    int64_t blocks = ncols * chunks;
    QNMT_LAUNCH(k_seg_maxabs, (unsigned)blocks, QT, 0, st, x, ncols, K, ldx, chunks, chunk_elems, col_seg,
                                                 seg_maxbits, vec4, tl_ndev);
    QNMT_CHECK_LAUNCH("k_seg_maxabs");
    QNMT_LAUNCH(k_encode, (unsigned)blocks, QT, 0, st, x, ncols, K, ldx, chunks, chunk_elems, col_seg,
                                             seg_maxbits, q, ldq, scales, mode, err_flag, vec4, tl_ndev);
    QNMT_CHECK_LAUNCH("k_encode");
    return QNMT_OK;
}

int quantize_encode_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                           int8_t* q, int64_t ldq, float* scales, const uint32_t* seg_maxbits, int32_t mode,
                           int32_t* err_flag, cudaStream_t st) {
    if (ncols <= 0 || K <= 0) return QNMT_OK;
    bool vec4 = (K % 4 == 0) && (ldx % 4 == 0) && (ldq % 4 == 0) &&
                ((uintptr_t)x % 16 == 0) && ((uintptr_t)q % 4 == 0);
    int64_t chunk_elems = 4096;
    int chunks = (int)cdiv(K, chunk_elems);
    QNMT_LAUNCH(k_encode, (unsigned)(ncols * chunks), QT, 0, st, x, ncols, K, ldx, chunks, chunk_elems, col_seg,
                                                       seg_maxbits, q, ldq, scales, mode, err_flag, vec4, tl_ndev);
    QNMT_CHECK_LAUNCH("k_encode");
    return QNMT_OK;
}

int quantize_max_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                        uint32_t* seg_maxbits, cudaStream_t st) {
    if (ncols <= 0 || K <= 0) return QNMT_OK;
    bool vec4 = (K % 4 == 0) && (ldx % 4 == 0) && ((uintptr_t)x % 16 == 0);
    int64_t chunk_elems = 4096;
    int chunks = (int)cdiv(K, chunk_elems);
    QNMT_LAUNCH(k_seg_maxabs, (unsigned)(ncols * chunks), QT, 0, st, x, ncols, K, ldx, chunks, chunk_elems, col_seg,
                                                           seg_maxbits, vec4, tl_ndev);
    QNMT_CHECK_LAUNCH("k_seg_maxabs");
    return QNMT_OK;
}

__global__ void k_dequantize(const int8_t* __restrict__ q, int64_t n, float scale, float* y) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = __fdiv_rn((float)q[i], scale);
}

}  // namespace qnmt

extern "C" {

int qnmt_quantize(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                  int32_t nseg, int8_t* q, int64_t ldq, float* scales, uint32_t* seg_maxbits,
                  int32_t mode, int32_t* err_flag, void* stream) {
    if (ncols < 0 || K < 0 || ldx < K || ldq < K || nseg < 1) {
        qnmt::set_error("qnmt_quantize: bad shape ncols=%lld K=%lld ldx=%lld ldq=%lld nseg=%d",
                        (long long)ncols, (long long)K, (long long)ldx, (long long)ldq, nseg);
        return QNMT_ERR_SHAPE;
    }
    return qnmt::quantize_launch(x, ncols, K, ldx, col_seg, nseg, q, ldq, scales, seg_maxbits,
                                 mode, err_flag, qnmt::as_stream(stream));
}

int qnmt_dequantize(const int8_t* q, int64_t n, float scale, float* y, void* stream) {
    if (n <= 0) return QNMT_OK;
    qnmt::k_dequantize<<<(unsigned)qnmt::cdiv(n, 256), 256, 0, qnmt::as_stream(stream)>>>(q, n, scale, y);
    QNMT_CHECK_LAUNCH("k_dequantize");
    return QNMT_OK;
}

}  // extern "C"
