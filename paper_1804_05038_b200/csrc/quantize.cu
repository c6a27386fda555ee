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

// ---------------------------------------------------------------------------
// k_quant_cluster: quantize_activations (qmath.py:157-182) of one small
// contiguous matrix in ONE launch -- the two-pass scheme above costs a memset
// and two dependent launches, more than the 0.25 MB of data.  A cluster of 8
// CTAs: every thread keeps its <= 4 float4 of x in registers, the CTA maxima
// meet through distributed shared memory, then every thread encodes its own
// values.  n = ncols * K <= QC_CAP elements, one segment.
// ---------------------------------------------------------------------------
constexpr int QC_T = 512, QC_CTAS = 8, QC_R = 4;
constexpr int64_t QC_CAP = (int64_t)QC_CTAS * QC_T * QC_R * 4;

__global__ void __cluster_dims__(QC_CTAS, 1, 1) __launch_bounds__(QC_T)
k_quant_cluster(const float* __restrict__ x, int64_t n4, int8_t* __restrict__ q, float* __restrict__ scale_out,
                uint32_t* maxbits_out, int32_t mode, int32_t* err_flag) {
    pdl_entry();
    __shared__ uint32_t red[QC_T / 32];
    __shared__ uint32_t cta_max;
    float4 v[QC_R];
    uint32_t m = 0;
    const int64_t i0 = (int64_t)blockIdx.x * QC_T + threadIdx.x;
#pragma unroll
    for (int r = 0; r < QC_R; ++r) {
        const int64_t i = i0 + (int64_t)r * QC_CTAS * QC_T;
        v[r] = i < n4 ? reinterpret_cast<const float4*>(x)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        m = max(max(m, max(__float_as_uint(v[r].x) & 0x7fffffffu, __float_as_uint(v[r].y) & 0x7fffffffu)),
                max(__float_as_uint(v[r].z) & 0x7fffffffu, __float_as_uint(v[r].w) & 0x7fffffffu));
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t mm = 0;
#pragma unroll
        for (int w = 0; w < QC_T / 32; ++w) mm = max(mm, red[w]);
        cta_max = mm;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t bits = 0;
    {
        const uint32_t local = (uint32_t)__cvta_generic_to_shared(&cta_max);
#pragma unroll
        for (uint32_t c = 0; c < QC_CTAS; ++c) {
            uint32_t ra, val;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local), "r"(c));
            asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(val) : "r"(ra) : "memory");
            bits = max(bits, val);
        }
    }
    // no CTA may exit while a peer still reads its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (blockIdx.x == 0 && threadIdx.x == 0 && maxbits_out) *maxbits_out = bits;
    if (bits >= 0x7f800000u) {   // non-finite input: flag, codes of a failed call are zeros (as k_encode)
        if (threadIdx.x == 0) set_flag(err_flag, mode == 0 ? QNMT_FLAG_INVALID : QNMT_FLAG_NUMERIC);
        bits = 0;
    }
    const float s = scale_from_maxbits(bits);
    if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = s;
#pragma unroll
    for (int r = 0; r < QC_R; ++r) {
        const int64_t i = i0 + (int64_t)r * QC_CTAS * QC_T;
        if (i < n4)
            reinterpret_cast<uint32_t*>(q)[i] = (uint32_t)(quant_code(v[r].x, s) & 0xff) |
                                                ((uint32_t)(quant_code(v[r].y, s) & 0xff) << 8) |
                                                ((uint32_t)(quant_code(v[r].z, s) & 0xff) << 16) |
                                                ((uint32_t)(quant_code(v[r].w, s) & 0xff) << 24);
    }
}

// one-launch quantization of a small contiguous single-segment matrix; false = not eligible
bool quantize_small_eligible(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int8_t* q, int64_t ldq) {
    return ldx == K && ldq == K && ncols * K > 0 && (ncols * K) % 4 == 0 && ncols * K <= QC_CAP &&
           (uintptr_t)x % 16 == 0 && (uintptr_t)q % 4 == 0 && tl_ndev == nullptr;
}

int quantize_small_launch(const float* x, int64_t ncols, int64_t K, int8_t* q, float* scale_out, uint32_t* maxbits_out,
                          int32_t mode, int32_t* err_flag, cudaStream_t st) {
    QNMT_LAUNCH(k_quant_cluster, QC_CTAS, QC_T, 0, st, x, ncols * K / 4, q, scale_out, maxbits_out, mode, err_flag);
    QNMT_CHECK_LAUNCH("k_quant_cluster");
    return QNMT_OK;
}

int quantize_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                    int32_t nseg, int8_t* q, int64_t ldq, float* scales, uint32_t* seg_maxbits,
                    int32_t mode, int32_t* err_flag, cudaStream_t st) {
    if (ncols <= 0 || K <= 0) return QNMT_OK;
    // small single-segment matrices (LinearOp.apply on a batch of columns): one cluster launch
    if (!col_seg && nseg == 1 && scales && seg_maxbits && quantize_small_eligible(x, ncols, K, ldx, q, ldq))
        return quantize_small_launch(x, ncols, K, q, scales, seg_maxbits, mode, err_flag, st);
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
