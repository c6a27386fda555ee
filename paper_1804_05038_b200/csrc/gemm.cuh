// gemm.cuh -- internal GEMM entry shared by the ABI wrapper and the engine.
#pragma once
#include "common.cuh"

namespace qnmt {

// GRU elementwise phases computed in the tcgen05 GEMM epilogue (layers.py:170-181)
// instead of a separate pass over the products (fused_q.cu k_gates_q / k_combine_q).
//   mode 1 (gates, on the cell's W_x GEMM with bias): rows m < H: z[n][m] =
//     sigmoid((dq + b) + g[n][m]); rows H <= m < 2H: out[n][m-H] = sigmoid((dq + b) +
//     g[n][m]) * h[n][m-H]; rows >= 2H are stored to Y as usual.  g = the U_zr h product.
//   mode 2 (combine, on the U_c GEMM, M = H): out[n][m] = (1 - z) h + z tanh(g[n][m] + dq),
//     g = the candidate rows of the W_x product.
// Both raise segmax[col_seg[n]] to max |out| bits (atomicMax) for the quantization
// of out that follows (quantize_encode_launch); non-finite pre-activations set err_flag.
struct GruEpi {
    int32_t mode = 0;
    int64_t H = 0;
    const float* g = nullptr;
    int64_t ldg = 0;
    const float* h = nullptr;
    int64_t ldh = 0;
    float* z = nullptr;
    float* out = nullptr;
    int64_t ldo = 0;
    uint32_t* segmax = nullptr;
    int32_t* err_flag = nullptr;
};

struct GemmArgs {
    const int8_t* W;
    int64_t M, K, ldw;
    const float* w_scales;
    int64_t w_rows_per_scale;
    const int8_t* X;
    int64_t N, ldx;
    const float* x_scales;
    const int32_t* col_seg;
    const float* bias;
    float* Y;
    int64_t ldy;
    int64_t* acc_out;
    int32_t flags;
    // optional epilogue addends (tcgen05 path only): y = ((dq + bias) + add1[n][m]) + add2[n][m]
    const float* add1 = nullptr;
    int64_t ld1 = 0;
    const float* add2 = nullptr;
    int64_t ld2 = 0;
    // optional GRU epilogue (tcgen05 path only), see GruEpi
    struct GruEpi gru = {};
};

int gemm_i8_launch(const GemmArgs& g, cudaStream_t st);
bool tc_eligible(const GemmArgs& g);
int gemm_tc_launch(const GemmArgs& g, cudaStream_t st);
// two plain products of one shape in one launch (k_gemm_tc_dual)
bool gemm_tc_dual_eligible(const GemmArgs& g0, const GemmArgs& g1);
int gemm_tc_dual_launch(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t st);
// size the stream's split-K workspace before graph capture ([N][M] int32 + tile counters)
int tc_split_reserve(cudaStream_t st, int64_t ws_elems, int64_t tiles);
extern int g_tc_split;
extern int g_gemm_impl;   // 0 auto, 1 CUDA-core dp4a only, 2 tcgen05 whenever eligible

int quantize_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                    int32_t nseg, int8_t* q, int64_t ldq, float* scales, uint32_t* seg_maxbits,
                    int32_t mode, int32_t* err_flag, cudaStream_t st);

bool quantize_small_eligible(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int8_t* q, int64_t ldq);
int quantize_small_launch(const float* x, int64_t ncols, int64_t K, int8_t* q, float* scale_out, uint32_t* maxbits_out,
                          int32_t mode, int32_t* err_flag, cudaStream_t st);

}  // namespace qnmt
