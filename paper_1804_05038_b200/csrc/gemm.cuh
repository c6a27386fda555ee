// gemm.cuh -- internal GEMM entry shared by the ABI wrapper and the engine.
#pragma once
#include "common.cuh"

namespace qnmt {

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
};

int gemm_i8_launch(const GemmArgs& g, cudaStream_t st);
bool tc_eligible(const GemmArgs& g);
int gemm_tc_launch(const GemmArgs& g, cudaStream_t st);
// size the stream's split-K workspace before graph capture ([N][M] int32 + tile counters)
int tc_split_reserve(cudaStream_t st, int64_t ws_elems, int64_t tiles);
extern int g_tc_split;
extern int g_gemm_impl;   // 0 auto, 1 CUDA-core dp4a only, 2 tcgen05 whenever eligible

int quantize_launch(const float* x, int64_t ncols, int64_t K, int64_t ldx, const int32_t* col_seg,
                    int32_t nseg, int8_t* q, int64_t ldq, float* scales, uint32_t* seg_maxbits,
                    int32_t mode, int32_t* err_flag, cudaStream_t st);

}  // namespace qnmt
