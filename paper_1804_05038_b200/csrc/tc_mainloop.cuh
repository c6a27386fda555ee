// tc_mainloop.cuh -- the warp-specialised tcgen05 int8 main loop shared by the
// plain GEMM (gemm_tcgen05.cu) and the fused vocab GEMM + softmax statistics
// (vocab_topk.cu).
//
//   D[i][j] = sum_k A[i][k] * B[j][k]   A tile [128 x 128 B], B tile [BN x 128 B]
//
// warp 0 lane 0: TMA producer into a STAGES-deep ring (SWIZZLE_128B, K-major);
// warp 1 lane 0: tcgen05.mma.cta_group::1.kind::i8 issuer, int32 accumulators in
//   TMEM, double-buffered (buffer b at column b*BN) so the epilogue of tile t
//   overlaps the MMAs of tile t+1.  Tiles t = blockIdx.x, +gridDim.x, ... (or a given
//   [t0, tiles) range with stride tstep);
//   t -> (a-block t / n_blocks, b-block t % n_blocks).
#pragma once
#include "tc_common.cuh"

namespace qnmt {

constexpr int TC_BM = 128;
constexpr int TC_BK = 128;   // bytes of K per stage (= int8 elements)

template <int BN, int STAGES_>
struct TcRing {
    static constexpr int A_BYTES = TC_BM * TC_BK;
    static constexpr int B_BYTES = BN * TC_BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = STAGES_;
    static constexpr int TMEM_COLS = 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;   // pow2
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// barriers live right after the ring: full[STAGES], empty[STAGES], tfull[2], tempty[2], tmem slot
template <class R>
struct TcBars {
    uint64_t* full;
    uint64_t* empty;
    uint64_t* tfull;
    uint64_t* tempty;
    uint32_t* tmem_slot;
    __device__ explicit TcBars(unsigned char* smem) {
        full = reinterpret_cast<uint64_t*>(smem + R::STAGES * R::STAGE_BYTES);
        empty = full + R::STAGES;
        tfull = empty + R::STAGES;
        tempty = tfull + 2;
        tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    }
};

// barrier init (warp 0 lane 0) + TMEM allocation (warp 1); ends with a CTA barrier.
template <class R>
__device__ __forceinline__ uint32_t tc_setup(const CUtensorMap* tmA, const CUtensorMap* tmB, const TcBars<R>& b,
                                             int epi_warps) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(tmA);
        tc::prefetch_tmap(tmB);
        for (int s = 0; s < R::STAGES; ++s) {
            tc::mbar_init(&b.full[s], 1);
            tc::mbar_init(&b.empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&b.tfull[i], 1);
            tc::mbar_init(&b.tempty[i], epi_warps);
        }
        tc::fence_mbar_init();
    }
    if (warp == 1) tc::tmem_alloc<R::TMEM_COLS>(b.tmem_slot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    return *b.tmem_slot;
}

// split-K: tile t covers output tile t / ksplit and k-blocks [kb0, kb1) of split t % ksplit
__device__ __forceinline__ void tc_krange(int tile, int ksplit, int k_blocks, int& mn, int& kb0, int& kb1) {
    if (ksplit <= 1) {
        mn = tile;
        kb0 = 0;
        kb1 = k_blocks;
        return;
    }
    const int kpb = (k_blocks + ksplit - 1) / ksplit;
    mn = tile / ksplit;
    kb0 = (tile % ksplit) * kpb;
    kb1 = min(k_blocks, kb0 + kpb);
}

// Static A operand (weights): the A blocks of the CTA's first tile can be requested before the
// programmatic-dependent-launch wait -- they do not depend on the predecessor kernel, so they
// stream from HBM while it (e.g. the activation quantization) still runs.  Warp 0 lane 0, after
// tc_setup; `pre` = min(STAGES, k_blocks) stages, each armed for the full stage (the B block is
// added by tc_produce(..., pre) after the wait).  Requires ksplit == 1, blockIdx.x < tiles and a
// host-known n_blocks.
template <class R>
__device__ __forceinline__ void tc_prefetch_a(const CUtensorMap* tmA, unsigned char* smem, const TcBars<R>& b,
                                              int n_blocks, int pre) {
    const int ab = (int)blockIdx.x / n_blocks;
    for (int s = 0; s < pre; ++s) {
        tc::mbar_arrive_expect_tx(&b.full[s], R::STAGE_BYTES);
        tc::tma_load_2d(smem + s * R::STAGE_BYTES, tmA, &b.full[s], s * TC_BK, ab * TC_BM);
    }
}

template <class R, int BN>
__device__ __forceinline__ void tc_produce(const CUtensorMap* tmA, const CUtensorMap* tmB, unsigned char* smem,
                                           const TcBars<R>& b, int tiles, int n_blocks, int k_blocks,
                                           int t0 = -1, int tstep = 0, int ksplit = 1, int pre = 0) {
    if ((threadIdx.x & 31) != 0) return;
    int stage = 0;
    uint32_t phase = 0;
    if (t0 < 0) {   // default: persistent round-robin
        t0 = blockIdx.x;
        tstep = gridDim.x;
    }
    for (int tile = t0; tile < tiles; tile += tstep) {
        int mn, kbs, kbe;
        tc_krange(tile, ksplit, k_blocks, mn, kbs, kbe);
        const int ab = mn / n_blocks, bb = mn % n_blocks;
        for (int kb = kbs; kb < kbe; ++kb) {
            tc::mbar_wait(&b.empty[stage], phase ^ 1);
            unsigned char* sa = smem + stage * R::STAGE_BYTES;
            unsigned char* sb = sa + R::A_BYTES;
            if (!(pre > 0 && tile == t0 && kb < pre)) {   // (else armed and A requested by tc_prefetch_a)
                tc::mbar_arrive_expect_tx(&b.full[stage], R::STAGE_BYTES);
                tc::tma_load_2d(sa, tmA, &b.full[stage], kb * TC_BK, ab * TC_BM);
            }
            tc::tma_load_2d(sb, tmB, &b.full[stage], kb * TC_BK, bb * BN);
            if (++stage == R::STAGES) { stage = 0; phase ^= 1; }
        }
    }
}

template <class R, int BN>
__device__ __forceinline__ void tc_issue(unsigned char* smem, const TcBars<R>& b, uint32_t tmem_base, int tiles,
                                         int k_blocks, int t0 = -1, int tstep = 0, int ksplit = 1) {
    constexpr uint32_t IDESC = tc::idesc_i8(TC_BM, BN);
    const int lane = threadIdx.x & 31;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    if (t0 < 0) {
        t0 = blockIdx.x;
        tstep = gridDim.x;
    }
    for (int tile = t0; tile < tiles; tile += tstep, ++it) {
        const int buf = it & 1;
        const uint32_t use = (uint32_t)(it >> 1) & 1u;
        tc::mbar_wait(&b.tempty[buf], use ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(buf * BN);
        int mn, kbs, kbe;
        tc_krange(tile, ksplit, k_blocks, mn, kbs, kbe);
        for (int kb = kbs; kb < kbe; ++kb) {
            tc::mbar_wait(&b.full[stage], phase);
            tc::tc_fence_after();
            if (lane == 0) {
                const uint32_t a0 = tc::smem_u32(smem + stage * R::STAGE_BYTES);
                const uint32_t b0 = a0 + R::A_BYTES;
#pragma unroll
                for (int k = 0; k < TC_BK / 32; ++k)
                    tc::mma_i8(d, tc::sw128_kmajor_desc(a0 + 32 * k), tc::sw128_kmajor_desc(b0 + 32 * k), IDESC,
                               (kb != kbs) || k != 0);
                tc::mma_commit(&b.empty[stage]);
                if (kb == kbe - 1) tc::mma_commit(&b.tfull[buf]);
            }
            __syncwarp();
            if (++stage == R::STAGES) { stage = 0; phase ^= 1; }
        }
    }
}

// host: K-major int8 tensor map with a [TC_BK x box_rows] box (cached per pointer/shape)
int tc_get_map(const int8_t* p, int64_t rows, int64_t cols, int64_t ld, int box_rows, CUtensorMap* out);
int tc_sm_count();

}  // namespace qnmt
