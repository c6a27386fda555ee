// common.cuh -- shared helpers for the qnmt B200 kernels (sm_100a).
//
// Numerics rules:
//  * f32 elementwise ops that the reference performs as separate numpy f32
//    ufuncs are written with __fadd_rn / __fmul_rn / __fsub_rn so ptxas can
//    never contract them into FMAs.
//  * sigmoid / tanh / exp / log are evaluated in fp64 and rounded once to f32
//    (the "Tier B" contract of oracle/qnmt_oracle.py).
//  * dequantization is fl32(f64(acc) / (f64(sa) * f64(sb))) (qmath.py:379-381).
#pragma once
#include <shared_mutex>

#include <cuda_runtime.h>

#include <mutex>
#include <utility>
#include <stdint.h>
#include <stdio.h>

#include "../../include/qnmt_b200.h"
#include "act.cuh"

namespace qnmt {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
void count_launch();

// Device-resident column count for graph-captured decode steps: when set, the
// launch helpers size grids for the host-side maximum and every kernel reads
// the live count from *tl_ndev (blocks beyond it exit immediately).
extern thread_local const int32_t* tl_ndev;
struct NdevScope {
    const int32_t* old;
    explicit NdevScope(const int32_t* p) : old(tl_ndev) { tl_ndev = p; }
    ~NdevScope() { tl_ndev = old; }
};

// Programmatic dependent launch (PDL): kernels of the decode path are launched
// with programmatic stream serialization, so a kernel's CTAs are scheduled while
// its predecessor's last CTAs still run; every such kernel calls pdl_entry()
// (wait for the predecessor's completion + memory, then let the successor
// launch) before touching data the predecessor wrote.  Both instructions are
// no-ops for a normal launch.  QNMT_PDL=0 in the environment disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() {
    pdl_wait();
    pdl_trigger();
}
bool pdl_enabled();

// Raise a kernel's dynamic shared-memory limit to at least `bytes` (host threads
// driving separate engines may race here: check-and-set under one lock so the
// limit only grows).  `done` is the caller's per-kernel high-water mark.
inline cudaError_t raise_smem_limit(const void* fn, size_t bytes, size_t& done) {
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (bytes <= done) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done = bytes;
    return e;
}

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                   Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define QNMT_LAUNCH(kern, grid, block, smem, st, ...)                                                   \
    do {                                                                                              \
        cudaError_t _le = ::qnmt::launch_k(kern, grid, block, smem, st, __VA_ARGS__);                  \
        if (_le != cudaSuccess) return ::qnmt::cuda_status(_le, #kern);                               \
    } while (0)

#define QNMT_CHECK_LAUNCH(where)                                              \
    do {                                                                      \
        ::qnmt::count_launch();                                               \
        cudaError_t _e = cudaGetLastError();                                  \
        if (_e != cudaSuccess) return ::qnmt::cuda_status(_e, where);         \
    } while (0)

#define QNMT_CUDA(call)                                                       \
    do {                                                                      \
        cudaError_t _e = (call);                                              \
        if (_e != cudaSuccess) return ::qnmt::cuda_status(_e, #call);         \
    } while (0)

// Stream captures vs device-wide synchronisation.  Engines capture their step graphs on their
// own (non-blocking) streams from whatever host thread decodes; a device-wide synchronisation or
// a cudaFree issued by ANOTHER thread at that moment (an engine being destroyed by the garbage
// collector, a history block being regrown) invalidates the capture in flight
// ("operation failed due to a previous error during capture").  Captures hold this gate shared,
// the device-wide calls hold it exclusively.  (status.cu defines it.)
extern std::shared_mutex g_capture_gate;

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// device math
// ---------------------------------------------------------------------------

// Tier-B transcendental helpers (evaluate in fp64, round once to f32): act.cuh
__device__ __forceinline__ bool beyond(const int32_t* n_dev, int64_t i) {
    return n_dev != nullptr && i >= (int64_t)*n_dev;
}

__device__ __forceinline__ bool is_finite_f(float x) {
    return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}

// Code assignment of qmath.py:119-133 for one value with scale s.
__device__ __forceinline__ int quant_code(float x, float s) {
    float v = __fmul_rn(x, s);
    float q = floorf(__fadd_rn(fabsf(v), 0.5f));
    if (v < 0.0f) q = -q;
    q = fminf(fmaxf(q, -127.0f), 127.0f);
    return (int)q;
}

// Scale rule of qmath.py:136-142 from the max magnitude (as u32 bits of |x|).
__device__ __forceinline__ float scale_from_maxbits(uint32_t bits) {
    float m = __uint_as_float(bits);
    return (bits == 0u) ? 1.0f : __fdiv_rn(127.0f, m);
}

// Dequantization of qmath.py:379-381.
__device__ __forceinline__ float dequant(long long acc, float sa, float sb) {
    double den = __dmul_rn((double)sa, (double)sb);
    return __double2float_rn(__ddiv_rn((double)acc, den));
}

// Same value as dequant(), but via a reciprocal multiply: q = acc * (1/sa)(1/sb)
// carries at most a few f64 ulps of error, so fl32(q) equals the correctly
// rounded fl32(acc / (sa*sb)) unless q lies within a few f64 ulps of an f32
// rounding midpoint (low 29 mantissa bits ~ 0x10000000) or outside the normal
// f32 range -- only then is the exact __ddiv_rn evaluated (~1e-7 of elements).
__device__ __forceinline__ float dequant_rcp(long long acc, double rcp, float sa, float sb) {
    double q = (double)acc * rcp;
    unsigned long long b = (unsigned long long)__double_as_longlong(q);
    int low = (int)(b & 0x1fffffffull);
    int ex = (int)((b >> 52) & 0x7ff);
    bool safe = (low - 0x10000000 > 64 || 0x10000000 - low > 64) && ex > 1023 - 125 && ex < 1023 + 127;
    if (acc == 0) return 0.0f;
    if (safe) return __double2float_rn(q);
    return dequant(acc, sa, sb);
}

// Predicate of dequant_rcp's fast path for q = acc * rcp: zero, or a normal-range
// value whose bits are more than 64 f64-ulps away from an f32 rounding midpoint.
// (double)v for an int32 v through the exponent field (fp64 pipe, exact):
// 2^52 + (v + 2^31) - (2^52 + 2^31) -- the XU conversion is the scarcer pipe in epilogues.
__device__ __forceinline__ double i2d_exact(int v) {
    return __hiloint2double(0x43300000, (int)((unsigned)v ^ 0x80000000u)) - 4503601774854144.0;
}

__device__ __forceinline__ bool dequant_rcp_safe(double q) {
    unsigned long long b = (unsigned long long)__double_as_longlong(q);
    int low = (int)(b & 0x1fffffffull);
    int ex = (int)((b >> 52) & 0x7ff);
    int d = low - 0x10000000;
    return ((b << 1) == 0ull) || ((d > 64 || d < -64) && ex > 1023 - 125 && ex < 1023 + 127);
}

__device__ __forceinline__ void set_flag(int32_t* flag, int bit) {
    if (flag) atomicOr(flag, bit);
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// 16-byte streaming load that bypasses L1 allocation (weights are read once).
__device__ __forceinline__ int4 ld_stream16(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

}  // namespace qnmt
