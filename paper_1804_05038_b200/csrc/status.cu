#include <stdlib.h>
// status.cu -- error plumbing and small utilities of the C ABI.
#include <stdarg.h>
#include <mutex>
#include <string.h>

#include "common.cuh"

namespace qnmt {

static thread_local char g_last_error[512] = "";
thread_local const int32_t* tl_ndev = nullptr;
static unsigned long long g_launches = 0;
std::shared_mutex g_capture_gate;   // see common.cuh

bool pdl_enabled() {
    static const bool on = [] {
        const char* v = getenv("QNMT_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}

void count_launch() { __atomic_fetch_add(&g_launches, 1ULL, __ATOMIC_RELAXED); }

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
    set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
    return QNMT_ERR_CUDA;
}

}  // namespace qnmt

extern "C" {

int qnmt_abi_version(void) { return QNMT_ABI_VERSION; }

const char* qnmt_last_error(void) { return qnmt::g_last_error; }

int64_t qnmt_kernel_launches(void) {
    return (int64_t)__atomic_load_n(&qnmt::g_launches, __ATOMIC_RELAXED);
}

int qnmt_device_sync(void) {
    std::unique_lock<std::shared_mutex> gate(qnmt::g_capture_gate);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return qnmt::cuda_status(e, "cudaDeviceSynchronize");
    return QNMT_OK;
}

}  // extern "C"
