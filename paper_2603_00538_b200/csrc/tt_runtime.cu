// Library plumbing: error text, device properties, measurement probes.
#include <stdarg.h>
#include <mutex>
#include "tt_common.cuh"

namespace tt {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return TT_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return TT_ERR_CUDA;
}

int sm_count() {
    static int cached = 0;
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

// Independent DFMA chains: 8 per thread, fully unrolled; the measured rate is the FP64
// issue ceiling the fused on-the-fly kernels are compared against.
__global__ void fp64_probe_kernel(int64_t iters, double* sink) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double m = 0.999999999, c = 1e-12;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
            a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
        }
    }
    sink[blockIdx.x * (int64_t)blockDim.x + threadIdx.x] = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
}

}  // namespace tt

using namespace tt;

extern "C" const char* tt_last_error(void) { return g_err; }

extern "C" int tt_version(void) { return 100; }

extern "C" int tt_device_sm_count(int* out) {
    *out = sm_count();
    return TT_OK;
}

extern "C" int tt_fp64_peak_probe(int64_t iters, double* sink, int* blocks_out, int* threads_out,
                                  void* stream) {
    int threads = 256;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fp64_probe_kernel, threads, 0);
    if (per_sm < 1) per_sm = 1;
    int blocks = sm_count() * per_sm;
    if (blocks_out) *blocks_out = blocks;
    if (threads_out) *threads_out = threads;
    if (!sink) return TT_OK;  // size query
    fp64_probe_kernel<<<blocks, threads, 0, as_stream(stream)>>>(iters, sink);
    return launch_check("fp64_probe_kernel");
}
