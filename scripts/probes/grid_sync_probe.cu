// Microbenchmark: cost of cooperative-groups grid.sync() on this GPU (measurement aid).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, double* sink) {
    cg::grid_group g = cg::this_grid();
    double a = threadIdx.x;
    for (int i = 0; i < iters; ++i) { a = a * 0.999 + 1.0; g.sync(); }
    if (a == 12345.0) sink[0] = a;
}
int main() {
    double* sink; cudaMalloc(&sink, 8);
    int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int cfg[][2] = {{256, 1}, {256, 4}, {512, 1}, {512, 2}, {1024, 1}};
    for (auto& c : cfg) {
        int blocks = sms * c[1], threads = c[0];
        int iters = 2000;
        void* args[] = {&iters, &sink};
        cudaLaunchCooperativeKernel((void*)k, blocks, threads, args, 0, 0);
        cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
        cudaEventRecord(s);
        cudaLaunchCooperativeKernel((void*)k, blocks, threads, args, 0, 0);
        cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e);
        printf("blocks %d x %d threads: %.3f us per grid.sync (%s)\n", blocks, threads, ms * 1000 / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
