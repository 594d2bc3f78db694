// Microbenchmark: cost of a cooperative-groups grid.sync() at the Lloyd loop's grid shape.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned long long* out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;
// a flat barrier: one arrival counter, generation flag polled by one thread per block
__global__ void k2(int iters, unsigned long long* out) {
    unsigned int gen = 0;
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            gen = g_gen;
            __threadfence();
            if (atomicAdd(&g_count, 1) == gridDim.x - 1) {
                g_count = 0;
                __threadfence();
                g_gen = gen + 1;
            } else {
                while (g_gen == gen) {}
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = iters;
}
int main() {
    unsigned long long* o;
    cudaMalloc(&o, 8);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 256, 0);
    int blocks = 148 * 3;
    for (int rep = 0; rep < 2; ++rep) {
        for (int which = 0; which < 2; ++which) {
            int iters = 3000;
            void* args[] = {&iters, &o};
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            if (which == 0) cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
            else cudaLaunchCooperativeKernel((void*)k2, blocks, 256, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("%s: %d blocks x 256: %.3f us per sync (%s)\n", which ? "flat" : "grid.sync", blocks,
                   ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
}
