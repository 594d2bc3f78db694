// Microbenchmark: dependent DADD chain latency, and the chain with an
// independent shared-memory table lookup per step (one thread per chain).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_dadd(const double* tab, const uint32_t* lab, int steps, double* out, long long* cyc) {
    __shared__ double st[256];
    for (int t = threadIdx.x; t < 256; t += blockDim.x) st[t] = tab[t];
    __syncthreads();
    double v = threadIdx.x;
    const double inc = tab[threadIdx.x & 255];
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < steps; ++i) v += inc;
    long long t1 = clock64();
#pragma unroll 16
    for (int i = 0; i < steps; ++i) v += st[(lab[i & 1023] + threadIdx.x) & 255];
    long long t2 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
    double *tab, *out; uint32_t* lab; long long* cyc;
    cudaMallocManaged(&tab, 256 * 8); cudaMallocManaged(&out, 1024 * 8);
    cudaMallocManaged(&lab, 1024 * 4); cudaMallocManaged(&cyc, 16);
    for (int i = 0; i < 256; ++i) tab[i] = 1.0 + i * 1e-3;
    for (int i = 0; i < 1024; ++i) lab[i] = (i * 2654435761u) >> 24;
    const int steps = 1 << 16;
    k_dadd<<<1, 32>>>(tab, lab, steps, out, cyc);
    cudaDeviceSynchronize();
    printf("dadd chain: %.2f cycles/step; with smem lookup: %.2f cycles/step\n",
           (double)cyc[0] / steps, (double)cyc[1] / steps);
    return 0;
}
