// Microbenchmark: latency per step of the quantize_lengths carry recurrence
// (inverse.hpp:63-74) on one thread, with different llround formulations,
// plus the plain DADD chain (v += inc). nvcc -O3 -fmad=false -arch=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double llround_d(double x) {
    double r = trunc(x);
    const double f = x - r;
    if (f >= 0.5) r += 1.0;
    else if (f <= -0.5) r -= 1.0;
    return r;
}

template <int MODE>
__global__ void k_chain(const double* l, int n, double* out, long long* cyc) {
    double carry = 0.0, acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        const double x = l[i & 1023] + carry;
        if (MODE == 0) {  // llround + int conversions
            long long r = llround(x);
            if (r < 1) r = 1;
            carry = x - (double)r;
        } else if (MODE == 1) {  // fp64-only llround
            double r = llround_d(x);
            if (r < 1.0) r = 1.0;
            carry = x - r;
        } else {  // plain DADD chain
            carry = x;
        }
        acc += carry;
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    cyc[0] = t1 - t0;
}

int main() {
    double *l, *out;
    long long* cyc;
    cudaMalloc(&l, 1024 * 8);
    cudaMalloc(&out, 1024 * 8);
    cudaMallocManaged(&cyc, 8);
    double h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = 1.0 + (i % 7) * 0.37;
    cudaMemcpy(l, h, sizeof h, cudaMemcpyHostToDevice);
    const int n = 1 << 20;
    const char* names[3] = {"llround+cvt", "fp64 llround", "dadd chain"};
    for (int m = 0; m < 3; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            if (m == 0) k_chain<0><<<1, 1>>>(l, n, out, cyc);
            if (m == 1) k_chain<1><<<1, 1>>>(l, n, out, cyc);
            if (m == 2) k_chain<2><<<1, 1>>>(l, n, out, cyc);
            cudaDeviceSynchronize();
        }
        printf("%-14s %.1f cycles/step\n", names[m], (double)cyc[0] / n);
    }
    return 0;
}
