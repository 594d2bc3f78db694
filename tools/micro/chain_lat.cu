// Microbenchmark: latency of the quantize carry step formulations (one chain per thread).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int V>
__device__ __forceinline__ double step(double l, double& carry) {
    const double x = l + carry;
    double r;
    if (V == 0) {
        r = floor(x + 0.5);
        if (x >= 0x1p52) r = x;
        if (x < 0.5) r = 1.0;
    } else if (V == 1) {
        r = fmax(floor(x + 0.5), 1.0);
    } else if (V == 2) {
        r = __dsub_rn(__dadd_rz(x + 0.5, 0x1p52), 0x1p52);
        r = fmax(r, 1.0);
    } else {
        r = floor(x + 0.5);
        if (x < 0.5) r = 1.0;
    }
    carry = x - r;
    return r;
}
template <int V>
__global__ void k(const double* tab, const uint8_t* lab, int steps, int nch, double* out, long long* qs) {
    __shared__ double st[256];
    for (int t = threadIdx.x; t < 256; t += blockDim.x) st[t] = tab[t];
    __syncthreads();
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nch) return;
    double carry = 0;
    long long q = 0;
#pragma unroll 16
    for (int i = 0; i < steps; ++i) {
        double r = step<V>(st[((unsigned)i * 2654435761u + (unsigned)c * 40503u) >> 24], carry);
        q += (long long)r;
    }
    out[c] = carry;
    qs[c] = q;
}
int main() {
    const int nch = 10000, steps = 20000;
    double htab[256];
    for (int i = 0; i < 256; ++i) htab[i] = (i % 7 == 0) ? 0.3 + i * 1e-3 : 1.0 + i * 0.0731;
    uint8_t* hl = new uint8_t[(size_t)nch * steps];
    uint64_t s = 1;
    for (size_t i = 0; i < (size_t)nch * steps; ++i) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; hl[i] = s >> 56; }
    double* tab; uint8_t* lab; double* out; long long* qs;
    cudaMalloc(&tab, 2048); cudaMalloc(&lab, (size_t)nch * steps); cudaMalloc(&out, nch * 8 * 4); cudaMalloc(&qs, nch * 8 * 4);
    cudaMemcpy(tab, htab, 2048, cudaMemcpyHostToDevice);
    cudaMemcpy(lab, hl, (size_t)nch * steps, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    void (*ks[4])(const double*, const uint8_t*, int, int, double*, long long*) = {k<0>, k<1>, k<2>, k<3>};

    for (int v = 0; v < 4; ++v) {
        ks[v]<<<(nch + 31) / 32, 32>>>(tab, lab, steps, nch, out + v * nch, qs + v * nch);
        cudaEventRecord(a);
        ks[v]<<<(nch + 31) / 32, 32>>>(tab, lab, steps, nch, out + v * nch, qs + v * nch);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("variant %d: %.3f ms, %.1f ns/step\n", v, ms, ms * 1e6 / steps);
    }
    double* ho = new double[nch * 4]; long long* hq = new long long[nch * 4];
    cudaMemcpy(ho, out, nch * 32, cudaMemcpyDeviceToHost);
    cudaMemcpy(hq, qs, nch * 32, cudaMemcpyDeviceToHost);
    for (int v = 1; v < 4; ++v) {
        int bad = 0;
        for (int c = 0; c < nch; ++c) bad += ho[c] != ho[v * nch + c] || hq[c] != hq[v * nch + c];
        printf("variant %d mismatches vs 0: %d\n", v, bad);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
