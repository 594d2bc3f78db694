// probe.cu — measured fp64 peak of this GPU (the roofline denominator for the
// fp64-bound kernels; MEASURED_PEAKS.json carries HBM and bf16 only).
// 8 independent DFMA chains per thread, 148*8 CTAs x 256 threads; flops are
// counted as 2 per DFMA.
#include "../../include/jabba_b200.h"
#include "jb_device.hpp"

namespace {
__global__ void k_dfma_chain(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
           x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        x0 = __fma_rn(x0, a, b);
        x1 = __fma_rn(x1, a, b);
        x2 = __fma_rn(x2, a, b);
        x3 = __fma_rn(x3, a, b);
        x4 = __fma_rn(x4, a, b);
        x5 = __fma_rn(x5, a, b);
        x6 = __fma_rn(x6, a, b);
        x7 = __fma_rn(x7, a, b);
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace

extern "C" jb_status jb_probe_fp64_tflops(int device, double* tflops) {
    using namespace jb;
    try {
        JB_CUDA(cudaSetDevice(device));
        DArr<double> out(1, 0);
        const int grid = num_sms() * 8, tb = 256, iters = 20000;
        k_dfma_chain<<<grid, tb>>>(out.p, 100, 0.999999, 1e-9);  // warm-up
        cudaEvent_t a, b;
        JB_CUDA(cudaEventCreate(&a));
        JB_CUDA(cudaEventCreate(&b));
        JB_CUDA(cudaEventRecord(a));
        k_dfma_chain<<<grid, tb>>>(out.p, iters, 0.999999, 1e-9);
        JB_CUDA(cudaEventRecord(b));
        JB_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        JB_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        out.release();
        JB_CUDA(cudaDeviceSynchronize());
        *tflops = 2.0 * 8.0 * iters * (double)grid * tb / (ms * 1e-3) / 1e12;
        return JB_OK;
    } catch (const Error& e) {
        return (jb_status)e.code;
    }
}
