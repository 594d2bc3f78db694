// inverse.cu — inverse symbolization on sm_100a (inverse.hpp:32-132,
// compression.hpp:87-103, 198-213).
//
// Two kernels:
//  1. one thread per segment runs the three inherently sequential
//     recurrences exactly as the reference does: inverse digitization
//     (:32-51), error-carrying rounding with clamp (quantize_lengths :63-74),
//     the backward length fix-up (match_total_length :81-93), and the running
//     start value v += inc (inverse_compress :94-101). It records, per piece,
//     the start value and the absolute output position.
//  2. one thread per piece writes its interpolated samples
//     v + inc * (i / len) straight into the (optionally stitched) output: the
//     bandwidth-bound fill.
#include <algorithm>

#include "jb_device.hpp"

namespace jb {

namespace {

constexpr int64_t SKIP_LAST = 1LL << 62;  // flag: don't write this piece's last sample

__global__ void k_inv_seq(InverseIn in, int64_t* __restrict__ qlen, double* __restrict__ vstart,
                          int64_t* __restrict__ pstart, double* __restrict__ out,
                          unsigned long long* __restrict__ err) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= in.n_seg) return;
    const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
    const double scl = in.scl, sl = in.sigma_len, si = in.sigma_inc;
    // inverse_digitize_series + quantize_lengths
    double carry = 0.0;
    int64_t total = 0;
    for (int64_t j = a; j < b; ++j) {
        const uint32_t lab = in.labels[j];
        if ((uint64_t)lab >= in.k) {
            atomicMin(err, (unsigned long long)(s * 16 + UNKNOWN_SYMBOL));
            return;
        }
        const double l = scl > 0.0 ? in.centers[2 * lab] * sl / scl : in.mean_lengths[lab];
        int64_t r = llround(l + carry);
        if (r < 1) r = 1;
        carry = l + carry - (double)r;
        qlen[j] = r;
        total += r;
    }
    // match_total_length
    int64_t residual = in.source_lengths[s] - total;
    for (int64_t j = b; j-- > a && residual != 0;) {
        int64_t adj = qlen[j] + residual;
        if (adj < 1) adj = 1;
        residual -= adj - qlen[j];
        qlen[j] = adj;
    }
    if (residual != 0 || b == a) {
        atomicMin(err, (unsigned long long)(s * 16 + INVALID_PIECE));
        return;
    }
    // inverse_compress: running value and output positions
    const int64_t base = in.out_offsets[s];
    const double anchor = in.anchors[s];
    out[base] = anchor;
    double v = anchor;
    int64_t pos = base;
    const bool drop_last = in.layout == 0 && s + 1 < in.n_seg;  // stitch_partitions
    for (int64_t j = a; j < b; ++j) {
        vstart[j] = v;
        pstart[j] = pos | ((drop_last && j == b - 1) ? SKIP_LAST : 0);
        const uint32_t lab = in.labels[j];
        v += in.centers[2 * lab + 1] * si;  // RealPiece::inc = c1 * sigma_inc
        pos += qlen[j];
    }
}

__global__ void k_inv_fill(InverseIn in, const int64_t* __restrict__ qlen,
                           const double* __restrict__ vstart, const int64_t* __restrict__ pstart,
                           double* __restrict__ out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < in.N;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = qlen[j];
        const int64_t ps = pstart[j];
        const int64_t p0 = ps & ~SKIP_LAST;
        const int64_t n_write = (ps & SKIP_LAST) ? len - 1 : len;
        const double v = vstart[j];
        const double inc = in.centers[2 * in.labels[j] + 1] * in.sigma_inc;
        const double l = (double)len;
        for (int64_t i = 1; i <= n_write; ++i) out[p0 + i] = v + inc * ((double)i / l);
    }
}

}  // namespace

void inverse_transform_device(const InverseIn& in, double* d_out, cudaStream_t st) {
    if (in.layout == 0 && in.n_seg == 0)
        throw Error(INVALID_INPUT, "stitch_partitions: no segments");
    DArr<int64_t> qlen(std::max<int64_t>(in.N, 1), st), pstart(std::max<int64_t>(in.N, 1), st);
    DArr<double> vstart(std::max<int64_t>(in.N, 1), st);
    DArr<unsigned long long> err(1, st);
    const unsigned long long none = ~0ULL;
    err.upload(&none, 1);
    {
        JB_PROF("inverse_seq", st);
        k_inv_seq<<<(int)((in.n_seg + 127) / 128), 128, 0, st>>>(in, qlen.p, vstart.p, pstart.p,
                                                              d_out, err.p);
    }
    JB_LAUNCH_CHECK();
    unsigned long long e;
    err.download(&e, 1);
    JB_CUDA(cudaStreamSynchronize(st));
    if (e != ~0ULL) {
        const int code = (int)(e % 16);
        const long long seg = (long long)(e / 16);
        if (code == UNKNOWN_SYMBOL)
            throw Error(UNKNOWN_SYMBOL,
                        "label not in codebook of size " + std::to_string(in.k) +
                            " (segment " + std::to_string(seg) + ")");
        throw Error(INVALID_PIECE, "cannot fit pieces into the segment's steps (segment " +
                                       std::to_string(seg) + ")");
    }
    if (in.N > 0) {
        const int grid =
            (int)std::max<int64_t>(1, std::min<int64_t>((in.N + 255) / 256, (int64_t)kSMs * 16));
        {
            JB_PROF("inverse_fill", st);
            k_inv_fill<<<grid, 256, 0, st>>>(in, qlen.p, vstart.p, pstart.p, d_out);
        }
        JB_LAUNCH_CHECK();
    }
}

}  // namespace jb
