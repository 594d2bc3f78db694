// inverse.cu — inverse symbolization on sm_100a (inverse.hpp:32-132,
// compression.hpp:87-103, 198-213).
//
// The reference's recurrences are sequential and stay sequential: one
// thread per segment runs the carry / length-fix-up / start-value chains in
// the reference's rounding (all segments are resident in one wave), then a
// piece-parallel fill writes the interpolated samples v + inc * (i / len)
// straight into the (optionally stitched, :198-213) output.
#include <algorithm>

#include "jb_device.hpp"

namespace jb {

namespace {

__global__ void k_inv_tables(const double* __restrict__ centers,
                             const double* __restrict__ mean_lengths, uint64_t k, double scl,
                             double sl, double si, double* __restrict__ rlen,
                             double* __restrict__ rinc) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < k;
         c += (uint64_t)gridDim.x * blockDim.x) {
        rlen[c] = scl > 0.0 ? centers[2 * c] * sl / scl : mean_lengths[c];
        rinc[c] = centers[2 * c + 1] * si;
    }
}

// llround (round half away from zero) of x, as a double, using only exact
// fp64 operations: trunc, the exact remainder x - trunc(x), one compare.
__device__ __forceinline__ double llround_d(double x) {
    double r = trunc(x);
    const double f = x - r;  // exact
    if (f >= 0.5) r += 1.0;
    else if (f <= -0.5) r -= 1.0;
    return r;
}

constexpr int64_t SKIP_LAST = 1LL << 62;  // flag: don't write this piece's last sample

// One thread per segment: the reference's sequential recurrences, exactly.
//   quantize_lengths (:63-74): r = llround(l + carry), clamp >= 1,
//     carry = (l + carry) - r  -- r kept as an exact double, so the carry
//     chain has no int<->fp conversions;
//   match_total_length (:81-93): backward cascade on the tail;
//   inverse_compress (:94-101): v += inc (start value of every piece) and
//     the running output position.
// The three chains are independent and run interleaved in one loop.
__global__ void __launch_bounds__(128) k_inv_chain(InverseIn in, const double* __restrict__ rlen,
                                                   const double* __restrict__ rinc,
                                                   int32_t* __restrict__ qlen,
                                                   double* __restrict__ vstart,
                                                   int64_t* __restrict__ pstart,
                                                   double* __restrict__ out,
                                                   unsigned long long* __restrict__ err) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= in.n_seg) return;
    const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
    for (int64_t j = a; j < b; ++j)  // inverse_digitize_series validates first (:41-44)
        if ((uint64_t)in.labels[j] >= in.k) {
            atomicMin(err, (unsigned long long)(s * 16 + UNKNOWN_SYMBOL));
            return;
        }
    const bool drop_last = in.layout == 0 && s + 1 < in.n_seg;  // stitch_partitions
    const int64_t base = in.out_offsets[s];
    double carry = 0.0, v = in.anchors[s];
    int64_t pos = base, total = 0;
    out[base] = v;
    int64_t j = a;
    constexpr int U = 4;
    for (; j + U <= b; j += U) {
        uint32_t lab[U];
#pragma unroll
        for (int u = 0; u < U; ++u) lab[u] = in.labels[j + u];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double l = __ldg(rlen + lab[u]);
            const double x = l + carry;
            double r = llround_d(x);
            if (r < 1.0) r = 1.0;
            carry = x - r;
            const int32_t q = (int32_t)r;
            qlen[j + u] = q;
            vstart[j + u] = v;
            pstart[j + u] = pos;
            v += __ldg(rinc + lab[u]);
            pos += q;
            total += q;
        }
    }
    for (; j < b; ++j) {
        const uint32_t lab = in.labels[j];
        const double l = __ldg(rlen + lab);
        const double x = l + carry;
        double r = llround_d(x);
        if (r < 1.0) r = 1.0;
        carry = x - r;
        const int32_t q = (int32_t)r;
        qlen[j] = q;
        vstart[j] = v;
        pstart[j] = pos;
        v += __ldg(rinc + lab);
        pos += q;
        total += q;
    }
    // match_total_length: backward cascade; positions after the first
    // modified piece are recomputed
    long long residual = in.source_lengths[s] - total;
    int64_t first_mod = b;
    for (int64_t t = b; t-- > a && residual != 0;) {
        long long adj = (long long)qlen[t] + residual;
        if (adj < 1) adj = 1;
        residual -= adj - qlen[t];
        qlen[t] = (int32_t)adj;
        first_mod = t;
    }
    if (residual != 0 || b == a) {
        atomicMin(err, (unsigned long long)(s * 16 + INVALID_PIECE));
        return;
    }
    if (first_mod < b) {
        int64_t p = pstart[first_mod];
        for (int64_t t = first_mod; t < b; ++t) {
            pstart[t] = p;
            p += qlen[t];
        }
    }
    if (drop_last) pstart[b - 1] |= SKIP_LAST;
}

// interpolation fill (inverse_compress :97-99): v + inc * (i / len)
__global__ void k_inv_fill(InverseIn in, const double* __restrict__ rinc,
                           const int32_t* __restrict__ qlen, const double* __restrict__ vstart,
                           const int64_t* __restrict__ pstart, double* __restrict__ out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < in.N;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = qlen[j];
        const int64_t ps = pstart[j];
        const int64_t p0 = ps & ~SKIP_LAST;
        const int64_t n_write = (ps & SKIP_LAST) ? len - 1 : len;
        const double v = vstart[j];
        const double inc = __ldg(rinc + in.labels[j]);
        const double l = (double)len;
        for (int64_t i = 1; i <= n_write; ++i) out[p0 + i] = v + inc * ((double)i / l);
    }
}

}  // namespace

void inverse_transform_device(const InverseIn& in, double* d_out, cudaStream_t st) {
    if (in.layout == 0 && in.n_seg == 0)
        throw Error(INVALID_INPUT, "stitch_partitions: no segments");
    DArr<int32_t> qlen(std::max<int64_t>(in.N, 1), st);
    const uint64_t kk = std::max<uint64_t>(in.k, 1);
    DArr<double> tab(2 * kk, st);
    DArr<unsigned long long> err(1, st);
    const unsigned long long none = ~0ULL;
    err.upload(&none, 1);
    if (in.k > 0) {
        k_inv_tables<<<(int)std::min<uint64_t>((in.k + 255) / 256, 1024), 256, 0, st>>>(
            in.centers, in.mean_lengths, in.k, in.scl, in.sigma_len, in.sigma_inc, tab.p,
            tab.p + kk);
        JB_LAUNCH_CHECK();
    }
    DArr<double> vstart(std::max<int64_t>(in.N, 1), st);
    DArr<int64_t> pstart(std::max<int64_t>(in.N, 1), st);
    {
        JB_PROF("inverse_chain", st);
        k_inv_chain<<<(int)((in.n_seg + 127) / 128), 128, 0, st>>>(
            in, tab.p, tab.p + kk, qlen.p, vstart.p, pstart.p, d_out, err.p);
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
        JB_PROF("inverse_fill", st);
        const int grid =
            (int)std::max<int64_t>(1, std::min<int64_t>((in.N + 255) / 256, (int64_t)kSMs * 16));
        k_inv_fill<<<grid, 256, 0, st>>>(in, tab.p + kk, qlen.p, vstart.p, pstart.p, d_out);
        JB_LAUNCH_CHECK();
    }
}

}  // namespace jb
