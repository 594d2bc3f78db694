// inverse.cu — inverse symbolization on sm_100a (inverse.hpp:32-132,
// compression.hpp:87-103, 198-213).
//
// One warp per segment. The recurrences of the reference are sequential and
// are kept sequential -- every lane replays the same chain on values
// broadcast by shuffles, so the rounding is the reference's exactly -- while
// all memory traffic is warp-coalesced:
//   pass 1  labels -> real lengths (inverse_digitize_series :32-51, per-label
//           table) -> error-carrying rounding with clamp (quantize_lengths
//           :63-74) -> int32 lengths, then the backward fix-up
//           (match_total_length :81-93);
//   pass 2  running start value v += inc (inverse_compress :94-101) and an
//           exact integer scan of the lengths give every piece its start
//           value and output position; the warp then writes the group's
//           samples v + inc * (i / len) contiguously, straight into the
//           (optionally stitched, :198-213) output.
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

constexpr int INV_TB = 256;

__global__ void __launch_bounds__(INV_TB) k_inv_warp(InverseIn in, const double* __restrict__ rlen,
                                                    const double* __restrict__ rinc,
                                                    int32_t* __restrict__ qlen,
                                                    double* __restrict__ out,
                                                    unsigned long long* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < in.n_seg;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
        // ---- pass 1: quantize ----
        double carry = 0.0;
        long long total = 0;
        bool bad = false;
        for (int64_t base = a; base < b; base += 32) {
            const int64_t j = base + lane;
            const bool valid = j < b;
            const uint32_t lab = valid ? in.labels[j] : 0u;
            if (__any_sync(FULL, valid && (uint64_t)lab >= in.k)) {
                bad = true;
                break;
            }
            const double l = valid ? __ldg(rlen + lab) : 0.0;
            const int cnt = (int)((b - base) < 32 ? (b - base) : 32);
            int myr = 0;
            // fully unrolled (cnt is warp-uniform): the 32 broadcasts are
            // independent of the carry, so only the rounding chain is serial
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const double li = __shfl_sync(FULL, l, i);
                if (i < cnt) {
                    const double x = li + carry;
                    long long r = llround(x);
                    if (r < 1) r = 1;
                    carry = x - (double)r;
                    if (lane == i) myr = (int)r;
                }
            }
            if (valid) qlen[j] = myr;
            long long t = myr;
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
            total += t;
        }
        if (bad) {
            if (lane == 0) atomicMin(err, (unsigned long long)(s * 16 + UNKNOWN_SYMBOL));
            continue;
        }
        // ---- match_total_length (backward cascade, almost always 1 piece) ----
        __syncwarp();
        int ok = 1;
        if (lane == 0) {
            long long residual = in.source_lengths[s] - total;
            for (int64_t j = b; j-- > a && residual != 0;) {
                long long adj = (long long)qlen[j] + residual;
                if (adj < 1) adj = 1;
                residual -= adj - qlen[j];
                qlen[j] = (int32_t)adj;
            }
            ok = (residual == 0 && b > a) ? 1 : 0;
            if (!ok) atomicMin(err, (unsigned long long)(s * 16 + INVALID_PIECE));
        }
        ok = __shfl_sync(FULL, ok, 0);
        if (!ok) continue;
        __syncwarp();
        // ---- pass 2: start values, positions, interpolation fill ----
        const bool drop_last = in.layout == 0 && s + 1 < in.n_seg;  // stitch_partitions
        int64_t pos = in.out_offsets[s];
        double v = in.anchors[s];
        if (lane == 0) out[pos] = v;
        for (int64_t base = a; base < b; base += 32) {
            const int64_t j = base + lane;
            const bool valid = j < b;
            const uint32_t lab = valid ? in.labels[j] : 0u;
            const int len = valid ? qlen[j] : 0;
            const double inc = valid ? __ldg(rinc + lab) : 0.0;
            const int cnt = (int)((b - base) < 32 ? (b - base) : 32);
            double myv = 0.0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {  // v += p.inc, sequential as the reference
                const double ii = __shfl_sync(FULL, inc, i);
                if (i < cnt) {
                    if (lane == i) myv = v;
                    v += ii;
                }
            }
            // inclusive scan of lengths (exact integers)
            long long incl = len;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const long long L = __shfl_sync(FULL, incl, 31);
            const bool last_group = base + 32 >= b;
            for (long long q0 = 1; q0 <= L; q0 += 32) {
                const long long q = q0 + lane;  // 1-based sample within the group
                // piece lo with excl_lo < q <= incl_lo: fixed 5-step search so
                // every lane executes the same full-mask shuffles
                int last_below = -1;  // last piece with incl < q
                for (int step = 16; step > 0; step >>= 1) {
                    const int t = last_below + step;
                    const long long cm = __shfl_sync(FULL, incl, t < 31 ? t : 31);
                    if (t < cnt && cm < q) last_below = t;
                }
                const int lo = last_below + 1 < 32 ? last_below + 1 : 31;
                const long long ci = __shfl_sync(FULL, incl, lo);
                const int li = __shfl_sync(FULL, len, lo);
                const double vi = __shfl_sync(FULL, myv, lo);
                const double ii = __shfl_sync(FULL, inc, lo);
                if (q <= L) {
                    const long long i = q - (ci - li);  // 1..len within piece lo
                    const bool skip = drop_last && last_group && q == L;
                    if (!skip) out[pos + q] = vi + ii * ((double)i / (double)li);
                }
            }
            pos += L;
        }
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
    {
        JB_PROF("inverse_warp", st);
        const int grid = (int)std::max<int64_t>(
            1, std::min<int64_t>((in.n_seg * 32 + INV_TB - 1) / INV_TB, (int64_t)kSMs * 16));
        k_inv_warp<<<grid, INV_TB, 0, st>>>(in, tab.p, tab.p + kk, qlen.p, d_out, err.p);
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
}

}  // namespace jb
