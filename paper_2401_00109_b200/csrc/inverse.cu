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

// Pass A -- one thread per segment runs the reference's sequential chains:
//   quantize_lengths (:63-74): r = llround(l + carry), clamp >= 1,
//     carry = (l + carry) - r  (r kept as an exact double: no int<->fp
//     conversions on the ~90-cycle critical path);
//   inverse_compress (:94-101): v += inc, and the running output position.
// Only the rounded lengths (int32, 16-byte vector stores on the aligned
// body) and, every GROUP pieces, checkpoints (v, position) leave the
// thread, so the per-thread streams cost ~5 B/piece. Then the backward
// fix-up (match_total_length :81-93) and a re-checkpoint of the tail.
constexpr int GROUP = 32;

struct ChainOut {
    int32_t* qlen;      // N
    double* vstart;     // N: start value of every piece
    double* ck_v;       // one per group (unused)
    int64_t* ck_pos;    // one per group
    int64_t* grp_off;   // n_seg + 1: first group of each segment
    int32_t* grp_seg;   // segment of every group
};

// inverse_digitize_series (:41-44): the first segment holding a label >= k
__global__ void k_inv_validate(InverseIn in, const int32_t* __restrict__ grp_seg,
                               unsigned long long* __restrict__ err) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < in.N;
         j += (int64_t)gridDim.x * blockDim.x)
        if ((uint64_t)in.labels[j] >= in.k) {
            // segment of piece j: binary search of the piece offsets
            int64_t lo = 0, hi = in.n_seg;
            while (hi - lo > 1) {
                const int64_t m = (lo + hi) >> 1;
                if (in.seg_offsets[m] <= j) lo = m;
                else hi = m;
            }
            atomicMin(err, (unsigned long long)(lo * 16 + UNKNOWN_SYMBOL));
        }
}

__global__ void k_group_segments(const int64_t* __restrict__ grp_off, int64_t n_seg,
                                 int32_t* __restrict__ grp_seg) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    for (int64_t g = grp_off[s]; g < grp_off[s + 1]; ++g) grp_seg[g] = (int32_t)s;
}

__device__ __forceinline__ void chain_step(double l, double& carry, int32_t& q) {
    const double x = l + carry;
    double r = llround_d(x);
    if (r < 1.0) r = 1.0;
    carry = x - r;
    q = (int32_t)r;
}

__global__ void __launch_bounds__(32) k_inv_chain(InverseIn in, const double* __restrict__ rlen,
                                                  const double* __restrict__ rinc, ChainOut co,
                                                  double* __restrict__ out,
                                                  unsigned long long* __restrict__ err) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= in.n_seg) return;
    const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
    // (labels were validated by k_inv_validate)
    const int64_t g0 = co.grp_off[s];
    double carry = 0.0, v = in.anchors[s];
    int64_t pos = in.out_offsets[s], total = 0;
    out[pos] = v;
    auto step = [&](int64_t j, uint32_t lab, double& vs) -> int32_t {
        if (((j - a) & (GROUP - 1)) == 0) co.ck_pos[g0 + ((j - a) >> 5)] = pos;
        int32_t q;
        chain_step(__ldg(rlen + lab), carry, q);
        vs = v;
        v += __ldg(rinc + lab);
        pos += q;
        total += q;
        return q;
    };
    int64_t j = a;
    double vs0, vs1, vs2, vs3;
    for (; j < b && (j & 3); ++j) {
        co.qlen[j] = step(j, in.labels[j], vs0);
        co.vstart[j] = vs0;
    }
    for (; j + 4 <= b; j += 4) {
        const uint4 L = *reinterpret_cast<const uint4*>(in.labels + j);
        int4 Q;
        Q.x = step(j, L.x, vs0);
        Q.y = step(j + 1, L.y, vs1);
        Q.z = step(j + 2, L.z, vs2);
        Q.w = step(j + 3, L.w, vs3);
        *reinterpret_cast<int4*>(co.qlen + j) = Q;
        *reinterpret_cast<double2*>(co.vstart + j) = make_double2(vs0, vs1);
        *reinterpret_cast<double2*>(co.vstart + j + 2) = make_double2(vs2, vs3);
    }
    for (; j < b; ++j) {
        co.qlen[j] = step(j, in.labels[j], vs0);
        co.vstart[j] = vs0;
    }
    // match_total_length: backward cascade
    long long residual = in.source_lengths[s] - total;
    int64_t first_mod = b;
    for (int64_t t = b; t-- > a && residual != 0;) {
        long long adj = (long long)co.qlen[t] + residual;
        if (adj < 1) adj = 1;
        residual -= adj - co.qlen[t];
        co.qlen[t] = (int32_t)adj;
        first_mod = t;
    }
    if (residual != 0 || b == a) {
        atomicMin(err, (unsigned long long)(s * 16 + INVALID_PIECE));
        return;
    }
    if (first_mod < b) {  // positions of the groups after the modified piece
        const int64_t gm = (first_mod - a) >> 5;
        int64_t p = co.ck_pos[g0 + gm];
        for (int64_t t = a + gm * GROUP; t < b; ++t) {
            if (((t - a) & (GROUP - 1)) == 0) co.ck_pos[g0 + ((t - a) >> 5)] = p;
            p += co.qlen[t];
        }
    }
}

// Pass B -- one warp per group of GROUP pieces: v within the group replayed
// sequentially from the checkpoint (shuffled, same rounding), positions by
// an exact integer scan, then the group's samples v + inc * (i / len)
// (inverse_compress :97-99) written contiguously into the output; a
// non-final part of a univariate-partitioned fit drops its last sample
// (stitch_partitions :198-213).
constexpr int DIV_MAX = 31;  // exact i/len table for len <= DIV_MAX (7.9 KB smem)

__global__ void __launch_bounds__(256) k_inv_fill(InverseIn in, const double* __restrict__ rinc,
                                                  ChainOut co, int64_t n_groups,
                                                  double* __restrict__ out) {
    __shared__ double div_tab[(DIV_MAX + 1) * (DIV_MAX + 1)];
    for (int t = threadIdx.x; t < (DIV_MAX + 1) * (DIV_MAX + 1); t += blockDim.x) {
        const int l = t / (DIV_MAX + 1), i = t % (DIV_MAX + 1);
        div_tab[t] = l > 0 ? (double)i / (double)l : 0.0;  // the same IEEE division
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < n_groups;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t s = co.grp_seg[g];
        const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
        const int64_t base = a + (g - co.grp_off[s]) * GROUP;
        const int cnt = (int)((b - base) < GROUP ? (b - base) : GROUP);
        const int64_t j = base + lane;
        const bool valid = lane < cnt;
        const int len = valid ? co.qlen[j] : 0;
        const double inc = valid ? __ldg(rinc + in.labels[j]) : 0.0;
        const double myv = valid ? co.vstart[j] : 0.0;
        long long incl = len;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const long long L = __shfl_sync(FULL, incl, 31);
        const int64_t pos = co.ck_pos[g];
        const bool drop_last = in.layout == 0 && (s + 1 < in.n_seg || in.drop_local_last) &&
                               base + GROUP >= b;
        for (long long q0 = 1; q0 <= L; q0 += 32) {
            const long long q = q0 + lane;  // 1-based sample within the group
            int last_below = -1;  // last piece with incl < q (fixed 5 steps)
            for (int st = 16; st > 0; st >>= 1) {
                const int t = last_below + st;
                const long long cm = __shfl_sync(FULL, incl, t < 31 ? t : 31);
                if (t < cnt && cm < q) last_below = t;
            }
            const int pc = last_below + 1 < 32 ? last_below + 1 : 31;
            const long long ci = __shfl_sync(FULL, incl, pc);
            const int li = __shfl_sync(FULL, len, pc);
            const double vi = __shfl_sync(FULL, myv, pc);
            const double ii = __shfl_sync(FULL, inc, pc);
            if (q <= L && !(drop_last && q == L)) {
                const long long i = q - (ci - li);  // 1..len within the piece
                // (double)i / l, IEEE-rounded; exact table for short pieces
                const double frac = li <= DIV_MAX ? div_tab[li * (DIV_MAX + 1) + (int)i]
                                                  : (double)i / (double)li;
                out[pos + q] = vi + ii * frac;
            }
        }
    }
}

}  // namespace

void inverse_transform_device(const InverseIn& in, double* d_out, cudaStream_t st) {
    if (in.layout == 0 && in.n_seg == 0)
        throw Error(INVALID_INPUT, "stitch_partitions: no segments");
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
    // group layout (host: segment piece counts are needed anyway for the offsets)
    std::vector<int64_t> h_off(in.n_seg + 1), h_goff(in.n_seg + 1);
    JB_CUDA(cudaMemcpyAsync(h_off.data(), in.seg_offsets, sizeof(int64_t) * (in.n_seg + 1),
                            cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    h_goff[0] = 0;
    for (int64_t s = 0; s < in.n_seg; ++s)
        h_goff[s + 1] = h_goff[s] + (h_off[s + 1] - h_off[s] + GROUP - 1) / GROUP;
    const int64_t n_groups = h_goff[in.n_seg];
    DArr<int64_t> goff(in.n_seg + 1, st);
    goff.upload(h_goff.data(), in.n_seg + 1);
    DArr<int32_t> qlen(std::max<int64_t>(in.N, 1) + 4, st);
    DArr<double> ck_v(1, st);
    DArr<int64_t> ck_pos(std::max<int64_t>(n_groups, 1), st);
    DArr<int32_t> gseg(std::max<int64_t>(n_groups, 1), st);
    DArr<double> vstart(std::max<int64_t>(in.N, 1) + 4, st);
    ChainOut co{qlen.p, vstart.p, ck_v.p, ck_pos.p, goff.p, gseg.p};
    k_group_segments<<<(int)((in.n_seg + 127) / 128), 128, 0, st>>>(goff.p, in.n_seg, gseg.p);
    JB_LAUNCH_CHECK();
    if (in.N > 0) {
        k_inv_validate<<<(int)std::max<int64_t>(1, std::min<int64_t>((in.N + 255) / 256, kSMs * 8)),
                         256, 0, st>>>(in, gseg.p, err.p);
        JB_LAUNCH_CHECK();
        unsigned long long e0;
        err.download(&e0, 1);
        JB_CUDA(cudaStreamSynchronize(st));
        if (e0 != ~0ULL)
            throw Error(UNKNOWN_SYMBOL, "label not in codebook of size " + std::to_string(in.k) +
                                            " (segment " + std::to_string(e0 / 16) + ")");
    }
    {
        JB_PROF("inverse_chain", st);
        k_inv_chain<<<(int)((in.n_seg + 31) / 32), 32, 0, st>>>(in, tab.p, tab.p + kk, co, d_out,
                                                                 err.p);
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
    if (n_groups > 0) {
        JB_PROF("inverse_fill", st);
        const int grid = (int)std::max<int64_t>(
            1, std::min<int64_t>((n_groups * 32 + 255) / 256, (int64_t)kSMs * 16));
        k_inv_fill<<<grid, 256, 0, st>>>(in, tab.p + kk, co, n_groups, d_out);
        JB_LAUNCH_CHECK();
    }
}

}  // namespace jb
