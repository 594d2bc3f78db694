// seqsum.cu — exact emulation of the reference's left-to-right fp64
// accumulation of NON-NEGATIVE terms, in parallel.
//
// The reference sums several non-negative quantities with a plain loop,
// `s += w` from s = 0 in index order:
//   * var_len of scale_pieces, w = (len - mean_len)^2   digitization.hpp:39-45
//   * the per-group sum of x = scl*len/sigma_len        digitization.hpp:224-231
// Both feed discrete decisions of the inverse (rlen = c_x*sigma_len/scl,
// inverse.hpp:46, then llround with carry, :63-74), so the device must produce
// the SAME double, not a more accurate one.
//
// Method. For s in the binade [2^e, 2^(e+1)) the grid is u_e = 2^(e-52), and
// as long as the result stays in that binade, fl(s + w) = s + u_e * inc(w)
// where inc(w) = w / u_e rounded to nearest; a tie (w / u_e = a + 1/2) rounds
// to the even significand, i.e. depends on the parity of M = s / u_e. Each term
// is therefore the map M -> M + (M even ? i_even : i_odd), and such maps
// compose associatively as pairs (i_even, i_odd). The sum is cut into blocks
// of kB terms; a block whose accumulator provably stays in one binade e
// (predicted from an approximate prefix, then VERIFIED while resolving) is
// summarised by its composed pair, blocks of 32 and 1024 into uniform parent
// pairs. One warp per segment then walks the blocks from the exact start
// value: a uniform node whose binade matches and whose result stays below
// 2^(e+1) is applied in O(1) -- exactly, by the argument above, since the
// accumulator is monotone -- and everything else (the first terms, binade
// crossings, mispredictions) is summed 32 terms at a time, falling back to
// the hardware fp64 add (the reference's own operation) term by term where a
// chunk crosses a binade or holds a tie. The prediction only decides speed:
// every O(1) step is checked, so the result is the sequential sum for any
// input (subnormal accumulators and zero included).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "jb_device.hpp"

namespace jb {

namespace {

constexpr int kB = 2048;       // terms per block (64 per lane)
constexpr int kNone = -100000; // "no uniform binade"

struct Pair {
    unsigned long long e, o;  // increments (units of u) for even / odd entry significand
};

__device__ __forceinline__ Pair compose(Pair f, Pair g) {
    Pair r;
    r.e = f.e + ((f.e & 1ULL) ? g.o : g.e);
    r.o = f.o + (((1ULL + f.o) & 1ULL) ? g.o : g.e);
    return r;
}

__device__ __forceinline__ double term_of_len(const SeqTerms& t, int32_t len) {
    const double l = (double)len;
    if (t.kind == SeqTerms::VAR_LEN) {
        const double dl = l - t.a;  // digitization.hpp:41,43
        return dl * dl;
    }
    return t.a * l / t.b;  // ScalingParams::apply core.hpp:131 (x)
}

__device__ __forceinline__ double term_at(const SeqTerms& t, int64_t i) {
    if (t.kind == SeqTerms::DIRECT) return t.w[i];
    if (t.kind == SeqTerms::SQDIFF) {
        const double d = t.w[i] - t.w2[i];  // metrics.hpp:25-26
        return d * d;
    }
    const double l = (double)t.len[i];
    if (t.kind == SeqTerms::VAR_LEN) {
        const double dl = l - t.a;  // digitization.hpp:41,43
        return dl * dl;
    }
    return t.a * l / t.b;  // ScalingParams::apply core.hpp:131 (x)
}

// w / 2^(e-52): the integer part a and the class of the remainder
// (0: below half, 1: above half, 2: exactly half). w >= 0 finite.
// Saturates at 2^57 (callers then fail the < 2^53 check; 32 saturated
// lanes still sum without wrapping).
__device__ __forceinline__ unsigned long long grid_units(double w, int e, int& cls) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(w);
    const int bexp = (int)((b >> 52) & 0x7FF);
    unsigned long long m = b & 0x000FFFFFFFFFFFFFULL;
    int ew;  // w = m * 2^(ew - 52)
    if (bexp == 0) {
        ew = -1022;
    } else {
        m |= 0x0010000000000000ULL;
        ew = bexp - 1023;
    }
    cls = 0;
    if (m == 0) return 0;
    const int up = ew - e;  // w / u_e = m * 2^up
    if (up >= 0) return up >= 5 ? (1ULL << 57) : (m << up);
    const int sh = -up;
    if (sh >= 55) return 0;  // < 1/2
    const unsigned long long a = sh >= 64 ? 0 : (m >> sh);
    const unsigned long long rem = m & ((1ULL << sh) - 1ULL);
    const unsigned long long half = 1ULL << (sh - 1);
    cls = rem > half ? 1 : (rem == half ? 2 : 0);
    return a;
}

__device__ __forceinline__ Pair term_pair(double w, int e) {
    int cls;
    const unsigned long long a = grid_units(w, e, cls);
    if (cls == 2) return Pair{a + (a & 1ULL), a + 1ULL - (a & 1ULL)};
    return Pair{a + (unsigned long long)cls, a + (unsigned long long)cls};
}

// binade exponent of a positive normal double, kNone otherwise
__device__ __forceinline__ int binade(double s) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(s);
    const int bexp = (int)((b >> 52) & 0x7FF);
    if ((b >> 63) || bexp == 0 || bexp == 0x7FF) return kNone;
    return bexp - 1023;
}

// s (binade e) advanced by the pair p: true and s updated iff the result stays
// in the binade (then it is exactly the sequential result)
__device__ __forceinline__ bool apply_pair(double& s, int e, Pair p) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(s);
    const unsigned long long M = (b & 0x000FFFFFFFFFFFFFULL) | 0x0010000000000000ULL;
    const unsigned long long inc = (M & 1ULL) ? p.o : p.e;
    if (inc >= (1ULL << 53)) return false;
    const unsigned long long Mn = M + inc;
    if (Mn >= (1ULL << 53)) return false;
    s = __longlong_as_double((long long)(((unsigned long long)(e + 1023) << 52) |
                                         (Mn & 0x000FFFFFFFFFFFFFULL)));
    return true;
}

struct SegDesc {
    const int64_t* blk;   // n_seg + 1: first block of each segment
    const int64_t* off;   // n_seg + 1: first term of each segment
    int64_t n_seg;
};

__device__ __forceinline__ int64_t seg_of_block(const SegDesc& sd, int64_t b) {
    int64_t lo = 0, hi = sd.n_seg;  // largest g with blk[g] <= b
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (sd.blk[mid] <= b) lo = mid;
        else hi = mid;
    }
    return lo;
}

// pass 1: approximate block sums (prediction only)
__global__ void k_ss_bsum(SeqTerms t, SegDesc sd, int64_t nblk, double* __restrict__ bsum,
                          int* __restrict__ bseg) {
    const int lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= nblk) return;
    const int64_t g = seg_of_block(sd, b);
    const int64_t i0 = sd.off[g] + (b - sd.blk[g]) * kB;
    const int64_t i1 = min(i0 + kB, sd.off[g + 1]);
    double s = 0.0;
    for (int64_t i = i0 + lane; i < i1; i += 32) s += term_at(t, i);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        bsum[b] = s;
        bseg[b] = (int)g;
    }
}

// pass 2: predicted binade of every block and its composed pair
__global__ void k_ss_pairs(SeqTerms t, SegDesc sd, int64_t nblk, const double* __restrict__ bsum,
                           const double* __restrict__ gpre, const int* __restrict__ bseg,
                           const double* __restrict__ s_in, const int64_t* __restrict__ gbase,
                           int* __restrict__ be, unsigned long long* __restrict__ pe,
                           unsigned long long* __restrict__ po) {
    const int lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= nblk) return;
    const int g = bseg[b];
    const int64_t b0 = sd.blk[g];
    const double P0 = s_in[g] + (gpre[b] - gpre[b0]);
    const double P1 = P0 + bsum[b];
    // |sequential - exact| <= (terms so far) * 2^-52 * s, plus slack for the
    // approximate (double) prefix; a misprediction only costs the fallback
    const int64_t i0 = sd.off[g] + (b - b0) * kB;
    const int64_t i1 = min(i0 + kB, sd.off[g + 1]);
    const double d = (double)(gbase[g] + (i1 - sd.off[g]) + (int64_t)(b - b0 + 2) * 64) * 0x1p-52 +
                     0x1p-40;
    const int e0 = binade(P0 * (1.0 - d)), e1 = binade(P1 * (1.0 + d));
    int e = (e0 != kNone && e0 == e1) ? e0 : kNone;
    Pair acc{0, 0};
    if (e != kNone) {
        unsigned long long sum = 0;
        bool tie = false, big = false;
        for (int64_t i = i0 + lane; i < i1; i += 32) {
            int cls;
            const unsigned long long a = grid_units(term_at(t, i), e, cls);
            big |= a >= (1ULL << 53);  // one term alone leaves the binade
            sum += a + (cls == 1 ? 1ULL : 0ULL);
            tie |= cls == 2;
        }
        big |= sum >= (1ULL << 54);  // (64 terms per lane: no wrap before this test)
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (__any_sync(0xffffffffu, big)) {
            e = kNone;
        } else if (__any_sync(0xffffffffu, tie)) {
            // ordered composition: chunks of 32 by a shuffle scan, in order
            Pair run{0, 0};
            for (int64_t c = i0; c < i1; c += 32) {
                const int64_t i = c + lane;
                Pair p = i < i1 ? term_pair(term_at(t, i), e) : Pair{0, 0};
                for (int o = 1; o < 32; o <<= 1) {
                    Pair q;
                    q.e = __shfl_up_sync(0xffffffffu, p.e, o);
                    q.o = __shfl_up_sync(0xffffffffu, p.o, o);
                    if (lane >= o) p = compose(q, p);
                }
                Pair tot;
                tot.e = __shfl_sync(0xffffffffu, p.e, 31);
                tot.o = __shfl_sync(0xffffffffu, p.o, 31);
                run = compose(run, tot);
            }
            acc = run;
        } else {
            acc = Pair{sum, sum};
        }
        if (acc.e >= (1ULL << 53) || acc.o >= (1ULL << 53)) e = kNone;
    }
    if (lane == 0) {
        be[b] = e;
        pe[b] = acc.e;
        po[b] = acc.o;
    }
}

// parents of 32 consecutive nodes: uniform iff all 32 children are uniform in
// the same binade and segment
__global__ void k_ss_level(int64_t nchild, int64_t seg_div, const int* __restrict__ ce,
                           const int* __restrict__ cseg,
                           const unsigned long long* __restrict__ cpe,
                           const unsigned long long* __restrict__ cpo, int64_t npar,
                           int* __restrict__ e_out, int* __restrict__ seg_out,
                           unsigned long long* __restrict__ pe_out,
                           unsigned long long* __restrict__ po_out) {
    const int lane = threadIdx.x & 31;
    const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (p >= npar) return;
    const int64_t c = p * 32 + lane;
    const bool have = c < nchild;
    const int e = have ? ce[c] : kNone;
    const int sg = have ? (cseg ? cseg[c] : (int)(c / seg_div)) : -1;
    Pair q = have ? Pair{cpe[c], cpo[c]} : Pair{0, 0};
    const int e0 = __shfl_sync(0xffffffffu, e, 0);
    const int s0 = __shfl_sync(0xffffffffu, sg, 0);
    const bool uni = __all_sync(0xffffffffu, have && e == e0 && sg == s0 && e != kNone);
    for (int o = 1; o < 32; o <<= 1) {
        Pair r;
        r.e = __shfl_up_sync(0xffffffffu, q.e, o);
        r.o = __shfl_up_sync(0xffffffffu, q.o, o);
        if (lane >= o) q = compose(r, q);
    }
    if (lane == 31) {
        const bool fits = q.e < (1ULL << 53) && q.o < (1ULL << 53);
        e_out[p] = uni && fits ? e0 : kNone;
        seg_out[p] = s0;
        pe_out[p] = q.e;
        po_out[p] = q.o;
    }
}

struct Level {
    const int* e;
    const int* seg;
    const unsigned long long* pe;
    const unsigned long long* po;
};

// the chunk fallback: terms [i0, i1) from s, 32 at a time (warp-uniform s)
__device__ void ss_terms(const SeqTerms& t, int64_t i0, int64_t i1, double& s) {
    const int lane = threadIdx.x & 31;
    for (int64_t c = i0; c < i1; c += 32) {
        const int64_t i = c + lane;
        const int n = (int)(i1 - c < 32 ? i1 - c : 32);
        const double w = i < i1 ? term_at(t, i) : 0.0;
        const int e = binade(s);
        if (e != kNone) {
            int cls;
            unsigned long long a = grid_units(w, e, cls);
            a += cls == 1 ? 1ULL : 0ULL;
            const bool tie = cls == 2;
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (!__any_sync(0xffffffffu, tie) && apply_pair(s, e, Pair{a, a})) continue;
        }
        for (int j = 0; j < n; ++j) s = s + __shfl_sync(0xffffffffu, w, j);  // the reference's add
    }
}

// one warp per segment: s_out[g] = sequential sum of the segment from s_in[g]
__global__ void k_ss_resolve(SeqTerms t, SegDesc sd, int64_t nblk, Level L1, Level L2, int64_t n2,
                             Level L3, int64_t n3, const double* __restrict__ s_in,
                             double* __restrict__ s_out) {
    const int lane = threadIdx.x & 31;
    const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= sd.n_seg) return;
    double s = s_in[g];
    const int64_t bend = sd.blk[g + 1];
    int64_t b = sd.blk[g];
    while (b < bend) {
        const int e = binade(s);
        if (e != kNone) {
            if ((b & 1023) == 0 && b + 1024 <= bend && (b >> 10) < n3) {
                const int64_t p = b >> 10;
                if (L3.e[p] == e && L3.seg[p] == (int)g && apply_pair(s, e, Pair{L3.pe[p], L3.po[p]})) {
                    b += 1024;
                    continue;
                }
            }
            if ((b & 31) == 0 && b + 32 <= bend && (b >> 5) < n2) {
                const int64_t p = b >> 5;
                if (L2.e[p] == e && L2.seg[p] == (int)g && apply_pair(s, e, Pair{L2.pe[p], L2.po[p]})) {
                    b += 32;
                    continue;
                }
            }
            if (L1.e[b] == e && apply_pair(s, e, Pair{L1.pe[b], L1.po[b]})) {
                ++b;
                continue;
            }
        }
        const int64_t i0 = sd.off[g] + (b - sd.blk[g]) * kB;
        const int64_t i1 = min(i0 + kB, sd.off[g + 1]);
        ss_terms(t, i0, i1, s);
        ++b;
    }
    if (lane == 0) s_out[g] = s;
}

int blocks_for_warps(int64_t warps) { return (int)std::max<int64_t>(1, (warps + 7) / 8); }

}  // namespace

void SeqSum::setup(const SeqTerms& t, const std::vector<int64_t>& seg_off, cudaStream_t st) {
    terms = t;
    stream = st;
    n_seg = (int64_t)seg_off.size() - 1;
    h_off = seg_off;
    h_blk.assign(n_seg + 1, 0);
    for (int64_t g = 0; g < n_seg; ++g)
        h_blk[g + 1] = h_blk[g] + (seg_off[g + 1] - seg_off[g] + kB - 1) / kB;
    nblk = h_blk[n_seg];
    d_blk.alloc(n_seg + 1, st);
    d_off.alloc(n_seg + 1, st);
    d_blk.upload(h_blk.data(), n_seg + 1);
    d_off.upload(h_off.data(), n_seg + 1);
    const size_t nb = (size_t)std::max<int64_t>(nblk, 1);
    bsum.alloc(nb, st);
    gpre.alloc(nb, st);
    bseg.alloc(nb, st);
    local_total.assign(n_seg, 0.0);
    if (nblk == 0) return;
    const SegDesc sd{d_blk.p, d_off.p, n_seg};
    {
        JB_PROF("seqsum_blocks", st);
        k_ss_bsum<<<blocks_for_warps(nblk), 256, 0, st>>>(t, sd, nblk, bsum.p, bseg.p);
    }
    JB_LAUNCH_CHECK();
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, bsum.p, gpre.p, nblk, st);
    DArr<uint8_t> tmp(std::max<size_t>(tb, 1), st);
    cub::DeviceScan::ExclusiveSum(tmp.p, tb, bsum.p, gpre.p, nblk, st);
    JB_LAUNCH_CHECK();
    // per-segment totals (approximate): for the start-value predictions of
    // the following ranks / for diagnostics
    std::vector<double> g(nblk), bs(nblk);
    gpre.download(g.data(), nblk);
    bsum.download(bs.data(), nblk);
    JB_CUDA(cudaStreamSynchronize(st));
    for (int64_t s = 0; s < n_seg; ++s) {
        if (h_blk[s + 1] == h_blk[s]) continue;
        local_total[s] = g[h_blk[s + 1] - 1] + bs[h_blk[s + 1] - 1] - g[h_blk[s]];
    }
}

void SeqSum::predict(const std::vector<double>& s_in_approx, const std::vector<int64_t>& terms_before) {
    cudaStream_t st = stream;
    const size_t nb = (size_t)std::max<int64_t>(nblk, 1);
    be.alloc(nb, st);
    pe.alloc(nb, st);
    po.alloc(nb, st);
    n2 = (nblk + 31) / 32;
    n3 = (n2 + 31) / 32;
    e2.alloc(std::max<int64_t>(n2, 1), st);
    s2.alloc(std::max<int64_t>(n2, 1), st);
    pe2.alloc(std::max<int64_t>(n2, 1), st);
    po2.alloc(std::max<int64_t>(n2, 1), st);
    e3.alloc(std::max<int64_t>(n3, 1), st);
    s3.alloc(std::max<int64_t>(n3, 1), st);
    pe3.alloc(std::max<int64_t>(n3, 1), st);
    po3.alloc(std::max<int64_t>(n3, 1), st);
    if (nblk == 0) return;
    DArr<double> sin_d(n_seg, st);
    sin_d.upload(s_in_approx.data(), n_seg);
    DArr<int64_t> gb(n_seg, st);
    gb.upload(terms_before.data(), n_seg);
    const SegDesc sd{d_blk.p, d_off.p, n_seg};
    {
        JB_PROF("seqsum_pairs", st);
        k_ss_pairs<<<blocks_for_warps(nblk), 256, 0, st>>>(terms, sd, nblk, bsum.p, gpre.p, bseg.p,
                                                           sin_d.p, gb.p, be.p, pe.p, po.p);
        JB_LAUNCH_CHECK();
        k_ss_level<<<blocks_for_warps(n2), 256, 0, st>>>(nblk, 1, be.p, bseg.p, pe.p, po.p, n2, e2.p,
                                                         s2.p, pe2.p, po2.p);
        JB_LAUNCH_CHECK();
        k_ss_level<<<blocks_for_warps(n3), 256, 0, st>>>(n2, 1, e2.p, s2.p, pe2.p, po2.p, n3, e3.p,
                                                         s3.p, pe3.p, po3.p);
        JB_LAUNCH_CHECK();
    }
    JB_CUDA(cudaStreamSynchronize(st));  // sin_d / gb are released on return
}

std::vector<double> SeqSum::resolve(const std::vector<double>& s_in) {
    cudaStream_t st = stream;
    std::vector<double> out(s_in);
    if (n_seg == 0) return out;
    DArr<double> din(n_seg, st), dout(n_seg, st);
    din.upload(s_in.data(), n_seg);
    const SegDesc sd{d_blk.p, d_off.p, n_seg};
    const Level L1{be.p, bseg.p, pe.p, po.p}, L2{e2.p, s2.p, pe2.p, po2.p},
        L3{e3.p, s3.p, pe3.p, po3.p};
    {
        JB_PROF("seqsum_resolve", st);
        k_ss_resolve<<<blocks_for_warps(n_seg), 256, 0, st>>>(terms, sd, nblk, L1, L2, n2, L3, n3,
                                                              din.p, dout.p);
    }
    JB_LAUNCH_CHECK();
    dout.download(out.data(), n_seg);
    JB_CUDA(cudaStreamSynchronize(st));
    return out;
}

std::vector<double> seq_sum_nonneg(const SeqTerms& t, const std::vector<int64_t>& seg_off,
                                   cudaStream_t st, const Comm* cm) {
    const int64_t n_seg = (int64_t)seg_off.size() - 1;
    SeqSum ss;
    ss.setup(t, seg_off, st);
    std::vector<double> s_in(n_seg, 0.0);
    std::vector<int64_t> before(n_seg, 0);
    if (!cm || !cm->dist()) {
        ss.predict(s_in, before);
        return ss.resolve(s_in);
    }
    // ranks hold consecutive pieces of every segment: rank r's terms follow
    // ranks 0..r-1's. Predictions from the gathered approximate totals, then
    // the exact start values are handed down the ranks one at a time.
    std::vector<double> tot = cm->gather(ss.local_total);
    std::vector<int64_t> cnt(n_seg);
    for (int64_t g = 0; g < n_seg; ++g) cnt[g] = seg_off[g + 1] - seg_off[g];
    std::vector<int64_t> cnts = cm->gather(cnt);
    std::vector<double> approx(n_seg, 0.0);
    for (int r = 0; r < cm->rank; ++r)
        for (int64_t g = 0; g < n_seg; ++g) {
            approx[g] += tot[(size_t)r * n_seg + g];
            before[g] += cnts[(size_t)r * n_seg + g];
        }
    ss.predict(approx, before);
    std::vector<double> cur(n_seg, 0.0);
    for (int r = 0; r < cm->world; ++r) {
        std::vector<double> mine = r == cm->rank ? ss.resolve(cur) : cur;
        std::vector<double> all = cm->gather(mine);
        std::copy(all.begin() + (size_t)r * n_seg, all.begin() + (size_t)(r + 1) * n_seg, cur.begin());
    }
    return cur;
}


// ---------------------------------------------------------------------------
// Range-histogram form (no pass over the data of its own): the producer
// kernel (scale's k_var_blocks for var_len, k_assign_stats for the group
// sums) counts, for every range of R consecutive pieces, the pieces of each
// group by length l <= RH and lists the longer ones. A record (r, g) -- the
// pieces of group g in range r, in index order -- then gets its binade
// prediction and its pair from the counts alone: sum_l h[l] * inc(T(l), e),
// order-free unless some present length is a tie at e (then the record is
// left to the fallback). Records are range-major (r * k + g, the layout the
// producer writes, so every pass reads it coalesced across groups); level
// nodes group 32 consecutive ranges of one group. One CTA per group walks its
// records from the exact start value; the fallback re-reads the range and
// keeps the members of g in order.

namespace {

// range-major (nr x k) -> group-major (k x nr), 32 x 32 tiles through shared memory
__global__ void k_rs_transpose(const double* __restrict__ in, int64_t nr, int k,
                               double* __restrict__ out) {
    __shared__ double tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32, g0 = (int64_t)blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t r = r0 + j, g = g0 + threadIdx.x;
        if (r < nr && g < k) tile[j][threadIdx.x] = in[r * k + g];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int64_t g = g0 + j, r = r0 + threadIdx.x;
        if (r < nr && g < k) out[g * nr + r] = tile[threadIdx.x][j];
    }
}

// K3: every record's predicted binade and pair (thread per record)
__global__ void k_rs_pairs(SeqTerms t, const uint16_t* __restrict__ hist,
                           const double* __restrict__ bsum, int64_t nr, int k, int RH,
                           const double* __restrict__ gpre, const double* __restrict__ s_in,
                           double rel, int* __restrict__ be, unsigned long long* __restrict__ pe,
                           unsigned long long* __restrict__ po) {
    __shared__ double T[64];
    if (threadIdx.x < RH) T[threadIdx.x] = term_of_len(t, threadIdx.x + 1);
    __syncthreads();
    const int64_t nrec = nr * k;
    for (int64_t rec = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; rec < nrec;
         rec += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = rec / k, g = rec - r * k;
        // gpre: exclusive prefix over ALL records in group-major order
        const double P0 = s_in[g] + (gpre[g * nr + r] - gpre[g * nr]);
        const double P1 = P0 + bsum[rec];
        const int e0 = binade(P0 * (1.0 - rel)), e1 = binade(P1 * (1.0 + rel));
        int e = (e0 != kNone && e0 == e1) ? e0 : kNone;
        unsigned long long A = 0;
        const uint16_t* h = hist + (r * RH) * k + g;
        for (int l = 0; l < RH && e != kNone; ++l) {
            const unsigned long long c = h[(int64_t)l * k];
            if (!c) continue;
            int cls;
            const unsigned long long a = grid_units(T[l], e, cls);
            const unsigned long long inc = a + (unsigned long long)cls;
            // tie, or the record leaves the binade (128-bit product: no wrap)
            const u128 add = (u128)c * (u128)inc;
            if (cls == 2 || add >= (u128)((1ULL << 53) - A)) e = kNone;
            else A += (unsigned long long)add;
        }
        be[rec] = e;
        pe[rec] = A;
        po[rec] = A;
    }
}

// the listed long pieces: their increments, atomically (order-free)
__global__ void k_rs_long(SeqTerms t, const uint32_t* __restrict__ idx,
                          const unsigned long long* __restrict__ count, int64_t R, int k,
                          const uint32_t* __restrict__ labels, int* __restrict__ be,
                          unsigned long long* __restrict__ pe, unsigned long long* __restrict__ po) {
    const int64_t n = (int64_t)*count;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx[j];
        const int64_t g = labels ? labels[i] : 0;
        const int64_t rec = (i / R) * k + g;
        const int e = be[rec];
        if (e == kNone) continue;
        int cls;
        const unsigned long long a = grid_units(term_of_len(t, t.len[i]), e, cls);
        if (cls == 2 || a >= (1ULL << 53)) {
            atomicExch(be + rec, kNone);
            continue;
        }
        const unsigned long long inc = a + (unsigned long long)cls;
        const unsigned long long old = atomicAdd(pe + rec, inc);
        atomicAdd(po + rec, inc);
        // past 2^53 the record leaves its binade: drop it (before any wrap)
        if (old + inc >= (1ULL << 53)) atomicExch(be + rec, kNone);
    }
}

// parent (j, g) of the 32 children (32 j .. 32 j + 31, g), range-major
__global__ void k_rs_level(int64_t nchild, int k, const int* __restrict__ ce,
                           const unsigned long long* __restrict__ cpe,
                           const unsigned long long* __restrict__ cpo, int64_t npar,
                           int* __restrict__ e_out, unsigned long long* __restrict__ pe_out,
                           unsigned long long* __restrict__ po_out) {
    const int lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (q >= npar * k) return;
    const int64_t j = q / k, g = q - j * k;
    const int64_t c = j * 32 + lane;
    const bool have = c < nchild;
    const int e = have ? ce[c * k + g] : kNone;
    Pair p = have ? Pair{cpe[c * k + g], cpo[c * k + g]} : Pair{0, 0};
    const int e0 = __shfl_sync(0xffffffffu, e, 0);
    const bool uni = __all_sync(0xffffffffu, have && e == e0 && e != kNone);
    for (int o = 1; o < 32; o <<= 1) {
        Pair r;
        r.e = __shfl_up_sync(0xffffffffu, p.e, o);
        r.o = __shfl_up_sync(0xffffffffu, p.o, o);
        if (lane >= o) p = compose(r, p);
    }
    if (lane == 31) {
        const bool fits = p.e < (1ULL << 53) && p.o < (1ULL << 53);
        e_out[q] = uni && fits ? e0 : kNone;
        pe_out[q] = p.e;
        po_out[q] = p.o;
    }
}

struct RLevel {
    const int* e;
    const unsigned long long* pe;
    const unsigned long long* po;
    int64_t n;  // nodes per group
};

// a window of 32 consecutive nodes of one group held by a warp's lanes: the
// walk pays one load per 32 steps instead of one dependent load per step
struct Window {
    int64_t base = -1;
    int e = 0;
    unsigned long long pe = 0, po = 0;
    __device__ __forceinline__ void get(const RLevel& L, int k, int64_t g, int64_t p, int& oe,
                                        Pair& pr) {
        const int lane = threadIdx.x & 31;
        if (base < 0 || p < base || p >= base + 32) {
            base = p;
            const int64_t q = p + lane;
            e = q < L.n ? L.e[q * k + g] : kNone;
            pe = q < L.n ? L.pe[q * k + g] : 0;
            po = q < L.n ? L.po[q * k + g] : 0;
        }
        const int src = (int)(p - base);
        oe = __shfl_sync(0xffffffffu, e, src);
        pr.e = __shfl_sync(0xffffffffu, pe, src);
        pr.o = __shfl_sync(0xffffffffu, po, src);
    }
};

__device__ void ss_chunks(const SeqTerms& t, const int32_t* lens, int cnt, double& s);

__device__ void ss_lens(const SeqTerms& t, const int32_t* lens, int cnt, double& s) {
    const int lane = threadIdx.x & 31;
    for (int c0 = 0; c0 < cnt; c0 += 1024) {
        // 1024 terms at once when none of them crosses a binade or ties:
        // lane-local sums, one warp reduction (one per 32 chunks)
        const int nb = cnt - c0 < 1024 ? cnt - c0 : 1024;
        const int e = binade(s);
        if (e != kNone && nb > 64) {
            unsigned long long a = 0;
            bool bad = false;
            for (int j = lane; j < nb; j += 32) {
                int cls;
                const unsigned long long q = grid_units(term_of_len(t, lens[c0 + j]), e, cls);
                bad |= cls == 2 || q >= (1ULL << 53);
                a += q + (cls == 1 ? 1ULL : 0ULL);
            }
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (!__any_sync(0xffffffffu, bad) && apply_pair(s, e, Pair{a, a})) continue;
        }
        ss_chunks(t, lens + c0, nb, s);
    }
}

__device__ void ss_chunks(const SeqTerms& t, const int32_t* lens, int cnt, double& s) {
    const int lane = threadIdx.x & 31;
    for (int c = 0; c < cnt; c += 32) {
        const int n = cnt - c < 32 ? cnt - c : 32;
        const double w = lane < n ? term_of_len(t, lens[c + lane]) : 0.0;
        const int e = binade(s);
        if (e != kNone) {
            int cls;
            unsigned long long a = grid_units(w, e, cls);
            a += cls == 1 ? 1ULL : 0ULL;
            const bool tie = cls == 2;
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (!__any_sync(0xffffffffu, tie) && apply_pair(s, e, Pair{a, a})) continue;
        }
        for (int j = 0; j < n; ++j) s = s + __shfl_sync(0xffffffffu, w, j);  // the reference's add
    }
}

constexpr int RS_TB = 256, RS_SUB = 1024;  // pieces per warp per fallback sub-range

// one CTA per group: walk its records; a record that cannot be applied in
// O(1) is summed from the range's pieces (members of g gathered in order)
__global__ void __launch_bounds__(RS_TB) k_rs_resolve(SeqTerms t, const uint32_t* __restrict__ labels,
                                                      int64_t n, int64_t R, int k, RLevel L1,
                                                      RLevel L2, RLevel L3,
                                                      const double* __restrict__ s_in,
                                                      double* __restrict__ s_out,
                                                      unsigned long long* __restrict__ diag) {
    // diag (optional): steps applied at level 3 / 2 / 1, fallbacks
    __shared__ int32_t s_len[RS_TB / 32][RS_SUB];
    __shared__ int s_cnt[RS_TB / 32];
    __shared__ double s_val;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t g = blockIdx.x;
    const int64_t nr = L1.n;
    double s = s_in[g];
    Window W1, W2, W3;
    int64_t r = 0;
    while (r < nr) {
        const int e = binade(s);
        if (e != kNone) {
            int ne;
            Pair pr;
            if ((r & 1023) == 0 && r + 1024 <= nr) {
                W3.get(L3, k, g, r >> 10, ne, pr);
                if (ne == e && apply_pair(s, e, pr)) {
                    r += 1024;
                    if (diag && threadIdx.x == 0) atomicAdd(diag + 0, 1ULL);
                    continue;
                }
            }
            if ((r & 31) == 0 && r + 32 <= nr) {
                W2.get(L2, k, g, r >> 5, ne, pr);
                if (ne == e && apply_pair(s, e, pr)) {
                    r += 32;
                    if (diag && threadIdx.x == 0) atomicAdd(diag + 1, 1ULL);
                    continue;
                }
            }
            W1.get(L1, k, g, r, ne, pr);
            if (ne == e && apply_pair(s, e, pr)) {
                ++r;
                if (diag && threadIdx.x == 0) atomicAdd(diag + 2, 1ULL);
                continue;
            }
        }
        if (diag && threadIdx.x == 0) atomicAdd(diag + 3, 1ULL);
        // fallback: the pieces of range r, the members of g in index order
        const int64_t i0 = r * R, i1 = min(i0 + R, n);
        for (int64_t sub = i0; sub < i1; sub += (int64_t)RS_SUB * (RS_TB / 32)) {
            const int64_t w0 = sub + (int64_t)w * RS_SUB;
            uint32_t lab[RS_SUB / 32];
            int32_t ln[RS_SUB / 32];
#pragma unroll
            for (int j = 0; j < RS_SUB / 32; ++j) {  // every load in flight at once
                const int64_t i = w0 + j * 32 + lane;
                lab[j] = i < i1 && labels ? labels[i] : 0u;
                ln[j] = i < i1 ? t.len[i] : 0;
            }
            int cnt = 0;
#pragma unroll
            for (int j = 0; j < RS_SUB / 32; ++j) {
                const int64_t i = w0 + j * 32 + lane;
                const bool in = i < i1 && lab[j] == (uint32_t)g;
                const unsigned m = __ballot_sync(0xffffffffu, in);
                if (in) s_len[w][cnt + __popc(m & ((1u << lane) - 1u))] = ln[j];
                cnt += __popc(m);
            }
            if (lane == 0) s_cnt[w] = cnt;
            __syncthreads();
            if (w == 0) {  // the regions in order; small ones chunk by chunk
                int tot = 0;
                for (int q = 0; q < RS_TB / 32; ++q) tot += s_cnt[q];
                for (int q = 0; q < RS_TB / 32; ++q)
                    if (s_cnt[q]) (tot > 256 ? ss_lens : ss_chunks)(t, s_len[q], s_cnt[q], s);
            }
            if (threadIdx.x == 0) s_val = s;
            __syncthreads();
            s = s_val;
            __syncthreads();
        }
        ++r;
    }
    if (threadIdx.x == 0) s_out[g] = s;
}

}  // namespace

std::vector<double> range_seq_sums(const RangeHist& h, const SeqTerms& t,
                                   const uint32_t* d_labels, cudaStream_t st, const Comm* cm) {
    const int k = h.k;
    const int64_t nr = h.nr, nrec = nr * (int64_t)k;
    std::vector<double> cur(k, 0.0);
    if (h.RH > 64) throw Error(INTERNAL, "range histogram wider than 64 lengths");
    const double* bsum = h.approx.p;  // the producer's per-record approximate sums
    DArr<double> gpre(std::max<int64_t>(nrec, 1), st);
    auto grid_for_n = [](int64_t m) {
        return (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, num_sms() * 16));
    };
    std::vector<double> local_total(k, 0.0);
    if (nrec > 0) {
        JB_PROF("seqsum_blocks", st);
        // per-group prefix: group-major copy, one scan over all records (each
        // group's base subtracted where it is read)
        DArr<double> gm(k > 1 ? nrec : 0, st);
        const double* src = bsum;
        if (k > 1) {
            k_rs_transpose<<<dim3((unsigned)((nr + 31) / 32), (unsigned)((k + 31) / 32)), dim3(32, 8),
                             0, st>>>(bsum, nr, k, gm.p);
            JB_LAUNCH_CHECK();
            src = gm.p;
        }
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, src, gpre.p, nrec, st);
        DArr<uint8_t> tmp(std::max<size_t>(tb, 1), st);
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, src, gpre.p, nrec, st);
        JB_LAUNCH_CHECK();
        if (cm && cm->dist()) {  // this rank's approximate group totals
            std::vector<double> pre = gpre.to_host(nrec);
            std::vector<double> last(k);
            for (int g = 0; g < k; ++g) {
                JB_CUDA(cudaMemcpyAsync(&last[g], src + (int64_t)g * nr + nr - 1, 8,
                                        cudaMemcpyDeviceToHost, st));
            }
            JB_CUDA(cudaStreamSynchronize(st));
            for (int g = 0; g < k; ++g)
                local_total[g] = pre[(int64_t)g * nr + nr - 1] + last[g] - pre[(int64_t)g * nr];
        }
    }
    std::vector<double> approx(k, 0.0);
    int64_t n_all = h.n;
    if (cm && cm->dist()) {  // predictions from the gathered approximate totals
        const std::vector<double> all = cm->gather(local_total);
        const std::vector<int64_t> ns = cm->gather(std::vector<int64_t>{h.n});
        n_all = 0;
        for (int r = 0; r < cm->world; ++r) {
            n_all += ns[r];
            if (r < cm->rank)
                for (int g = 0; g < k; ++g) approx[g] += all[(size_t)r * k + g];
        }
    }
    // |sequential - exact| <= (terms so far) * 2^-52 * s; plus the double prefix's slack
    const double rel = (double)(n_all + 64) * 0x1p-52 + 0x1p-40;
    const int64_t n2 = (nr + 31) / 32, n3 = (n2 + 31) / 32;
    auto mx1 = [](int64_t v) { return std::max<int64_t>(v, 1); };
    DArr<int> be(mx1(nrec), st), e2(mx1(n2 * k), st), e3(mx1(n3 * k), st);
    DArr<unsigned long long> pe(mx1(nrec), st), po(mx1(nrec), st), pe2(mx1(n2 * k), st),
        po2(mx1(n2 * k), st), pe3(mx1(n3 * k), st), po3(mx1(n3 * k), st);
    DArr<double> sin_d(k, st), sout_d(k, st);
    if (nrec > 0) {
        sin_d.upload(approx.data(), k);
        JB_PROF("seqsum_pairs", st);
        k_rs_pairs<<<grid_for_n(nrec), 256, 0, st>>>(t, h.hist.p, bsum, nr, k, h.RH, gpre.p,
                                                     sin_d.p, rel, be.p, pe.p, po.p);
        JB_LAUNCH_CHECK();
        if (h.long_idx.p)
            k_rs_long<<<num_sms() * 4, 256, 0, st>>>(t, h.long_idx.p, h.long_n.p, h.R, k, d_labels, be.p,
                                                pe.p, po.p);
        JB_LAUNCH_CHECK();
        k_rs_level<<<blocks_for_warps(n2 * k), 256, 0, st>>>(nr, k, be.p, pe.p, po.p, n2, e2.p,
                                                             pe2.p, po2.p);
        JB_LAUNCH_CHECK();
        k_rs_level<<<blocks_for_warps(n3 * k), 256, 0, st>>>(n2, k, e2.p, pe2.p, po2.p, n3, e3.p,
                                                             pe3.p, po3.p);
        JB_LAUNCH_CHECK();
    }
    const RLevel L1{be.p, pe.p, po.p, nr}, L2{e2.p, pe2.p, po2.p, n2}, L3{e3.p, pe3.p, po3.p, n3};
    auto resolve = [&](const std::vector<double>& sin) {
        std::vector<double> out(sin);
        if (nrec == 0) return out;
        sin_d.upload(sin.data(), k);
        static const bool stats = getenv("JB_SEQSUM_STATS") != nullptr;
        DArr<unsigned long long> diag(stats ? 4 : 0, st);
        if (stats) diag.zero();
        {
            JB_PROF(k == 1 ? "seqsum_resolve_one" : "seqsum_resolve_groups", st);
            k_rs_resolve<<<k, RS_TB, 0, st>>>(t, d_labels, h.n, h.R, k, L1, L2, L3, sin_d.p,
                                              sout_d.p, stats ? diag.p : nullptr);
        }
        JB_LAUNCH_CHECK();
        if (stats) {
            const auto d = diag.to_host(4);
            fprintf(stderr, "[jb] seqsum k=%d records=%lld R=%lld: L3 %llu L2 %llu L1 %llu fallbacks %llu\n",
                    k, (long long)nrec, (long long)h.R, d[0], d[1], d[2], d[3]);
        }
        sout_d.download(out.data(), k);
        JB_CUDA(cudaStreamSynchronize(st));
        return out;
    };
    if (!cm || !cm->dist()) return resolve(cur);
    for (int r = 0; r < cm->world; ++r) {  // exact start values handed down the ranks
        std::vector<double> mine = r == cm->rank ? resolve(cur) : cur;
        std::vector<double> all = cm->gather(mine);
        std::copy(all.begin() + (size_t)r * k, all.begin() + (size_t)(r + 1) * k, cur.begin());
    }
    return cur;
}

}  // namespace jb
