// digitize.cu — scaling (digitization.hpp:25-59), nearest-center assignment
// with group statistics (clustering.hpp:146-163, digitization.hpp:217-253),
// relabeling by cardinality rank (:255-291).
//
// Sums that the reference accumulates sequentially in fp64 are accumulated
// here as 128-bit fixed-point integers (jb_common.cuh): deterministic for any
// grid or GPU count, and within an ulp-scale of the sequential result.
#include <cub/cub.cuh>

#include <cmath>

#include "jb_device.hpp"
#include "jb_grid.cuh"
#include "jb_rowgrid.cuh"

namespace jb {

namespace {

__device__ __forceinline__ unsigned long long ord_bits(double x) {
    // order-preserving map of any double to u64
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
inline double ord_to_double(unsigned long long u) {
    const unsigned long long b = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFULL) : ~u;
    double d;
    memcpy(&d, &b, 8);
    return d;
}

template <int TB>
__device__ __forceinline__ i128 block_sum_i128(i128 v) {
    __shared__ unsigned long long lo[TB / 32], hi[TB / 32];
    v = fx_warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        lo[w] = (unsigned long long)(u128)v;
        hi[w] = (unsigned long long)((u128)v >> 64);
    }
    __syncthreads();
    i128 r = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < TB / 32; ++i) r += (i128)(((u128)hi[i] << 64) | (u128)lo[i]);
    __syncthreads();
    return r;
}

constexpr int kTB = 256;

// sum of inc (+ its extremes: with the piece-length extremes of k_emit they
// give the points' bounding box, x = scl*len/sl and y = inc/si being monotone)
__global__ void k_sum_inc(const double* __restrict__ inc, int64_t n, int E,
                          unsigned long long* __restrict__ acc, unsigned long long* __restrict__ mm) {
    i128 s = 0;
    unsigned long long imn = ~0ULL, imx = 0;
    constexpr int U = 4;  // independent loads in flight per thread
    for (int64_t b = blockIdx.x * (int64_t)kTB * U + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * kTB * U) {
        double V[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = b + (int64_t)u * kTB;
            V[u] = i < n ? inc[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (b + (int64_t)u * kTB >= n) break;
            s += fx_from_double(V[u], E);
            imn = min(imn, ord_bits(V[u]));
            imx = max(imx, ord_bits(V[u]));
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        imn = min(imn, __shfl_xor_sync(0xffffffffu, imn, o));
        imx = max(imx, __shfl_xor_sync(0xffffffffu, imx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, imn);
        atomicMax(mm + 1, imx);
    }
    s = block_sum_i128<kTB>(s);
    if (threadIdx.x == 0) fx_atomic_add(acc, s);
}

// scale_pieces' second pass (digitization.hpp:39-45), split by input so the
// two halves run on different streams: var_inc as an exact fixed-point sum
// (k_var_inc, reads inc only) ...
__global__ void k_var_inc(const double* __restrict__ inc, int64_t n, double mean_inc, int Ei,
                          unsigned long long* __restrict__ acc) {
    i128 si = 0;
    constexpr int U = 4;  // independent loads in flight per thread
    for (int64_t b = blockIdx.x * (int64_t)kTB * U + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * kTB * U) {
        double V[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = b + (int64_t)u * kTB;
            V[u] = i < n ? inc[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (b + (int64_t)u * kTB >= n) break;
            const double di = V[u] - mean_inc;  // digitization.hpp:42,44
            si += fx_from_double(di * di, Ei);
        }
    }
    si = block_sum_i128<kTB>(si);
    if (threadIdx.x == 0) fx_atomic_add(acc + 2, si);
}

// ... and var_len's range histogram (k_len_hist, reads len only; seqsum.cu:
// ranges of VB_R pieces, counts per length <= RH, longer pieces listed) from
// which the reference's sequential var_len is reproduced bit for bit. It
// needs only mean_len = total steps / N, known before any pass. Warp per range.
constexpr int VB_R = 2048;

// SMALL (RH <= 16, e.g. config 4's lengths 1..9): each lane counts its 64
// pieces of a range in two registers of 8-bit fields (no shared-memory
// atomics, no match), widened to 16-bit fields for the warp reduction.
__device__ __forceinline__ unsigned long long spread8to16(uint32_t x) {
    return (unsigned long long)(x & 0xFFu) | ((unsigned long long)(x & 0xFF00u) << 8) |
           ((unsigned long long)(x & 0xFF0000u) << 16) | ((unsigned long long)(x & 0xFF000000u) << 24);
}

template <bool SMALL>
__global__ void __launch_bounds__(256) k_len_hist(
    const int32_t* __restrict__ len, int64_t n, double mean_len, uint16_t* __restrict__ hist,
    double* __restrict__ approx, uint32_t* __restrict__ long_idx,
    unsigned long long* __restrict__ long_n, int RH) {
    __shared__ uint32_t sh[8][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nr = (n + VB_R - 1) / VB_R;
    for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < nr; r += (int64_t)gridDim.x * 8) {
        if (!SMALL) {
            for (int l = lane; l < RH; l += 32) sh[w][l] = 0;
            __syncwarp();
        }
        unsigned long long c0 = 0, c1 = 0;
        double lsum = 0.0;
        const int64_t i0 = r * VB_R, i1 = min(i0 + VB_R, n);
        for (int64_t c = i0; c < i1; c += 32 * 8) {
            int32_t L[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t i = c + u * 32 + lane;
                L[u] = i < i1 ? len[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t i = c + u * 32 + lane;
                const bool v = i < i1;
                const int l = L[u];
                const bool in = v && l >= 1 && l <= RH;
                if (SMALL) {
                    const unsigned long long one = in ? 1ull << (8 * ((l - 1) & 7)) : 0ull;
                    if (l <= 8) c0 += one;
                    else c1 += one;
                } else {
                    const unsigned grp = __match_any_sync(0xffffffffu, in ? l : -1);
                    if (in && (__ffs(grp) - 1) == lane) atomicAdd(&sh[w][l - 1], (uint32_t)__popc(grp));
                }
                const bool lg = v && !in;
                const unsigned lm = __ballot_sync(0xffffffffu, lg);
                if (lm) {
                    unsigned long long b = 0;
                    if (lane == __ffs(lm) - 1) b = atomicAdd(long_n, (unsigned long long)__popc(lm));
                    b = __shfl_sync(0xffffffffu, b, __ffs(lm) - 1);
                    if (lg) {
                        long_idx[b + __popc(lm & ((1u << lane) - 1u))] = (uint32_t)i;
                        const double dl = (double)l - mean_len;
                        lsum += dl * dl;
                    }
                }
            }
        }
        if (SMALL) {
            unsigned long long e[4] = {spread8to16((uint32_t)c0), spread8to16((uint32_t)(c0 >> 32)),
                                       spread8to16((uint32_t)c1), spread8to16((uint32_t)(c1 >> 32))};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                for (int o = 16; o; o >>= 1) e[q] += __shfl_xor_sync(0xffffffffu, e[q], o);
            if (lane < RH) {
                const unsigned long long ew = lane < 4 ? e[0] : lane < 8 ? e[1] : lane < 12 ? e[2] : e[3];
                const uint32_t cnt = (uint32_t)(ew >> (16 * (lane & 3))) & 0xFFFFu;
                hist[r * RH + lane] = (uint16_t)cnt;
                const double dl = (double)(lane + 1) - mean_len;
                lsum += (double)cnt * (dl * dl);  // the record's approximate sum
            }
        } else {
            __syncwarp();
            for (int l = lane; l < RH; l += 32) {
                hist[r * RH + l] = (uint16_t)sh[w][l];
                const double dl = (double)(l + 1) - mean_len;
                lsum += (double)sh[w][l] * (dl * dl);  // the record's approximate sum
            }
        }
        for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if (lane == 0) approx[r] = lsum;
        __syncwarp();
    }
}

// ScalingParams::apply (core.hpp:130-132): materialised points (GA only)
__global__ void k_scale(const int32_t* __restrict__ len, const double* __restrict__ inc,
                        int64_t n, double scl, double sl, double si, double* __restrict__ pts) {
    for (int64_t i = blockIdx.x * (int64_t)kTB + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * kTB)
        reinterpret_cast<double2*>(pts)[i] = make_double2(scl * (double)len[i] / sl, inc[i] / si);
}

int grid_for(int64_t n) {
    const int64_t b = (n + kTB - 1) / kTB;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 8));
}

}  // namespace

void scale_pieces(const Pieces& pc, int64_t total_steps, double scl, Scaled& out,
                  cudaStream_t st, const Comm* cm, cudaStream_t aux) {
    const Comm one;
    const Comm& C = cm ? *cm : one;
    // global N, max|inc|, max len (identical fixed-point exponents on every rank)
    int64_t N = pc.N;
    double max_abs_inc = pc.max_abs_inc;
    int32_t max_len = pc.max_len;
    if (C.dist()) {
        struct Loc {
            int64_t n;
            double mi;
            int64_t ml;
        } loc{pc.N, pc.max_abs_inc, pc.max_len};
        std::vector<Loc> all(C.world);
        C.allgather(&loc, sizeof loc, all.data());
        N = 0;
        for (const auto& l : all) {
            N += l.n;
            max_abs_inc = std::max(max_abs_inc, l.mi);
            max_len = std::max<int32_t>(max_len, (int32_t)l.ml);
        }
    }
    if (N == 0) throw Error(INVALID_INPUT, "digitize: no pieces");
    if (scl < 0.0) throw Error(INVALID_INPUT, "scale_pieces: scl must be >= 0");
    const double n = (double)N;
    // Two independent chains: the increments (sum -> mean_inc -> var_inc, HBM
    // bound) on `si_st` and the lengths (range histogram -> the sequential
    // var_len of seqsum.cu, latency bound) on `st`. With an aux stream they
    // overlap; without one they run back to back on `st` (same results: every
    // sum is exact or bit-exact sequential, whatever the schedule).
    cudaStream_t si_st = aux ? aux : st;
    if (aux) {  // the pieces were written on st
        cudaEvent_t ev;
        JB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        JB_CUDA(cudaEventRecord(ev, st));
        JB_CUDA(cudaStreamWaitEvent(aux, ev, 0));
        JB_CUDA(cudaEventDestroy(ev));
    }
    // sum of lens over all pieces == total steps of all segments (exact)
    DArr<unsigned long long> acc(6, si_st);
    acc.zero();
    const int Einc = fx_exponent_for(max_abs_inc * n * 1.0000001 + 1e-300);
    DArr<unsigned long long> mm(2, si_st);  // extremes of inc (order-preserving bits)
    {
        const unsigned long long init[2] = {~0ULL, 0ULL};
        mm.upload(init, 2);
    }
    if (pc.N > 0) {
        JB_PROF("scale_sum_inc", si_st);
        k_sum_inc<<<grid_for(pc.N), kTB, 0, si_st>>>(pc.inc.p, pc.N, Einc, acc.p, mm.p);
    }
    JB_LAUNCH_CHECK();
    // mean_len: sequential double sum of integer lens is exact (< 2^53)
    const double mean_len = (double)total_steps / n;
    RangeHist vh;  // var_len's range histogram (seqsum.cu)
    const int RH = (int)std::min<int32_t>(std::max<int32_t>(pc.max_len, 1), 64);
    vh.alloc(pc.N, VB_R, 1, RH, pc.max_len > RH, st);
    if (pc.N > 0) {
        JB_PROF("scale_len_hist", st);
        const int64_t nr = vh.nr;
        auto kern = RH <= 16 ? k_len_hist<true> : k_len_hist<false>;
        kern<<<(int)std::max<int64_t>(1, std::min<int64_t>((nr + 7) / 8, (int64_t)num_sms() * 8)), 256,
               0, st>>>(pc.len.p, pc.N, mean_len, vh.hist.p, vh.approx.p, vh.long_idx.p, vh.long_n.p,
                        RH);
    }
    JB_LAUNCH_CHECK();
    if (!aux) JB_TRACE("scale: sum inc + len hist", st);
    std::vector<unsigned long long> h = acc.to_host(2);
    h = C.sum_i128(h);
    const std::vector<unsigned long long> hm = mm.to_host(2);
    const double mean_inc = fx_to_double(fx_load(h.data()), Einc) / n;

    const double dimax = max_abs_inc + std::fabs(mean_inc) + 1e-300;
    const int Ei = fx_exponent_for(dimax * dimax * n * 1.001 + 1e-300);
    acc.zero();
    if (pc.N > 0) {
        JB_PROF("scale_sum_var", si_st);
        k_var_inc<<<grid_for(pc.N), kTB, 0, si_st>>>(pc.inc.p, pc.N, mean_inc, Ei, acc.p);
    }
    JB_LAUNCH_CHECK();
    if (!aux) JB_TRACE("scale: var inc", st);
    // var_len: the reference's left-to-right sum of (len - mean_len)^2,
    // bit-exact (seqsum.cu); sigma_len then fixes every x = scl*len/sigma_len
    // and every reconstructed length (inverse.hpp:46)
    SeqTerms vt;
    vt.len = pc.len.p;
    vt.kind = SeqTerms::VAR_LEN;
    vt.a = mean_len;
    const double var_len = range_seq_sums(vh, vt, nullptr, st, cm)[0];
    JB_TRACE("scale: var len (sequential)", st);
    h = acc.to_host(4);  // joins the increments' stream
    h = C.sum_i128(h);
    const double var_inc = fx_to_double(fx_load(h.data() + 2), Ei);
    double sl = N > 1 ? std::sqrt(var_len / (n - 1.0)) : 0.0;
    double si = N > 1 ? std::sqrt(var_inc / (n - 1.0)) : 0.0;
    if (sl <= 0.0) sl = 1.0;
    if (si <= 0.0) si = 1.0;
    out.scl = scl;
    out.sigma_len = sl;
    out.sigma_inc = si;

    // bounding box of all points from the extremes of len and inc
    std::vector<unsigned long long> hb = {
        pc.N > 0 ? (unsigned long long)pc.min_len : ~0ULL, (unsigned long long)pc.max_len,
        hm[0], hm[1]};
    if (C.dist()) {
        auto all = C.gather(hb);
        for (int j = 0; j < 4; ++j) hb[j] = all[j];  // rank 0's extremes, then the others
        for (int r = 1; r < C.world; ++r) {
            hb[0] = std::min(hb[0], all[4 * r]);
            hb[1] = std::max(hb[1], all[4 * r + 1]);
            hb[2] = std::min(hb[2], all[4 * r + 2]);
            hb[3] = std::max(hb[3], all[4 * r + 3]);
        }
    }
    out.xmin = scl * (double)(int32_t)hb[0] / sl;  // k_scale's expressions, monotone
    out.xmax = scl * (double)(int32_t)hb[1] / sl;
    out.ymin = ord_to_double(hb[2]) / si;
    out.ymax = ord_to_double(hb[3]) / si;
    out.N_global = N;
    out.max_len_global = max_len;
}

PtsView points_view(const Pieces& pc, const Scaled& sc) {
    PtsView v;
    v.pts = sc.pts.p ? reinterpret_cast<const double2*>(sc.pts.p) : nullptr;
    v.len = pc.len.p;
    v.inc = pc.inc.p;
    v.scl = sc.scl;
    v.sl = sc.sigma_len;
    v.si = sc.sigma_inc;
    v.rsi = div_by_recip(sc.sigma_inc);
    return v;
}

void materialize_points(const Pieces& pc, Scaled& sc, cudaStream_t st) {
    if (sc.pts.p || pc.N == 0) return;
    sc.pts.alloc(2 * pc.N, st);
    JB_PROF("scale_points", st);
    k_scale<<<grid_for(pc.N), kTB, 0, st>>>(pc.len.p, pc.inc.p, pc.N, sc.scl, sc.sigma_len,
                                           sc.sigma_inc, sc.pts.p);
    JB_LAUNCH_CHECK();
}


// ---------------------------------------------------------------------------
// Nearest-center assignment + group statistics.

namespace {

// Group statistics of digitize (digitization.hpp:217-231) fused with the
// final assignment: count, first index, sum of lengths, sums of x and y.
// Only native 32-bit shared-memory atomics (64-bit ones are CAS loops):
//  * count, length sum and x sum come from a per-block histogram over
//    (piece length, cluster): x = scl*len/sigma_len is a function of len, so
//    the exact fixed-point x sum is sum_l hist[l] * fx(x_l);
//  * y (biased fixed point fx(y) + B in [0, 2^62)) is split into three
//    21-bit limbs, each accumulated in a u32 counter; 2048 points cannot
//    overflow a counter, so the counters are folded into 64-bit per-cluster
//    totals every two 1024-point rounds;
//  * first index: u32 atomicMin, taken only when it can lower the minimum.
// Pieces longer than the histogram (rare) go straight to global 64-bit
// atomics (native in L2). Everything is exact integer arithmetic, hence
// independent of the schedule; the host removes the bias (count * B).
constexpr int AS_TB = 256, AS_U = 4;
#ifndef JB_AS_MINB
#define JB_AS_MINB 4  // 64 registers, no spills: 4 CTAs per SM (3 at 75 registers: 7.55 -> 7.23 ms, config 4)
#endif
constexpr int kXRow = 64;

// Per-range output of the group statistics (seqsum.cu RangeHist): per range
// of R pieces (a multiple of AS_TB * AS_U) the (length, cluster) counts and
// the long pieces' approximate x sums; long pieces listed. hist == null: none.
struct RangeOut {
    uint16_t* hist = nullptr;
    double* approx = nullptr;  // per (range, cluster): approximate sum of the pieces' x
    uint32_t* long_idx = nullptr;
    unsigned long long* long_n = nullptr;
    int64_t R = 1024;
};

__global__ void __launch_bounds__(AS_TB, JB_AS_MINB) k_assign_stats(
    const PtsView pv, const int32_t* __restrict__ len, int64_t n,
    const double* __restrict__ centers, int k, int do_assign, uint32_t* __restrict__ labels,
    int Ex, int Ey, unsigned long long Bx, unsigned long long By,
    unsigned long long* __restrict__ gacc, CandGrid cg, RowGrid rg, int RH, RangeOut ro) {
    // gacc layout: count(k) len(k) first(k) sx(2k) sy(2k), sums biased
    extern __shared__ unsigned long long smem64[];
    double* cx = reinterpret_cast<double*>(smem64);
    double* cy = cx + k;
    unsigned long long* yacc = smem64 + (do_assign ? 2 * k : 0);  // 3k limb totals
    unsigned long long* tot = yacc + 3 * k;                        // 4k: count, len, x (lo, hi)
    double* lxr = reinterpret_cast<double*>(tot + 4 * k);          // k: this range's long x
    uint32_t* hist = reinterpret_cast<uint32_t*>(lxr + k);         // RH x k (this range)
    uint32_t* ylimb = hist + (size_t)RH * k;                        // 3k
    uint32_t* first = ylimb + 3 * k;                                // k
    for (int c = threadIdx.x; c < k; c += AS_TB) {
        if (do_assign) {
            cx[c] = centers[2 * c];
            cy[c] = centers[2 * c + 1];
        }
        yacc[c] = yacc[k + c] = yacc[2 * k + c] = 0;
        tot[c] = tot[k + c] = tot[2 * k + c] = tot[3 * k + c] = 0;
        lxr[c] = 0.0;
        ylimb[c] = ylimb[k + c] = ylimb[2 * k + c] = 0;
        first[c] = 0xFFFFFFFFu;
    }
    for (int j = threadIdx.x; j < RH * k; j += AS_TB) hist[j] = 0;
    __shared__ double s_xrow[kXRow];  // x of short pieces: k_scale's expression, once
    for (int l = threadIdx.x; l < kXRow; l += AS_TB) s_xrow[l] = pv.scl * (double)l / pv.sl;
    __syncthreads();
    auto fold = [&]() {
        __syncthreads();
        for (int c = threadIdx.x; c < 3 * k; c += AS_TB) {
            yacc[c] += ylimb[c];
            ylimb[c] = 0;
        }
        __syncthreads();
    };
    const int64_t R = ro.R, nr = (n + R - 1) / R;
    int round = 0;
    for (int64_t r = blockIdx.x; r < nr; r += gridDim.x) {
        const int64_t rend = min(n, (r + 1) * R);
        for (int64_t base0 = r * R; base0 < rend; base0 += (int64_t)AS_TB * AS_U) {
            const int64_t base = base0 + threadIdx.x;
            double2 pp[AS_U];
            int32_t ll[AS_U];
            uint32_t lb[AS_U];
#pragma unroll
            for (int u = 0; u < AS_U; ++u) {
                const int64_t i = base + (int64_t)u * AS_TB;
                pp[u] = make_double2(0.0, 0.0);
                ll[u] = 0;
                lb[u] = 0;
                if (i < rend) {
                    ll[u] = len[i];
                    if (pv.pts) {
                        pp[u] = pv.pts[i];
                    } else {  // x from len (k_scale's expression), y = inc / si
                        pp[u].y = pv.inc[i];
                    }
                    if (!do_assign) lb[u] = labels[i];
                }
            }
            if (!pv.pts) {
#pragma unroll
                for (int u = 0; u < AS_U; ++u) {
                    const int32_t l = ll[u];
                    pp[u] = make_double2(l >= 0 && l < kXRow ? s_xrow[l] : pv.scl * (double)l / pv.sl,
                                         div_by(pp[u].y, pv.si, pv.rsi));
                }
            }
            uint64_t cw[AS_U];  // row-cell words, all in flight before the searches
            if (do_assign) {
#pragma unroll
                for (int u = 0; u < AS_U; ++u) cw[u] = row_cell_word<true>(rg, ll[u], pp[u].y);
            }
#pragma unroll
            for (int u = 0; u < AS_U; ++u) {
                const int64_t i = base + (int64_t)u * AS_TB;
                const bool valid = i < rend;
                const double2 p = pp[u];
                const int32_t l = ll[u];
                uint32_t lab = lb[u];
                bool lg = false;
                if (valid) {
                    if (do_assign) {
                        lab = row_nearest_w(cg, rg.spill, cw[u], p.x, p.y, cx, cy, k);
                        labels[i] = lab;
                    }
                    if ((uint32_t)i < first[lab]) atomicMin(first + lab, (uint32_t)i);
                    if (l >= 1 && l <= RH) {
                        atomicAdd(hist + (size_t)(l - 1) * k + lab, 1u);
                    } else {  // rare: long piece
                        lg = true;
                        atomicAdd(gacc + lab, 1ULL);
                        atomicAdd(gacc + k + lab, (unsigned long long)l);
                        fx_atomic_add_small(gacc + 3 * k + 2 * lab,
                                            (u128)(fx_from_double(p.x, Ex) + (i128)Bx));
                        if (ro.hist) atomicAdd(lxr + lab, p.x);
                    }
                    const unsigned long long yb = (unsigned long long)(fx_from_double(p.y, Ey) + (i128)By);
                    atomicAdd(ylimb + lab, (uint32_t)(yb & 0x1FFFFFu));
                    atomicAdd(ylimb + k + lab, (uint32_t)((yb >> 21) & 0x1FFFFFu));
                    atomicAdd(ylimb + 2 * k + lab, (uint32_t)(yb >> 42));
                }
                if (ro.hist) {  // list the long pieces (one counter atomic per warp)
                    const unsigned lm = __ballot_sync(0xffffffffu, lg);
                    if (lm) {
                        const int lane = threadIdx.x & 31;
                        unsigned long long b = 0;
                        if (lane == __ffs(lm) - 1) b = atomicAdd(ro.long_n, (unsigned long long)__popc(lm));
                        b = __shfl_sync(0xffffffffu, b, __ffs(lm) - 1);
                        if (lg) ro.long_idx[b + __popc(lm & ((1u << lane) - 1u))] = (uint32_t)i;
                    }
                }
            }
            if (++round & 1) continue;
            fold();
        }
        // end of range r: fold its counts into the block totals, write its record
        __syncthreads();
        for (int c = threadIdx.x; c < k; c += AS_TB) {
            unsigned long long cnt = 0, ls = 0;
            u128 sx = 0;
            double ax = lxr[c];
            for (int l = 1; l <= RH; ++l) {
                const uint32_t h = hist[(size_t)(l - 1) * k + c];
                if (!h) continue;
                cnt += h;
                ls += (unsigned long long)h * (unsigned long long)l;
                const double xl = row_x(rg, l);
                const u128 xb = (u128)(fx_from_double(xl, Ex) + (i128)Bx);
                sx += xb * (u128)h;
                ax += (double)h * xl;
            }
            tot[c] += cnt;
            tot[k + c] += ls;
            const u128 t0 = ((u128)tot[3 * k + c] << 64 | tot[2 * k + c]) + sx;
            tot[2 * k + c] = (unsigned long long)t0;
            tot[3 * k + c] = (unsigned long long)(t0 >> 64);
            if (ro.hist) ro.approx[r * k + c] = ax;
            lxr[c] = 0.0;
        }
        __syncthreads();
        for (int j = threadIdx.x; j < RH * k; j += AS_TB) {
            if (ro.hist) ro.hist[r * RH * k + j] = (uint16_t)hist[j];
            hist[j] = 0;
        }
        __syncthreads();
    }
    fold();
    for (int c = threadIdx.x; c < k; c += AS_TB) {
        if (tot[c]) {
            atomicAdd(gacc + c, tot[c]);
            atomicAdd(gacc + k + c, tot[k + c]);
            fx_atomic_add(gacc + 3 * k + 2 * c, (i128)(((u128)tot[3 * k + c] << 64) | tot[2 * k + c]));
        }
        const u128 sy = (u128)yacc[c] + ((u128)yacc[k + c] << 21) + ((u128)yacc[2 * k + c] << 42);
        if (sy) fx_atomic_add(gacc + 5 * k + 2 * c, (i128)sy);
        if (first[c] != 0xFFFFFFFFu) atomicMin(gacc + 2 * k + c, (unsigned long long)first[c]);
    }
}

// Large alphabets (GA can form thousands of groups; labels are given): the
// same exact statistics with global 64-bit atomics (native in L2).
__global__ void k_stats_global(const PtsView pv, const int32_t* __restrict__ len,
                               int64_t n, const uint32_t* __restrict__ labels, int k, int Ex,
                               int Ey, unsigned long long Bx, unsigned long long By,
                               unsigned long long* __restrict__ gacc) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t lab = labels[i];
        const double2 p = pv.at(i);
        atomicAdd(gacc + lab, 1ULL);
        atomicAdd(gacc + k + lab, (unsigned long long)len[i]);
        if ((unsigned long long)i < gacc[2 * k + lab]) atomicMin(gacc + 2 * k + lab, (unsigned long long)i);
        fx_atomic_add_small(gacc + 3 * k + 2 * lab, (u128)(fx_from_double(p.x, Ex) + (i128)Bx));
        fx_atomic_add_small(gacc + 5 * k + 2 * lab, (u128)(fx_from_double(p.y, Ey) + (i128)By));
    }
}

// out may be the input itself (in place) or a second array
__global__ void k_relabel(const uint32_t* labels, uint32_t* out, int64_t n,
                          const uint32_t* __restrict__ rank_of, int k) {
    extern __shared__ uint32_t rk[];
    for (int c = threadIdx.x; c < k; c += blockDim.x) rk[c] = rank_of[c];
    __syncthreads();
    // 16-byte accesses, two in flight per thread (labels are 256-byte aligned)
    const uint4* l4 = reinterpret_cast<const uint4*>(labels);
    uint4* o4 = reinterpret_cast<uint4*>(out);
    const int64_t n4 = n >> 2, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += 2 * stride) {
        uint4 a = l4[i], b = make_uint4(0, 0, 0, 0);
        const bool two = i + stride < n4;
        if (two) b = l4[i + stride];
        o4[i] = make_uint4(rk[a.x], rk[a.y], rk[a.z], rk[a.w]);
        if (two) o4[i + stride] = make_uint4(rk[b.x], rk[b.y], rk[b.z], rk[b.w]);
    }
    for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = rk[labels[i]];
}

__global__ void k_relabel_global(const uint32_t* labels, uint32_t* out, int64_t n,
                                 const uint32_t* __restrict__ rank_of) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = rank_of[labels[i]];
}

__global__ void k_sample_len(const uint64_t* __restrict__ sample,
                             const uint32_t* __restrict__ slab, int64_t S,
                             const int32_t* __restrict__ len, unsigned long long* __restrict__ ls,
                             unsigned long long* __restrict__ lc) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S;
         s += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t g = slab[s];
        atomicAdd(ls + g, (unsigned long long)len[sample[s]]);
        atomicAdd(lc + g, 1ULL);
    }
}

__global__ void k_gather(const double2* __restrict__ pts, const uint64_t* __restrict__ idx,
                         int64_t S, double2* __restrict__ out) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S;
         s += (int64_t)gridDim.x * blockDim.x)
        out[s] = pts[idx[s]];
}

}  // namespace

void assign_and_stats(const PtsView& pv, const int32_t* d_len, int64_t n,
                      const std::vector<double>& centers, uint64_t k, const BBox& bb,
                      bool do_assign, uint32_t* d_labels, GroupStats& gs, cudaStream_t st,
                      int32_t max_len, double scl, double sigma_len, const Comm* cm,
                      int64_t first_base, RangeHist* rh) {
    DArr<double> dc(std::max<uint64_t>(2 * k, 1), st);
    if (centers.size() >= 2 * k) dc.upload(centers.data(), 2 * k);  // GA: no centers needed
    else if (do_assign) throw Error(INTERNAL, "assignment without centers");
    DArr<unsigned long long> acc(7 * k, st);  // cl(k) len(k) first(k) sx(2k) sy(2k)
    acc.zero();
    JB_CUDA(cudaMemsetAsync(acc.p + 2 * k, 0xFF, sizeof(unsigned long long) * k, st));
    const double mx = std::max(std::fabs(bb.xmin), std::fabs(bb.xmax));
    const double my = std::max(std::fabs(bb.ymin), std::fabs(bb.ymax));
    (void)n;
    // biased per-element fixed point: fx(v) + B in [0, 2^62)
    auto exp_for = [](double m) {
        const int e = fx_exponent_for(m + 1e-300);  // 125 - e', m < 2^e'
        return e - 125 + 61;                         // 61 - e'
    };
    const int Ex = exp_for(mx), Ey = exp_for(my);
    const unsigned long long Bx = (unsigned long long)fx_from_double(mx, Ex);
    const unsigned long long By = (unsigned long long)fx_from_double(my, Ey);
    if (n >= (1LL << 32)) throw Error(INVALID_INPUT, "more than 2^32 pieces on one GPU");
    if (k > 2048 && do_assign)
        throw Error(INVALID_INPUT, "k > 2048 is not supported by the assignment kernel");
    // histogram rows: piece lengths 1..RH (longer pieces take the global path)
    int64_t rh_ = std::min<int64_t>(std::max<int32_t>(max_len, 1), 64);
    rh_ = std::min<int64_t>(rh_, std::max<int64_t>(1, 8192 / (int64_t)std::max<uint64_t>(k, 1)));
    const int RH = (int)rh_;
    const size_t smem = (do_assign ? sizeof(double) * 2 * k : 0) + sizeof(unsigned long long) * 7 * k +
                        sizeof(double) * k + sizeof(uint32_t) * ((size_t)RH * k + 4 * k);
    if (k <= 2048)
        JB_CUDA(cudaFuncSetAttribute(k_assign_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 1)));
    RowGrid rg = make_row_grid_desc(bb.ymin, bb.ymax, scl, sigma_len, max_len, 1 << 20);
    CandGrid cg{};
    DArr<uint16_t> cg_cnt, cg_cand;
    DArr<uint64_t> rg_cell;
    DArr<uint16_t> rg_spill;
    if (do_assign) {
        // exact candidate grids over the points' bounding box (jb_grid.cuh,
        // jb_rowgrid.cuh): rows for short pieces, 2-D for the rest
        const int G = grid_side_for(k), cap = 32;
        cg = make_grid_desc(bb.xmin, bb.xmax, bb.ymin, bb.ymax, G, cap);
        cg_cnt.alloc((size_t)G * G, st);
        cg_cand.alloc((size_t)G * G * cap, st);
        cg.cnt = cg_cnt.p;
        cg.cand = cg_cand.p;
        rg_cell.alloc((size_t)rg.R * rg.Gy, st);
        rg.cell = rg_cell.p;
        rg_spill.alloc((size_t)rg.R * rg.Gy * kSpill, st);
        rg.spill = rg_spill.p;
        JB_PROF("assign_grid", st);
        launch_grid_build(cg, dc.p, (int)k, st);
        JB_LAUNCH_CHECK();
        launch_row_grid_build(rg, dc.p, (int)k, st);
        JB_LAUNCH_CHECK();
    }
    if (k > 2048) {
        if (n > 0) {
            JB_PROF("assign_stats", st);
            k_stats_global<<<(int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 8)),
                             256, 0, st>>>(pv, d_len, n, d_labels,
                                           (int)k, Ex, Ey, Bx, By, acc.p);
        }
        JB_LAUNCH_CHECK();
    } else {
    int per_sm = 1;
    JB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_assign_stats, AS_TB, smem));
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((n + AS_TB * AS_U - 1) / (AS_TB * AS_U),
                             (int64_t)num_sms() * std::max(per_sm, 1)));
    // ranges: about one per block, at most 32768 pieces (u16 counts), a
    // multiple of the 1024-piece chunk
    constexpr int64_t kChunk = (int64_t)AS_TB * AS_U;
    const int64_t R = std::min<int64_t>(32768, std::max<int64_t>(kChunk, (n / grid) / kChunk * kChunk));
    RangeOut ro;
    ro.R = R;
    if (rh) {
        rh->alloc(n, R, (int)k, RH, max_len > RH, st);
        ro.hist = rh->hist.p;
        ro.approx = rh->approx.p;
        ro.long_idx = rh->long_idx.p;
        ro.long_n = rh->long_n.p;
    }
    if (n > 0) {
        JB_PROF("assign_stats", st);
        k_assign_stats<<<grid, AS_TB, smem, st>>>(pv, d_len, n,
                                                  dc.p, (int)k, do_assign ? 1 : 0, d_labels, Ex, Ey,
                                                  Bx, By, acc.p, cg, rg, RH, ro);
    }
    JB_LAUNCH_CHECK();
    }
    std::vector<unsigned long long> h = acc.to_host(7 * k);
    // exact per-cluster records: count, len sum, first index (global), unbiased sums
    std::vector<unsigned long long> rec(7 * k);
    for (uint64_t c = 0; c < k; ++c) {
        const i128 cnt = (i128)h[c];
        const u128 ux = (u128)(fx_load(&h[3 * k + 2 * c]) - cnt * (i128)Bx);
        const u128 uy = (u128)(fx_load(&h[5 * k + 2 * c]) - cnt * (i128)By);
        rec[7 * c + 0] = h[c];
        rec[7 * c + 1] = h[k + c];
        rec[7 * c + 2] = h[2 * k + c] == ~0ULL ? ~0ULL : h[2 * k + c] + (unsigned long long)first_base;
        rec[7 * c + 3] = (unsigned long long)ux;
        rec[7 * c + 4] = (unsigned long long)(ux >> 64);
        rec[7 * c + 5] = (unsigned long long)uy;
        rec[7 * c + 6] = (unsigned long long)(uy >> 64);
    }
    if (cm && cm->dist()) {  // group statistics of all ranks (exact integers)
        const auto all = cm->gather(rec);
        std::copy(all.begin(), all.begin() + 7 * k, rec.begin());  // rank 0's, then the others
        for (int r = 1; r < cm->world; ++r)
            for (uint64_t c = 0; c < k; ++c) {
                const unsigned long long* o = &all[(size_t)r * 7 * k + 7 * c];
                rec[7 * c + 0] += o[0];
                rec[7 * c + 1] += o[1];
                rec[7 * c + 2] = std::min(rec[7 * c + 2], o[2]);
                u128 x = ((u128)rec[7 * c + 4] << 64) | rec[7 * c + 3];
                u128 y = ((u128)rec[7 * c + 6] << 64) | rec[7 * c + 5];
                x += ((u128)o[4] << 64) | o[3];
                y += ((u128)o[6] << 64) | o[5];
                rec[7 * c + 3] = (unsigned long long)x;
                rec[7 * c + 4] = (unsigned long long)(x >> 64);
                rec[7 * c + 5] = (unsigned long long)y;
                rec[7 * c + 6] = (unsigned long long)(y >> 64);
            }
    }
    gs.counts.resize(k);
    gs.len_sums.resize(k);
    gs.first_seen.resize(k);
    gs.sum_x.resize(k);
    gs.sum_y.resize(k);
    for (uint64_t c = 0; c < k; ++c) {
        gs.counts[c] = rec[7 * c];
        gs.len_sums[c] = rec[7 * c + 1];
        gs.first_seen[c] = rec[7 * c + 2];
        gs.sum_x[c] = fx_to_double((i128)(((u128)rec[7 * c + 4] << 64) | rec[7 * c + 3]), Ex);
        gs.sum_y[c] = fx_to_double((i128)(((u128)rec[7 * c + 6] << 64) | rec[7 * c + 5]), Ey);
    }
}

namespace {
// first position of each key in a sorted key array (k + 1 offsets)
__global__ void k_key_offsets(const uint32_t* __restrict__ keys, int64_t n, int64_t k,
                              int64_t* __restrict__ off) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g > k) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)keys[mid] < g) lo = mid + 1;
        else hi = mid;
    }
    off[g] = lo;
}
}  // namespace

std::vector<double> exact_group_sum_x(const int32_t* d_len, const uint32_t* d_labels, int64_t n,
                                      uint64_t k, double scl, double sigma_len, cudaStream_t st,
                                      const Comm* cm) {
    // the pieces of each group in index order: a stable sort of the lengths
    // by label, then the groups' sequential sums (digitization.hpp:224-231)
    std::vector<int64_t> off(k + 1, 0);
    DArr<int32_t> slen(std::max<int64_t>(n, 1), st);
    if (n > 0) {
        DArr<uint32_t> skey(n, st);
        int bits = 1;
        while (bits < 32 && (1ULL << bits) < k) ++bits;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, d_labels, skey.p, d_len, slen.p, n, 0, bits, st);
        DArr<uint8_t> tmp(std::max<size_t>(tb, 1), st);
        {
            JB_PROF("group_sort", st);
            cub::DeviceRadixSort::SortPairs(tmp.p, tb, d_labels, skey.p, d_len, slen.p, n, 0, bits,
                                            st);
        }
        JB_LAUNCH_CHECK();
        DArr<int64_t> doff(k + 1, st);
        k_key_offsets<<<(int)((k + 256) / 256), 256, 0, st>>>(skey.p, n, (int64_t)k, doff.p);
        JB_LAUNCH_CHECK();
        doff.download(off.data(), k + 1);
        JB_CUDA(cudaStreamSynchronize(st));
    }
    SeqTerms t;
    t.len = slen.p;
    t.kind = SeqTerms::X;
    t.a = scl;
    t.b = sigma_len;
    return seq_sum_nonneg(t, off, st, cm);
}

void relabel(uint32_t* d_labels, int64_t n, const std::vector<uint32_t>& rank_of,
             cudaStream_t st, uint32_t* d_out, bool sync) {
    const int k = (int)rank_of.size();
    uint32_t* out = d_out ? d_out : d_labels;
    DArr<uint32_t> rk(k, st);  // returns to st's cache: reuse is ordered after the kernel
    rk.upload(rank_of.data(), k);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 8));
    JB_PROF("relabel", st);
    if ((size_t)k * 4 <= 48 * 1024 && (((uintptr_t)d_labels | (uintptr_t)out) & 15) == 0)
        k_relabel<<<grid, 256, k * 4, st>>>(d_labels, out, n, rk.p, k);
    else
        k_relabel_global<<<grid, 256, 0, st>>>(d_labels, out, n, rk.p);
    JB_LAUNCH_CHECK();
    if (sync) JB_CUDA(cudaStreamSynchronize(st));
}

void sample_len_stats(const uint64_t* d_sample, const uint32_t* d_sample_labels, int64_t S,
                      const int32_t* d_len, uint64_t k, std::vector<uint64_t>& len_sum,
                      std::vector<uint64_t>& count, cudaStream_t st) {
    DArr<unsigned long long> acc(2 * k, st);
    acc.zero();
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((S + 255) / 256, num_sms() * 8));
    k_sample_len<<<grid, 256, 0, st>>>(d_sample, d_sample_labels, S, d_len, acc.p, acc.p + k);
    JB_LAUNCH_CHECK();
    auto h = acc.to_host(2 * k);
    len_sum.assign(h.begin(), h.begin() + k);
    count.assign(h.begin() + k, h.end());
}

void gather_points(const double* d_pts, const uint64_t* d_idx, int64_t S, double* d_out,
                   cudaStream_t st) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((S + 255) / 256, num_sms() * 8));
    {
        JB_PROF("sample_gather", st);
        k_gather<<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(d_pts), d_idx, S,
                                   reinterpret_cast<double2*>(d_out));
    }
    JB_LAUNCH_CHECK();
}

}  // namespace jb

// ---------------------------------------------------------------------------
// symbolize_with (digitization.hpp:297-307): held-out pieces against a
// fitted codebook -- ScalingParams::apply (core.hpp:130-132) then
// Codebook::nearest (core.hpp:147-160, lowest index on ties), through the
// same exact grid assignment as the fit.

namespace jb {
namespace {

__global__ void k_piece_extremes(const int32_t* __restrict__ len, const double* __restrict__ inc,
                                 int64_t n, unsigned long long* __restrict__ mm,
                                 int* __restrict__ nonfinite) {
    unsigned long long lmn = ~0ULL, lmx = 0, imn = ~0ULL, imx = 0;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        // order-preserving u64 of the signed len
        const unsigned long long l = (unsigned long long)((long long)len[i]) ^ 0x8000000000000000ULL;
        const double v = inc[i];
        bad |= !isfinite(v);
        lmn = min(lmn, l);
        lmx = max(lmx, l);
        imn = min(imn, ord_bits(v));
        imx = max(imx, ord_bits(v));
    }
    for (int o = 16; o > 0; o >>= 1) {
        lmn = min(lmn, __shfl_xor_sync(0xffffffffu, lmn, o));
        lmx = max(lmx, __shfl_xor_sync(0xffffffffu, lmx, o));
        imn = min(imn, __shfl_xor_sync(0xffffffffu, imn, o));
        imx = max(imx, __shfl_xor_sync(0xffffffffu, imx, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm + 0, lmn);
        atomicMax(mm + 1, lmx);
        atomicMin(mm + 2, imn);
        atomicMax(mm + 3, imx);
        if (bad) atomicExch(nonfinite, 1);
    }
}

// Codebook::nearest over all centers (large or degenerate codebooks)
__global__ void k_nearest_all(const PtsView pv, int64_t n, const double* __restrict__ centers,
                              uint64_t k, uint32_t* __restrict__ labels) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 q = pv.at(i);
        uint64_t best = 0;
        double bd = __longlong_as_double(0x7FF0000000000000LL);  // +inf
        for (uint64_t c = 0; c < k; ++c) {
            const double d = dist2(q.x, q.y, centers[2 * c], centers[2 * c + 1]);
            if (d < bd) {
                bd = d;
                best = c;
            }
        }
        labels[i] = (uint32_t)best;
    }
}

}  // namespace

void symbolize_pieces(const int32_t* d_len, const double* d_inc, int64_t n,
                      const std::vector<double>& centers, uint64_t k, const double scaling[3],
                      uint32_t* d_labels, cudaStream_t st) {
    if (k == 0) throw Error(INVALID_INPUT, "symbolize_with: empty codebook");
    if (n == 0) return;
    PtsView pv;
    pv.len = d_len;
    pv.inc = d_inc;
    pv.scl = scaling[0];
    pv.sl = scaling[1];
    pv.si = scaling[2];
    pv.rsi = div_by_recip(pv.si);
    DArr<unsigned long long> mm(4, st);
    const unsigned long long init[4] = {~0ULL, 0ULL, ~0ULL, 0ULL};
    mm.upload(init, 4);
    DArr<int> bad(1, st);
    bad.zero();
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 8));
    k_piece_extremes<<<grid, 256, 0, st>>>(d_len, d_inc, n, mm.p, bad.p);
    JB_LAUNCH_CHECK();
    std::vector<unsigned long long> h = mm.to_host(4);
    int hbad = 0;
    bad.download(&hbad, 1);
    JB_CUDA(cudaStreamSynchronize(st));
    const long long lmin = (long long)(h[0] ^ 0x8000000000000000ULL);
    const long long lmax = (long long)(h[1] ^ 0x8000000000000000ULL);
    BBox bb{pv.scl * (double)lmin / pv.sl, pv.scl * (double)lmax / pv.sl,
            ord_to_double(h[2]) / pv.si, ord_to_double(h[3]) / pv.si};
    bool grid_ok = !hbad && k <= 2048 && std::isfinite(pv.scl) && pv.scl >= 0.0 &&
                   std::isfinite(pv.sl) && pv.sl > 0.0 && std::isfinite(pv.si) && pv.si > 0.0 &&
                   std::isfinite(bb.xmin) && std::isfinite(bb.xmax) && std::isfinite(bb.ymin) &&
                   std::isfinite(bb.ymax) && lmin >= INT32_MIN && lmax <= INT32_MAX;
    for (uint64_t i = 0; i < 2 * k && grid_ok; ++i) grid_ok = std::isfinite(centers[i]);
    if (grid_ok) {
        GroupStats gs;
        assign_and_stats(pv, d_len, n, centers, k, bb, true, d_labels, gs, st,
                         (int32_t)std::max<long long>(lmax, 1), pv.scl, pv.sl);
        return;
    }
    DArr<double> dc(2 * k, st);
    dc.upload(centers.data(), 2 * k);
    JB_PROF("symbolize_nearest_all", st);
    k_nearest_all<<<grid, 256, 0, st>>>(pv, n, dc.p, k, d_labels);
    JB_LAUNCH_CHECK();
    JB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace jb
