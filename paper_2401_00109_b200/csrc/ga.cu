// ga.cu — greedy aggregation (clustering.hpp:292-375) on sm_100a.
//
// The reference sweeps points in stable key order: an unassigned point
// becomes a starting point and claims every unassigned later point of its key
// window (early stop on key gap > alpha) within distance alpha. The sweep is
// reproduced exactly in BATCHES by one cooperative kernel:
//   A. (one block) the next GA_M undecided points in key order (no owner yet)
//      are the candidates; every earlier point is decided. One warp walks
//      them in order with the candidates in registers: the smallest undecided
//      candidate is a start and claims the later undecided candidates of its
//      window within alpha (all tests of a step in flight together). After
//      GA_SMAX starts the batch is cut at the next undecided candidate.
//   B. (whole grid) every new start claims the undecided points of its
//      window within alpha; a point reached by several takes the FIRST start
//      (atomicMin on the sorted position), exactly as the sequential sweep.
// Work is the sequential sweep's (the starts' windows) plus one test per
// (start, later candidate) pair; a batch costs two grid barriers. Keys are
// sorted with a stable CUB radix sort on (key, index), matching
// std::stable_sort (:335-338). JB_GA_TRACE=1 prints block 0's cycles per
// phase and the batch statistics.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "jb_device.hpp"

namespace jb {

namespace {

__device__ __forceinline__ unsigned long long key_bits(double k) {
    if (k == 0.0) k = 0.0;  // -0.0 == +0.0 under operator<: canonicalize
    const unsigned long long b = (unsigned long long)__double_as_longlong(k);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__global__ void k_keys_norm(const double2* __restrict__ pts, int64_t n,
                            unsigned long long* __restrict__ kb, uint32_t* __restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        kb[i] = key_bits(sqrt(p.x * p.x + p.y * p.y));  // sort_keys two_norm (:294-297)
        idx[i] = (uint32_t)i;
    }
}

__global__ void k_keys_pca(const double2* __restrict__ pts, int64_t n, double vx, double vy,
                           double mx, double my, unsigned long long* __restrict__ kb,
                           uint32_t* __restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        kb[i] = key_bits(vx * (p.x - mx) + vy * (p.y - my));  // :321-322
        idx[i] = (uint32_t)i;
    }
}

__global__ void k_moments(const double2* __restrict__ pts, int64_t n, double mx, double my,
                          int Ex, int Ey, int Exx, int Exy, int Eyy, int pass,
                          unsigned long long* __restrict__ acc) {
    i128 a = 0, b = 0, c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        if (pass == 0) {
            a += fx_from_double(p.x, Ex);
            b += fx_from_double(p.y, Ey);
        } else {
            const double dx = p.x - mx, dy = p.y - my;
            a += fx_from_double(dx * dx, Exx);
            b += fx_from_double(dx * dy, Exy);
            c += fx_from_double(dy * dy, Eyy);
        }
    }
    a = fx_warp_sum(a);
    b = fx_warp_sum(b);
    c = fx_warp_sum(c);
    if ((threadIdx.x & 31) == 0) {
        fx_atomic_add(acc, a);
        fx_atomic_add(acc + 2, b);
        fx_atomic_add(acc + 4, c);
    }
}

__device__ __forceinline__ double key_from_bits(unsigned long long u) {
    const unsigned long long b = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFULL) : ~u;
    return __longlong_as_double((long long)b);
}

// sorted points + window ends: wend[i] = first j > i with key_j - key_i > alpha
__global__ void k_windows(const double2* __restrict__ pts, const unsigned long long* __restrict__ skb,
                          const uint32_t* __restrict__ sidx, int64_t n, double alpha,
                          int early_stop, double2* __restrict__ spt, double* __restrict__ skey,
                          int64_t* __restrict__ wend) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        spt[i] = pts[sidx[i]];
        const double ki = key_from_bits(skb[i]);
        skey[i] = ki;
        if (!early_stop) {
            wend[i] = n;
            continue;
        }
        int64_t a = i + 1, b = n;  // first j in [i+1, n) with key_j - ki > alpha, else n
        while (a < b) {
            const int64_t m = (a + b) >> 1;
            if (key_from_bits(skb[m]) - ki > alpha) b = m;
            else a = m + 1;
        }
        wend[i] = a;
    }
}

constexpr int GA_M = 256;   // candidates per batch (= block size of the sweep)
constexpr int GA_SMAX = 64; // starts per batch at most
constexpr unsigned long long kNoOwner = ~0ULL;

struct GaSweep {
    const double2* spt;
    const int64_t* wend;
    int64_t n;
    double alpha2;
    unsigned long long* owner;   // claiming start (sorted position; a start owns itself),
                                 // kNoOwner: undecided
    int64_t* real;               // GA_M: the batch's starts
    int64_t* wpre;               // GA_M + 1: prefix of their window sizes
    int* ctl;                    // [0] done, [1] starts in this batch, [2] batches
    int64_t* cursor;             // every position before it is decided
    unsigned long long* trace;   // JB_GA_TRACE: per batch 4 globaltimer stamps (else null)
};

constexpr int kGaTraceMax = 8192;

__device__ __forceinline__ void ga_stamp(const GaSweep& a, int round, int k) {
    // the warp sync holds the read until a preceding bar.sync has completed
    // (the clock read itself may issue before a deferred-blocking barrier)
    if (a.trace && blockIdx.x == 0 && threadIdx.x < 32 && round < kGaTraceMax) {
        __syncwarp();
        if (threadIdx.x == 0) a.trace[16 * round + k] = (unsigned long long)clock64();
    }
}

__device__ void ga_phase_a(const GaSweep& a, int round) {
    __shared__ int64_t cand[GA_M];
    __shared__ uint32_t adj[GA_M][GA_M / 32];
    __shared__ int wcnt[GA_M / 32];
    __shared__ int s_m, s_nreal;
    __shared__ int64_t s_real[GA_M], s_pre[GA_M + 1];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) s_m = 0;
    __syncthreads();
    // from the cursor rounded down to 8 (every earlier position is decided:
    // owner set). A position is a candidate iff no start owns it yet, so the
    // scan reads only the owners: GA_SCAN consecutive ones per thread and
    // pass, 16-byte loads, so a stretch the last claims covered is crossed in
    // few passes
    int64_t p0 = *a.cursor & ~(int64_t)7;
    constexpr int GA_SCAN = 8;
    while (s_m < GA_M && p0 < a.n) {
        const int64_t pb = p0 + (int64_t)t * GA_SCAN;
        uint32_t cm = 0;  // candidate bits of this thread's positions
        if (pb + GA_SCAN <= a.n) {
            const ulonglong2* o2 = reinterpret_cast<const ulonglong2*>(a.owner + pb);
            ulonglong2 v[GA_SCAN / 2];
#pragma unroll
            for (int r = 0; r < GA_SCAN / 2; ++r) v[r] = __ldcg(o2 + r);
#pragma unroll
            for (int r = 0; r < GA_SCAN / 2; ++r)
                cm |= (v[r].x == kNoOwner ? 1u : 0u) << (2 * r) |
                      (v[r].y == kNoOwner ? 2u : 0u) << (2 * r);
        } else {
            for (int r = 0; r < GA_SCAN; ++r)
                if (pb + r < a.n && __ldcg(a.owner + pb + r) == kNoOwner) cm |= 1u << r;
        }
        const int cnt = __popc(cm);
        int incl = cnt;  // block exclusive scan of the counts, in position order
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wcnt[w] = incl;
        __syncthreads();
        int off = s_m + incl - cnt;
        for (int q = 0; q < w; ++q) off += wcnt[q];
        for (uint32_t bits = cm; bits && off < GA_M; bits &= bits - 1) cand[off++] = pb + __ffs(bits) - 1;
        __syncthreads();
        if (t == 0) {
            int tot = s_m;
            for (int q = 0; q < GA_M / 32; ++q) tot += wcnt[q];
            s_m = tot < GA_M ? tot : GA_M;
        }
        p0 += (int64_t)GA_M * GA_SCAN;
        __syncthreads();
    }
    ga_stamp(a, round, 4);
    const int m = s_m;
    if (m == 0) {
        if (t == 0) a.ctl[0] = 1;
        return;
    }
    // the candidates' points and window ends, staged once (the pair tests
    // below read each of them up to GA_M times)
    __shared__ double2 s_pt[GA_M];
    __shared__ int64_t s_wend[GA_M];
    if (t < m) {
        s_pt[t] = a.spt[cand[t]];
        s_wend[t] = a.wend[cand[t]];
    }
    __syncthreads();
    ga_stamp(a, round, 5);
    // Starts in order (warp 0; lane l holds candidates 32k+l in registers):
    // the smallest undecided candidate is a start, and it claims every later
    // undecided candidate of its window within alpha (the sequential sweep
    // restricted to the batch). After GA_SMAX starts the batch is cut at
    // the next undecided candidate, which the next batch takes up.
    __shared__ int s_first[GA_M];
    __shared__ int s_cut;
    if (w == 0) {
        constexpr int NK = GA_M / 32;
        double2 cp[NK];
        int64_t cj[NK];
        uint32_t und = 0u;  // bit k: candidate 32k+lane undecided
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const int c = 32 * k + lane;
            cp[k] = s_pt[c];
            cj[k] = cand[c];
            if (c < m) und |= 1u << k;
        }
        int cut = m, nst = 0;
        for (;;) {
            const unsigned mine = und ? 32u * (__ffs(und) - 1) + lane : 0xffffffffu;
            const unsigned cu = __reduce_min_sync(0xffffffffu, mine);
            if (cu == 0xffffffffu) break;
            const int c = (int)cu;
            if (nst == GA_SMAX) {
                cut = c;
                break;
            }
            ++nst;
            if (lane == (c & 31)) und &= ~(1u << (c >> 5));
            if (lane == 0) s_first[c] = -1;
            const double2 pc = s_pt[c];
            const int64_t wc = s_wend[c];
            uint32_t hit = 0u;  // all NK tests independent (in flight together)
#pragma unroll
            for (int k = 0; k < NK; ++k) {
                const double d = dist2(pc.x, pc.y, cp[k].x, cp[k].y);
                hit |= (uint32_t)((cj[k] < wc) & (d <= a.alpha2)) << k;
            }
            hit &= und;
            und &= ~hit;
#pragma unroll
            for (int k = 0; k < NK; ++k)
                if ((hit >> k) & 1u) s_first[32 * k + lane] = c;
        }
        if (lane == 0) s_cut = cut;
    }
    __syncthreads();
    ga_stamp(a, round, 6);
    const int mc = s_cut;  // candidates decided in this batch
    // claims written in parallel; the starts compacted in candidate order with
    // the prefix of their window sizes (the windows' points after the start)
    const bool isst = t < mc && s_first[t] < 0;
    if (t < mc) {
        const int64_t j = cand[t];
        a.owner[j] = isst ? (unsigned long long)j : (unsigned long long)cand[s_first[t]];
    }
    const int64_t win = isst ? s_wend[t] - cand[t] - 1 : 0;
    int rk = isst ? 1 : 0;
    int64_t wp = win;
    for (int o = 1; o < 32; o <<= 1) {
        const int yr = __shfl_up_sync(0xffffffffu, rk, o);
        const int64_t yw = __shfl_up_sync(0xffffffffu, wp, o);
        if (lane >= o) {
            rk += yr;
            wp += yw;
        }
    }
    __shared__ int s_wr[GA_M / 32];
    __shared__ int64_t s_ww[GA_M / 32];
    if (lane == 31) {
        s_wr[w] = rk;
        s_ww[w] = wp;
    }
    __syncthreads();
    int rb = 0;
    int64_t wb = 0;
    for (int q = 0; q < w; ++q) {
        rb += s_wr[q];
        wb += s_ww[q];
    }
    if (isst) {
        const int r = rb + rk - 1;
        s_real[r] = cand[t];
        s_pre[r] = wb + wp - win;
    }
    if (t == 0) {
        int nr = 0;
        int64_t tw = 0;
        for (int q = 0; q < GA_M / 32; ++q) {
            nr += s_wr[q];
            tw += s_ww[q];
        }
        s_nreal = nr;
        s_pre[nr] = tw;
        if (a.trace && round < kGaTraceMax) {
            a.trace[16 * round + 8] = (unsigned long long)tw;
            a.trace[16 * round + 9] = (unsigned long long)nr;
        }
        *a.cursor = mc < m ? cand[mc] : cand[m - 1] + 1;
        a.ctl[1] = nr;
        a.ctl[2] += 1;
    }
    __syncthreads();
    for (int r = t; r < s_nreal; r += GA_M) a.real[r] = s_real[r];
    for (int r = t; r <= s_nreal; r += GA_M) a.wpre[r] = s_pre[r];
}

// every new start claims the unassigned points of its window within alpha;
// the batch's starts (sorted position, point, window prefix) staged in
// shared memory for the per-position lookups
__device__ void ga_phase_b(const GaSweep& a) {
    __shared__ int64_t s_wp[GA_M + 1], s_rl[GA_M];
    __shared__ double2 s_ps[GA_M];
    const int nr = __ldcg(a.ctl + 1);
    for (int r = threadIdx.x; r <= nr; r += blockDim.x) {
        s_wp[r] = __ldcg(a.wpre + r);
        if (r < nr) {
            const int64_t sr = __ldcg(a.real + r);
            s_rl[r] = sr;
            s_ps[r] = a.spt[sr];
        }
    }
    __syncthreads();
    const int64_t total = s_wp[nr];
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nr;  // the start whose window slice holds q
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_wp[mid] <= q) lo = mid;
            else hi = mid;
        }
        const int64_t s = s_rl[lo];
        const int64_t j = s + 1 + (q - s_wp[lo]);
        if (__ldcg(a.owner + j) <= (unsigned long long)s) continue;  // decided before s
        const double2 ps = s_ps[lo], pj = a.spt[j];
        if (dist2(ps.x, ps.y, pj.x, pj.y) <= a.alpha2)
            atomicMin(a.owner + j, (unsigned long long)s);  // the first start claims it
    }
    __syncthreads();  // s_* are rewritten by the next batch's phase
}

__global__ void __launch_bounds__(GA_M) k_ga_sweep(GaSweep a) {
    namespace cgx = cooperative_groups;
    cgx::grid_group grid = cgx::this_grid();
    for (int round = 0;; ++round) {
        ga_stamp(a, round, 0);
        if (blockIdx.x == 0) ga_phase_a(a, round);
        ga_stamp(a, round, 1);
        grid.sync();
        ga_stamp(a, round, 2);
        if (((volatile int*)a.ctl)[0]) break;
        ga_phase_b(a);
        ga_stamp(a, round, 3);
        grid.sync();
    }
}

__global__ void k_start_flags(const unsigned long long* __restrict__ owner, int64_t n,
                              int64_t* __restrict__ is_start) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        is_start[j] = owner[j] == (unsigned long long)j ? 1 : 0;
}

__global__ void k_ga_labels(const unsigned long long* __restrict__ owner,
                            const int64_t* __restrict__ gid,
                            const uint32_t* __restrict__ sidx, int64_t n,
                            uint32_t* __restrict__ labels) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        labels[sidx[j]] = (uint32_t)gid[owner[j]];
}

int gcap(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8));
}

}  // namespace

void greedy_aggregate_device(const double* d_pts, int64_t n, double alpha, int sort_key,
                             bool early_stop, const BBox& bb, GAOut& out, cudaStream_t st) {
    if (!(alpha > 0.0)) throw Error(INVALID_INPUT, "GAConfig: alpha must be > 0");
    if (n <= 0) throw Error(INVALID_INPUT, "greedy_aggregate: no points");
    if (n >= (1LL << 32)) throw Error(INVALID_INPUT, "greedy_aggregate: too many points");
    const double2* pts = reinterpret_cast<const double2*>(d_pts);
    const double alpha2 = alpha * alpha;
    DArr<unsigned long long> kb(n, st), skb(n, st);
    DArr<uint32_t> idx(n, st), sidx(n, st);
    if (sort_key == 1) {
        k_keys_norm<<<gcap(n), 256, 0, st>>>(pts, n, kb.p, idx.p);
    } else {
        // sort_keys first principal component (:299-323): moments on device
        // (exact fixed point), angle with the host libm as the reference does
        DArr<unsigned long long> acc(6, st);
        const double bound = std::max(std::max(std::fabs(bb.xmin), std::fabs(bb.xmax)),
                                      std::max(std::fabs(bb.ymin), std::fabs(bb.ymax)));
        const double dn = (double)n;
        const int Ex = fx_exponent_for(bound * dn * 1.001 + 1e-300);
        acc.zero();
        k_moments<<<gcap(n), 256, 0, st>>>(pts, n, 0, 0, Ex, Ex, 0, 0, 0, 0, acc.p);
        JB_LAUNCH_CHECK();
        auto h1 = acc.to_host(6);
        const double mx = fx_to_double(fx_load(&h1[0]), Ex) / dn;
        const double my = fx_to_double(fx_load(&h1[2]), Ex) / dn;
        const double b2 = (2 * bound) * (2 * bound) * dn * 1.001 + 1e-300;
        const int E2 = fx_exponent_for(b2);
        acc.zero();
        k_moments<<<gcap(n), 256, 0, st>>>(pts, n, mx, my, 0, 0, E2, E2, E2, 1, acc.p);
        JB_LAUNCH_CHECK();
        auto h2 = acc.to_host(6);
        const double sxx = fx_to_double(fx_load(&h2[0]), E2);
        const double sxy = fx_to_double(fx_load(&h2[2]), E2);
        const double syy = fx_to_double(fx_load(&h2[4]), E2);
        const double theta = 0.5 * std::atan2(2.0 * sxy, sxx - syy);
        double vx = std::cos(theta), vy = std::sin(theta);
        if (vx < 0.0 || (vx == 0.0 && vy < 0.0)) {
            vx = -vx;
            vy = -vy;
        }
        k_keys_pca<<<gcap(n), 256, 0, st>>>(pts, n, vx, vy, mx, my, kb.p, idx.p);
    }
    JB_LAUNCH_CHECK();
    {
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, kb.p, skb.p, idx.p, sidx.p, n, 0, 64, st);
        DArr<uint8_t> tmp(tb, st);
        cub::DeviceRadixSort::SortPairs(tmp.p, tb, kb.p, skb.p, idx.p, sidx.p, n, 0, 64, st);
        JB_LAUNCH_CHECK();
    }
    DArr<double2> spt(n, st);
    DArr<double> skey(n, st);
    DArr<int64_t> wend(n, st);
    DArr<unsigned long long> owner(n, st);
    {
        JB_PROF("ga_windows", st);
        k_windows<<<gcap(n), 256, 0, st>>>(pts, skb.p, sidx.p, n, alpha, early_stop ? 1 : 0, spt.p,
                                       skey.p, wend.p);
    }
    JB_LAUNCH_CHECK();
    JB_CUDA(cudaMemsetAsync(owner.p, 0xFF, sizeof(unsigned long long) * n, st));
    DArr<int64_t> real(GA_M, st), wpre(GA_M + 1, st), cursor(1, st);
    DArr<int> ctl(3, st);
    ctl.zero();
    cursor.zero();
    const char* tr = std::getenv("JB_GA_TRACE");
    const bool trace = tr && tr[0] == '1';
    DArr<unsigned long long> trbuf(trace ? 16 * kGaTraceMax : 0, st);
    if (trace) trbuf.zero();
    GaSweep a{spt.p, wend.p, n, alpha2, owner.p, real.p, wpre.p, ctl.p, cursor.p,
              trace ? trbuf.p : nullptr};
    int per_sm = 0;
    JB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ga_sweep, GA_M, 0));
    if (per_sm < 1) throw Error(INTERNAL, "greedy_aggregate: sweep kernel does not fit");
    void* args[] = {&a};
    {
        JB_PROF("ga_sweep", st);
        JB_CUDA(cudaLaunchCooperativeKernel((const void*)k_ga_sweep,
                                            dim3(num_sms() * std::min(per_sm, 2)), dim3(GA_M), args, 0,
                                            st));
    }
    JB_LAUNCH_CHECK();
    int hctl[3];
    ctl.download(hctl, 3);
    JB_CUDA(cudaStreamSynchronize(st));
    const int rounds = hctl[2];
    if (trace) {  // mean SM cycles per batch of each phase (block 0's clock)
        auto h = trbuf.to_host(16 * kGaTraceMax);
        const int nb = std::min(rounds, kGaTraceMax - 1);
        const char* names[7] = {"select", "stage", "starts", "claims", "sync", "B", "sync"};
        const int from[7] = {0, 4, 5, 6, 1, 2, 3}, to[7] = {4, 5, 6, 1, 2, 3, 16};
        double s[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int r = 0; r < nb; ++r)
            for (int k = 0; k < 7; ++k) s[k] += (double)(h[16 * r + to[k]] - h[16 * r + from[k]]);
        std::fprintf(stderr, "ga trace: %d batches, kcycles/batch:", nb);
        for (int k = 0; k < 7; ++k) std::fprintf(stderr, " %s %.2f", names[k], s[k] / nb / 1e3);
        // claim positions and starts per batch: mean, quantiles
        std::vector<unsigned long long> tot(nb), nst(nb);
        for (int r = 0; r < nb; ++r) {
            tot[r] = h[16 * r + 8];
            nst[r] = h[16 * r + 9];
        }
        std::sort(tot.begin(), tot.end());
        std::sort(nst.begin(), nst.end());
        std::fprintf(stderr, "; claims/batch p50 %llu p90 %llu max %llu; starts/batch p50 %llu max %llu\n",
                     tot[nb / 2], tot[nb * 9 / 10], tot[nb - 1], nst[nb / 2], nst[nb - 1]);
    }
    // group ids in sorted order of their starting points
    DArr<int64_t> flg(n + 1, st), gid(n + 1, st);
    k_start_flags<<<gcap(n), 256, 0, st>>>(owner.p, n, flg.p);
    JB_CUDA(cudaMemsetAsync(flg.p + n, 0, 8, st));
    {
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, flg.p, gid.p, n + 1, st);
        DArr<uint8_t> tmp(tb, st);
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, flg.p, gid.p, n + 1, st);
        JB_LAUNCH_CHECK();
    }
    int64_t groups = 0;
    JB_CUDA(cudaMemcpyAsync(&groups, gid.p + n, 8, cudaMemcpyDeviceToHost, st));
    out.labels.alloc(n, st);
    k_ga_labels<<<gcap(n), 256, 0, st>>>(owner.p, gid.p, sidx.p, n, out.labels.p);
    JB_LAUNCH_CHECK();
    JB_CUDA(cudaStreamSynchronize(st));
    out.groups = (uint64_t)groups;
    out.rounds = rounds;
}

}  // namespace jb
