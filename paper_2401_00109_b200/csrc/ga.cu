// ga.cu — greedy aggregation (clustering.hpp:292-375) on sm_100a.
//
// The reference sweep visits points in stable key order; an unassigned point
// becomes a starting point and claims every unassigned later point inside its
// key window (early stop on key gap > alpha) within distance alpha. Equivalently
// (the lexicographically-first maximal independent set in sorted order):
//   * the earlier neighbours of sorted position j form N-(j) = {i in [lo(j), j):
//     dist2(p_i, p_j) <= alpha^2}, where lo(j) is the first i whose window
//     reaches j (windows are monotone in i because keys are sorted);
//   * j is claimed by the FIRST starting point in N-(j); j is a starting point
//     iff N-(j) holds none.
// Each round, every undecided j scans N-(j) in order from where it last
// stopped, skipping claimed neighbours: a start decides it (claimed), an
// undecided neighbour suspends it, reaching j makes it a start. Decisions are
// final, so rounds repeat until none is undecided; the result is exactly the
// sequential sweep's. Keys are sorted with a stable CUB radix sort on
// (key, index), matching std::stable_sort (:335-338).
#include <cub/cub.cuh>

#include <cmath>

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

// lo(j) = first i with wend[i] > j (wend is non-decreasing)
__global__ void k_lo(const int64_t* __restrict__ wend, int64_t n, int64_t* __restrict__ resume) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = 0, b = j;
        while (a < b) {
            const int64_t m = (a + b) >> 1;
            if (wend[m] > j) b = m;
            else a = m + 1;
        }
        resume[j] = a;
    }
}

// status: 0 undecided, 1 starting point, 2 claimed (owner = claiming start)
__global__ void k_round(const double2* __restrict__ spt, int64_t n, double alpha2,
                        const int64_t* __restrict__ list, int64_t n_list,
                        uint8_t* __restrict__ status, int64_t* __restrict__ resume,
                        int64_t* __restrict__ owner, unsigned long long* __restrict__ pending) {
    unsigned long long my_pending = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_list;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = list ? list[t] : t;
        if (*(volatile const uint8_t*)(status + j)) continue;
        const double2 pj = spt[j];
        int64_t i = resume[j];
        int decided = 0;
        for (; i < j; ++i) {
            const double2 pi = spt[i];
            if (dist2(pi.x, pi.y, pj.x, pj.y) <= alpha2) {
                const uint8_t si = *(volatile const uint8_t*)(status + i);
                if (si == 0) break;  // wait for i
                if (si == 1) {
                    owner[j] = i;
                    decided = 2;
                    break;
                }
            }
        }
        if (!decided && i == j) decided = 1;
        if (decided) {
            if (decided == 1) owner[j] = j;
            __threadfence();
            *(volatile uint8_t*)(status + j) = (uint8_t)decided;
        } else {
            resume[j] = i;
            ++my_pending;
        }
    }
    for (int o = 16; o > 0; o >>= 1) my_pending += __shfl_down_sync(0xffffffffu, my_pending, o);
    if ((threadIdx.x & 31) == 0 && my_pending) atomicAdd(pending, my_pending);
}

__global__ void k_start_flags(const uint8_t* __restrict__ status, int64_t n,
                              int64_t* __restrict__ is_start) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        is_start[j] = status[j] == 1 ? 1 : 0;
}

__global__ void k_ga_labels(const int64_t* __restrict__ owner, const int64_t* __restrict__ gid,
                            const uint32_t* __restrict__ sidx, int64_t n,
                            uint32_t* __restrict__ labels) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        labels[sidx[j]] = (uint32_t)gid[owner[j]];
}

__global__ void k_compact_pending(const uint8_t* __restrict__ status,
                                  const int64_t* __restrict__ list, int64_t n_list,
                                  int64_t* __restrict__ out, unsigned long long* __restrict__ cnt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_list;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = list ? list[t] : t;
        if (status[j] == 0) out[atomicAdd(cnt, 1ULL)] = j;
    }
}

int gcap(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)kSMs * 8));
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
    DArr<int64_t> wend(n, st), resume(n, st), owner(n, st);
    {
        JB_PROF("ga_windows", st);
        k_windows<<<gcap(n), 256, 0, st>>>(pts, skb.p, sidx.p, n, alpha, early_stop ? 1 : 0, spt.p,
                                       skey.p, wend.p);
    }
    JB_LAUNCH_CHECK();
    k_lo<<<gcap(n), 256, 0, st>>>(wend.p, n, resume.p);
    JB_LAUNCH_CHECK();
    DArr<uint8_t> status(n, st);
    status.zero();
    DArr<unsigned long long> pend(2, st);
    DArr<int64_t> listA(n, st), listB(n, st);
    int64_t* list = nullptr;  // nullptr = all positions
    int64_t n_list = n;
    int rounds = 0;
    for (;;) {
        pend.zero();
        {
            JB_PROF("ga_round", st);
            k_round<<<gcap(n_list), 256, 0, st>>>(spt.p, n, alpha2, list, n_list, status.p,
                                              resume.p, owner.p, pend.p);
        }
        JB_LAUNCH_CHECK();
        ++rounds;
        unsigned long long p = 0;
        pend.download(&p, 1);
        JB_CUDA(cudaStreamSynchronize(st));
        if (p == 0) break;
        if ((int64_t)p * 4 < n_list) {  // shrink the work list
            int64_t* dst = (list == listA.p) ? listB.p : listA.p;
            JB_CUDA(cudaMemsetAsync(pend.p + 1, 0, 8, st));
            k_compact_pending<<<gcap(n_list), 256, 0, st>>>(status.p, list, n_list, dst,
                                                            pend.p + 1);
            JB_LAUNCH_CHECK();
            unsigned long long c = 0;
            JB_CUDA(cudaMemcpyAsync(&c, pend.p + 1, 8, cudaMemcpyDeviceToHost, st));
            JB_CUDA(cudaStreamSynchronize(st));
            list = dst;
            n_list = (int64_t)c;
        }
    }
    // group ids in sorted order of their starting points
    DArr<int64_t> flg(n + 1, st), gid(n + 1, st);
    k_start_flags<<<gcap(n), 256, 0, st>>>(status.p, n, flg.p);
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
