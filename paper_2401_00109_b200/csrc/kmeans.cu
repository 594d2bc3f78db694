// kmeans.cu — sampled k-means++ on sm_100a (clustering.hpp:59-275).
//
//  * std::mt19937_64 generated on device; uniform_int / uniform_real mapped
//    exactly as libstdc++ (GCC 13) does: 128-bit Lemire downscaling with its
//    rejection loop, and generate_canonical = double(x) / 2^64.
//  * sample_indices (partial Fisher-Yates, :74-85) resolved in parallel:
//    idx[i] = value at position j_i just before swap i, recovered from the
//    "last earlier swap that touched this position" chains after one stable
//    radix sort of (j_i, i).
//  * d2_seed (:92-131): per round one fused pass (D^2 min-update + block
//    partial sums) and one single-block pick; the sums are exact 128-bit
//    fixed point, so the weighted pick is deterministic. The engine draw
//    cursor lives on device, so the k rounds run without host round trips.
//  * lloyd_once (:200-220): assignment with the exact tie rule, cluster sums
//    maintained incrementally as exact fixed-point integers (only points
//    whose label changed contribute), empty-cluster repair exactly as
//    update_means (:181-197).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "jb_device.hpp"

namespace jb {

namespace {

// ---------------------------------------------------------------------------
// std::mt19937_64

constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ULL, MT_LM = 0x7FFFFFFFULL;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ULL;

__device__ __forceinline__ uint64_t mt_twist(uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t x = (cur & MT_UM) | (nxt & MT_LM);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    return far ^ xa;
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

// One CTA walks the engine sequentially: each refill of 312 words is done in
// two dependency-free halves (words 0..155 read only old state; 156..311 read
// the fresh 0..155), then tempered in parallel.
__global__ void __launch_bounds__(320) k_mt_generate(uint64_t seed, uint64_t count,
                                                     uint64_t* __restrict__ out) {
    __shared__ uint64_t mt[312];
    const int t = threadIdx.x;
    if (t == 0) {
        mt[0] = seed;
        for (int i = 1; i < 312; ++i)
            mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    }
    __syncthreads();
    for (uint64_t base = 0; base < count; base += 312) {
        uint64_t v = 0;
        if (t < 156) v = mt_twist(mt[t], mt[t + 1], mt[t + 156]);
        __syncthreads();
        if (t < 156) mt[t] = v;
        __syncthreads();
        if (t >= 156 && t < 312) v = mt_twist(mt[t], mt[(t + 1) % 312], mt[t - 156]);
        __syncthreads();
        if (t >= 156 && t < 312) mt[t] = v;
        __syncthreads();
        if (t < 312 && base + t < count) out[base + t] = mt_temper(mt[t]);
    }
}

// libstdc++ _S_nd<unsigned __int128>: returns true if the draw is accepted
__device__ __forceinline__ bool lemire(uint64_t x, uint64_t erange, uint64_t& r) {
    const u128 prod = (u128)x * erange;
    const uint64_t low = (uint64_t)prod;
    r = (uint64_t)(prod >> 64);
    if (low < erange) {
        const uint64_t thresh = (0 - erange) % erange;
        if (low < thresh) return false;
    }
    return true;
}

// j_i = i + uniform_int(0, n-1-i) for i in [0,S), draws aligned by a small
// piecewise shift table (rejections are ~1e-10 per draw and handled by the
// host loop in sample_indices_device).
__global__ void k_fy_map(const uint64_t* __restrict__ raw, uint64_t n, uint64_t S,
                         const uint64_t* __restrict__ bp_i, const uint64_t* __restrict__ bp_sh,
                         int nbp, uint64_t* __restrict__ j_out, uint32_t* __restrict__ vals,
                         unsigned long long* __restrict__ first_reject) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t sh = 0;
        bool fixed = false;
        for (int b = 0; b < nbp; ++b) {
            if (i == bp_i[b]) fixed = true;  // host resolved this draw
            if (i >= bp_i[b]) sh = bp_sh[b];
        }
        const uint64_t erange = n - i;  // urange + 1
        uint64_t r;
        const bool ok = lemire(raw[i + sh], erange, r);
        if (!ok && !fixed) atomicMin(first_reject, (unsigned long long)i);
        j_out[i] = i + r;
        vals[i] = (uint32_t)i;
    }
}

__global__ void k_fy_links(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                           uint64_t S, uint32_t* __restrict__ P, uint32_t* __restrict__ L) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < S;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[r];
        const uint32_t i = vals[r];
        const bool same_prev = r > 0 && keys[r - 1] == key;
        P[i] = same_prev ? vals[r - 1] : 0xFFFFFFFFu;
        const bool group_last = (r + 1 == S) || keys[r + 1] != key;
        if (group_last && key < S) {
            // last swap (< key) that wrote position `key`
            if ((uint64_t)i < key) L[key] = i;
            else L[key] = same_prev ? vals[r - 1] : 0xFFFFFFFFu;
        }
    }
}

__global__ void k_fy_resolve(const uint64_t* __restrict__ j, const uint32_t* __restrict__ P,
                             const uint32_t* __restrict__ L, uint64_t S,
                             uint64_t* __restrict__ idx) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = P[i];
        if (p == 0xFFFFFFFFu) {
            idx[i] = j[i];
        } else {
            uint32_t q = p;  // g(q) = end of the chain q -> L[q] -> ...
            while (L[q] != 0xFFFFFFFFu) q = L[q];
            idx[i] = q;
        }
    }
}

int grid_cap(uint64_t n, int tb = 256, int per_sm = 8) {
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + tb - 1) / tb, (uint64_t)kSMs * per_sm));
}

}  // namespace

void mt19937_64_generate(uint64_t seed, uint64_t count, DArr<uint64_t>& out, cudaStream_t st) {
    out.alloc(count, st);
    {
        JB_PROF("mt19937_64", st);
        k_mt_generate<<<1, 320, 0, st>>>(seed, count, out.p);
    }
    JB_LAUNCH_CHECK();
}

uint64_t sample_indices_device(uint64_t n, uint64_t S, const uint64_t* d_raw, uint64_t raw_count,
                               DArr<uint64_t>& idx, cudaStream_t st) {
    if (n >= (1ULL << 32)) throw Error(INVALID_INPUT, "sampling: more than 2^32 pieces");
    DArr<uint64_t> j(S, st), keys_s(S, st);
    DArr<uint32_t> vals(S, st), vals_s(S, st);
    DArr<unsigned long long> rej(1, st);
    std::vector<uint64_t> bpi, bps;
    DArr<uint64_t> dbp(64, st);
    for (int round = 0;; ++round) {
        if (bpi.size() > 30) throw Error(INTERNAL, "sampling: too many rejections");
        std::vector<uint64_t> tab(bpi);
        tab.insert(tab.end(), bps.begin(), bps.end());
        dbp.upload(tab.data(), tab.size());
        const unsigned long long none = ~0ULL;
        rej.upload(&none, 1);
        {
            JB_PROF("sample_fy_map", st);
            k_fy_map<<<grid_cap(S), 256, 0, st>>>(d_raw, n, S, dbp.p, dbp.p + bpi.size(),
                                              (int)bpi.size(), j.p, vals.p, rej.p);
        }
        JB_LAUNCH_CHECK();
        unsigned long long r0;
        rej.download(&r0, 1);
        JB_CUDA(cudaStreamSynchronize(st));
        if (r0 == ~0ULL) break;
        // replay the rejection loop for draw r0 on the host (libstdc++ _S_nd)
        const uint64_t i0 = r0;
        uint64_t cur_sh = 0;
        for (size_t b = 0; b < bpi.size(); ++b)
            if (i0 >= bpi[b]) cur_sh = bps[b];
        const uint64_t erange = n - i0;
        uint64_t t = i0 + cur_sh;
        uint64_t extra = 0;
        for (;;) {
            if (t + 1 >= raw_count) throw Error(INTERNAL, "sampling: raw stream exhausted");
            uint64_t x;
            JB_CUDA(cudaMemcpy(&x, d_raw + t, 8, cudaMemcpyDeviceToHost));
            const u128 prod = (u128)x * erange;
            const uint64_t low = (uint64_t)prod;
            const uint64_t thresh = (0 - erange) % erange;
            if (!(low < erange && low < thresh)) break;
            ++t;
            ++extra;
        }
        // draw i0 uses raw[i0+cur_sh+extra]; later draws shift by `extra` more
        bpi.push_back(i0);
        bps.push_back(cur_sh + extra);
        (void)round;
    }
    uint64_t total_shift = bps.empty() ? 0 : bps.back();
    // stable radix sort of (j, i) by j
    int end_bit = 1;
    while (end_bit < 64 && (n >> end_bit) != 0) ++end_bit;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, j.p, keys_s.p, vals.p, vals_s.p, (int64_t)S, 0,
                                    end_bit, st);
    DArr<uint8_t> tmp(tb, st);
    cub::DeviceRadixSort::SortPairs(tmp.p, tb, j.p, keys_s.p, vals.p, vals_s.p, (int64_t)S, 0,
                                    end_bit, st);
    JB_LAUNCH_CHECK();
    DArr<uint32_t> P(S, st), L(S, st);
    JB_CUDA(cudaMemsetAsync(L.p, 0xFF, sizeof(uint32_t) * S, st));
    k_fy_links<<<grid_cap(S), 256, 0, st>>>(keys_s.p, vals_s.p, S, P.p, L.p);
    JB_LAUNCH_CHECK();
    idx.alloc(S, st);
    {
        JB_PROF("sample_fy_resolve", st);
        k_fy_resolve<<<grid_cap(S), 256, 0, st>>>(j.p, P.p, L.p, S, idx.p);
    }
    JB_LAUNCH_CHECK();
    return S + total_shift;
}

// ---------------------------------------------------------------------------
// D^2 seeding

namespace {

constexpr int D2_TB = 256;
constexpr int D2_ITEMS = 8;
constexpr int D2_R = D2_TB * D2_ITEMS;  // elements per partial-sum block

struct SeedState {
    uint64_t cursor;    // next engine draw
    int64_t last;       // index of the latest center in the sample
    int32_t degenerate; // total == 0 round happened
    int32_t pad;
};

// d2[i] = min(d2[i], dist2(p_i, c_last)) (or init when `init`), plus the
// block's exact fixed-point partial sum of d2.
__global__ void __launch_bounds__(D2_TB) k_d2_update(const double2* __restrict__ pts, int64_t n,
                                                    double* __restrict__ d2,
                                                    const SeedState* __restrict__ ss, int init,
                                                    int E, unsigned long long* __restrict__ part) {
    const int64_t c = ss->last;
    const double2 cc = pts[c];
    const int64_t b0 = (int64_t)blockIdx.x * D2_R;
    i128 s = 0;
#pragma unroll
    for (int it = 0; it < D2_ITEMS; ++it) {
        const int64_t i = b0 + it * D2_TB + threadIdx.x;
        if (i < n) {
            const double2 p = pts[i];
            const double dd = dist2(p.x, p.y, cc.x, cc.y);
            double v;
            if (init) {
                v = dd;
            } else {
                v = d2[i];
                if (dd < v) v = dd;  // std::min(a, b) == (b < a) ? b : a
            }
            d2[i] = v;
            s += fx_from_double(v, E);
        }
    }
    __shared__ unsigned long long lo[D2_TB / 32], hi[D2_TB / 32];
    s = fx_warp_sum(s);
    if ((threadIdx.x & 31) == 0) {
        lo[threadIdx.x >> 5] = (unsigned long long)(u128)s;
        hi[threadIdx.x >> 5] = (unsigned long long)((u128)s >> 64);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        i128 t = 0;
        for (int w = 0; w < D2_TB / 32; ++w) t += (i128)(((u128)hi[w] << 64) | (u128)lo[w]);
        part[2 * blockIdx.x] = (unsigned long long)(u128)t;
        part[2 * blockIdx.x + 1] = (unsigned long long)((u128)t >> 64);
    }
}

// floor(u * 2^E) for u >= 0 as an integer (u * 2^E < 2^126)
__device__ __forceinline__ i128 fx_floor(double u, int E) {
    return fx_from_double(u, E);  // magnitude truncation == floor for u >= 0
}

constexpr int PICK_TB = 1024;

// First center: uniform_int(0, n-1) (clustering.hpp:103-104).
__global__ void k_pick_first(const uint64_t* __restrict__ raw, uint64_t n, SeedState* ss,
                             int64_t* __restrict__ chosen) {
    uint64_t cur = ss->cursor, r;
    while (!lemire(raw[cur], n, r)) ++cur;
    ss->cursor = cur + 1;
    ss->last = (int64_t)r;
    chosen[0] = (int64_t)r;
}

// One D^2 round pick: total > 0 ? weighted_index (:59-71) : first unchosen.
// Single block: find the partial-sum block holding the crossing, then the
// element; all prefix arithmetic is exact 128-bit integer.
__global__ void __launch_bounds__(PICK_TB) k_pick(const uint64_t* __restrict__ raw,
                                                  const double* __restrict__ d2, int64_t n,
                                                  int nblocks,
                                                  const unsigned long long* __restrict__ part,
                                                  int E, SeedState* ss,
                                                  int64_t* __restrict__ chosen, int c) {
    __shared__ unsigned long long s_lo[PICK_TB], s_hi[PICK_TB];
    __shared__ unsigned long long s_total[2], s_before[2];
    __shared__ int s_found_block;
    __shared__ unsigned long long s_found_elem;
    const int t = threadIdx.x;
    const int per = (nblocks + PICK_TB - 1) / PICK_TB;
    const int b_lo = min(nblocks, t * per), b_hi = min(nblocks, b_lo + per);
    i128 local = 0;
    for (int b = b_lo; b < b_hi; ++b) local += fx_load(part + 2 * b);
    s_lo[t] = (unsigned long long)(u128)local;
    s_hi[t] = (unsigned long long)((u128)local >> 64);
    __syncthreads();
    if (t == 0) {  // exclusive scan of the per-thread totals (deterministic)
        i128 run = 0;
        for (int i = 0; i < PICK_TB; ++i) {
            const i128 v = (i128)(((u128)s_hi[i] << 64) | (u128)s_lo[i]);
            s_lo[i] = (unsigned long long)(u128)run;
            s_hi[i] = (unsigned long long)((u128)run >> 64);
            run += v;
        }
        s_total[0] = (unsigned long long)(u128)run;
        s_total[1] = (unsigned long long)((u128)run >> 64);
        s_found_block = 0x7FFFFFFF;
        s_found_elem = ~0ULL;
    }
    __syncthreads();
    const double total = fx_to_double(fx_load(s_total), E);
    if (!(total > 0.0)) {
        // every remaining point duplicates a center: first free slot (:120-124)
        if (t == 0) {
            int64_t next = 0;
            for (;;) {
                bool taken = false;
                for (int q = 0; q < c; ++q) taken |= chosen[q] == next;
                if (!taken) break;
                ++next;
            }
            chosen[c] = next;
            ss->last = next;
            ss->degenerate = 1;
        }
        return;
    }
    const uint64_t x = raw[ss->cursor];
    double canon = __ull2double_rn(x) * 0x1p-64;  // generate_canonical<double,53>
    if (canon >= 1.0) canon = 0x1.fffffffffffffp-1;  // nextafter(1, 0)
    const double u = canon * total + 0.0;             // uniform_real(0, total)
    const i128 U = fx_floor(u, E);
    // first partial-sum block whose inclusive prefix exceeds U
    int my_block = 0x7FFFFFFF;
    i128 my_before = 0;
    {
        i128 run = (i128)(((u128)s_hi[t] << 64) | (u128)s_lo[t]);
        for (int b = b_lo; b < b_hi; ++b) {
            const i128 v = fx_load(part + 2 * b);
            if (U < run + v) {
                my_block = b;
                my_before = run;
                atomicMin(&s_found_block, b);
                break;
            }
            run += v;
        }
    }
    __syncthreads();
    const int fb = s_found_block;
    if (fb == 0x7FFFFFFF) {
        // roundoff spill: last positive-weight index (:67-70)
        if (t == 0) {
            int64_t next = n - 1;
            for (int64_t i = n - 1; i >= 0; --i)
                if (d2[i] > 0.0) {
                    next = i;
                    break;
                }
            chosen[c] = next;
            ss->last = next;
            ss->cursor += 1;
        }
        return;
    }
    if (my_block == fb) {
        s_before[0] = (unsigned long long)(u128)my_before;
        s_before[1] = (unsigned long long)((u128)my_before >> 64);
    }
    __syncthreads();
    // within block fb: 1024 threads x 2 elements, exclusive scan of pairs
    const int64_t e0 = (int64_t)fb * D2_R + 2 * t;
    i128 a = 0, bsum = 0;
    if (e0 < n) a = fx_from_double(d2[e0], E);
    if (e0 + 1 < n) bsum = fx_from_double(d2[e0 + 1], E);
    const i128 pair = a + bsum;
    s_lo[t] = (unsigned long long)(u128)pair;
    s_hi[t] = (unsigned long long)((u128)pair >> 64);
    __syncthreads();
    if (t == 0) {
        i128 run = fx_load(s_before);
        for (int i = 0; i < PICK_TB; ++i) {
            const i128 v = (i128)(((u128)s_hi[i] << 64) | (u128)s_lo[i]);
            s_lo[i] = (unsigned long long)(u128)run;
            s_hi[i] = (unsigned long long)((u128)run >> 64);
            run += v;
        }
    }
    __syncthreads();
    {
        const i128 before = (i128)(((u128)s_hi[t] << 64) | (u128)s_lo[t]);
        unsigned long long hit = ~0ULL;
        if (e0 < n && U < before + a) hit = (unsigned long long)e0;
        else if (e0 + 1 < n && U < before + a + bsum) hit = (unsigned long long)(e0 + 1);
        if (hit != ~0ULL) atomicMin(&s_found_elem, hit);
    }
    __syncthreads();
    if (t == 0) {
        const int64_t next = (int64_t)s_found_elem;
        chosen[c] = next;
        ss->last = next;
        ss->cursor += 1;
    }
}

__global__ void k_copy_center(const double2* __restrict__ pts, const int64_t* __restrict__ chosen,
                              int k, double* __restrict__ centers) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const double2 p = pts[chosen[c]];
        centers[2 * c] = p.x;
        centers[2 * c + 1] = p.y;
    }
}

// ---------------------------------------------------------------------------
// Lloyd

struct ClusterAcc {
    unsigned long long* sx;   // 2k
    unsigned long long* sy;   // 2k
    unsigned long long* cnt;  // k (two's complement deltas)
};

// labels := nearest(centers); cluster sums updated by the delta of every
// label change (full accumulation when `full`). Also counts changes.
__global__ void k_lloyd_assign(const double2* __restrict__ pts, int64_t n,
                               const double* __restrict__ centers, int k,
                               uint32_t* __restrict__ labels, int full, int Ex, int Ey,
                               ClusterAcc acc, unsigned long long* __restrict__ changed) {
    extern __shared__ unsigned char smem[];
    double* cx = reinterpret_cast<double*>(smem);
    double* cy = cx + k;
    unsigned long long* s_sx = reinterpret_cast<unsigned long long*>(cy + k);
    unsigned long long* s_sy = s_sx + 2 * k;
    unsigned long long* s_cnt = s_sy + 2 * k;
    __shared__ unsigned long long s_changed;
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        cx[c] = centers[2 * c];
        cy[c] = centers[2 * c + 1];
        s_sx[2 * c] = s_sx[2 * c + 1] = 0;
        s_sy[2 * c] = s_sy[2 * c + 1] = 0;
        s_cnt[c] = 0;
    }
    if (threadIdx.x == 0) s_changed = 0;
    __syncthreads();
    unsigned long long my_changed = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        uint32_t best = 0;
        double bd = __longlong_as_double(0x7FF0000000000000LL);
        for (int c = 0; c < k; ++c) {
            const double d = dist2(p.x, p.y, cx[c], cy[c]);
            if (d < bd) {
                bd = d;
                best = (uint32_t)c;
            }
        }
        if (full) {
            labels[i] = best;
            fx_atomic_add(s_sx + 2 * best, fx_from_double(p.x, Ex));
            fx_atomic_add(s_sy + 2 * best, fx_from_double(p.y, Ey));
            atomicAdd(s_cnt + best, 1ULL);
        } else {
            const uint32_t old = labels[i];
            if (old != best) {
                labels[i] = best;
                ++my_changed;
                const i128 fx = fx_from_double(p.x, Ex), fy = fx_from_double(p.y, Ey);
                fx_atomic_add(s_sx + 2 * best, fx);
                fx_atomic_add(s_sy + 2 * best, fy);
                atomicAdd(s_cnt + best, 1ULL);
                fx_atomic_add(s_sx + 2 * old, -fx);
                fx_atomic_add(s_sy + 2 * old, -fy);
                atomicAdd(s_cnt + old, ~0ULL);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) my_changed += __shfl_down_sync(0xffffffffu, my_changed, o);
    if ((threadIdx.x & 31) == 0 && my_changed) atomicAdd(&s_changed, my_changed);
    __syncthreads();
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const i128 vx = fx_load(s_sx + 2 * c), vy = fx_load(s_sy + 2 * c);
        if (vx) fx_atomic_add(acc.sx + 2 * c, vx);
        if (vy) fx_atomic_add(acc.sy + 2 * c, vy);
        if (s_cnt[c]) atomicAdd(acc.cnt + c, s_cnt[c]);
    }
    if (threadIdx.x == 0 && s_changed) atomicAdd(changed, s_changed);
}

// centers[c] = sums[c] / counts[c] for non-empty clusters (update_means
// :177-180); reports the empty clusters in index order.
__global__ void k_means(ClusterAcc acc, int k, int Ex, int Ey, double* __restrict__ centers,
                        int* __restrict__ empties, int* __restrict__ n_empty) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const long long cnt = (long long)acc.cnt[c];
        if (cnt > 0) {
            centers[2 * c] = fx_to_double(fx_load(acc.sx + 2 * c), Ex) / (double)cnt;
            centers[2 * c + 1] = fx_to_double(fx_load(acc.sy + 2 * c), Ey) / (double)cnt;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int ne = 0;
        for (int c = 0; c < k; ++c)
            if ((long long)acc.cnt[c] <= 0) empties[ne++] = c;
        *n_empty = ne;
    }
}

// farthest point among clusters with count > 1 (update_means :183-192):
// max distance, lowest index on ties. Per-block candidates.
__global__ void k_far_block(const double2* __restrict__ pts, int64_t n,
                            const uint32_t* __restrict__ labels,
                            const double* __restrict__ centers,
                            const unsigned long long* __restrict__ cnt,
                            unsigned long long* __restrict__ out) {
    double bd = -1.0;
    int64_t bi = INT64_MAX;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t l = labels[i];
        if ((long long)cnt[l] <= 1) continue;
        const double2 p = pts[i];
        const double d = dist2(p.x, p.y, centers[2 * l], centers[2 * l + 1]);
        if (d > bd || (d == bd && i < bi)) {
            bd = d;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_down_sync(0xffffffffu, bd, o);
        const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (od > bd || (od == bd && oi < bi)) {
            bd = od;
            bi = oi;
        }
    }
    __shared__ double sd[32];
    __shared__ int64_t si[32];
    if ((threadIdx.x & 31) == 0) {
        sd[threadIdx.x >> 5] = bd;
        si[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sd[w] > bd || (sd[w] == bd && si[w] < bi)) {
                bd = sd[w];
                bi = si[w];
            }
        out[2 * blockIdx.x] = (unsigned long long)__double_as_longlong(bd);
        out[2 * blockIdx.x + 1] = (unsigned long long)bi;
    }
}

// re-seed empty cluster c at the farthest point (update_means :193-196)
__global__ void k_repair(const double2* __restrict__ pts, uint32_t* __restrict__ labels,
                         double* __restrict__ centers, ClusterAcc acc, int Ex, int Ey,
                         const unsigned long long* __restrict__ blk, int nblk, int c) {
    double bd = -1.0;
    int64_t bi = INT64_MAX;
    for (int b = 0; b < nblk; ++b) {
        const double d = __longlong_as_double((long long)blk[2 * b]);
        const int64_t i = (int64_t)blk[2 * b + 1];
        if (d > bd || (d == bd && i < bi)) {
            bd = d;
            bi = i;
        }
    }
    const int64_t far_i = (bi == INT64_MAX) ? 0 : bi;  // no candidate: far_i stays 0
    const uint32_t donor = labels[far_i];
    const double2 p = pts[far_i];
    const i128 fx = fx_from_double(p.x, Ex), fy = fx_from_double(p.y, Ey);
    fx_atomic_add(acc.sx + 2 * donor, -fx);
    fx_atomic_add(acc.sy + 2 * donor, -fy);
    acc.cnt[donor] -= 1;
    labels[far_i] = (uint32_t)c;
    // counts[c] = 1 and sums[c] = p (the cluster was empty: its sums are 0
    // up to exactness of the integer bookkeeping)
    acc.sx[2 * c] = 0;
    acc.sx[2 * c + 1] = 0;
    acc.sy[2 * c] = 0;
    acc.sy[2 * c + 1] = 0;
    fx_atomic_add(acc.sx + 2 * c, fx);
    fx_atomic_add(acc.sy + 2 * c, fy);
    acc.cnt[c] = 1;
    centers[2 * c] = p.x;
    centers[2 * c + 1] = p.y;
}

__global__ void k_sse(const double2* __restrict__ pts, int64_t n,
                      const uint32_t* __restrict__ labels, const double* __restrict__ centers,
                      int E, unsigned long long* __restrict__ acc) {
    i128 s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t l = labels[i];
        const double2 p = pts[i];
        s += fx_from_double(dist2(p.x, p.y, centers[2 * l], centers[2 * l + 1]), E);
    }
    s = fx_warp_sum(s);
    if ((threadIdx.x & 31) == 0) fx_atomic_add(acc, s);
}

}  // namespace

namespace {

struct LloydCtx {
    const double* pts;
    int64_t n;
    int k;
    int Ex, Ey;
    BBox bb;
    cudaStream_t st;
    DArr<double> centers;
    DArr<uint32_t> labels;
    DArr<unsigned long long> acc;  // 5k: sx(2k) sy(2k) cnt(k)
    DArr<unsigned long long> changed;
    DArr<int> empties;  // k + 1 (last = count)
    DArr<unsigned long long> far_blk;
    ClusterAcc cacc() { return ClusterAcc{acc.p, acc.p + 2 * k, acc.p + 4 * k}; }
    size_t smem() const { return sizeof(double) * 2 * k + sizeof(unsigned long long) * 5 * k; }
    int grid_assign() const {
        return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)kSMs * 2));
    }
};

void lloyd_assign(LloydCtx& L, bool full) {
    JB_CUDA(cudaMemsetAsync(L.changed.p, 0, 8, L.st));
    JB_PROF("lloyd_assign", L.st);
    k_lloyd_assign<<<L.grid_assign(), 256, L.smem(), L.st>>>(
        reinterpret_cast<const double2*>(L.pts), L.n, L.centers.p, L.k, L.labels.p, full ? 1 : 0,
        L.Ex, L.Ey, L.cacc(), L.changed.p);
    JB_LAUNCH_CHECK();
}

// update_means (:167-198) with the exact repair sequence
void lloyd_update_means(LloydCtx& L) {
    {
        JB_PROF("lloyd_means", L.st);
        k_means<<<1, 1024, 0, L.st>>>(L.cacc(), L.k, L.Ex, L.Ey, L.centers.p, L.empties.p,
                                  L.empties.p + L.k);
    }
    JB_LAUNCH_CHECK();
    int ne = 0;
    JB_CUDA(cudaMemcpyAsync(&ne, L.empties.p + L.k, sizeof(int), cudaMemcpyDeviceToHost, L.st));
    JB_CUDA(cudaStreamSynchronize(L.st));
    if (ne == 0) return;
    std::vector<int> em(ne);
    JB_CUDA(cudaMemcpy(em.data(), L.empties.p, sizeof(int) * ne, cudaMemcpyDeviceToHost));
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((L.n + 255) / 256, kSMs * 4));
    if (L.far_blk.n < (size_t)(2 * nblk)) L.far_blk.alloc(2 * nblk, L.st);
    for (int c : em) {
        k_far_block<<<nblk, 256, 0, L.st>>>(reinterpret_cast<const double2*>(L.pts), L.n,
                                            L.labels.p, L.centers.p, L.cacc().cnt, L.far_blk.p);
        JB_LAUNCH_CHECK();
        k_repair<<<1, 1, 0, L.st>>>(reinterpret_cast<const double2*>(L.pts), L.labels.p,
                                    L.centers.p, L.cacc(), L.Ex, L.Ey, L.far_blk.p, nblk, c);
        JB_LAUNCH_CHECK();
    }
}

}  // namespace

void lloyd_best_device(const double* d_pts, int64_t n, uint64_t k, uint64_t max_iters,
                       uint64_t n_init, const uint64_t* d_raw, uint64_t raw_count,
                       uint64_t* cursor, const BBox& bb, KMeansOut& out, cudaStream_t st) {
    if (k < 1) throw Error(INVALID_INPUT, "d2_seed: k must be >= 1");
    if ((int64_t)k > n) throw Error(INVALID_INPUT, "d2_seed: k exceeds points");
    if (k > 4096) throw Error(INVALID_INPUT, "k > 4096 is not supported by the Lloyd kernel");
    const double mx = std::max(std::fabs(bb.xmin), std::fabs(bb.xmax));
    const double my = std::max(std::fabs(bb.ymin), std::fabs(bb.ymax));
    const double wx = bb.xmax - bb.xmin, wy = bb.ymax - bb.ymin;
    const double d2max = (wx * wx + wy * wy) * (1.0 + 1e-9) + 1e-300;
    const int Ed2 = fx_exponent_for(d2max * (double)n * 1.001);

    LloydCtx L;
    L.pts = d_pts;
    L.n = n;
    L.k = (int)k;
    L.Ex = fx_exponent_for(mx * (double)n * 1.001 + 1e-300);
    L.Ey = fx_exponent_for(my * (double)n * 1.001 + 1e-300);
    L.bb = bb;
    L.st = st;
    L.centers.alloc(2 * k, st);
    L.labels.alloc(n, st);
    L.acc.alloc(5 * k, st);
    L.changed.alloc(1, st);
    L.empties.alloc(k + 1, st);
    JB_CUDA(cudaFuncSetAttribute(k_lloyd_assign, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)L.smem()));

    const int nblocks = (int)((n + D2_R - 1) / D2_R);
    DArr<double> d2(n, st);
    DArr<unsigned long long> part(2 * nblocks, st);
    DArr<SeedState> ss(1, st);
    DArr<int64_t> chosen(k, st);

    double best_sse = 0.0;
    for (uint64_t restart = 0; restart < n_init; ++restart) {
        // ---- d2_seed ----
        SeedState h{*cursor, 0, 0, 0};
        ss.upload(&h, 1);
        k_pick_first<<<1, 1, 0, st>>>(d_raw, (uint64_t)n, ss.p, chosen.p);
        JB_LAUNCH_CHECK();
        {
            JB_PROF("d2_update", st);
            k_d2_update<<<nblocks, D2_TB, 0, st>>>(reinterpret_cast<const double2*>(d_pts), n,
                                                   d2.p, ss.p, 1, Ed2, part.p);
        }
        JB_LAUNCH_CHECK();
        for (uint64_t c = 1; c < k; ++c) {
            {
                JB_PROF("d2_pick", st);
                k_pick<<<1, PICK_TB, 0, st>>>(d_raw, d2.p, n, nblocks, part.p, Ed2, ss.p, chosen.p,
                                          (int)c);
            }
            JB_LAUNCH_CHECK();
            if (c + 1 < k) {
                JB_PROF("d2_update", st);
                k_d2_update<<<nblocks, D2_TB, 0, st>>>(reinterpret_cast<const double2*>(d_pts),
                                                       n, d2.p, ss.p, 0, Ed2, part.p);
                JB_LAUNCH_CHECK();
            }
        }
        k_copy_center<<<1, 256, 0, st>>>(reinterpret_cast<const double2*>(d_pts), chosen.p,
                                         (int)k, L.centers.p);
        JB_LAUNCH_CHECK();
        ss.download(&h, 1);
        JB_CUDA(cudaStreamSynchronize(st));
        if (h.cursor > raw_count) throw Error(INTERNAL, "rng stream exhausted");
        *cursor = h.cursor;

        // ---- Lloyd ----
        L.acc.zero();
        lloyd_assign(L, true);
        uint64_t it = 0;
        for (; it < max_iters; ++it) {
            lloyd_update_means(L);
            lloyd_assign(L, false);
            unsigned long long ch = 0;
            JB_CUDA(cudaMemcpyAsync(&ch, L.changed.p, 8, cudaMemcpyDeviceToHost, st));
            JB_CUDA(cudaStreamSynchronize(st));
            if (ch == 0) {
                ++it;
                break;
            }
        }
        lloyd_update_means(L);
        double sse = 0.0;
        if (n_init > 1) {
            DArr<unsigned long long> sacc(2, st);
            sacc.zero();
            k_sse<<<(int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, kSMs * 8)), 256,
                    0, st>>>(reinterpret_cast<const double2*>(d_pts), n, L.labels.p, L.centers.p,
                             Ed2, sacc.p);
            JB_LAUNCH_CHECK();
            auto hs = sacc.to_host(2);
            sse = fx_to_double(fx_load(hs.data()), Ed2);
        }
        if (restart == 0 || sse < best_sse) {
            best_sse = sse;
            out.k = k;
            out.centers = L.centers.to_host(2 * k);
            out.labels.alloc(n, st);
            JB_CUDA(cudaMemcpyAsync(out.labels.p, L.labels.p, sizeof(uint32_t) * n,
                                    cudaMemcpyDeviceToDevice, st));
            out.iterations = it;
            out.sse = sse;
        }
    }
    JB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace jb
