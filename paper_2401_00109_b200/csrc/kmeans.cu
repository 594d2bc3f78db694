// kmeans.cu — sampled k-means++ on sm_100a (clustering.hpp:59-275).
//
//  * std::mt19937_64 generated on device; uniform_int / uniform_real mapped
//    exactly as libstdc++ (GCC 13) does: 128-bit Lemire downscaling with its
//    rejection loop, and generate_canonical = double(x) / 2^64.
//  * sample_indices (partial Fisher-Yates, :74-85) resolved in parallel:
//    idx[i] = value at position j_i just before swap i, recovered from the
//    "last earlier swap that touched this position" chains after one stable
//    radix sort of (j_i, i).
//  * the points are put in Morton order once; warp tiles of 128 consecutive
//    points then cover small boxes.
//  * d2_seed (:92-131): per round one tile pass (D^2 min-update, skipping
//    every tile whose box cannot beat its current max D^2; exact deltas of
//    per-original-block 128-bit fixed-point partial sums) and one
//    single-block pick in ORIGINAL sample order. The engine draw cursor lives
//    on device, so the k rounds run without host round trips.
//  * lloyd_once (:200-220): per tile, the exact candidate centers of the
//    tile's box, then nearest_center over them with the exact tie rule;
//    cluster sums maintained incrementally as exact fixed-point integers
//    (only points whose label changed contribute), empty-cluster repair
//    exactly as update_means (:181-197).
#include <cub/cub.cuh>

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "jb_device.hpp"
#include "jb_grid.cuh"
#include "jb_rowgrid.cuh"

#include <cooperative_groups.h>

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

// Multi-CTA engine: CTA c produces draws [c*b, (c+1)*b). Its starting
// window (x_{cb} .. x_{cb+311}) is p(A) applied to the seeded window, p the
// build-time jump polynomial t^(cb) mod phi (mt64_jump.c): one table entry
// when SUB == 1, else the product of a coarse jump (floor(c/SUB)*SUB*b) and
// a fine one ((c%SUB)*b), applied in turn. Applying a polynomial is the XOR
// of the windows x_{i..i+311} over its set coefficients i (64 batches of 312
// windows; only set bits are visited). The 31 low bits of the window's first
// word may differ from the sequential engine, but the twist never reads
// them. buf[312+i] = twist(buf[i], buf[i+1], buf[i+156]) is x_{k+312} =
// f(x_k, x_{k+1}, x_{k+156}) on a 624-word sliding buffer.
__global__ void __launch_bounds__(320) k_mt_jump_generate(uint64_t seed, uint64_t count,
                                                          uint64_t b, int SUB,
                                                          const uint64_t* __restrict__ jump,
                                                          const uint64_t* __restrict__ sub,
                                                          uint64_t* __restrict__ out) {
    __shared__ uint64_t buf[624];
    __shared__ uint64_t acc[312];
    __shared__ uint64_t gbits[312];
    const int t = threadIdx.x;
    const uint64_t start = (uint64_t)blockIdx.x * b;
    if (start >= count) return;
    const uint64_t nout = min(b, count - start);
    if (t == 0) {
        buf[0] = seed;
        for (int i = 1; i < 312; ++i)
            buf[i] = 6364136223846793005ULL * (buf[i - 1] ^ (buf[i - 1] >> 62)) + (uint64_t)i;
    }
    __syncthreads();
    auto advance = [&]() {  // buf[312..623] from buf[0..311]
        if (t < 156) buf[312 + t] = mt_twist(buf[t], buf[t + 1], buf[t + 156]);
        __syncthreads();
        if (t >= 156 && t < 312) buf[312 + t] = mt_twist(buf[t], buf[t + 1], buf[t + 156]);
        __syncthreads();
    };
    auto slide = [&]() {  // buf[0..311] = buf[312..623]
        uint64_t v = 0;
        if (t < 312) v = buf[312 + t];
        __syncthreads();
        if (t < 312) buf[t] = v;
        __syncthreads();
    };
    auto apply = [&](const uint64_t* __restrict__ poly) {  // buf[0..311] := poly(A) buf
        if (t < 312) {
            gbits[t] = poly[t];
            acc[t] = 0;
        }
        __syncthreads();
        for (int bb = 0; bb < 64; ++bb) {
            advance();
            if (t < 312) {
                uint64_t a = acc[t];
                const int b0 = 312 * bb, b1 = min(b0 + 312, 19937);
                for (int bit = b0; bit < b1;) {  // set coefficients in [b0, b1)
                    const int sh = bit & 63, take = min(64 - sh, b1 - bit);
                    uint64_t m = gbits[bit >> 6] >> sh;
                    if (take < 64) m &= (1ULL << take) - 1ULL;
                    while (m) {
                        const int k = __ffsll((long long)m) - 1;
                        m &= m - 1ULL;
                        a ^= buf[bit - b0 + k + t];
                    }
                    bit += take;
                }
                acc[t] = a;
            }
            __syncthreads();
            slide();
        }
        if (t < 312) buf[t] = acc[t];
        __syncthreads();
    };
    if (SUB == 1) {
        if (blockIdx.x > 0) apply(sub + (size_t)blockIdx.x * 312);
    } else {
        const int big = (int)(blockIdx.x / SUB), small = (int)(blockIdx.x % SUB);
        if (big > 0) apply(jump + (size_t)big * 312);
        if (small > 0) apply(sub + (size_t)small * 312);
    }
    for (uint64_t base = 0; base < nout; base += 312) {
        advance();
        if (t < 312 && base + t < nout) out[start + base + t] = mt_temper(buf[312 + t]);
        slide();
    }
}

// libstdc++ _S_nd<unsigned __int128> on the host (distributed seeding)
inline bool lemire_host(uint64_t x, uint64_t erange, uint64_t& r) {
    const u128 prod = (u128)x * erange;
    const uint64_t low = (uint64_t)prod;
    r = (uint64_t)(prod >> 64);
    if (low < erange) {
        const uint64_t thresh = (0 - erange) % erange;
        if (low < thresh) return false;
    }
    return true;
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
                         int nbp, uint32_t* __restrict__ j_out, uint32_t* __restrict__ vals,
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
        j_out[i] = (uint32_t)(i + r);  // < n < 2^32
        vals[i] = (uint32_t)i;
    }
}

// P is pre-filled with "none": only the (few) swaps that share their j with an
// earlier swap are written
__global__ void k_fy_links(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                           uint64_t S, uint32_t* __restrict__ P, uint32_t* __restrict__ L) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < S;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[r];
        const uint32_t i = vals[r];
        const bool same_prev = r > 0 && keys[r - 1] == key;
        if (same_prev) P[i] = vals[r - 1];
        const bool group_last = (r + 1 == S) || keys[r + 1] != key;
        if (group_last && key < S) {
            // last swap (< key) that wrote position `key`
            if ((uint64_t)i < key) L[key] = i;
            else L[key] = same_prev ? vals[r - 1] : 0xFFFFFFFFu;
        }
    }
}

__global__ void k_fy_resolve(const uint32_t* __restrict__ j, const uint32_t* __restrict__ P,
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
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + tb - 1) / tb, (uint64_t)num_sms() * per_sm));
}

}  // namespace

namespace {
// jump tables produced by mt64_jump at build time, next to libjabba_b200.so
struct JumpTable {
    uint64_t B = 0, count = 0;
    uint64_t* d = nullptr;  // device copy (process lifetime)
};
struct JumpTables {
    bool tried = false;
    int device = -1;
    JumpTable big, sub;  // sub: SUB = big.B / sub.B jumps inside one big block
};
JumpTables g_jump;
std::mutex g_jump_mu;

bool load_jump(const std::string& path, JumpTable& jt) {
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) return false;
    uint64_t hdr[4];
    std::vector<uint64_t> tab;
    bool ok = fread(hdr, 8, 4, f) == 4 && hdr[0] == 0x4A4D54364A4D5031ULL && hdr[3] == 312;
    if (ok) {
        tab.resize(hdr[2] * 312);
        ok = fread(tab.data(), 8, tab.size(), f) == tab.size();
    }
    fclose(f);
    if (!ok) return false;
    if (cudaMalloc((void**)&jt.d, tab.size() * 8) != cudaSuccess) {
        jt.d = nullptr;
        return false;
    }
    cudaMemcpy(jt.d, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice);
    jt.B = hdr[1];
    jt.count = hdr[2];
    return true;
}

const JumpTables* jump_tables() {
    std::lock_guard<std::mutex> lk(g_jump_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_jump.tried && g_jump.device == dev) return g_jump.big.d ? &g_jump : nullptr;
    g_jump.tried = true;
    g_jump.device = dev;
    g_jump.big = JumpTable{};
    g_jump.sub = JumpTable{};
    Dl_info info;
    if (!dladdr((void*)&jump_tables, &info) || !info.dli_fname) return nullptr;
    std::string dir(info.dli_fname);
    dir = dir.substr(0, dir.rfind('/') + 1);
    if (!load_jump(dir + "mt64_jump.bin", g_jump.big)) return nullptr;
    if (!load_jump(dir + "mt64_jump_small.bin", g_jump.sub) || g_jump.sub.B == 0 ||
        g_jump.big.B % g_jump.sub.B || g_jump.big.B / g_jump.sub.B > g_jump.sub.count)
        g_jump.sub = JumpTable{};  // big blocks only
    return &g_jump;
}
}  // namespace

void mt19937_64_generate(uint64_t seed, uint64_t count, DArr<uint64_t>& out, cudaStream_t st) {
    out.alloc(count, st);
    const JumpTables* jt = jump_tables();
    JB_PROF("mt19937_64", st);
    if (jt && jt->sub.d && (count + jt->sub.B - 1) / jt->sub.B <= jt->sub.count) {
        // one fine jump per CTA: ~340 CTAs of 2^18 draws for config 4
        const int ctas = (int)((count + jt->sub.B - 1) / jt->sub.B);
        k_mt_jump_generate<<<ctas, 320, 0, st>>>(seed, count, jt->sub.B, 1, jt->big.d, jt->sub.d,
                                                 out.p);
    } else if (jt && (count + jt->big.B - 1) / jt->big.B <= jt->big.count) {
        // coarse + fine jumps (fine table present) or coarse blocks only
        // (SUB == 1 with the coarse table in the fine slot: coarse blocks only)
        const int SUB = jt->sub.d ? (int)(jt->big.B / jt->sub.B) : 1;
        const uint64_t b = jt->big.B / SUB;
        const int ctas = (int)((count + b - 1) / b);
        k_mt_jump_generate<<<ctas, 320, 0, st>>>(seed, count, b, SUB, jt->big.d,
                                                 SUB > 1 ? jt->sub.d : jt->big.d, out.p);
    } else {  // no table (or beyond it): one CTA walks the engine
        k_mt_generate<<<1, 320, 0, st>>>(seed, count, out.p);
    }
    JB_LAUNCH_CHECK();
}

uint64_t sample_indices_device(uint64_t n, uint64_t S, const uint64_t* d_raw, uint64_t raw_count,
                               DArr<uint64_t>& idx, cudaStream_t st, SampleOrder* jorder) {
    if (n >= (1ULL << 32)) throw Error(INVALID_INPUT, "sampling: more than 2^32 pieces");
    DArr<uint32_t> j(S, st), keys_s(S, st);  // j_i < n < 2^32
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
    while (end_bit < 32 && (n >> end_bit) != 0) ++end_bit;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, j.p, keys_s.p, vals.p, vals_s.p, (int64_t)S, 0,
                                    end_bit, st);
    DArr<uint8_t> tmp(tb, st);
    cub::DeviceRadixSort::SortPairs(tmp.p, tb, j.p, keys_s.p, vals.p, vals_s.p, (int64_t)S, 0,
                                    end_bit, st);
    JB_LAUNCH_CHECK();
    DArr<uint32_t> P(S, st), L(S, st);
    JB_CUDA(cudaMemsetAsync(L.p, 0xFF, sizeof(uint32_t) * S, st));
    JB_CUDA(cudaMemsetAsync(P.p, 0xFF, sizeof(uint32_t) * S, st));
    k_fy_links<<<grid_cap(S), 256, 0, st>>>(keys_s.p, vals_s.p, S, P.p, L.p);
    JB_LAUNCH_CHECK();
    idx.alloc(S, st);
    {
        JB_PROF("sample_fy_resolve", st);
        k_fy_resolve<<<grid_cap(S), 256, 0, st>>>(j.p, P.p, L.p, S, idx.p);
    }
    JB_LAUNCH_CHECK();
    if (jorder) {
        jorder->j = std::move(keys_s);
        jorder->i = std::move(vals_s);
    }
    return S + total_shift;
}

// ---------------------------------------------------------------------------
// Spatial order of the k-means points.
//
// The points are visited in Morton (Z) order so that every warp tile of
// TILE consecutive points covers a small box. This is a pure re-ordering:
// labels, sums (exact integers) and the convergence test are order
// independent, the D^2 pick keeps the ORIGINAL sample order through exact
// per-original-block partial sums, and every tie-break that depends on an
// index (lowest index on equal distance) uses the original index.

namespace {

constexpr int TILE = 128;  // points per warp tile
constexpr int D2_R = 2048; // original-order elements per partial-sum block

__device__ __forceinline__ uint32_t spread16(uint32_t v) {
    v &= 0xFFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

// Morton keys of the sample points; also gathers the points (and their
// piece lengths) into sample order, so the sorted gather reads a compact
// array instead of chasing idx into the full point array again.
__global__ void k_morton(const PtsView pv, const uint64_t* __restrict__ idx,
                         int64_t n, double x0, double sx, double y0, double sy,
                         uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                         double2* __restrict__ cpts, const int32_t* __restrict__ len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t src = idx ? idx[i] : (uint64_t)i;
        const double2 p = pv.at(src);
        // with piece lengths the record carries (length, y): x is the length's
        // row coordinate (pv.at's expression), recomputed in the sorted gather
        cpts[i] = len ? make_double2((double)len[src], p.y) : p;
        const uint32_t qx = (uint32_t)fmin(fmax((p.x - x0) * sx, 0.0), 65535.0);
        const uint32_t qy = (uint32_t)fmin(fmax((p.y - y0) * sy, 0.0), 65535.0);
        keys[i] = spread16(qx) | (spread16(qy) << 1);
        vals[i] = (uint32_t)i;
    }
}

// one random 16-byte record read per point (plus the pos scatter)
__global__ void k_sorted_gather(const double2* __restrict__ cpts, const uint32_t* __restrict__ orig,
                                int64_t n, double2* __restrict__ spts, uint32_t* __restrict__ pos,
                                double scl, double sl, int32_t* __restrict__ slen) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t o = orig[r];
        const double2 c = cpts[o];
        if (slen) {
            const int32_t l = (int32_t)c.x;
            spts[r] = make_double2(scl * (double)l / sl, c.y);
            slen[r] = l;
        } else {
            spts[r] = c;
        }
        pos[o] = (uint32_t)r;
    }
}

// Spatial pass in swap-target order (SampleOrder), for points on the row
// grid's vertical lines: the r-th entry is swap i = order_i[r]; the first of
// a run of equal targets has idx[i] = j (no earlier swap touched position j:
// k_fy_links), the rest take the resolved idx[i]. Piece reads follow
// ascending j, so len/inc stream instead of two random reads per point. The
// key orders by (piece length, y): every tile lies on one line (x is a
// function of the length) with the smallest y extent a sort can give. The
// (y, len, i) record rides through the radix sort as its value, so the
// sorted order needs no random gather.
struct SRec {
    double y;
    int32_t len;
    uint32_t i;
};

__global__ void k_rowkey_jorder(const PtsView pv, const uint64_t* __restrict__ idx,
                                const uint32_t* __restrict__ oj, const uint32_t* __restrict__ oi,
                                int64_t n, int qbits, uint32_t lcap, double y0, double sy,
                                uint32_t* __restrict__ keys, SRec* __restrict__ rec) {
    const double qmax = (double)((1u << qbits) - 1u);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = oj[r], i = oi[r];
        const bool first = r == 0 || oj[r - 1] != j;
        const uint64_t src = first ? (uint64_t)j : idx[i];
        const int32_t l = pv.len[src];
        const double y = div_by(pv.inc[src], pv.si, pv.rsi);  // pv.at's y
        rec[r] = SRec{y, l, i};
        const uint32_t qy = (uint32_t)fmin(fmax((y - y0) * sy, 0.0), qmax);
        keys[r] = (min((uint32_t)l, lcap) << qbits) | qy;
    }
}

// sorted records -> points (pv.at's x from the length), lengths, original
// sample positions, and the inverse permutation
__global__ void k_rec_unpack(const SRec* __restrict__ srec, int64_t n, double2* __restrict__ spts,
                             uint32_t* __restrict__ orig, uint32_t* __restrict__ pos, double scl,
                             double sl, int32_t* __restrict__ slen) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const SRec c = srec[s];
        spts[s] = make_double2(scl * (double)c.len / sl, c.y);
        slen[s] = c.len;
        orig[s] = c.i;
    }
}

// pos = inverse of orig, scattered in passes over ranges [lo, hi) of the
// original index small enough to stay resident in L2 (the full 4n-byte
// scatter would miss to DRAM on every 4-byte write)
__global__ void k_pos_scatter(const uint32_t* __restrict__ orig, int64_t n, uint32_t lo,
                              uint32_t hi, uint32_t* __restrict__ pos) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t o = orig[s];
        if (o >= lo && o < hi) pos[o] = (uint32_t)s;
    }
}

// box = (x0, x1, y0, y1)
__global__ void k_tile_boxes(const double2* __restrict__ spts, int64_t n,
                             double4* __restrict__ tbox, const int32_t* __restrict__ slen,
                             int32_t* __restrict__ tlen) {
    const int lane = threadIdx.x & 31;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < ntiles;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
        int lmin = 0x7FFFFFFF, lmax = -1;
        for (int i = 0; i < TILE / 32; ++i) {
            const int64_t r = t * TILE + i * 32 + lane;
            if (r < n) {
                const double2 p = spts[r];
                x0 = fmin(x0, p.x);
                x1 = fmax(x1, p.x);
                y0 = fmin(y0, p.y);
                y1 = fmax(y1, p.y);
                if (slen) {
                    lmin = min(lmin, slen[r]);
                    lmax = max(lmax, slen[r]);
                }
            }
        }
        if (slen) {  // the tile's common piece length, or 0
            lmin = __reduce_min_sync(0xffffffffu, lmin);
            lmax = __reduce_max_sync(0xffffffffu, lmax);
            if (lane == 0) tlen[t] = lmin == lmax ? lmin : 0;
        }
        for (int o = 16; o > 0; o >>= 1) {
            x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, o));
            x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, o));
            y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, o));
            y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, o));
        }
        if (lane == 0) tbox[t] = make_double4(x0, x1, y0, y1);
    }
}

// Squared distance bounds between center c and box b. Each carries at most
// ~4 ulps of relative rounding error, which the 1e-12 margins below absorb:
// a center is dropped only when for EVERY point of the box its rounded
// reference distance (dx*dx+dy*dy, no FMA) is strictly larger than that of
// the center realising the min-max bound -- so it can be neither the
// argmin nor a lower-index tie.
__device__ __forceinline__ void box_d2(double cx, double cy, const double4& b, double& dmin2,
                                       double& dmax2) {
    const double ex = fmax(fmax(b.x - cx, cx - b.y), 0.0);
    const double ey = fmax(fmax(b.z - cy, cy - b.w), 0.0);
    dmin2 = ex * ex + ey * ey;
    const double fx = fmax(fabs(b.x - cx), fabs(b.y - cx));
    const double fy = fmax(fabs(b.z - cy), fabs(b.w - cy));
    dmax2 = fx * fx + fy * fy;
}

constexpr double kKeepMargin = 1e-12;

// block-wide exclusive scan of int128 values (blockDim.x a multiple of 32)
__device__ __forceinline__ i128 block_exscan_i128(i128 v, i128* total,
                                                  unsigned long long* s_lo,
                                                  unsigned long long* s_hi) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned long long lo = (unsigned long long)(u128)v, hi = (unsigned long long)((u128)v >> 64);
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long plo = __shfl_up_sync(0xffffffffu, lo, o);
        const unsigned long long phi = __shfl_up_sync(0xffffffffu, hi, o);
        if (lane >= o) {
            const unsigned long long nlo = lo + plo;
            hi = hi + phi + (nlo < lo ? 1ULL : 0ULL);
            lo = nlo;
        }
    }
    if (lane == 31) {
        s_lo[w] = lo;
        s_hi[w] = hi;
    }
    __syncthreads();
    if (w == 0) {
        const bool in = lane < (int)(blockDim.x >> 5);
        unsigned long long a = in ? s_lo[lane] : 0ULL, b = in ? s_hi[lane] : 0ULL;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long plo = __shfl_up_sync(0xffffffffu, a, o);
            const unsigned long long phi = __shfl_up_sync(0xffffffffu, b, o);
            if (lane >= o) {
                const unsigned long long nlo = a + plo;
                b = b + phi + (nlo < a ? 1ULL : 0ULL);
                a = nlo;
            }
        }
        s_lo[lane] = a;  // inclusive warp prefix
        s_hi[lane] = b;
    }
    __syncthreads();
    const i128 incl = (i128)(((u128)hi << 64) | (u128)lo);
    const i128 wpre = w > 0 ? (i128)(((u128)s_hi[w - 1] << 64) | (u128)s_lo[w - 1]) : (i128)0;
    *total = (i128)(((u128)s_hi[31] << 64) | (u128)s_lo[31]);
    __syncthreads();
    return wpre + incl - v;
}

// ---------------------------------------------------------------------------
// D^2 seeding (d2_seed clustering.hpp:92-131)

struct SeedState {
    uint64_t cursor;    // next engine draw
    int64_t last;       // ORIGINAL index of the latest center
    int32_t degenerate; // a total == 0 round happened
    int32_t pad;
};

// First center: uniform_int(0, n-1) (clustering.hpp:103-104).
__global__ void k_pick_first(const uint64_t* __restrict__ raw, uint64_t n, SeedState* ss,
                             int64_t* __restrict__ chosen) {
    uint64_t cur = ss->cursor, r;
    while (!lemire(raw[cur], n, r)) ++cur;
    ss->cursor = cur + 1;
    ss->last = (int64_t)r;
    chosen[0] = (int64_t)r;
}

// D^2 round, pass 1 (thread per tile): a tile needs work only if some point
// of its box can come closer to the new center than the tile's current max
// d2; every other tile keeps all its d2 (the rounded distances of its points
// are all > max d2 >= d2, so std::min leaves them unchanged).
// tile boxes for the D^2 cull in fp32, rounded outward (a superset box): the
// cull reads 20 B per tile instead of 40; with tmax rounded up, the test can
// only keep more tiles, never skip one the exact test keeps
__global__ void k_cull_boxes(const double4* __restrict__ tbox, int64_t ntiles,
                             float4* __restrict__ cbox) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        const double4 b = tbox[t];
        cbox[t] = make_float4(__double2float_rd(b.x), __double2float_ru(b.y),
                              __double2float_rd(b.z), __double2float_ru(b.w));
    }
}

__global__ void k_d2_cull(const float4* __restrict__ cbox, const float* __restrict__ tmax,
                          int64_t ntiles, const double2* __restrict__ spts,
                          const uint32_t* __restrict__ pos, const SeedState* __restrict__ ss,
                          uint32_t* __restrict__ work, unsigned long long* __restrict__ nwork,
                          const double2* __restrict__ cur) {
    const double2 c = cur ? *cur : spts[pos[ss->last]];
    const int lane = threadIdx.x & 31;
    constexpr int U = 4;  // tiles per thread per pass, loads issued together
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count (t0 - lane is the warp's first tile)
    for (int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t0 - lane < ntiles;
         t0 += U * stride) {
        float4 f[U];
        float tm[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t t = t0 + u * stride;
            f[u] = t < ntiles ? cbox[t] : make_float4(0.f, 0.f, 0.f, 0.f);
            tm[u] = t < ntiles ? tmax[t] : -INFINITY;  // -inf: never needed
        }
        unsigned m[U];
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double dmin2, dmax2;
            box_d2(c.x, c.y, make_double4(f[u].x, f[u].y, f[u].z, f[u].w), dmin2, dmax2);
            m[u] = __ballot_sync(0xffffffffu, !(dmin2 * (1.0 - kKeepMargin) > (double)tm[u]));
            cnt += __popc(m[u]);
        }
        if (!cnt) continue;  // warp-uniform
        // one atomic per warp and pass (a per-tile atomic on one counter serialises)
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(nwork, (unsigned long long)cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if ((m[u] >> lane) & 1u)
                work[base + __popc(m[u] & ((1u << lane) - 1u))] = (uint32_t)(t0 + u * stride);
            base += __popc(m[u]);
        }
    }
}

// D^2 round, pass 2 (warp per listed tile; init: every tile): d2 = min(d2,
// dist2(p, c_last)), the tile's new max d2, and exact deltas of the
// per-ORIGINAL-block partial sums (the pick scans in sample order).
__global__ void __launch_bounds__(256) k_d2_tiles(
    const double2* __restrict__ spts, const uint32_t* __restrict__ orig,
    const uint32_t* __restrict__ pos, int64_t n, const uint32_t* __restrict__ work,
    const unsigned long long* __restrict__ nwork, float* __restrict__ tmax,
    double* __restrict__ d2s, const SeedState* __restrict__ ss, int init, int E,
    unsigned long long* __restrict__ part, const double2* __restrict__ cur,
    const uint32_t* __restrict__ gkey, unsigned long long* __restrict__ diag, int limbs44 = 0) {
    // cur: center given directly (distributed fit); gkey: partial-sum block
    // key per sorted point (global sample position) instead of orig; diag:
    // tiles updated (diagnostics); limbs44: the init round's partials as
    // k_d2_seed's (bits 0-43, bits 44-107) limbs, fire-and-forget REDs
    const int lane = threadIdx.x & 31;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    const int64_t nw = init ? ntiles : (int64_t)*nwork;
    if (diag && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(diag, (unsigned long long)nw);
    const double2 c = cur ? *cur : spts[pos[ss->last]];
    const uint32_t* key = gkey ? gkey : orig;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t t = init ? w : (int64_t)work[w];
        double2 p[TILE / 32];
        double old[TILE / 32];
        uint32_t o[TILE / 32];
#pragma unroll
        for (int i = 0; i < TILE / 32; ++i) {
            const int64_t r = t * TILE + i * 32 + lane;
            if (r < n) {
                p[i] = spts[r];
                old[i] = init ? 0.0 : d2s[r];
                o[i] = key[r];
            }
        }
        double mx = 0.0;
#pragma unroll
        for (int i = 0; i < TILE / 32; ++i) {
            const int64_t r = t * TILE + i * 32 + lane;
            if (r >= n) break;
            const double dd = dist2(p[i].x, p[i].y, c.x, c.y);
            double v;
            if (init) {
                v = dd;
                d2s[r] = v;
                if (part && limbs44) {
                    const u128 f = (u128)fx_from_double(v, E);
                    unsigned long long* q2 = part + 2 * (o[i] / D2_R);
                    red_add_u64(q2, (unsigned long long)f & ((1ULL << 44) - 1));
                    red_add_u64(q2 + 1, (unsigned long long)(f >> 44));
                } else if (part) {
                    fx_atomic_add(part + 2 * (o[i] / D2_R), fx_from_double(v, E));
                }
            } else {
                v = old[i];
                if (dd < v) {  // std::min(d2, dd)
                    fx_atomic_add(part + 2 * (o[i] / D2_R),
                                  fx_from_double(dd, E) - fx_from_double(v, E));
                    v = dd;
                    d2s[r] = v;
                }
            }
            mx = fmax(mx, v);
        }
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        if (lane == 0) tmax[t] = __double2float_ru(mx);  // an upper bound for the cull
    }
}

constexpr int PICK_TB = 1024;

// warp-inclusive scan of int128 values (exact: integer adds with carries)
__device__ __forceinline__ i128 warp_incl_scan_i128(i128 v) {
    const int lane = threadIdx.x & 31;
    unsigned long long lo = (unsigned long long)(u128)v, hi = (unsigned long long)((u128)v >> 64);
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long plo = __shfl_up_sync(0xffffffffu, lo, o);
        const unsigned long long phi = __shfl_up_sync(0xffffffffu, hi, o);
        if (lane >= o) {
            const unsigned long long nlo = lo + plo;
            hi = hi + phi + (nlo < lo ? 1ULL : 0ULL);
            lo = nlo;
        }
    }
    return (i128)(((u128)hi << 64) | (u128)lo);
}

__device__ __forceinline__ i128 shfl_i128(i128 v, int src) {
    const unsigned long long lo = __shfl_sync(0xffffffffu, (unsigned long long)(u128)v, src);
    const unsigned long long hi = __shfl_sync(0xffffffffu, (unsigned long long)((u128)v >> 64), src);
    return (i128)(((u128)hi << 64) | (u128)lo);
}

// One D^2 round pick: total > 0 ? weighted_index (:59-71) : first unchosen.
// Finds the original-order partial-sum block holding the crossing, then the
// element (d2 gathered through pos[]); all prefix arithmetic is exact. Warp w
// owns a contiguous range of blocks read with coalesced loads; the warp
// holding the crossing scans its range 32 blocks at a time.
__global__ void __launch_bounds__(PICK_TB) k_pick(const uint64_t* __restrict__ raw,
                                                  const double* __restrict__ d2s,
                                                  const uint32_t* __restrict__ pos, int64_t n,
                                                  int nblocks,
                                                  const unsigned long long* __restrict__ part,
                                                  int E, SeedState* ss,
                                                  int64_t* __restrict__ chosen, int c,
                                                  unsigned long long* __restrict__ nwork_reset) {
    __shared__ unsigned long long s_lo[32], s_hi[32];
    __shared__ unsigned long long s_wt_lo[32], s_wt_hi[32];
    __shared__ int s_found_block;
    __shared__ unsigned long long s_found_elem;
    __shared__ unsigned long long s_before[2];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // the next cull's counter (the previous round's k_d2_tiles, which read
    // it, finished before this launch): no separate memset per round
    if (t == 0 && nwork_reset) *nwork_reset = 0;
    constexpr int NW = PICK_TB / 32;
    const int R = ((nblocks + NW - 1) / NW + 31) & ~31;  // blocks per warp, multiple of 32
    const int b0 = min(nblocks, w * R), b1 = min(nblocks, b0 + R);
    i128 local = 0;
    // 8 independent loads in flight per lane (a plain strided loop would wait
    // one L2 round trip per block: ~42 per lane at config 4)
    for (int b = b0 + lane; b < b1; b += 32 * 8) {
        unsigned long long lo[8], hi[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int bb = b + 32 * u;
            lo[u] = bb < b1 ? part[2 * bb] : 0ULL;
            hi[u] = bb < b1 ? part[2 * bb + 1] : 0ULL;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) local += (i128)(((u128)hi[u] << 64) | (u128)lo[u]);
    }
    local = fx_warp_sum(local);  // lane 0 holds the warp's total
    if (lane == 0) {
        s_wt_lo[w] = (unsigned long long)(u128)local;
        s_wt_hi[w] = (unsigned long long)((u128)local >> 64);
    }
    if (t == 0) {
        s_found_block = 0x7FFFFFFF;
        s_found_elem = ~0ULL;
    }
    __syncthreads();
    // every warp scans the NW warp totals (cheap; no extra barrier)
    const i128 wt = (i128)(((u128)s_wt_hi[lane] << 64) | (u128)s_wt_lo[lane]);
    const i128 wincl = warp_incl_scan_i128(wt);
    const i128 total_fx = shfl_i128(wincl, 31);
    const double total = fx_to_double(total_fx, E);
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
    const i128 U = fx_from_double(u, E);               // floor(u * 2^E), u >= 0
    // the warp range holding the crossing: first warp with U < inclusive prefix
    const unsigned crossing = __ballot_sync(0xffffffffu, U < wincl);
    // that range's block sums staged in shared memory by the whole block at
    // once (one coalesced round trip), then walked by warp 0
    constexpr int STAGE = 2048;
    __shared__ unsigned long long s_rng[STAGE][2];
    const int fwb = crossing ? __ffs(crossing) - 1 : 0;
    const int r0 = min(nblocks, fwb * R), r1 = min(nblocks, r0 + R);
    const bool staged = crossing && r1 - r0 <= STAGE;
    constexpr int MAXCH = STAGE / 32;
    __shared__ unsigned long long s_chk[MAXCH][2];  // 32-block chunk sums of the staged range
    if (staged) {
        for (int q = t; q < r1 - r0; q += PICK_TB) {
            s_rng[q][0] = part[2 * (r0 + q)];
            s_rng[q][1] = part[2 * (r0 + q) + 1];
        }
    }
    __syncthreads();
    const int nchk = (r1 - r0 + 31) / 32;
    if (staged) {  // one warp per chunk sum, all in parallel
        for (int j = w; j < nchk; j += NW) {
            const int q = 32 * j + lane;
            const i128 v = q < r1 - r0 ? (i128)(((u128)s_rng[q][1] << 64) | s_rng[q][0]) : (i128)0;
            const i128 cs = fx_warp_sum(v);
            if (lane == 0) {
                s_chk[j][0] = (unsigned long long)(u128)cs;
                s_chk[j][1] = (unsigned long long)((u128)cs >> 64);
            }
        }
    }
    __syncthreads();
    if (w == 0 && crossing) {  // warp 0 resolves the block inside that range
        const int fw = __ffs(crossing) - 1;
        const i128 prev = shfl_i128(wincl, fw > 0 ? fw - 1 : 0);
        i128 run = fw > 0 ? prev : (i128)0;  // exclusive prefix of warp fw's range
        const int c0 = min(nblocks, fw * R), c1 = min(nblocks, c0 + R);
        int start = c0;
        if (staged) {  // the chunk holding the crossing, from the chunk sums
            int jf = -1;
            for (int j0 = 0; j0 < nchk && jf < 0; j0 += 32) {
                const int j = j0 + lane;
                const i128 v = j < nchk ? (i128)(((u128)s_chk[j][1] << 64) | s_chk[j][0]) : (i128)0;
                const i128 incl = warp_incl_scan_i128(v);
                const unsigned hit = __ballot_sync(0xffffffffu, j < nchk && U < run + incl);
                if (hit) {
                    const int hl = __ffs(hit) - 1;
                    jf = j0 + hl;
                    run += shfl_i128(incl, hl) - shfl_i128(v, hl);
                } else {
                    run += shfl_i128(incl, 31);
                }
            }
            start = jf >= 0 ? c0 + 32 * jf : c1;
        }
        for (int bb = start; bb < c1; bb += 32) {
            const int b = bb + lane;
            const i128 v = b >= c1 ? (i128)0
                           : staged ? (i128)(((u128)s_rng[b - c0][1] << 64) | s_rng[b - c0][0])
                                    : fx_load(part + 2 * b);
            const i128 incl = warp_incl_scan_i128(v);
            const unsigned hit = __ballot_sync(0xffffffffu, b < c1 && U < run + incl);
            if (hit) {
                const int hl = __ffs(hit) - 1;
                const i128 before = run + shfl_i128(incl, hl) - shfl_i128(v, hl);
                if (lane == 0) {
                    s_found_block = bb + hl;
                    s_before[0] = (unsigned long long)(u128)before;
                    s_before[1] = (unsigned long long)((u128)before >> 64);
                }
                break;
            }
            run += shfl_i128(incl, 31);
        }
    }
    __syncthreads();
    const int fb = s_found_block;
    if (fb == 0x7FFFFFFF) {
        // roundoff spill: last positive-weight index (:67-70)
        if (t == 0) {
            int64_t next = n - 1;
            for (int64_t i = n - 1; i >= 0; --i)
                if (d2s[pos[i]] > 0.0) {
                    next = i;
                    break;
                }
            chosen[c] = next;
            ss->last = next;
            ss->cursor += 1;
        }
        return;
    }
    const i128 before_block = fx_load(s_before);
    // within block fb: 1024 threads x 2 elements (original order)
    const int64_t e0 = (int64_t)fb * D2_R + 2 * t;
    i128 a = 0, bsum = 0;
    if (e0 < n) a = fx_from_double(d2s[pos[e0]], E);
    if (e0 + 1 < n) bsum = fx_from_double(d2s[pos[e0 + 1]], E);
    i128 dummy;
    const i128 ex2 = block_exscan_i128(a + bsum, &dummy, s_lo, s_hi);
    {
        const i128 before = before_block + ex2;
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


// The same pick by a thread-block CLUSTER of PC CTAs: CTA r stages its
// contiguous share of the block partials in shared memory and sums them; the
// PC range totals are exchanged through distributed shared memory; the CTA
// whose range holds u finds the block from its staged partials and the
// element inside it exactly as k_pick. One CTA read ~700 KB of partials per
// round (config 4); eight read 87 KB each, in parallel.
constexpr int PC = 8;
constexpr size_t kPickClusterSmem = 200 * 1024;  // staged partials per CTA

__global__ void __cluster_dims__(PC, 1, 1) __launch_bounds__(PICK_TB)
    k_pick_cluster(const uint64_t* __restrict__ raw, const double* __restrict__ d2s,
                   const uint32_t* __restrict__ pos, int64_t n, int nblocks,
                   const unsigned long long* __restrict__ part, int E, SeedState* ss,
                   int64_t* __restrict__ chosen, int c, unsigned long long* __restrict__ nwork_reset) {
    namespace cgx = cooperative_groups;
    cgx::cluster_group cl = cgx::this_cluster();
    extern __shared__ unsigned long long s_part[];  // my blocks: (lo, hi) pairs
    __shared__ unsigned long long s_lo[32], s_hi[32];
    __shared__ unsigned long long s_tot[2];
    __shared__ int s_fb;
    __shared__ unsigned long long s_before[2];
    __shared__ unsigned long long s_found_elem;
    const int t = threadIdx.x, lane = t & 31;
    const int r = (int)cl.block_rank();
    const int per = (nblocks + PC - 1) / PC;
    const int b0 = min(nblocks, r * per), b1 = min(nblocks, b0 + per), nb = b1 - b0;
    if (r == 0 && t == 0 && nwork_reset) *nwork_reset = 0;
    // stage my partials (8 independent 16-byte loads in flight per thread)
    const ulonglong2* p2 = reinterpret_cast<const ulonglong2*>(part) + b0;
    ulonglong2* s2 = reinterpret_cast<ulonglong2*>(s_part);
    for (int q0 = t; q0 < nb; q0 += PICK_TB * 8) {
        ulonglong2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * PICK_TB;
            v[u] = q < nb ? p2[q] : make_ulonglong2(0ULL, 0ULL);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int q = q0 + u * PICK_TB;
            if (q < nb) s2[q] = v[u];
        }
    }
    __syncthreads();
    // thread t owns blocks [b0 + t*qn, ...) of my range: its sum, then a block scan
    const int qn = (nb + PICK_TB - 1) / PICK_TB;
    const int q0 = min(nb, t * qn), q1 = min(nb, q0 + qn);
    i128 mine = 0;
    for (int q = q0; q < q1; ++q) mine += (i128)(((u128)s2[q].y << 64) | (u128)s2[q].x);
    i128 range_total;
    const i128 excl = block_exscan_i128(mine, &range_total, s_lo, s_hi);
    if (t == 0) {
        s_tot[0] = (unsigned long long)(u128)range_total;
        s_tot[1] = (unsigned long long)((u128)range_total >> 64);
        s_fb = 0x7FFFFFFF;
        s_found_elem = ~0ULL;
    }
    cl.sync();
    // the PC range totals (DSMEM): prefix, total, u -- identical on every CTA
    i128 pre_r = 0, total_fx = 0;
    int rc = -1;
    for (int q = 0; q < PC; ++q) {
        const unsigned long long* rt = cl.map_shared_rank(s_tot, q);
        const i128 v = (i128)(((u128)rt[1] << 64) | (u128)rt[0]);
        if (q < r) pre_r += v;
        total_fx += v;
    }
    const double total = fx_to_double(total_fx, E);
    bool spill = false;
    i128 U = 0;
    if (total > 0.0) {
        const uint64_t x = raw[ss->cursor];
        double canon = __ull2double_rn(x) * 0x1p-64;  // generate_canonical<double,53>
        if (canon >= 1.0) canon = 0x1.fffffffffffffp-1;
        const double u = canon * total + 0.0;  // uniform_real(0, total)
        U = fx_from_double(u, E);
        i128 run = 0;
        for (int q = 0; q < PC && rc < 0; ++q) {
            const unsigned long long* rt = cl.map_shared_rank(s_tot, q);
            run += (i128)(((u128)rt[1] << 64) | (u128)rt[0]);
            if (U < run) rc = q;
        }
        spill = rc < 0;
    }
    cl.sync();  // no CTA leaves while its totals may still be read
    if (!(total > 0.0) || spill) {  // rare paths, serially as k_pick
        if (r == 0 && t == 0) {
            int64_t next;
            if (!(total > 0.0)) {  // every remaining point duplicates a center (:120-124)
                next = 0;
                for (;;) {
                    bool taken = false;
                    for (int q = 0; q < c; ++q) taken |= chosen[q] == next;
                    if (!taken) break;
                    ++next;
                }
                ss->degenerate = 1;
            } else {  // roundoff spill: last positive-weight index (:67-70)
                next = n - 1;
                for (int64_t i = n - 1; i >= 0; --i)
                    if (d2s[pos[i]] > 0.0) {
                        next = i;
                        break;
                    }
                ss->cursor += 1;
            }
            chosen[c] = next;
            ss->last = next;
        }
        return;
    }
    if (r != rc) return;
    // my range holds the crossing: the owning thread finds the block
    const i128 lo_t = pre_r + excl;
    if (U >= lo_t && U < lo_t + mine) {
        i128 run = lo_t;
        for (int q = q0; q < q1; ++q) {
            const i128 v = (i128)(((u128)s2[q].y << 64) | (u128)s2[q].x);
            if (U < run + v) {
                s_fb = b0 + q;
                s_before[0] = (unsigned long long)(u128)run;
                s_before[1] = (unsigned long long)((u128)run >> 64);
                break;
            }
            run += v;
        }
    }
    __syncthreads();
    const int fb = s_fb;
    if (fb == 0x7FFFFFFF) {  // cannot happen for U < total; stay safe: spill rule
        if (t == 0) {
            int64_t next = n - 1;
            for (int64_t i = n - 1; i >= 0; --i)
                if (d2s[pos[i]] > 0.0) {
                    next = i;
                    break;
                }
            chosen[c] = next;
            ss->last = next;
            ss->cursor += 1;
        }
        return;
    }
    const i128 before_block = fx_load(s_before);
    const int64_t e0 = (int64_t)fb * D2_R + 2 * t;  // 1024 threads x 2 elements
    i128 a = 0, bsum = 0;
    if (e0 < n) a = fx_from_double(d2s[pos[e0]], E);
    if (e0 + 1 < n) bsum = fx_from_double(d2s[pos[e0 + 1]], E);
    i128 dummy;
    const i128 ex2 = block_exscan_i128(a + bsum, &dummy, s_lo, s_hi);
    {
        const i128 before = before_block + ex2;
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
    (void)lane;
}

// ---- persistent D^2 seeding: every round of d2_seed in ONE cooperative
// launch (clustering.hpp:112-129). Per round:
//   (1) CTA b sums its contiguous range of the original-order block
//       partials into rtot[b], keeping the partials in shared memory;
//       grid barrier;
//   (2) every CTA scans the range totals (u, total: identical everywhere)
//       and so knows the range holding the crossing; ITS CTA alone finds the
//       block (from its staged partials) and the element (d2 of the block's
//       2048 points) and publishes it through a round-tagged flag -- the
//       others wait on the flag instead of a grid barrier, so nothing
//       changes the d2 values while they are being read;
//   (3) CTA b culls its own tiles (t = b, b + G, ...: a compact set of kept
//       tiles spreads over all CTAs) against the new center and updates the
//       kept ones with its warps; grid barrier.
// Tile -> CTA ownership is static: each CTA keeps its tiles' cull boxes and
// max d2 in shared memory for the whole launch, and d2 of a tile is only
// ever written by one SM; data other CTAs wrote inside the launch is read
// with ld.global.cg (L2).
//
// Fixed point: d2 -> floor(d2 * 2^E) with E chosen so the initial total is
// < 2^107 (18 bits below the per-round path's scale, still ~2^-100 of the
// total per unit), so every block partial lies in [0, 2^107) and is known
// from its value mod 2^108. A block partial is two u64 limbs, L (bits 0-43
// of each addend) and H (bits 44-107, wrapping): a changed point adds
// (new - old) mod 2^108 as two fire-and-forget atomics, with no carry round
// trip (a (lo, hi) int128 add must learn the low word's carry). The range
// owner folds L into H every round, before any add, so L never overflows.
// The prefix arithmetic is exact on these integers, as in k_pick. If the
// total reaches 0 (every remaining point duplicates a center), the launch
// stops before that round (flag[1]) and the per-round path finishes.
#ifndef JB_D2P_TB
#define JB_D2P_TB 512  // 128 registers, no spills (1024 threads: 64 registers, 172 bytes spilled): 8.39 -> 7.93 ms; 256: 8.76
#endif
constexpr int D2P_TB = JB_D2P_TB;

struct D2Seed {
    const double2* spts;
    const uint32_t* orig;
    const uint32_t* pos;
    int64_t n;
    const float4* cbox;
    float* tmax;
    int64_t ntiles;
    double* d2s;
    const unsigned long long* part;  // (lo, hi) partials after the init round
    unsigned long long* part2;       // this launch's block partials: (L, H) limbs
    int nblocks;
    int E;
    const uint64_t* raw;
    SeedState* ss;
    int64_t* chosen;
    int k;
    unsigned long long* rtot;  // (lo, hi) per CTA
    int* flag;                 // [0] last published round (0 before launch), [1] exit round
    unsigned long long* diag;
    unsigned long long* phase;  // optional (JB_D2_PHASES): summed ns of 5 phases, CTAs 0 and 1
    int ntl;                    // tiles per CTA (shared-memory arrays)
    unsigned long long* rounds; // optional (JB_D2_PHASES): CTA 0 per round: cull+update ns, kept tiles
};

constexpr unsigned long long kM44 = (1ULL << 44) - 1;

__device__ __forceinline__ i128 ldcg_i128(const unsigned long long* p) {
    const unsigned long long lo = __ldcg(p), hi = __ldcg(p + 1);
    return (i128)(((u128)hi << 64) | (u128)lo);
}

__global__ void __launch_bounds__(D2P_TB, 1) k_d2_seed(D2Seed P) {
    namespace cgx = cooperative_groups;
    cgx::grid_group grid = cgx::this_grid();
    extern __shared__ unsigned long long s_dyn[];
    const int ntl = P.ntl;
    const int G = (int)gridDim.x, b = (int)blockIdx.x;
    const int BR = (P.nblocks + G - 1) / G;  // blocks per range
    float4* s_box = reinterpret_cast<float4*>(s_dyn);                      // my tiles' cull boxes
    unsigned long long* s_part = s_dyn + 2 * ntl;                          // my range's partials (lo, hi)
    float* s_tmax = reinterpret_cast<float*>(s_part + 2 * BR);             // my tiles' max d2
    uint32_t* s_list = reinterpret_cast<uint32_t*>(s_tmax + ntl);          // kept tiles (local)
    __shared__ unsigned long long s_lo[32], s_hi[32];
    __shared__ int s_cnt, s_rc, s_fb;
    __shared__ unsigned long long s_before[2], s_bbefore[2];
    __shared__ long long s_next;
    constexpr int NW = D2P_TB / 32;
    constexpr int EP = D2_R / D2P_TB;  // elements of a block per thread
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint64_t cursor = P.ss->cursor;
    int64_t last = P.ss->last;
    const int QB = (BR + D2P_TB - 1) / D2P_TB;  // blocks per thread
    const int r0 = min(P.nblocks, b * BR), r1 = min(P.nblocks, r0 + BR);
    const int q0 = min(r1, r0 + t * QB), q1 = min(r1, q0 + QB);
    for (int i = t; i < ntl; i += D2P_TB) {
        const int64_t tt = (int64_t)b + (int64_t)i * G;
        s_box[i] = tt < P.ntiles ? P.cbox[tt] : make_float4(0.f, 0.f, 0.f, 0.f);
        s_tmax[i] = tt < P.ntiles ? P.tmax[tt] : -INFINITY;  // -inf: never kept
    }
    unsigned long long kept = 0;
    unsigned long long tprev = 0;
    auto stamp = [&](int i) {  // JB_D2_PHASES: CTA 0 and 1 sum their phase times
        if (P.phase && t == 0 && b < 2) {
            unsigned long long v;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
            if (i > 0) atomicAdd(P.phase + 5 * b + i - 1, v - tprev);
            tprev = v;
        }
    };
    int c = 1;
    for (; c < P.k; ++c) {
        stamp(0);
        // ---- (1) my range total; partials normalised and staged ----
        i128 mine = 0;
        for (int j = q0; j < q1; ++j) {
            // (the init round wrote the same limbs: k_d2_tiles, limbs44)
            const unsigned long long L = __ldcg(P.part2 + 2 * j), H = __ldcg(P.part2 + 2 * j + 1);
            const u128 v = ((u128)L + ((u128)H << 44)) & (((u128)1 << 108) - 1);
            __stcg(P.part2 + 2 * j, (unsigned long long)v & kM44);
            __stcg(P.part2 + 2 * j + 1, (unsigned long long)(v >> 44));
            s_part[2 * (j - r0)] = (unsigned long long)v;
            s_part[2 * (j - r0) + 1] = (unsigned long long)(v >> 64);
            mine += (i128)v;
        }
        i128 my_ex;  // this thread's blocks before it in the range (kept for the pick)
        {
            i128 rt;
            my_ex = block_exscan_i128(mine, &rt, s_lo, s_hi);
            if (t == 0) {
                __stcg(P.rtot + 2 * b, (unsigned long long)(u128)rt);
                __stcg(P.rtot + 2 * b + 1, (unsigned long long)((u128)rt >> 64));
            }
        }
        stamp(1);
        grid.sync();
        stamp(2);
        // ---- (2) the pick ----
        const i128 vr = t < G ? ldcg_i128(P.rtot + 2 * t) : (i128)0;
        i128 total_fx;
        const i128 exr = block_exscan_i128(vr, &total_fx, s_lo, s_hi);
        if (total_fx == 0) break;  // uniform: the per-round path finishes
        const double total = fx_to_double(total_fx, P.E);
        const uint64_t x = P.raw[cursor];
        double canon = __ull2double_rn(x) * 0x1p-64;  // generate_canonical<double,53>
        if (canon >= 1.0) canon = 0x1.fffffffffffffp-1;
        const double u = canon * total + 0.0;  // uniform_real(0, total)
        const i128 U = fx_from_double(u, P.E);
        if (t == 0) s_rc = -1;
        __syncthreads();
        if (t < G && U >= exr && U < exr + vr) {  // unique: vr > 0 there
            s_rc = t;
            s_before[0] = (unsigned long long)(u128)exr;
            s_before[1] = (unsigned long long)((u128)exr >> 64);
        }
        __syncthreads();
        const int rc = s_rc;
        // the owner: the crossing range's CTA, or CTA 0 on a roundoff spill
        // (U >= total): the same decision on every CTA
        const int owner = rc >= 0 ? rc : 0;
        int64_t next;
        if (b == owner) {
            if (t == 0) {
                s_fb = -1;
                s_next = -1;
            }
            __syncthreads();
            if (rc >= 0) {
                i128 dummy;
                const i128 ex = fx_load(s_before) + my_ex;
                if (U >= ex && U < ex + mine) {
                    i128 run = ex;
                    for (int j = q0; j < q1; ++j) {
                        const i128 v = fx_load(s_part + 2 * (j - r0));
                        if (U < run + v) {
                            s_fb = j;
                            s_bbefore[0] = (unsigned long long)(u128)run;
                            s_bbefore[1] = (unsigned long long)((u128)run >> 64);
                            break;
                        }
                        run += v;
                    }
                }
                __syncthreads();
                const int fb = s_fb;  // found: U lies inside this range
                const int64_t e0 = (int64_t)fb * D2_R + (int64_t)EP * t;
                i128 a[EP];
                i128 ts = 0;
#pragma unroll
                for (int i = 0; i < EP; ++i) {
                    const int64_t e = e0 + i;
                    a[i] = (fb >= 0 && e < P.n) ? fx_from_double(__ldcg(P.d2s + P.pos[e]), P.E)
                                                : (i128)0;
                    ts += a[i];
                }
                const i128 ex3 = fx_load(s_bbefore) + block_exscan_i128(ts, &dummy, s_lo, s_hi);
                if (fb >= 0 && U >= ex3 && U < ex3 + ts) {
                    i128 run = ex3;
#pragma unroll
                    for (int i = 0; i < EP; ++i) {
                        run += a[i];
                        if (U < run) {
                            s_next = e0 + i;
                            break;
                        }
                    }
                }
                __syncthreads();
            }
            if (t == 0) {
                long long nx = s_next;
                if (nx < 0) {  // roundoff spill: last positive-weight index (:67-70)
                    nx = P.n - 1;
                    for (int64_t i = P.n - 1; i >= 0; --i)
                        if (__ldcg(P.d2s + P.pos[i]) > 0.0) {
                            nx = i;
                            break;
                        }
                }
                P.chosen[c] = nx;
                s_next = nx;
                __threadfence();
                atomicExch(P.flag, c);  // publish round c
            }
            __syncthreads();
            next = s_next;
        } else {
            if (t == 0) {
                while (*(volatile int*)P.flag < c) {
                }
                __threadfence();
                s_next = __ldcg((const long long*)P.chosen + c);
            }
            __syncthreads();
            next = s_next;
        }
        cursor += 1;
        last = next;
        stamp(3);
        unsigned long long t3 = 0;
        if (P.rounds && b == 0 && t == 0 && c < 1024) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
        if (c + 1 >= P.k) {
            c = P.k;
            break;
        }
        // ---- (3) cull + update my tiles against the new center ----
        const double2 cc = P.spts[P.pos[next]];
        if (t == 0) s_cnt = 0;
        __syncthreads();
        for (int i0 = 0; i0 < ntl; i0 += D2P_TB) {  // block-uniform trip count
            const int i = i0 + t;
            bool keep = false;
            if (i < ntl) {
                const float4 f = s_box[i];
                double dmin2, dmax2;
                box_d2(cc.x, cc.y, make_double4(f.x, f.y, f.z, f.w), dmin2, dmax2);
                keep = !(dmin2 * (1.0 - kKeepMargin) > (double)s_tmax[i]);
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (m) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&s_cnt, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (keep) s_list[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)i;
            }
        }
        __syncthreads();
        const int cnt = s_cnt;
        if (t == 0) kept += (unsigned long long)cnt;
        for (int li = w; li < cnt; li += NW) {
            const int il = (int)s_list[li];
            const int64_t tl = (int64_t)b + (int64_t)il * G;
            double2 p[TILE / 32];
            double old[TILE / 32];
            uint32_t o[TILE / 32];
#pragma unroll
            for (int ii = 0; ii < TILE / 32; ++ii) {
                const int64_t r = tl * TILE + ii * 32 + lane;
                if (r < P.n) {
                    p[ii] = P.spts[r];
                    old[ii] = __ldcg(P.d2s + r);
                    o[ii] = P.orig[r];
                }
            }
            double mx = 0.0;
#pragma unroll
            for (int ii = 0; ii < TILE / 32; ++ii) {
                const int64_t r = tl * TILE + ii * 32 + lane;
                if (r >= P.n) break;
                const double dd = dist2(p[ii].x, p[ii].y, cc.x, cc.y);
                double v = old[ii];
                if (dd < v) {  // std::min(d2, dd)
                    const u128 dl = (u128)(fx_from_double(dd, P.E) - fx_from_double(v, P.E));
                    unsigned long long* q2 = P.part2 + 2 * (o[ii] / D2_R);
                    red_add_u64(q2, (unsigned long long)dl & kM44);
                    red_add_u64(q2 + 1, (unsigned long long)(dl >> 44));  // bits 44-107 (mod 2^64)
                    v = dd;
                    __stcg(P.d2s + r, v);
                }
                mx = fmax(mx, v);
            }
            for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            if (lane == 0) s_tmax[il] = __double2float_ru(mx);
        }
        stamp(4);
        if (P.rounds && b == 0 && t == 0 && c < 1024) {
            unsigned long long v;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
            P.rounds[2 * c] = v - t3;
            P.rounds[2 * c + 1] = (unsigned long long)cnt;
        }
        grid.sync();
        stamp(5);
    }
    if (c < P.k) {  // early exit before round c: the tile maxima back for the per-round path
        for (int i = t; i < ntl; i += D2P_TB) {
            const int64_t tt = (int64_t)b + (int64_t)i * G;
            if (tt < P.ntiles) P.tmax[tt] = s_tmax[i];
        }
    }
    if (b == 0 && t == 0) {
        P.ss->cursor = cursor;
        P.ss->last = last;
        P.flag[1] = c;
    }
    if (t == 0 && P.diag && kept) atomicAdd(P.diag, kept);
}

// the device supports cooperative launches (cached per process)
bool coop_ok() {
    static int coop = -1;
    if (coop < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) != cudaSuccess) {
            cudaGetLastError();
            coop = 0;
        }
    }
    return coop != 0;
}

// (lo, hi) partials of every block from the current d2 (the per-round
// path's 128-bit scale), after an early exit of k_d2_seed
__global__ void k_part_rebuild(const double* __restrict__ d2s, const uint32_t* __restrict__ orig,
                               int64_t n, int E, unsigned long long* __restrict__ part) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        fx_atomic_add_small(part + 2 * (orig[r] / D2_R), (u128)fx_from_double(d2s[r], E));
}

struct D2Plan {
    int G = 0;  // 0: no persistent launch
    int ntl = 0;
    size_t smem = 0;
};

// the persistent seeding grid: one 1024-thread CTA per SM, its tiles' cull
// state and its range of partials in shared memory
D2Plan d2_plan(int64_t ntiles, int nblocks) {
    D2Plan p;
    if (!coop_ok()) return p;
    const int G = num_sms();
    if (G > D2P_TB) return p;
    const int ntl = (int)((ntiles + G - 1) / G);
    const int BR = (nblocks + G - 1) / G;
    const size_t smem = 24 * (size_t)ntl + 16 * (size_t)BR;
    if (smem > 200 * 1024) return p;
    if (cudaFuncSetAttribute(k_d2_seed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return p;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_d2_seed, D2P_TB, smem) != cudaSuccess ||
        occ < 1) {
        cudaGetLastError();
        return p;
    }
    p.G = G;
    p.ntl = ntl;
    p.smem = smem;
    return p;
}

// Rounds 1.. of d2_seed in one cooperative launch; returns the round the
// per-round path continues from (k when done; 1 when the launch failed).
uint64_t d2_seed_persistent(const D2Plan& pl, const double2* spts, const uint32_t* orig,
                            const uint32_t* pos, int64_t n, const float4* cbox, float* tmax,
                            int64_t ntiles, double* d2s, unsigned long long* part,
                            unsigned long long* part2, int nblocks,
                            int E, const uint64_t* raw, SeedState* ss, int64_t* chosen, int k,
                            unsigned long long* diag, cudaStream_t st) {
    static const bool phases = getenv("JB_D2_PHASES") != nullptr;
    const int G = pl.G;
    DArr<unsigned long long> aux(2 * G + 1 + 10 + 2048, st);  // range totals, flags, phase sums, rounds
    JB_CUDA(cudaMemsetAsync(aux.p + 2 * G, 0, 8 * (11 + 2048), st));
    int* flag = reinterpret_cast<int*>(aux.p + 2 * G);
    D2Seed a{spts, orig, pos, n, cbox, tmax, ntiles, d2s, part, part2, nblocks, E, raw, ss,
             chosen, k, aux.p, flag, diag, phases ? aux.p + 2 * G + 1 : nullptr, pl.ntl,
             phases ? aux.p + 2 * G + 11 : nullptr};
    void* args[] = {&a};
    {
        JB_PROF("d2_seed", st);
        const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_d2_seed, dim3(G),
                                                          dim3(D2P_TB), args, pl.smem, st);
        if (e != cudaSuccess) {  // cannot co-schedule: the per-round path from round 1
            cudaGetLastError();
            return 1;
        }
    }
    JB_LAUNCH_CHECK();
    int hf[2];
    JB_CUDA(cudaMemcpyAsync(hf, flag, 8, cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    if (phases) {
        unsigned long long h[10];
        JB_CUDA(cudaMemcpy(h, aux.p + 2 * G + 1, 80, cudaMemcpyDeviceToHost));
        const double r = std::max(k - 1, 1), r2 = std::max(k - 2, 1);
        for (int q = 0; q < 2; ++q)
            fprintf(stderr, "[jb] d2 phases CTA %d (us/round, G=%d): sums %.2f sync1 %.2f "
                            "pick %.2f cull+update %.2f sync2 %.2f\n",
                    q, G, h[5 * q] * 1e-3 / r, h[5 * q + 1] * 1e-3 / r, h[5 * q + 2] * 1e-3 / r,
                    h[5 * q + 3] * 1e-3 / r2, h[5 * q + 4] * 1e-3 / r2);
        std::vector<unsigned long long> hr(2048);
        JB_CUDA(cudaMemcpy(hr.data(), aux.p + 2 * G + 11, 8 * 2048, cudaMemcpyDeviceToHost));
        std::string line;
        double tot = 0, tail = 0;
        int ntail = 0;
        for (int c = 1; c < std::min(k, 1024); ++c) {
            tot += hr[2 * c] * 1e-3;
            if (c <= 12) line += " " + std::to_string((int)(hr[2 * c] * 1e-3)) + "us/" + std::to_string(hr[2 * c + 1]);
            else { tail += hr[2 * c] * 1e-3; ++ntail; }
        }
        fprintf(stderr, "[jb] d2 CTA 0 cull+update per round (us/kept tiles):%s | rounds 13..: %.2f us avg | total %.0f us\n",
                line.c_str(), ntail ? tail / ntail : 0.0, tot);
    }
    return (uint64_t)hf[1];
}

__global__ void k_copy_center(const double2* __restrict__ spts, const uint32_t* __restrict__ pos,
                              const int64_t* __restrict__ chosen, int k,
                              double* __restrict__ centers) {
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const double2 p = spts[pos[chosen[c]]];
        centers[2 * c] = p.x;
        centers[2 * c + 1] = p.y;
    }
}

// ---------------------------------------------------------------------------
// Lloyd

struct ClusterAcc {
    unsigned long long* sx;   // 3k: l3 limbs per cluster
    unsigned long long* sy;   // 3k
    unsigned long long* cnt;  // k (two's complement deltas)
};

constexpr int LL_TB = 256;

// ---- tile-level skipping --------------------------------------------------
// A tile (TILE consecutive Morton-ordered points, box tbox[t]) is SINGLE with
// center c when c is the only possible reference argmin for every point of
// the box: the union of the candidate lists of the grid cells covering the
// box is pruned again with the tile's own (much smaller) box by the same
// min-max argument (jb_grid.cuh); the survivors are a superset of the
// argmins, so one survivor decides every label. A tile that is SINGLE with
// the same center as when it was last processed holds that label on every
// point already: it is skipped without reading its points.
constexpr uint32_t MIXED = 0xFFFFFFFFu;

// Row tile (every point of one length l, so x0 == x1 == x_l): the union of
// the candidate words of the row cells covering [y0, y1], pruned again with
// the tile box. Returns false when a cell overflows or the span is long.
__device__ __forceinline__ bool row_tile_single(const RowGrid& rg, int l, const double4& b,
                                                const double* centers,
                                                uint32_t& single) {
    int iy0 = (int)((b.z - rg.y0) * rg.invh), iy1 = (int)((b.w - rg.y0) * rg.invh);
    iy0 = min(max(iy0, 0), rg.Gy - 1);
    iy1 = min(max(iy1, 0), rg.Gy - 1);
    const int nc = iy1 - iy0 + 1;
    if (nc > 8) return false;
    const unsigned long long* row =
        reinterpret_cast<const unsigned long long*>(rg.cell) + (size_t)(l - 1) * rg.Gy + iy0;
    uint64_t wv[8];  // all cell words first: independent loads
#pragma unroll
    for (int j = 0; j < 8; ++j) wv[j] = j < nc ? __ldcg(row + j) : ~0ull;
    double M = INFINITY;
    for (int j = 0; j < 8; ++j) {
        if (j >= nc) break;
        if ((wv[j] & 0xFFFF) >= kRowOverflow) return false;  // overflow / not built
        const int m = row_word_count(wv[j]);
        for (int q = 0; q < m; ++q) {
            const uint32_t c = row_word_cand(rg.spill, wv[j], q);
            double dmn, dmx;
            box_d2(centers[2 * c], centers[2 * c + 1], b, dmn, dmx);
            M = fmin(M, dmx);
        }
    }
    const double thr = M * (1.0 + kKeepMargin) + 1e-300;
    uint32_t first = MIXED;
    for (int j = 0; j < 8; ++j) {
        if (j >= nc) break;
        const int m = row_word_count(wv[j]);
        for (int q = 0; q < m; ++q) {
            const uint32_t c = row_word_cand(rg.spill, wv[j], q);
            double dmn, dmx;
            box_d2(centers[2 * c], centers[2 * c + 1], b, dmn, dmx);
            if (dmn <= thr) {
                if (first == MIXED) first = c;
                else if (c != first) {
                    single = MIXED;
                    return true;
                }
            }
        }
    }
    single = first;
    return true;
}

// Single-center test of a box b (tile or super-tile) with common piece length
// l (0: mixed): the row grid when it applies, else the 2-D grid cells.
__device__ __forceinline__ uint32_t box_single(const double4& b, int l, const CandGrid& g,
                                               const RowGrid& rg,
                                               const double* centers) {
    uint32_t single;
    if (l >= 1 && l <= rg.R && row_tile_single(rg, l, b, centers, single)) return single;
    if (g.G == 0) return MIXED;  // no 2-D grid (row grid in use)
    int ix0 = (int)((b.x - g.x0) * g.invw), ix1 = (int)((b.y - g.x0) * g.invw);
    int iy0 = (int)((b.z - g.y0) * g.invh), iy1 = (int)((b.w - g.y0) * g.invh);
    ix0 = min(max(ix0, 0), g.G - 1);
    ix1 = min(max(ix1, 0), g.G - 1);
    iy0 = min(max(iy0, 0), g.G - 1);
    iy1 = min(max(iy1, 0), g.G - 1);
    if ((ix1 - ix0 + 1) * (iy1 - iy0 + 1) > 4) return MIXED;
    double M = INFINITY;
    for (int iy = iy0; iy <= iy1; ++iy)
        for (int ix = ix0; ix <= ix1; ++ix) {
            const int cell = iy * g.G + ix;
            const int n = __ldg(g.cnt + cell);
            if (n == 0xFFFF) return MIXED;
            const uint16_t* cl = g.cand + (size_t)cell * g.cap;
            for (int j = 0; j < n; ++j) {
                const int c = __ldg(cl + j);
                double dmn, dmx;
                box_d2(centers[2 * c], centers[2 * c + 1], b, dmn, dmx);
                M = fmin(M, dmx);
            }
        }
    const double thr = M * (1.0 + kKeepMargin) + 1e-300;
    uint32_t first = MIXED;
    for (int iy = iy0; iy <= iy1; ++iy)
        for (int ix = ix0; ix <= ix1; ++ix) {
            const int cell = iy * g.G + ix;
            const int n = __ldg(g.cnt + cell);
            const uint16_t* cl = g.cand + (size_t)cell * g.cap;
            for (int j = 0; j < n; ++j) {
                const uint32_t c = __ldg(cl + j);
                double dmn, dmx;
                box_d2(centers[2 * c], centers[2 * c + 1], b, dmn, dmx);
                if (dmn <= thr) {
                    if (first == MIXED) first = c;
                    else if (c != first) return MIXED;
                }
            }
        }
    return first;
}

// box_single by a group of 8 lanes (lane `sub` takes row cell word sub, its
// <= 4 candidates): the same candidate set, the same M (fmin is exact and
// order free), the same threshold and the same dmn <= thr tests as the
// serial loop, and SINGLE iff every passing candidate is one center -- so
// the same answer with a short critical path. Every lane of the warp must
// call it (shuffles over the full mask); l and b are uniform per group.
__device__ __forceinline__ uint32_t box_single_g8(const double4& b, int l, const CandGrid& g,
                                                  const RowGrid& rg, const double* centers,
                                                  int sub) {
    bool row = l >= 1 && l <= rg.R;
    int iy0 = 0, nc = 0;
    if (row) {
        iy0 = (int)((b.z - rg.y0) * rg.invh);
        int iy1 = (int)((b.w - rg.y0) * rg.invh);
        iy0 = min(max(iy0, 0), rg.Gy - 1);
        iy1 = min(max(iy1, 0), rg.Gy - 1);
        nc = iy1 - iy0 + 1;
        row = nc <= 8;
    }
    uint64_t wv = ~0ull;
    if (row && sub < nc)
        wv = __ldcg(reinterpret_cast<const unsigned long long*>(rg.cell) + (size_t)(l - 1) * rg.Gy +
                    iy0 + sub);
    bool bad = row && sub < nc && (wv & 0xFFFF) >= kRowOverflow;
    double M = INFINITY;
    int ncand = 0;
    if (row && sub < nc && !bad) {
        ncand = row_word_count(wv);
        for (int q = 0; q < ncand; ++q) {
            const uint32_t c = row_word_cand(rg.spill, wv, q);
            double dmn, dmx;
            box_d2(centers[2 * c], centers[2 * c + 1], b, dmn, dmx);
            M = fmin(M, dmx);
        }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        M = fmin(M, __shfl_xor_sync(0xffffffffu, M, o));
        bad |= __shfl_xor_sync(0xffffffffu, (int)bad, o) != 0;
    }
    const double thr = M * (1.0 + kKeepMargin) + 1e-300;
    uint32_t cmin = MIXED, cmax = 0;  // passing candidates (cmax: c + 1)
    for (int q = 0; q < ncand; ++q) {
        const uint32_t c = row_word_cand(rg.spill, wv, q);
        double dmn, dmx;
        box_d2(centers[2 * c], centers[2 * c + 1], b, dmn, dmx);
        if (dmn <= thr) {
            cmin = min(cmin, c);
            cmax = max(cmax, c + 1);
        }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        cmin = min(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
        cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    if (row && !bad) return (cmax != 0 && cmin + 1 == cmax) ? cmin : MIXED;
    if (g.G == 0) return MIXED;
    return box_single(b, l, g, rg, centers);  // 2-D grid: every lane the serial test
}

// Super-tile check (32 consecutive tiles = 4096 points), 8 lanes each. A
// super-tile whose box is SINGLE with the center it was SINGLE with last
// time holds that label on all its points (its state is reset to MIXED
// whenever a point of it is relabeled outside this scheme, k_repair): it is
// skipped. The others are listed for k_lloyd_work. State: tlab[ntiles + s].
__device__ __forceinline__ void super_check_body(const double4* __restrict__ sbox, const int32_t* __restrict__ slenc,
                              int64_t ntiles, CandGrid g, const double* centers,
                              uint32_t* __restrict__ tlab, uint32_t* __restrict__ swork,
                              unsigned long long* __restrict__ nswork,
                              const int* __restrict__ skip_flag, int force_all, RowGrid rg,
                              int k) {
    if (skip_flag && (skip_flag[0] | skip_flag[1])) return;
    extern __shared__ double s_centers[];  // 2k: the candidate tests read them repeatedly
    if (centers != s_centers) {  // (the persistent loop passes its shared copy)
        for (int i = threadIdx.x; i < 2 * k; i += blockDim.x) s_centers[i] = centers[i];
        __syncthreads();
        centers = s_centers;
    }
    const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
    const int64_t nsuper = (ntiles + 31) / 32;
    uint32_t* stlab = tlab + ntiles;
    // 8 lanes per super-tile (box_single_g8), 4 super-tiles per warp pass
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t wstride = (((int64_t)gridDim.x * blockDim.x) >> 5) * 4;
    for (int64_t s0 = warp * 4; s0 < nsuper; s0 += wstride) {
        const int64_t sidx = s0 + grp;
        const bool valid = sidx < nsuper;
        const double4 b = valid ? sbox[sidx] : make_double4(0.0, 0.0, 0.0, 0.0);
        const int l = valid && slenc ? slenc[sidx] : 0;
        const uint32_t ss = force_all ? MIXED : box_single_g8(b, l, g, rg, centers, sub);
        bool need = false;
        if (valid && sub == 0) {
            need = force_all || ss == MIXED || ss != stlab[sidx];
            if (need) stlab[sidx] = ss;  // all its points carry ss after this iteration
        }
        const unsigned m = __ballot_sync(0xffffffffu, need);
        unsigned long long base = 0;
        if (lane == 0 && m) base = atomicAdd(nswork, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (need) swork[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)sidx;
    }
}

__global__ void k_super_check(const double4* __restrict__ sbox, const int32_t* __restrict__ slenc,
                              int64_t ntiles, CandGrid g, const double* centers,
                              uint32_t* __restrict__ tlab, uint32_t* __restrict__ swork,
                              unsigned long long* __restrict__ nswork,
                              const int* __restrict__ skip_flag, int force_all, RowGrid rg,
                              int k) {
    super_check_body(sbox, slenc, ntiles, g, centers, tlab, swork, nswork, skip_flag, force_all, rg, k);
}

// Tiles of the listed super-tiles (8 lanes per tile over the flattened
// (super-tile, tile) list): the
// tiles whose single-center state changed or is MIXED are listed for
// k_lloyd_work with their new state in tnew.
__device__ __forceinline__ void tile_expand_body(const uint32_t* __restrict__ swork,
                              const unsigned long long* __restrict__ nswork,
                              const double4* __restrict__ tbox, const int32_t* __restrict__ tlen,
                              int64_t ntiles, CandGrid g, const double* centers,
                              const uint32_t* __restrict__ tlab, uint32_t* __restrict__ tnew,
                              uint32_t* __restrict__ work, unsigned long long* __restrict__ nwork,
                              const int* __restrict__ skip_flag, int force_all, RowGrid rg,
                              int k) {
    if (skip_flag && (skip_flag[0] | skip_flag[1])) return;
    extern __shared__ double s_centers[];
    for (int i = threadIdx.x; i < 2 * k; i += blockDim.x) s_centers[i] = centers[i];
    __syncthreads();
    centers = s_centers;
    const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
    const int64_t items = (int64_t)*nswork * 32;  // (listed super-tile, tile) pairs
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t wstride = (((int64_t)gridDim.x * blockDim.x) >> 5) * 4;
    for (int64_t i0 = warp * 4; i0 < items; i0 += wstride) {  // 8 lanes per tile
        const int64_t it = i0 + grp;
        const int64_t t = it < items ? (int64_t)swork[it >> 5] * 32 + (it & 31) : ntiles;
        const bool valid = t < ntiles;
        const double4 b = valid ? tbox[t] : make_double4(0.0, 0.0, 0.0, 0.0);
        const int l = valid && tlen ? tlen[t] : 0;
        const uint32_t single = force_all ? MIXED : box_single_g8(b, l, g, rg, centers, sub);
        bool add = false;
        if (valid && sub == 0) {
            tnew[t] = single;
            add = force_all || single == MIXED || single != tlab[t];
        }
        const unsigned am = __ballot_sync(0xffffffffu, add);
        unsigned long long base = 0;
        if (lane == 0 && am) base = atomicAdd(nwork, (unsigned long long)__popc(am));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (add) work[base + __popc(am & ((1u << lane) - 1u))] = (uint32_t)t;
    }
}

__global__ void k_tile_expand(const uint32_t* __restrict__ swork,
                              const unsigned long long* __restrict__ nswork,
                              const double4* __restrict__ tbox, const int32_t* __restrict__ tlen,
                              int64_t ntiles, CandGrid g, const double* centers,
                              const uint32_t* __restrict__ tlab, uint32_t* __restrict__ tnew,
                              uint32_t* __restrict__ work, unsigned long long* __restrict__ nwork,
                              const int* __restrict__ skip_flag, int force_all, RowGrid rg,
                              int k) {
    tile_expand_body(swork, nswork, tbox, tlen, ntiles, g, centers, tlab, tnew, work, nwork, skip_flag, force_all, rg, k);
}

// super-tile boxes and common lengths (32 tiles each)
__global__ void k_super_boxes(const double4* __restrict__ tbox, const int32_t* __restrict__ tlen,
                              int64_t ntiles, double4* __restrict__ sbox,
                              int32_t* __restrict__ slenc) {
    const int lane = threadIdx.x & 31;
    const int64_t nsuper = (ntiles + 31) / 32;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < nsuper;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t t = s * 32 + lane;
        double4 b = make_double4(INFINITY, -INFINITY, INFINITY, -INFINITY);
        int lmin = 0x7FFFFFFF, lmax = -1;
        if (t < ntiles) {
            b = tbox[t];
            const int l = tlen ? tlen[t] : 0;
            lmin = l;
            lmax = l;
        }
        for (int o = 16; o > 0; o >>= 1) {
            b.x = fmin(b.x, __shfl_xor_sync(0xffffffffu, b.x, o));
            b.y = fmax(b.y, __shfl_xor_sync(0xffffffffu, b.y, o));
            b.z = fmin(b.z, __shfl_xor_sync(0xffffffffu, b.z, o));
            b.w = fmax(b.w, __shfl_xor_sync(0xffffffffu, b.w, o));
        }
        lmin = __reduce_min_sync(0xffffffffu, lmin);
        lmax = __reduce_max_sync(0xffffffffu, lmax);
        if (lane == 0) {
            sbox[s] = b;
            slenc[s] = (lmin == lmax && lmin > 0) ? lmin : 0;
        }
    }
}

// One warp per listed tile: labels := the single center, or nearest_center
// through the grids; exact integer deltas of the cluster sums. The first
// (full) assignment accumulates per block in shared memory; the incremental
// ones move few points, so each (old, new) label group of a warp adds its
// deltas straight to the global accumulators (native 64-bit atomics in L2).
// One listed tile, one warp: labels := the single center, or nearest_center
// through the grids; exact integer deltas of the cluster sums (FULL: into
// the block's shared accumulators s_sx/s_sy/s_cnt; else (old, new) groups
// straight to the global limbs).
template <bool FULL>
__device__ __forceinline__ void lloyd_tile(
    uint32_t t, uint32_t single, const double2* __restrict__ spts, int64_t n,
    const double* __restrict__ cx, const double* __restrict__ cy, int k, CandGrid g,
    uint32_t* __restrict__ labs, uint32_t* __restrict__ tlab, int Ex, int Ey, ClusterAcc acc,
    RowGrid rg, const int32_t* __restrict__ slen, AggScratch* agg,
    unsigned long long* s_sx, unsigned long long* s_sy, unsigned long long* s_cnt,
    unsigned long long& my_changed) {
    const int lane = threadIdx.x & 31;
    uint32_t old[TILE / 32];
#pragma unroll
    for (int i = 0; i < TILE / 32; ++i) {
        const int64_t r = (int64_t)t * TILE + i * 32 + lane;
        old[i] = (r < n && !FULL) ? __ldcg(labs + r) : 0u;  // written by other SMs in-kernel
    }
    // all loads of the tile first (points, lengths, then row-cell words),
    // so a tile costs about three dependent memory latencies, not twelve
    double2 pt[TILE / 32];
    int32_t ln[TILE / 32];
    uint64_t cw[TILE / 32];
    uint32_t bst[TILE / 32];
#pragma unroll
    for (int i = 0; i < TILE / 32; ++i) {
        const int64_t r = (int64_t)t * TILE + i * 32 + lane;
        const bool valid = r < n;
        // not gated on old[i]: the point loads go out with the label loads
        // (one memory round trip instead of two; unused points cost 2 KB)
        pt[i] = valid ? spts[r] : make_double2(0.0, 0.0);
        ln[i] = (valid && single == MIXED && slen) ? slen[r] : 0;
    }
    if (single == MIXED && slen) {
#pragma unroll
        for (int i = 0; i < TILE / 32; ++i) {
            cw[i] = ~0ull;  // not built: fallback
            if (ln[i] >= 1 && ln[i] <= rg.R) {
                int iy = (int)((pt[i].y - rg.y0) * rg.invh);
                iy = min(max(iy, 0), rg.Gy - 1);
                cw[i] = __ldcg(reinterpret_cast<const unsigned long long*>(rg.cell) +
                               (size_t)(ln[i] - 1) * rg.Gy + iy);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < TILE / 32; ++i) {
        const int64_t r = (int64_t)t * TILE + i * 32 + lane;
        bst[i] = single;
        if (r < n && single == MIXED)
            bst[i] = slen ? row_pick(cw[i], g, rg.spill, pt[i].x, pt[i].y, cx, cy, k)
                          : grid_nearest(g, pt[i].x, pt[i].y, cx, cy, k);
    }
    auto flush = [&](uint32_t kk, u128 sa, u128 sb, unsigned long long, int cnt) {
        if (FULL) {
            fx_atomic_add(s_sx + 2 * kk, (i128)sa);
            fx_atomic_add(s_sy + 2 * kk, (i128)sb);
            atomicAdd(s_cnt + kk, (unsigned long long)cnt);
        } else {
            const uint32_t nb = kk & 0xFFFFu, ob = kk >> 16;
            l3_add(acc.sx + 3 * nb, (i128)sa);
            l3_add(acc.sy + 3 * nb, (i128)sb);
            atomicAdd(acc.cnt + nb, (unsigned long long)cnt);
            l3_add(acc.sx + 3 * ob, -(i128)sa);
            l3_add(acc.sy + 3 * ob, -(i128)sb);
            atomicAdd(acc.cnt + ob, (unsigned long long)(-(long long)cnt));
        }
    };
    bool mv[TILE / 32];
    uint32_t key[TILE / 32];
    uint32_t key0 = 0xFFFFFFFFu;  // the first moved point's key (lane order, round order)
#pragma unroll
    for (int i = 0; i < TILE / 32; ++i) {
        const int64_t r = (int64_t)t * TILE + i * 32 + lane;
        const bool valid = r < n;
        const uint32_t best = valid ? bst[i] : 0u;
        mv[i] = valid && (FULL || old[i] != best);
        if (mv[i]) labs[r] = best;
        if (!FULL && mv[i]) ++my_changed;
        key[i] = FULL ? best : ((old[i] << 16) | best);
        const unsigned bm = __ballot_sync(0xffffffffu, mv[i]);
        if (key0 == 0xFFFFFFFFu && bm) key0 = __shfl_sync(0xffffffffu, key[i], __ffs(bm) - 1);
    }
    bool uni = true;  // every moved point shares one (old, new) pair: the SINGLE-tile case
#pragma unroll
    for (int i = 0; i < TILE / 32; ++i) uni &= !mv[i] || key[i] == key0;
    uni = __all_sync(0xffffffffu, uni);
    if (uni) {
        if (key0 != 0xFFFFFFFFu) {  // one tree reduction and one set of atomics per tile
            i128 sa = 0, sb = 0;
            int cnt = 0;
#pragma unroll
            for (int i = 0; i < TILE / 32; ++i)
                if (mv[i]) {
                    sa += fx_from_double(pt[i].x, Ex);
                    sb += fx_from_double(pt[i].y, Ey);
                    ++cnt;
                }
            sa = fx_warp_sum(sa);
            sb = fx_warp_sum(sb);
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
            if (lane == 0) flush(key0, (u128)sa, (u128)sb, 0ULL, cnt);
        }
    } else {
        // group lanes by (old, new) label pair; one set of atomics per group
#pragma unroll
        for (int i = 0; i < TILE / 32; ++i) {
            const i128 fx = mv[i] ? fx_from_double(pt[i].x, Ex) : (i128)0;
            const i128 fy = mv[i] ? fx_from_double(pt[i].y, Ey) : (i128)0;
            warp_aggregate(mv[i], key[i], (u128)fx, (u128)fy, 0ULL, agg, flush);
        }
    }
    if (lane == 0) tlab[t] = single;
}

// One warp per listed tile (lloyd_tile). The first (full) assignment
// accumulates per block in shared memory; the incremental ones move few
// points, so each (old, new) label group of a warp adds its deltas straight
// to the global accumulators (native 64-bit atomics in L2).
template <bool FULL>
__device__ __forceinline__ void lloyd_work_body(
    const double2* __restrict__ spts, int64_t n, const double* __restrict__ centers, int k,
    CandGrid g, uint32_t* __restrict__ labs, const uint32_t* __restrict__ work,
    const unsigned long long* __restrict__ nwork, const uint32_t* __restrict__ tnew,
    uint32_t* __restrict__ tlab, int Ex, int Ey, ClusterAcc acc,
    unsigned long long* __restrict__ changed, const int* __restrict__ skip_flag, RowGrid rg,
    const int32_t* __restrict__ slen) {
    extern __shared__ unsigned char smem[];
    if (skip_flag && (skip_flag[0] | skip_flag[1])) return;
    double* cx = reinterpret_cast<double*>(smem);
    double* cy = cx + k;
    unsigned long long* s_sx = reinterpret_cast<unsigned long long*>(cy + k);  // FULL only
    unsigned long long* s_sy = s_sx + 2 * k;
    unsigned long long* s_cnt = s_sy + 2 * k;
    __shared__ unsigned long long s_changed;
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        cx[c] = centers[2 * c];
        cy[c] = centers[2 * c + 1];
        if (FULL) {
            s_sx[2 * c] = s_sx[2 * c + 1] = 0;
            s_sy[2 * c] = s_sy[2 * c + 1] = 0;
            s_cnt[c] = 0;
        }
    }
    if (threadIdx.x == 0) s_changed = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    __shared__ AggScratch agg_all[LL_TB / 32];
    AggScratch* agg = agg_all + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)*nwork;
    unsigned long long my_changed = 0;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t t = work[w];
        lloyd_tile<FULL>(t, tnew[t], spts, n, cx, cy, k, g, labs, tlab, Ex, Ey, acc, rg, slen, agg,
                         s_sx, s_sy, s_cnt, my_changed);
    }
    for (int o = 16; o > 0; o >>= 1) my_changed += __shfl_down_sync(0xffffffffu, my_changed, o);
    if (lane == 0 && my_changed) atomicAdd(&s_changed, my_changed);
    __syncthreads();
    if (FULL) {
        for (int c = threadIdx.x; c < k; c += blockDim.x) {
            const i128 vx = fx_load(s_sx + 2 * c), vy = fx_load(s_sy + 2 * c);
            if (vx) l3_add(acc.sx + 3 * c, vx);
            if (vy) l3_add(acc.sy + 3 * c, vy);
            if (s_cnt[c]) atomicAdd(acc.cnt + c, s_cnt[c]);
        }
    }
    if (threadIdx.x == 0 && s_changed) atomicAdd(changed, s_changed);
}

template <bool FULL>
__global__ void __launch_bounds__(LL_TB) k_lloyd_work(
    const double2* __restrict__ spts, int64_t n, const double* __restrict__ centers, int k,
    CandGrid g, uint32_t* __restrict__ labs, const uint32_t* __restrict__ work,
    const unsigned long long* __restrict__ nwork, const uint32_t* __restrict__ tnew,
    uint32_t* __restrict__ tlab, int Ex, int Ey, ClusterAcc acc,
    unsigned long long* __restrict__ changed, const int* __restrict__ skip_flag, RowGrid rg,
    const int32_t* __restrict__ slen) {
    lloyd_work_body<FULL>(spts, n, centers, k, g, labs, work, nwork, tnew, tlab, Ex, Ey, acc, changed, skip_flag, rg, slen);
}

// centers[c] = sums[c] / counts[c] for non-empty clusters (update_means
// :177-180); reports the empty clusters in index order.
// mov (optional, persistent loop): [0] displacement accumulated since the
// last row-grid build (double), [1] rebuild flag for this iteration (as
// double), [2] the allowed displacement D = slack / 2. The row grid is rebuilt
// only when a center may have moved more than D since the last build.
__device__ __forceinline__ void means_body(ClusterAcc acc, int k, int Ex, int Ey,
                                               double* __restrict__ centers,
                                               int* __restrict__ empties, int* __restrict__ n_empty,
                                               const int* __restrict__ gate,
                                               double* __restrict__ mov = nullptr) {
    if (gate && (gate[0] | gate[1])) return;  // uniform over the block
    __shared__ int wc[32];
    __shared__ int base;
    __shared__ double wmax[32];
    double dmax = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int c0 = 0; c0 < k; c0 += blockDim.x) {
        const int c = c0 + threadIdx.x;
        bool empty = false;
        if (c < k) {
            const long long cnt = (long long)acc.cnt[c];
            const i128 sx = l3_load(acc.sx + 3 * c), sy = l3_load(acc.sy + 3 * c);
            l3_store(acc.sx + 3 * c, sx);  // renormalise the limbs once per iteration
            l3_store(acc.sy + 3 * c, sy);
            if (cnt > 0) {
                const double nx = fx_to_double(sx, Ex) / (double)cnt;
                const double ny = fx_to_double(sy, Ey) / (double)cnt;
                if (mov) {  // displacement, rounded up
                    const double dx = nx - centers[2 * c], dy = ny - centers[2 * c + 1];
                    dmax = fmax(dmax, sqrt(dx * dx + dy * dy) * (1.0 + 1e-12) + 1e-300);
                }
                centers[2 * c] = nx;
                centers[2 * c + 1] = ny;
            } else {
                empty = true;
            }
        }
        // empty clusters listed in index order (block-wide ballot compaction)
        const unsigned m = __ballot_sync(0xffffffffu, empty);
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        int off = base;
        for (int w = 0; w < warp; ++w) off += wc[w];
        if (empty) empties[off + __popc(m & ((1u << lane) - 1u))] = c;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) base += wc[w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_empty = base;
    if (mov) {
        for (int o = 16; o > 0; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        if (lane == 0) wmax[warp] = dmax;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) dmax = fmax(dmax, wmax[w]);
            const double acc_d = mov[0] + dmax;  // triangle inequality: a bound
            if (!(acc_d <= mov[2])) {  // also NaN / +inf (forced)
                mov[0] = 0.0;
                mov[1] = 1.0;
            } else {
                mov[0] = acc_d;
                mov[1] = 0.0;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_means(ClusterAcc acc, int k, int Ex, int Ey,
                                               double* __restrict__ centers,
                                               int* __restrict__ empties, int* __restrict__ n_empty,
                                               const int* __restrict__ gate) {
    means_body(acc, k, Ex, Ey, centers, empties, n_empty, gate);
}

// farthest point among clusters with count > 1 (update_means :183-192):
// max distance, lowest ORIGINAL index on ties. Per-block candidates
// (distance bits, original index, sorted position).
__global__ void k_far_block(const double2* __restrict__ spts, const uint32_t* __restrict__ orig,
                            int64_t n, const uint32_t* __restrict__ labs,
                            const double* __restrict__ centers,
                            const unsigned long long* __restrict__ cnt,
                            unsigned long long* __restrict__ out) {
    double bd = -1.0;
    int64_t bi = INT64_MAX, br = -1;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t l = labs[r];
        if ((long long)cnt[l] <= 1) continue;
        const double2 p = spts[r];
        const double d = dist2(p.x, p.y, centers[2 * l], centers[2 * l + 1]);
        const int64_t o = orig[r];
        if (d > bd || (d == bd && o < bi)) {
            bd = d;
            bi = o;
            br = r;
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double od = __shfl_down_sync(0xffffffffu, bd, off);
        const int64_t oi = __shfl_down_sync(0xffffffffu, bi, off);
        const int64_t orr = __shfl_down_sync(0xffffffffu, br, off);
        if (od > bd || (od == bd && oi < bi)) {
            bd = od;
            bi = oi;
            br = orr;
        }
    }
    __shared__ double sd[32];
    __shared__ int64_t si[32], sr[32];
    if ((threadIdx.x & 31) == 0) {
        sd[threadIdx.x >> 5] = bd;
        si[threadIdx.x >> 5] = bi;
        sr[threadIdx.x >> 5] = br;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (sd[w] > bd || (sd[w] == bd && si[w] < bi)) {
                bd = sd[w];
                bi = si[w];
                br = sr[w];
            }
        out[3 * blockIdx.x] = (unsigned long long)__double_as_longlong(bd);
        out[3 * blockIdx.x + 1] = (unsigned long long)bi;
        out[3 * blockIdx.x + 2] = (unsigned long long)br;
    }
}

// re-seed empty cluster c at the farthest point (update_means :193-196)
__global__ void k_repair(const double2* __restrict__ spts, const uint32_t* __restrict__ pos,
                         uint32_t* __restrict__ labs, double* __restrict__ centers, ClusterAcc acc,
                         int Ex, int Ey, const unsigned long long* __restrict__ blk, int nblk,
                         int c, uint32_t* __restrict__ tlab, int64_t ntiles) {
    double bd = -1.0;
    int64_t bi = INT64_MAX, br = -1;
    for (int b = 0; b < nblk; ++b) {
        const double d = __longlong_as_double((long long)blk[3 * b]);
        const int64_t i = (int64_t)blk[3 * b + 1];
        if (d > bd || (d == bd && i < bi)) {
            bd = d;
            bi = i;
            br = (int64_t)blk[3 * b + 2];
        }
    }
    if (br < 0) br = pos[0];  // no candidate: far_i stays 0 (original index)
    const uint32_t donor = labs[br];
    const double2 p = spts[br];
    const i128 fx = fx_from_double(p.x, Ex), fy = fx_from_double(p.y, Ey);
    l3_store(acc.sx + 3 * donor, l3_load(acc.sx + 3 * donor) - fx);
    l3_store(acc.sy + 3 * donor, l3_load(acc.sy + 3 * donor) - fy);
    acc.cnt[donor] -= 1;
    labs[br] = (uint32_t)c;
    tlab[br / TILE] = MIXED;  // the tile no longer holds one label
    tlab[ntiles + br / (TILE * 32)] = MIXED;  // nor its super-tile
    l3_store(acc.sx + 3 * c, fx);
    l3_store(acc.sy + 3 * c, fy);
    acc.cnt[c] = 1;
    centers[2 * c] = p.x;
    centers[2 * c + 1] = p.y;
}

__global__ void k_sse(const double2* __restrict__ spts, int64_t n,
                      const uint32_t* __restrict__ labs, const double* __restrict__ centers,
                      int E, unsigned long long* __restrict__ acc) {
    i128 s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t l = labs[i];
        const double2 p = spts[i];
        s += fx_from_double(dist2(p.x, p.y, centers[2 * l], centers[2 * l + 1]), E);
    }
    s = fx_warp_sum(s);
    if ((threadIdx.x & 31) == 0) fx_atomic_add(acc, s);
}

__global__ void k_unsort_labels(const uint32_t* __restrict__ labs,
                                const uint32_t* __restrict__ orig, int64_t n,
                                uint32_t* __restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        out[orig[r]] = labs[r];
}

struct LloydCtx {
    const double2* spts;
    const uint32_t* orig;
    const uint32_t* pos;
    int64_t n;
    int k;
    int Ex, Ey;
    cudaStream_t st;
    DArr<double> centers;
    DArr<double> mov;              // persistent loop: row-grid movement state
    DArr<uint32_t> labs;           // sorted order
    DArr<unsigned long long> acc;  // 5k: sx(2k) sy(2k) cnt(k)
    DArr<unsigned long long> flags;  // [0] changed
    DArr<int> empties;             // k + 1 (last = count)
    DArr<unsigned long long> far_blk;
    CandGrid cg;
    DArr<uint16_t> cg_cnt, cg_cand;
    const double4* tbox = nullptr;
    int64_t ntiles = 0;
    DArr<uint32_t> tlab, tnew, work;  // tile | super-tile states, new tile states, listed tiles
    DArr<uint32_t> swork;             // listed super-tiles
    DArr<unsigned long long> nswork;
    DArr<unsigned long long> nwork, diag;
    RowGrid rg{};                   // rg.R == 0: no row grid
    DArr<uint64_t> rg_cell;
    DArr<uint16_t> rg_spill;
    DArr<int> rg_blocks;            // row-grid segments holding points
    int rg_nblocks = 0;
    const int32_t* slen = nullptr;  // piece length per sorted point
    const int32_t* tlen = nullptr;  // common piece length per tile (0: mixed)
    DArr<double4> sbox;             // super-tile boxes (32 tiles)
    DArr<int32_t> slenc;            // super-tile common piece length (0: mixed)
    int64_t nsuper() const { return (ntiles + 31) / 32; }
    int64_t nstate() const { return std::max<int64_t>(ntiles, 1) + nsuper(); }  // tlab | stlab
    DArr<unsigned long long> dacc;  // distributed fit: this rank's deltas (5k)
    bool use_dacc = false;
    ClusterAcc cacc() { return ClusterAcc{acc.p, acc.p + 3 * k, acc.p + 6 * k}; }
    // label-change counter: in the distributed fit it trails the deltas
    // (dacc[7k]) so one all-reduce carries both
    unsigned long long* changed_ptr() { return use_dacc ? dacc.p + 7 * k : flags.p; }
    ClusterAcc tacc() {  // where the assignment writes
        return use_dacc ? ClusterAcc{dacc.p, dacc.p + 3 * k, dacc.p + 6 * k} : cacc();
    }
    size_t smem(bool full) const {
        return sizeof(double) * 2 * k + (full ? sizeof(unsigned long long) * 5 * k : 0);
    }
    int grid() const {
        return (int)std::max<int64_t>(1, std::min<int64_t>((n + LL_TB - 1) / LL_TB,
                                                           (int64_t)num_sms() * 6));
    }
};

// end of one batched Lloyd iteration (lloyd_once :209-213): ++iterations,
// stop when no label changed; resets the per-iteration counters. Gated like
// the other kernels, so iterations launched past convergence are no-ops.
__device__ __forceinline__ void iter_end_body(int* __restrict__ state, unsigned long long* __restrict__ changed,
                           unsigned long long* __restrict__ nwork,
                           unsigned long long* __restrict__ nswork,
                           unsigned long long* __restrict__ diag) {
    if (state[0] | state[1]) return;  // pending repair / converged
    state[2] += 1;
    diag[0] += *nwork;  // diagnostics: tiles / super-tiles listed, labels changed
    diag[2] += *nswork;
    diag[1] += *changed;
    if (*changed == 0) state[1] = 1;
    *changed = 0;
    *nwork = 0;
    *nswork = 0;
}

__global__ void k_iter_end(int* __restrict__ state, unsigned long long* __restrict__ changed,
                           unsigned long long* __restrict__ nwork,
                           unsigned long long* __restrict__ nswork,
                           unsigned long long* __restrict__ diag) {
    iter_end_body(state, changed, nwork, nswork, diag);
}

void lloyd_assign(LloydCtx& L, bool full, bool gate_on_empties) {
    const int* gate = gate_on_empties ? L.empties.p + L.k : nullptr;
    if (L.n == 0) return;  // a rank may hold no sample points
    {
        JB_PROF("lloyd_grid", L.st);
        if (L.cg.G > 0) launch_grid_build(L.cg, L.centers.p, L.k, L.st);
        if (L.rg.R > 0)
            launch_row_grid_build(L.rg, L.centers.p, L.k, L.st, L.rg_blocks.p, L.rg_nblocks);
    }
    JB_LAUNCH_CHECK();
    {
        JB_PROF("lloyd_tile_check", L.st);
        k_super_check<<<(int)std::max<int64_t>(1, std::min<int64_t>((L.nsuper() + 255) / 256,
                                                                   num_sms() * 16)),
                        256, sizeof(double) * 2 * L.k, L.st>>>(
            L.sbox.p, L.rg.R > 0 ? L.slenc.p : nullptr, L.ntiles, L.cg, L.centers.p, L.tlab.p,
            L.swork.p, L.nswork.p, gate, full ? 1 : 0, L.rg, L.k);
        k_tile_expand<<<full ? (int)std::max<int64_t>(1, std::min<int64_t>((L.nsuper() + 7) / 8,
                                                                            num_sms() * 16))
                             : num_sms() * 4,
                        256, sizeof(double) * 2 * L.k, L.st>>>(
            L.swork.p, L.nswork.p, L.tbox, L.rg.R > 0 ? L.tlen : nullptr, L.ntiles, L.cg,
            L.centers.p, L.tlab.p, L.tnew.p, L.work.p, L.nwork.p, gate, full ? 1 : 0, L.rg, L.k);
    }
    JB_LAUNCH_CHECK();
    JB_PROF("lloyd_assign", L.st);
    auto kern = full ? k_lloyd_work<true> : k_lloyd_work<false>;
    kern<<<L.grid(), LL_TB, L.smem(full), L.st>>>(
        L.spts, L.n, L.centers.p, L.k, L.cg, L.labs.p, L.work.p, L.nwork.p, L.tnew.p, L.tlab.p,
        L.Ex, L.Ey, L.tacc(), L.changed_ptr(), gate, L.rg, L.rg.R > 0 ? L.slen : nullptr);
    JB_LAUNCH_CHECK();
}

void lloyd_means(LloydCtx& L, bool gated) {
    JB_PROF("lloyd_means", L.st);
    k_means<<<1, 256, 0, L.st>>>(L.cacc(), L.k, L.Ex, L.Ey, L.centers.p, L.empties.p,
                                  L.empties.p + L.k, gated ? L.empties.p + L.k : nullptr);
    JB_LAUNCH_CHECK();
}

// Persistent Lloyd loop (single GPU, row grid in use): every phase of an
// iteration -- update_means (block 0), row-grid rebuild, super-tile check,
// tile expansion, re-assignment, iteration end (block 0) -- runs in ONE
// cooperative launch separated by grid-wide barriers, for up to `budget`
// iterations, stopping at convergence or when update_means reports empty
// clusters (re-seeded on the host path). Same phase bodies as the
// multi-kernel path, so the same arithmetic.
struct PersistArgs {
    ClusterAcc acc;
    int k, Ex, Ey;
    double* centers;
    int* empties;  // k entries, then state: n_empty | converged | iterations
    RowGrid rg;
    const int* rg_blocks;
    int rg_nblocks;
    const double4* sbox;
    const int32_t* slenc;
    int64_t ntiles;
    CandGrid cg;
    uint32_t* tlab;
    uint32_t* swork;
    unsigned long long* nswork;
    const double4* tbox;
    const int32_t* tlen;
    uint32_t* tnew;
    uint32_t* work;
    unsigned long long* nwork;
    const double2* spts;
    int64_t n;
    uint32_t* labs;
    unsigned long long* changed;
    const int32_t* slen;
    unsigned long long* diag;
    int budget;
    unsigned long long* tstamp;  // optional: 8 globaltimer stamps per iteration (block 0; [7] the slowest block)
    double* mov;                 // row-grid movement state (means_body)
    unsigned long long* cnt2;    // persistent loop: changed[2], listed super-tiles[2], listed tiles[2] (by parity)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// update_means (clustering.hpp:177-180) computed by EVERY block from the
// global limbs into its shared copy of the centers (identical on every
// block: the same integers, the same operations), so no block waits for
// another to publish them. Returns the number of empty clusters (listed in
// index order into empties when non-null) and the largest center
// displacement (rounded up), both uniform over the block.
__device__ __forceinline__ void means_local(ClusterAcc acc, int k, int Ex, int Ey, double* s_c,
                                            double* cx, double* cy, int* __restrict__ empties,
                                            int& n_empty, double& dmax_out) {
    // two block barriers: the displacement maximum as the bits of a
    // non-negative double (ordered like the value) and the empty count by
    // shared-memory atomics; the ordered empty list only when one is empty
    __shared__ unsigned long long s_dmax;
    __shared__ int s_ne;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        s_dmax = 0ull;
        s_ne = 0;
    }
    __syncthreads();
    double dmax = 0.0;
    int ne = 0;
    for (int c = threadIdx.x; c < k; c += blockDim.x) {
        const long long cnt = (long long)__ldcg(acc.cnt + c);
        const i128 sx = (i128)((u128)__ldcg(acc.sx + 3 * c) + ((u128)__ldcg(acc.sx + 3 * c + 1) << 32) +
                               ((u128)__ldcg(acc.sx + 3 * c + 2) << 64));
        const i128 sy = (i128)((u128)__ldcg(acc.sy + 3 * c) + ((u128)__ldcg(acc.sy + 3 * c + 1) << 32) +
                               ((u128)__ldcg(acc.sy + 3 * c + 2) << 64));
        if (cnt > 0) {
            const double nx = fx_to_double(sx, Ex) / (double)cnt;
            const double ny = fx_to_double(sy, Ey) / (double)cnt;
            const double dx = nx - s_c[2 * c], dy = ny - s_c[2 * c + 1];
            dmax = fmax(dmax, sqrt(dx * dx + dy * dy) * (1.0 + 1e-12) + 1e-300);
            s_c[2 * c] = nx;
            s_c[2 * c + 1] = ny;
            cx[c] = nx;
            cy[c] = ny;
        } else {
            ++ne;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        ne += __shfl_xor_sync(0xffffffffu, ne, o);
    }
    if (lane == 0) {
        atomicMax(&s_dmax, (unsigned long long)__double_as_longlong(dmax));
        if (ne) atomicAdd(&s_ne, ne);
    }
    __syncthreads();
    n_empty = s_ne;
    dmax_out = __longlong_as_double((long long)s_dmax);
    if (n_empty > 0 && empties && threadIdx.x == 0) {  // rare: the host repairs; index order
        int m = 0;
        for (int c = 0; c < k; ++c)
            if ((long long)__ldcg(acc.cnt + c) <= 0) empties[m++] = c;
    }
}

// Lloyd iterations (lloyd_once :200-220) in one cooperative launch, three grid
// barriers per iteration:
//   every block: update_means into its shared centers (means_local); stop on
//     an empty cluster (host repair); row-grid rebuild when the centers may
//     have moved more than half a cell since the last one (+ barrier);
//     super-tile check -> global list of super-tiles;       barrier B1
//   (listed super-tile, 4 of its tiles) per warp: the tiles' single-center
//     tests; the tiles that need a reassignment go to one global tile list
//     (one reservation per block pass);                     barrier B1.5
//   the list's tiles spread evenly over all warps of the grid (lloyd_tile);
//                                                           barrier B2
//   every block: iteration end (count, stop when no label changed).
// The tile list replaced per-block queues drained by the block's own warps:
// the slowest block then ended its work 17.0 us after B1 (mean work 9.7 us),
// with the list 13.5 us (config 4: 29.6 -> 26.2 us per iteration).
// Counters alternate by iteration parity, so a counter is cleared only once
// every block is past reading it. Block 0 folds the low limbs of the cluster
// sums upward with atomics while the other blocks add to them.
// 80 registers (3 blocks per SM): with 2 the grid is 296 blocks, and the
// iterations take longer than the few spilled registers cost.
__global__ void __launch_bounds__(256, 3) k_lloyd_persistent(PersistArgs a) {
    namespace cgx = cooperative_groups;
    cgx::grid_group grid = cgx::this_grid();
    extern __shared__ double s_cen[];  // [0, 2k) centers (x, y); [2k, 4k) cx | cy
    const int k = a.k;
    double* cx = s_cen + 2 * k;
    double* cy = cx + k;
    __shared__ AggScratch agg_all[8];
    AggScratch* agg = agg_all + (threadIdx.x >> 5);
    __shared__ unsigned long long s_changed;
    __shared__ unsigned long long s_q[32];  // block tile queue: (single << 32) | tile
    __shared__ int s_qn;
    if (threadIdx.x == 0) s_qn = 0;
    int* state = a.empties + k;
    if (state[0] | state[1]) return;  // pending repair / converged (uniform)
    for (int i = threadIdx.x; i < 2 * k; i += blockDim.x) s_cen[i] = a.centers[i];
    double mov0 = a.mov[0];  // displacement since the last row-grid build (+inf: build now)
    const double movD = a.mov[2];
    const bool ts = a.tstamp && blockIdx.x == 0 && threadIdx.x == 0;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    __syncthreads();
    for (int b = 0; b < a.budget; ++b) {
        const int par = b & 1;
        if (ts && b < 512) a.tstamp[8 * b] = gtimer();
        int n_empty;
        double dmax;
        means_local(a.acc, k, a.Ex, a.Ey, s_cen, cx, cy, blockIdx.x == 0 ? a.empties : nullptr, n_empty,
                    dmax);
        if (n_empty > 0) {
            if (lead) state[0] = n_empty;
            break;
        }
        const double acc_d = mov0 + dmax;  // triangle inequality: a bound
        const bool rebuild = !(acc_d <= movD);
        mov0 = rebuild ? 0.0 : acc_d;
        if (ts && b < 512) a.tstamp[8 * b + 1] = gtimer();
        if (rebuild) {
            row_grid_build_body(a.rg, s_cen, k, a.rg_blocks, a.rg_nblocks);
            grid.sync();
        }
        if (ts && b < 512) a.tstamp[8 * b + 2] = gtimer();
        super_check_body(a.sbox, a.slenc, a.ntiles, a.cg, s_cen, a.tlab, a.swork, a.cnt2 + 2 + par,
                         nullptr, 0, a.rg, k);
        if (threadIdx.x == 0) s_changed = 0;
        if (a.tstamp && blockIdx.x == 0 && b < 512) {  // check done (block 0)
            __syncthreads();
            if (threadIdx.x == 0) a.tstamp[8 * b + 6] = gtimer();
        }
        grid.sync();  // B1
        if (ts && b < 512) a.tstamp[8 * b + 3] = gtimer();
        if (lead) {  // counters of the other parity: last read before B2 of b - 1
            a.cnt2[par ^ 1] = 0;
            a.cnt2[2 + (par ^ 1)] = 0;
            a.cnt2[4 + (par ^ 1)] = 0;
        }
        if (blockIdx.x == 0) {  // fold the low limbs of the cluster sums (value-preserving)
            for (int q = threadIdx.x; q < 2 * k; q += blockDim.x) {
                unsigned long long* l3 = (q < k ? a.acc.sx : a.acc.sy) + 3 * (q % k);
                const unsigned long long L = atomicExch(l3, 0ULL);
                atomicAdd(l3, L & 0xFFFFFFFFull);
                atomicAdd(l3 + 1, L >> 32);
                const unsigned long long M = atomicExch(l3 + 1, 0ULL);
                atomicAdd(l3 + 1, M & 0xFFFFFFFFull);
                atomicAdd(l3 + 2, M >> 32);
            }
        }
        const int64_t items = (int64_t)__ldcg(a.cnt2 + 2 + par) * 8;
        unsigned long long my_changed = 0, my_tiles = 0;
        {
            // W1: every warp tests its items (balanced by count) and the
            // block's tiles that need a reassignment go to one global list (one
            // reservation per block pass); barrier; W2: the list's tiles spread
            // evenly over all warps of the grid
            const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
            const int wib = threadIdx.x >> 5;
            unsigned long long* nlist = a.cnt2 + 4 + par;
            for (int64_t b0 = (int64_t)blockIdx.x * 8; b0 < items; b0 += (int64_t)gridDim.x * 8) {
                const int64_t it = b0 + wib;
                if (it < items) {
                    const int64_t t = (int64_t)__ldcg(a.swork + (it >> 3)) * 32 + (it & 7) * 4 + grp;
                    const bool tv = t < a.ntiles;
                    const double4 tb = tv ? a.tbox[t] : make_double4(0.0, 0.0, 0.0, 0.0);
                    const int tl = tv && a.tlen ? a.tlen[t] : 0;
                    const uint32_t single = box_single_g8(tb, tl, a.cg, a.rg, s_cen, sub);
                    const bool add = tv && sub == 0 && (single == MIXED || single != __ldcg(a.tlab + t));
                    if (add) {
                        a.tnew[t] = single;
                        s_q[atomicAdd(&s_qn, 1)] = (unsigned long long)t;
                    }
                }
                __syncthreads();
                const int nq = s_qn;
                if (nq) {
                    __shared__ unsigned long long s_base;
                    if (threadIdx.x == 0) s_base = atomicAdd(nlist, (unsigned long long)nq);
                    __syncthreads();
                    if (threadIdx.x < nq) a.work[s_base + threadIdx.x] = (uint32_t)s_q[threadIdx.x];
                }
                __syncthreads();
                if (threadIdx.x == 0) s_qn = 0;
                __syncthreads();
            }
            grid.sync();  // B1.5: the tile list is complete
            const int64_t nw = (int64_t)__ldcg(nlist);
            const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
            for (int64_t q = (((int64_t)blockIdx.x * blockDim.x) >> 5) + wib; q < nw; q += W) {
                const uint32_t t = __ldcg(a.work + q);
                lloyd_tile<false>(t, __ldcg(a.tnew + t), a.spts, a.n, cx, cy, k, a.cg, a.labs, a.tlab,
                                  a.Ex, a.Ey, a.acc, a.rg, a.slen, agg, nullptr, nullptr, nullptr,
                                  my_changed);
                ++my_tiles;
            }
        }
        if ((threadIdx.x & 31) == 0 && my_tiles) atomicAdd(a.diag, my_tiles);
        for (int o = 16; o > 0; o >>= 1) my_changed += __shfl_down_sync(0xffffffffu, my_changed, o);
        if ((threadIdx.x & 31) == 0 && my_changed) atomicAdd(&s_changed, my_changed);
        __syncthreads();
        if (threadIdx.x == 0 && s_changed) atomicAdd(a.cnt2 + par, s_changed);
        if (ts && b < 512) a.tstamp[8 * b + 4] = gtimer();
        if (a.tstamp && b < 512 && threadIdx.x == 0) atomicMax(a.tstamp + 8 * b + 7, gtimer());
        grid.sync();  // B2
        if (ts && b < 512) a.tstamp[8 * b + 5] = gtimer();
        // iteration end (iter_end_body), on every block
        const unsigned long long chg = __ldcg(a.cnt2 + par);
        if (lead) {
            state[2] += 1;
            a.diag[1] += chg;  // labels changed
            a.diag[2] += __ldcg(a.cnt2 + 2 + par);  // super-tiles listed
        }
        if (chg == 0) {
            if (lead) state[1] = 1;
            break;
        }
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < 2 * k; i += blockDim.x) a.centers[i] = s_cen[i];
    }
}

// the persistent loop applies when the row grid carries the assignment
// (no 2-D grid) and the device can co-schedule the grid
bool lloyd_persistent(LloydCtx& L, int budget) {
    static const bool phase_times = getenv("JB_LLOYD_PHASES") != nullptr;
    if (L.rg.R == 0 || L.cg.G != 0 || L.n == 0 || dbg_on()) return false;
    static int coop = -1;
    if (coop < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    }
    if (!coop) return false;
    const size_t smem = sizeof(double) * 4 * L.k;  // centers (x, y) + cx | cy
    if (smem > 200 * 1024 ||
        cudaFuncSetAttribute(k_lloyd_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lloyd_persistent, 256, smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (per_sm < 1) return false;
    static const int per_sm_cap = getenv("JB_LLOYD_PER_SM") ? atoi(getenv("JB_LLOYD_PER_SM")) : 3;
    if (per_sm_cap > 0) per_sm = std::min(per_sm, per_sm_cap);  // grid barriers: fewer blocks
    PersistArgs a;
    a.acc = L.cacc();
    a.k = L.k;
    a.Ex = L.Ex;
    a.Ey = L.Ey;
    a.centers = L.centers.p;
    a.empties = L.empties.p;
    a.rg = L.rg;
    a.rg_blocks = L.rg_blocks.p;
    a.rg_nblocks = L.rg_nblocks;
    a.sbox = L.sbox.p;
    a.slenc = L.slenc.p;
    a.ntiles = L.ntiles;
    a.cg = L.cg;
    a.tlab = L.tlab.p;
    a.swork = L.swork.p;
    a.nswork = L.nswork.p;
    a.tbox = L.tbox;
    a.tlen = L.tlen;
    a.tnew = L.tnew.p;
    a.work = L.work.p;
    a.nwork = L.nwork.p;
    a.spts = L.spts;
    a.n = L.n;
    a.labs = L.labs.p;
    a.changed = L.flags.p;
    a.slen = L.slen;
    a.diag = L.diag.p;
    a.budget = budget;
    // grid slack: centers may drift h / 2 (half a row-grid cell) between
    // rebuilds; the first iteration of every launch rebuilds (+inf)
    if (L.mov.n == 0) L.mov.alloc(3, L.st);
    {
        const double init[3] = {INFINITY, 1.0, 0.5 * L.rg.slack};
        L.mov.upload(init, 3);
    }
    a.mov = L.mov.p;
    DArr<unsigned long long> tsb(phase_times ? 8 * 512 : 0, L.st);
    if (phase_times) tsb.zero();
    a.tstamp = phase_times ? tsb.p : nullptr;
    DArr<unsigned long long> cnt2(6, L.st);
    cnt2.zero();
    a.cnt2 = cnt2.p;
    void* args[] = {&a};
    {
        JB_PROF("lloyd_persistent", L.st);
        const cudaError_t e = cudaLaunchCooperativeKernel(
            (const void*)k_lloyd_persistent, dim3(num_sms() * per_sm), dim3(256), args, smem, L.st);
        if (e != cudaSuccess) {  // cannot co-schedule (MPS/MIG limits): multi-kernel path
            cudaGetLastError();
            return false;
        }
    }
    if (phase_times) {  // JB_LLOYD_PHASES=1: mean phase latencies (us) on stderr
        auto h = tsb.to_host(8 * 512);
        double acc[5] = {0, 0, 0, 0, 0};
        int cnt = 0;
        double chk = 0, lastw = 0;
        for (int b = 0; b < 512 && h[8 * b + 5]; ++b, ++cnt) {
            for (int q = 0; q < 5; ++q) acc[q] += (double)(h[8 * b + q + 1] - h[8 * b + q]) * 1e-3;
            chk += (double)(h[8 * b + 6] - h[8 * b + 2]) * 1e-3;
            lastw += (double)(h[8 * b + 7] - h[8 * b + 3]) * 1e-3;
        }
        if (cnt) {
            int rebuilds = 0;
            double quart[4][5] = {};
            for (int b = 0; b < cnt; ++b) {
                rebuilds += (h[8 * b + 2] - h[8 * b + 1]) > 1500;
                for (int q = 0; q < 5; ++q)
                    quart[4 * b / cnt][q] += (double)(h[8 * b + q + 1] - h[8 * b + q]) * 1e-3;
            }
            fprintf(stderr, "[jb] lloyd phases over %d iters (us): means %.1f grid %.1f check+B1 %.1f "
                            "work %.1f B2 %.1f (grid %d x 256), %d grid rebuilds\n",
                    cnt, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt,
                    num_sms() * per_sm, rebuilds);
            fprintf(stderr, "[jb] lloyd: block-0 check %.1f us (B1 wait = check+B1 - this), "
                            "slowest block's work end %.1f us after B1 exit\n", chk / cnt, lastw / cnt);
            for (int qq = 0; qq < 4; ++qq)
                fprintf(stderr, "[jb]   quarter %d: means %.1f grid %.1f check+B1 %.1f work %.1f B2 %.1f\n",
                        qq, quart[qq][0] / (cnt / 4.0), quart[qq][1] / (cnt / 4.0),
                        quart[qq][2] / (cnt / 4.0), quart[qq][3] / (cnt / 4.0),
                        quart[qq][4] / (cnt / 4.0));
        }
    }
    return true;
}

struct LoopState {
    int n_empty, converged, iters;
};

LoopState lloyd_state(LloydCtx& L) {
    LoopState h;
    JB_CUDA(cudaMemcpyAsync(&h, L.empties.p + L.k, sizeof h, cudaMemcpyDeviceToHost, L.st));
    JB_CUDA(cudaStreamSynchronize(L.st));
    return h;
}

// empty-cluster re-seeding (update_means :181-197), in cluster order
void lloyd_repair(LloydCtx& L, int ne) {
    std::vector<int> em(ne);
    JB_CUDA(cudaMemcpyAsync(em.data(), L.empties.p, sizeof(int) * ne, cudaMemcpyDeviceToHost,
                            L.st));
    JB_CUDA(cudaStreamSynchronize(L.st));
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((L.n + 255) / 256, num_sms() * 4));
    if (L.far_blk.n < (size_t)(3 * nblk)) L.far_blk.alloc(3 * nblk, L.st);
    for (int c : em) {
        k_far_block<<<nblk, 256, 0, L.st>>>(L.spts, L.orig, L.n, L.labs.p, L.centers.p,
                                            L.cacc().cnt, L.far_blk.p);
        JB_LAUNCH_CHECK();
        k_repair<<<1, 1, 0, L.st>>>(L.spts, L.pos, L.labs.p, L.centers.p, L.cacc(), L.Ex, L.Ey,
                                    L.far_blk.p, nblk, c, L.tlab.p, L.ntiles);
        JB_LAUNCH_CHECK();
    }
    const int zero = 0;
    JB_CUDA(cudaMemcpyAsync(L.empties.p + L.k, &zero, sizeof(int), cudaMemcpyHostToDevice, L.st));
}

// update_means for the final centers (after the loop): means + repairs
void lloyd_update_means_sync(LloydCtx& L) {
    lloyd_means(L, false);
    int ne = 0;
    JB_CUDA(cudaMemcpyAsync(&ne, L.empties.p + L.k, sizeof(int), cudaMemcpyDeviceToHost, L.st));
    JB_CUDA(cudaStreamSynchronize(L.st));
    if (ne) lloyd_repair(L, ne);
}

}  // namespace

void lloyd_best_device(const PtsView& pv, const uint64_t* d_idx, int64_t n, uint64_t k,
                       uint64_t max_iters, uint64_t n_init, const uint64_t* d_raw,
                       uint64_t raw_count, uint64_t* cursor, const BBox& bb, KMeansOut& out,
                       cudaStream_t st, const PieceRows& rows, const SampleOrder* jorder) {
    if (k < 1) throw Error(INVALID_INPUT, "d2_seed: k must be >= 1");
    if ((int64_t)k > n) throw Error(INVALID_INPUT, "d2_seed: k exceeds points");
    if (k > 2048) throw Error(INVALID_INPUT, "k > 2048 is not supported by the Lloyd kernel");
    if (n >= (1LL << 32)) throw Error(INVALID_INPUT, "k-means on more than 2^32 points");
    const double mx = std::max(std::fabs(bb.xmin), std::fabs(bb.xmax));
    const double my = std::max(std::fabs(bb.ymin), std::fabs(bb.ymax));
    const double wx = bb.xmax - bb.xmin, wy = bb.ymax - bb.ymin;
    const double d2max = (wx * wx + wy * wy) * (1.0 + 1e-9) + 1e-300;
    const int Ed2 = fx_exponent_for(d2max * (double)n * 1.001);

    // ---- Morton order of the points ----
    DArr<double2> spts(n, st);
    DArr<uint32_t> orig(n, st), pos(n, st);
    DArr<int32_t> slen(rows.len ? n : 0, st), tlen((n + TILE - 1) / TILE, st);
    {
        DArr<uint32_t> keys(n, st), skeys(n, st), vals(n, st);
        const double sx = wx > 0 ? 65535.0 / wx : 0.0, sy = wy > 0 ? 65535.0 / wy : 0.0;
        const bool jo = jorder && d_idx && rows.len && !pv.pts && pv.len == rows.len &&
                        jorder->j.n >= (size_t)n && jorder->i.n >= (size_t)n;
        if (jo) {  // piece reads in ascending piece order, (length, y) key (k_rowkey_jorder)
            int lbits = 1;
            const uint32_t lcap = (uint32_t)std::min<int32_t>(std::max<int32_t>(rows.max_len, 1), 255);
            while ((1u << lbits) <= lcap) ++lbits;
            const int end_bit = lbits + 18 <= 24 ? 24 : 32;
            const int qbits = end_bit - lbits;
            const double syq = wy > 0 ? (double)((1u << qbits) - 1u) / wy : 0.0;
            DArr<SRec> rec(n, st), srec(n, st);
            {
                JB_PROF("sample_order", st);
                k_rowkey_jorder<<<grid_cap(n), 256, 0, st>>>(pv, d_idx, jorder->j.p, jorder->i.p, n,
                                                             qbits, lcap, bb.ymin, syq, keys.p, rec.p);
            }
            JB_LAUNCH_CHECK();
            size_t tb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, rec.p, srec.p, n, 0,
                                            end_bit, st);
            DArr<uint8_t> tmp(tb, st);
            cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, rec.p, srec.p, n, 0,
                                            end_bit, st);
            JB_LAUNCH_CHECK();
            {
                JB_PROF("sample_unpack", st);
                k_rec_unpack<<<grid_cap(n), 256, 0, st>>>(srec.p, n, spts.p, orig.p, pos.p, pv.scl,
                                                          pv.sl, slen.p);
                // ~48 MB of pos per pass: resident in the 126 MB L2 while scattered
                const int64_t span = (int64_t)12 << 20;
                for (int64_t lo = 0; lo < n; lo += span)
                    k_pos_scatter<<<grid_cap(n), 256, 0, st>>>(
                        orig.p, n, (uint32_t)lo, (uint32_t)std::min<int64_t>(n, lo + span), pos.p);
            }
            JB_LAUNCH_CHECK();
        } else {
            DArr<double2> cpts(n, st);
            k_morton<<<grid_cap(n), 256, 0, st>>>(pv, d_idx, n, bb.xmin, sx, bb.ymin, sy, keys.p,
                                                  vals.p, cpts.p, rows.len);
            JB_LAUNCH_CHECK();
            size_t tb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, vals.p, orig.p, n, 0, 32,
                                            st);
            DArr<uint8_t> tmp(tb, st);
            cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, vals.p, orig.p, n, 0, 32,
                                            st);
            JB_LAUNCH_CHECK();
            k_sorted_gather<<<grid_cap(n), 256, 0, st>>>(cpts.p, orig.p, n, spts.p, pos.p, pv.scl,
                                                         pv.sl, rows.len ? slen.p : nullptr);
            JB_LAUNCH_CHECK();
        }
    }
    JB_TRACE("kmeans: morton order", st);
    const int64_t ntiles = (n + TILE - 1) / TILE;
    DArr<double4> tbox(ntiles, st);
    DArr<float> tmax(ntiles, st);  // per-tile max d2, rounded up (D^2 cull)
    const int tile_grid = (int)std::max<int64_t>(1, std::min<int64_t>((ntiles + 7) / 8, num_sms() * 8));
    k_tile_boxes<<<tile_grid, 256, 0, st>>>(spts.p, n, tbox.p, rows.len ? slen.p : nullptr,
                                            tlen.p);
    DArr<float4> cbox(ntiles, st);
    k_cull_boxes<<<grid_cap(ntiles), 256, 0, st>>>(tbox.p, ntiles, cbox.p);
    JB_LAUNCH_CHECK();

    LloydCtx L;
    L.spts = spts.p;
    L.orig = orig.p;
    L.pos = pos.p;
    L.n = n;
    L.k = (int)k;
    L.Ex = fx_exponent_for(mx * (double)n * 1.001 + 1e-300);
    L.Ey = fx_exponent_for(my * (double)n * 1.001 + 1e-300);
    L.st = st;
    L.centers.alloc(2 * k, st);
    L.labs.alloc(n, st);
    L.acc.alloc(7 * k, st);
    L.flags.alloc(1, st);
    L.empties.alloc(k + 4, st);  // list | n_empty | converged | iterations | gate
    L.diag.alloc(4, st);
    L.empties.zero();
    {
        const int G = grid_side_for(k), cap = 32;
        L.cg = make_grid_desc(bb.xmin, bb.xmax, bb.ymin, bb.ymax, G, cap);
        L.cg_cnt.alloc((size_t)G * G, st);
        L.cg_cand.alloc((size_t)G * G * cap, st);
        L.cg.cnt = L.cg_cnt.p;
        L.cg.cand = L.cg_cand.p;
    }
    if (rows.len) {  // exact row grid over the integer piece lengths (jb_rowgrid.cuh)
        // every piece length up to 4096 gets a row (a length beyond the rows
        // is compared with all k centers, every iteration); long rows hold
        // few points, and only the occupied segments are ever built
        const int32_t R = std::min<int32_t>(std::max<int32_t>(rows.max_len, 1), 4096);
        const int64_t budget = std::min<int64_t>(1 << 23, std::max<int64_t>(1 << 16, (int64_t)R * 2048));
        L.rg = make_row_grid_desc(bb.ymin, bb.ymax, rows.scl, rows.sl, rows.max_len, budget, 4096);
        static const double slack_h = getenv("JB_RG_SLACK") ? atof(getenv("JB_RG_SLACK")) : 4.0;
        L.rg.slack = slack_h * L.rg.h;  // persistent loop: rebuild only after slack / 2 of movement
        L.rg_cell.alloc((size_t)L.rg.R * L.rg.Gy, st);
        L.rg.cell = L.rg_cell.p;
        L.rg_spill.alloc((size_t)L.rg.R * L.rg.Gy * kSpill, st);
        L.rg.spill = L.rg_spill.p;
        L.slen = slen.p;
        L.tlen = tlen.p;
        // only segments holding points are rebuilt each iteration; the others
        // stay "not built" (all ones) and send their queries to the fallback
        JB_CUDA(cudaMemsetAsync(L.rg_cell.p, 0xFF, sizeof(uint64_t) * L.rg.R * L.rg.Gy, st));
        const int nseg_all = row_grid_segments(L.rg);
        DArr<int> occ(nseg_all, st);
        occ.zero();
        if (n > 0)
            k_row_occupancy<<<grid_cap(n), 256, 0, st>>>(L.rg, spts.p, slen.p, n, occ.p);
        JB_LAUNCH_CHECK();
        std::vector<int> h_occ = occ.to_host(nseg_all), blocks;
        for (int b = 0; b < nseg_all; ++b)
            if (h_occ[b]) blocks.push_back(b);
        L.rg_nblocks = (int)blocks.size();
        L.rg_blocks.alloc(std::max<size_t>(blocks.size(), 1), st);
        L.rg_blocks.upload(blocks.data(), blocks.size());
        // the 2-D grid would only serve mixed-length tiles (-> per point) and
        // lengths beyond the rows / overflowing row cells (-> all centers)
        L.cg.G = 0;
    }
    L.tbox = tbox.p;
    L.ntiles = ntiles;
    L.tlab.alloc(L.nstate(), st);
    L.sbox.alloc(std::max<int64_t>(L.nsuper(), 1), st);
    L.slenc.alloc(std::max<int64_t>(L.nsuper(), 1), st);
    if (ntiles > 0)
        k_super_boxes<<<(int)std::max<int64_t>(1, std::min<int64_t>((L.nsuper() + 7) / 8, num_sms() * 8)),
                        256, 0, st>>>(tbox.p, rows.len ? tlen.p : nullptr, ntiles, L.sbox.p,
                                      L.slenc.p);
    L.work.alloc(std::max<int64_t>(ntiles, 1), st);
    L.tnew.alloc(std::max<int64_t>(ntiles, 1), st);
    L.swork.alloc(std::max<int64_t>(L.nsuper(), 1), st);
    L.nswork.alloc(1, st);
    L.nswork.zero();
    L.nwork.alloc(1, st);
    JB_CUDA(cudaMemsetAsync(L.tlab.p, 0xFF, sizeof(uint32_t) * L.nstate(), st));
    JB_CUDA(cudaFuncSetAttribute(k_lloyd_work<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)L.smem(true)));
    JB_CUDA(cudaFuncSetAttribute(k_lloyd_work<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)L.smem(false)));

    const int nblocks = (int)((n + D2_R - 1) / D2_R);
    DArr<uint32_t> d2_work(ntiles, st);
    DArr<unsigned long long> d2_nwork(1, st);
    const int cull_grid =
        (int)std::max<int64_t>(1, std::min<int64_t>((ntiles + 1023) / 1024, num_sms() * 8));
    DArr<double> d2s(n, st);
    DArr<unsigned long long> part(2 * nblocks, st);
    DArr<SeedState> ss(1, st);
    DArr<int64_t> chosen(k, st);
    DArr<unsigned long long> d2_diag(1, st);
    d2_diag.zero();

    double best_sse = 0.0;
    for (uint64_t restart = 0; restart < n_init; ++restart) {
        // ---- d2_seed ----
        SeedState h{*cursor, 0, 0, 0};
        ss.upload(&h, 1);
        part.zero();
        // all rounds in one cooperative launch when the device can co-schedule
        // it (two-limb partials, E - 18: k_d2_seed), else -- or from the
        // round where it stops -- one pick + cull + update launch per round
        // on the 128-bit scale
        const D2Plan plan = (k > 1 && !getenv("JB_D2_NO_PERSIST")) ? d2_plan(ntiles, nblocks)
                                                                    : D2Plan{};
        const int Einit = plan.G ? Ed2 - 18 : Ed2;
        k_pick_first<<<1, 1, 0, st>>>(d_raw, (uint64_t)n, ss.p, chosen.p);
        JB_LAUNCH_CHECK();
        // the cooperative kernel's partials (two-limb layout), filled by the init round
        DArr<unsigned long long> part2(plan.G ? 2 * (size_t)std::max(nblocks, 1) : 0, st);
        if (plan.G) part2.zero();
        {
            JB_PROF("d2_update", st);
            k_d2_tiles<<<tile_grid, 256, 0, st>>>(spts.p, orig.p, pos.p, n, nullptr, nullptr,
                                                  tmax.p, d2s.p, ss.p, 1, Einit,
                                                  plan.G ? part2.p : part.p, nullptr, nullptr,
                                                  d2_diag.p, plan.G ? 1 : 0);
        }
        JB_LAUNCH_CHECK();
        uint64_t c_from = 1;
        if (plan.G) {
            c_from = d2_seed_persistent(plan, spts.p, orig.p, pos.p, n, cbox.p, tmax.p, ntiles,
                                        d2s.p, part.p, part2.p, nblocks, Ed2 - 18, d_raw, ss.p,
                                        chosen.p, (int)k, d2_diag.p, st);
            if (c_from < k) {  // rebuild the partials on the 128-bit scale
                part.zero();
                k_part_rebuild<<<grid_cap(n), 256, 0, st>>>(d2s.p, orig.p, n, Ed2, part.p);
                JB_LAUNCH_CHECK();
            }
        }
        // cluster pick when every CTA's share of the partials fits its smem
        const size_t pick_smem = 16 * (size_t)((nblocks + PC - 1) / PC);
        const bool cluster_pick = pick_smem <= kPickClusterSmem;
        if (cluster_pick && c_from < k)
            JB_CUDA(cudaFuncSetAttribute(k_pick_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(pick_smem, 16)));
        for (uint64_t c = c_from; c < k; ++c) {
            {
                JB_PROF("d2_pick", st);
                if (cluster_pick)
                    k_pick_cluster<<<PC, PICK_TB, std::max<size_t>(pick_smem, 16), st>>>(
                        d_raw, d2s.p, pos.p, n, nblocks, part.p, Ed2, ss.p, chosen.p, (int)c,
                        d2_nwork.p);
                else
                    k_pick<<<1, PICK_TB, 0, st>>>(d_raw, d2s.p, pos.p, n, nblocks, part.p, Ed2,
                                                  ss.p, chosen.p, (int)c, d2_nwork.p);
            }
            JB_LAUNCH_CHECK();
            if (c + 1 < k) {
                JB_PROF("d2_update", st);
                k_d2_cull<<<cull_grid, 256, 0, st>>>(cbox.p, tmax.p, ntiles, spts.p, pos.p, ss.p,
                                                     d2_work.p, d2_nwork.p, nullptr);
                k_d2_tiles<<<tile_grid, 256, 0, st>>>(spts.p, orig.p, pos.p, n, d2_work.p,
                                                      d2_nwork.p, tmax.p, d2s.p, ss.p, 0, Ed2,
                                                      part.p, nullptr, nullptr, d2_diag.p);
                JB_LAUNCH_CHECK();
            }
        }
        k_copy_center<<<1, 256, 0, st>>>(spts.p, pos.p, chosen.p, (int)k, L.centers.p);
        JB_LAUNCH_CHECK();
        ss.download(&h, 1);
        JB_CUDA(cudaStreamSynchronize(st));
        if (h.cursor > raw_count) throw Error(INTERNAL, "rng stream exhausted");
        *cursor = h.cursor;
        if (dbg_on()) {
            auto ch = chosen.to_host(k);
            auto cc = L.centers.to_host(2 * k);
            fprintf(stderr, "[jb] seeds: S=%lld Ed2=%d Ex=%d Ey=%d chosen[0..3]=%lld %lld %lld %lld hash=%016llx cursor=%llu\n",
                    (long long)n, Ed2, L.Ex, L.Ey, (long long)ch[0], (long long)ch[std::min<uint64_t>(1, k - 1)],
                    (long long)ch[std::min<uint64_t>(2, k - 1)], (long long)ch[k - 1],
                    (unsigned long long)dbg_hash(cc.data(), 16 * k), (unsigned long long)h.cursor);
        }
        JB_TRACE("kmeans: d2 seeding", st);

        // ---- Lloyd (lloyd_once :200-220) ----
        // Iterations are launched in batches; device-side state gates every
        // kernel (pending empty-cluster repair, convergence) so the host
        // syncs once per batch. Iterations launched after convergence are
        // no-ops; the count is taken on the device.
        L.acc.zero();
        JB_CUDA(cudaMemsetAsync(L.tlab.p, 0xFF, sizeof(uint32_t) * L.nstate(), st));
        JB_CUDA(cudaMemsetAsync(L.empties.p + L.k, 0, 3 * sizeof(int), st));
        L.diag.zero();
        JB_CUDA(cudaMemsetAsync(L.flags.p, 0, 8, st));
        JB_CUDA(cudaMemsetAsync(L.nwork.p, 0, 8, st));
        JB_CUDA(cudaMemsetAsync(L.nswork.p, 0, 8, st));
        lloyd_assign(L, true, false);  // assign_all(points, seeds) (:204)
        JB_CUDA(cudaMemsetAsync(L.flags.p, 0, 8, st));
        JB_CUDA(cudaMemsetAsync(L.nwork.p, 0, 8, st));
        JB_CUDA(cudaMemsetAsync(L.nswork.p, 0, 8, st));
        uint64_t it = 0;
        const uint64_t kBatch = dbg_on() ? 1 : 16;
        while (it < max_iters) {
            const uint64_t B = std::min<uint64_t>(kBatch, max_iters - it);
            if (!lloyd_persistent(L, (int)std::min<uint64_t>(max_iters - it, 1u << 30))) {
                for (uint64_t b = 0; b < B; ++b) {
                    lloyd_means(L, true);          // update_means ...
                    lloyd_assign(L, false, true);  // ... assign_all, label comparison
                    k_iter_end<<<1, 1, 0, st>>>(L.empties.p + L.k, L.flags.p, L.nwork.p,
                                                L.nswork.p, L.diag.p);
                    JB_LAUNCH_CHECK();
                }
            }
            LoopState h = lloyd_state(L);
            it = (uint64_t)h.iters;
            if (dbg_on()) {
                auto cc = L.centers.to_host(2 * k);
                auto dg = L.diag.to_host(4);
                fprintf(stderr, "[jb] iter %d: empty=%d conv=%d cum_changed=%llu cum_tiles=%llu cum_need_supers=%llu centers=%016llx\n",
                        h.iters, h.n_empty, h.converged, dg[1], dg[0], dg[2],
                        (unsigned long long)dbg_hash(cc.data(), 16 * k));
            }
            if (h.converged) break;
            if (h.n_empty) {  // empty clusters: re-seed on the host path, finish the iteration
                lloyd_repair(L, h.n_empty);
                lloyd_assign(L, false, true);
                k_iter_end<<<1, 1, 0, st>>>(L.empties.p + L.k, L.flags.p, L.nwork.p, L.nswork.p,
                                            L.diag.p);
                JB_LAUNCH_CHECK();
                h = lloyd_state(L);
                it = (uint64_t)h.iters;
                if (h.converged) break;
            }
        }
        JB_CUDA(cudaMemsetAsync(L.empties.p + L.k, 0, 2 * sizeof(int), st));  // ungate
        {
            unsigned long long diag[2];
            JB_CUDA(cudaMemcpyAsync(diag, L.diag.p, 16, cudaMemcpyDeviceToHost, st));
            JB_CUDA(cudaStreamSynchronize(st));
            out.work_tiles = diag[0];
            out.changed_labels = diag[1];
            JB_CUDA(cudaMemcpyAsync(diag, d2_diag.p, 8, cudaMemcpyDeviceToHost, st));
            JB_CUDA(cudaStreamSynchronize(st));
            out.d2_tiles = diag[0];
        }
        lloyd_update_means_sync(L);
        JB_TRACE("kmeans: lloyd", st);
        double sse = 0.0;
        if (n_init > 1) {
            DArr<unsigned long long> sacc(2, st);
            sacc.zero();
            k_sse<<<grid_cap(n), 256, 0, st>>>(spts.p, n, L.labs.p, L.centers.p, Ed2, sacc.p);
            JB_LAUNCH_CHECK();
            auto hs = sacc.to_host(2);
            sse = fx_to_double(fx_load(hs.data()), Ed2);
        }
        if (restart == 0 || sse < best_sse) {
            best_sse = sse;
            out.k = k;
            out.centers = L.centers.to_host(2 * k);
            if (n_init == 1) {  // unsorted on demand (kmeans_labels)
                out.slabs = std::move(L.labs);
            } else {
                out.slabs.alloc(n, st);
                JB_CUDA(cudaMemcpyAsync(out.slabs.p, L.labs.p, sizeof(uint32_t) * n,
                                        cudaMemcpyDeviceToDevice, st));
            }
            JB_LAUNCH_CHECK();
            out.iterations = it;
            out.sse = sse;
        }
    }
    out.sorig = std::move(orig);
    JB_CUDA(cudaStreamSynchronize(st));
}

void kmeans_labels(KMeansOut& out, int64_t n, cudaStream_t st) {
    if (out.labels.p || !out.slabs.p) return;
    out.labels.alloc(std::max<int64_t>(n, 1), st);
    if (n > 0) {
        k_unsort_labels<<<grid_cap(n), 256, 0, st>>>(out.slabs.p, out.sorig.p, n, out.labels.p);
        JB_LAUNCH_CHECK();
    }
}

}  // namespace jb

// ===========================================================================
// Distributed k-means++ (one joint fit sharded over ranks).
//
// Every rank holds the sample entries whose pieces it owns (global sample
// positions gpos, ascending). All exchanges are exact integers or the
// owner's exact doubles, so every rank makes the same decisions as the
// single-GPU path:
//  * D^2 round: this rank's per-global-block partial sums -> allgather ->
//    exact global prefix on the host -> block; the block's 2048 weights from
//    their owners -> element; the chosen point's coordinates from its owner.
//  * Lloyd iteration: this rank's exact cluster-sum deltas and change count
//    -> allgather -> identical global accumulators on every rank.
//  * Empty clusters: per-rank farthest candidates -> global (max d, lowest
//    global sample position) -> applied by every rank (labels by the owner).

namespace jb {
namespace {

// ---------------------------------------------------------------------------
// Device-side exchanges of the joint fit. Every exchanged quantity is a
// vector of u64 words whose word-wise sum over ranks is the wanted result
// (l3 limbs, 32-bit halves of int128 partials, or one owner's bits with
// zeros elsewhere), so a sum all-reduce is exact and identical on every
// rank. Transport: NCCL on the fit's stream when every rank drives its own
// GPU (the libnccl the process already loaded -- torch's -- else the
// system's, found at run time), else staged through the caller's host
// allgather (jb_comm), e.g. gloo ranks sharing one GPU in the tests.

struct NcclApi {
    bool tried = false;
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;
std::map<std::tuple<const void*, int, int, int>, ncclComm_t> g_nccl_comms;

const NcclApi* nccl_api() {
    if (!g_nccl.tried) {
        g_nccl.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (h) {
            g_nccl.get_unique_id = (decltype(g_nccl.get_unique_id))dlsym(h, "ncclGetUniqueId");
            g_nccl.comm_init_rank = (decltype(g_nccl.comm_init_rank))dlsym(h, "ncclCommInitRank");
            g_nccl.all_reduce = (decltype(g_nccl.all_reduce))dlsym(h, "ncclAllReduce");
            g_nccl.error_string = (decltype(g_nccl.error_string))dlsym(h, "ncclGetErrorString");
            if (g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.all_reduce &&
                g_nccl.error_string)
                g_nccl.h = h;
        }
    }
    return g_nccl.h ? &g_nccl : nullptr;
}

struct DevComm {
    const Comm* cm = nullptr;
    ncclComm_t nc = nullptr;  // null: staged through cm's host allgather

    // a collective call: the same on every rank (the bus-id exchange and the
    // NCCL bootstrap go through the host allgather)
    void init(const Comm& c, cudaStream_t st) {
        cm = &c;
        if (!c.dist() || getenv("JB_DIST_STAGED")) return;
        int dev = 0;
        JB_CUDA(cudaGetDevice(&dev));
        char bus[32] = {0};
        JB_CUDA(cudaDeviceGetPCIBusId(bus, sizeof bus, dev));
        std::vector<char> all(32 * (size_t)c.world);
        c.allgather(bus, 32, all.data());
        bool distinct = true;  // NCCL needs one GPU per rank
        for (int a = 0; a < c.world && distinct; ++a)
            for (int b = a + 1; b < c.world; ++b)
                if (!strncmp(&all[32 * a], &all[32 * b], 32)) distinct = false;
        int ok = distinct && nccl_api() != nullptr;
        std::vector<int> oks(c.world);
        c.allgather(&ok, sizeof ok, oks.data());
        for (int v : oks) ok &= v;
        if (!ok) return;
        std::lock_guard<std::mutex> lk(g_nccl_mu);
        const auto key = std::make_tuple((const void*)c.c, c.rank, c.world, dev);
        auto it = g_nccl_comms.find(key);
        if (it != g_nccl_comms.end()) {
            nc = it->second;
            return;
        }
        ncclUniqueId id;
        memset(&id, 0, sizeof id);
        if (c.rank == 0 && g_nccl.get_unique_id(&id) != ncclSuccess)
            throw Error(NCCL_ERROR, "ncclGetUniqueId failed");
        std::vector<ncclUniqueId> ids(c.world);
        c.allgather(&id, sizeof id, ids.data());
        const ncclResult_t r = g_nccl.comm_init_rank(&nc, c.world, ids[0], c.rank);
        if (r != ncclSuccess)
            throw Error(NCCL_ERROR, std::string("ncclCommInitRank: ") + g_nccl.error_string(r));
        g_nccl_comms[key] = nc;
        (void)st;
    }

    // p[0..count) = word-wise sum over ranks (mod 2^64), in stream order
    void allreduce_u64(unsigned long long* p, size_t count, cudaStream_t st) const {
        if (!cm->dist() || count == 0) return;
        if (nc) {
            const ncclResult_t r =
                g_nccl.all_reduce(p, p, count, ncclUint64, ncclSum, nc, st);
            if (r != ncclSuccess)
                throw Error(NCCL_ERROR, std::string("ncclAllReduce: ") + g_nccl.error_string(r));
            return;
        }
        std::vector<unsigned long long> h(count);
        JB_CUDA(cudaMemcpyAsync(h.data(), p, 8 * count, cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        const auto all = cm->gather(h);
        for (size_t i = 0; i < count; ++i) {
            unsigned long long v = 0;
            for (int r = 0; r < cm->world; ++r) v += all[(size_t)r * count + i];
            h[i] = v;
        }
        JB_CUDA(cudaMemcpyAsync(p, h.data(), 8 * count, cudaMemcpyHostToDevice, st));
        JB_CUDA(cudaStreamSynchronize(st));
    }
    bool nccl() const { return nc != nullptr; }
};

__global__ void k_gkey(const uint32_t* __restrict__ gpos, const uint32_t* __restrict__ orig,
                       int64_t n, uint32_t* __restrict__ gkey) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        gkey[r] = gpos[orig[r]];
}

// local entry holding global sample position q (gpos ascending), or -1
__global__ void k_find_gpos(const uint32_t* __restrict__ gpos, int64_t n, uint64_t q,
                            long long* __restrict__ out) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (gpos[m] < q) lo = m + 1;
        else hi = m;
    }
    *out = (lo < n && gpos[lo] == q) ? lo : -1;
}

// d2 of this rank's entries of global block b into w[0..R) (zeros elsewhere)
__global__ void k_block_weights(const uint32_t* __restrict__ gpos, const uint32_t* __restrict__ pos,
                                int64_t n, const double* __restrict__ d2s, uint64_t b,
                                double* __restrict__ w) {
    const uint64_t q0 = b * D2_R, q1 = q0 + D2_R;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (gpos[m] < q0) lo = m + 1;
        else hi = m;
    }
    for (int64_t i = lo + threadIdx.x; i < n && gpos[i] < q1; i += blockDim.x)
        w[gpos[i] - q0] = d2s[pos[i]];
}

// largest global position with d2 > 0 (roundoff spill of weighted_index)
__global__ void k_last_positive(const uint32_t* __restrict__ gpos, const uint32_t* __restrict__ pos,
                                int64_t n, const double* __restrict__ d2s,
                                long long* __restrict__ out) {
    long long best = -1;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        if (d2s[pos[i]] > 0.0) best = max(best, (long long)gpos[i]);
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

// re-seed empty cluster c at the globally chosen far point (update_means :193-196)
__global__ void k_repair_dist(unsigned long long* __restrict__ acc, double* __restrict__ centers,
                              uint32_t* __restrict__ labs, uint32_t* __restrict__ tlab, int k,
                              int Ex, int Ey, int c, int donor, double px, double py,
                              long long owner_r, int64_t ntiles) {
    const i128 fx = fx_from_double(px, Ex), fy = fx_from_double(py, Ey);
    ClusterAcc a{acc, acc + 3 * k, acc + 6 * k};
    l3_store(a.sx + 3 * donor, l3_load(a.sx + 3 * donor) - fx);
    l3_store(a.sy + 3 * donor, l3_load(a.sy + 3 * donor) - fy);
    a.cnt[donor] -= 1;
    l3_store(a.sx + 3 * c, fx);
    l3_store(a.sy + 3 * c, fy);
    a.cnt[c] = 1;
    centers[2 * c] = px;
    centers[2 * c + 1] = py;
    if (owner_r >= 0) {
        labs[owner_r] = (uint32_t)c;
        tlab[owner_r / TILE] = MIXED;
        tlab[ntiles + owner_r / (TILE * 32)] = MIXED;
    }
}

// ---- device-side distributed D^2 round (no host round trip) ----

// int128 (lo, hi) partials <-> three additive words (bits 0-31 and 32-63 of
// lo, and hi): a word-wise sum over ranks recombines to the exact total
__global__ void k_part_split(const unsigned long long* __restrict__ part, int nblocks,
                             unsigned long long* __restrict__ p3) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += gridDim.x * blockDim.x) {
        const unsigned long long lo = part[2 * b], hi = part[2 * b + 1];
        p3[3 * b] = lo & 0xFFFFFFFFull;
        p3[3 * b + 1] = lo >> 32;
        p3[3 * b + 2] = hi;
    }
}

__global__ void k_part_join(const unsigned long long* __restrict__ p3, int nblocks,
                            unsigned long long* __restrict__ gpart) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += gridDim.x * blockDim.x) {
        const u128 v = (u128)p3[3 * b] + ((u128)p3[3 * b + 1] << 32) + ((u128)p3[3 * b + 2] << 64);
        gpart[2 * b] = (unsigned long long)v;
        gpart[2 * b + 1] = (unsigned long long)(v >> 64);
    }
}

struct DPick {
    unsigned long long U[2], before[2];
    long long fb;  // crossing block, -1: none (degenerate round or spill)
    int deg;       // this round: every remaining point duplicates a center
    int spill;     // sticky: a roundoff spill happened (host re-runs the seeding)
};

// total, u and the crossing block of the global partial sums (k_pick's
// arithmetic): 1024 threads over contiguous block ranges, one exact scan
__global__ void __launch_bounds__(PICK_TB) k_dpick_block(const uint64_t* __restrict__ raw,
                                                         const unsigned long long* __restrict__ gpart,
                                                         int nblocks, int E, SeedState* ss,
                                                         int64_t* __restrict__ chosen, int c,
                                                         DPick* dp) {
    __shared__ unsigned long long s_lo[32], s_hi[32];
    __shared__ unsigned long long s_found;
    const int t = threadIdx.x;
    const int per = (nblocks + PICK_TB - 1) / PICK_TB;
    const int b0 = min(nblocks, t * per), b1 = min(nblocks, b0 + per);
    i128 local = 0;
    for (int b = b0; b < b1; ++b) local += fx_load(gpart + 2 * b);
    if (t == 0) s_found = ~0ULL;
    i128 total;
    const i128 ex = block_exscan_i128(local, &total, s_lo, s_hi);
    const double total_d = fx_to_double(total, E);
    if (!(total_d > 0.0)) {  // every remaining point duplicates a center (:120-124)
        if (t == 0) {
            int64_t next = 0;
            for (;;) {
                bool taken = false;
                for (int q = 0; q < c; ++q) taken |= chosen[q] == next;
                if (!taken) break;
                ++next;
            }
            chosen[c] = next;
            ss->degenerate = 1;
            dp->deg = 1;
            dp->fb = -1;
        }
        return;
    }
    const uint64_t x = raw[ss->cursor];
    double canon = __ull2double_rn(x) * 0x1p-64;  // generate_canonical<double,53>
    if (canon >= 1.0) canon = 0x1.fffffffffffffp-1;
    const double u = canon * total_d + 0.0;
    const i128 U = fx_from_double(u, E);
    i128 run = ex;
    int mine = -1;
    for (int b = b0; b < b1; ++b) {
        const i128 v = fx_load(gpart + 2 * b);
        if (U < run + v) {
            mine = b;
            break;
        }
        run += v;
    }
    if (mine >= 0) atomicMin(&s_found, (unsigned long long)mine);
    __syncthreads();
    if (t == 0) {
        dp->deg = 0;
        dp->fb = s_found == ~0ULL ? -1 : (long long)s_found;
        dp->U[0] = (unsigned long long)(u128)U;
        dp->U[1] = (unsigned long long)((u128)U >> 64);
        if (s_found == ~0ULL) dp->spill = 1;
    }
    if (mine >= 0 && (unsigned long long)mine == s_found) {
        dp->before[0] = (unsigned long long)(u128)run;
        dp->before[1] = (unsigned long long)((u128)run >> 64);
    }
}

// this rank's d2 bits of the crossing block's entries (zeros elsewhere)
__global__ void k_dblock_weights(const uint32_t* __restrict__ gpos, const uint32_t* __restrict__ pos,
                                 int64_t n, const double* __restrict__ d2s, const DPick* dp,
                                 unsigned long long* __restrict__ w) {
    if (dp->fb < 0) return;
    const uint64_t q0 = (uint64_t)dp->fb * D2_R, q1 = q0 + D2_R;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (gpos[m] < q0) lo = m + 1;
        else hi = m;
    }
    for (int64_t i = lo + threadIdx.x; i < n && gpos[i] < q1; i += blockDim.x)
        w[gpos[i] - q0] = (unsigned long long)__double_as_longlong(d2s[pos[i]]);
}

// the element inside the crossing block from the gathered weights
__global__ void __launch_bounds__(PICK_TB) k_dpick_elem(const unsigned long long* __restrict__ w,
                                                        DPick* dp, int E, SeedState* ss,
                                                        int64_t* __restrict__ chosen, int c,
                                                        uint64_t S) {
    __shared__ unsigned long long s_lo[32], s_hi[32];
    __shared__ unsigned long long s_found;
    if (dp->deg) return;
    const int t = threadIdx.x;
    if (dp->fb < 0) {  // roundoff spill (:67-70): the host re-runs the seeding
        if (t == 0) chosen[c] = (int64_t)S - 1;
        return;
    }
    if (t == 0) s_found = ~0ULL;
    const uint64_t e0 = (uint64_t)dp->fb * D2_R + 2 * t;
    i128 a = 0, b = 0;
    if (e0 < S) a = fx_from_double(__longlong_as_double((long long)w[2 * t]), E);
    if (e0 + 1 < S) b = fx_from_double(__longlong_as_double((long long)w[2 * t + 1]), E);
    i128 dummy;
    const i128 ex2 = block_exscan_i128(a + b, &dummy, s_lo, s_hi);
    const i128 U = fx_load(dp->U), before = fx_load(dp->before) + ex2;
    unsigned long long hit = ~0ULL;
    if (e0 < S && U < before + a) hit = e0;
    else if (e0 + 1 < S && U < before + a + b) hit = e0 + 1;
    if (hit != ~0ULL) atomicMin(&s_found, hit);
    __syncthreads();
    if (t == 0) {
        if (s_found == ~0ULL) {
            dp->spill = 1;
            chosen[c] = (int64_t)S - 1;
        } else {
            chosen[c] = (int64_t)s_found;
        }
        ss->cursor += 1;
    }
}

// the chosen point's bits from its owner (zeros on the other ranks)
__global__ void k_dcenter_bits(const uint32_t* __restrict__ gpos, const uint32_t* __restrict__ pos,
                               const double2* __restrict__ spts, int64_t n,
                               const int64_t* __restrict__ chosen, int c,
                               unsigned long long* __restrict__ cb) {
    const uint64_t q = (uint64_t)chosen[c];
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (gpos[m] < q) lo = m + 1;
        else hi = m;
    }
    cb[0] = cb[1] = 0;
    if (lo < n && gpos[lo] == q) {
        const double2 p = spts[pos[lo]];
        cb[0] = (unsigned long long)__double_as_longlong(p.x);
        cb[1] = (unsigned long long)__double_as_longlong(p.y);
    }
}

__global__ void k_dstore_center(const unsigned long long* __restrict__ cb, double* __restrict__ centers,
                                int c) {
    centers[2 * c] = __longlong_as_double((long long)cb[0]);
    centers[2 * c + 1] = __longlong_as_double((long long)cb[1]);
}

// Lloyd iteration end of the joint fit (device loop): acc += the all-reduced
// deltas; ++iterations; converged when no label changed anywhere. Gated like
// k_iter_end (pending empty-cluster repair / converged: no-op).
__global__ void k_dist_accum(unsigned long long* __restrict__ acc,
                             unsigned long long* __restrict__ dacc, int k,
                             int* __restrict__ state, unsigned long long* __restrict__ changed,
                             unsigned long long* __restrict__ nwork,
                             unsigned long long* __restrict__ nswork,
                             unsigned long long* __restrict__ diag, int count_iter) {
    if (count_iter && (state[0] | state[1])) return;
    for (int i = threadIdx.x; i < 7 * k; i += blockDim.x) {
        acc[i] += dacc[i];
        dacc[i] = 0;
    }
    if (threadIdx.x == 0) {
        if (count_iter) {
            state[2] += 1;
            diag[0] += *nwork;
            diag[2] += *nswork;
            diag[1] += *changed;
            if (*changed == 0) state[1] = 1;
        }
        *changed = 0;
        *nwork = 0;
        *nswork = 0;
    }
}

struct FarRec {
    double d;
    long long gp;  // global sample position (INT64_MAX: none)
    long long r;   // this rank's sorted position
    double x, y;
    long long donor;
};

}  // namespace

void lloyd_best_dist(const Comm& cm, const PtsView& pv, const uint64_t* d_lidx,
                     const uint32_t* d_gpos, int64_t n, uint64_t S, uint64_t k, uint64_t max_iters,
                     uint64_t n_init, const uint64_t* d_raw, uint64_t raw_count, uint64_t* cursor,
                     const BBox& bb, KMeansOut& out, cudaStream_t st, const PieceRows& rows) {
    if (k < 1) throw Error(INVALID_INPUT, "d2_seed: k must be >= 1");
    if (k > S) throw Error(INVALID_INPUT, "d2_seed: k exceeds points");
    if (k > 2048) throw Error(INVALID_INPUT, "k > 2048 is not supported by the Lloyd kernel");
    if (S >= (1ULL << 32)) throw Error(INVALID_INPUT, "k-means on more than 2^32 points");
    const double mx = std::max(std::fabs(bb.xmin), std::fabs(bb.xmax));
    const double my = std::max(std::fabs(bb.ymin), std::fabs(bb.ymax));
    const double wx = bb.xmax - bb.xmin, wy = bb.ymax - bb.ymin;
    const double d2max = (wx * wx + wy * wy) * (1.0 + 1e-9) + 1e-300;
    const int Ed2 = fx_exponent_for(d2max * (double)S * 1.001);
    const int64_t nn = std::max<int64_t>(n, 1);

    // ---- Morton order of this rank's points ----
    DArr<double2> spts(nn, st);
    DArr<uint32_t> orig(nn, st), pos(nn, st), gkey(nn, st);
    DArr<int32_t> slen(rows.len ? nn : 0, st), tlen(std::max<int64_t>((n + TILE - 1) / TILE, 1), st);
    if (n > 0) {
        DArr<uint32_t> keys(n, st), skeys(n, st), vals(n, st);
        const double sx = wx > 0 ? 65535.0 / wx : 0.0, sy = wy > 0 ? 65535.0 / wy : 0.0;
        DArr<double2> cpts(n, st);
        k_morton<<<grid_cap(n), 256, 0, st>>>(pv, d_lidx, n, bb.xmin, sx, bb.ymin, sy, keys.p,
                                              vals.p, cpts.p, rows.len);
        JB_LAUNCH_CHECK();
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, vals.p, orig.p, n, 0, 32,
                                        st);
        DArr<uint8_t> tmp(tb, st);
        cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, vals.p, orig.p, n, 0, 32, st);
        k_sorted_gather<<<grid_cap(n), 256, 0, st>>>(cpts.p, orig.p, n, spts.p, pos.p, pv.scl,
                                                     pv.sl, rows.len ? slen.p : nullptr);
        k_gkey<<<grid_cap(n), 256, 0, st>>>(d_gpos, orig.p, n, gkey.p);
        JB_LAUNCH_CHECK();
    }
    const int64_t ntiles = (n + TILE - 1) / TILE;
    DArr<double4> tbox(std::max<int64_t>(ntiles, 1), st);
    DArr<float> tmax(std::max<int64_t>(ntiles, 1), st);  // per-tile max d2, rounded up
    const int tile_grid = (int)std::max<int64_t>(1, std::min<int64_t>((ntiles + 7) / 8, num_sms() * 8));
    if (n > 0)
        k_tile_boxes<<<tile_grid, 256, 0, st>>>(spts.p, n, tbox.p, rows.len ? slen.p : nullptr,
                                                tlen.p);
    DArr<float4> cbox(std::max<int64_t>(ntiles, 1), st);
    if (n > 0) k_cull_boxes<<<grid_cap(ntiles), 256, 0, st>>>(tbox.p, ntiles, cbox.p);
    JB_LAUNCH_CHECK();

    LloydCtx L;
    L.spts = spts.p;
    L.orig = gkey.p;  // tie-breaks by global sample position
    L.pos = pos.p;
    L.n = n;
    L.k = (int)k;
    L.Ex = fx_exponent_for(mx * (double)S * 1.001 + 1e-300);
    L.Ey = fx_exponent_for(my * (double)S * 1.001 + 1e-300);
    L.st = st;
    L.centers.alloc(2 * k, st);
    L.labs.alloc(nn, st);
    L.acc.alloc(7 * k, st);
    L.dacc.alloc(7 * k + 1, st);  // deltas + change count (changed_ptr)
    L.use_dacc = true;
    L.flags.alloc(1, st);
    L.empties.alloc(k + 4, st);
    L.empties.zero();
    L.diag.alloc(4, st);
    {
        const int G = grid_side_for(k), cap = 32;
        L.cg = make_grid_desc(bb.xmin, bb.xmax, bb.ymin, bb.ymax, G, cap);
        L.cg_cnt.alloc((size_t)G * G, st);
        L.cg_cand.alloc((size_t)G * G * cap, st);
        L.cg.cnt = L.cg_cnt.p;
        L.cg.cand = L.cg_cand.p;
    }
    if (rows.len) {  // exact row grid over the integer piece lengths (jb_rowgrid.cuh)
        const int32_t R = std::min<int32_t>(std::max<int32_t>(rows.max_len, 1), 4096);
        const int64_t budget = std::min<int64_t>(1 << 23, std::max<int64_t>(1 << 16, (int64_t)R * 2048));
        L.rg = make_row_grid_desc(bb.ymin, bb.ymax, rows.scl, rows.sl, rows.max_len, budget, 4096);
        L.rg_cell.alloc((size_t)L.rg.R * L.rg.Gy, st);
        L.rg.cell = L.rg_cell.p;
        L.rg_spill.alloc((size_t)L.rg.R * L.rg.Gy * kSpill, st);
        L.rg.spill = L.rg_spill.p;
        L.slen = slen.p;
        L.tlen = tlen.p;
        // only segments holding points are rebuilt each iteration; the others
        // stay "not built" (all ones) and send their queries to the fallback
        JB_CUDA(cudaMemsetAsync(L.rg_cell.p, 0xFF, sizeof(uint64_t) * L.rg.R * L.rg.Gy, st));
        const int nseg_all = row_grid_segments(L.rg);
        DArr<int> occ(nseg_all, st);
        occ.zero();
        if (n > 0)
            k_row_occupancy<<<grid_cap(n), 256, 0, st>>>(L.rg, spts.p, slen.p, n, occ.p);
        JB_LAUNCH_CHECK();
        std::vector<int> h_occ = occ.to_host(nseg_all), blocks;
        for (int b = 0; b < nseg_all; ++b)
            if (h_occ[b]) blocks.push_back(b);
        L.rg_nblocks = (int)blocks.size();
        L.rg_blocks.alloc(std::max<size_t>(blocks.size(), 1), st);
        L.rg_blocks.upload(blocks.data(), blocks.size());
        // the 2-D grid would only serve mixed-length tiles (-> per point) and
        // lengths beyond the rows / overflowing row cells (-> all centers)
        L.cg.G = 0;
    }
    L.tbox = tbox.p;
    L.ntiles = ntiles;
    L.tlab.alloc(L.nstate(), st);
    L.sbox.alloc(std::max<int64_t>(L.nsuper(), 1), st);
    L.slenc.alloc(std::max<int64_t>(L.nsuper(), 1), st);
    if (ntiles > 0)
        k_super_boxes<<<(int)std::max<int64_t>(1, std::min<int64_t>((L.nsuper() + 7) / 8, num_sms() * 8)),
                        256, 0, st>>>(tbox.p, rows.len ? tlen.p : nullptr, ntiles, L.sbox.p,
                                      L.slenc.p);
    L.work.alloc(std::max<int64_t>(ntiles, 1), st);
    L.tnew.alloc(std::max<int64_t>(ntiles, 1), st);
    L.swork.alloc(std::max<int64_t>(L.nsuper(), 1), st);
    L.nswork.alloc(1, st);
    L.nswork.zero();
    L.nwork.alloc(1, st);
    JB_CUDA(cudaFuncSetAttribute(k_lloyd_work<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)L.smem(true)));
    JB_CUDA(cudaFuncSetAttribute(k_lloyd_work<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)L.smem(false)));

    const uint64_t nblocks = (S + D2_R - 1) / D2_R;
    DArr<uint32_t> d2_work(std::max<int64_t>(ntiles, 1), st);
    DArr<unsigned long long> d2_nwork(1, st);
    const int cull_grid =
        (int)std::max<int64_t>(1, std::min<int64_t>((ntiles + 1023) / 1024, num_sms() * 8));
    DArr<double> d2s(nn, st);
    DArr<unsigned long long> part(2 * nblocks, st);
    DArr<SeedState> ss(1, st);
    DArr<double2> cur(1, st);
    DArr<double> wblk(D2_R, st);
    DArr<long long> dll(1, st);

    // the engine draws the seeding consumes (identical on every rank)
    const uint64_t tail_n = std::min<uint64_t>(raw_count - *cursor, (k + 1) * n_init + 4096);
    std::vector<uint64_t> raw_h(tail_n);
    JB_CUDA(cudaMemcpyAsync(raw_h.data(), d_raw + *cursor, 8 * tail_n, cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    const uint64_t raw_base = *cursor;
    auto draw = [&](uint64_t at) {
        if (at - raw_base >= tail_n) throw Error(INTERNAL, "rng stream exhausted");
        return raw_h[at - raw_base];
    };

    // coordinates of global sample position q, from its owner
    auto center_of = [&](uint64_t q) -> std::pair<double, double> {
        struct Rec {
            long long has;
            double x, y;
        } rec{0, 0.0, 0.0};
        if (n > 0) {
            k_find_gpos<<<1, 1, 0, st>>>(d_gpos, n, q, dll.p);
            long long i = -1;
            dll.download(&i, 1);
            JB_CUDA(cudaStreamSynchronize(st));
            if (i >= 0) {
                uint64_t li;
                double2 p;
                JB_CUDA(cudaMemcpyAsync(&li, d_lidx + i, 8, cudaMemcpyDeviceToHost, st));
                JB_CUDA(cudaStreamSynchronize(st));
                if (pv.pts) {
                    JB_CUDA(cudaMemcpyAsync(&p, pv.pts + li, 16, cudaMemcpyDeviceToHost, st));
                    JB_CUDA(cudaStreamSynchronize(st));
                } else {  // the point from its piece (k_scale's expressions, host IEEE)
                    int32_t L;
                    double I;
                    JB_CUDA(cudaMemcpyAsync(&L, pv.len + li, 4, cudaMemcpyDeviceToHost, st));
                    JB_CUDA(cudaMemcpyAsync(&I, pv.inc + li, 8, cudaMemcpyDeviceToHost, st));
                    JB_CUDA(cudaStreamSynchronize(st));
                    p = make_double2(pv.scl * (double)L / pv.sl, I / pv.si);
                }
                rec = Rec{1, p.x, p.y};
            }
        }
        std::vector<Rec> all(cm.world);
        cm.allgather(&rec, sizeof rec, all.data());
        for (const auto& r : all)
            if (r.has) return {r.x, r.y};
        throw Error(INTERNAL, "distributed seeding: no owner for a sample position");
    };

    auto repair_dist = [&]() {  // update_means :181-197 across ranks
        lloyd_means(L, false);
        int ne = 0;
        JB_CUDA(cudaMemcpyAsync(&ne, L.empties.p + L.k, sizeof(int), cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        if (!ne) return;
        std::vector<int> em(ne);
        L.empties.download(em.data(), ne);
        JB_CUDA(cudaStreamSynchronize(st));
        const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, num_sms() * 4));
        if (L.far_blk.n < (size_t)(3 * nblk)) L.far_blk.alloc(3 * nblk, st);
        for (int c : em) {
            FarRec mine{-1.0, INT64_MAX, -1, 0.0, 0.0, -1};
            if (n > 0) {
                k_far_block<<<nblk, 256, 0, st>>>(spts.p, gkey.p, n, L.labs.p, L.centers.p,
                                                  L.cacc().cnt, L.far_blk.p);
                JB_LAUNCH_CHECK();
                auto blk = L.far_blk.to_host(3 * nblk);
                for (int b = 0; b < nblk; ++b) {
                    double d;
                    memcpy(&d, &blk[3 * b], 8);
                    const long long gp = (long long)blk[3 * b + 1];
                    if (d > mine.d || (d == mine.d && gp < mine.gp)) {
                        mine.d = d;
                        mine.gp = gp;
                        mine.r = (long long)blk[3 * b + 2];
                    }
                }
                if (mine.r >= 0) {
                    double2 p;
                    uint32_t lab;
                    JB_CUDA(cudaMemcpyAsync(&p, spts.p + mine.r, 16, cudaMemcpyDeviceToHost, st));
                    JB_CUDA(cudaMemcpyAsync(&lab, L.labs.p + mine.r, 4, cudaMemcpyDeviceToHost, st));
                    JB_CUDA(cudaStreamSynchronize(st));
                    mine.x = p.x;
                    mine.y = p.y;
                    mine.donor = lab;
                }
            }
            std::vector<FarRec> all(cm.world);
            cm.allgather(&mine, sizeof mine, all.data());
            int owner = -1;
            FarRec best{-1.0, INT64_MAX, -1, 0.0, 0.0, -1};
            for (int r = 0; r < cm.world; ++r)
                if (all[r].r >= 0 &&
                    (all[r].d > best.d || (all[r].d == best.d && all[r].gp < best.gp))) {
                    best = all[r];
                    owner = r;
                }
            if (owner < 0) {  // no cluster with count > 1: far_i stays 0 (global position 0)
                const auto xy = center_of(0);
                // owner of position 0 supplies its label
                struct L0 {
                    long long has, lab, r;
                } l0{0, 0, -1};
                if (n > 0) {
                    k_find_gpos<<<1, 1, 0, st>>>(d_gpos, n, 0, dll.p);
                    long long i = -1;
                    dll.download(&i, 1);
                    JB_CUDA(cudaStreamSynchronize(st));
                    if (i >= 0) {
                        uint32_t pr, lab;
                        JB_CUDA(cudaMemcpyAsync(&pr, pos.p + i, 4, cudaMemcpyDeviceToHost, st));
                        JB_CUDA(cudaStreamSynchronize(st));
                        JB_CUDA(cudaMemcpyAsync(&lab, L.labs.p + pr, 4, cudaMemcpyDeviceToHost, st));
                        JB_CUDA(cudaStreamSynchronize(st));
                        l0 = L0{1, lab, (long long)pr};
                    }
                }
                std::vector<L0> a0(cm.world);
                cm.allgather(&l0, sizeof l0, a0.data());
                for (int r = 0; r < cm.world; ++r)
                    if (a0[r].has) {
                        best = FarRec{0.0, 0, a0[r].r, xy.first, xy.second, a0[r].lab};
                        owner = r;
                    }
            }
            k_repair_dist<<<1, 1, 0, st>>>(L.acc.p, L.centers.p, L.labs.p, L.tlab.p, (int)k, L.Ex,
                                           L.Ey, c, (int)best.donor, best.x, best.y,
                                           owner == cm.rank ? best.r : -1, L.ntiles);
            JB_LAUNCH_CHECK();
        }
        const int zero = 0;
        JB_CUDA(cudaMemcpyAsync(L.empties.p + L.k, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    };

    // host-driven seeding: every decision on the host from allgathered
    // partials (kept as the fallback of the device path's roundoff spill)
    auto seed_host = [&]() {
            std::vector<uint64_t> chosen;
            std::vector<double> ch_xy;
            uint64_t cur_draw = *cursor, r0;
            while (!lemire_host(draw(cur_draw), S, r0)) ++cur_draw;
            cur_draw += 1;
            chosen.push_back(r0);
            auto xy = center_of(r0);
            ch_xy.push_back(xy.first);
            ch_xy.push_back(xy.second);
            double2 hc = make_double2(xy.first, xy.second);
            cur.upload(&hc, 1);
            part.zero();
            if (n > 0) {
                JB_PROF("d2_update", st);
                k_d2_tiles<<<tile_grid, 256, 0, st>>>(spts.p, orig.p, pos.p, n, nullptr, nullptr,
                                                      tmax.p, d2s.p, ss.p, 1, Ed2, part.p, cur.p,
                                                      gkey.p, nullptr);
            }
            JB_LAUNCH_CHECK();
            for (uint64_t c = 1; c < k; ++c) {
                std::vector<unsigned long long> hp = part.to_host(2 * nblocks);
                hp = cm.sum_i128(hp);
                i128 total = 0;
                for (uint64_t b = 0; b < nblocks; ++b) total += fx_load(&hp[2 * b]);
                const double total_d = fx_to_double(total, Ed2);
                uint64_t next;
                if (!(total_d > 0.0)) {  // every remaining point duplicates a center (:120-124)
                    next = 0;
                    while (std::find(chosen.begin(), chosen.end(), next) != chosen.end()) ++next;
                } else {
                    const uint64_t x = draw(cur_draw);
                    double canon = (double)x * 0x1p-64;  // generate_canonical<double,53>
                    if (canon >= 1.0) canon = 0x1.fffffffffffffp-1;
                    const double u = canon * total_d + 0.0;
                    const i128 U = fx_from_double(u, Ed2);
                    i128 run = 0;
                    uint64_t fb = nblocks;
                    for (uint64_t b = 0; b < nblocks; ++b) {
                        const i128 v = fx_load(&hp[2 * b]);
                        if (U < run + v) {
                            fb = b;
                            break;
                        }
                        run += v;
                    }
                    if (fb == nblocks) {  // roundoff spill: last positive-weight index (:67-70)
                        long long lp = -1;
                        if (n > 0) {
                            dll.upload(&lp, 1);
                            k_last_positive<<<1, 256, 0, st>>>(d_gpos, pos.p, n, d2s.p, dll.p);
                            dll.download(&lp, 1);
                            JB_CUDA(cudaStreamSynchronize(st));
                        }
                        std::vector<long long> all(cm.world);
                        cm.allgather(&lp, sizeof lp, all.data());
                        long long m = (long long)S - 1, best = -1;
                        for (auto v : all) best = std::max(best, v);
                        next = best >= 0 ? (uint64_t)best : (uint64_t)m;
                    } else {
                        wblk.zero();
                        if (n > 0) k_block_weights<<<1, 256, 0, st>>>(d_gpos, pos.p, n, d2s.p, fb, wblk.p);
                        JB_LAUNCH_CHECK();
                        std::vector<double> w = wblk.to_host(D2_R);
                        const auto all = cm.gather(w);  // every position owned by exactly one rank
                        next = UINT64_MAX;
                        i128 before = run;
                        for (uint64_t e = 0; e < D2_R && fb * D2_R + e < S; ++e) {
                            double we = 0.0;
                            for (int r = 0; r < cm.world; ++r) we += all[(size_t)r * D2_R + e];
                            const i128 a = fx_from_double(we, Ed2);
                            if (U < before + a) {
                                next = fb * D2_R + e;
                                break;
                            }
                            before += a;
                        }
                        if (next == UINT64_MAX) throw Error(INTERNAL, "distributed D2 pick failed");
                    }
                    cur_draw += 1;
                }
                chosen.push_back(next);
                xy = center_of(next);
                ch_xy.push_back(xy.first);
                ch_xy.push_back(xy.second);
                if (c + 1 < k && n > 0) {
                    hc = make_double2(xy.first, xy.second);
                    cur.upload(&hc, 1);
                    JB_PROF("d2_update", st);
                    JB_CUDA(cudaMemsetAsync(d2_nwork.p, 0, 8, st));
                    k_d2_cull<<<cull_grid, 256, 0, st>>>(cbox.p, tmax.p, ntiles, spts.p, pos.p, ss.p,
                                                         d2_work.p, d2_nwork.p, cur.p);
                    k_d2_tiles<<<tile_grid, 256, 0, st>>>(spts.p, orig.p, pos.p, n, d2_work.p,
                                                          d2_nwork.p, tmax.p, d2s.p, ss.p, 0, Ed2,
                                                          part.p, cur.p, gkey.p, nullptr);
                    JB_LAUNCH_CHECK();
                }
            }
            *cursor = cur_draw;
            L.centers.upload(ch_xy.data(), 2 * k);
            if (dbg_on())
                fprintf(stderr, "[jb r%d] dist seeds: S=%llu n=%lld Ed2=%d Ex=%d Ey=%d chosen[0..3]=%llu %llu %llu %llu hash=%016llx cursor=%llu\n",
                        cm.rank, (unsigned long long)S, (long long)n, Ed2, L.Ex, L.Ey,
                        (unsigned long long)chosen[0], (unsigned long long)chosen[std::min<uint64_t>(1, k - 1)],
                        (unsigned long long)chosen[std::min<uint64_t>(2, k - 1)], (unsigned long long)chosen[k - 1],
                        (unsigned long long)dbg_hash(ch_xy.data(), 16 * k), (unsigned long long)cur_draw);
    };

    // device-driven seeding: partials all-reduced on the stream (DevComm),
    // every rank picks the same point on device; false on a roundoff spill
    DevComm dc;
    dc.init(cm, st);
    if (dbg_on())
        fprintf(stderr, "[jb r%d] dist exchanges: %s\n", cm.rank,
                dc.nccl() ? "NCCL on the stream" : "staged through the host allgather");
    auto seed_device = [&]() -> bool {
        DArr<SeedState> dss(1, st);
        const SeedState h0{*cursor, 0, 0, 0};
        dss.upload(&h0, 1);
        DArr<int64_t> dch(k, st);
        DArr<DPick> dp(1, st);
        dp.zero();
        DArr<unsigned long long> p3(3 * nblocks, st), gpart(2 * nblocks, st), w(D2_R, st), cb(2, st);
        const double2* curp = reinterpret_cast<const double2*>(cb.p);
        const int pg = (int)std::max<uint64_t>(1, std::min<uint64_t>((nblocks + 255) / 256, num_sms() * 4));
        part.zero();
        k_pick_first<<<1, 1, 0, st>>>(d_raw, S, dss.p, dch.p);
        k_dcenter_bits<<<1, 1, 0, st>>>(d_gpos, pos.p, spts.p, n, dch.p, 0, cb.p);
        JB_LAUNCH_CHECK();
        dc.allreduce_u64(cb.p, 2, st);
        k_dstore_center<<<1, 1, 0, st>>>(cb.p, L.centers.p, 0);
        if (n > 0) {
            JB_PROF("d2_update", st);
            k_d2_tiles<<<tile_grid, 256, 0, st>>>(spts.p, orig.p, pos.p, n, nullptr, nullptr,
                                                  tmax.p, d2s.p, ss.p, 1, Ed2, part.p, curp,
                                                  gkey.p, nullptr);
        }
        JB_LAUNCH_CHECK();
        for (uint64_t c = 1; c < k; ++c) {
            {
                JB_PROF("d2_pick", st);
                k_part_split<<<pg, 256, 0, st>>>(part.p, (int)nblocks, p3.p);
                dc.allreduce_u64(p3.p, 3 * nblocks, st);
                k_part_join<<<pg, 256, 0, st>>>(p3.p, (int)nblocks, gpart.p);
                k_dpick_block<<<1, PICK_TB, 0, st>>>(d_raw, gpart.p, (int)nblocks, Ed2, dss.p,
                                                     dch.p, (int)c, dp.p);
                w.zero();
                if (n > 0) k_dblock_weights<<<1, 256, 0, st>>>(d_gpos, pos.p, n, d2s.p, dp.p, w.p);
                JB_LAUNCH_CHECK();
                dc.allreduce_u64(w.p, D2_R, st);
                k_dpick_elem<<<1, PICK_TB, 0, st>>>(w.p, dp.p, Ed2, dss.p, dch.p, (int)c, S);
                k_dcenter_bits<<<1, 1, 0, st>>>(d_gpos, pos.p, spts.p, n, dch.p, (int)c, cb.p);
                JB_LAUNCH_CHECK();
                dc.allreduce_u64(cb.p, 2, st);
                k_dstore_center<<<1, 1, 0, st>>>(cb.p, L.centers.p, (int)c);
            }
            if (c + 1 < k && n > 0) {
                JB_PROF("d2_update", st);
                JB_CUDA(cudaMemsetAsync(d2_nwork.p, 0, 8, st));
                k_d2_cull<<<cull_grid, 256, 0, st>>>(cbox.p, tmax.p, ntiles, spts.p, pos.p, ss.p,
                                                     d2_work.p, d2_nwork.p, curp);
                k_d2_tiles<<<tile_grid, 256, 0, st>>>(spts.p, orig.p, pos.p, n, d2_work.p,
                                                      d2_nwork.p, tmax.p, d2s.p, ss.p, 0, Ed2,
                                                      part.p, curp, gkey.p, nullptr);
            }
            JB_LAUNCH_CHECK();
        }
        SeedState hs;
        DPick hp;
        dss.download(&hs, 1);
        dp.download(&hp, 1);
        JB_CUDA(cudaStreamSynchronize(st));
        if (hp.spill) return false;
        if (hs.cursor > raw_count) throw Error(INTERNAL, "rng stream exhausted");
        *cursor = hs.cursor;
        return true;
    };

    double best_sse = 0.0;
    for (uint64_t restart = 0; restart < n_init; ++restart) {
        // ---- d2_seed (clustering.hpp:92-131) ----
        {
            const uint64_t cursor0 = *cursor;
            if (getenv("JB_DIST_HOST_SEED") || !seed_device()) {
                *cursor = cursor0;
                seed_host();
            }
        }


        // ---- Lloyd (lloyd_once :200-220): device loop, one all-reduce of the
        // exact cluster-sum deltas + change count per iteration, host sync
        // once per batch (empty clusters: re-seeded on the host path) ----
        auto exchange_dev = [&](bool count_iter) {
            dc.allreduce_u64(L.dacc.p, 7 * k + 1, st);
            k_dist_accum<<<1, 256, 0, st>>>(L.acc.p, L.dacc.p, (int)k, L.empties.p + L.k,
                                             L.changed_ptr(),
                                             L.nwork.p, L.nswork.p, L.diag.p, count_iter ? 1 : 0);
            JB_LAUNCH_CHECK();
        };
        L.acc.zero();
        L.dacc.zero();
        L.diag.zero();
        JB_CUDA(cudaMemsetAsync(L.tlab.p, 0xFF, sizeof(uint32_t) * L.nstate(), st));
        JB_CUDA(cudaMemsetAsync(L.empties.p + L.k, 0, 3 * sizeof(int), st));
        JB_CUDA(cudaMemsetAsync(L.flags.p, 0, 8, st));
        JB_CUDA(cudaMemsetAsync(L.nwork.p, 0, 8, st));
        JB_CUDA(cudaMemsetAsync(L.nswork.p, 0, 8, st));
        lloyd_assign(L, true, false);  // assign_all(points, seeds) (:204)
        exchange_dev(false);
        uint64_t it = 0;
        const uint64_t kBatch = dbg_on() ? 1 : 16;
        while (it < max_iters) {
            const uint64_t B = std::min<uint64_t>(kBatch, max_iters - it);
            for (uint64_t b = 0; b < B; ++b) {
                lloyd_means(L, true);          // update_means ...
                lloyd_assign(L, false, true);  // ... assign_all, label comparison
                exchange_dev(true);
            }
            LoopState h = lloyd_state(L);
            it = (uint64_t)h.iters;
            if (dbg_on()) {
                auto cc = L.centers.to_host(2 * k);
                fprintf(stderr, "[jb r%d] dist iter %d: empty=%d conv=%d centers=%016llx\n", cm.rank,
                        h.iters, h.n_empty, h.converged,
                        (unsigned long long)dbg_hash(cc.data(), 16 * k));
            }
            if (h.converged) break;
            if (h.n_empty) {  // re-seed the empty clusters, finish the iteration
                repair_dist();
                lloyd_assign(L, false, true);
                exchange_dev(true);
                h = lloyd_state(L);
                it = (uint64_t)h.iters;
                if (h.converged) break;
            }
        }
        repair_dist();  // final update_means
        double sse = 0.0;
        if (n_init > 1) {
            DArr<unsigned long long> sacc(2, st);
            sacc.zero();
            if (n > 0)
                k_sse<<<grid_cap(n), 256, 0, st>>>(spts.p, n, L.labs.p, L.centers.p, Ed2, sacc.p);
            JB_LAUNCH_CHECK();
            auto hs = cm.sum_i128(sacc.to_host(2));
            sse = fx_to_double(fx_load(hs.data()), Ed2);
        }
        if (restart == 0 || sse < best_sse) {
            best_sse = sse;
            out.k = k;
            out.centers = L.centers.to_host(2 * k);
            out.slabs.alloc(nn, st);
            if (n > 0) {
                JB_CUDA(cudaMemcpyAsync(out.slabs.p, L.labs.p, sizeof(uint32_t) * n,
                                        cudaMemcpyDeviceToDevice, st));
                JB_LAUNCH_CHECK();
            }
            out.iterations = it;
            out.sse = sse;
        }
    }
    out.sorig = std::move(orig);
    JB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace jb
