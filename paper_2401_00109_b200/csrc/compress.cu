// compress.cu — tol-bounded greedy piecewise-linear compression on sm_100a.
//
// Reference: detail::compress_range (compression.hpp:31-66), compress
// (:70-83), partitional_compress (:167-193). The greedy parse is a
// deterministic orbit p -> f(p) (f = piece end from start p), so the work is
// split into fixed-size chunks of start positions and every chunk is parsed
// SPECULATIVELY from its own first position by one thread. Orbits merge once
// they share a point, so the true parse is recovered by (1) propagating true
// chunk exits left to right with a parallel fixed-point iteration that
// re-parses only the prefix of a chunk before the true orbit meets the
// speculative one (usually zero pieces), then (2) rewriting only those
// prefixes. All arithmetic in f is the reference's, in the reference's order,
// compiled with -fmad=false, so boundaries and increments are bit-exact.
#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <vector>

#include "jb_device.hpp"

namespace jb {

// RN(1/d) and RN(1/d^2) for d <= kRcpG (L1-resident through __ldg): the
// FMA-corrected quotients (div_cr) of the deviation test for long pieces
// (config 5: pieces up to ~3000 samples), instead of the division sequence.
constexpr int kRcpG = 4096;
__device__ double g_rcp1[kRcpG + 1], g_rcp2[kRcpG + 1];

void upload_recips(cudaStream_t st) {  // once per device
    static std::mutex mu;
    static std::vector<int> done;
    static std::vector<double> r1(kRcpG + 1), r2(kRcpG + 1);
    int dev = 0;
    JB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(done.begin(), done.end(), dev) != done.end()) return;
    for (int t = 0; t <= kRcpG; ++t) {
        const double dd = (double)(t > 0 ? t : 1);
        r1[t] = 1.0 / dd;  // IEEE, as the device's 1.0 / dd
        r2[t] = 1.0 / (dd * dd);
    }
    JB_CUDA(cudaMemcpyToSymbolAsync(g_rcp1, r1.data(), sizeof(double) * (kRcpG + 1), 0,
                                    cudaMemcpyHostToDevice, st));
    JB_CUDA(cudaMemcpyToSymbolAsync(g_rcp2, r2.data(), sizeof(double) * (kRcpG + 1), 0,
                                    cudaMemcpyHostToDevice, st));
    JB_CUDA(cudaStreamSynchronize(st));
    done.push_back(dev);
}

// a = yy / (d d), b = 2 y / d as the reference rounds them (compression.hpp:52)
__device__ __forceinline__ void dev_quotients(double y, double yy, double d, int64_t L,
                                              const double* r1s, const double* r2s, int rs,
                                              double& a, double& b) {
    const double y2 = 2.0 * y, ay = fabs(y);
    if (L <= kRcpG && ((ay >= 0x1p-450 && ay <= 0x1p500) || y == 0.0)) {
        const double q1 = L <= rs ? r1s[L] : __ldg(g_rcp1 + L);
        const double q2 = L <= rs ? r2s[L] : __ldg(g_rcp2 + L);
        a = yy == 0.0 ? yy : div_cr(yy, d * d, q2);
        b = y2 == 0.0 ? y2 : div_cr(y2, d, q1);  // 0 / d keeps the zero's sign
    } else {
        a = yy / (d * d);
        b = y2 / d;
    }
}

// Greedy piece end from `start` (compression.hpp:38-61), bit-exact. The
// test at d = 1 cannot break (cand > start + 1 fails), so its deviation is not
// evaluated; for d = 2^m the two divisions are multiplications by the exact
// power of two 2^-m (a product and a quotient of the same real value round
// identically). `bad` collects non-finite candidates (compression.hpp:73-74).
__device__ __forceinline__ int64_t piece_end(const double* __restrict__ v, int64_t start,
                                             int64_t last, double tol2, int64_t max_len,
                                             bool* bad = nullptr) {
    const double base = v[start];
    double s2 = 0.0, s3 = 0.0;
    // sum_{i<=d} i^2 kept as a running integer-valued double: identical to the
    // reference's d*(d+1)*(2d+1)/6 while d*(d+1)*(2d+1) < 2^53 (every value
    // involved is an exactly representable integer), the formula beyond that
    double sq = 0.0;
    int64_t end = start;
    for (;;) {
        const int64_t cand = end + 1;
        if (cand > last) break;
        const double vc = v[cand];
        if (bad && !isfinite(vc)) *bad = true;
        const double y = vc - base;
        const int64_t L = cand - start;
        const double d = (double)L;
        const double yy = y * y;
        const double ns2 = s2 + yy;
        const double ns3 = s3 + d * y;
        sq += d * d;
        if (L > 1) {
            double sum_d2 = sq;
            if (L > 165000) sum_d2 = d * (d + 1.0) * (2.0 * d + 1.0) / 6.0;
            double a, b;  // inc * inc / (len * len), 2.0 * inc / len
            if ((L & (L - 1)) == 0) {
                const int m = __ffsll(L) - 1;
                const double inv = __longlong_as_double((long long)(1023 - m) << 52);
                a = yy * (inv * inv);
                b = (2.0 * y) * inv;
            } else {
                dev_quotients(y, yy, d, L, nullptr, nullptr, 0, a, b);
            }
            const double sq_dev = a * sum_d2 - b * ns3 + ns2;
            if (sq_dev > (d - 1.0) * tol2) break;
        }
        end = cand;
        s2 = ns2;
        s3 = ns3;
        if (max_len > 0 && end - start >= max_len) break;
    }
    return end;
}

struct ChunkGeom {
    const int64_t* seg_first;
    const int64_t* seg_steps;
    const int64_t* chunk_off;  // n_seg + 1
    int64_t n_seg;
    int64_t C;
    const int32_t* chunk_seg;  // segment of every chunk (no binary search per chunk)
};

__device__ __forceinline__ void chunk_bounds(const ChunkGeom& g, int64_t ch, int64_t& s,
                                             int64_t& c, int64_t& lo, int64_t& hi,
                                             int64_t& last) {
    s = g.chunk_seg[ch];  // chunk_off[s] <= ch < chunk_off[s+1]
    c = ch - g.chunk_off[s];
    const int64_t first = g.seg_first[s];
    last = first + g.seg_steps[s];
    lo = first + c * g.C;
    hi = lo + g.C < last ? lo + g.C : last;
}

// Piece starts are kept as one bit per sample position, chunk-relative:
// chunk ch owns words fb[ch * W .. ch * W + W), W = C / 32, bit (p - lo).
__device__ __forceinline__ bool fbit(const uint32_t* __restrict__ fb, int64_t ch, int W,
                                     int64_t rel) {
    return (fb[ch * W + (rel >> 5)] >> (rel & 31)) & 1u;
}

constexpr int kRcp = 256;  // k_spec reciprocal tables cover d <= kRcp

// Phase 1: speculative parse of every chunk from its first start position,
// streamed: each sample is loaded once (one register ahead) and tested once
// against the open piece. When the test fails, the piece closes at the
// previous sample, which opens the next piece, and the failing sample
// becomes that piece's d = 1 candidate (always accepted, compression.hpp:54).
// Identical decisions to piece_end, with no re-loads and a uniform
// per-sample loop across the warp.
#ifndef JB_SPEC_MINB
#define JB_SPEC_MINB 8  // 64 registers (8 bytes spilled): 8 CTAs per SM, 6.01 -> 5.67 ms (9: 56 registers, 7.98 ms)
#endif
__global__ void __launch_bounds__(128, JB_SPEC_MINB) k_spec(const double* __restrict__ v, ChunkGeom g,
                                              int64_t n_chunks, double tol2, int64_t max_len,
                                              uint32_t* __restrict__ fb,
                                              int64_t* __restrict__ exit_spec,
                                              int* __restrict__ bad) {
    // RN(1/d) and RN(1/d^2) for the FMA quotients (div_cr)
    __shared__ double s_r1[kRcp + 1], s_r2[kRcp + 1];
    for (int t = threadIdx.x; t <= kRcp; t += blockDim.x) {
        const double dd = (double)(t > 0 ? t : 1);
        s_r1[t] = 1.0 / dd;
        s_r2[t] = 1.0 / (dd * dd);
    }
    __syncthreads();
    const int64_t ch = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (ch >= n_chunks) return;
    int64_t s, c, lo, hi, last;
    chunk_bounds(g, ch, s, c, lo, hi, last);
    const int W = (int)(g.C >> 5);
    uint32_t* my = fb + ch * W;
    uint32_t word = 1u;  // bit of lo: the chunk's first start
    int wi = 0;
    auto flag = [&](int64_t p) {
        const int rel = (int)(p - lo);
        while (wi < (rel >> 5)) {
            my[wi++] = word;
            word = 0;
        }
        word |= 1u << (rel & 31);
    };
    double prev = v[lo];            // v[i - 1]
    bool nonfinite = !isfinite(prev);
    double base = prev;             // v[start]
    int64_t start = lo, L = 0;      // open piece: start, current length
    double s2 = 0.0, s3 = 0.0, sq = 0.0;
    int64_t i = lo + 1;
    double vc = i <= last ? __ldg(v + i) : 0.0;
    int64_t exit_p = -1;
    for (;;) {
        if (i > last) {  // every candidate accepted: the piece ends at last
            exit_p = last;
            break;
        }
        const double vn = i + 1 <= last ? __ldg(v + i + 1) : 0.0;  // next sample in flight
        nonfinite |= !isfinite(vc);
        const int64_t Ln = L + 1;
        const double y = vc - base;
        const double d = (double)Ln;
        const double yy = y * y;
        const double ns2 = s2 + yy;
        const double ns3 = s3 + d * y;
        const double nsq = sq + d * d;
        bool brk = false;
        if (Ln > 1) {
            double sum_d2 = nsq;
            if (Ln > 165000) sum_d2 = d * (d + 1.0) * (2.0 * d + 1.0) / 6.0;
            double a, b;  // inc * inc / (len * len), 2.0 * inc / len
            dev_quotients(y, yy, d, Ln, s_r1, s_r2, kRcp, a, b);
            const double sq_dev = a * sum_d2 - b * ns3 + ns2;
            brk = sq_dev > (d - 1.0) * tol2;
        }
        if (brk) {
            // the piece ends at i - 1, which starts the next one
            start = i - 1;
            if (start >= hi) {
                exit_p = start;
                break;
            }
            flag(start);
            base = prev;
            const double y1 = vc - base;  // candidate i at d = 1 (same operations)
            s2 = 0.0 + y1 * y1;
            s3 = 0.0 + 1.0 * y1;
            sq = 0.0 + 1.0;
            L = 1;
        } else {
            s2 = ns2;
            s3 = ns3;
            sq = nsq;
            L = Ln;
        }
        if (max_len > 0 && L >= max_len) {  // closes at i (compression.hpp:61-63)
            start = i;
            if (start >= hi) {
                exit_p = start;
                break;
            }
            flag(start);
            base = vc;
            s2 = s3 = sq = 0.0;
            L = 0;
        }
        prev = vc;
        vc = vn;
        ++i;
    }
    for (; wi < W; ++wi) {
        my[wi] = word;
        word = 0;
    }
    exit_spec[ch] = exit_p;
    if (nonfinite) atomicExch(bad, 1);
}

// Phase 2: E_out[c] = F_c(E_in[c-1]), F_c = exit of chunk c when the true
// orbit enters it at t. Only chunks whose entry changed in the previous round
// (dirty_in[c-1]) are re-evaluated: long pieces make chains of chunks whose
// orbits merge late (config 5: ~50 rounds), and a full re-parse of every
// chunk per round would cost a whole compression pass each time.
__global__ void k_fix(const double* __restrict__ v, ChunkGeom g, int64_t n_chunks, double tol2,
                      int64_t max_len, const uint32_t* __restrict__ fb,
                      const int64_t* __restrict__ exit_spec, const int64_t* __restrict__ E_in,
                      int64_t* __restrict__ E_out, int* __restrict__ changed,
                      const uint8_t* __restrict__ dirty_in, uint8_t* __restrict__ dirty_out) {
    const int64_t ch = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (ch >= n_chunks) return;
    if (dirty_in && !(ch > 0 && dirty_in[ch - 1])) {  // entry unchanged: so is the exit
        E_out[ch] = E_in[ch];
        dirty_out[ch] = 0;
        return;
    }
    int64_t s, c, lo, hi, last;
    chunk_bounds(g, ch, s, c, lo, hi, last);
    const int W = (int)(g.C >> 5);
    int64_t r;
    if (c == 0) {
        r = exit_spec[ch];
    } else {
        const int64_t t = E_in[ch - 1];
        if (t >= hi) {
            r = t;
        } else if (fbit(fb, ch, W, t - lo)) {
            r = exit_spec[ch];
        } else {
            int64_t q = t;
            do {
                q = piece_end(v, q, last, tol2, max_len);
            } while (q < hi && !fbit(fb, ch, W, q - lo));
            r = q < hi ? exit_spec[ch] : q;
        }
    }
    E_out[ch] = r;
    const bool ch_ = r != E_in[ch];
    if (dirty_out) dirty_out[ch] = ch_ ? 1 : 0;
    if (ch_) atomicExch(changed, 1);
}

// Greedy piece end from `start` (compression.hpp:38-61) evaluated by a whole
// warp, 32 candidates per step: lane j tests d = c0 + j - start. The running
// sums s2 = sum y^2 and s3 = sum d*y stay the reference's sequential fp64
// sums: each lane adds the step's terms of lanes 0..j to the carried sum in
// order (predicated adds over a shared-memory broadcast of the terms), which
// is the same chain of roundings. The piece ends before the first lane that
// fails the test, passes `last` or exceeds max_len (all three give
// end = cand - 1). Uniform result.
__device__ __forceinline__ int64_t piece_end_warp(const double* __restrict__ v, int64_t start,
                                                  int64_t last, double tol2, int64_t max_len,
                                                  double* sh /* 64 doubles per warp */) {
    const int lane = threadIdx.x & 31;
    const double base = __ldg(v + start);
    double s2 = 0.0, s3 = 0.0;  // carried sums through the previous step
    for (int64_t c0 = start + 1;; c0 += 32) {
        const int64_t cand = c0 + lane;
        const int64_t L = cand - start;
        const bool in = cand <= last && (max_len <= 0 || L <= max_len);
        const double vc = in ? __ldg(v + cand) : base;
        const double y = vc - base;
        const double d = (double)L;
        const double yy = y * y, dy = d * y;
        sh[lane] = yy;
        sh[32 + lane] = dy;
        __syncwarp();
        double n2 = s2, n3 = s3;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const double a2 = sh[i], a3 = sh[32 + i];
            if (i <= lane) {
                n2 += a2;
                n3 += a3;
            }
        }
        __syncwarp();
        bool stop = !in;
        if (in && L > 1) {
            // sum_{i<=d} i^2: the exact integer while d(d+1)(2d+1) < 2^53,
            // where the reference's formula is exact too; the formula beyond
            const double sum_d2 = L <= 165000 ? (double)(L * (L + 1) * (2 * L + 1) / 6)
                                              : d * (d + 1.0) * (2.0 * d + 1.0) / 6.0;
            double a, b;  // inc * inc / (len * len), 2.0 * inc / len
            dev_quotients(y, yy, d, L, nullptr, nullptr, 0, a, b);
            const double sq_dev = a * sum_d2 - b * n3 + n2;
            stop = sq_dev > (d - 1.0) * tol2;
        }
        const unsigned m = __ballot_sync(0xffffffffu, stop);
        if (m) return c0 + (__ffs(m) - 1) - 1;
        s2 = __shfl_sync(0xffffffffu, n2, 31);
        s3 = __shfl_sync(0xffffffffu, n3, 31);
    }
}

// Phase 2b (chains that merge late, config 5's long pieces): one WARP per
// segment walks its chunks in order from the true entry -- the exact
// sequential fixed point -- and rewrites each chunk's flags to the true orbit
// on the way (so Phase 3 is skipped). A chunk whose entry is a speculative
// start costs O(1); otherwise the warp parses from the entry until the true
// orbit meets a speculative start or leaves the chunk. The chunk's W flag
// words live in lanes 0..W-1.
constexpr int kWalkTB = 128;
__global__ void __launch_bounds__(kWalkTB) k_walk(const double* __restrict__ v, ChunkGeom g,
                                                  double tol2, int64_t max_len,
                                                  uint32_t* __restrict__ fb,
                                                  const int64_t* __restrict__ exit_spec,
                                                  int64_t* __restrict__ E) {
    __shared__ double s_terms[kWalkTB / 32][64];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (s >= g.n_seg) return;
    const int64_t c0 = g.chunk_off[s], c1 = g.chunk_off[s + 1];
    const int W = (int)(g.C >> 5);
    int64_t t = g.seg_first[s];  // true entry of the current chunk
    for (int64_t ch = c0; ch < c1; ++ch) {
        int64_t ss, c, lo, hi, last;
        chunk_bounds(g, ch, ss, c, lo, hi, last);
        uint32_t word = lane < W ? fb[ch * W + lane] : 0u;
        // clear bits of positions [p0, p1) (chunk-relative)
        auto clear = [&](int64_t p0, int64_t p1) {
            const int64_t w0 = 32 * (int64_t)lane;
            const int64_t a = p0 - lo > w0 ? p0 - lo - w0 : 0;
            const int64_t b = p1 - lo - w0 < 32 ? p1 - lo - w0 : 32;
            if (a < b) {
                const uint32_t hm = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
                word &= ~(hm & ~((1u << a) - 1u));
            }
        };
        auto test = [&](int64_t p) {
            const int rel = (int)(p - lo);
            return (__shfl_sync(0xffffffffu, word, rel >> 5) >> (rel & 31)) & 1u;
        };
        auto set = [&](int64_t p) {
            const int rel = (int)(p - lo);
            if (lane == (rel >> 5)) word |= 1u << (rel & 31);
        };
        int64_t r;
        if (t >= hi) {
            word = 0;
            r = t;
        } else {
            clear(lo, t);
            if (test(t)) {
                r = exit_spec[ch];
            } else {
                set(t);
                int64_t p = t;
                for (;;) {
                    const int64_t q = piece_end_warp(v, p, last, tol2, max_len, s_terms[wib]);
                    clear(p + 1, q < hi ? q : hi);
                    if (q >= hi) {
                        r = q;
                        break;
                    }
                    if (test(q)) {
                        r = exit_spec[ch];
                        break;
                    }
                    set(q);
                    p = q;
                }
            }
        }
        if (lane < W) fb[ch * W + lane] = word;
        if (lane == 0) E[ch] = r;
        t = r;
    }
}

// Phase 3: rewrite each chunk's flags to the true orbit.
__global__ void k_apply(const double* __restrict__ v, ChunkGeom g, int64_t n_chunks, double tol2,
                        int64_t max_len, uint32_t* __restrict__ fb,
                        const int64_t* __restrict__ E) {
    const int64_t ch = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (ch >= n_chunks) return;
    int64_t s, c, lo, hi, last;
    chunk_bounds(g, ch, s, c, lo, hi, last);
    const int W = (int)(g.C >> 5);
    uint32_t* my = fb + ch * W;
    auto clear_range = [&](int64_t p0, int64_t p1) {  // bits of [p0, p1)
        for (int64_t p = p0; p < p1; ++p) my[(p - lo) >> 5] &= ~(1u << ((p - lo) & 31));
    };
    const int64_t T = c == 0 ? lo : E[ch - 1];
    if (T >= hi) {
        for (int w = 0; w < W; ++w) my[w] = 0;
    } else {
        clear_range(lo, T);
        if (!fbit(fb, ch, W, T - lo)) {
            int64_t p = T;
            my[(p - lo) >> 5] |= 1u << ((p - lo) & 31);
            for (;;) {
                const int64_t q = piece_end(v, p, last, tol2, max_len);
                const int64_t z = q < hi ? q : hi;
                clear_range(p + 1, z);
                if (q >= hi || fbit(fb, ch, W, q - lo)) break;
                my[(q - lo) >> 5] |= 1u << ((q - lo) & 31);
                p = q;
            }
        }
    }
}

// Phase 4a: pieces per chunk.
__global__ void k_count(ChunkGeom g, int64_t n_chunks, const uint32_t* __restrict__ fb,
                        int64_t* __restrict__ count) {
    const int W = (int)(g.C >> 5);
    for (int64_t ch = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ch < n_chunks;
         ch += (int64_t)gridDim.x * blockDim.x) {
        int n = 0;
        for (int w = 0; w < W; ++w) n += __popc(fb[ch * W + w]);
        count[ch] = n;
    }
}

constexpr int kEmitW = 8;  // flag words per chunk at most (C <= 256)

// Phase 4b: emit (len, inc) pieces in input order, one warp per chunk, a
// lane per sample position of each 32-bit flag word: a flagged lane's piece
// ends at the next set bit (this word, a later word, or the chunk's true exit
// E); its output slot is the chunk base plus the set bits before it, so the
// loads of v and the stores of len/inc are coalesced. Also max|inc| and max
// len for the fixed-point exponents downstream.
__global__ void k_emit(const double* __restrict__ v, ChunkGeom g, int64_t n_chunks,
                       const uint32_t* __restrict__ fb, const int64_t* __restrict__ E,
                       const int64_t* __restrict__ base, int32_t* __restrict__ out_len,
                       double* __restrict__ out_inc, unsigned long long* __restrict__ max_inc_bits,
                       int* __restrict__ max_len) {  // [0] max, [1] min
    const int lane = threadIdx.x & 31;
    const int W = (int)(g.C >> 5);
    double mi = 0.0;
    int ml = 0, mn = 0x7FFFFFFF;
    for (int64_t ch = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; ch < n_chunks;
         ch += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int64_t s, c, lo, hi, last;
        chunk_bounds(g, ch, s, c, lo, hi, last);
        const uint32_t mine = lane < W ? fb[ch * W + lane] : 0u;  // all words of the chunk
        // the chunk's samples, one per (word, lane), all loads in flight at
        // once: v[p] is a register and v[e] a shuffle when e lies in the same
        // or the next word (a load otherwise: pieces longer than a word)
        double vr[kEmitW];
#pragma unroll
        for (int w = 0; w < kEmitW; ++w) {
            const int64_t q = lo + 32 * w + lane;
            vr[w] = (w < W && q <= last) ? __ldg(v + q) : 0.0;
        }
        const int64_t Ech = E[ch];
        int64_t j = base[ch];
#pragma unroll
        for (int w = 0; w < kEmitW; ++w) {
            if (w >= W) break;
            const uint32_t m = __shfl_sync(0xffffffffu, mine, w);
            if (!m) continue;
            // next start after this word: first set bit of a later word
            uint32_t later = lane > w ? mine : 0u;
            const unsigned nz = __ballot_sync(0xffffffffu, later != 0);
            int64_t nxt = Ech;
            if (nz) {
                const int wl = __ffs(nz) - 1;
                const uint32_t mw = __shfl_sync(0xffffffffu, mine, wl);
                nxt = lo + 32 * wl + (__ffs(mw) - 1);
            }
            const bool f = (m >> lane) & 1u;
            const int64_t p = lo + 32 * w + lane;
            const uint32_t above = lane < 31 ? (m >> (lane + 1)) : 0u;
            const int64_t e = above ? p + __ffs(above) : nxt;
            const int64_t re = e - lo - 32 * w;  // e relative to this word
            const double e0 = __shfl_sync(0xffffffffu, vr[w], (int)(re & 31));
            const double e1 = w + 1 < kEmitW ? __shfl_sync(0xffffffffu, vr[(w + 1) % kEmitW], (int)(re & 31))
                                             : 0.0;
            if (f) {
                const double ve = re < 32 ? e0 : (re < 64 && w + 1 < W ? e1 : __ldg(v + e));
                const double inc = ve - vr[w];
                const int64_t k = j + __popc(m & ((1u << lane) - 1u));
                out_len[k] = (int32_t)(e - p);
                out_inc[k] = inc;
                mi = fmax(mi, fabs(inc));
                ml = max(ml, (int)(e - p));
                mn = min(mn, (int)(e - p));
            }
            j += __popc(m);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mi = fmax(mi, __shfl_down_sync(0xffffffffu, mi, o));
        ml = max(ml, __shfl_down_sync(0xffffffffu, ml, o));
        mn = min(mn, __shfl_down_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
        atomicMax(max_inc_bits, dbits(mi));
        atomicMax(max_len, ml);
        atomicMin(max_len + 1, mn);
    }
}

__global__ void k_chunk_seg(const int64_t* __restrict__ chunk_off, int64_t n_seg,
                            int32_t* __restrict__ chunk_seg) {
    for (int64_t sidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sidx < n_seg;
         sidx += (int64_t)gridDim.x * blockDim.x)
        for (int64_t ch = chunk_off[sidx]; ch < chunk_off[sidx + 1]; ++ch)
            chunk_seg[ch] = (int32_t)sidx;
}

__global__ void k_seg_offsets(const int64_t* __restrict__ chunk_off,
                              const int64_t* __restrict__ base, int64_t n_seg, int64_t total,
                              int64_t* __restrict__ seg_off) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s < n_seg) seg_off[s] = base[chunk_off[s]];
    if (s == n_seg) seg_off[s] = total;
}

void compress_segments(const double* d_values, const SegTable& seg, double tol,
                       int64_t max_piece_len, Pieces& out, cudaStream_t st, int* n_fix_iters) {
    const int64_t n_seg = seg.n_seg;
    upload_recips(st);
    // chunk size: enough chunks to fill 148 SMs, clamped to [32, 256] steps
    int64_t C = 256;
    while (C > 32 && seg.total_steps / C < (int64_t)num_sms() * 1024) C >>= 1;
    std::vector<int64_t> h_chunk_off(n_seg + 1);
    int64_t max_last = 0;
    h_chunk_off[0] = 0;
    for (int64_t s = 0; s < n_seg; ++s) {
        h_chunk_off[s + 1] = h_chunk_off[s] + (seg.h_steps[s] + C - 1) / C;
        max_last = std::max(max_last, seg.h_first[s] + seg.h_steps[s]);
    }
    const int64_t n_chunks = h_chunk_off[n_seg];
    DArr<int64_t> chunk_off(n_seg + 1, st);
    chunk_off.upload(h_chunk_off.data(), n_seg + 1);
    DArr<int32_t> chunk_seg(std::max<int64_t>(n_chunks, 1), st);
    k_chunk_seg<<<ceil_div(n_seg, 256), 256, 0, st>>>(chunk_off.p, n_seg, chunk_seg.p);
    JB_LAUNCH_CHECK();
    ChunkGeom g{seg.first.p, seg.steps.p, chunk_off.p, n_seg, C, chunk_seg.p};

    const double tol2 = tol * tol;
    const int W = (int)(C / 32);
    DArr<uint32_t> flags(n_chunks * W, st);  // every word is written by k_spec
    DArr<int64_t> exit_spec(n_chunks, st), Ea(n_chunks, st), Eb(n_chunks, st), cnt(n_chunks, st);
    DArr<int> dflag(2, st);
    dflag.zero();
    const int TB = 128;
    const int nb = ceil_div(n_chunks, TB);
    {
        JB_PROF("compress_spec", st);
        k_spec<<<nb, TB, 0, st>>>(d_values, g, n_chunks, tol2, max_piece_len, flags.p, exit_spec.p,
                              dflag.p);
    }
    JB_LAUNCH_CHECK();
    int hflag[2];
    dflag.download(hflag, 1);
    JB_CUDA(cudaStreamSynchronize(st));
    if (hflag[0]) throw Error(INVALID_INPUT, "compression input has non-finite values");

    JB_CUDA(cudaMemcpyAsync(Ea.p, exit_spec.p, sizeof(int64_t) * n_chunks,
                            cudaMemcpyDeviceToDevice, st));
    int iters = 0;
    // the warp walk is sequential per segment: used unless one segment is so
    // long that its walk would outlast the parallel rounds
    int64_t max_steps = 0;
    for (int64_t s = 0; s < n_seg; ++s) max_steps = std::max(max_steps, seg.h_steps[s]);
    const bool walk_ok = max_steps <= (int64_t(1) << 22) && !getenv("JB_NO_WALK");
    bool walked = false;
    DArr<uint8_t> dirty_a(n_chunks, st), dirty_b(n_chunks, st);
    for (;;) {
        JB_CUDA(cudaMemsetAsync(dflag.p + 1, 0, sizeof(int), st));
        {
            JB_PROF("compress_fix", st);
            k_fix<<<nb, TB, 0, st>>>(d_values, g, n_chunks, tol2, max_piece_len, flags.p,
                                 exit_spec.p, Ea.p, Eb.p, dflag.p + 1,
                                 iters == 0 ? nullptr : dirty_a.p, dirty_b.p);
        }
        JB_LAUNCH_CHECK();
        std::swap(dirty_a, dirty_b);
        ++iters;
        int ch;
        JB_CUDA(cudaMemcpyAsync(&ch, dflag.p + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        std::swap(Ea, Eb);
        if (!ch) break;
        if (walk_ok) {  // still moving: walk the segments sequentially (exact)
            JB_PROF("compress_walk", st);
            k_walk<<<ceil_div(n_seg * 32, kWalkTB), kWalkTB, 0, st>>>(
                d_values, g, tol2, max_piece_len, flags.p, exit_spec.p, Ea.p);
            JB_LAUNCH_CHECK();
            ++iters;
            walked = true;
            break;
        }
    }
    if (n_fix_iters) *n_fix_iters = iters;
    if (!walked) {
        JB_PROF("compress_apply", st);
        k_apply<<<nb, TB, 0, st>>>(d_values, g, n_chunks, tol2, max_piece_len, flags.p, Ea.p);
        JB_LAUNCH_CHECK();
    }
    const int wgrid = (int)std::max<int64_t>(
        1, std::min<int64_t>((n_chunks * 32 + 255) / 256, (int64_t)num_sms() * 16));
    {
        JB_PROF("compress_count", st);
        k_count<<<nb, TB, 0, st>>>(g, n_chunks, flags.p, cnt.p);
    }
    JB_LAUNCH_CHECK();

    DArr<int64_t> base(n_chunks + 1, st);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, base.p, n_chunks + 1, st);
    // the scan input needs a trailing zero so base[n_chunks] is the total
    DArr<int64_t> cnt1(n_chunks + 1, st);
    JB_CUDA(cudaMemcpyAsync(cnt1.p, cnt.p, sizeof(int64_t) * n_chunks, cudaMemcpyDeviceToDevice,
                            st));
    JB_CUDA(cudaMemsetAsync(cnt1.p + n_chunks, 0, sizeof(int64_t), st));
    DArr<uint8_t> tmp(tmp_bytes, st);
    cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt1.p, base.p, n_chunks + 1, st);
    JB_LAUNCH_CHECK();
    int64_t N = 0;
    JB_CUDA(cudaMemcpyAsync(&N, base.p + n_chunks, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));

    out.N = N;
    out.len.alloc(N, st);
    out.inc.alloc(N, st);
    out.seg_offsets.alloc(n_seg + 1, st);
    DArr<unsigned long long> mx(1, st);
    mx.zero();
    DArr<int> ml(2, st);
    {
        const int init[2] = {0, 0x7FFFFFFF};
        ml.upload(init, 2);
    }
    {
        JB_PROF("compress_emit", st);
        k_emit<<<wgrid, 256, 0, st>>>(d_values, g, n_chunks, flags.p, Ea.p, base.p, out.len.p,
                                      out.inc.p, mx.p, ml.p);
    }
    JB_LAUNCH_CHECK();
    k_seg_offsets<<<ceil_div(n_seg + 1, 256), 256, 0, st>>>(chunk_off.p, base.p, n_seg, N,
                                                            out.seg_offsets.p);
    JB_LAUNCH_CHECK();
    unsigned long long hmx = 0;
    int hml[2] = {0, 0};
    mx.download(&hmx, 1);
    ml.download(hml, 2);
    JB_CUDA(cudaStreamSynchronize(st));
    memcpy(&out.max_abs_inc, &hmx, 8);
    out.max_len = hml[0];
    out.min_len = N > 0 ? hml[1] : 0;
}

}  // namespace jb
