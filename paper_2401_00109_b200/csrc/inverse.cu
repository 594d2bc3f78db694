// inverse.cu — inverse symbolization on sm_100a (inverse.hpp:32-132,
// compression.hpp:87-103, 198-213).
//
// The reference's recurrences are sequential and stay sequential, but they
// are split so that each runs with nothing else on its critical path: per
// segment, one thread runs the length-carry chain (quantize_lengths :63-74)
// and a thread of ANOTHER warp the start-value chain (inverse_compress
// :94-101), both in the reference's rounding. Group sums, the residual
// fix-up (match_total_length :81-93) and output positions are then exact
// integer work, and a piece-parallel fill writes the interpolated samples
// v + inc * (i / len) straight into the (optionally stitched, :198-213)
// output.
#include <algorithm>

#include <cub/device/device_scan.cuh>

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


constexpr int GROUP = 32;  // pieces per fill unit
// errors: lowest segment first, and within a segment the label check first
// (reconstruct processes series in order; inverse_digitize_series checks
// labels before quantize/match_total_length): code = segment * 4 + rank
constexpr int kErrLabel = 0, kErrPiece = 1;

// quantize_lengths' step (:68-70): r = max(1, llround(x)), x = l + carry,
// carry = x - r (exact). For x >= 0.5, llround(x) == floor(fl(x + 0.5)):
// the sum is exact except where the rounding cannot move the floor (it
// only rounds when x + 0.5 lies in a binade above x's, i.e. at or above the
// power of two that is the result); tests/test_round_identity.py checks the
// identity. x < 0.5 clamps to 1. Five dependent fp64 operations per step
// instead of eight.
__device__ __forceinline__ void chain_step(double l, double& carry, int32_t& q) {
    const double x = l + carry;
    double r = floor(x + 0.5);
    if (x >= 0x1p52) r = x;  // already an integer
    if (x < 0.5) r = 1.0;
    carry = x - r;
    q = (int32_t)r;
}

constexpr size_t kInvTabSmem = 160 * 1024;  // larger codebooks read the tables from L1/L2


// Pass A -- the two chains of 32 segments: warp 0 the length carry
// (qlen), warp 1 the start values (vstart), one segment per lane. A lane's
// labels stream through a private shared-memory ring filled by asynchronous
// 16-byte copies (cp.async) RD tiles ahead, so the in-order warp never waits
// on memory: each step is its fp64 chain plus a shared-memory read.
constexpr int RT = 16;                    // labels per ring tile
constexpr int RD = 8;                     // tiles in flight
constexpr int RSTRIDE = RT * RD * 4 + 16; // bytes per lane (padded: conflict-free LDS.128)

__device__ __forceinline__ void ring_issue(unsigned char* my, const uint32_t* __restrict__ src,
                                           int slot) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(my + slot * RT * 4);
#pragma unroll
    for (int m = 0; m < RT / 4; ++m)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * m),
                     "l"(src + 4 * m));
}
__device__ __forceinline__ void ring_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void ring_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <bool SMEM_TABS>
__global__ void __launch_bounds__(64) k_inv_chains(InverseIn in, const double* __restrict__ rlen,
                                                   const double* __restrict__ rinc,
                                                   int32_t* __restrict__ qlen,
                                                   double* __restrict__ vstart,
                                                   const int64_t* __restrict__ grp_off,
                                                   int64_t* __restrict__ gsum,
                                                   unsigned long long* __restrict__ err,
                                                   const int64_t* __restrict__ list,
                                                   int64_t nlist) {
    // The carry warp also validates every label (inverse_digitize_series
    // :41-44) and sums the quantized lengths of each group of GROUP pieces;
    // both are off its fp64 critical path. list: the segments to process
    // (null: all); grp_off is indexed by list position.
    extern __shared__ double s_tabs[];  // rlen(k) | rinc(k)
    __shared__ __align__(16) unsigned char ring[64 * RSTRIDE];
    if (SMEM_TABS) {
        for (int c = threadIdx.x; c < (int)in.k; c += blockDim.x) {
            s_tabs[c] = rlen[c];
            s_tabs[in.k + c] = rinc[c];
        }
        __syncthreads();
    }
    const double* tabs = SMEM_TABS ? s_tabs : rlen;  // global: rinc follows rlen
    const int kk = (int)in.k;
    const bool cwarp = threadIdx.x < 32;  // carry warp / start-value warp
    const int64_t li = blockIdx.x * (int64_t)32 + (threadIdx.x & 31);
    if (li >= nlist) return;
    const int64_t s = list ? list[li] : li;
    unsigned char* my = ring + threadIdx.x * RSTRIDE;
    const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
    const double* tl = cwarp ? tabs : tabs + kk;
    double carry = 0.0, v = in.anchors[s];
    bool badlab = false;
    int64_t g = grp_off[li];
    long long gacc = 0;
    int gcnt = 0;
    auto lab_ok = [&](uint32_t lab) -> uint32_t {  // invalid labels flag the segment
        const bool bad = lab >= (uint32_t)kk;
        badlab |= bad;
        return bad ? 0u : lab;
    };
    auto gadd = [&](int32_t q) {
        gacc += q;
        if (++gcnt == GROUP) {
            gsum[g++] = gacc;
            gacc = 0;
            gcnt = 0;
        }
    };
    auto one = [&](int64_t j, uint32_t lab) {
        if (cwarp) {
            int32_t q;
            chain_step(tl[lab_ok(lab)], carry, q);
            qlen[j] = q;
            gadd(q);
        } else {
            vstart[j] = v;
            v += tl[lab < (uint32_t)kk ? lab : 0u];
        }
    };
    int64_t j = a;
    for (; j < b && (j & 3); ++j) one(j, in.labels[j]);
    const int64_t jb = j;
    const int64_t ntile = (b - jb) / RT;
    for (int t = 0; t < RD - 1; ++t) {
        if (t < ntile) ring_issue(my, in.labels + jb + (int64_t)t * RT, t);
        ring_commit();
    }
    for (int64_t t = 0; t < ntile; ++t) {
        if (t + RD - 1 < ntile) ring_issue(my, in.labels + jb + (t + RD - 1) * RT, (int)((t + RD - 1) % RD));
        ring_commit();
        ring_wait<RD - 1>();  // tile t has landed
        const uint4* src = reinterpret_cast<const uint4*>(my + (t % RD) * RT * 4);
        const int64_t j0 = jb + t * RT;
#pragma unroll
        for (int m = 0; m < RT / 4; ++m) {
            const uint4 L = src[m];
            const int64_t jj = j0 + 4 * m;
            if (cwarp) {
                int4 Q;
                chain_step(tl[lab_ok(L.x)], carry, Q.x);
                chain_step(tl[lab_ok(L.y)], carry, Q.y);
                chain_step(tl[lab_ok(L.z)], carry, Q.z);
                chain_step(tl[lab_ok(L.w)], carry, Q.w);
                *reinterpret_cast<int4*>(qlen + jj) = Q;
                gadd(Q.x);
                gadd(Q.y);
                gadd(Q.z);
                gadd(Q.w);
            } else {
                const double v0 = v;  // invalid labels: the carry warp reports them
                const double v1 = v0 + tl[L.x < (uint32_t)kk ? L.x : 0u];
                const double v2 = v1 + tl[L.y < (uint32_t)kk ? L.y : 0u];
                const double v3 = v2 + tl[L.z < (uint32_t)kk ? L.z : 0u];
                v = v3 + tl[L.w < (uint32_t)kk ? L.w : 0u];
                *reinterpret_cast<double2*>(vstart + jj) = make_double2(v0, v1);
                *reinterpret_cast<double2*>(vstart + jj + 2) = make_double2(v2, v3);
            }
        }
    }
    for (j = jb + ntile * RT; j < b; ++j) one(j, in.labels[j]);
    if (cwarp) {
        if (gcnt) gsum[g] = gacc;
        if (badlab) atomicMin(err, (unsigned long long)(s * 4 + kErrLabel));
    }
}

// Per segment (warp): match_total_length's backward cascade (lane 0), then
// the output position of every group (exact scan of the group sums) and
// the fill records. Errors: the lowest failing segment wins.
struct GroupRec {
    int64_t base;  // first piece
    int64_t pos;   // output index of the sample before the group's first sample
};

__global__ void k_inv_segfix(InverseIn in, int32_t* __restrict__ qlen,
                             const int64_t* __restrict__ grp_off, int64_t* __restrict__ gsum,
                             GroupRec* __restrict__ rec, int32_t* __restrict__ gmeta,
                             double* __restrict__ out, unsigned long long* __restrict__ err,
                             const int64_t* __restrict__ list, int64_t nlist) {
    const int lane = threadIdx.x & 31;
    for (int64_t li = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; li < nlist;
         li += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t s = list ? list[li] : li;
        const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
        const int64_t g0 = grp_off[li], g1 = grp_off[li + 1];
        long long total = 0;
        for (int64_t g = g0 + lane; g < g1; g += 32) total += gsum[g];
        for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
        int bad = 0;
        if (lane == 0) {
            long long residual = in.source_lengths[s] - total;
            for (int64_t t = b; t-- > a && residual != 0;) {
                long long adj = (long long)qlen[t] + residual;
                if (adj < 1) adj = 1;
                const long long delta = adj - qlen[t];
                residual -= delta;
                qlen[t] = (int32_t)adj;
                gsum[g0 + (t - a) / GROUP] += delta;
            }
            bad = residual != 0 || b == a;
            if (bad) atomicMin(err, (unsigned long long)(s * 4 + kErrPiece));
            else out[in.out_offsets[s]] = in.anchors[s];
        }
        bad = __shfl_sync(0xffffffffu, bad, 0);
        if (bad) continue;
        __syncwarp();
        // group positions: exclusive scan of the group sums
        const bool drop = in.layout == 0 && (s + 1 < in.n_seg || in.drop_local_last);
        long long run = in.out_offsets[s];
        for (int64_t g = g0; g < g1; g += 32) {
            const int64_t gg = g + lane;
            const long long v = gg < g1 ? gsum[gg] : 0;
            long long incl = v;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (gg < g1) {
                const int64_t base = a + (gg - g0) * GROUP;
                const int cnt = (int)(b - base < GROUP ? b - base : GROUP);
                rec[gg] = GroupRec{base, run + incl - v};
                gmeta[gg] = cnt | ((drop && gg == g1 - 1) ? 0x100 : 0);
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

// Pass B -- one warp per group of GROUP pieces. A lane writes its own
// piece's samples v + inc * (i / len) (inverse_compress :97-99; positions
// from the group's exact scan); a group holding a long piece switches to a
// sample-parallel layout. A non-final part of a univariate-partitioned fit
// drops its last sample (stitch_partitions :198-213).
constexpr int DIV_MAX = 31;  // exact i/len table for len <= DIV_MAX (7.9 KB smem)
constexpr int LANE_MAX = 16; // pieces up to this length: lane per piece
constexpr int FILL_TB = 256;

__global__ void __launch_bounds__(FILL_TB) k_inv_fill(InverseIn in, const double* __restrict__ rinc,
                                                  const int32_t* __restrict__ qlen,
                                                  const double* __restrict__ vstart,
                                                  const GroupRec* __restrict__ rec,
                                                  const int32_t* __restrict__ gmeta,
                                                  int64_t n_groups, double* __restrict__ out) {
    __shared__ double div_tab[(DIV_MAX + 1) * (DIV_MAX + 1)];
    __shared__ double s_stage[FILL_TB / 32][32 * LANE_MAX];
    extern __shared__ double s_inc[];
    const int kk = (int)in.k;
    const bool inc_smem = (size_t)kk * sizeof(double) <= kInvTabSmem / 2;
    for (int t = threadIdx.x; t < (DIV_MAX + 1) * (DIV_MAX + 1); t += blockDim.x) {
        const int l = t / (DIV_MAX + 1), i = t % (DIV_MAX + 1);
        div_tab[t] = l > 0 ? (double)i / (double)l : 0.0;  // the same IEEE division
    }
    if (inc_smem)
        for (int c = threadIdx.x; c < kk; c += blockDim.x) s_inc[c] = rinc[c];
    __syncthreads();
    const double* tinc = inc_smem ? s_inc : rinc;
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < n_groups;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const GroupRec r = rec[g];
        const int meta = gmeta[g];
        const int cnt = meta & 0xFF;
        const bool drop_last = (meta & 0x100) != 0;  // the group holds the dropped sample
        const int64_t j = r.base + lane;
        const bool valid = lane < cnt;
        const int len = valid ? qlen[j] : 0;
        const double inc = valid ? tinc[in.labels[j]] : 0.0;
        const double myv = valid ? vstart[j] : 0.0;
        long long incl = len;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const int maxlen = __reduce_max_sync(FULL, len);
        const long long L = __shfl_sync(FULL, incl, 31);
        if (maxlen <= LANE_MAX) {
            // lane per piece into the warp's staging row, then one coalesced copy
            double* st = s_stage[threadIdx.x >> 5];
            if (valid) {
                const int p0 = (int)(incl - len);
                for (int i = 1; i <= len; ++i)
                    st[p0 + i - 1] = myv + inc * div_tab[len * (DIV_MAX + 1) + i];
            }
            __syncwarp();
            const int Le = (int)L - (drop_last ? 1 : 0);
            for (int q = lane; q < Le; q += 32) out[r.pos + 1 + q] = st[q];
            __syncwarp();
            continue;
        }
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
                out[r.pos + q] = vi + ii * frac;
            }
        }
    }
}

// ---- fused path (the common case) ----
// One block = 32 segments, three warp-specialized roles connected by
// shared-memory rings with mbarrier full/empty handshakes, so each role runs
// at its own pace and the carry chain -- the latency-bound critical path --
// never waits on the others while the rings have room:
//  * the value warp (warp 1), lane = segment, streams the labels through a
//    cp.async ring, checks them (inverse_digitize_series :41-44), runs the
//    start-value chain (inverse_compress :94-101) and looks up each piece's
//    real length and increment;
//  * the carry warp (warp 0), lane = segment, runs only the length-carry
//    chain (quantize_lengths :63-74) on real lengths waiting in shared
//    memory and records each piece's quantized length and last output
//    position;
//  * the writer warps store every sample at its final position, lane per
//    piece: a piece's last sample v + inc * (q / q) is the next piece's start
//    value (inc * 1.0 == inc), so the common one-sample piece costs a
//    shared-memory load and a store; the other samples of longer pieces
//    (v + inc * (i / q)) go through a flattened per-warp queue.
// The last TAILT tiles of a segment are not written in the loop: their
// lengths, start values and increments go to a global scratch, the carry warp
// applies match_total_length's backward cascade (:81-93) there once the
// segment's chain is done (the cascade moves only the tail, so every piece
// written in the loop sits at its final position), and all warps write the
// tails after the loop. A cascade reaching past the tail sends the call to
// the general path (counted in err[1]).
#ifndef JB_FUSED_NOWRITE
#define JB_FUSED_NOWRITE 0
#endif
#ifndef JB_FUSED_PROF  // experiment builds: per-role busy / waiting cycles
#define JB_FUSED_PROF 0
#endif
#if JB_FUSED_PROF
__device__ unsigned long long g_fused_prof[8];
#define FP_WAIT(call)                                \
    do {                                             \
        const long long t0_ = clock64();             \
        call;                                        \
        fp_wait += clock64() - t0_;                  \
    } while (0)
#else
#define FP_WAIT(call) call
#endif
constexpr int FRD = 4;                    // label tiles in flight (value warp)
constexpr int FLSTR = FRD * RT * 4 + 16;  // label ring bytes per lane
constexpr int DL = 2, DQ = 2, DV = 4;     // ring depths: real lengths, quantized, start values
constexpr int LVS = RT + 2;               // real-length row (padded: conflict-free 128-bit)
constexpr int QPS = RT + 4;               // quantized-length / last-position row (padded)
constexpr int VSS = RT + 1;               // (start value, increment) x RT + the value after
constexpr int FDIV = 16;                  // exact i / q table for q <= FDIV
constexpr int FWW = 4;                    // writer warps
constexpr int FUSED_TB = 32 * (2 + FWW);
constexpr int TAILT = 16;                 // tiles per segment left to the tail pass
constexpr int WP = 16 / FWW;              // (segment, tile) half-warp pairs per writer warp
constexpr int WQ = WP * 32;               // queue entries per writer warp
constexpr int NBAR = 2 * (DL + DQ + DV);

struct FusedSmem {  // rows 16-byte aligned (cp.async, 128-bit accesses)
    unsigned long long bar[NBAR];  // full / empty mbarriers of the three rings
    unsigned char lab[32 * FLSTR];
    double2 vs[DV][32 * VSS];
    double lv[DL][32 * LVS];
    int32_t q[DQ][32 * QPS];       // quantized length (0: nothing to write in the loop)
    int32_t pe[DQ][32 * QPS];      // last output position, from the segment's anchor
    double div[(FDIV + 1) * (FDIV + 1)];
    long long oo[32];              // output index of each segment's anchor
    int32_t E[32];                 // the segment's last position (-1: none)
    int ntile[32];
    int bail[32];
    uint16_t wq[FWW][WQ];          // queued pieces: segment << 4 | piece
};
static_assert(32 * FLSTR % 16 == 0 && LVS * 8 % 16 == 0 && QPS * 4 % 16 == 0 && NBAR % 2 == 0,
              "fused ring rows must stay 16-byte aligned");

struct TailScratch {  // per segment (from off[s]): its tail pieces + 1
    const int64_t* off;
    int32_t* q;
    int32_t* pe;
    double* inc;
    double* v;  // start values; the entry after the last piece: the value after it
};

// tail layout: the same integer expressions as k_inv_fused
__device__ __forceinline__ int64_t tail_first_piece(int64_t a, int64_t b) {
    const int64_t base = a & ~(int64_t)3;
    const int ntile = b > a ? (int)((b - base + RT - 1) / RT) : 0;
    const int tt0 = ntile > TAILT ? ntile - TAILT : 0;
    return max(a, base + (int64_t)tt0 * RT);
}
__global__ void k_tail_sizes(const int64_t* __restrict__ seg_offsets, int64_t n_seg,
                             int64_t* __restrict__ sz) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_seg;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = seg_offsets[s], b = seg_offsets[s + 1];
        sz[s] = b - tail_first_piece(a, b) + 1;
    }
}

__device__ __forceinline__ void ring_issue_z(unsigned char* my, const uint32_t* __restrict__ labels,
                                             int64_t idx, int64_t n, int slot) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(my + slot * RT * 4);
#pragma unroll
    for (int m = 0; m < RT / 4; ++m) {
        const int64_t i = idx + 4 * m;  // 16-byte chunk: zero-filled past the label array
        const int64_t rem = n - i;
        const unsigned nb = rem >= 4 ? 16u : rem > 0 ? (unsigned)rem * 4u : 0u;
        const uint32_t* src = nb ? labels + i : labels;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + 16 * m),
                     "l"(src), "r"(nb));
    }
}

__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(b)),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(b))
                 : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
        "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep instead of spinning
        : "memory");
}

// A warp writes the samples of up to 32 pieces, lane per piece: q samples
// ending at position pe (from the segment anchor at ob), the last one vnext,
// the others vv + inc * (i / q); positions beyond E are dropped. (Tail pass.)
__device__ __forceinline__ void emit_pieces(int q, int pe, int E, double* ob, double vnext,
                                            double vv, double inc, const double* div) {
    const unsigned FULL = 0xffffffffu;
    if (q > 0 && pe <= E) ob[pe] = vnext;
    const int qmax = __reduce_max_sync(FULL, q);
    if (qmax <= 1) return;
    const int lane = threadIdx.x & 31;
    const unsigned mq = __ballot_sync(FULL, q > 1);
    unsigned lm = mq;
    while (lm) {  // a piece at a time, its other samples across the warp
        const int src = __ffs(lm) - 1;
        lm &= lm - 1;
        const int qs = __shfl_sync(FULL, q, src);
        const int ps = __shfl_sync(FULL, pe - q + 1, src);
        const int es = __shfl_sync(FULL, E, src);
        const double vs = __shfl_sync(FULL, vv, src);
        const double is = __shfl_sync(FULL, inc, src);
        double* os =
            reinterpret_cast<double*>(__shfl_sync(FULL, reinterpret_cast<unsigned long long>(ob), src));
        for (int i = 1 + lane; i < qs; i += 32)
            if (ps + i - 1 <= es) {
                const double fr = qs <= FDIV ? div[qs * (FDIV + 1) + i] : (double)i / (double)qs;
                os[ps + i - 1] = vs + is * fr;
            }
    }
}

template <bool SMEM_TABS>
__global__ void __launch_bounds__(FUSED_TB, 3) k_inv_fused(InverseIn in, const double* __restrict__ rlen,
                                                           const double* __restrict__ rinc,
                                                           double* __restrict__ out, TailScratch tail,
                                                           unsigned long long* __restrict__ err,
                                                           unsigned char* __restrict__ bailed) {
    extern __shared__ __align__(128) unsigned char dsm[];
    const int kk = (int)in.k;
    const size_t toff = SMEM_TABS ? ((size_t)2 * kk * sizeof(double) + 127) & ~(size_t)127 : 0;
    double* s_tabs = reinterpret_cast<double*>(dsm);
    FusedSmem& S = *reinterpret_cast<FusedSmem*>(dsm + toff);
    if (SMEM_TABS)
        for (int c = threadIdx.x; c < kk; c += blockDim.x) {
            s_tabs[c] = rlen[c];
            s_tabs[kk + c] = rinc[c];
        }
    for (int t = threadIdx.x; t < (FDIV + 1) * (FDIV + 1); t += blockDim.x) {
        const int l = t / (FDIV + 1), i = t % (FDIV + 1);
        S.div[t] = l > 0 ? (double)i / (double)l : 0.0;  // the same IEEE division
    }
    unsigned long long* LVF = S.bar;
    unsigned long long* LVE = LVF + DL;
    unsigned long long* QF = LVE + DL;
    unsigned long long* QE = QF + DQ;
    unsigned long long* VF = QE + DQ;
    unsigned long long* VE = VF + DV;
    if (threadIdx.x == 0) {
        for (int k = 0; k < DL; ++k) {
            mb_init(LVF + k, 32);
            mb_init(LVE + k, 32);
        }
        for (int k = 0; k < DQ; ++k) {
            mb_init(QF + k, 32);
            mb_init(QE + k, 32 * FWW);
        }
        for (int k = 0; k < DV; ++k) {
            mb_init(VF + k, 32);
            mb_init(VE + k, 32 * FWW);
        }
    }
    const double* tlen = SMEM_TABS ? s_tabs : rlen;
    const double* tinc = SMEM_TABS ? s_tabs + kk : rinc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // segment of this lane (carry and value warps)
    const int64_t s = blockIdx.x * (int64_t)32 + lane;
    const bool live = s < in.n_seg;
    int64_t a = 0, b = 0;
    if (warp < 2 && live) {
        a = in.seg_offsets[s];
        b = in.seg_offsets[s + 1];
    }
    const int64_t base = a & ~(int64_t)3;  // 16-byte aligned label tiles
    const int ntile = b > a ? (int)((b - base + RT - 1) / RT) : 0;
    const int tt0 = ntile > TAILT ? ntile - TAILT : 0;    // first tail tile
    const int64_t jlo = max(a, base + (int64_t)tt0 * RT);  // first tail piece
    const int64_t tofs = live && warp < 2 ? tail.off[s] - jlo : 0;  // scratch index of piece j
    if (warp == 0) {
        long long E = -1;
        if (live) {
            const long long o = in.out_offsets[s];
            const bool drop = in.layout == 0 && (s + 1 < in.n_seg || in.drop_local_last);
            E = in.source_lengths[s] - (drop ? 1 : 0);
            if (E >= 0) out[o] = in.anchors[s];
            S.oo[lane] = o;
        } else {
            S.oo[lane] = 0;
        }
        S.E[lane] = (int32_t)(E < 0x7FFFFFFFLL ? E : 0);
        S.ntile[lane] = ntile;
        S.bail[lane] = E >= 0x7FFFFFFFLL;  // positions from the anchor are ints
    }
    __syncthreads();
    int maxT = 0;
    for (int l = 0; l < 32; ++l) maxT = max(maxT, S.ntile[l]);

    long long fp_wait = 0, fp_t0 = clock64();
    (void)fp_wait;
    (void)fp_t0;
    if (warp == 1) {
        // ---- value warp ----
        unsigned char* lrow = S.lab + lane * FLSTR;
        double v = live ? in.anchors[s] : 0.0;
        bool badlab = false;
        for (int t = 0; t < FRD - 1; ++t) {
            if (t < ntile) ring_issue_z(lrow, in.labels, base + (int64_t)t * RT, in.N, t);
            ring_commit();
        }
        for (int it = 0; it < maxT; ++it) {
            const int k = it % DL, kv = it % DV;
            FP_WAIT(mb_wait(LVE + k, ((it / DL) & 1) ^ 1));
            FP_WAIT(mb_wait(VE + kv, ((it / DV) & 1) ^ 1));
            const int tn = it + FRD - 1;
            if (tn < ntile) ring_issue_z(lrow, in.labels, base + (int64_t)tn * RT, in.N, tn % FRD);
            ring_commit();
            ring_wait<FRD - 1>();  // tile it has landed
            if (it < ntile) {
                const uint32_t* lt = reinterpret_cast<const uint32_t*>(lrow + (it % FRD) * RT * 4);
                double2* vt = S.vs[kv] + lane * VSS;
                double* lv = S.lv[k] + lane * LVS;
                const int64_t jt = base + (int64_t)it * RT;
                if (jt >= a && jt + RT <= b) {
#pragma unroll
                    for (int mm = 0; mm < RT / 4; ++mm) {
                        const uint4 L = reinterpret_cast<const uint4*>(lt)[mm];
                        uint32_t l[4] = {L.x, L.y, L.z, L.w};
                        double inc[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            badlab |= l[e] >= (uint32_t)kk;
                            l[e] = l[e] < (uint32_t)kk ? l[e] : 0u;
                            inc[e] = tinc[l[e]];
                        }
                        reinterpret_cast<double2*>(lv)[2 * mm] = make_double2(tlen[l[0]], tlen[l[1]]);
                        reinterpret_cast<double2*>(lv)[2 * mm + 1] =
                            make_double2(tlen[l[2]], tlen[l[3]]);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            vt[4 * mm + e] = make_double2(v, inc[e]);
                            v += inc[e];
                        }
                    }
                } else {
                    for (int mm = 0; mm < RT; ++mm) {
                        const int64_t j = jt + mm;
                        double inc = 0.0;
                        lv[mm] = 0.0;
                        if (j >= a && j < b) {
                            uint32_t l = lt[mm];
                            badlab |= l >= (uint32_t)kk;
                            l = l < (uint32_t)kk ? l : 0u;
                            lv[mm] = tlen[l];
                            inc = tinc[l];
                        }
                        vt[mm] = make_double2(v, inc);
                        v += inc;
                    }
                }
                vt[RT] = make_double2(v, 0.0);  // the start value after the tile
                if (it >= tt0) {  // tail tile: start values and increments to the scratch
                    for (int mm = 0; mm < RT; ++mm) {
                        const int64_t j = jt + mm;
                        if (j >= jlo && j < b) {
                            tail.v[tofs + j] = vt[mm].x;
                            tail.inc[tofs + j] = vt[mm].y;
                        }
                    }
                    if (it == ntile - 1) tail.v[tofs + b] = v;
                }
            }
            mb_arrive(LVF + k);
            mb_arrive(VF + kv);
        }
        if (badlab) atomicMin(err, (unsigned long long)(s * 4 + kErrLabel));
    } else if (warp == 0) {
        // ---- carry warp ----
        double carry = 0.0;
        long long total = 0, pos = 1, pos_tail = 1;  // positions from the anchor
        bool bail = S.bail[lane];
        if (bail) {
            atomicAdd(err + 1, 1ULL);
            bailed[s] = 1;
        }
        auto do_bail = [&]() {
            if (!bail) {
                bail = true;
                atomicAdd(err + 1, 1ULL);
                bailed[s] = 1;
            }
        };
        for (int it = 0; it < maxT; ++it) {
            const int k = it % DL, kq = it % DQ;
            FP_WAIT(mb_wait(LVF + k, (it / DL) & 1));
            double l[RT];
            const double* lv = S.lv[k] + lane * LVS;
#pragma unroll
            for (int mm = 0; mm < RT / 2; ++mm) {
                const double2 d = reinterpret_cast<const double2*>(lv)[mm];
                l[2 * mm] = d.x;
                l[2 * mm + 1] = d.y;
            }
            mb_arrive(LVE + k);
            int32_t* qt = S.q[kq] + lane * QPS;
            int32_t* pt = S.pe[kq] + lane * QPS;
            int32_t Q[RT];
            const int64_t jt = base + (int64_t)it * RT;
            if (it < ntile) {
                if (it == tt0) pos_tail = pos;
                if (jt >= a && jt + RT <= b) {
#pragma unroll
                    for (int mm = 0; mm < RT; ++mm) chain_step(l[mm], carry, Q[mm]);
                } else {
                    for (int mm = 0; mm < RT; ++mm) {
                        const int64_t j = jt + mm;
                        Q[mm] = 0;
                        if (j >= a && j < b) chain_step(l[mm], carry, Q[mm]);
                    }
                }
            }
            FP_WAIT(mb_wait(QE + kq, ((it / DQ) & 1) ^ 1));
            if (it < tt0 && !bail) {
#pragma unroll
                for (int mm = 0; mm < RT / 4; ++mm) {
                    int4 q4, p4;
                    q4.x = Q[4 * mm];
                    q4.y = Q[4 * mm + 1];
                    q4.z = Q[4 * mm + 2];
                    q4.w = Q[4 * mm + 3];
                    p4.x = (int)(pos += q4.x) - 1;
                    p4.y = (int)(pos += q4.y) - 1;
                    p4.z = (int)(pos += q4.z) - 1;
                    p4.w = (int)(pos += q4.w) - 1;
                    reinterpret_cast<int4*>(qt)[mm] = q4;
                    reinterpret_cast<int4*>(pt)[mm] = p4;
                }
            } else {  // tail tile, finished or bailed segment: nothing to write in the loop
#pragma unroll
                for (int mm = 0; mm < RT / 4; ++mm)
                    reinterpret_cast<int4*>(qt)[mm] = make_int4(0, 0, 0, 0);
                if (it < ntile) {
#pragma unroll
                    for (int mm = 0; mm < RT; ++mm) {
                        const int64_t j = jt + mm;
                        if (it >= tt0 && j >= jlo && j < b) tail.q[tofs + j] = Q[mm];
                        pos += Q[mm];
                    }
                }
            }
            mb_arrive(QF + kq);
            if (it < ntile) {
                if (pos > 0x7FFFFFFFLL) do_bail();
                if (it == ntile - 1) {  // match_total_length on the tail
                    total = pos - 1;
                    long long residual = in.source_lengths[s] - total;
                    int32_t* tq = tail.q + tofs;  // indexed by piece
                    for (int64_t j = b - 1; j >= jlo && residual != 0; --j) {
                        long long adj = (long long)tq[j] + residual;
                        if (adj < 1) adj = 1;
                        residual -= adj - tq[j];
                        tq[j] = (int32_t)adj;
                    }
                    if (residual != 0) {
                        if (jlo == a) atomicMin(err, (unsigned long long)(s * 4 + kErrPiece));
                        else do_bail();
                    }
                    long long pp = pos_tail;
                    int32_t* tp = tail.pe + tofs;
                    for (int64_t j = jlo; j < b; ++j) {
                        pp += tq[j];
                        tp[j] = (int32_t)(pp - 1);
                    }
                    if (pp > 0x7FFFFFFFLL) do_bail();
                }
            }
        }
        (void)total;
        if (live && b == a) atomicMin(err, (unsigned long long)(s * 4 + kErrPiece));
        S.bail[lane] = bail;
    } else if (!JB_FUSED_NOWRITE) {
        // ---- writer warps: lane m of half h holds piece m of segment L ----
        const int wi = warp - 2, m = lane & 15;
        int wE[WP];
        double* wout[WP];
#pragma unroll
        for (int k = 0; k < WP; ++k) {
            const int L = 2 * wi + (lane >> 4) + 2 * FWW * k;
            wE[k] = S.E[L];
            wout[k] = out + S.oo[L];  // derived from the kernel argument: global stores
        }
        for (int it = 0; it < maxT; ++it) {
            const int kq = it % DQ, kv = it % DV;
            FP_WAIT(mb_wait(QF + kq, (it / DQ) & 1));
            FP_WAIT(mb_wait(VF + kv, (it / DV) & 1));
            // all shared-memory reads of the WP segment pairs first (independent,
            // in flight together), then the stores, then the queue of longer pieces
            int qk[WP], pek[WP];
            double vk[WP];
#pragma unroll
            for (int k = 0; k < WP; ++k) {
                const int L = 2 * wi + (lane >> 4) + 2 * FWW * k;
                qk[k] = S.q[kq][L * QPS + m];
                pek[k] = S.pe[kq][L * QPS + m];
                vk[k] = S.vs[kv][L * VSS + m + 1].x;
            }
#pragma unroll
            for (int k = 0; k < WP; ++k)
                if (qk[k] > 0 && pek[k] <= wE[k]) wout[k][pek[k]] = vk[k];
            int nq = 0;
#pragma unroll
            for (int k = 0; k < WP; ++k) {
                const int L = 2 * wi + (lane >> 4) + 2 * FWW * k;
                const unsigned mq = __ballot_sync(0xffffffffu, qk[k] > 1);
                if (qk[k] > 1) S.wq[wi][nq + __popc(mq & ((1u << lane) - 1u))] = (uint16_t)(L << 4 | m);
                nq += __popc(mq);
            }
            __syncwarp();
            // the other samples of the queued pieces, flattened over the warp
            for (int e0 = 0; e0 < nq; e0 += 32) {
                const int e = e0 + lane;
                const int ent = e < nq ? S.wq[wi][e] : 0;
                const int cnt = e < nq ? S.q[kq][(ent >> 4) * QPS + (ent & 15)] - 1 : 0;
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int ex = incl - cnt;
                const int tot = __shfl_sync(0xffffffffu, incl, 31);
                for (int c0 = 0; c0 < tot; c0 += 32) {
                    const int c = c0 + lane;
                    int p = 0;  // last entry with ex <= c: the one holding sample c
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1) {
                        const int x = __shfl_sync(0xffffffffu, ex, p + st);
                        if (x <= c) p += st;
                    }
                    const int xp = __shfl_sync(0xffffffffu, ex, p);
                    const int en = __shfl_sync(0xffffffffu, ent, p);
                    if (c < tot) {
                        const int L = en >> 4, mm = en & 15;
                        const int q = S.q[kq][L * QPS + mm];
                        const int P0 = S.pe[kq][L * QPS + mm] - q + 1;
                        const int i = c - xp + 1;  // 1 .. q-1
                        if (P0 + i - 1 <= S.E[L]) {
                            const double2 vi = S.vs[kv][L * VSS + mm];
                            const double fr =
                                q <= FDIV ? S.div[q * (FDIV + 1) + i] : (double)i / (double)q;
                            out[S.oo[L] + P0 + i - 1] = vi.x + vi.y * fr;
                        }
                    }
                }
            }
            __syncwarp();
            mb_arrive(QE + kq);
            mb_arrive(VE + kv);
        }
    }
    if (JB_FUSED_NOWRITE && warp >= 2) {  // keep the handshakes balanced
        for (int it = 0; it < maxT; ++it) {
            mb_wait(QF + it % DQ, (it / DQ) & 1);
            mb_wait(VF + it % DV, (it / DV) & 1);
            mb_arrive(QE + it % DQ);
            mb_arrive(VE + it % DV);
        }
    }
#if JB_FUSED_PROF
    if (lane == 0) {
        const int role = warp < 2 ? warp : 2;
        atomicAdd(&g_fused_prof[2 * role], (unsigned long long)(clock64() - fp_t0));
        atomicAdd(&g_fused_prof[2 * role + 1], (unsigned long long)fp_wait);
    }
#endif
    __syncthreads();
    if (warp == 0) S.ntile[lane] = (int)(live && b > a ? b - jlo : 0);  // tail pieces
    __syncthreads();
    if (JB_FUSED_NOWRITE) return;
    // tail pass: a warp per segment, lane per piece
    constexpr int NW = FUSED_TB / 32;
    for (int L = warp; L < 32; L += NW) {
        const int64_t sg = blockIdx.x * (int64_t)32 + L;
        const int cnt = S.ntile[L];
        if (S.bail[L] || cnt == 0) continue;
        const int E = S.E[L];
        double* ob = out + S.oo[L];
        const int64_t so = tail.off[sg];
        for (int c = 0; c < cnt; c += 32) {
            const int64_t u = so + c + lane;
            int q = 0, pe = 0;
            double vn = 0.0, vv = 0.0, inc = 0.0;
            if (c + lane < cnt) {
                q = tail.q[u];
                pe = tail.pe[u];
                vn = tail.v[u + 1];
                if (q > 1) {
                    vv = tail.v[u];
                    inc = tail.inc[u];
                }
            }
            emit_pieces(q, pe, E, ob, vn, vv, inc, S.div);
        }
    }
}

}  // namespace

static void throw_inverse_error(unsigned long long e, uint64_t k) {
    if (e == ~0ULL) return;
    const long long seg = (long long)(e / 4);
    if (e % 4 == kErrLabel)
        throw Error(UNKNOWN_SYMBOL, "label not in codebook of size " + std::to_string(k) +
                                        " (segment " + std::to_string(seg) + ")");
    throw Error(INVALID_PIECE, "cannot fit pieces into the segment's steps (segment " +
                                   std::to_string(seg) + ")");
}

// The general path: both chains write per-piece state (qlen, vstart), the
// cascade and positions run per segment, and a piece-parallel pass fills.
// Used when some segment's cascade reaches further back than the fused
// kernel's window.
static void inverse_general(const InverseIn& in, const double* tabp, uint64_t kk,
                            DArr<unsigned long long>& err, double* d_out, cudaStream_t st,
                            const std::vector<int64_t>* segs = nullptr) {
    // segs: the segments to (re)write (null: all). Group layout on the host
    // (segment piece counts are needed anyway for the offsets), by list position
    std::vector<int64_t> h_off(in.n_seg + 1);
    JB_CUDA(cudaMemcpyAsync(h_off.data(), in.seg_offsets, sizeof(int64_t) * (in.n_seg + 1),
                            cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    const int64_t nlist = segs ? (int64_t)segs->size() : in.n_seg;
    std::vector<int64_t> h_goff(nlist + 1);
    h_goff[0] = 0;
    for (int64_t li = 0; li < nlist; ++li) {
        const int64_t s = segs ? (*segs)[li] : li;
        h_goff[li + 1] = h_goff[li] + (h_off[s + 1] - h_off[s] + GROUP - 1) / GROUP;
    }
    const int64_t n_groups = h_goff[nlist];
    DArr<int64_t> goff(nlist + 1, st), dlist(segs ? std::max<int64_t>(nlist, 1) : 0, st);
    goff.upload(h_goff.data(), nlist + 1);
    if (segs) dlist.upload(segs->data(), nlist);
    const int64_t* lp = segs ? dlist.p : nullptr;
    const int64_t ng = std::max<int64_t>(n_groups, 1);
    DArr<int32_t> qlen(std::max<int64_t>(in.N, 1) + 4, st), gmeta(ng, st);
    DArr<double> vstart(std::max<int64_t>(in.N, 1) + 4, st);
    DArr<int64_t> gsum(ng, st);
    DArr<GroupRec> rec(ng, st);
    const size_t tsmem = sizeof(double) * 2 * kk <= kInvTabSmem ? sizeof(double) * 2 * kk : 0;
    {
        JB_PROF("inverse_chain", st);
        auto kern = tsmem ? k_inv_chains<true> : k_inv_chains<false>;
        if (tsmem + 64 * RSTRIDE > 48 * 1024)
            JB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tsmem));
        kern<<<(int)std::max<int64_t>(1, (nlist + 31) / 32), 64, tsmem, st>>>(
            in, tabp, tabp + kk, qlen.p, vstart.p, goff.p, gsum.p, err.p, lp, nlist);
        JB_LAUNCH_CHECK();
        k_inv_segfix<<<(int)std::max<int64_t>(1, std::min<int64_t>((nlist * 32 + 255) / 256,
                                                                   (int64_t)num_sms() * 16)),
                       256, 0, st>>>(in, qlen.p, goff.p, gsum.p, rec.p, gmeta.p, d_out, err.p, lp,
                                     nlist);
        JB_LAUNCH_CHECK();
    }
    unsigned long long e;
    err.download(&e, 1);
    JB_CUDA(cudaStreamSynchronize(st));
    throw_inverse_error(e, in.k);
    if (n_groups > 0) {
        JB_PROF("inverse_fill", st);
        const size_t fsmem = sizeof(double) * kk <= kInvTabSmem / 2 ? sizeof(double) * kk : 0;
        if (fsmem > 8 * 1024)  // 40 KB static (division table + staging rows)
            JB_CUDA(cudaFuncSetAttribute(k_inv_fill, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)fsmem));
        const int grid = (int)std::max<int64_t>(
            1, std::min<int64_t>((n_groups * 32 + FILL_TB - 1) / FILL_TB, (int64_t)num_sms() * 16));
        k_inv_fill<<<grid, FILL_TB, fsmem, st>>>(in, tabp + kk, qlen.p, vstart.p, rec.p, gmeta.p,
                                             n_groups, d_out);
        JB_LAUNCH_CHECK();
    }
}

void inverse_transform_device(const InverseIn& in, double* d_out, cudaStream_t st) {
    if (in.layout == 0 && in.n_seg == 0)
        throw Error(INVALID_INPUT, "stitch_partitions: no segments");
    const uint64_t kk = std::max<uint64_t>(in.k, 1);
    DArr<double> tab(2 * kk, st);
    DArr<unsigned long long> err(2, st);  // [0] lowest error code, [1] segments needing the general path
    const unsigned long long init[2] = {~0ULL, 0ULL};
    err.upload(init, 2);
    if (in.k > 0) {
        k_inv_tables<<<(int)std::min<uint64_t>((in.k + 255) / 256, 1024), 256, 0, st>>>(
            in.centers, in.mean_lengths, in.k, in.scl, in.sigma_len, in.sigma_inc, tab.p,
            tab.p + kk);
        JB_LAUNCH_CHECK();
    }
    if (in.n_seg == 0) return;
    unsigned long long h[2];
    DArr<unsigned char> bailed;  // segments whose cascade left the fused kernel's window
    {
        JB_PROF("inverse_fused", st);
        const size_t tsmem = sizeof(double) * 2 * kk <= kInvTabSmem ? sizeof(double) * 2 * kk : 0;
        const size_t smem = tsmem + sizeof(FusedSmem) + 128;
        auto kern = tsmem ? k_inv_fused<true> : k_inv_fused<false>;
        JB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // tail scratch offsets: exclusive scan of (tail pieces + 1)
        DArr<int64_t> tsz(in.n_seg + 1, st), toff(in.n_seg + 1, st);
        k_tail_sizes<<<(int)std::min<int64_t>((in.n_seg + 255) / 256, 4096), 256, 0, st>>>(
            in.seg_offsets, in.n_seg, tsz.p);
        JB_LAUNCH_CHECK();
        JB_CUDA(cudaMemsetAsync(tsz.p + in.n_seg, 0, sizeof(int64_t), st));
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, tsz.p, toff.p, in.n_seg + 1, st);
        DArr<uint8_t> tmp(tb, st);
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, tsz.p, toff.p, in.n_seg + 1, st);
        int64_t ntail = 0;
        JB_CUDA(cudaMemcpyAsync(&ntail, toff.p + in.n_seg, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        DArr<int32_t> tq(ntail, st), tpe(ntail, st);
        DArr<double> tinc(ntail, st), tv(ntail, st);
        const TailScratch tail{toff.p, tq.p, tpe.p, tinc.p, tv.p};
        bailed.alloc(in.n_seg, st);
        bailed.zero();
        kern<<<(int)((in.n_seg + 31) / 32), FUSED_TB, smem, st>>>(in, tab.p, tab.p + kk, d_out,
                                                                   tail, err.p, bailed.p);
        JB_LAUNCH_CHECK();
        err.download(h, 2);
        JB_CUDA(cudaStreamSynchronize(st));
    }
#if JB_FUSED_PROF
    {
        unsigned long long pr[8];
        JB_CUDA(cudaMemcpyFromSymbol(pr, g_fused_prof, sizeof(pr)));
        const double nb = (double)((in.n_seg + 31) / 32);
        fprintf(stderr, "[jb] fused roles (Mcycles per block): carry %.2f (wait %.2f) value %.2f (wait %.2f) writers %.2f (wait %.2f)\n",
                pr[0] / nb / 1e6, pr[1] / nb / 1e6, pr[2] / nb / 1e6, pr[3] / nb / 1e6,
                pr[4] / nb / FWW / 1e6, pr[5] / nb / FWW / 1e6);
        const unsigned long long z[8] = {};
        JB_CUDA(cudaMemcpyToSymbol(g_fused_prof, z, sizeof(z)));
    }
#endif
    if (h[1] != 0) {  // cascades outside the window: those segments again, on the general path
        std::vector<unsigned char> hb(in.n_seg);
        bailed.download(hb.data(), in.n_seg);
        JB_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> segs;
        for (int64_t s = 0; s < in.n_seg; ++s)
            if (hb[s]) segs.push_back(s);
        // err[0] keeps the fused pass's errors (labels everywhere, cascades of
        // the other segments); the listed segments' own cascades are decided now
        const unsigned long long keep[2] = {h[0], 0ULL};
        err.upload(keep, 2);
        inverse_general(in, tab.p, kk, err, d_out, st, &segs);
        return;
    }
    throw_inverse_error(h[0], in.k);
}

}  // namespace jb
