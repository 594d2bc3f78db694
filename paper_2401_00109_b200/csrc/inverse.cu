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
                                                   unsigned long long* __restrict__ err) {
    // The carry warp also validates every label (inverse_digitize_series
    // :41-44) and sums the quantized lengths of each group of GROUP pieces;
    // both are off its fp64 critical path.
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
    const int64_t s = blockIdx.x * (int64_t)32 + (threadIdx.x & 31);
    if (s >= in.n_seg) return;
    unsigned char* my = ring + threadIdx.x * RSTRIDE;
    const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
    const double* tl = cwarp ? tabs : tabs + kk;
    double carry = 0.0, v = in.anchors[s];
    bool badlab = false;
    int64_t g = grp_off[s];
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
                             double* __restrict__ out, unsigned long long* __restrict__ err) {
    const int lane = threadIdx.x & 31;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < in.n_seg;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = in.seg_offsets[s], b = in.seg_offsets[s + 1];
        const int64_t g0 = grp_off[s], g1 = grp_off[s + 1];
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
// One block = 32 segments. Warp 0 runs, one lane per segment, both
// sequential chains in the reference's rounding -- the length carry
// (quantize_lengths :63-74) and the start values (inverse_compress :94-101),
// independent of each other so they overlap -- into rings of per-piece
// quantized lengths and start values, plus each tile's first output
// position. The writer warps trail it by FD tiles and emit every sample at
// its final position: a half-warp per (segment, tile), lane m holding piece
// m, samples assigned to lanes 16 at a time (coalesced stores), the piece of
// a sample found by a 4-step search over the tile's exclusive length scan.
// When a segment's last tile is done, warp 0 applies match_total_length's
// backward cascade (:81-93) to the pieces still in the ring -- the cascade
// only moves the tail, so every piece already written sits at its final
// position -- and recomputes the window's tile positions. A cascade that
// reaches past the window sends the call to the general path (err[1]).
constexpr int FD = 4;                    // tiles between warp 0 and the writers (cascade window)
constexpr int FRD = 6;                   // label tiles in flight
constexpr int FS = FRD + FD;             // label ring tiles
constexpr int FLSTR = FS * RT * 4 + 16;  // label ring bytes per lane
constexpr int FQ = (FD + 1) * RT;        // ring entries per lane
constexpr int FWW = 7;                   // writer warps
constexpr int FUSED_TB = 32 * (1 + FWW);
constexpr long long kTileSamplesMax = 1LL << 30;  // larger tiles: general path
constexpr int kLanePiece = 8;  // pieces up to this length: lane per piece; longer: warp per piece

struct FusedSmem {
    double div[(DIV_MAX + 1) * (DIV_MAX + 1)];
    double vs[32 * FQ];       // start value of each piece
    int32_t q[32 * FQ];       // quantized length of each piece (0: outside the segment)
    int32_t ex[32 * FQ];      // its first sample's offset from the tile's first sample
    long long pos[FD + 1][32];// output position of each tile's first sample
    long long E[32];          // last output position of each segment
    int ntile[32];
    int bail[32];
    unsigned char lab[32 * FLSTR];
};

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

template <bool SMEM_TABS>
__global__ void __launch_bounds__(FUSED_TB) k_inv_fused(InverseIn in, const double* __restrict__ rlen,
                                                        const double* __restrict__ rinc,
                                                        double* __restrict__ out,
                                                        unsigned long long* __restrict__ err) {
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
    for (int t = threadIdx.x; t < (DIV_MAX + 1) * (DIV_MAX + 1); t += blockDim.x) {
        const int l = t / (DIV_MAX + 1), i = t % (DIV_MAX + 1);
        S.div[t] = l > 0 ? (double)i / (double)l : 0.0;  // the same IEEE division
    }
    const double* tlen = SMEM_TABS ? s_tabs : rlen;
    const double* tinc = SMEM_TABS ? s_tabs + kk : rinc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;

    // warp 0: lane = segment
    const int64_t s = blockIdx.x * (int64_t)32 + lane;
    int64_t a = 0, b = 0, base = 0;
    int ntile = 0;
    double carry = 0.0, v = 0.0;
    long long total = 0, pos = 0;
    bool badlab = false;
    unsigned char* lrow = S.lab + lane * FLSTR;
    int32_t* qrow = S.q + lane * FQ;
    int32_t* xrow = S.ex + lane * FQ;
    double* vrow = S.vs + lane * FQ;
    if (warp == 0) {
        const bool live = s < in.n_seg;
        long long E = -1;
        if (live) {
            a = in.seg_offsets[s];
            b = in.seg_offsets[s + 1];
            const long long o = in.out_offsets[s];
            const bool drop = in.layout == 0 && (s + 1 < in.n_seg || in.drop_local_last);
            E = o + in.source_lengths[s] - (drop ? 1 : 0);
            v = in.anchors[s];
            if (E >= o) out[o] = v;
            pos = o + 1;
        }
        base = a & ~(int64_t)3;  // 16-byte aligned label tiles
        ntile = b > a ? (int)((b - base + RT - 1) / RT) : 0;
        S.E[lane] = E;
        S.ntile[lane] = ntile;
        S.bail[lane] = 0;
        for (int t = 0; t < FRD - 1; ++t) {
            if (t < ntile) ring_issue_z(lrow, in.labels, base + (int64_t)t * RT, in.N, t % FS);
            ring_commit();
        }
    }
    __syncthreads();
    int maxT = 0;
    for (int l = 0; l < 32; ++l) maxT = max(maxT, S.ntile[l]);
    auto lab_ok = [&](uint32_t lab) -> uint32_t {
        const bool bad = lab >= (uint32_t)kk;
        badlab |= bad;
        return bad ? 0u : lab;
    };

    for (int it = 0; it < maxT + FD; ++it) {
        if (warp == 0) {
            if (it < ntile) {
                const int tn = it + FRD - 1;
                if (tn < ntile) ring_issue_z(lrow, in.labels, base + (int64_t)tn * RT, in.N, tn % FS);
                ring_commit();
                ring_wait<FRD - 1>();  // tile it has landed
                const uint32_t* lt = reinterpret_cast<const uint32_t*>(lrow + (it % FS) * RT * 4);
                const int slot = it % (FD + 1);
                int32_t* qt = qrow + slot * RT;
                int32_t* xt = xrow + slot * RT;
                double* vt = vrow + slot * RT;
                const int64_t jt = base + (int64_t)it * RT;
                S.pos[slot][lane] = pos;
                long long tsum = 0;
                if (jt >= a && jt + RT <= b) {
#pragma unroll
                    for (int m = 0; m < RT / 4; ++m) {
                        const uint4 L = reinterpret_cast<const uint4*>(lt)[m];
                        const uint32_t l0 = lab_ok(L.x), l1 = lab_ok(L.y), l2 = lab_ok(L.z),
                                       l3 = lab_ok(L.w);
                        int4 Q;
                        chain_step(tlen[l0], carry, Q.x);
                        chain_step(tlen[l1], carry, Q.y);
                        chain_step(tlen[l2], carry, Q.z);
                        chain_step(tlen[l3], carry, Q.w);
                        reinterpret_cast<int4*>(qt)[m] = Q;
                        int4 X;
                        X.x = (int)tsum;
                        X.y = X.x + Q.x;
                        X.z = X.y + Q.y;
                        X.w = X.z + Q.z;
                        reinterpret_cast<int4*>(xt)[m] = X;
                        tsum += (long long)Q.x + Q.y + Q.z + Q.w;
                        const double v0 = v, v1 = v0 + tinc[l0], v2 = v1 + tinc[l1],
                                     v3 = v2 + tinc[l2];
                        v = v3 + tinc[l3];
                        reinterpret_cast<double2*>(vt)[2 * m] = make_double2(v0, v1);
                        reinterpret_cast<double2*>(vt)[2 * m + 1] = make_double2(v2, v3);
                    }
                } else {
                    for (int m = 0; m < RT; ++m) {
                        const int64_t j = jt + m;
                        int32_t q = 0;
                        vt[m] = v;
                        if (j >= a && j < b) {
                            const uint32_t l = lab_ok(lt[m]);
                            chain_step(tlen[l], carry, q);
                            v += tinc[l];
                        }
                        qt[m] = q;
                        xt[m] = (int)tsum;
                        tsum += q;
                    }
                }
                total += tsum;
                pos += tsum;
                if (tsum > kTileSamplesMax && !S.bail[lane]) {  // the writers count in int
                    S.bail[lane] = 1;
                    atomicAdd(err + 1, 1ULL);
                }
                if (it == ntile - 1) {  // match_total_length on the window
                    long long residual = in.source_lengths[s] - total;
                    const int t0 = ntile - FD > 0 ? ntile - FD : 0;
                    const int64_t jlo = max(a, base + (int64_t)t0 * RT);
                    for (int64_t j = b - 1; j >= jlo && residual != 0; --j) {
                        const int64_t r = j - base;
                        int32_t* qp = qrow + (int)((r / RT) % (FD + 1)) * RT + (int)(r % RT);
                        long long adj = (long long)*qp + residual;
                        if (adj < 1) adj = 1;
                        residual -= adj - *qp;
                        *qp = (int32_t)adj;
                    }
                    if (residual != 0) {
                        if (jlo == a) {
                            atomicMin(err, (unsigned long long)(s * 4 + kErrPiece));
                        } else {
                            S.bail[lane] = 1;
                            atomicAdd(err + 1, 1ULL);
                        }
                    }
                    // the window's tile positions after the cascade
                    long long pp = S.pos[t0 % (FD + 1)][lane];
                    for (int t = t0; t < ntile; ++t) {
                        S.pos[t % (FD + 1)][lane] = pp;
                        const int32_t* qq = qrow + (t % (FD + 1)) * RT;
                        int32_t* xx = xrow + (t % (FD + 1)) * RT;
                        long long ts = 0;
                        for (int m = 0; m < RT; ++m) {
                            xx[m] = (int)ts;
                            ts += qq[m];
                        }
                        pp += ts;
                        if (ts > kTileSamplesMax && !S.bail[lane]) {
                            S.bail[lane] = 1;
                            atomicAdd(err + 1, 1ULL);
                        }
                    }
                }
            }
        } else {
            const int t = it - FD;
            if (t >= 0) {
                const int h = lane >> 4, m = lane & 15;
                const int slot = t % (FD + 1);
                for (int L0 = 2 * (warp - 1); L0 < 32; L0 += 2 * FWW) {
                    // lane per piece: a half-warp per segment
                    const int L = L0 + h;
                    const bool act = t < S.ntile[L] && !S.bail[L];
                    const int r = L * FQ + slot * RT + m;
                    const int q = act ? S.q[r] : 0;
                    double vv = 0.0, inc = 0.0;
                    long long P0 = 0, E = -1;
                    if (q > 0) {
                        vv = S.vs[r];
                        const uint32_t lab = reinterpret_cast<const uint32_t*>(
                            S.lab + L * FLSTR + (t % FS) * RT * 4)[m];
                        inc = tinc[lab < (uint32_t)kk ? lab : 0u];
                        P0 = S.pos[slot][L] + S.ex[r];
                        E = S.E[L];
                    }
                    const int qmax = __reduce_max_sync(FULL, q);
                    const int lim = min(qmax, kLanePiece);
                    for (int i = 1; i <= lim; ++i) {
                        const long long P = P0 + i - 1;
                        if (i <= q && P <= E) {
                            const double fr = q <= DIV_MAX ? S.div[q * (DIV_MAX + 1) + i]
                                                           : (double)i / (double)q;
                            out[P] = vv + inc * fr;
                        }
                    }
                    if (qmax > kLanePiece) {  // long pieces: the warp writes 32 samples at a time
                        unsigned lm = __ballot_sync(FULL, q > kLanePiece);
                        while (lm) {
                            const int src = __ffs(lm) - 1;
                            lm &= lm - 1;
                            const int qs = __shfl_sync(FULL, q, src);
                            const long long ps = __shfl_sync(FULL, P0, src);
                            const long long es = __shfl_sync(FULL, E, src);
                            const double vs = __shfl_sync(FULL, vv, src);
                            const double is = __shfl_sync(FULL, inc, src);
                            for (int i = kLanePiece + 1 + lane; i <= qs; i += 32) {
                                const long long P = ps + i - 1;
                                if (P <= es) {
                                    const double fr = qs <= DIV_MAX
                                                          ? S.div[qs * (DIV_MAX + 1) + i]
                                                          : (double)i / (double)qs;
                                    out[P] = vs + is * fr;
                                }
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    if (warp == 0) {
        if (s < in.n_seg && b == a) atomicMin(err, (unsigned long long)(s * 4 + kErrPiece));
        if (badlab) atomicMin(err, (unsigned long long)(s * 4 + kErrLabel));
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
                            DArr<unsigned long long>& err, double* d_out, cudaStream_t st) {
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
        kern<<<(int)((in.n_seg + 31) / 32), 64, tsmem, st>>>(in, tabp, tabp + kk, qlen.p,
                                                              vstart.p, goff.p, gsum.p, err.p);
        JB_LAUNCH_CHECK();
        k_inv_segfix<<<(int)std::max<int64_t>(1, std::min<int64_t>((in.n_seg * 32 + 255) / 256,
                                                                   (int64_t)kSMs * 16)),
                       256, 0, st>>>(in, qlen.p, goff.p, gsum.p, rec.p, gmeta.p, d_out, err.p);
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
            1, std::min<int64_t>((n_groups * 32 + FILL_TB - 1) / FILL_TB, (int64_t)kSMs * 16));
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
    {
        JB_PROF("inverse_fused", st);
        const size_t tsmem = sizeof(double) * 2 * kk <= kInvTabSmem ? sizeof(double) * 2 * kk : 0;
        const size_t smem = tsmem + sizeof(FusedSmem) + 128;
        auto kern = tsmem ? k_inv_fused<true> : k_inv_fused<false>;
        JB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(int)((in.n_seg + 31) / 32), FUSED_TB, smem, st>>>(in, tab.p, tab.p + kk, d_out, err.p);
        JB_LAUNCH_CHECK();
        err.download(h, 2);
        JB_CUDA(cudaStreamSynchronize(st));
    }
    if (h[1] != 0) {  // a cascade outside the window: redo everything on the general path
        err.upload(init, 2);
        inverse_general(in, tab.p, kk, err, d_out, st);
        return;
    }
    throw_inverse_error(h[0], in.k);
}

}  // namespace jb
