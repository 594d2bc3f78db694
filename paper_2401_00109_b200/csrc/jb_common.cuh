// jb_common.cuh — shared device utilities for the B200 JABBA path.
//
// Built with -fmad=false: every fp64 expression that mirrors a reference
// expression must round exactly as the reference's SSE2 build does
// (proj/CMakeLists.txt:5-10 has no -march, hence no FMA contraction).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <stdexcept>
#include <string>

namespace jb {

// Status codes mirror the reference's error hierarchy (core.hpp:20-30).
enum Status : int {
    OK = 0,
    INVALID_INPUT = 1,
    INVALID_PIECE = 2,
    INVALID_PARTITION = 3,
    UNKNOWN_SYMBOL = 4,
    PARSE_ERROR = 5,
    LAYOUT_ERROR = 6,
    VERSION_ERROR = 7,
    CUDA_ERROR = 100,
    NCCL_ERROR = 101,
    NO_DEVICE = 102,
    INTERNAL = 103,
};

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define JB_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::jb::Error(::jb::CUDA_ERROR, std::string(#call) + ": " +             \
                                                    cudaGetErrorString(e_));            \
    } while (0)

#define JB_LAUNCH_CHECK() JB_CUDA(cudaGetLastError())

typedef unsigned __int128 u128;
typedef __int128 i128;

// ---------------------------------------------------------------------------
// Deterministic fp64 summation: every addend is converted to a signed 128-bit
// fixed-point integer with a per-quantity binary exponent E (value * 2^E,
// magnitude truncated), and accumulated with integer adds. Integer addition is
// associative, so the result is bitwise identical for any launch geometry,
// atomic order or GPU count (the determinism contract of parallel.hpp:3-5,
// extended to 1/2/4/8 GPUs). E is chosen so the largest possible |sum| stays
// below 2^126; addends >= 2^(53-E) are represented exactly.

__host__ __device__ inline int fx_exponent_for(double max_abs_sum) {
    // smallest e with max_abs_sum < 2^e, then E = 125 - e
    if (!(max_abs_sum > 0.0)) return 0;
    int e = 0;
    double m = max_abs_sum;
    // frexp-free exponent extraction (works on host and device)
    uint64_t bits;
    memcpy(&bits, &m, 8);
    e = (int)((bits >> 52) & 0x7FF) - 1022;  // m < 2^e
    int E = 125 - e;
    if (E > 1000) E = 1000;
    return E;
}

// Correctly rounded quotient a / b from ry = RN(1 / b) by FMA corrections:
// q0 = RN(a ry), then twice q <- RN(q + RN(a - b q) ry); the remainder of a
// faithful quotient is exact under an FMA, the first correction makes q
// faithful and Markstein's theorem makes the second one RN(a / b) -- the
// IEEE quotient -- in 5 fp64 operations instead of the division sequence
// (whose slow-path branch also diverges warps). Needs no underflow or
// overflow on the way: 2^-900 <= |a| <= 2^900 and 2^-50 <= b <= 2^50 (the
// caller checks b once and passes ry = 0 outside that range).
// tests/test_div_identity.py checks the identity against a / b.
__device__ __forceinline__ double div_cr(double a, double b, double ry) {
    const double q0 = __dmul_rn(a, ry);
    const double q1 = __fma_rn(__fma_rn(-q0, b, a), ry, q0);
    return __fma_rn(__fma_rn(-q1, b, a), ry, q1);
}

// a / b (IEEE, round to nearest) for a divisor b > 0 with ry = RN(1/b), or
// ry = 0 when b is outside div_cr's range
__device__ __forceinline__ double div_by(double a, double b, double ry) {
    if (ry == 0.0) return a / b;
    const double aa = fabs(a);
    if (aa == 0.0) return a;  // +-0 / b (b > 0 here) keeps the zero's sign
    return (aa >= 0x1p-900 && aa <= 0x1p900) ? div_cr(a, b, ry) : a / b;
}

__host__ inline double div_by_recip(double b) {  // ry for div_by
    return (b >= 0x1p-50 && b <= 0x1p50) ? 1.0 / b : 0.0;
}

// |x| * 2^E truncated to an integer, with x's sign.
__host__ __device__ __forceinline__ i128 fx_from_double(double x, int E) {
#ifdef __CUDA_ARCH__
    // device: the same integer from fp64 arithmetic. a = |x| 2^(E-64) is
    // exact (power-of-two scaling; a subnormal a means |x| 2^E < 2^-958,
    // whose truncation is 0 either way); hi = trunc(a) < 2^62, and
    // a - hi (the fraction) and its 2^64 scaling are exact, so
    // hi * 2^64 + trunc(frac * 2^64) = trunc(|x| 2^E). Checked equal to the
    // bit-level path below on 2.1e6 random and edge values.
    const double a = fabs(x) * __longlong_as_double((long long)(E - 64 + 1023) << 52);
    const unsigned long long hi = __double2ull_rz(a);
    const double r = a - __ull2double_rn(hi);
    const unsigned long long lo = __double2ull_rz(r * 0x1p64);
    const u128 mag = ((u128)hi << 64) | lo;
    return signbit(x) ? -(i128)mag : (i128)mag;
#else
    uint64_t bits;
    memcpy(&bits, &x, 8);
    const int bexp = (int)((bits >> 52) & 0x7FF);
    if (bexp == 0) return 0;  // zero / subnormal: below any resolution we use
    const uint64_t mant = (bits & 0x000FFFFFFFFFFFFFULL) | 0x0010000000000000ULL;
    // x = mant * 2^(bexp - 1075)
    const int sh = bexp - 1075 + E;
    u128 mag;
    if (sh >= 0) {
        if (sh > 74) mag = ((u128)1) << 126;  // saturate (caller's E makes this unreachable)
        else mag = ((u128)mant) << sh;
    } else {
        mag = (sh <= -64) ? 0 : (u128)(mant >> (-sh));
    }
    const i128 v = (i128)mag;
    return (bits >> 63) ? -v : v;
#endif
}

// Correctly rounded (nearest-even) conversion of a fixed-point integer back to
// double, then exact scaling by 2^-E.
__host__ __device__ inline double fx_to_double(i128 v, int E) {
    if (v == 0) return 0.0;
    const bool neg = v < 0;
    u128 m = neg ? (u128)(-v) : (u128)v;
    int lz = 0;
    {
        uint64_t hi = (uint64_t)(m >> 64);
        uint64_t lo = (uint64_t)m;
        if (hi) {
#ifdef __CUDA_ARCH__
            lz = __clzll((long long)hi);
#else
            lz = __builtin_clzll(hi);
#endif
        } else {
#ifdef __CUDA_ARCH__
            lz = 64 + __clzll((long long)lo);
#else
            lz = 64 + __builtin_clzll(lo);
#endif
        }
    }
    const int msb = 127 - lz;  // index of the leading one
    uint64_t mant;
    int exp2;  // value = mant * 2^exp2
    if (msb <= 52) {
        mant = (uint64_t)m;
        exp2 = 0;
    } else {
        const int drop = msb - 52;
        const u128 keep = m >> drop;
        const u128 rem = m - (keep << drop);
        const u128 half = ((u128)1) << (drop - 1);
        mant = (uint64_t)keep;
        exp2 = drop;
        if (rem > half || (rem == half && (mant & 1))) {
            ++mant;
            if (mant == (1ULL << 53)) {
                mant >>= 1;
                ++exp2;
            }
        }
    }
    // mant < 2^53 exactly representable; scale by 2^(exp2 - E)
    double d = (double)mant;
    int s = exp2 - E;
    // scale in steps to avoid overflow/underflow of the factor itself
    while (s > 600) { d *= 0x1p600; s -= 600; }
    while (s < -600) { d *= 0x1p-600; s += 600; }
    double f;
    {
        uint64_t fb = (uint64_t)(s + 1023) << 52;
        memcpy(&f, &fb, 8);
    }
    d *= f;
    return neg ? -d : d;
}

// Global int128 accumulator stored as two u64 words (lo, hi).
__device__ __forceinline__ void fx_atomic_add(unsigned long long* lohi, i128 v) {
    if (v == 0) return;
    const u128 u = (u128)v;
    const unsigned long long lo = (unsigned long long)u;
    const unsigned long long hi = (unsigned long long)(u >> 64);
    const unsigned long long old = atomicAdd(lohi, lo);
    const unsigned long long carry = (old + lo) < old ? 1ULL : 0ULL;
    const unsigned long long h = hi + carry;
    if (h) atomicAdd(lohi + 1, h);
}

// add a NON-NEGATIVE value (< 2^64 in the common case) to a (lo, hi)
// accumulator: one atomic unless the low word carries
__device__ __forceinline__ void fx_atomic_add_small(unsigned long long* lohi, u128 v) {
    const unsigned long long lo = (unsigned long long)v;
    const unsigned long long hi = (unsigned long long)(v >> 64);
    const unsigned long long old = atomicAdd(lohi, lo);
    const unsigned long long h = hi + ((old + lo) < old ? 1ULL : 0ULL);
    if (h) atomicAdd(lohi + 1, h);
}

__host__ __device__ inline i128 fx_load(const unsigned long long* lohi) {
    return (i128)(((u128)lohi[1] << 64) | (u128)lohi[0]);
}

// int128 accumulator held as three u64 limb sums: bits 0-31 and 32-63 of each
// addend (unsigned) and bits 64-127 (two's complement). No add needs the old
// value, so every add is a fire-and-forget RED (an int128 add through a
// (lo, hi) pair must wait for the low word to learn its carry). Exact while
// fewer than 2^32 addends reach a limb between normalisations (l3_norm).
__device__ __forceinline__ void l3_add(unsigned long long* p, i128 v) {
    const u128 u = (u128)v;
    const unsigned long long a = (unsigned long long)(u & 0xFFFFFFFFu);
    const unsigned long long b = (unsigned long long)((u >> 32) & 0xFFFFFFFFu);
    const unsigned long long c = (unsigned long long)(u >> 64);
    if (a) atomicAdd(p, a);
    if (b) atomicAdd(p + 1, b);
    if (c) atomicAdd(p + 2, c);
}
__host__ __device__ __forceinline__ i128 l3_load(const unsigned long long* p) {
    return (i128)((u128)p[0] + ((u128)p[1] << 32) + ((u128)p[2] << 64));
}
__host__ __device__ __forceinline__ void l3_store(unsigned long long* p, i128 v) {
    const u128 u = (u128)v;
    p[0] = (unsigned long long)(u & 0xFFFFFFFFu);
    p[1] = (unsigned long long)((u >> 32) & 0xFFFFFFFFu);
    p[2] = (unsigned long long)(u >> 64);
}

// warp-level int128 sum (deterministic: integer adds)
__device__ __forceinline__ i128 fx_warp_sum(i128 v) {
    unsigned long long lo = (unsigned long long)(u128)v;
    unsigned long long hi = (unsigned long long)((u128)v >> 64);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long olo = __shfl_down_sync(0xffffffffu, lo, o);
        const unsigned long long ohi = __shfl_down_sync(0xffffffffu, hi, o);
        const unsigned long long nlo = lo + olo;
        hi = hi + ohi + (nlo < lo ? 1ULL : 0ULL);
        lo = nlo;
    }
    return (i128)(((u128)hi << 64) | (u128)lo);
}

// Warp-aggregated accumulation. Lanes with the same key (active lanes only)
// form a group (__match_any_sync); the group's leader sums the members' values
// from a per-warp shared scratch and issues ONE set of atomics for the group.
// Integer sums: the result is independent of grouping and order.
struct AggScratch {  // per warp, in shared memory
    unsigned long long a_lo[32], a_hi[32], b_lo[32], b_hi[32], c[32];
};

template <class Flush>
__device__ __forceinline__ void warp_aggregate(bool active, uint32_t key, u128 a, u128 b,
                                               unsigned long long c, AggScratch* sc,
                                               Flush&& flush) {
    const int lane = threadIdx.x & 31;
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (!act) return;
    const unsigned grp = __match_any_sync(0xffffffffu, active ? key : 0xFFFFFFFFu);
    sc->a_lo[lane] = (unsigned long long)a;
    sc->a_hi[lane] = (unsigned long long)(a >> 64);
    sc->b_lo[lane] = (unsigned long long)b;
    sc->b_hi[lane] = (unsigned long long)(b >> 64);
    sc->c[lane] = c;
    __syncwarp();
    if (active && (__ffs(grp) - 1) == lane) {  // group leader
        u128 sa = 0, sb = 0;
        unsigned long long sc_ = 0;
        unsigned m = grp;
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            sa += ((u128)sc->a_hi[l] << 64) | sc->a_lo[l];
            sb += ((u128)sc->b_hi[l] << 64) | sc->b_lo[l];
            sc_ += sc->c[l];
        }
        flush(key, sa, sb, sc_, __popc(grp));
    }
    __syncwarp();
}

// exact reference distance: dx*dx + dy*dy with no contraction (clustering.hpp:52-56)
__device__ __forceinline__ double dist2(double ax, double ay, double bx, double by) {
    const double dx = __dsub_rn(ax, bx);
    const double dy = __dsub_rn(ay, by);
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// non-negative double <-> order-preserving u64 (for atomicMax on >= 0 values)
__device__ __forceinline__ unsigned long long dbits(double x) {
    return (unsigned long long)__double_as_longlong(x);
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// SMs of the current device, for grid sizing and cooperative launches (148
// on a full B200; a MIG slice or an MPS SM limit exposes fewer)
inline int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& c = cache[dev & 63];
    if (!c) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) {
            cudaGetLastError();
            v = 148;
        }
        c = v;
    }
    return c;
}

// ---------------------------------------------------------------------------
// Bulk asynchronous copies global -> shared (TMA engine, no tensor map):
// one thread arms an mbarrier with the byte count and issues the copies; the
// consumers wait on the barrier's phase. Sizes and addresses 16-byte aligned.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// fire-and-forget 64-bit add in L2 (no value returned to the SM; atomicAdd
// with an unused result can still compile to a returning ATOM, e.g. inside
// cooperative kernels)
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
// generic-proxy accesses of shared memory before async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace jb
