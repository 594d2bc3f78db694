/*
 * mt64_jump.c — build-time generator of std::mt19937_64 jump polynomials.
 *
 * The device engine (kmeans.cu) lets CTA c produce engine draws
 * [c*B, (c+1)*B) of the reference's stream (clustering.hpp:74-85, 103-104:
 * one std::mt19937_64 per fit). CTA c needs the state window at time c*B,
 * i.e. A^(c*B) applied to the seeded window, which equals g_c(A) applied to
 * it, with g_c(t) = t^(c*B) mod phi(t) and phi the degree-19937
 * characteristic polynomial of the generator (up to the 31 unused low bits of
 * the window's first word, which the next twist never reads).
 *
 * phi is recovered with Berlekamp-Massey from bit 0 of the output stream;
 * g_c = g_{c-1} * (t^B mod phi) mod phi. The table depends only on B, not on
 * the seed. Output: <out> = header {magic, B, count, words} + count polynomials
 * of 312 little-endian 64-bit words (bit i = coefficient of t^i).
 *
 * usage: mt64_jump <out> [log2_B=22] [count=1024]
 * (the chain g_c is split into per-thread stretches with OpenMP)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NW 312      /* 64-bit words per polynomial (19968 bits) */
#define DEG 19937

typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

static int getb(const uint64_t* p, int i) { return (int)((p[i >> 6] >> (i & 63)) & 1ULL); }
static void flipb(uint64_t* p, int i) { p[i >> 6] ^= 1ULL << (i & 63); }

/* Berlekamp-Massey over GF(2); returns the connection polynomial C (C[0]=1)
 * as coefficients c_0..c_L; the characteristic polynomial is its reversal. */
static int berlekamp_massey(const uint8_t* s, int n, uint8_t* C) {
    uint8_t* B = calloc(n + 1, 1);
    uint8_t* T = calloc(n + 1, 1);
    memset(C, 0, n + 1);
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int i = 0; i < n; ++i) {
        int d = s[i];
        for (int j = 1; j <= L; ++j) d ^= C[j] & s[i - j];
        if (!d) {
            ++m;
        } else if (2 * L <= i) {
            memcpy(T, C, n + 1);
            for (int j = 0; j + m <= n; ++j) C[j + m] ^= B[j];
            L = i + 1 - L;
            memcpy(B, T, n + 1);
            m = 1;
        } else {
            for (int j = 0; j + m <= n; ++j) C[j + m] ^= B[j];
            ++m;
        }
    }
    free(B);
    free(T);
    return L;
}

static uint64_t phi[NW];  /* characteristic polynomial, degree DEG */

/* a <- a * t mod phi */
static void mul_t(uint64_t* a) {
    const int top = getb(a, DEG - 1);
    for (int w = NW - 1; w > 0; --w) a[w] = (a[w] << 1) | (a[w - 1] >> 63);
    a[0] <<= 1;
    if (top) for (int w = 0; w < NW; ++w) a[w] ^= phi[w];
    /* clear bits >= DEG */
    a[DEG >> 6] &= (1ULL << (DEG & 63)) - 1ULL;
    for (int w = (DEG >> 6) + 1; w < NW; ++w) a[w] = 0;
}

/* r <- a * b mod phi */
static void mulmod(const uint64_t* a, const uint64_t* b, uint64_t* r) {
    uint64_t acc[NW], sh[NW];
    memset(acc, 0, sizeof acc);
    memcpy(sh, a, sizeof sh);
    for (int i = 0; i < DEG; ++i) {
        if (getb(b, i))
            for (int w = 0; w < NW; ++w) acc[w] ^= sh[w];
        mul_t(sh);
    }
    memcpy(r, acc, sizeof acc);
}

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: %s <out> [log2_B] [count]\n", argv[0]);
        return 2;
    }
    const int logB = argc > 2 ? atoi(argv[2]) : 22;
    const int count = argc > 3 ? atoi(argv[3]) : 1024;
    /* bit-0 sequence of the outputs */
    const int n = 2 * DEG + 64;
    uint8_t* s = malloc(n);
    mt64 g;
    mt_seed(&g, 5489ULL);
    for (int i = 0; i < n; ++i) s[i] = (uint8_t)(mt_next(&g) & 1ULL);
    uint8_t* C = malloc(n + 1);
    const int L = berlekamp_massey(s, n, C);
    if (L != DEG) {
        fprintf(stderr, "unexpected linear complexity %d\n", L);
        return 1;
    }
    /* characteristic polynomial: phi(t) = t^L * C(1/t) -> coefficient of t^i is C[L-i] */
    memset(phi, 0, sizeof phi);
    for (int i = 0; i <= L; ++i)
        if (C[L - i] && i < DEG) flipb(phi, i); /* t^DEG is implicit (reduction) */
    /* P = t^B mod phi by repeated squaring of t (squaring = mulmod) */
    uint64_t P[NW], cur[NW], nxt[NW];
    memset(P, 0, sizeof P);
    flipb(P, 1); /* t */
    for (int i = 0; i < logB; ++i) {
        mulmod(P, P, nxt);
        memcpy(P, nxt, sizeof P);
    }
    uint64_t* out = calloc((size_t)count * NW, 8);
    /* per-thread stretches: start = P^c0 by binary powering, then chain */
#pragma omp parallel
    {
#ifdef _OPENMP
        extern int omp_get_thread_num(void);
        extern int omp_get_num_threads(void);
        const int tid = omp_get_thread_num(), nt = omp_get_num_threads();
#else
        const int tid = 0, nt = 1;
#endif
        const int per = (count + nt - 1) / nt;
        const int c0 = tid * per, c1 = c0 + per < count ? c0 + per : count;
        if (c0 < c1) {
            uint64_t acc[NW], base[NW], t[NW];
            memset(acc, 0, sizeof acc);
            flipb(acc, 0);
            memcpy(base, P, sizeof base);
            for (int e = c0; e; e >>= 1) {
                if (e & 1) {
                    mulmod(acc, base, t);
                    memcpy(acc, t, sizeof acc);
                }
                if (e >> 1) {
                    mulmod(base, base, t);
                    memcpy(base, t, sizeof base);
                }
            }
            for (int c = c0; c < c1; ++c) {
                memcpy(out + (size_t)c * NW, acc, sizeof acc);
                if (c + 1 < c1) {
                    mulmod(acc, P, t);
                    memcpy(acc, t, sizeof acc);
                }
            }
        }
    }
    (void)cur;
    (void)nxt;
    FILE* f = fopen(argv[1], "wb");
    if (!f) return 1;
    const uint64_t hdr[4] = {0x4A4D54364A4D5031ULL, 1ULL << logB, (uint64_t)count, NW};
    fwrite(hdr, 8, 4, f);
    fwrite(out, 8, (size_t)count * NW, f);
    fclose(f);
    free(out);
    free(s);
    free(C);
    return 0;
}
