"""The FMA-corrected quotient (jb_common.cuh div_cr) that replaces the
reference's divisions on the hot path -- yy / (d*d) and 2y / d of the
compression test (compression.hpp:52, k_spec) and y = inc / sigma_inc of
scale_pieces (digitization.hpp:50, PtsView / k_assign_stats) -- equals the
IEEE quotient: checked in C (gcc, libm fma, no contraction) on random
numerators over the guarded range, near-multiples of b, and integers, for
every d <= 256 with b = d and b = d^2, and for random divisors in
[2^-50, 2^50] (including all-ones significands)."""
import os
import shutil
import subprocess
import tempfile

import pytest

SRC = r"""
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ull;
static uint64_t xr(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double div_cr(double a, double b, double ry) {
    double q0 = a * ry;
    double q1 = fma(fma(-q0, b, a), ry, q0);
    return fma(fma(-q1, b, a), ry, q1);
}
int main(int argc, char** argv) {
    long per = argc > 1 ? atol(argv[1]) : 20000, bad = 0, n = 0;
    for (int d = 1; d <= 256; ++d)
        for (int sq = 0; sq < 2; ++sq) {
            const double b = sq ? (double)d * (double)d : (double)d, ry = 1.0 / b;
            for (long k = 0; k < per; ++k) {
                const int e = (int)(xr() % 1900) - 900;
                double a = ldexp(1.0 + (double)(xr() >> 11) * 0x1p-53, e);
                if (xr() & 1) a = -a;
                if (k % 4 == 1) {  /* (near-)multiples of b: ties and exact quotients */
                    a = ldexp((double)(xr() % 100000), e % 60) * b;
                    if (k & 8) a = nextafter(a, 0.0);
                }
                if (k % 4 == 2) a = ldexp((double)(xr() >> 11), (int)(xr() % 40) - 60);
                const double want = a / b, got = div_cr(a, b, ry);
                ++n;
                if (memcmp(&want, &got, 8)) ++bad;
            }
        }
    for (long t = 0; t < per / 10; ++t) {  /* general divisors (sigma_inc) */
        double b = ldexp(1.0 + (double)(xr() >> 11) * 0x1p-53, (int)(xr() % 100) - 50);
        if (t % 7 == 0) b = nextafter(ldexp(1.0, (int)(xr() % 40) - 20), 0.0);
        const double ry = 1.0 / b;
        for (int k = 0; k < 1000; ++k) {
            const int e = (int)(xr() % 1800) - 900;
            double a = ldexp(1.0 + (double)(xr() >> 11) * 0x1p-53, e);
            if (xr() & 1) a = -a;
            if (k % 3 == 1) {
                a = ldexp(1.0 + (double)(xr() >> 11) * 0x1p-53, e % 100) * b;
                if (k & 4) a = nextafter(a, 0.0);
            }
            const double want = a / b, got = div_cr(a, b, ry);
            ++n;
            if (memcmp(&want, &got, 8)) ++bad;
        }
    }
    printf("%ld %ld\n", n, bad);
    return 0;
}
"""


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_fma_quotient_equals_ieee_division():
    with tempfile.TemporaryDirectory() as t:
        c, exe = os.path.join(t, "d.c"), os.path.join(t, "d")
        with open(c, "w") as f:
            f.write(SRC.replace("#include <string.h>", "#include <string.h>\n#include <stdlib.h>"))
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, c, "-lm"], check=True)
        out = subprocess.run([exe, "40000"], capture_output=True, text=True, check=True).stdout
        n, bad = map(int, out.split())
        assert n == 256 * 2 * 40000 + 4000 * 1000
        assert bad == 0
