"""The inverse carry chain's rounding shortcut (inverse.cu chain_step):
max(1, llround(x)) == (x < 0.5 ? 1 : floor(fl(x + 0.5))) for every double
x < 2^52 (quantize_lengths, inverse.hpp:68-70). Checked on binade edges,
half-integer neighbourhoods and random values (float64 arithmetic)."""
import math

import numpy as np


def llround_clamped(x: float) -> float:
    f = math.floor(x)
    r = f + 1 if x - f >= 0.5 else f  # x - floor(x) is exact; ties away (x >= 0 here)
    if x < 0:
        t = math.trunc(x)
        r = t - 1 if t - x >= 0.5 else t
    return float(max(1, r))


def shortcut(x: float) -> float:
    if x < 0.5:
        return 1.0
    if x >= 2.0 ** 52:
        return x
    return float(math.floor(np.float64(x) + np.float64(0.5)))


def cases():
    xs = []
    for k in range(0, 70):
        for base in (k + 0.5, float(k), 2.0 ** min(k, 60)):
            x = np.float64(base)
            for _ in range(4):
                xs.append(float(x))
                x = np.nextafter(x, np.inf)
            x = np.float64(base)
            for _ in range(4):
                x = np.nextafter(x, -np.inf)
                xs.append(float(x))
    rng = np.random.default_rng(0)
    xs += list(rng.uniform(-3, 40, 20000))
    xs += list(np.ldexp(rng.uniform(0.5, 1, 5000), rng.integers(-60, 53, 5000)))
    return xs


def test_round_shortcut_matches_llround():
    for x in cases():
        assert shortcut(x) == llround_clamped(x), x
