"""CPU tests of the C-ABI boundary: the library loads, exports every symbol
include/jabba_b200.h declares, and its host-only entry points (segment
planning, tokens, defaults) behave like the reference. No GPU compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2401_00109_b200 import _native as N
from paper_2401_00109_b200 import api

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "jabba_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(jb_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = N.lib()
    decl = declared_symbols()
    assert len(decl) >= 20
    for s in decl:
        assert hasattr(L, s), s
    assert sorted(N.EXPORTS) == decl


def test_abi_version_and_defaults():
    L = N.lib()
    assert L.jb_abi_version() == 1
    c = N.JbConfig()
    L.jb_config_default(C.byref(c))
    # reference defaults: compression.hpp:19-20, clustering.hpp:20-24,37-39,
    # digitization.hpp:78,111-112, jabba.hpp:20
    assert (c.tol, c.max_piece_len, c.backend, c.scl) == (0.1, 0, 2, 1.0)
    assert (c.k, c.r, c.max_iters, c.n_init, c.seed) == (8, 1.0, 300, 1, 0)
    assert (c.alpha, c.sort_key, c.early_stop, c.eta, c.threads) == (0.5, 0, 1, 1.0, 1)


@pytest.mark.parametrize("lengths,layout,parts", [
    ([13], 0, 3), ([12], 0, 3), ([4000], 0, 8), ([10, 20, 30], 2, 1), ([100, 100], 1, 1),
    ([10001, 10001], 2, 4), ([100000] * 3, 2, 8), ([7], 0, 6), ([2], 2, 1),
])
def test_plan_segments_matches_oracle(oracle, lengths, layout, parts):
    st, f0, s0 = oracle.plan_segments(lengths, layout, parts)
    f1, s1 = api.plan_segments(lengths, layout, parts)
    assert st == 0
    assert np.array_equal(f0, f1) and np.array_equal(s0, s1)


@pytest.mark.parametrize("lengths,layout,parts,exc", [
    ([4], 0, 4, api.InvalidPartition),         # split_series m > steps
    ([10], 0, 0, api.InvalidPartition),        # m == 0
    ([10, 10], 0, 2, api.LayoutError),         # partitioned needs one series
    ([10, 9], 1, 1, api.LayoutError),          # ragged multivariate
    ([], 2, 1, api.InvalidInput),              # empty dataset
])
def test_plan_segments_errors(lengths, layout, parts, exc):
    with pytest.raises(exc):
        api.plan_segments(lengths, layout, parts)


def test_symbol_tokens():
    # core.hpp:186-193
    assert api.symbol_token(0, 3) == "A"
    assert api.symbol_token(61, 94) == "~"
    assert api.symbol_token(62, 94) == "!"
    assert api.symbol_token(93, 94) == "@"
    assert api.symbol_token(57, 120) == "#57"


def test_no_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(api.DeviceError):
        api.Engine(0)
