"""ctypes bindings to the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``liboracle.so``         -- oracle/jabba_oracle.c, the plain-C restatement.
* ``_ref/libjabba_ref.so`` -- the unmodified reference headers bound by
  oracle/ref_shim.cpp (built in the dev container; the prebuilt .so travels
  to the GPU box).

Both expose the same flat conventions as include/jabba_b200.h.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libjabba_ref.so")

i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class JoConfig(C.Structure):
    _fields_ = [
        ("tol", C.c_double), ("max_piece_len", C.c_int64), ("backend", C.c_int32),
        ("scl", C.c_double), ("k", C.c_uint64), ("r", C.c_double),
        ("max_iters", C.c_uint64), ("n_init", C.c_uint64), ("seed", C.c_uint64),
        ("alpha", C.c_double), ("sort_key", C.c_int32), ("early_stop", C.c_int32),
        ("has_alpha_len", C.c_int32), ("alpha_len", C.c_double),
        ("has_alpha_inc", C.c_int32), ("alpha_inc", C.c_double), ("eta", C.c_double),
        ("threads", C.c_uint32),
    ]


class JoFit(C.Structure):
    _fields_ = [
        ("n_seg", C.c_int64), ("n_pieces", C.c_int64),
        ("piece_offsets", C.POINTER(C.c_int64)), ("piece_len", C.POINTER(C.c_int64)),
        ("piece_inc", C.POINTER(C.c_double)), ("anchors", C.POINTER(C.c_double)),
        ("source_lengths", C.POINTER(C.c_int64)), ("k", C.c_uint64),
        ("centers", C.POINTER(C.c_double)), ("mean_lengths", C.POINTER(C.c_double)),
        ("scaling", C.c_double * 3), ("labels", C.POINTER(C.c_uint32)),
        ("iterations", C.c_uint64), ("sample_size", C.c_uint64),
    ]


BACKENDS = {"vq": 0, "svq": 1, "ga": 2, "ga-auto": 3, "ga-hier": 4}


def make_config(**kw) -> JoConfig:
    """Reference defaults (compression.hpp:18-20, clustering.hpp:19-41,
    digitization.hpp:78,110-117, jabba.hpp:17-21) overridden by kw."""
    d = dict(tol=0.1, max_piece_len=0, backend="ga", scl=1.0, k=8, r=1.0, max_iters=300,
             n_init=1, seed=0, alpha=0.5, sort_key=0, early_stop=1, alpha_len=None,
             alpha_inc=None, eta=1.0, threads=1)
    d.update(kw)
    c = JoConfig()
    c.tol, c.max_piece_len = d["tol"], d["max_piece_len"]
    b = d["backend"]
    c.backend = BACKENDS[b] if isinstance(b, str) else int(b)
    c.scl, c.k, c.r = d["scl"], d["k"], d["r"]
    c.max_iters, c.n_init, c.seed = d["max_iters"], d["n_init"], d["seed"]
    c.alpha = d["alpha"]
    sk = d["sort_key"]
    c.sort_key = (1 if sk in ("two_norm", 1) else 0) if not isinstance(sk, int) else sk
    c.early_stop = int(bool(d["early_stop"]))
    c.has_alpha_len = d["alpha_len"] is not None
    c.alpha_len = d["alpha_len"] or 0.0
    c.has_alpha_inc = d["alpha_inc"] is not None
    c.alpha_inc = d["alpha_inc"] or 0.0
    c.eta, c.threads = d["eta"], d["threads"]
    return c


@dataclass
class FitArrays:
    status: int
    piece_offsets: np.ndarray
    piece_len: np.ndarray
    piece_inc: np.ndarray
    anchors: np.ndarray
    source_lengths: np.ndarray
    k: int
    centers: np.ndarray
    mean_lengths: np.ndarray
    scaling: np.ndarray
    labels: np.ndarray
    iterations: int = 0
    sample_size: int = 0
    error: str = ""


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def build():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class _Lib:
    prefix = ""

    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.L = C.CDLL(path)
        self.p = prefix
        L, p = self.L, prefix
        getattr(L, p + "last_error").restype = C.c_char_p

    def err(self):
        return getattr(self.L, self.p + "last_error")().decode()

    def _unpack(self, st, r: JoFit, free):
        if st != 0:
            free(C.byref(r))
            return FitArrays(st, *([None] * 5), 0, None, None, None, None, error=self.err())
        n, ns, k = r.n_pieces, r.n_seg, r.k
        out = FitArrays(
            st, _arr(r.piece_offsets, ns + 1, np.int64), _arr(r.piece_len, n, np.int64),
            _arr(r.piece_inc, n, np.float64), _arr(r.anchors, ns, np.float64),
            _arr(r.source_lengths, ns, np.int64), int(k),
            _arr(r.centers, 2 * k, np.float64).reshape(-1, 2),
            _arr(r.mean_lengths, k, np.float64), np.array(list(r.scaling)),
            _arr(r.labels, n, np.uint32), int(r.iterations), int(r.sample_size))
        free(C.byref(r))
        return out


class Oracle(_Lib):
    """The C restatement (oracle/jabba_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        super().__init__(ORACLE_SO, "jo_")

    def symbolize_with(self, centers, scaling, lens, incs):
        """symbolize_with (digitization.hpp:297-307) -> (status, labels)."""
        c = np.ascontiguousarray(centers, np.float64).reshape(-1)
        sc = np.ascontiguousarray(scaling, np.float64)
        lens = np.ascontiguousarray(lens, np.int64)
        incs = np.ascontiguousarray(incs, np.float64)
        labels = np.zeros(max(len(lens), 1), np.uint32)
        f = getattr(self.L, self.p + "symbolize_with")
        f.argtypes = [f64p, C.c_uint64, f64p, i64p, f64p, C.c_int64, u32p]
        st = f(c, len(c) // 2, sc, lens, incs, len(lens), labels)
        return st, labels[: len(lens)]

    def plan_segments(self, series_lengths, layout, parts):
        sl = np.ascontiguousarray(series_lengths, np.int64)
        cap = int(len(sl) * max(parts, 1))
        first = np.zeros(cap, np.int64)
        steps = np.zeros(cap, np.int64)
        nseg = C.c_int64(0)
        f = self.L.jo_plan_segments
        f.argtypes = [i64p, C.c_int64, C.c_int32, C.c_int64, i64p, i64p, C.POINTER(C.c_int64)]
        st = f(sl, len(sl), layout, parts, first, steps, C.byref(nseg))
        if st:
            return st, None, None
        return 0, first[: nseg.value].copy(), steps[: nseg.value].copy()

    def fit(self, values, seg_first, seg_steps, layout, cfg: JoConfig) -> FitArrays:
        f = self.L.jo_fit
        f.argtypes = [f64p, i64p, i64p, C.c_int64, C.POINTER(JoConfig), C.POINTER(JoFit)]
        r = JoFit()
        st = f(np.ascontiguousarray(values, np.float64), np.ascontiguousarray(seg_first, np.int64),
               np.ascontiguousarray(seg_steps, np.int64), len(seg_first), C.byref(cfg), C.byref(r))
        return self._unpack(st, r, self.L.jo_fit_free)

    def reconstruct(self, fit: FitArrays, layout, labels=None):
        size_f = self.L.jo_reconstruct_size
        size_f.argtypes = [i64p, C.c_int64, C.c_int32]
        size_f.restype = C.c_int64
        n = size_f(fit.source_lengths, len(fit.source_lengths), layout)
        out = np.zeros(max(n, 1), np.float64)
        f = self.L.jo_reconstruct
        f.argtypes = [f64p, f64p, C.c_uint64, f64p, u32p, i64p, f64p, i64p, C.c_int64,
                      C.c_int32, f64p]
        lab = fit.labels if labels is None else labels
        st = f(np.ascontiguousarray(fit.centers.reshape(-1)), fit.mean_lengths, fit.k,
               np.ascontiguousarray(fit.scaling), np.ascontiguousarray(lab, np.uint32),
               fit.piece_offsets, fit.anchors, fit.source_lengths, len(fit.source_lengths),
               layout, out)
        return st, out[:n]

    def quantize_lengths(self, real):
        real = np.ascontiguousarray(real, np.float64)
        out = np.zeros(len(real), np.int64)
        f = self.L.jo_quantize_lengths
        f.argtypes = [f64p, C.c_int64, i64p]
        f(real, len(real), out)
        return out

    def match_total_length(self, lens, target):
        lens = np.ascontiguousarray(lens, np.int64).copy()
        f = self.L.jo_match_total_length
        f.argtypes = [i64p, C.c_int64, C.c_int64]
        st = f(lens, len(lens), target)
        return st, lens

    def auto_alpha(self, n, N, tol, eta):
        f = self.L.jo_auto_alpha
        f.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_int)]
        f.restype = C.c_double
        st = C.c_int(0)
        a = f(n, N, tol, eta, C.byref(st))
        return st.value, a

    def inverse_compress(self, lens, incs, anchor):
        lens = np.ascontiguousarray(lens, np.int64)
        incs = np.ascontiguousarray(incs, np.float64)
        out = np.zeros(int(lens.sum()) + 1 if len(lens) else 1, np.float64)
        f = self.L.jo_inverse_compress
        f.argtypes = [i64p, f64p, C.c_int64, C.c_double, f64p]
        st = f(lens, incs, len(lens), anchor, out)
        return st, out

    def greedy_aggregate(self, pts, alpha, sort_key=0, early_stop=1):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        n = len(pts)
        labels = np.zeros(max(n, 1), np.uint32)
        sp = np.zeros(max(n, 1), np.int64)
        ng = C.c_int64(0)
        f = getattr(self.L, self.p + "greedy_aggregate")
        f.argtypes = [f64p, C.c_int64, C.c_double, C.c_int32, C.c_int32, u32p,
                      C.POINTER(C.c_int64), i64p]
        st = f(pts.reshape(-1), n, alpha, sort_key, early_stop, labels, C.byref(ng), sp)
        return st, labels[:n], sp[: ng.value]

    def kmeans(self, pts, k, max_iters=300, n_init=1, seed=0):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        n = len(pts)
        labels = np.zeros(max(n, 1), np.uint32)
        centers = np.zeros(2 * k, np.float64)
        it = C.c_uint64(0)
        f = getattr(self.L, self.p + "kmeans")
        f.argtypes = [f64p, C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u32p,
                      f64p, C.POINTER(C.c_uint64)]
        st = f(pts.reshape(-1), n, k, max_iters, n_init, seed, labels, centers, C.byref(it))
        return st, labels[:n], centers.reshape(-1, 2), it.value

    def sample_indices(self, n, s, seed):
        out = np.zeros(max(s, 1), np.uint64)
        f = getattr(self.L, self.p + "sample_indices")
        f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        f(n, s, seed, out)
        return out[:s]

    def mt_stream(self, seed, count):
        out = np.zeros(count, np.uint64)
        f = getattr(self.L, self.p + "mt_stream")
        f.argtypes = [C.c_uint64, C.c_uint64, u64p]
        f(seed, count, out)
        return out

    def uniform_int_stream(self, seed, lo, hi, count):
        out = np.zeros(count, np.uint64)
        f = getattr(self.L, self.p + "uniform_int_stream")
        f.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        f(seed, lo, hi, count, out)
        return out

    def uniform_real_stream(self, seed, lo, hi, count):
        out = np.zeros(count, np.float64)
        f = getattr(self.L, self.p + "uniform_real_stream")
        f.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64, f64p]
        f(seed, lo, hi, count, out)
        return out


class Reference(Oracle):
    """The unmodified reference, bound by oracle/ref_shim.cpp."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        _Lib.__init__(self, REF_SO, "jref_")

    def fit(self, values, seg_first, seg_steps, layout, cfg: JoConfig) -> FitArrays:
        f = self.L.jref_fit
        f.argtypes = [f64p, i64p, i64p, C.c_int64, C.c_int32, C.POINTER(JoConfig),
                      C.POINTER(JoFit)]
        r = JoFit()
        st = f(np.ascontiguousarray(values, np.float64), np.ascontiguousarray(seg_first, np.int64),
               np.ascontiguousarray(seg_steps, np.int64), len(seg_first), layout, C.byref(cfg),
               C.byref(r))
        return self._unpack(st, r, self.L.jref_fit_free)

    def reconstruct(self, fit: FitArrays, layout, labels=None):
        n = Oracle.__new__(Oracle)
        total = int((fit.source_lengths + 1).sum())
        if layout == 0:
            total -= len(fit.source_lengths) - 1
        out = np.zeros(max(total, 1), np.float64)
        f = self.L.jref_reconstruct
        f.argtypes = [f64p, f64p, C.c_uint64, f64p, u32p, i64p, f64p, i64p, C.c_int64,
                      C.c_int32, f64p]
        lab = fit.labels if labels is None else labels
        st = f(np.ascontiguousarray(fit.centers.reshape(-1)), fit.mean_lengths, fit.k,
               np.ascontiguousarray(fit.scaling), np.ascontiguousarray(lab, np.uint32),
               fit.piece_offsets, fit.anchors, fit.source_lengths, len(fit.source_lengths),
               layout, out)
        del n
        return st, out[:total]

    def quantize_lengths(self, real):
        real = np.ascontiguousarray(real, np.float64)
        out = np.zeros(len(real), np.int64)
        f = self.L.jref_quantize_lengths
        f.argtypes = [f64p, C.c_int64, i64p]
        f(real, len(real), out)
        return out

    def auto_alpha(self, n, N, tol, eta):
        f = self.L.jref_auto_alpha
        f.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_int)]
        f.restype = C.c_double
        st = C.c_int(0)
        a = f(n, N, tol, eta, C.byref(st))
        return st.value, a
