"""Reference-shaped host API over the B200 C ABI.

Mirrors the reference's public C++ surface (/root/reference/proj/include/jabba):
types of core.hpp (TimeSeries, Dataset, Piece, PieceSequence, ScalingParams,
Codebook, SymbolicResult), the configs (CompressionConfig, VQConfig, GAConfig,
DigitizeConfig, JabbaConfig), the errors (core.hpp:20-30), and the two entry
points ``jabba_fit`` (jabba.hpp:30-36) / ``reconstruct`` (inverse.hpp:127-132),
exported under the BASELINE names ``fit_transform`` / ``inverse_transform``.

All compute runs in libjabba_b200.so on the GPU. ``Engine.fit_arrays`` is
the flat, zero-copy entry used by the benchmark (values may already live in
HBM as a CUDA tensor).
"""
from __future__ import annotations

import atexit
import ctypes as C
import enum
import weakref
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N


# ---------------------------------------------------------------------------
# errors (core.hpp:20-30)

class JabbaError(RuntimeError):
    pass


class InvalidInput(JabbaError):
    pass


class InvalidPiece(JabbaError):
    pass


class InvalidPartition(JabbaError):
    pass


class UnknownSymbol(JabbaError):
    pass


class ParseError(JabbaError):
    pass


class LayoutError(JabbaError):
    pass


class VersionError(JabbaError):
    pass


class DeviceError(JabbaError):
    pass


_ERRORS = {1: InvalidInput, 2: InvalidPiece, 3: InvalidPartition, 4: UnknownSymbol,
           5: ParseError, 6: LayoutError, 7: VersionError}


def _check(rc: int):
    if rc != 0:
        raise _ERRORS.get(rc, DeviceError)(f"[{rc}] {N.last_error()}")


# ---------------------------------------------------------------------------
# domain types (core.hpp)

class Layout(enum.IntEnum):  # core.hpp:55
    univariate_partitioned = 0
    multivariate = 1
    collection = 2


class Backend(enum.IntEnum):  # digitization.hpp:88
    vq = 0
    sampling_vq = 1
    ga = 2
    ga_auto = 3
    ga_hier = 4


class SortKey(enum.IntEnum):  # clustering.hpp:34
    first_principal_component = 0
    two_norm = 1


def backend_from_string(s: str) -> Backend:  # digitization.hpp:101-108
    m = {"vq": Backend.vq, "svq": Backend.sampling_vq, "ga": Backend.ga,
         "ga-auto": Backend.ga_auto, "ga-hier": Backend.ga_hier}
    if s not in m:
        raise InvalidInput(f'unknown backend "{s}"')
    return m[s]


_BACKEND_TAG = {Backend.vq: "vq", Backend.sampling_vq: "svq", Backend.ga: "ga",
                Backend.ga_auto: "ga-auto", Backend.ga_hier: "ga-hier"}


@dataclass
class TimeSeries:  # core.hpp:35-53
    values: np.ndarray
    id: str = ""

    def __post_init__(self):
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    def steps(self) -> int:
        return max(0, self.values.size - 1)


@dataclass
class Dataset:  # core.hpp:68-99
    series: List[TimeSeries]
    layout: Layout = Layout.collection
    m: int = 0
    parts: int = 1  # extension: split every member series (configs 2 and 5)

    @staticmethod
    def partitioned(ts: TimeSeries, partitions: int) -> "Dataset":
        return Dataset([ts], Layout.univariate_partitioned, partitions, partitions)

    @staticmethod
    def multivariate(dims: Sequence[TimeSeries]) -> "Dataset":
        d = Dataset(list(dims), Layout.multivariate, len(dims))
        for s in d.series:
            if s.values.size != d.series[0].values.size:
                raise LayoutError("multivariate dataset has ragged dimensions")
        return d

    @staticmethod
    def collection(members: Sequence[TimeSeries], parts: int = 1) -> "Dataset":
        return Dataset(list(members), Layout.collection, len(members), parts)


@dataclass
class Piece:  # core.hpp:104-107
    len: int
    inc: float


@dataclass
class PieceSequence:  # core.hpp:109-120
    pieces: List[Piece]
    anchor: float
    source_id: str
    source_length: int

    def total_len(self) -> int:
        return sum(p.len for p in self.pieces)


@dataclass
class CompressedBatch:  # compression.hpp:107-133
    segments: List[PieceSequence]
    layout: Layout

    def total_pieces(self) -> int:
        return sum(len(s.pieces) for s in self.segments)

    def total_steps(self) -> int:
        return sum(s.source_length for s in self.segments)

    def boundaries(self) -> List[int]:
        return list(np.cumsum([len(s.pieces) for s in self.segments]))


@dataclass
class ScalingParams:  # core.hpp:125-133
    scl: float = 1.0
    sigma_len: float = 1.0
    sigma_inc: float = 1.0

    def apply(self, p: Piece):
        return (self.scl * float(p.len) / self.sigma_len, p.inc / self.sigma_inc)


def symbol_token(rank: int, alphabet_size: int) -> str:  # core.hpp:186-193
    buf = C.create_string_buffer(32)
    N.lib().jb_symbol_token(rank, alphabet_size, buf)
    return buf.value.decode()


@dataclass
class Codebook:  # core.hpp:137-181
    centers: np.ndarray             # (k, 2) scaled space
    symbols: List[str]
    mean_lengths: np.ndarray
    scaling: ScalingParams
    digitizer_tag: str = ""

    def size(self) -> int:
        return len(self.centers)

    def index_of(self, token: str) -> int:
        try:
            return self.symbols.index(token)
        except ValueError:
            raise UnknownSymbol(f'token not in codebook alphabet: "{token}"') from None


@dataclass
class SymbolicSeries:  # SymbolicResult::Series core.hpp:197-202
    id: str
    anchor: float
    source_length: int
    labels: np.ndarray


@dataclass
class SymbolicResult:  # core.hpp:196-215
    codebook: Codebook
    series: List[SymbolicSeries]
    layout: Layout = Layout.collection

    def tokens(self, i: int) -> List[str]:
        return [self.codebook.symbols[l] for l in self.series[i].labels]


# ---------------------------------------------------------------------------
# configs

@dataclass
class CompressionConfig:  # compression.hpp:18-26
    tol: float = 0.1
    max_piece_len: int = 0


@dataclass
class VQConfig:  # clustering.hpp:19-32
    k: int = 8
    r: float = 1.0
    max_iters: int = 300
    n_init: int = 1
    seed: int = 0


@dataclass
class GAConfig:  # clustering.hpp:36-48
    alpha: float = 0.5
    sort_key: SortKey = SortKey.first_principal_component
    early_stop: bool = True
    alpha_len: Optional[float] = None
    alpha_inc: Optional[float] = None


@dataclass
class AutoDigitizeConfig:  # digitization.hpp:77-83
    eta: float = 1.0


@dataclass
class DigitizeConfig:  # digitization.hpp:110-117
    backend: Backend = Backend.ga
    scl: float = 1.0
    vq: VQConfig = field(default_factory=VQConfig)
    ga: GAConfig = field(default_factory=GAConfig)
    auto_digitize: AutoDigitizeConfig = field(default_factory=AutoDigitizeConfig)
    tol: float = 0.0


@dataclass
class JabbaConfig:  # jabba.hpp:17-21
    compression: CompressionConfig = field(default_factory=CompressionConfig)
    digitize: DigitizeConfig = field(default_factory=DigitizeConfig)
    threads: int = 1

    @staticmethod
    def of(tol=0.1, backend="ga", scl=1.0, k=8, r=1.0, max_iters=300, n_init=1, seed=0,
           alpha=0.5, sort_key=0, early_stop=True, alpha_len=None, alpha_inc=None, eta=1.0,
           max_piece_len=0, threads=1) -> "JabbaConfig":
        """Flat constructor with the BASELINE parameter names."""
        b = backend_from_string(backend) if isinstance(backend, str) else Backend(backend)
        sk = SortKey.two_norm if sort_key in ("two_norm", 1) else SortKey.first_principal_component
        return JabbaConfig(
            CompressionConfig(tol, max_piece_len),
            DigitizeConfig(b, scl, VQConfig(k, r, max_iters, n_init, seed),
                           GAConfig(alpha, sk, bool(early_stop), alpha_len, alpha_inc),
                           AutoDigitizeConfig(eta)),
            threads)

    def to_c(self) -> N.JbConfig:
        c = N.JbConfig()
        c.tol = self.compression.tol
        c.max_piece_len = self.compression.max_piece_len
        d = self.digitize
        c.backend = int(d.backend)
        c.scl = d.scl
        c.k, c.r, c.max_iters, c.n_init, c.seed = d.vq.k, d.vq.r, d.vq.max_iters, d.vq.n_init, d.vq.seed
        c.alpha = d.ga.alpha
        c.sort_key = int(d.ga.sort_key)
        c.early_stop = int(bool(d.ga.early_stop))
        c.has_alpha_len = d.ga.alpha_len is not None
        c.alpha_len = d.ga.alpha_len or 0.0
        c.has_alpha_inc = d.ga.alpha_inc is not None
        c.alpha_inc = d.ga.alpha_inc or 0.0
        c.eta = d.auto_digitize.eta
        c.threads = self.threads
        return c


@dataclass
class JabbaFit:  # jabba.hpp:23-26
    batch: CompressedBatch
    symbolic: SymbolicResult


# ---------------------------------------------------------------------------
# engine (device context)

def plan_segments(series_lengths, layout: int, parts: int):
    """jb_plan_segments: Dataset layout checks + split_series."""
    sl = np.ascontiguousarray(series_lengths, np.int64)
    cap = max(1, len(sl) * max(int(parts), 1))
    first = np.zeros(cap, np.int64)
    steps = np.zeros(cap, np.int64)
    nseg = C.c_int64(0)
    _check(N.lib().jb_plan_segments(sl, len(sl), int(layout), int(parts), first, steps,
                                    C.byref(nseg)))
    return first[: nseg.value].copy(), steps[: nseg.value].copy()


_LIVE = weakref.WeakSet()


@atexit.register
def _release_all():
    """Free device-resident handles while the CUDA runtime is still alive
    (interpreter teardown order is otherwise unspecified)."""
    fits = [o for o in list(_LIVE) if isinstance(o, NativeFit)]
    engines = [o for o in list(_LIVE) if isinstance(o, Engine)]
    for o in fits + engines:
        o.close()


class NativeFit:
    """Device-resident result of one fit_transform (owns a jb_fit handle)."""

    def __init__(self, engine: "Engine", handle: C.c_void_p):
        self.engine = engine
        self.h = handle
        _LIVE.add(self)
        L = N.lib()
        self.n_seg = L.jb_fit_n_segments(handle)
        self.n_pieces = L.jb_fit_n_pieces(handle)
        self.k = L.jb_fit_k(handle)
        self.layout = L.jb_fit_layout(handle)

    def close(self):
        if getattr(self, "h", None) and N is not None and N._lib is not None:
            N._lib.jb_fit_free(self.h)
        self.h = None

    def __del__(self):
        self.close()

    def pieces(self):
        off = np.zeros(self.n_seg + 1, np.int64)
        ln = np.zeros(max(self.n_pieces, 1), np.int64)
        inc = np.zeros(max(self.n_pieces, 1), np.float64)
        _check(N.lib().jb_fit_copy_pieces(self.h, off.ctypes.data, ln.ctypes.data,
                                          inc.ctypes.data))
        return off, ln[: self.n_pieces], inc[: self.n_pieces]

    def piece_offsets(self) -> np.ndarray:
        """First piece of every segment (n_seg + 1 offsets), without the pieces."""
        off = np.zeros(self.n_seg + 1, np.int64)
        _check(N.lib().jb_fit_copy_pieces(self.h, off.ctypes.data, None, None))
        return off

    def symbolic_arrays(self, labels=True):
        k = self.k
        lab = np.zeros(max(self.n_pieces, 1), np.uint32)
        cen = np.zeros(max(2 * k, 1), np.float64)
        ml = np.zeros(max(k, 1), np.float64)
        sc = np.zeros(3, np.float64)
        anc = np.zeros(self.n_seg, np.float64)
        sl = np.zeros(self.n_seg, np.int64)
        _check(N.lib().jb_fit_copy_symbolic(self.h, lab.ctypes.data if labels else None,
                                            cen.ctypes.data, ml.ctypes.data, sc.ctypes.data,
                                            anc.ctypes.data, sl.ctypes.data))
        return dict(labels=lab[: self.n_pieces], centers=cen[: 2 * k].reshape(-1, 2),
                    mean_lengths=ml[:k], scaling=sc, anchors=anc, source_lengths=sl)

    def labels_into(self, out: np.ndarray):
        """Copy ranked labels into a caller buffer (e.g. pinned host memory)."""
        _check(N.lib().jb_fit_copy_symbolic(self.h, out.ctypes.data, None, None, None, None,
                                            None))

    def stats(self):
        it, ss, dr = C.c_uint64(), C.c_uint64(), C.c_uint64()
        fr, gr = C.c_int32(), C.c_int32()
        ph = np.zeros(8, np.float64)
        _check(N.lib().jb_fit_stats(self.h, C.byref(it), C.byref(ss), C.byref(dr), C.byref(fr),
                                    C.byref(gr), ph.ctypes.data))
        return dict(iterations=it.value, sample_size=ss.value, draws=dr.value,
                    fix_rounds=fr.value, ga_rounds=gr.value,
                    ms=dict(zip(["compress", "scale", "backend", "stats", "total"], ph[:5])),
                    lloyd_tiles_processed=int(ph[5]), lloyd_labels_changed=int(ph[6]),
                    d2_tiles_updated=int(ph[7]))

    def reconstruct_size(self) -> int:
        return N.lib().jb_fit_reconstruct_size(self.h)

    def inverse(self, out=None, out_ptr: Optional[int] = None, on_device=False):
        """inverse_transform on the device-resident fit. Returns (values, offsets)
        (values is `out` or a new host array); with on_device=True writes to
        the device pointer out_ptr."""
        n = self.reconstruct_size()
        n_out = 1 if self.layout == 0 else self.n_seg
        off = np.zeros(n_out + 1, np.int64)
        if on_device:
            _check(N.lib().jb_fit_inverse_transform(self.engine.ctx, self.h, C.c_void_p(out_ptr),
                                                    1, off.ctypes.data))
            return None, off
        if out is None:
            out = np.empty(max(n, 1), np.float64)
        _check(N.lib().jb_fit_inverse_transform(self.engine.ctx, self.h, out.ctypes.data, 0,
                                                off.ctypes.data))
        return out[:n], off


class Engine:
    """A CUDA context + stream on one device (jb_context)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(N.lib().jb_context_create(int(device), C.byref(h)))
        self.ctx = h
        self.device = device
        _LIVE.add(self)

    def close(self):
        if getattr(self, "ctx", None) and N is not None and N._lib is not None:
            N._lib.jb_context_destroy(self.ctx)
        self.ctx = None

    def __del__(self):
        self.close()

    def fit_arrays(self, values, seg_first, seg_steps, layout: int, cfg: JabbaConfig,
                   device_ptr: Optional[int] = None, n_values: Optional[int] = None) -> NativeFit:
        """fit_transform on a flat segment table. `values` is a host float64
        array, or pass device_ptr (+ n_values) for HBM-resident input."""
        sf = np.ascontiguousarray(seg_first, np.int64)
        ss = np.ascontiguousarray(seg_steps, np.int64)
        c = cfg.to_c()
        h = C.c_void_p()
        if device_ptr is not None:
            _check(N.lib().jb_fit_transform(self.ctx, C.c_void_p(device_ptr), int(n_values), 1, sf,
                                            ss, len(sf), int(layout), C.byref(c), C.byref(h)))
        else:
            v = np.ascontiguousarray(values, np.float64)
            _check(N.lib().jb_fit_transform(self.ctx, v.ctypes.data, v.size, 0, sf, ss, len(sf),
                                            int(layout), C.byref(c), C.byref(h)))
        return NativeFit(self, h)

    def mt19937_64_stream(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(max(count, 1), np.uint64)
        _check(N.lib().jb_mt19937_64_stream(self.ctx, seed, count, out.ctypes.data))
        return out[:count]

    def sample_indices(self, n: int, sample_size: int, seed: int) -> np.ndarray:
        out = np.zeros(max(sample_size, 1), np.uint64)
        _check(N.lib().jb_sample_indices(self.ctx, n, sample_size, seed, out.ctypes.data))
        return out[:sample_size]

    def kmeans(self, points, k: int, max_iters: int = 300, n_init: int = 1, seed: int = 0):
        """jabba::kmeans (clustering.hpp:224-236) on device: (labels, centers, iterations)."""
        p = np.ascontiguousarray(points, np.float64).reshape(-1, 2)
        n = len(p)
        labels = np.zeros(max(n, 1), np.uint32)
        centers = np.zeros(max(2 * k, 1), np.float64)
        it = C.c_uint64(0)
        _check(N.lib().jb_kmeans(self.ctx, p.ctypes.data, n, k, max_iters, n_init, seed,
                                 labels.ctypes.data, centers.ctypes.data, C.byref(it)))
        return labels[:n], centers[: 2 * k].reshape(-1, 2), it.value

    def mse(self, a, b) -> float:
        """jabba::mse (metrics.hpp:18-29) on device, bit-exact."""
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        if len(a) != len(b):
            raise InvalidInput(f"mse: length mismatch ({len(a)} vs {len(b)})")
        out = C.c_double(0)
        _check(N.lib().jb_mse(self.ctx, a.ctypes.data, b.ctypes.data, len(a), 0, C.byref(out)))
        return out.value

    def seq_sum_nonneg(self, terms, seg_off=None) -> np.ndarray:
        """The reference's sequential ``s += w`` over non-negative terms
        (digitization.hpp:39-45, 224-231), per segment, bit-exact on device."""
        w = np.ascontiguousarray(terms, np.float64)
        off = np.ascontiguousarray([0, len(w)] if seg_off is None else seg_off, np.int64)
        out = np.zeros(max(len(off) - 1, 1), np.float64)
        _check(N.lib().jb_seq_sum_nonneg(self.ctx, w.ctypes.data, off.ctypes.data, len(off) - 1,
                                         out.ctypes.data))
        return out[: len(off) - 1]

    def inverse_arrays(self, centers, mean_lengths, scaling, labels, piece_offsets, anchors,
                       source_lengths, layout: int) -> np.ndarray:
        sl = np.ascontiguousarray(source_lengths, np.int64)
        n = N.lib().jb_reconstruct_size(sl, len(sl), int(layout))
        out = np.empty(max(n, 1), np.float64)
        cen = np.ascontiguousarray(centers, np.float64).reshape(-1)
        _check(N.lib().jb_inverse_transform(
            self.ctx, cen, np.ascontiguousarray(mean_lengths, np.float64), len(cen) // 2,
            np.ascontiguousarray(scaling, np.float64), np.ascontiguousarray(labels, np.uint32),
            np.ascontiguousarray(piece_offsets, np.int64), np.ascontiguousarray(anchors, np.float64),
            sl, len(sl), int(layout), out.ctypes.data))
        return out[:n]

    def symbolize_arrays(self, centers, scaling, lens, incs, device_ptrs=None) -> np.ndarray:
        """symbolize_with (digitization.hpp:297-307) on the GPU: labels of the
        pieces (lens, incs) against the codebook (centers (k, 2), scaling).
        device_ptrs = (len_i64_ptr, inc_ptr, labels_ptr, n): device arrays."""
        cen = np.ascontiguousarray(centers, np.float64).reshape(-1)
        sc = np.ascontiguousarray(scaling, np.float64)
        if device_ptrs is not None:
            lp, ip, op, n = device_ptrs
            _check(N.lib().jb_symbolize_with(self.ctx, cen, len(cen) // 2, sc, C.c_void_p(lp),
                                             C.c_void_p(ip), int(n), 1, C.c_void_p(op)))
            return None
        lens = np.ascontiguousarray(lens, np.int64)
        incs = np.ascontiguousarray(incs, np.float64)
        out = np.empty(max(len(lens), 1), np.uint32)
        _check(N.lib().jb_symbolize_with(self.ctx, cen, len(cen) // 2, sc, lens.ctypes.data,
                                         incs.ctypes.data, len(lens), 0, out.ctypes.data))
        return out[: len(lens)]


# ---------------------------------------------------------------------------
# multi-GPU: one joint fit sharded over ranks (jb_fit_transform_dist)

def shard_segments(seg_steps, world: int, rank: int):
    """Contiguous segment range [s0, s1) of `rank`, balanced by steps
    (compression, scaling, final assignment and inverse work are all
    proportional to samples)."""
    steps = np.asarray(seg_steps, np.int64)
    n = len(steps)
    if world > n:
        raise InvalidPartition(f"{n} segments cannot be sharded over {world} ranks")
    cum = np.concatenate([[0], np.cumsum(steps)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(cum, total * r / world, side="left"))
        c = max(c, cuts[-1] + 1)              # every rank gets >= 1 segment
        c = min(c, n - (world - r))
        cuts.append(c)
    cuts.append(n)
    return cuts[rank], cuts[rank + 1]


def local_view(seg_first, seg_steps, s0: int, s1: int):
    """Sample range [lo, hi] this rank needs for segments [s0, s1) and the
    segment table rebased onto it (split segments share boundary samples)."""
    f = np.asarray(seg_first, np.int64)[s0:s1]
    st = np.asarray(seg_steps, np.int64)[s0:s1]
    lo = int(f[0])
    hi = int((f + st).max())
    return lo, hi, f - lo, st


class TorchComm:
    """jb_comm over torch.distributed: an exact allgather of host bytes
    (gloo on host tensors; nccl staged through the rank's GPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        world = self.world

        def _allgather(user, send, nbytes, recv):
            try:
                if nbytes == 0:
                    return 0
                src = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(send))
                t = torch.from_numpy(src.copy())
                if backend == "nccl":
                    t = t.to(device)
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t, group=group)
                cat = torch.cat(outs).cpu().numpy()
                C.memmove(recv, cat.ctypes.data, nbytes * world)
                return 0
            except Exception:  # noqa: BLE001 -- reported as JB_NCCL_ERROR by the library
                return 1

        self._fn = N.ALLGATHER_FN(_allgather)
        self.c = N.JbComm(None, self.rank, self.world, self._fn)


def fit_arrays_dist(engine: "Engine", comm: TorchComm, values_local, seg_first_local,
                    seg_steps_local, n_seg_global: int, layout: int, cfg: JabbaConfig,
                    device_ptr: Optional[int] = None, n_values: Optional[int] = None) -> "NativeFit":
    """This rank's part of a joint fit_transform (see jb_fit_transform_dist)."""
    sf = np.ascontiguousarray(seg_first_local, np.int64)
    ss = np.ascontiguousarray(seg_steps_local, np.int64)
    c = cfg.to_c()
    h = C.c_void_p()
    if device_ptr is not None:
        _check(N.lib().jb_fit_transform_dist(engine.ctx, C.byref(comm.c), C.c_void_p(device_ptr),
                                             int(n_values), 1, sf, ss, len(sf), n_seg_global,
                                             int(layout), C.byref(c), C.byref(h)))
    else:
        v = np.ascontiguousarray(values_local, np.float64)
        _check(N.lib().jb_fit_transform_dist(engine.ctx, C.byref(comm.c), v.ctypes.data, v.size,
                                             0, sf, ss, len(sf), n_seg_global, int(layout),
                                             C.byref(c), C.byref(h)))
    return NativeFit(engine, h)


_default_engine: Optional[Engine] = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine(0)
    return _default_engine


# ---------------------------------------------------------------------------
# reference entry points

def _flatten(dataset: Dataset):
    if not dataset.series:
        raise InvalidInput("empty dataset")
    lengths = np.array([s.values.size for s in dataset.series], np.int64)
    parts = dataset.m if dataset.layout == Layout.univariate_partitioned else dataset.parts
    if dataset.layout != Layout.univariate_partitioned and dataset.m != len(dataset.series):
        raise LayoutError("dataset m does not match member count")
    first, steps = plan_segments(lengths, int(dataset.layout), parts)
    values = np.concatenate([s.values for s in dataset.series]) if len(dataset.series) > 1 \
        else dataset.series[0].values
    # segment ids: split parts are "<id>[s]" (compression.hpp:153)
    ids = []
    for s in dataset.series:
        if dataset.layout == Layout.univariate_partitioned or parts > 1:
            ids += [f"{s.id}[{i}]" for i in range(parts)]
        else:
            ids.append(s.id)
    return values, first, steps, ids


def jabba_fit(dataset: Dataset, cfg: JabbaConfig, engine: Optional[Engine] = None) -> JabbaFit:
    """jabba_fit (jabba.hpp:30-36): compress all segments, digitize jointly."""
    eng = engine or default_engine()
    values, first, steps, ids = _flatten(dataset)
    nf = eng.fit_arrays(values, first, steps, int(dataset.layout), cfg)
    off, ln, inc = nf.pieces()
    sym = nf.symbolic_arrays()
    segs = []
    for s in range(nf.n_seg):
        a, b = off[s], off[s + 1]
        segs.append(PieceSequence([Piece(int(l), float(x)) for l, x in zip(ln[a:b], inc[a:b])],
                                  float(sym["anchors"][s]), ids[s], int(sym["source_lengths"][s])))
    k = nf.k
    cb = Codebook(sym["centers"], [symbol_token(r, k) for r in range(k)], sym["mean_lengths"],
                  ScalingParams(*sym["scaling"]), _BACKEND_TAG[cfg.digitize.backend])
    series = [SymbolicSeries(ids[s], float(sym["anchors"][s]), int(sym["source_lengths"][s]),
                             sym["labels"][off[s]:off[s + 1]].copy()) for s in range(nf.n_seg)]
    layout = Layout(dataset.layout)
    return JabbaFit(CompressedBatch(segs, layout), SymbolicResult(cb, series, layout))


fit_transform = jabba_fit


def reconstruct(symbolic: SymbolicResult, engine: Optional[Engine] = None) -> List[TimeSeries]:
    """reconstruct (inverse.hpp:127-132): inverse_symbolize, stitched for a
    univariate-partitioned fit."""
    eng = engine or default_engine()
    cb = symbolic.codebook
    ser = symbolic.series
    offs = np.zeros(len(ser) + 1, np.int64)
    offs[1:] = np.cumsum([len(s.labels) for s in ser])
    labels = np.concatenate([np.asarray(s.labels, np.uint32) for s in ser]) if ser else \
        np.zeros(0, np.uint32)
    sc = cb.scaling
    out = eng.inverse_arrays(np.asarray(cb.centers, np.float64).reshape(-1, 2),
                             np.asarray(cb.mean_lengths, np.float64),
                             np.array([sc.scl, sc.sigma_len, sc.sigma_inc]), labels, offs,
                             np.array([s.anchor for s in ser], np.float64),
                             np.array([s.source_length for s in ser], np.int64),
                             int(symbolic.layout))
    if symbolic.layout == Layout.univariate_partitioned:
        name = ser[0].id
        if "[" in name:
            name = name[: name.index("[")]
        return [TimeSeries(out, name)]
    res, pos = [], 0
    for s in ser:
        n = s.source_length + 1
        res.append(TimeSeries(out[pos:pos + n].copy(), s.id))
        pos += n
    return res


inverse_transform = reconstruct


def symbolize_with(codebook: Codebook, seq: PieceSequence,
                   engine: Optional[Engine] = None) -> SymbolicSeries:
    """symbolize_with (digitization.hpp:297-307): held-out pieces against a
    fitted codebook, on the GPU (Codebook::nearest of ScalingParams::apply,
    lowest index on ties)."""
    eng = engine or default_engine()
    if codebook.size() == 0:
        raise InvalidInput("symbolize_with: empty codebook")
    sc = codebook.scaling
    lens = np.array([p.len for p in seq.pieces], np.int64)
    incs = np.array([p.inc for p in seq.pieces], np.float64)
    labels = eng.symbolize_arrays(np.asarray(codebook.centers, np.float64).reshape(-1, 2),
                                  [sc.scl, sc.sigma_len, sc.sigma_inc], lens, incs)
    return SymbolicSeries(seq.source_id, seq.anchor, seq.source_length, labels)
