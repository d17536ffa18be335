"""Python mirror of the reference ACE API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference C++ headers
(/root/reference/proj/include/ace/{srp,sketch,detect,estimators,dataset,
errors}.hpp), so parity tests read like the reference's own tests.  Every
hash / insert / score / detect call goes through libace_dev.so
(include/ace_b200.h); W generation goes through libace.so (the C++ host
layer).  Nothing here computes on the CPU.

Point matrices may be numpy arrays (host memory, copied in by the library) or
CUDA torch tensors (device memory, used in place).  1-D inputs are one point
(the reference's std::span<const double> API); 2-D inputs are batches
(extension).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

# ---------------------------------------------------------------- errors ----
# reference errors.hpp:9-26


class ContractViolation(ValueError):
    """Caller broke a documented precondition (std::invalid_argument)."""


class DataError(RuntimeError):
    """Input data is malformed."""


class InconsistentDelete(RuntimeError):
    """Delete of an item the sketch never saw (sketch unchanged)."""


class UnsupportedOperation(RuntimeError):
    """Operation not available under the current configuration."""


class CudaError(RuntimeError):
    """CUDA runtime failure (exit code 3 in the reference CLI)."""


_STATUS = {
    N.ACE_E_CONTRACT: ContractViolation,
    N.ACE_E_UNSUPPORTED: UnsupportedOperation,
    N.ACE_E_INCONSISTENT: InconsistentDelete,
    N.ACE_E_DATA: DataError,
    N.ACE_E_CUDA: CudaError,
    N.ACE_E_NOMEM: MemoryError,
}


def _check(status: int) -> None:
    if status != N.ACE_OK:
        raise _STATUS.get(status, RuntimeError)(N.last_error())


# ------------------------------------------------------------- helpers ------

POINT_MAX_ROWS = 32  # per-point path (include/ace_b200.h, ace_sketch_insert)


class _Points:
    """A point matrix as (pointer, dtype, n, ld, where) + keepalive."""

    def __init__(self, x, dim: int):
        self.keep = x
        if hasattr(x, "is_cuda") and hasattr(x, "data_ptr"):  # torch tensor
            t = x
            if t.dim() == 1:
                t = t.reshape(1, -1)
            if t.dim() != 2:
                raise ContractViolation("points must be 1-D or 2-D")
            if t.stride(1) != 1:
                t = t.contiguous()
            self.keep = t
            name = str(t.dtype)
            if name == "torch.float32":
                self.dtype = N.ACE_F32
            elif name == "torch.float64":
                self.dtype = N.ACE_F64
            else:
                t = t.float()
                self.keep = t
                self.dtype = N.ACE_F32
            self.n, cols = int(t.shape[0]), int(t.shape[1])
            self.ld = int(t.stride(0)) if self.n > 1 else cols
            self.where = N.ACE_DEVICE if t.is_cuda else N.ACE_HOST
            self.ptr = t.data_ptr()
        else:
            a = np.asarray(x)
            if a.dtype not in (np.float32, np.float64):
                a = a.astype(np.float64)
            if a.ndim == 1:
                a = a.reshape(1, -1)
            if a.ndim != 2:
                raise ContractViolation("points must be 1-D or 2-D")
            a = np.ascontiguousarray(a)
            self.keep = a
            self.dtype = N.ACE_F32 if a.dtype == np.float32 else N.ACE_F64
            self.n, cols = a.shape
            self.ld = cols
            self.where = N.ACE_HOST
            self.ptr = a.ctypes.data
        if cols != dim:
            raise ContractViolation(
                f"AceSketch: expected vector of length {dim}, received {cols}")


def generate_directions(seed: int, dim: int, k_bits: int, num_tables: int) -> np.ndarray:
    """W, (K*L) x dim binary64, row t*K+b (srp.cpp:36-48), from libace.so."""
    w = np.empty((k_bits * num_tables, dim), dtype=np.float64)
    if N.host().ace_generate_directions(seed, dim, k_bits, num_tables, w.ctypes.data) != 0:
        raise ContractViolation("generate_directions: bad configuration")
    return w


_M64 = (1 << 64) - 1


def mix_seed(seed: int, index: int) -> int:
    """rng::mix_seed (rng.hpp:19-22): splitmix64 of seed ^ golden * (index + 1)."""
    z = ((seed ^ ((0x9e3779b97f4a7c15 * (index + 1)) & _M64)) + 0x9e3779b97f4a7c15) & _M64
    z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & _M64
    z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & _M64
    return z ^ (z >> 31)


def _bits_to_bool(bits: np.ndarray, n: int) -> np.ndarray:
    return np.unpackbits(bits.view(np.uint8), bitorder="little")[:n].astype(bool)


# ----------------------------------------------------------------- srp -------
# reference srp.hpp:10-79


@dataclass
class SrpConfig:
    dim: int = 0
    k_bits: int = 15
    num_tables: int = 50
    seed: int = 0
    noise_scale: float = 0.0
    cache_projections: bool = True


def check_srp_config(cfg: SrpConfig) -> None:
    """SrpFamily's configuration checks (srp.cpp:25-32)."""
    if cfg.dim == 0:
        raise ContractViolation("SrpFamily: dim must be >= 1")
    if cfg.k_bits < 1 or cfg.k_bits > 30:
        raise ContractViolation("SrpFamily: k_bits must be in [1, 30]")
    if cfg.num_tables < 1:
        raise ContractViolation("SrpFamily: num_tables must be >= 1")
    if cfg.noise_scale < 0.0:
        raise ContractViolation("SrpFamily: noise_scale must be >= 0")


class SrpFamily:
    """Seeded SRP family; W generated on the host, hashing on the GPU."""

    def __init__(self, cfg: SrpConfig):
        check_srp_config(cfg)
        self._cfg = SrpConfig(**cfg.__dict__)
        self._w = generate_directions(cfg.seed, cfg.dim, cfg.k_bits, cfg.num_tables)
        self._dev: Optional[C.c_void_p] = None
        self._owner = True
        # noisy variant (srp.cpp:34, 97-101): aux stream seed and tick counter
        self._noise_seed = mix_seed(cfg.seed, 0x6e6f697365)
        self._noise_ctr = 0

    def _copy(self) -> "SrpFamily":
        """Copy semantics of the reference (srp.cpp:51-64): same W (device
        handle shared), own noise counter starting at the current value."""
        o = SrpFamily.__new__(SrpFamily)
        o.__dict__.update(self.__dict__)
        o._owner = False
        o._parent = self if self._owner else self._parent  # keeps the shared device handle alive
        return o

    # device handle, created on first use
    @property
    def handle(self) -> C.c_void_p:
        if not self._owner:
            return self._parent.handle
        if self._dev is None:
            h = C.c_void_p()
            _check(N.dev().ace_family_create(self._cfg.dim, self._cfg.k_bits, self._cfg.num_tables,
                                             self._cfg.noise_scale, self._w.ctypes.data, C.byref(h)))
            self._dev = h
        return self._dev

    def __del__(self):
        try:
            if self._owner and self._dev is not None:
                N.dev().ace_family_destroy(self._dev)
        except Exception:
            pass

    def config(self) -> SrpConfig:
        return self._cfg

    def set_kernel(self, which: str) -> None:
        """Projection kernel: "auto", "simt" or "tc" (tcgen05)."""
        code = {"auto": 0, "simt": 1, "tc": 2}[which]
        _check(N.dev().ace_family_set_kernel(self.handle, code))

    def kernel(self) -> str:
        return {1: "simt", 2: "tc"}[N.dev().ace_family_kernel(self.handle)]

    def num_buckets(self) -> int:
        return 1 << self._cfg.k_bits

    def direction(self, table: int, b: int) -> np.ndarray:
        if table >= self._cfg.num_tables or b >= self._cfg.k_bits or table < 0 or b < 0:
            raise ContractViolation("SrpFamily: direction index out of range")
        return self._w[table * self._cfg.k_bits + b].copy()

    @property
    def directions(self) -> np.ndarray:
        return self._w

    def projection_bytes(self) -> int:
        return self._w.nbytes if self._cfg.cache_projections else 0

    def reset_noise_stream(self, aux_seed: int) -> None:
        """srp.cpp:126-129."""
        self._noise_seed = int(aux_seed) & _M64
        self._noise_ctr = 0

    def draw_noise(self, count: int) -> np.ndarray:
        """Reserve `count` ticks; the terms noise_scale * N(0,1) (glibc libm, libace.so)."""
        out = np.empty(count, dtype=np.float64)
        tick0 = self._noise_ctr
        self._noise_ctr += count
        if count and N.host().ace_noise_terms(self._noise_seed, tick0, count, self._cfg.noise_scale,
                                              out.ctypes.data) != 0:
            raise ContractViolation("ace_noise_terms failed")
        return out

    def noisy_ids(self, x, t0: int, nt: int, b0: int, nb: int) -> np.ndarray:
        """Noisy bucket ids (nt, n): bits [b0, b0+nb) of tables [t0, t0+nt),
        ticks in point / table / bit order (srp.cpp:93-104)."""
        p = _Points(x, self._cfg.dim)
        noise = self.draw_noise(p.n * nt * nb)
        ids = np.empty((nt, p.n), dtype=np.uint32)
        if p.n and nt:
            _check(N.dev().ace_family_buckets_noisy(self.handle, p.ptr, p.dtype, p.n, p.ld, p.where, t0, nt, b0,
                                                    nb, noise.ctypes.data, N.ACE_HOST, ids.ctypes.data,
                                                    N.ACE_HOST))
        return ids

    def buckets(self, x, stats: Optional[N.AceHashStats] = None) -> np.ndarray:
        """Bucket ids, shape (L, n) uint32 (batched SrpFamily::bucket)."""
        if self._cfg.noise_scale > 0:
            return self.noisy_ids(x, 0, self._cfg.num_tables, 0, self._cfg.k_bits)
        p = _Points(x, self._cfg.dim)
        ids = np.empty((self._cfg.num_tables, p.n), dtype=np.uint32)
        st = stats if stats is not None else N.AceHashStats()
        if p.n:
            _check(N.dev().ace_family_buckets(self.handle, p.ptr, p.dtype, p.n, p.ld, p.where,
                                              ids.ctypes.data, N.ACE_HOST, C.byref(st)))
        return ids

    def bucket(self, table: int, x) -> int:
        self._check_indices(table, 0, x)
        if self._cfg.noise_scale > 0:
            return int(self.noisy_ids(np.asarray(x, dtype=np.float64), table, 1, 0, self._cfg.k_bits)[0, 0])
        return int(self.buckets(np.asarray(x, dtype=np.float64))[table, 0])

    def bit(self, table: int, b: int, x) -> int:
        self._check_indices(table, b, x)
        if self._cfg.noise_scale > 0:  # one tick
            return int(self.noisy_ids(np.asarray(x, dtype=np.float64), table, 1, b, 1)[0, 0])
        return (self.bucket(table, x) >> (self._cfg.k_bits - 1 - b)) & 1

    def _check_indices(self, table: int, b: int, x) -> None:
        n = np.asarray(x).shape[-1]
        if n != self._cfg.dim:
            raise ContractViolation(
                f"SrpFamily: expected vector of length {self._cfg.dim}, received {n}")
        if table >= self._cfg.num_tables:
            raise ContractViolation("SrpFamily: table index out of range")
        if b >= self._cfg.k_bits:
            raise ContractViolation("SrpFamily: bit index out of range")

    def __eq__(self, other) -> bool:
        a, b = self._cfg, other._cfg
        return (a.dim, a.k_bits, a.num_tables, a.seed, a.noise_scale) == (
            b.dim, b.k_bits, b.num_tables, b.seed, b.noise_scale)


# --------------------------------------------------------------- sketch ------
# reference sketch.hpp:11-84


class CounterWidth(enum.IntEnum):
    k16 = 16
    k32 = 32


@dataclass
class ScoreEstimate:
    value: float = 0.0
    k_bits: int = 0
    num_tables: int = 0


class AceSketch:
    kHeaderBytes = 53

    def __init__(self, family: SrpFamily, width: CounterWidth = CounterWidth.k16):
        self._family = family._copy()  # by value, as the reference (sketch.hpp:77)
        self._width = CounterWidth(width)
        h = C.c_void_p()
        _check(N.dev().ace_sketch_create(family.handle, int(self._width), C.byref(h)))
        self._h = h
        self.last_stats = N.AceHashStats()

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None:
                N.dev().ace_sketch_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def copy(self) -> "AceSketch":
        other = AceSketch.__new__(AceSketch)
        other._family = self._family
        other._width = self._width
        h = C.c_void_p()
        _check(N.dev().ace_sketch_clone(self._h, C.byref(h)))
        other._h = h
        other.last_stats = N.AceHashStats()
        return other

    __copy__ = copy

    def reset(self) -> None:
        _check(N.dev().ace_sketch_reset(self._h))

    def set_option(self, option: int, value: int) -> None:
        """Per-sketch execution option (N.ACE_OPT_*); results do not change."""
        _check(N.dev().ace_sketch_set_option(self._h, int(option), int(value)))

    def set_stream(self, stream_ptr: int) -> None:
        _check(N.dev().ace_sketch_set_stream(self._h, stream_ptr))

    def _dim(self) -> int:
        return self._family.config().dim

    def _noisy(self) -> bool:
        return self._family.config().noise_scale > 0

    def insert(self, x) -> None:
        """AceSketch::insert (sketch.cpp:50-72); 2-D input inserts rows in order."""
        if self._noisy():
            ids = np.ascontiguousarray(self._family.buckets(x))
            _check(N.dev().ace_sketch_insert_ids(self._h, ids.ctypes.data, ids.shape[1], N.ACE_HOST))
            return
        p = _Points(x, self._dim())
        if p.n <= POINT_MAX_ROWS and p.where == N.ACE_HOST:
            # a few host rows: the per-point path (one launch, no wait; no stats)
            self.last_stats = N.AceHashStats()
            _check(N.dev().ace_sketch_insert(self._h, p.ptr, p.dtype, p.n, p.ld, p.where, None))
            return
        _check(N.dev().ace_sketch_insert(self._h, p.ptr, p.dtype, p.n, p.ld, p.where,
                                         C.byref(self.last_stats)))

    def remove(self, x) -> None:
        """AceSketch::remove (sketch.cpp:74-106); batches are all-or-nothing."""
        if self._family.config().noise_scale > 0:
            raise UnsupportedOperation(
                "AceSketch: delete is unsupported with noisy hashes (buckets are not reproducible)")
        p = _Points(x, self._dim())
        _check(N.dev().ace_sketch_remove(self._h, p.ptr, p.dtype, p.n, p.ld, p.where,
                                         C.byref(self.last_stats)))

    def score(self, q) -> ScoreEstimate:
        """AceSketch::score (sketch.cpp:108-116) for one point."""
        q = np.asarray(q)
        if q.ndim != 1:
            raise ContractViolation("AceSketch::score takes one point; use score_batch")
        v = self.score_batch(q)
        cfg = self._family.config()
        return ScoreEstimate(float(v[0]), cfg.k_bits, cfg.num_tables)

    def score_batch(self, x, out=None, sums=None):
        """Scores S_i / L of every row (float64).  With `out`/`sums` CUDA
        tensors the results stay on the device."""
        if self._noisy():
            ids = np.ascontiguousarray(self._family.buckets(x))
            res = np.empty(ids.shape[1], dtype=np.float64)
            if ids.shape[1]:
                _check(N.dev().ace_sketch_score_ids(self._h, ids.ctypes.data, ids.shape[1], N.ACE_HOST,
                                                    res.ctypes.data, None, N.ACE_HOST))
            return res
        p = _Points(x, self._dim())
        if out is not None or sums is not None:
            _check(N.dev().ace_sketch_score(
                self._h, p.ptr, p.dtype, p.n, p.ld, p.where,
                out.data_ptr() if out is not None else None,
                sums.data_ptr() if sums is not None else None, N.ACE_DEVICE,
                C.byref(self.last_stats)))
            return out
        res = np.empty(p.n, dtype=np.float64)
        if p.n:
            _check(N.dev().ace_sketch_score(self._h, p.ptr, p.dtype, p.n, p.ld, p.where,
                                            res.ctypes.data, None, N.ACE_HOST,
                                            C.byref(self.last_stats)))
        return res

    def score_sums(self, x) -> np.ndarray:
        """Integer S_i (uint64) of every row."""
        p = _Points(x, self._dim())
        res = np.empty(p.n, dtype=np.uint64)
        if p.n:
            _check(N.dev().ace_sketch_score(self._h, p.ptr, p.dtype, p.n, p.ld, p.where, None,
                                            res.ctypes.data, N.ACE_HOST, C.byref(self.last_stats)))
        return res

    def _info(self):
        n, m, s = C.c_uint64(), C.c_double(), C.c_int()
        _check(N.dev().ace_sketch_info(self._h, C.byref(n), C.byref(m), C.byref(s)))
        return n.value, m.value, bool(s.value)

    def size(self) -> int:
        return self._info()[0]

    def mean(self) -> float:
        return self._info()[1]

    def saturated(self) -> bool:
        return self._info()[2]

    def family(self) -> SrpFamily:
        return self._family

    def counter_width(self) -> CounterWidth:
        return self._width

    def num_counters(self) -> int:
        cfg = self._family.config()
        return cfg.num_tables << cfg.k_bits

    def counter_bytes(self) -> int:
        return self.num_counters() * (2 if self._width == CounterWidth.k16 else 4)

    def memory_bytes(self) -> int:
        return self.counter_bytes() + self.kHeaderBytes

    def counters_u32(self) -> np.ndarray:
        out = np.empty(self.num_counters(), dtype=np.uint32)
        _check(N.dev().ace_sketch_counters_u32(self._h, out.ctypes.data, N.ACE_HOST))
        return out

    def counters_flat(self) -> np.ndarray:
        return self.counters_u32().astype(np.uint64)

    def counter(self, table: int, bucket: int) -> int:
        cfg = self._family.config()
        if table >= cfg.num_tables or bucket >= (1 << cfg.k_bits) or table < 0 or bucket < 0:
            raise ContractViolation("AceSketch: counter index out of range")
        v = C.c_uint64()
        _check(N.dev().ace_sketch_counter(self._h, table, bucket, C.byref(v)))
        return int(v.value)

    @classmethod
    def restore(cls, family: SrpFamily, width: CounterWidth, counters, n: int, mean: float,
                saturated: bool) -> "AceSketch":
        s = cls(family, width)
        c = np.ascontiguousarray(np.asarray(counters, dtype=np.uint64))
        _check(N.dev().ace_sketch_restore(s._h, c.ctypes.data, c.size, n, mean, int(saturated)))
        return s

    # -- pipelines (extensions) --
    def build_detect(self, x, flags_out=None, scores_out=None) -> "DetectionReport":
        """insert every row (build_sketch) then detect_batch over the same rows."""
        return _detect(self, x, build=True, flags_out=flags_out, scores_out=scores_out)

    def stream_batch(self, x, alpha: float, scores: bool = False, flags_out=None):
        """Score a batch against the current counts (flag score <= mean - alpha,
        none while empty), then insert it.  Returns (flags bool array or the
        device bitmap, scores or None, AceStreamReport)."""
        p = _Points(x, self._dim())
        rep = N.AceStreamReport()
        if flags_out is not None:
            _check(N.dev().ace_sketch_stream_batch(self._h, p.ptr, p.dtype, p.n, p.ld, p.where,
                                                   float(alpha), flags_out.data_ptr(), None,
                                                   N.ACE_DEVICE, C.byref(rep),
                                                   C.byref(self.last_stats)))
            return flags_out, None, rep
        bits = np.zeros((p.n + 31) // 32, dtype=np.uint32)
        sc = np.empty(p.n, dtype=np.float64) if scores else None
        _check(N.dev().ace_sketch_stream_batch(self._h, p.ptr, p.dtype, p.n, p.ld, p.where,
                                               float(alpha), bits.ctypes.data,
                                               sc.ctypes.data if sc is not None else None,
                                               N.ACE_HOST, C.byref(rep), C.byref(self.last_stats)))
        return _bits_to_bool(bits, p.n), sc, rep


    def stream_run(self, x, batch: int, alpha: float, flags_out=None, latencies: bool = True):
        """The streaming driver over consecutive batches of `batch` rows (score
        against counts at batch start, flag score <= mean - alpha, insert), queued
        without host synchronisation.  Returns (flags bool array or the device
        bitmap, per-batch device latency in ms, AceStreamReport with run totals)."""
        p = _Points(x, self._dim())
        rep = N.AceStreamReport()
        nb = (p.n + batch - 1) // batch
        lat = np.empty(nb, dtype=np.float32) if latencies else None
        if flags_out is not None:
            _check(N.dev().ace_sketch_stream_run(self._h, p.ptr, p.dtype, p.n, p.ld, p.where, batch,
                                                 float(alpha), flags_out.data_ptr(), N.ACE_DEVICE,
                                                 lat.ctypes.data if lat is not None else None,
                                                 C.byref(rep), C.byref(self.last_stats)))
            return flags_out, lat, rep
        bits = np.zeros((p.n + 31) // 32, dtype=np.uint32)
        _check(N.dev().ace_sketch_stream_run(self._h, p.ptr, p.dtype, p.n, p.ld, p.where, batch,
                                             float(alpha), bits.ctypes.data, N.ACE_HOST,
                                             lat.ctypes.data if lat is not None else None,
                                             C.byref(rep), C.byref(self.last_stats)))
        return _bits_to_bool(bits, p.n), lat, rep


# --------------------------------------------------------------- dataset -----
# reference dataset.hpp:14-31


@dataclass
class Dataset:
    values: np.ndarray
    labels: Optional[np.ndarray] = None
    name: str = ""

    @property
    def rows(self) -> int:
        return int(self.values.shape[0])

    @property
    def cols(self) -> int:
        return int(self.values.shape[1])

    def row(self, i: int) -> np.ndarray:
        return self.values[i]

    def labeled_anomalies(self) -> int:
        return 0 if self.labels is None else int(np.count_nonzero(self.labels))


# ---------------------------------------------------------------- detect -----
# reference detect.hpp:12-36


@dataclass
class DetectionReport:
    reported: int = 0
    correctly_reported: int = 0
    missed: int = 0
    total_labeled_anomalies: int = 0
    has_labels: bool = False
    threshold: float = 0.0
    score_mean: float = 0.0
    score_stddev: float = 0.0
    elapsed_seconds: float = 0.0
    # extensions
    flags: Optional[np.ndarray] = field(default=None, repr=False)
    scores: Optional[np.ndarray] = field(default=None, repr=False)
    ambiguous: int = 0
    replayed: bool = False
    stats: Optional[N.AceHashStats] = field(default=None, repr=False)


def _detect(sketch: AceSketch, data, build: bool, flags_out=None, scores_out=None,
            want_scores: bool = False) -> DetectionReport:
    values = data.values if isinstance(data, Dataset) else data
    labels = data.labels if isinstance(data, Dataset) else None
    p = _Points(values, sketch._dim())
    if p.n == 0:
        raise ContractViolation("detect_batch: empty dataset")
    if sketch._noisy():
        return _detect_noisy(sketch, values, labels, build, want_scores)
    rep = N.AceBatchReport()
    st = N.AceHashStats()
    fn = N.dev().ace_sketch_build_detect if build else N.dev().ace_sketch_detect_batch
    if flags_out is not None:
        _check(fn(sketch._h, p.ptr, p.dtype, p.n, p.ld, p.where, flags_out.data_ptr(),
                  scores_out.data_ptr() if scores_out is not None else None, N.ACE_DEVICE,
                  C.byref(rep), C.byref(st)))
        flags = None
        scores = None
    else:
        bits = np.zeros((p.n + 31) // 32, dtype=np.uint32)
        scores = np.empty(p.n, dtype=np.float64) if want_scores else None
        _check(fn(sketch._h, p.ptr, p.dtype, p.n, p.ld, p.where, bits.ctypes.data,
                  scores.ctypes.data if scores is not None else None, N.ACE_HOST,
                  C.byref(rep), C.byref(st)))
        flags = _bits_to_bool(bits, p.n)
    out = DetectionReport(
        reported=int(rep.reported), threshold=rep.threshold, score_mean=rep.score_mean,
        score_stddev=rep.score_stddev, elapsed_seconds=rep.elapsed_seconds, flags=flags,
        scores=scores, ambiguous=int(rep.ambiguous), replayed=bool(rep.replayed), stats=st)
    if labels is not None and flags is not None:  # detect.cpp:59-68
        lab = np.asarray(labels) != 0
        out.has_labels = True
        out.total_labeled_anomalies = int(lab.sum())
        out.correctly_reported = int((flags & lab).sum())
        out.missed = int((~flags & lab).sum())
    sketch.last_stats = st
    return out


def _detect_noisy(sketch: AceSketch, values, labels, build: bool, want_scores: bool) -> DetectionReport:
    """Noisy variant: device scores with fresh noise (ticks in row order, the
    reference's threads=1 order), then the reference's own statistics
    (detect.cpp:44-60: sequential binary64 sums, population sigma, s < thr)."""
    import time
    t0 = time.perf_counter()
    if build:
        sketch.insert(values)
    sc = sketch.score_batch(values)
    total = 0.0
    for v in sc:
        total += float(v)
    mean = total / len(sc)
    var = 0.0
    for v in sc:
        var += (float(v) - mean) * (float(v) - mean)
    sd = math.sqrt(var / len(sc))
    thr = mean - sd
    flags = sc < thr
    out = DetectionReport(reported=int(flags.sum()), threshold=thr, score_mean=mean, score_stddev=sd,
                          elapsed_seconds=time.perf_counter() - t0, flags=flags,
                          scores=sc if want_scores else None, stats=N.AceHashStats())
    if labels is not None:
        lab = np.asarray(labels) != 0
        out.has_labels = True
        out.total_labeled_anomalies = int(lab.sum())
        out.correctly_reported = int((flags & lab).sum())
        out.missed = int((~flags & lab).sum())
    return out


def detect_batch(sketch: AceSketch, data, threads: int = 0, want_scores: bool = False) -> DetectionReport:
    """detect_batch (detect.cpp:12-74); `threads` is accepted for API parity."""
    values = data.values if isinstance(data, Dataset) else data
    if int(values.shape[-1]) != sketch._dim():
        raise ContractViolation("detect_batch: data dimension mismatch")
    return _detect(sketch, data, build=False, want_scores=want_scores)


def detect_stream(sketch: AceSketch, q, alpha: float):
    """detect_stream (detect.cpp:76-84): (ScoreEstimate, score <= mean - alpha)."""
    if alpha < 0.0:
        raise ContractViolation("detect_stream: alpha must be >= 0")
    cfg = sketch.family().config()
    qa = np.asarray(q)
    if cfg.noise_scale > 0 or qa.ndim != 1 or qa.shape[0] != cfg.dim:
        if sketch.size() == 0:
            raise ContractViolation("detect_stream: empty sketch")
        est = sketch.score(q)
        return est, est.value <= sketch.mean() - alpha
    p = _Points(qa, cfg.dim)
    v, f = C.c_double(), C.c_uint8()
    _check(N.dev().ace_sketch_detect_stream(sketch._h, p.ptr, p.dtype, 1, p.ld, p.where, float(alpha),
                                            C.byref(v), C.byref(f)))
    return ScoreEstimate(v.value, cfg.k_bits, cfg.num_tables), bool(f.value)


# ------------------------------------------------------------ estimators -----

def build_sketch(data, k_bits: int, num_tables: int, seed: int, noise_scale: float = 0.0,
                 width: CounterWidth = CounterWidth.k16) -> AceSketch:
    """build_sketch (estimators.cpp:79-92): insert every row in order."""
    values = data.values if isinstance(data, Dataset) else data
    if values.shape[0] == 0:
        raise ContractViolation("build_sketch: empty dataset")
    fam = SrpFamily(SrpConfig(dim=int(values.shape[1]), k_bits=k_bits, num_tables=num_tables,
                              seed=seed, noise_scale=noise_scale))
    sk = AceSketch(fam, width)
    sk.insert(values)
    return sk


# ACE1 sketch files (reference io.hpp:23-27)
from .sketch_io import load_dataset, load_sketch, save_sketch  # noqa: E402
