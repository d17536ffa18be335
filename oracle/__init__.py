"""Parity checkers (TEST INFRASTRUCTURE ONLY).

`Oracle`    — ctypes over _build/libaceoracle.so, the plain-C restatement of the
              reference algorithm (ace_oracle.c, each function cites the
              reference file:line it follows).
`Reference` — ctypes over _ref/libaceref.so, the UNMODIFIED reference sources
              compiled by oracle/Makefile plus the extern "C" harness
              ref_driver.cpp.  Built in the dev container (where
              /root/reference exists) and shipped prebuilt to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
--impl reference legs may import this package — as the checker or the timed
CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libaceoracle.so"
REF_SO = HERE / "_ref" / "libaceref.so"

_vp, _u64, _u32, _i, _d = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
_P = C.POINTER


def _threads() -> int:
    return max(1, os.cpu_count() or 1)


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32)


class Oracle:
    """The C restatement (ace_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: make -C oracle oracle")
        L = C.CDLL(str(path))
        L.ora_mix_seed.restype = _u64
        L.ora_mix_seed.argtypes = [_u64, _u64]
        L.ora_directions.restype = None
        L.ora_directions.argtypes = [_u64, _u64, _u32, _u32, _vp]
        L.ora_bucket.restype = _u32
        L.ora_bucket.argtypes = [_vp, _u64, _u32, _u64, _vp]
        L.ora_project.restype = _d
        L.ora_project.argtypes = [_vp, _vp, _u64]
        L.ora_buckets.restype = _u64
        L.ora_buckets.argtypes = [_vp, _u64, _u32, _u32, _vp, _i, _u64, _vp, _i, _d]
        L.ora_buckets_fast.restype = _u64
        L.ora_buckets_fast.argtypes = [_vp, _u64, _u32, _u32, _vp, _i, _u64, _vp, _i, _d]
        L.ora_sketch_new.restype = _vp
        L.ora_sketch_new.argtypes = [_u32, _u32, _u32]
        L.ora_sketch_free.argtypes = [_vp]
        L.ora_sketch_size.restype = _u64
        L.ora_sketch_size.argtypes = [_vp]
        L.ora_sketch_mean.restype = _d
        L.ora_sketch_mean.argtypes = [_vp]
        L.ora_sketch_saturated.restype = _i
        L.ora_sketch_saturated.argtypes = [_vp]
        L.ora_sketch_counters.argtypes = [_vp, _vp]
        L.ora_insert_batch.argtypes = [_vp, _vp, _u64]
        L.ora_remove_ids.restype = _i
        L.ora_remove_ids.argtypes = [_vp, _vp, _u64]
        L.ora_score_batch.argtypes = [_vp, _vp, _u64, _vp, _vp]
        L.ora_detect_batch_from_scores.restype = _u64
        L.ora_detect_batch_from_scores.argtypes = [_vp, _u64, _P(_d), _P(_d), _P(_d), _vp]
        L.ora_stream_batch.restype = _u64
        L.ora_stream_batch.argtypes = [_vp, _vp, _u64, _d, _vp, _vp]
        self.L = L

    def directions(self, seed, dim, k, l) -> np.ndarray:
        w = np.empty((k * l, dim), dtype=np.float64)
        self.L.ora_directions(seed, dim, k, l, w.ctypes.data)
        return w

    def buckets(self, w, x, k, l, threads=None, rel_eps=0.0, fast=True):
        """(ids (L, n) uint32, near-tie count below rel_eps).  fast: the
        row-blocked fold (ora_buckets_fast, same bits); else the scalar one."""
        x = np.ascontiguousarray(x)
        is64 = x.dtype == np.float64
        if not is64:
            x = _f32(x)
        n, dim = x.shape
        ids = np.empty((l, n), dtype=np.uint32)
        fn = self.L.ora_buckets_fast if fast else self.L.ora_buckets
        near = fn(np.ascontiguousarray(w).ctypes.data, dim, k, l, x.ctypes.data,
                  int(is64), n, ids.ctypes.data, threads or _threads(), rel_eps)
        return ids, int(near)

    def project(self, wrow, x) -> float:
        wrow = np.ascontiguousarray(wrow, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.L.ora_project(wrow.ctypes.data, x.ctypes.data, x.size)

    def sketch(self, k, l, width=32) -> "OracleSketch":
        return OracleSketch(self, k, l, width)


class OracleSketch:
    def __init__(self, o: Oracle, k, l, width):
        self.o, self.k, self.l = o, k, l
        self.h = o.L.ora_sketch_new(k, l, width)

    def __del__(self):
        try:
            self.o.L.ora_sketch_free(self.h)
        except Exception:
            pass

    def insert_ids(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        self.o.L.ora_insert_batch(self.h, ids.ctypes.data, ids.shape[1])

    def remove_ids_point(self, ids_col) -> bool:
        ids_col = np.ascontiguousarray(ids_col, dtype=np.uint32)
        return self.o.L.ora_remove_ids(self.h, ids_col.ctypes.data, 1) == 0

    def score_ids(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        n = ids.shape[1]
        sc = np.empty(n, dtype=np.float64)
        sums = np.empty(n, dtype=np.uint64)
        self.o.L.ora_score_batch(self.h, ids.ctypes.data, n, sc.ctypes.data, sums.ctypes.data)
        return sc, sums

    def stream_ids(self, ids, alpha):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        n = ids.shape[1]
        sc = np.empty(n, dtype=np.float64)
        fl = np.empty(n, dtype=np.uint8)
        self.o.L.ora_stream_batch(self.h, ids.ctypes.data, n, alpha, sc.ctypes.data, fl.ctypes.data)
        return fl.astype(bool), sc

    def counters(self):
        out = np.empty(self.l << self.k, dtype=np.uint64)
        self.o.L.ora_sketch_counters(self.h, out.ctypes.data)
        return out

    def size(self):
        return self.o.L.ora_sketch_size(self.h)

    def mean(self):
        return self.o.L.ora_sketch_mean(self.h)

    def saturated(self):
        return bool(self.o.L.ora_sketch_saturated(self.h))


def detect_from_scores(o: Oracle, scores):
    """detect.cpp:44-68 on given scores: (mean, sd, thr, flags)."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    m, s, t = _d(), _d(), _d()
    fl = np.empty(scores.size, dtype=np.uint8)
    o.L.ora_detect_batch_from_scores(scores.ctypes.data, scores.size, C.byref(m), C.byref(s),
                                     C.byref(t), fl.ctypes.data)
    return m.value, s.value, t.value, fl.astype(bool)


class Reference:
    """The compiled reference (oracle/_ref/libaceref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: make -C oracle ref (needs /root/reference)")
        L = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_directions.restype = _i
        L.ref_directions.argtypes = [_u64, _u64, _u32, _u32, _vp]
        L.ref_buckets.restype = _i
        L.ref_buckets.argtypes = [_u64, _u64, _u32, _u32, _vp, _u64, _vp, _i]
        L.ref_sketch_new.restype = _vp
        L.ref_sketch_new.argtypes = [_u64, _u64, _u32, _u32, _u32]
        L.ref_sketch_free.argtypes = [_vp]
        L.ref_sketch_insert.restype = _i
        L.ref_sketch_insert.argtypes = [_vp, _vp, _u64, _u64]
        L.ref_sketch_insert_f64.restype = _i
        L.ref_sketch_insert_f64.argtypes = [_vp, _vp, _u64, _u64]
        L.ref_sketch_remove.restype = _i
        L.ref_sketch_remove.argtypes = [_vp, _vp, _u64, _u64]
        L.ref_sketch_score.restype = _i
        L.ref_sketch_score.argtypes = [_vp, _vp, _u64, _u64, _vp]
        L.ref_sketch_size.restype = _u64
        L.ref_sketch_size.argtypes = [_vp]
        L.ref_sketch_mean.restype = _d
        L.ref_sketch_mean.argtypes = [_vp]
        L.ref_sketch_saturated.restype = _i
        L.ref_sketch_saturated.argtypes = [_vp]
        L.ref_sketch_counters.argtypes = [_vp, _vp]
        L.ref_detect_batch.restype = _i
        L.ref_detect_batch.argtypes = [_vp, _vp, _u64, _u64, C.c_uint, _P(_d), _P(_d), _P(_d),
                                       _P(_u64), _P(_d), _vp]
        L.ref_stream_batch.restype = _i
        L.ref_stream_batch.argtypes = [_vp, _vp, _u64, _u64, _d, _vp, _vp]
        L.ref_time_build_detect.restype = _i
        L.ref_time_build_detect.argtypes = [_u64, _vp, _u64, _u64, _u32, _u32, C.c_uint, _P(_d),
                                            _P(_d), _P(_u64)]
        L.ref_time_point.restype = _i
        L.ref_time_point.argtypes = [_u64, _vp, _u64, _u64, _u64, _u32, _u32, _d, _P(_d), _P(_u64), _vp, _vp]
        L.ref_time_stream.restype = _i
        L.ref_time_stream.argtypes = [_u64, _vp, _u64, _u64, _u32, _u32, _u64, _d, C.c_uint, _P(_d), _P(_d),
                                      _P(_u64)]
        L.ref_save_sketch.restype = _i
        L.ref_save_sketch.argtypes = [_vp, C.c_char_p]
        L.ref_load_sketch.restype = _vp
        L.ref_load_sketch.argtypes = [C.c_char_p, _P(_i)]
        L.ref_sketch_config.argtypes = [_vp, _P(_u64), _P(_u32), _P(_u32), _P(_u64), _P(_u32)]
        L.ref_sketch_new_noisy.restype = _vp
        L.ref_sketch_new_noisy.argtypes = [_u64, _u64, _u32, _u32, _u32, _d]
        L.ref_sketch_reset_noise.argtypes = [_vp, _u64]
        L.ref_noisy_calls.restype = _i
        L.ref_noisy_calls.argtypes = [_u64, _u64, _u32, _u32, _d, _i, _u64, _vp, _u64, _u32, _u32, _i, _vp]
        L.ref_noisy_sequence.restype = _i
        L.ref_noisy_sequence.argtypes = [_u64, _u64, _u32, _u32, _d, _u64, _vp, _vp, _u64, _vp]
        L.ref_load_dataset.restype = _i
        L.ref_load_dataset.argtypes = [C.c_char_p, _i, _i, _vp, _vp, _vp, _vp]
        L.ref_free.argtypes = [_vp]
        self.L = L

    def _ok(self, rc):
        if rc != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def load_dataset(self, path, label_column=None):
        """ace::io::load_dataset: (values (rows, cols) f64, labels u8 or None);
        DataError -> ValueError with the reference's message."""
        vals, labs = _vp(), _vp()
        rows, cols = _u64(), _u64()
        rc = self.L.ref_load_dataset(str(path).encode(), int(label_column is not None), int(label_column or 0),
                                     C.byref(vals), C.byref(rows), C.byref(cols), C.byref(labs))
        if rc != 0:
            raise (ValueError if rc == -3 else RuntimeError)(self.L.ref_last_error().decode())
        n, d = rows.value, cols.value
        v = np.ctypeslib.as_array(C.cast(vals, _P(_d)), shape=(n * d,)).copy().reshape(n, d)
        lab = None
        if labs.value:
            lab = np.ctypeslib.as_array(C.cast(labs, _P(C.c_uint8)), shape=(n,)).copy()
            self.L.ref_free(labs)
        self.L.ref_free(vals)
        return v, lab

    def noisy_calls(self, seed, dim, k, l, noise, x, t0, nt, b=-1, aux=None):
        """A noisy family's bucket (b < 0) or bit(t, b) calls, rows in order,
        tables t0..t0+nt-1; ids (nt, n)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        n = x.shape[0]
        ids = np.empty((nt, n), dtype=np.uint32)
        self._ok(self.L.ref_noisy_calls(seed, dim, k, l, noise, int(aux is not None), aux or 0, x.ctypes.data, n,
                                        t0, nt, b, ids.ctypes.data))
        return ids

    def noisy_sequence(self, seed, dim, k, l, noise, aux, x, ops):
        """Calls (row, table, b) on one noisy family after reset_noise_stream(aux);
        b < 0 is bucket(table, x[row]), else bit(table, b, x[row])."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        o = np.ascontiguousarray(np.asarray(ops, dtype=np.int32).reshape(-1, 3))
        out = np.empty(o.shape[0], dtype=np.uint32)
        self._ok(self.L.ref_noisy_sequence(seed, dim, k, l, noise, aux, x.ctypes.data, o.ctypes.data, o.shape[0],
                                           out.ctypes.data))
        return out

    def noisy_sketch(self, seed, dim, k, l, noise, width=32, aux=None) -> "RefSketch":
        r = RefSketch.__new__(RefSketch)
        r.r, r.dim, r.k, r.l = self, dim, k, l
        r.h = self.L.ref_sketch_new_noisy(seed, dim, k, l, width, noise)
        if not r.h:
            raise RuntimeError(self.L.ref_last_error().decode())
        if aux is not None:
            self.L.ref_sketch_reset_noise(r.h, aux)
        return r

    def load_sketch(self, path) -> "RefSketch":
        """ace::io::load_sketch (io.cpp:213-244); DataError -> ValueError."""
        st = _i()
        h = self.L.ref_load_sketch(str(path).encode(), C.byref(st))
        if not h:
            msg = self.L.ref_last_error().decode()
            raise (ValueError if st.value == -3 else RuntimeError)(msg)
        dim, seed = _u64(), _u64()
        k, l, width = _u32(), _u32(), _u32()
        self.L.ref_sketch_config(h, C.byref(dim), C.byref(k), C.byref(l), C.byref(seed), C.byref(width))
        r = RefSketch.__new__(RefSketch)
        r.r, r.dim, r.k, r.l, r.h = self, dim.value, k.value, l.value, h
        r.seed, r.width = seed.value, width.value
        return r

    def directions(self, seed, dim, k, l):
        w = np.empty((k * l, dim), dtype=np.float64)
        self._ok(self.L.ref_directions(seed, dim, k, l, w.ctypes.data))
        return w

    def buckets(self, seed, x, k, l, threads=None):
        x = _f32(x)
        n, dim = x.shape
        ids = np.empty((l, n), dtype=np.uint32)
        self._ok(self.L.ref_buckets(seed, dim, k, l, x.ctypes.data, n, ids.ctypes.data,
                                    threads or _threads()))
        return ids

    def sketch(self, seed, dim, k, l, width=32) -> "RefSketch":
        return RefSketch(self, seed, dim, k, l, width)

    def time_build_detect(self, seed, x, k, l, threads=0):
        x = _f32(x)
        n, dim = x.shape
        ti, td, rep = _d(), _d(), _u64()
        self._ok(self.L.ref_time_build_detect(seed, x.ctypes.data, n, dim, k, l, threads,
                                              C.byref(ti), C.byref(td), C.byref(rep)))
        return ti.value, td.value, rep.value


    def time_stream(self, seed, x, k, l, batch, alpha, threads=0):
        """(seconds scoring on `threads` cores, seconds inserting on one core,
        reported) of the stream-ordered reference loop over the rows."""
        x = _f32(x)
        n, dim = x.shape
        ts, ti, rep = _d(), _d(), _u64()
        self._ok(self.L.ref_time_stream(seed, x.ctypes.data, n, dim, k, l, batch, alpha, threads, C.byref(ts),
                                        C.byref(ti), C.byref(rep)))
        return ts.value, ti.value, rep.value

    def time_point(self, seed, x, n_build, k, l, alpha, outputs=False):
        """(seconds, reported[, scores, flags]) of the per-point loop
        detect_stream + insert over rows n_build.. of x (ace_cli stream
        --adapt), after an untimed build from the first n_build rows."""
        x = _f32(x)
        n, dim = x.shape
        q = n - n_build
        sec, rep = _d(), _u64()
        sc = np.empty(q, dtype=np.float64) if outputs else None
        fl = np.empty(q, dtype=np.uint8) if outputs else None
        self._ok(self.L.ref_time_point(seed, x.ctypes.data, n_build, q, dim, k, l, alpha, C.byref(sec), C.byref(rep),
                                       sc.ctypes.data if outputs else None, fl.ctypes.data if outputs else None))
        return (sec.value, rep.value, sc, fl) if outputs else (sec.value, rep.value)


class RefSketch:
    def __init__(self, r: Reference, seed, dim, k, l, width):
        self.r, self.dim, self.k, self.l = r, dim, k, l
        self.h = r.L.ref_sketch_new(seed, dim, k, l, width)
        if not self.h:
            raise RuntimeError(r.L.ref_last_error().decode())

    def __del__(self):
        try:
            self.r.L.ref_sketch_free(self.h)
        except Exception:
            pass

    def insert(self, x):
        x = np.ascontiguousarray(x)
        if x.ndim == 1:
            x = x.reshape(1, -1)
        if x.dtype == np.float64:
            self.r._ok(self.r.L.ref_sketch_insert_f64(self.h, x.ctypes.data, x.shape[0], self.dim))
        else:
            x = _f32(x)
            self.r._ok(self.r.L.ref_sketch_insert(self.h, x.ctypes.data, x.shape[0], self.dim))

    def remove(self, x) -> int:
        x = _f32(x).reshape(-1, self.dim)
        return self.r.L.ref_sketch_remove(self.h, x.ctypes.data, x.shape[0], self.dim)

    def score(self, x):
        x = _f32(x).reshape(-1, self.dim)
        out = np.empty(x.shape[0], dtype=np.float64)
        self.r._ok(self.r.L.ref_sketch_score(self.h, x.ctypes.data, x.shape[0], self.dim,
                                             out.ctypes.data))
        return out

    def detect_batch(self, x, threads=0):
        x = _f32(x)
        m, s, t, e = _d(), _d(), _d(), _d()
        rep = _u64()
        fl = np.empty(x.shape[0], dtype=np.uint8)
        self.r._ok(self.r.L.ref_detect_batch(self.h, x.ctypes.data, x.shape[0], self.dim, threads,
                                             C.byref(m), C.byref(s), C.byref(t), C.byref(rep),
                                             C.byref(e), fl.ctypes.data))
        return dict(mean=m.value, sd=s.value, thr=t.value, reported=rep.value,
                    elapsed=e.value, flags=fl.astype(bool))

    def stream_batch(self, x, alpha):
        x = _f32(x)
        sc = np.empty(x.shape[0], dtype=np.float64)
        fl = np.empty(x.shape[0], dtype=np.uint8)
        self.r._ok(self.r.L.ref_stream_batch(self.h, x.ctypes.data, x.shape[0], self.dim, alpha,
                                             sc.ctypes.data, fl.ctypes.data))
        return fl.astype(bool), sc

    def counters(self):
        out = np.empty(self.l << self.k, dtype=np.uint64)
        self.r.L.ref_sketch_counters(self.h, out.ctypes.data)
        return out

    def size(self):
        return self.r.L.ref_sketch_size(self.h)

    def mean(self):
        return self.r.L.ref_sketch_mean(self.h)

    def saturated(self):
        return bool(self.r.L.ref_sketch_saturated(self.h))

    def save(self, path):
        """ace::io::save_sketch (io.cpp:184-211)."""
        self.r._ok(self.r.L.ref_save_sketch(self.h, str(path).encode()))
