"""ACE1 sketch files (reference io.hpp:23-27, io.cpp:184-244) and CSV
ingestion (io.hpp:16-21, io.cpp:89-182, parsed by libace.so on all host
threads).

Layout, little-endian, 53-byte header (AceSketch::kHeaderBytes):
    "ACE1" | dim u32 | k_bits u32 | num_tables u32 | width u32 (16/32) |
    seed u64 | noise_scale f64 | n u64 | mean f64 | saturated u8 |
    L * 2^K counters, table-major, u16 or u32 by width.
The counters come from (and go back to) the device sketch; the file bytes are
what the reference's save_sketch writes for the same state.
"""
from __future__ import annotations

import ctypes as C
import struct

import numpy as np

from . import _native as N
from . import ace

MAGIC = b"ACE1"
_HDR = struct.Struct("<4sIIIIQdQdB")
assert _HDR.size == 53


def ace1_bytes(dim, k_bits, num_tables, width, seed, noise_scale, n, mean, saturated, counters) -> bytes:
    """The file image for a sketch state (io.cpp:187-210)."""
    c = np.asarray(counters, dtype=np.uint64)
    if c.size != num_tables << k_bits:
        raise ace.ContractViolation("ACE1: counter payload does not match L * 2^K")
    head = _HDR.pack(MAGIC, dim, k_bits, num_tables, width, seed, float(noise_scale), n, float(mean),
                     1 if saturated else 0)
    body = c.astype("<u2" if width == 16 else "<u4").tobytes()
    return head + body


def parse_ace1(data: bytes):
    """(header dict, counters uint64) with the reference loader's checks
    (io.cpp:213-244): bad magic / bad width / truncation -> DataError."""
    if len(data) < 4 or data[:4] != MAGIC:
        raise ace.DataError("bad magic in sketch file")
    if len(data) < _HDR.size:
        raise ace.DataError("sketch file truncated")
    magic, dim, k, l, width, seed, noise, n, mean, sat = _HDR.unpack_from(data, 0)
    if width not in (16, 32):
        raise ace.DataError(f"sketch file counter width must be 16 or 32, got {width}")
    # the reference constructs the family (validating the configuration) first
    cfg = ace.SrpConfig(dim=dim, k_bits=k, num_tables=l, seed=seed, noise_scale=noise)
    ace.check_srp_config(cfg)
    total = l << k
    esz = 2 if width == 16 else 4
    if len(data) < _HDR.size + total * esz:
        raise ace.DataError("sketch file truncated")
    counters = np.frombuffer(data, dtype="<u2" if width == 16 else "<u4", count=total,
                             offset=_HDR.size).astype(np.uint64)
    return dict(cfg=cfg, width=width, n=n, mean=mean, saturated=bool(sat)), counters


def save_sketch(sketch: "ace.AceSketch", path) -> None:
    """ace::io::save_sketch."""
    cfg = sketch.family().config()
    width = 16 if sketch.counter_width() == ace.CounterWidth.k16 else 32
    img = ace1_bytes(cfg.dim, cfg.k_bits, cfg.num_tables, width, cfg.seed, cfg.noise_scale, sketch.size(),
                     sketch.mean(), sketch.saturated(), sketch.counters_flat())
    try:
        with open(path, "wb") as f:
            f.write(img)
    except OSError as e:
        raise ace.DataError(f"cannot open sketch file for write: {path}") from e


def load_sketch(path) -> "ace.AceSketch":
    """ace::io::load_sketch: restores counters, n, mean (reported exactly until
    the next update) and the saturation flag on the device."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise ace.DataError(f"cannot open sketch file: {path}") from e
    h, counters = parse_ace1(data)
    fam = ace.SrpFamily(h["cfg"])
    width = ace.CounterWidth.k16 if h["width"] == 16 else ace.CounterWidth.k32
    return ace.AceSketch.restore(fam, width, counters, h["n"], h["mean"], h["saturated"])


def load_dataset(path, label_column=None) -> "ace.Dataset":
    """ace::io::load_dataset: header auto-detected, optional 0/1 label column
    (negative counts from the end), all-zero rows rejected (DataError)."""
    vals, labs = C.c_void_p(), C.c_void_p()
    rows, cols = C.c_uint64(), C.c_uint64()
    rc = N.host().ace_load_dataset_csv(str(path).encode(), int(label_column is not None),
                                       int(label_column or 0), C.byref(vals), C.byref(rows), C.byref(cols),
                                       C.byref(labs))
    if rc != 0:
        msg = N.host().ace_host_last_error().decode()
        raise (ace.DataError if rc == N.ACE_E_DATA else ace.ContractViolation)(msg)
    try:
        n, d = rows.value, cols.value
        values = np.ctypeslib.as_array(C.cast(vals, C.POINTER(C.c_double)), shape=(n * d,)).copy().reshape(n, d)
        labels = None
        if labs.value:
            labels = np.ctypeslib.as_array(C.cast(labs, C.POINTER(C.c_uint8)), shape=(n,)).copy()
    finally:
        N.host().ace_free(vals)
        if labs.value:
            N.host().ace_free(labs)
    return ace.Dataset(values=values, labels=labels, name=str(path))
