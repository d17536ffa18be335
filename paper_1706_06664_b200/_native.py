"""ctypes bindings of the native libraries (include/ace_b200.h).

Loading fails loudly: there is no Python or CPU fallback for any hot-path
operation.  Libraries live in-tree under paper_1706_06664_b200/lib/ (built by
paper_1706_06664_b200.build / __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"

ACE_OK, ACE_E_CONTRACT, ACE_E_UNSUPPORTED, ACE_E_INCONSISTENT, ACE_E_DATA, ACE_E_CUDA, ACE_E_NOMEM = range(7)
ACE_F32, ACE_F64 = 0, 1
ACE_HOST, ACE_DEVICE = 0, 1
ACE_OPT_H2D_CHUNKS, ACE_OPT_DEFER_INSERT, ACE_OPT_STREAM_GROUP, ACE_OPT_STREAM_PIPE = 1, 2, 3, 4


class AceHashStats(C.Structure):
    _fields_ = [("projections", C.c_uint64), ("rechecked", C.c_uint64), ("flipped", C.c_uint64),
                ("near_ties", C.c_uint64)]


class AceBatchReport(C.Structure):
    _fields_ = [
        ("score_mean", C.c_double),
        ("score_stddev", C.c_double),
        ("threshold", C.c_double),
        ("reported", C.c_uint64),
        ("ambiguous", C.c_uint64),
        ("replayed", C.c_int),
        ("elapsed_seconds", C.c_double),
    ]


class AceStreamReport(C.Structure):
    _fields_ = [
        ("mean_before", C.c_double),
        ("cut", C.c_double),
        ("reported", C.c_uint64),
        ("ambiguous", C.c_uint64),
    ]


_vp, _u64, _u32, _i, _d = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
_P = C.POINTER

# name -> (restype, argtypes) for every symbol declared in include/ace_b200.h
ABI = {
    "ace_last_error": (C.c_char_p, []),
    "ace_version": (C.c_char_p, []),
    "ace_device_available": (_i, []),
    "ace_kernel_launches": (_u64, []),
    "ace_family_create": (_i, [_u64, _u32, _u32, _d, _vp, _P(_vp)]),
    "ace_family_destroy": (_i, [_vp]),
    "ace_family_set_kernel": (_i, [_vp, _i]),
    "ace_family_kernel": (_i, [_vp]),
    "ace_family_buckets": (_i, [_vp, _vp, _i, _u64, _u64, _i, _vp, _i, _P(AceHashStats)]),
    "ace_sketch_create": (_i, [_vp, _u32, _P(_vp)]),
    "ace_sketch_clone": (_i, [_vp, _P(_vp)]),
    "ace_sketch_destroy": (_i, [_vp]),
    "ace_sketch_reset": (_i, [_vp]),
    "ace_sketch_set_stream": (_i, [_vp, _vp]),
    "ace_sketch_set_option": (_i, [_vp, _i, C.c_int64]),
    "ace_sketch_insert": (_i, [_vp, _vp, _i, _u64, _u64, _i, _P(AceHashStats)]),
    "ace_sketch_remove": (_i, [_vp, _vp, _i, _u64, _u64, _i, _P(AceHashStats)]),
    "ace_sketch_score": (_i, [_vp, _vp, _i, _u64, _u64, _i, _vp, _vp, _i, _P(AceHashStats)]),
    "ace_sketch_detect_batch": (_i, [_vp, _vp, _i, _u64, _u64, _i, _vp, _vp, _i,
                                     _P(AceBatchReport), _P(AceHashStats)]),
    "ace_sketch_build_detect": (_i, [_vp, _vp, _i, _u64, _u64, _i, _vp, _vp, _i,
                                     _P(AceBatchReport), _P(AceHashStats)]),
    "ace_sketch_stream_batch": (_i, [_vp, _vp, _i, _u64, _u64, _i, _d, _vp, _vp, _i,
                                     _P(AceStreamReport), _P(AceHashStats)]),
    "ace_sketch_stream_run": (_i, [_vp, _vp, _i, _u64, _u64, _i, _u64, _d, _vp, _i, _vp,
                                   _P(AceStreamReport), _P(AceHashStats)]),
    "ace_sketch_detect_stream": (_i, [_vp, _vp, _i, _u64, _u64, _i, _d, _vp, _vp]),
    "ace_sketch_counter": (_i, [_vp, _u32, _u64, _P(_u64)]),
    "ace_sketch_info": (_i, [_vp, _P(_u64), _P(_d), _P(_i)]),
    "ace_sketch_counters": (_i, [_vp, _vp]),
    "ace_sketch_counters_u32": (_i, [_vp, _vp, _i]),
    "ace_sketch_restore": (_i, [_vp, _vp, _u64, _u64, _d, _i]),
    "ace_sketch_device_counters": (_vp, [_vp]),
    "ace_sketch_set_timing": (_i, [_vp, _i]),
    "ace_sketch_timings": (_i, [_vp, _vp]),
}

ABI.update({
    "ace_family_buckets_noisy": (_i, [_vp, _vp, _i, _u64, _u64, _i, _u32, _u32, _u32, _u32, _vp, _i, _vp, _i]),
    "ace_sketch_insert_ids": (_i, [_vp, _vp, _u64, _i]),
    "ace_sketch_score_ids": (_i, [_vp, _vp, _u64, _i, _vp, _vp, _i]),
})

HOST_ABI = {
    "ace_generate_directions": (_i, [_u64, _u64, _u32, _u32, _vp]),
    "ace_load_dataset_csv": (_i, [C.c_char_p, _i, _i, _vp, _vp, _vp, _vp]),
    "ace_host_last_error": (C.c_char_p, []),
    "ace_free": (None, [_vp]),
    "ace_noise_terms": (_i, [_u64, _u64, _u64, _d, _vp]),
}

DATAGEN_ABI = {
    "ace_datagen_dim": (_u64, [_i]),
    "ace_datagen_host": (_i, [_i, _u64, _u64, _u64, _vp, _vp, _i]),
    "ace_datagen_device": (_i, [_i, _u64, _u64, _u64, _vp, _vp, _vp]),
}


def _load(name: str, table: dict) -> C.CDLL:
    path = LIB_DIR / name
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build the native libraries first "
            "(python -m paper_1706_06664_b200.build); there is no fallback path")
    lib = C.CDLL(str(path), mode=C.RTLD_LOCAL)
    for sym, (res, args) in table.items():
        fn = getattr(lib, sym)
        fn.restype = res
        fn.argtypes = args
    return lib


_dev = _host = _datagen = None


def dev() -> C.CDLL:
    global _dev
    if _dev is None:
        _dev = _load("libace_dev.so", ABI)
    return _dev


def host() -> C.CDLL:
    global _host
    if _host is None:
        dev()
        _host = _load("libace.so", HOST_ABI)
    return _host


def datagen() -> C.CDLL:
    global _datagen
    if _datagen is None:
        _datagen = _load("libace_datagen.so", DATAGEN_ABI)
    return _datagen


def last_error() -> str:
    msg = dev().ace_last_error()
    return msg.decode() if msg else ""
