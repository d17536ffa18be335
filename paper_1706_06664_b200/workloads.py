"""The five BASELINE.json configurations as seeded synthetic workloads.

Rows come from libace_datagen.so (csrc/datagen_core.h): bit-identical on the
host and on the device, so full-size inputs are generated in HBM while the CPU
oracle regenerates any row range on the host.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class Workload:
    cfg: int
    name: str
    n: int
    dim: int
    k_bits: int
    num_tables: int
    mode: str            # "batch" (insert all, then detect) or "stream"
    batch: int = 0       # stream batch size
    alpha: float = 1.0   # stream: flag score <= mean - alpha
    data_seed: int = 20261019
    w_seed: int = 1      # SRP seed (CLI examples use --seed 1)


CONFIGS = {
    1: Workload(1, "clusters8_d40", 100_000, 40, 15, 50, "batch"),
    2: Workload(2, "kdd_mixed_d120", 500_000, 120, 15, 50, "batch"),
    3: Workload(3, "iid_d128_k16_l100", 10_000_000, 128, 16, 100, "batch"),
    4: Workload(4, "lowrank_d4096_k18_l64", 1_000_000, 4096, 18, 64, "batch"),
    5: Workload(5, "drift_stream_d64", 100_000_000, 64, 15, 50, "stream", batch=65_536),
}


def host_rows(cfg: int, row0: int, nrows: int, seed: int | None = None, threads: int | None = None):
    """(X float32 [nrows, dim], labels uint8 [nrows]) generated on the host."""
    w = CONFIGS[cfg]
    seed = w.data_seed if seed is None else seed
    x = np.empty((nrows, w.dim), dtype=np.float32)
    lab = np.empty(nrows, dtype=np.uint8)
    th = threads or max(1, os.cpu_count() or 1)
    if nrows and N.datagen().ace_datagen_host(cfg, seed, row0, nrows, x.ctypes.data,
                                              lab.ctypes.data, th) != 0:
        raise RuntimeError("datagen failed")
    return x, lab


def device_rows(cfg: int, row0: int, nrows: int, out_ptr: int, labels_ptr: int | None = None,
                seed: int | None = None, stream: int | None = None) -> None:
    """Same rows generated straight into device memory (out_ptr: float32 CUDA)."""
    w = CONFIGS[cfg]
    seed = w.data_seed if seed is None else seed
    if nrows and N.datagen().ace_datagen_device(cfg, seed, row0, nrows, out_ptr, labels_ptr,
                                                stream) != 0:
        raise RuntimeError("device datagen failed")
