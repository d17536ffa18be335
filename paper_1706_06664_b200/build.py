"""Build the native libraries in-tree (paper_1706_06664_b200/lib/).

  libace_dev.so      CUDA kernels + C ABI (include/ace_b200.h), sm_100a
  libace.so          C++ drop-in API (include/ace/*.hpp) over libace_dev.so
  libace_datagen.so  synthetic workload generators (host + device)

and the parity checkers under oracle/ (test infrastructure; see oracle/Makefile).
Run: python -m paper_1706_06664_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
INC = ROOT / "include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found")


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_dev(force: bool = False) -> Path:
    out = LIB / "libace_dev.so"
    srcs = [CSRC / "ace_api.cu", CSRC / "ace_kernels.cu", CSRC / "ace_hash_tc.cu", CSRC / "ace_hash_tck.cu"]
    deps = srcs + list(CSRC.glob("*.cuh")) + [INC / "ace_b200.h"]
    if force or _stale(out, deps):
        _run([_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-shared", f"-I{INC}", "-o", str(out), *map(str, srcs)])
    return out


def build_host(force: bool = False) -> Path:
    out = LIB / "libace.so"
    src = CSRC / "ace_host.cpp"
    deps = [src, INC / "ace_b200.h", *INC.glob("ace/*.hpp"), LIB / "libace_dev.so"]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wl,-Bsymbolic", f"-I{INC}", "-o",
              str(out), str(src), f"-L{LIB}", "-lace_dev", "-Wl,-rpath,$ORIGIN"])
    return out


def build_datagen(force: bool = False) -> Path:
    out = LIB / "libace_datagen.so"
    srcs = [CSRC / "datagen.cu", CSRC / "datagen_core.h"]
    if force or _stale(out, srcs):
        _run([_nvcc(), *ARCH, "-O3", "--fmad=false", "-Xcompiler", "-ffp-contract=off",
              "-Xcompiler", "-fPIC", "-shared", "-o", str(out), str(CSRC / "datagen.cu")])
    return out


def build_cpp_test(force: bool = False) -> Path:
    """The drop-in C++ test program (tests/cpp/test_dropin.cpp) against
    include/ace/*.hpp + libace.so; run on the GPU by tests/test_cpp_dropin_gpu.py."""
    out = LIB / "ace_dropin_test"
    src = ROOT / "tests" / "cpp" / "test_dropin.cpp"
    if src.exists() and (force or _stale(out, [src, LIB / "libace.so", *INC.glob("ace/*.hpp")])):
        _run(["g++", "-std=c++20", "-O2", f"-I{INC}", "-o", str(out), str(src), f"-L{LIB}", "-lace",
              "-lace_dev", "-Wl,-rpath,$ORIGIN"])
    return out


def build_point_bench(force: bool = False) -> Path:
    """The per-point API timing program (tests/cpp/point_bench.cpp) against
    include/ace/*.hpp + libace.so; driven by bench.py --api point."""
    out = LIB / "ace_point_bench"
    src = ROOT / "tests" / "cpp" / "point_bench.cpp"
    if src.exists() and (force or _stale(out, [src, LIB / "libace.so", *INC.glob("ace/*.hpp")])):
        _run(["g++", "-std=c++20", "-O2", f"-I{INC}", "-o", str(out), str(src), f"-L{LIB}", "-lace",
              "-lace_dev", "-Wl,-rpath,$ORIGIN"])
    return out


def build_oracle() -> None:
    """C restatement always; the reference build only where its sources exist."""
    _run(["make", "-C", str(ROOT / "oracle"), "oracle"])
    if Path("/root/reference/proj/src/srp.cpp").exists():
        _run(["make", "-C", str(ROOT / "oracle"), "ref"])


def build_all(force: bool = False) -> None:
    LIB.mkdir(exist_ok=True)
    build_dev(force)
    build_host(force)
    build_datagen(force)
    build_cpp_test(force)
    build_point_bench(force)
    build_oracle()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
