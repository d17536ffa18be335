"""CPU tests of the boundary: every symbol declared in include/ace_b200.h is
exported by libace_dev.so; the C++ drop-in and generator libraries load;
without a GPU the library reports that instead of computing on the CPU."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1706_06664_b200 import _native as N
from paper_1706_06664_b200 import ace

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "ace_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ace_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(str(N.LIB_DIR / "libace_dev.so"))
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes table covers exactly the header
    assert sorted(N.ABI) == syms


def test_dropin_library_loads():
    lib = N.host()
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "ace_host.h").read_text(), flags=re.S)
    host_syms = sorted(set(re.findall(r"\b(ace_[a-z0-9_]+)\s*\(", text)))
    assert host_syms and all(hasattr(lib, s) for s in host_syms)
    assert sorted(N.HOST_ABI) == host_syms
    # C++ API symbols of the drop-in (mangled) are present
    names = (N.LIB_DIR / "libace.so").read_bytes()
    for frag in (b"SrpFamily", b"AceSketch", b"detect_batch", b"detect_stream", b"build_sketch"):
        assert frag in names


def test_status_codes_map_to_reference_exceptions():
    assert ace._STATUS[N.ACE_E_CONTRACT] is ace.ContractViolation
    assert issubclass(ace.ContractViolation, ValueError)  # std::invalid_argument
    assert ace._STATUS[N.ACE_E_INCONSISTENT] is ace.InconsistentDelete
    assert ace._STATUS[N.ACE_E_UNSUPPORTED] is ace.UnsupportedOperation


def test_config_validation_on_host():
    for bad in [dict(dim=0), dict(dim=2, k_bits=0), dict(dim=2, k_bits=31), dict(dim=2, num_tables=0),
                dict(dim=2, noise_scale=-1.0)]:
        with pytest.raises(ace.ContractViolation):
            ace.SrpFamily(ace.SrpConfig(**bad))


@pytest.mark.skipif(N.dev().ace_device_available(), reason="GPU present")
def test_no_cpu_fallback_without_gpu():
    fam = ace.SrpFamily(ace.SrpConfig(dim=4, k_bits=3, num_tables=2, seed=1))
    with pytest.raises(ace.CudaError):
        fam.buckets(np.ones((2, 4), dtype=np.float32))
