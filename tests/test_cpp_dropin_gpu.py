"""The C++ drop-in (include/ace/*.hpp + libace.so) passes the reference's
known-answer tests restated in tests/cpp/test_dropin.cpp."""
import subprocess

import pytest

from paper_1706_06664_b200 import _native as N

pytestmark = pytest.mark.gpu


def test_cpp_dropin_kats(cuda):
    exe = N.LIB_DIR / "ace_dropin_test"
    assert exe.exists(), "built by __graft_entry__.build()"
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
