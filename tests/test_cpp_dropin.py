"""The C++ drop-in (include/wallace_b200.hpp) builds against the C-ABI, and on
a GPU passes the reference's generator test cases bit-for-bit against the
reference library (tests/cpp/test_dropin.cpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def _build():
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmaxent_ref.so")):
        pytest.skip("oracle/_ref not built")
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return os.path.join(CPP, "test_dropin")


def test_cpp_dropin_builds():
    assert os.access(_build(), os.X_OK)


@pytest.mark.gpu
def test_cpp_dropin_reference_cases(cuda):
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
