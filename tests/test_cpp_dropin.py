"""The C++ drop-in headers (include/dfuse/*.hpp): they compile against the
reference's API as a C++ user would include it (CPU), and the reference's
KATs restated in tests/cpp/test_dropin.cpp pass through them on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2207_12244_b200")
OUT = os.path.join(ROOT, "build", "test_dropin")


def _build():
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "include", "compat"), SRC, "-o", OUT, "-L" + LIBDIR,
           "-ldfuse_cuda", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]


def test_dropin_headers_compile():
    _build()
    assert os.path.exists(OUT)


@pytest.mark.gpu
def test_dropin_kats_on_gpu():
    _build()
    r = subprocess.run([OUT], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
