"""TEST INFRASTRUCTURE ONLY -- the parity checkers (see dfuse_oracle.h).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. The product package
(paper_2207_12244_b200) never imports it.

    oracle()     plain-C restatement (liborc.so), Bindings with prefix orc_
    reference()  the reference's own headers compiled unmodified
                 (_ref/libdfuse_ref.so), Bindings with prefix ref_
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libdfuse_ref.so")

_cache = {}


def build(force: bool = False) -> None:
    """make -C oracle (liborc.so always; _ref only where /root/reference exists)."""
    if force or not os.path.exists(ORC_SO) or (
            os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str, prefix: str, name: str):
    from paper_2207_12244_b200._ffi import Bindings

    if path not in _cache:
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (reference sources absent here?)")
        lib = C.CDLL(path)
        _cache[path] = Bindings(lib, prefix, None, name)
    return _cache[path]


def oracle():
    return _load(ORC_SO, "orc_", "oracle")


def reference():
    return _load(REF_SO, "ref_", "reference")


def have_reference() -> bool:
    return os.path.exists(REF_SO) or os.path.isdir("/root/reference/proj")


def hypot(x: float, y: float) -> float:
    lib = oracle().lib
    f = lib.orc_hypot
    f.restype = C.c_double
    f.argtypes = [C.c_double, C.c_double]
    return f(x, y)
