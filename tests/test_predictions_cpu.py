"""Keyframe-creation inputs on the host side, CPU only:
the DFPRED writer used by the tests against the reference's own
save_predictions / load_predictions (predictions.hpp:69-145), the library's
DFPRED header checks against load_predictions' error codes on the same
corrupted files (the reference's own KATs, test_predictions.cpp:38-101), and
the oracle's focal_adjust / median_predicted_depth against the reference."""
import ctypes as C
import math
import struct

import numpy as np
import pytest

from paper_2207_12244_b200 import api, synth
from paper_2207_12244_b200._ffi import DfuseError, ERR_NAMES
from helpers import synth_oracle


def smooth_gt(w, h, phase=1.3):  # test_predictions.cpp:15-24 (fixed phase)
    x = np.arange(w)[None, :]
    y = np.arange(h)[:, None]
    return 2.0 + 0.8 * np.sin(0.13 * x + phase) + 0.5 * np.cos(0.21 * y)


def planes_of(p):
    return np.concatenate([a.ravel() for a in p.planes()])


def ref_save(ref, tmp_path, p, name="p.dfpred"):
    h, w = p.log_depth.shape
    path = str(tmp_path / name)
    flat = np.ascontiguousarray(planes_of(p))
    assert ref.lib.ref_save_predictions(path.encode(), w, h, flat.ctypes.data_as(C.c_void_p),
                                        C.c_double(p.source_focal)) == 0
    return path


def ref_load(ref, path, w, h):
    out = np.zeros(6 * w * h)
    f = C.c_double(0)
    msg = C.create_string_buffer(512)
    rc = ref.lib.ref_load_predictions(path.encode(), w, h, out.ctypes.data_as(C.c_void_p),
                                      C.byref(f), msg, 512)
    return rc, out, f.value, msg.value.decode()


def test_writer_matches_reference_save(ref, tmp_path):
    p = synth_oracle(smooth_gt(31, 17), 0.25, 0.04, 42, 210.5)
    ours = synth.to_dfpred(p, 210.5)
    theirs = open(ref_save(ref, tmp_path, p), "rb").read()
    assert ours == theirs  # byte for byte (test_predictions.cpp:38-61)
    assert api.dfpred_header(ours) == (31, 17, 210.5)
    path = tmp_path / "ours.dfpred"
    path.write_bytes(ours)
    rc, planes, f, _ = ref_load(ref, str(path), 31, 17)
    assert rc == 0 and f == 210.5
    assert np.array_equal(planes, planes_of(p))


def corruptions(p):
    good = synth.to_dfpred(p, 200.0)
    n = p.log_depth.size
    yield "bad magic", b"XFPR" + good[4:]
    yield "version", good[:4] + struct.pack("<I", 2) + good[8:]
    yield "zero width", good[:8] + struct.pack("<I", 0) + good[12:]
    yield "huge height", good[:12] + struct.pack("<I", 70000) + good[16:]
    yield "channels", good[:16] + struct.pack("<I", 5) + good[20:]
    yield "zero focal", good[:20] + struct.pack("<I", 0) + good[24:]
    yield "short header", good[:17]


def test_header_checks_match_reference(ref, tmp_path):
    p = synth_oracle(smooth_gt(8, 6), 0.1, 0.02, 3, 200.0)
    for what, data in corruptions(p):
        path = tmp_path / "c.dfpred"
        path.write_bytes(data)
        rc_ref, _, _, _ = ref_load(ref, str(path), 8, 6)
        assert rc_ref != 0, what
        with pytest.raises(DfuseError) as e:
            api.dfpred_header(data)
        assert e.value.code == ERR_NAMES[rc_ref - 1], what


def test_reference_corruption_kats_on_the_reference(ref, tmp_path):
    """test_predictions.cpp:63-101 replayed on the reference build: the codes
    and message contents the device ingest must reproduce (test_gpu_keyframe)."""
    p = synth_oracle(smooth_gt(8, 6), 0.1, 0.02, 3, 200.0)
    good = bytearray(synth.to_dfpred(p, 200.0))
    n = 8 * 6
    off = 24 + n * 4 + 5 * 4  # log_depth_var[5]
    bad = bytes(good[:off]) + struct.pack("<f", 0.0) + bytes(good[off + 4:])
    path = tmp_path / "v.dfpred"
    path.write_bytes(bad)
    rc, _, _, msg = ref_load(ref, str(path), 8, 6)
    assert ERR_NAMES[rc - 1] == "NonPositiveVariance"
    assert "log_depth_var" in msg and str(off) in msg
    path.write_bytes(bytes(good[:24 + 3 * n * 4 + 10]))  # inside grad_x_var
    rc, _, _, msg = ref_load(ref, str(path), 8, 6)
    assert ERR_NAMES[rc - 1] == "TruncatedFile" and "grad_x_var" in msg


@pytest.mark.parametrize("src,test", [(300.0, 300.0), (300.0, 600.0), (300.0, 612.0),
                                      (525.0, 262.5)])
def test_focal_adjust_oracle_is_the_reference(orc, ref, src, test):
    p = synth_oracle(smooth_gt(12, 9), 0.2, 0.05, 5, src)
    a = np.ascontiguousarray(p.log_depth.copy())
    b = a.copy()
    assert orc.lib.orc_focal_adjust(12, 9, a.ctypes.data_as(C.c_void_p), C.c_double(src),
                                    C.c_double(test)) == 0
    assert ref.lib.ref_focal_adjust(12, 9, b.ctypes.data_as(C.c_void_p), C.c_double(src),
                                    C.c_double(test)) == 0
    assert a.tobytes() == b.tobytes()
    if test == 600.0:  # test_predictions.cpp:103-115
        assert np.allclose(a - p.log_depth, np.log(2.0), rtol=1e-12, atol=0)
    for bad in (0.0, -2.0):
        assert orc.lib.orc_focal_adjust(12, 9, a.ctypes.data_as(C.c_void_p), C.c_double(src),
                                        C.c_double(bad)) == ERR_NAMES.index("NonPositiveFocal") + 1


def test_median_oracle(orc):
    orc.lib.orc_median_predicted_depth.restype = C.c_double
    rng = np.random.default_rng(7)
    for n in (1, 2, 7, 640 * 48):
        v = rng.normal(0.3, 0.5, n)
        got = orc.lib.orc_median_predicted_depth(v.ctypes.data_as(C.c_void_p), C.c_long(n))
        assert got == math.exp(np.partition(v, n // 2)[n // 2])  # glibc exp, as std::exp
