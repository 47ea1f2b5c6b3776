"""Scoring oracle, CPU only: the C restatement of
pct_within_10 / median_abs_rel / export_depth_image's quantisation against
the reference build's own eval.hpp (oracle/_ref, OpenCV calls stood in by
oracle/compat_cv), and the reference's eval KATs (test_eval.cpp:21-110)."""
import ctypes as C

import numpy as np
import pytest

from paper_2207_12244_b200._ffi import ERR_NAMES

P = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data_as(P)


def orc_pct(orc, est, gt, gv, ev=None):
    out = C.c_double(0)
    rc = orc.lib.orc_pct_within_10(C.c_long(est.size), _p(est), _p(ev), _p(gt), _p(gv),
                                   C.byref(out))
    return rc, out.value


def ref_pct(ref, est, gt, gv, ev=None):
    out = C.c_double(0)
    h, w = est.shape
    rc = ref.lib.ref_pct_within_10(w, h, _p(est), _p(ev), _p(gt), _p(gv), C.byref(out))
    return rc, out.value


def orc_med(orc, est, gt, gv, ev=None):
    orc.lib.orc_median_abs_rel.restype = C.c_double
    return orc.lib.orc_median_abs_rel(C.c_long(est.size), _p(est), _p(ev), _p(gt), _p(gv))


def ref_med(ref, est, gt, gv, ev=None):
    out = C.c_double(0)
    h, w = est.shape
    assert ref.lib.ref_median_abs_rel(w, h, _p(est), _p(ev), _p(gt), _p(gv), C.byref(out)) == 0
    return out.value


def random_case(seed, h, w, holes=0.2, undefined=0.1):
    rng = np.random.default_rng(seed)
    gt = rng.uniform(0.5, 5.0, (h, w))
    est = gt * rng.uniform(0.8, 1.25, (h, w))
    edge = rng.uniform(size=(h, w)) < 0.05
    est[edge] = gt[edge] * 1.10  # exactly-10% ratios (eval.hpp:27-29)
    gv = (rng.uniform(size=(h, w)) >= holes).astype(np.uint8)
    ev = (rng.uniform(size=(h, w)) >= undefined).astype(np.uint8)
    return est, gt, gv, ev


def ones(w):
    return np.ones((1, w)), np.ones((1, w), np.uint8)


def test_reference_eval_kats(orc):
    gt, gv = ones(3)  # test_eval.cpp:21-32
    est = np.ones((1, 3))
    assert orc_pct(orc, est, gt, gv)[1] == 100.0
    est[0, 1], est[0, 2] = 1.05, 1.2
    assert abs(orc_pct(orc, est, gt, gv)[1] - 200.0 / 3.0) < 1e-9
    assert orc_pct(orc, np.full((1, 3), 1.11), gt, gv)[1] == 0.0
    gt, gv = ones(4)  # test_eval.cpp:34-46
    gt[0, 1:] = [2.0, 0.37, 5.5]
    assert orc_pct(orc, 1.10 * gt, gt, gv)[1] == 100.0
    assert orc_pct(orc, 1.101 * gt, gt, gv)[1] == 0.0
    gt, gv = ones(4)  # test_eval.cpp:48-58
    ev = np.array([[1, 1, 1, 0]], np.uint8)
    assert orc_pct(orc, np.ones((1, 4)), gt, gv, ev)[1] == 75.0
    gv[0, 3] = 0
    assert orc_pct(orc, np.ones((1, 4)), gt, gv, ev)[1] == 100.0
    gt, gv = ones(3)  # test_eval.cpp:60-74
    rc, _ = orc_pct(orc, np.ones((1, 3)), gt, np.zeros((1, 3), np.uint8))
    assert ERR_NAMES[rc - 1] == "NoValidGroundTruth"


@pytest.mark.parametrize("seed,shape", [(1, (1, 1)), (2, (7, 5)), (3, (48, 64)), (4, (120, 160))])
def test_oracle_is_the_reference(orc, ref, seed, shape):
    est, gt, gv, ev = random_case(seed, *shape)
    for e in (None, ev):
        assert orc_pct(orc, est, gt, gv, e) == ref_pct(ref, est, gt, gv, e)
        assert orc_med(orc, est, gt, gv, e) == ref_med(ref, est, gt, gv, e)
    rc_o, _ = orc_pct(orc, est, gt, np.zeros_like(gv))
    rc_r, _ = ref_pct(ref, est, gt, np.zeros_like(gv))
    assert rc_o == rc_r != 0
    assert orc_med(orc, est, gt, np.zeros_like(gv)) == ref_med(ref, est, gt, np.zeros_like(gv))


def test_export_quantisation_is_the_reference(orc, ref):
    rng = np.random.default_rng(9)
    ld = rng.uniform(-8.0, 3.5, (31, 17))  # exp up to ~33 m: saturates at 5000 units/m
    ld[0, :4] = [np.log(0.5 / 5000.0), np.log(1.5 / 5000.0), -50.0, 20.0]  # .5 ties, 0, clamp
    for scale in (5000.0, 1000.0, 1.0):
        a = np.zeros(ld.shape, np.uint16)
        b = np.zeros(ld.shape, np.uint16)
        orc.lib.orc_export_depth_u16(C.c_long(ld.size), _p(ld), C.c_double(scale), _p(a))
        assert ref.lib.ref_export_depth_u16(17, 31, _p(ld), C.c_double(scale), _p(b)) == 0
        assert np.array_equal(a, b)
