"""The C-ABI library: it loads without a GPU and exports every entry point
include/dfuse_cuda.h declares; a context cannot be created without an sm_100
device (no CPU fallback). CPU only: no compute call is made here."""
import ctypes as C
import os
import re

import pytest

from paper_2207_12244_b200 import _ffi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dfuse_cuda.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dfuse_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared()
    for n in ("dfuse_texture_mask", "dfuse_search_depth", "dfuse_update_semidense",
              "dfuse_stereo_update", "dfuse_assemble_normal_equations", "dfuse_total_cost",
              "dfuse_cost_gradient", "dfuse_stencil_apply", "dfuse_solve_depth_step",
              "dfuse_solve_scale_step", "dfuse_optimize", "dfuse_kf_create",
              "dfuse_kf_process_frame", "dfuse_make_epipolar_geometry", "dfuse_stereo_scan",
              "dfuse_search_depth_gen", "dfuse_bkf_connect"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = api.lib()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_layouts_match_header():
    # sizes the C side relies on (112-byte EpipolarObservation, semidense.hpp:38-44)
    assert C.sizeof(_ffi.ObsC) == 112
    assert C.sizeof(_ffi.EpiGeom) == 15 * 8 + 40
    assert C.sizeof(_ffi.RobustCfgC) == 4 * 8 + 4 * 4
    assert C.sizeof(_ffi.SolverStatsC) == 16 + 512 * 4 + 2 * 512 * 8


def test_error_names_follow_reference_enum():
    lib = api.lib()
    assert lib.dfuse_err_name(0) == b"Ok"
    for i, name in enumerate(_ffi.ERR_NAMES):
        assert lib.dfuse_err_name(i + 1).decode() == name
    assert lib.dfuse_abi_version() == 1


def test_geometry_is_host_code_and_matches_oracle(orc):
    import numpy as np

    from paper_2207_12244_b200 import synth

    lib = api.lib()
    b = _ffi.Bindings(lib, "dfuse_", C.c_void_p(1), "cuda-host")  # geometry takes no ctx
    spec = synth.CONFIGS["C2"]
    rng = np.random.default_rng(3)
    for _ in range(20):
        q, t = synth.random_pose(spec, rng)
        assert bytes(b.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t,
                                              spec.camera())) == bytes(
            orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera()))


def test_no_context_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    rc = api.lib().dfuse_ctx_create(0, C.byref(h))
    assert rc == _ffi.E_CUDA and not h.value
