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


SCAN_SRC = os.path.join(ROOT, "tests", "cpp", "test_scan_loop.cpp")
SCAN_OUT = os.path.join(ROOT, "build", "test_scan_loop")


def _build_scan():
    os.makedirs(os.path.dirname(SCAN_OUT), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-fopenmp", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(ROOT, "include", "compat"), SCAN_SRC, "-o", SCAN_OUT,
           "-L" + LIBDIR, "-ldfuse_cuda", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]


def test_scan_loop_compiles():
    _build_scan()
    assert os.path.exists(SCAN_OUT)


@pytest.mark.gpu
def test_reference_scan_loop_through_dropin(tmp_path, orc):
    """The reference's stereo_scan loop (OpenMP over rows, one search_depth
    per masked pixel, pipeline.hpp:167-178) through the drop-in headers at C1:
    every frame's observations and the final semi-dense map are bit-exact
    against the oracle, the one-launch dfuse::stereo_scan returns the same
    vector, and each frame uploads its tracked image once (I0 once in all)."""
    import numpy as np

    from paper_2207_12244_b200 import synth
    from paper_2207_12244_b200._ffi import SemiDenseMap

    _build_scan()
    spec = synth.CONFIGS["C1"]
    seq = synth.make_sequence(spec, 21, frames=3)
    W, H = spec.width, spec.height
    inp = tmp_path / "scan_in.bin"
    with open(inp, "wb") as f:
        f.write(np.array([W, H, len(seq.frames)], np.int32).tobytes())
        f.write(np.array([spec.fx, spec.fy, spec.cx, spec.cy], np.float64).tobytes())
        s = spec.search
        f.write(np.array([s.min_depth, s.max_depth, s.max_rms_error], np.float64).tobytes())
        f.write(np.ascontiguousarray(seq.I0, np.float32).tobytes())
        for q, t, I1 in seq.frames:
            f.write(np.asarray(q, np.float64).tobytes() + np.asarray(t, np.float64).tobytes())
            f.write(np.ascontiguousarray(I1, np.float32).tobytes())
    outp = tmp_path / "scan_out.bin"
    env = dict(os.environ, OMP_NUM_THREADS="8")
    r = subprocess.run([SCAN_OUT, str(inp), str(outp)], capture_output=True, text=True,
                       timeout=600, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    raw = outp.read_bytes()
    nF = len(seq.frames)
    recs = np.frombuffer(raw[:16 * nF], np.int32).reshape(nF, 4)
    P = W * H
    o = 16 * nF
    depth = np.frombuffer(raw[o:o + 8 * P], np.float64)
    var = np.frombuffer(raw[o + 8 * P:o + 16 * P], np.float64)
    valid = np.frombuffer(raw[o + 16 * P:o + 17 * P], np.uint8)
    cnt = int(np.frombuffer(raw[o + 17 * P:o + 17 * P + 4], np.int32)[0])
    # the oracle pipeline: stereo_scan + update_semidense per frame
    mask = orc.texture_mask(seq.I0, 0.02)
    semi = SemiDenseMap.empty(W, H)
    for k, (q, t, I1) in enumerate(seq.frames):
        g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
        res = orc.stereo_update(g, seq.I0, I1, mask, semi, spec.search, want_obs=False)
        semi = res.semi
        n_obs, uploads, same, threads = recs[k]
        assert n_obs == res.n_obs
        assert same == 1  # one-launch scan == per-pixel loop, bit for bit
        assert uploads <= (2 if k == 0 else 1), uploads  # I1 (and I0 on the first frame)
        assert threads == 8
    assert depth.tobytes() == semi.depth.tobytes()
    assert var.tobytes() == semi.variance.tobytes()
    assert valid.tobytes() == semi.valid.tobytes()
    assert cnt == semi.inlier_count


def test_stereo_scan_template_matches_the_reference_shape():
    """dfuse::gpu::stereo_scan instantiates with types shaped like the
    reference's Keyframe / Frame / PipelineConfig (compile only)."""
    src = os.path.join(ROOT, "tests", "cpp", "test_scan_template.cpp")
    out = os.path.join(ROOT, "build", "test_scan_template")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                        "-I" + os.path.join(ROOT, "include", "compat"), src, "-o", out,
                        "-L" + LIBDIR, "-ldfuse_cuda", "-Wl,-rpath," + LIBDIR],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
