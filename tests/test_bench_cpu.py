"""bench.py host logic on CPU: the step schedule, the shared config dict of
the two arms, C3 keyframe sharding, and `--gpus N` failing loudly when N
GPUs are not visible."""
import os
import subprocess
import sys

import bench
from paper_2207_12244_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _Args:
    seed = 0
    keyframes = 0
    regime = "defaults"
    bands = 0


def test_schedule_walks_each_keyframe_in_order():
    s = bench.schedule(3, 10, 35)
    assert s[:10] == [(0, k) for k in range(10)]
    assert s[10:20] == [(1, k) for k in range(10)]
    assert s[30:] == [(0, k) for k in range(5)]  # wraps round the rank's keyframes


def test_c3_keyframes_shard_mod_n_and_cover_the_batch():
    spec = synth.CONFIGS["C3"]
    for n in (1, 2, 4, 8):
        owned = [bench.keyframe_ids(_Args, spec, n, r) for r in range(n)]
        assert sorted(k for ks in owned for k in ks) == list(range(64))
        for r, ks in enumerate(owned):
            assert all(k % n == r for k in ks)
    # distinct seeds per keyframe; C2 streams are per rank
    assert len({bench.keyframe_seed(_Args, spec, k, False) for k in range(64)}) == 64
    assert bench.keyframe_ids(_Args, synth.CONFIGS["C2"], 4, 3) == [3]


def test_both_arms_print_the_same_config_dict():
    spec = synth.CONFIGS["C2"]
    cfg = bench.solver_cfg(spec, "defaults")
    a = bench.config_dict(_Args, spec, cfg, 1, False, 1)
    b = bench.config_dict(_Args, spec, cfg, 1, False, 1)
    assert a == b and a["gn_iterations"] == 10 and a["cg_max_iters"] == 200
    f = bench.solver_cfg(spec, "fixed")
    assert f.cg_tol == 0.0 and f.cg_max_iters == 5


def test_gpus_n_without_gpus_fails_loudly():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1"], capture_output=True, text=True, timeout=300,
                       env={k: v for k, v in os.environ.items() if k != "WORLD_SIZE"})
    assert r.returncode != 0
    assert "GPU(s) visible" in r.stderr
