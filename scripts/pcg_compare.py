"""Diagnostics: per-phase PCG cycles (DFUSE_TRACE=1) on a random 640x480
system vs the normal equations of a real C2 keyframe update."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from helpers import make_random_problem  # noqa: E402
from paper_2207_12244_b200 import api, synth  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig, SemiDenseMap, init_state  # noqa: E402

ctx = api.context(0)
gpu = ctx.api
cfg = RobustConfig(cg_tol=0.0, cg_max_iters=200)
st, semi, pred = make_random_problem(5, 640, 480)
eq = gpu.assemble_normal_equations(st, semi, pred)
print("random system", file=sys.stderr)
gpu.solve_depth_step(eq, cfg)

spec = synth.CONFIGS["C2"]
seq = synth.make_sequence(spec, 0, frames=2)
mask = gpu.texture_mask(seq.I0, 0.02)
semi = SemiDenseMap.empty(spec.width, spec.height)
for q, t, I1 in seq.frames:
    g = gpu.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
    semi = gpu.stereo_update(g, seq.I0, I1, mask, semi, spec.search).semi
st = init_state(seq.pred)
eq = gpu.assemble_normal_equations(st, semi, seq.pred)
print("C2 system", file=sys.stderr)
gpu.solve_depth_step(eq, cfg)
print("C2 optimize", file=sys.stderr)
gpu.optimize(st, semi, seq.pred, RobustConfig())
print("C2 optimize gn=1, 200 fixed PCG iterations", file=sys.stderr)
gpu.optimize(st, semi, seq.pred, RobustConfig(gn_iterations=1, cg_tol=0.0, cg_max_iters=200))
print("C2 optimize gn=5, 40 fixed PCG iterations", file=sys.stderr)
gpu.optimize(st, semi, seq.pred, RobustConfig(gn_iterations=5, cg_tol=0.0, cg_max_iters=40))
print("standalone PCG, 40 iterations x5", file=sys.stderr)
for _ in range(5):
    gpu.solve_depth_step(eq, RobustConfig(cg_tol=0.0, cg_max_iters=40))
