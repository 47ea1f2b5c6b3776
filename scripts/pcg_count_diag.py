"""Diagnostics: per-GN PCG counts of the GPU session against the oracle on a
free-running sequence (C1 by default), and against the oracle re-seeded with
the GPU's input state each frame.
usage: python scripts/pcg_count_diag.py [config] [frames] [solver path]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2207_12244_b200 import api, synth  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig, SemiDenseMap, init_state  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = synth.CONFIGS[name]
seq = synth.make_sequence(spec, 0, frames=nf)
orc = oracle.oracle()
cfg = RobustConfig(gn_iterations=spec.gn_iterations)
ctx = api.context(0)
ctx.set_solver_path(sys.argv[3] if len(sys.argv) > 3 else "auto")
kf = api.Keyframe(ctx, spec.camera(), seq.I0, seq.pred, 0.02)
mask = orc.texture_mask(seq.I0, 0.02)
semi = SemiDenseMap.empty(spec.width, spec.height)
st_free = init_state(seq.pred)
for k, (q, t, I1) in enumerate(seq.frames):
    g = orc.make_epipolar_geometry(synth.IDENTITY_Q, np.zeros(3), q, t, spec.camera())
    before, _, _ = kf.download()
    res = kf.process_frame(g, I1, spec.search, cfg, "full")
    semi = orc.stereo_update(g, seq.I0, I1, mask, semi, spec.search, want_obs=False).semi
    st_free, so_free = orc.optimize(st_free, semi, seq.pred, cfg, with_stats=True)
    st_seed, so_seed = orc.optimize(before, semi, seq.pred, cfg, with_stats=True)
    gpu = [res.stats.pcg_iters[i] for i in range(res.stats.gn_done)]
    free = list(so_free.pcg_iters[:so_free.gn_done])
    seed = list(so_seed.pcg_iters[:so_seed.gn_done])
    dfree = [a - b for a, b in zip(gpu, free)]
    dseed = [a - b for a, b in zip(gpu, seed)]
    print(f"frame {k}: gpu {sum(gpu)} free {sum(free)} seeded {sum(seed)}; "
          f"max |d| free {max(map(abs, dfree))} seeded {max(map(abs, dseed))}")
    print("  gpu ", gpu)
    print("  free", free)
    print("  seed", seed)
