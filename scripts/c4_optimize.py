"""Profiling driver: one optimize() on a 3840x2160 random problem (the C4
raster; the streaming PCG path), fixed effort: GN steps from argv[1]
(default 5), 5 PCG iterations each."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests"))
from helpers import make_random_problem  # noqa: E402
from paper_2207_12244_b200 import api  # noqa: E402
from paper_2207_12244_b200._ffi import RobustConfig  # noqa: E402

gn = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = api.context(0)
st, semi, pred = make_random_problem(4, 3840, 2160, outlier_fraction=0.05)
cfg = RobustConfig(gn_iterations=gn, cg_tol=0.0, cg_max_iters=5)
for rep in range(2):
    t0 = time.perf_counter()
    out, stats = ctx.api.optimize(st, semi, pred, cfg, with_stats=True)
    print(f"optimize gn={gn}: {1e3 * (time.perf_counter() - t0):.1f} ms (host, incl. copies) "
          f"pcg {stats.pcg_total}", file=sys.stderr)
