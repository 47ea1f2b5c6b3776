#!/bin/bash
# A/B of library builds on the GPU box: bench.py (C2 by default; BENCH_ARGS
# adds flags), both solver regimes in one run, twice, for every library named
# in LIBS (paths relative to the package). Prints value, fixed-effort value
# and the two stage times.
# usage: LIBS="libdfuse_old.so libdfuse_cuda.so" bash scripts/ab_bench.sh
LIBS=${LIBS:-"libdfuse_old.so libdfuse_cuda.so"}
for r in 1 2; do
  for lib in $LIBS; do
    DFUSE_LIB=$PWD/paper_2207_12244_b200/$lib timeout 300 python bench.py --no-cpu-baseline \
      --no-e2e --steps ${STEPS:-100} $BENCH_ARGS 2>&1 | tail -1 |
      python -c "
import json,sys
d=json.loads(sys.stdin.read()); f=d.get('fixed_effort') or {}
print('$lib', 'value', d['value'], 'fixed', f.get('value'), 'stereo_ms', d['stage_ms']['stereo'],
      'opt_ms', d['stage_ms']['optimise'], 'fixed_opt_ms', (f.get('stage_ms') or {}).get('optimise'),
      'pcg', d.get('pcg_iters_per_update'))"
  done
done
