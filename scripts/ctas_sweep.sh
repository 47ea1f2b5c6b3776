#!/bin/bash
# Solver grid sweep: bench.py updates/s and stage times at several persistent
# CTA counts (dfuse_ctx_set_solver_ctas). usage: CONFIG=C1 bash scripts/ctas_sweep.sh 37 74 148
for n in "$@"; do
  python bench.py --config ${CONFIG:-C1} --steps ${STEPS:-60} --no-cpu-baseline --no-e2e \
    ${FIXED:---no-fixed} --solver-ctas $n 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
f = d.get('fixed_effort') or {}
print('ctas', $n, 'value', d['value'], 'stage_ms', d['stage_ms']['stereo'], d['stage_ms']['optimise'],
      'pcg', d['pcg_iters_per_update'], 'fixed', f.get('value'))"
done
