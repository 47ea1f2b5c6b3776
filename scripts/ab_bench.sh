#!/bin/bash
# A/B of library builds on the GPU box: bench.py (C2) in both solver regimes,
# twice, for every library named in LIBS (paths relative to the package).
# usage: LIBS="libdfuse_old.so libdfuse_cuda.so" bash scripts/ab_bench.sh
LIBS=${LIBS:-"libdfuse_old.so libdfuse_cuda.so"}
for r in 1 2; do
  for lib in $LIBS; do
    for reg in defaults fixed; do
      DFUSE_LIB=$PWD/paper_2207_12244_b200/$lib timeout 200 python bench.py --no-cpu-baseline \
        --no-e2e --regime $reg --steps 200 $BENCH_ARGS 2>&1 | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib','$reg',d['value'])"
    done
  done
done
