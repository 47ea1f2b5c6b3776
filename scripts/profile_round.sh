#!/bin/bash
# Bench lines + ncu evidence for one build, on the GPU box (gpurun).
# usage: bash scripts/profile_round.sh TAG   -> gpurun_out/TAG_*
T=${1:?tag}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${T}_bench_c2.json 2> $O/${T}_bench_c2.err
python bench.py --regime fixed > $O/${T}_bench_c2_fixed.json 2> $O/${T}_bench_c2_fixed.err
python bench.py --config C5 > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err
python bench.py --config C1 > $O/${T}_bench_c1.json 2> $O/${T}_bench_c1.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
python bench.py --config C4 --regime fixed --steps 3 --warmup 3 --no-cpu-baseline \
    > $O/${T}_bench_c4_fixed.json 2> $O/${T}_bench_c4_fixed.err
python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err
# launch list (the command first ran clean without ncu above)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    --no-e2e > $O/${T}_ncu_launch.log 2>&1
# one full capture of each hot kernel
ncu --set full --import-source on --clock-control none -k regex:"k_stereo|k_fusion" -s 4 -c 2 \
    -o $O/prof_${T} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/${T}_ncu_full.log 2>&1
# per-phase trace of the solver (diagnostics build)
if [ -f paper_2207_12244_b200/libdfuse_cuda_diag.so ]; then
  DFUSE_TRACE=1 DFUSE_LIB=$PWD/paper_2207_12244_b200/libdfuse_cuda_diag.so python scripts/trace_fixed.py \
    > $O/${T}_trace.log 2>&1
fi
tail -c 600 $O/${T}_bench_c2.json
