#!/bin/bash
# Bench lines + ncu evidence for one build, on the GPU box (gpurun).
# usage: bash scripts/profile_round.sh TAG   -> gpurun_out/TAG_*
T=${1:?tag}
O=gpurun_out
mkdir -p $O
# bench lines (C2 carries the fixed-effort sub-object, e2e and the CPU leg)
python bench.py > $O/${T}_bench_c2.json 2> $O/${T}_bench_c2.err
python bench.py --config C5 --no-fixed > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err
python bench.py --config C1 --no-fixed > $O/${T}_bench_c1.json 2> $O/${T}_bench_c1.err
python bench.py --config C3 --steps 640 --no-fixed > $O/${T}_bench_c3.json 2> $O/${T}_bench_c3.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
python bench.py --config C4 --steps 3 --warmup 3 > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err
# launch list (the command first ran clean without ncu above)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    --no-e2e --no-fixed > $O/${T}_ncu_launch.log 2>&1
# one full capture of each hot kernel (frame 2: a heavy stereo frame)
ncu --set full --import-source on --clock-control none -k regex:"^(k_stereo|k_fusion)$" -s 4 -c 2 \
    -o $O/prof_${T} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-fixed \
    > $O/${T}_ncu_full.log 2>&1
# the streaming solver at 4K (fixed effort: one optimize of 500 GN x 5 PCG)
ncu --set full --import-source on --clock-control none -k regex:"k_fusion" -c 1 \
    -o $O/prof_${T}_c4 python bench.py --config C4 --regime fixed --frames 1 --steps 1 \
    --warmup 3 --no-cpu-baseline --no-e2e --no-fixed > $O/${T}_ncu_c4.log 2>&1
# per-phase trace of the solver (diagnostics build)
if [ -f paper_2207_12244_b200/libdfuse_cuda_diag.so ]; then
  DFUSE_TRACE=1 DFUSE_LIB=$PWD/paper_2207_12244_b200/libdfuse_cuda_diag.so \
    python scripts/trace_frames.py auto 2 > $O/${T}_trace.log 2>&1
fi
tail -c 600 $O/${T}_bench_c2.json
