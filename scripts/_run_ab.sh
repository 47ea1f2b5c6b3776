DFUSE_LIB=$PWD/paper_2207_12244_b200/libdfuse_v3.so python -m pytest tests/test_gpu_fusion.py -x -q -m gpu 2>&1 | tail -2
STEPS=200 LIBS="libdfuse_old.so libdfuse_cuda.so libdfuse_v3.so" bash scripts/ab_bench.sh
