# FD single-round bf16-residual whitening + split Gram commits + TMEM alloc on warp 1:
# GPU suite, then FD-frame A/B against the two-round whitening build (ab_libs/libdp_wz2.so)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_wz.log 2>&1; tail -3 gpurun_out/pytest_wz.log
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
run fdwz_new1
DP_LIB_PATH=$PWD/ab_libs/libdp_wz2.so run fdwz_wz2_1
run fdwz_new2
DP_LIB_PATH=$PWD/ab_libs/libdp_wz2.so run fdwz_wz2_2
