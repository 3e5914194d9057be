# FD precode remap + staged s: GPU suite, then FD-frame A/B against the previous build (ab_libs/libdp_old.so)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_fdpc.log 2>&1; tail -3 gpurun_out/pytest_fdpc.log
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
run fdpc_new1
DP_LIB_PATH=$PWD/ab_libs/libdp_old.so run fdpc_old1
run fdpc_new2
DP_LIB_PATH=$PWD/ab_libs/libdp_old.so run fdpc_old2
