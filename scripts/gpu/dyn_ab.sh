# gram_tc2 with dynamic items (global counter) vs static blockIdx.x + k gridDim.x (ab_libs/libdp_prev.so)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_dyn.log 2>&1; tail -3 gpurun_out/pytest_dyn.log
for m in pd fd; do timeout 300 python scripts/diag_frames.py $m > gpurun_out/dyn_diag_$m.log 2>&1; tail -2 gpurun_out/dyn_diag_$m.log; done
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 "${@:2}" > gpurun_out/$1.json 2>&1; }
for i in 1 2; do run dyn_new_$i; DP_LIB_PATH=$PWD/ab_libs/libdp_prev.so run dyn_old_$i; done
run dyn_new_pd --mode pd; DP_LIB_PATH=$PWD/ab_libs/libdp_prev.so run dyn_old_pd --mode pd
