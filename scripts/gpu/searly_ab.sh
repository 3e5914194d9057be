# PD solve: s fetched before griddepcontrol.wait (new) vs after (ab_libs/libdp_prev.so)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_searly.log 2>&1; tail -3 gpurun_out/pytest_searly.log
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 "${@:2}" > gpurun_out/$1.json 2>&1; }
for i in 1 2; do run se_new_pd_$i --mode pd; DP_LIB_PATH=$PWD/ab_libs/libdp_prev.so run se_old_pd_$i --mode pd; done
run se_new_both; DP_LIB_PATH=$PWD/ab_libs/libdp_prev.so run se_old_both
