# fd_fused_kernel<16> at 4 CTAs / SM (128 registers) vs 3 (ab_libs/libdp_prev.so): cfg3 and Fig. 2(a)/(c) FD frames
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "fd or fig or cfg3 or fuzz or small or unequal" > gpurun_out/pytest_fd16.log 2>&1; tail -3 gpurun_out/pytest_fd16.log
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 "${@:2}" > gpurun_out/$1.json 2>&1; }
for c in 3 fig2a fig2c; do
run fd16_new_$c --config $c
DP_LIB_PATH=$PWD/ab_libs/libdp_prev.so run fd16_old_$c --config $c
run fd16_new2_$c --config $c
done
