# fd_fused_kernel replicas splitting the whitening's symbols (whiten_Tg_rep) + the relaxed replica rule
# (one precode row per lane) vs the previous build: small-U configs, PD and FD frames
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "fd or fig or cfg2 or cfg3 or fuzz or small or unequal or pd or host" > gpurun_out/pytest_rep.log 2>&1; tail -3 gpurun_out/pytest_rep.log
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 "${@:2}" > gpurun_out/$1.json 2>&1; }
for c in 2 3 fig2a fig2c fig2d fig2e; do
run rep_new_$c --config $c
DP_LIB_PATH=$PWD/ab_libs/libdp_prev.so run rep_old_$c --config $c
done
