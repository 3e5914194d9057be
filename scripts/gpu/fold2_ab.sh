# FD scalars: fd_finish_kernel with batched loads after the FD kernel (new default at Cl = 8) vs the
# 2-CTA thread-block-cluster fold (DP_FD_CLUSTER_FOLD=1): FD tests, FD frames, default step
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "fd or unequal or fuzz or host or force_comm or consecutive or symbol or full_size or small or mrt or ber or deterministic" > gpurun_out/pytest_fold2.log 2>&1; tail -3 gpurun_out/pytest_fold2.log
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 "${@:2}" > gpurun_out/$1.json 2>&1; }
for i in 1 2; do run f2_new_$i --mode fd; DP_FD_CLUSTER_FOLD=1 run f2_old_$i --mode fd; done
run f2_new_both; DP_FD_CLUSTER_FOLD=1 run f2_old_both
