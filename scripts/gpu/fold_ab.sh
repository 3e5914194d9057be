# FD per-subcarrier scalars: in-kernel 2-CTA-cluster fold (default) vs the separate finish kernel (DP_NO_FOLD)
set -x
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
for i in 1 2; do run fold_$i; DP_NO_FOLD=1 run nofold_$i; done
