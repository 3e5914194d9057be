# FD-frame timing ablation (diagnostics builds, ab_libs/): default, no sweep, no SIMT precode, no Gram UMMAs
set -x
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
run abl_def
for v in 1 2 4; do DP_LIB_PATH=ab_libs/libdp_abl$v.so run abl_$v; done
