# FD-frame A/B: default build vs ab_libs/libdp_$B.so (cfg4), interleaved, twice each
set -x
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
for r in 1 2; do
  run ab_def_$r
  DP_LIB_PATH=ab_libs/libdp_$B.so run ab_${B}_$r
done
