# A/B of libdp builds on the FD frame (cfg4): each variant twice, interleaved
for r in 1 2; do for v in A B; do
  DP_LIB_PATH=scratch_libs/libdp_$v.so python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/ab_${v}_$r.json 2>&1
done; done
