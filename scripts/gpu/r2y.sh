for r in 1 2; do
timeout 150 python bench.py --mode pd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 > gpurun_out/r2y_pd_nw4_$r.json 2>&1
DP_SOLVE_NW=2 timeout 150 python bench.py --mode pd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 > gpurun_out/r2y_pd_nw2_$r.json 2>&1
DP_SOLVE_SG=1 timeout 150 python bench.py --mode pd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 > gpurun_out/r2y_pd_sg_$r.json 2>&1
done
