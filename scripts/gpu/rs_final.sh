# per-rank shapes of cfg4 at world 1 (B/N antennas, C/N clusters) after the last session's changes
set -x
for n in 2 4 8; do timeout 300 python bench.py --rank-shape $n --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 > gpurun_out/rs_final_$n.json 2>&1; done
