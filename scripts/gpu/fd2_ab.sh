# FD-frame A/B of the FD kernel variants (cfg4), interleaved, twice each; then GPU parity file
set -x
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
for r in 1 2; do
  run fd2_n3_$r
  DP_FD2_MINB2=1 run fd2_n2_$r
  DP_FD_TC1=1 run fd2_o_$r
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/fd2_pytest.log
