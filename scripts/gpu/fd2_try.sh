# fd_tc2 first run: GPU parity tests, then FD-frame A/B (new default vs DP_FD_TC1) twice each
set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/fd2_pytest.log
for r in 1 2; do
  timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/fd2_new_$r.json 2>&1
  DP_FD_TC1=1 timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/fd2_old_$r.json 2>&1
done
