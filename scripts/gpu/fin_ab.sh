# fd_finish_kernel with one lane per cluster (ordered shuffle sums): GPU suite, FD frames, default step
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_fin.log 2>&1; tail -3 gpurun_out/pytest_fin.log
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 "${@:2}" > gpurun_out/$1.json 2>&1; }
run fin_fd1 --mode fd; run fin_fd2 --mode fd; run fin_both
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 3 --warmup 2 --profile-run --mode fd > /dev/null 2>&1
