mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench.txt 2>&1
echo "bench rc=$?" >> gpurun_out/bench.txt
timeout -s KILL 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
DP_NO_HANDOFF=1 timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --mode pd > gpurun_out/bench_noh.txt 2>&1
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --mode pd > gpurun_out/bench_h.txt 2>&1
