mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gram or pd" > gpurun_out/pytest_gram.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gram.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench.txt 2>&1
timeout 300 python scripts/imbalance_probe.py > gpurun_out/imbalance.txt 2>&1
