mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python bench.py --config 2 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg2_$i.json 2>/dev/null
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg3_$i.json 2>/dev/null
done
timeout 600 python -m pytest tests/test_gpu_unequal.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_fuzz.txt 2>&1
