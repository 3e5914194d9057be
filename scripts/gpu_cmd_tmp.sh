mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_unequal.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_fuzz.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_fuzz.txt
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --mode fd --cluster-sizes 64,32,32,32,32,32,16,16 > gpurun_out/b_uneq.txt 2>&1
DP_VAR_SERIAL=1 timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --mode fd --cluster-sizes 64,32,32,32,32,32,16,16 > gpurun_out/b_uneq_serial.txt 2>&1
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --cluster-sizes 64,32,32,32,32,32,16,16 > gpurun_out/b_uneq_both.txt 2>&1
