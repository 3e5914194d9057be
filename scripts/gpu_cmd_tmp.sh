mkdir -p gpurun_out
for i in 1 2; do
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --mode pd > gpurun_out/b64_$i.txt 2>&1
DP_GRAM_CH32=1 timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --mode pd > gpurun_out/b32_$i.txt 2>&1
done
DP_GRAM_CH32=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gram or pd" > gpurun_out/pytest_gram.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gram.txt
