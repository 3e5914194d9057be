mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gram or pd" > gpurun_out/pytest_gram.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gram.txt
for i in 1 2; do
timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_s3_$i.txt 2>&1
done
