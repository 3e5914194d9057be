mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_unequal.py tests/test_ber.py -x -q > gpurun_out/pytest_fuzz.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_fuzz.txt
timeout 900 python scripts/ber_partition.py --frames 20 --out gpurun_out/ber_partition.json > gpurun_out/ber_partition.log 2>&1
