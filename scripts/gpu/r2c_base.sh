# round-2 session-2 baseline: gpu tests, default bench, ncu source-level capture of the four cfg4 kernels
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2c_pytest.log
python bench.py > gpurun_out/r2c_b4.json 2> gpurun_out/r2c_b4.err
ncu --set full --clock-control none --import-source on -k 'regex:fd_tc|gram_tc2|solve_mw|precode_tc2' -s 8 -c 4 -o gpurun_out/r2c_cfg4 python bench.py --steps 2 --warmup 2 --profile-run --no-cpu-baseline --no-e2e --no-apply --latency-frames 2 > gpurun_out/r2c_ncu.log 2>&1
ls -la gpurun_out | tail
