# DP_FLAG_HOST_ASYNC: host-pointer tests, then the default bench line (e2e async + sync)
set -x
timeout 600 python -m pytest tests -m gpu -x -q -k "host" > gpurun_out/pytest_async.log 2>&1; tail -3 gpurun_out/pytest_async.log
timeout 400 python bench.py --steps 200 --latency-frames 50 --no-apply > gpurun_out/async_b4.json 2> gpurun_out/async_b4.err
timeout 400 python bench.py --config 3 --steps 200 --latency-frames 50 --no-apply --no-cpu-baseline > gpurun_out/async_b3.json 2> gpurun_out/async_b3.err
