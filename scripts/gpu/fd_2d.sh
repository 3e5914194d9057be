# 2-D sweep: GPU parity file first (stop on failure), then FD-frame A/B against the column sweep
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/fd2d_pytest.log
B=sw1 bash scripts/gpu/fd_ab2.sh
