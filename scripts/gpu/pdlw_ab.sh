# FD kernel: griddepcontrol.wait moved from the start to just before the x stores; GPU suite, default step
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pdlw.log 2>&1; tail -3 gpurun_out/pytest_pdlw.log
timeout 300 python scripts/diag_frames.py > gpurun_out/pdlw_diag.log 2>&1; tail -3 gpurun_out/pdlw_diag.log
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 "${@:2}" > gpurun_out/$1.json 2>&1; }
run pdlw_both1; run pdlw_both2; run pdlw_fd --mode fd
