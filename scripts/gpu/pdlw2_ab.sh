# late griddepcontrol.wait in fd_tc, fd_fused, fd_small: GPU suite, back-to-back frame diagnostics, bench lines
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pdlw2.log 2>&1; tail -3 gpurun_out/pytest_pdlw2.log
for m in pd fd; do timeout 300 python scripts/diag_frames.py $m > gpurun_out/pdlw2_diag_$m.log 2>&1; tail -2 gpurun_out/pdlw2_diag_$m.log; done
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 100 "${@:2}" > gpurun_out/$1.json 2>&1; }
run pw2_both; run pw2_fd --mode fd; run pw2_c3 --config 3; run pw2_c2 --config 2; run pw2_fig2d --config fig2d
