mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_r01j.json 2> gpurun_out/bench_r01j.err
timeout 300 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_r01j_cfg2.json 2>/dev/null
timeout 300 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_r01j_cfg3.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01j.csv python bench.py --profile-run --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fd_tc_kernel|gram_tc2|solve_mw|precode_tc2" -c 4 -o gpurun_out/k_r01j -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --eager > /dev/null 2>&1
