# blocked PD solve: GPU suite, then PD-frame A/B against the scalar-loop solve (DP_SOLVE_BLK=0)
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_blk.log 2>&1; tail -5 gpurun_out/pytest_blk.log
run() { timeout 300 python bench.py --mode pd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
run pdb_blk1
DP_SOLVE_BLK=0 run pdb_blk0
run pdb_blk1b
ncu --set full --clock-control none --import-source on -k regex:solve -s 2 -c 1 -o gpurun_out/pdb_blk python bench.py --mode pd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ncu -i gpurun_out/pdb_blk.ncu-rep --page raw --csv > gpurun_out/pdb_blk.raw.csv 2>/dev/null
ncu -i gpurun_out/pdb_blk.ncu-rep --page source --csv > gpurun_out/pdb_blk.src.csv 2>/dev/null
