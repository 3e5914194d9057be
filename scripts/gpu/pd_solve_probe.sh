# PD solve variants (cfg4 PD frames) and one ncu capture of each solve kernel
set -x
run() { timeout 300 python bench.py --mode pd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
run pds_mw4
DP_SOLVE_NW=2 run pds_mw2
DP_SOLVE_SG=1 run pds_sg
ncu --set full --clock-control none --import-source on -k regex:solve -s 2 -c 1 -o gpurun_out/pds_mw4 python bench.py --mode pd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
DP_SOLVE_SG=1 ncu --set full --clock-control none --import-source on -k regex:solve -s 2 -c 1 -o gpurun_out/pds_sg python bench.py --mode pd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
