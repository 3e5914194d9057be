# PD solve: one warp per problem with 1 / 2 / 4 warps per CTA (DP_SOLVE_WPC), cfg4 PD frames,
# plus an ncu capture of the 4-warp-CTA variant
set -x
run() { timeout 300 python bench.py --mode pd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
DP_SOLVE_SG=1 DP_SOLVE_WPC=1 run pdw_1
DP_SOLVE_SG=1 DP_SOLVE_WPC=2 run pdw_2
DP_SOLVE_SG=1 DP_SOLVE_WPC=4 run pdw_4
DP_SOLVE_SG=1 DP_SOLVE_WPC=4 ncu --set full --clock-control none --import-source on -k regex:solve -s 2 -c 1 -o gpurun_out/pdw_4 python bench.py --mode pd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ncu -i gpurun_out/pdw_4.ncu-rep --page raw --csv > gpurun_out/pdw_4.raw.csv 2>/dev/null
