# ncu --set full of the FD kernel variants (one launch each, after warm-up), for A/B comparisons
set -x
ncu --set full --clock-control none --import-source on -k regex:fd_tc -s 2 -c 1 -o gpurun_out/${TAG:-fd}_new python bench.py --mode fd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
DP_FD_TC1=1 ncu --set full --clock-control none --import-source on -k regex:fd_tc -s 2 -c 1 -o gpurun_out/${TAG:-fd}_old python bench.py --mode fd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -3
