mkdir -p gpurun_out
DP_SOLVE_SG=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:"solve_kernel" -s 2 -c 1 -o gpurun_out/k_solve_sg python bench.py --profile-run --steps 3 --warmup 2 --mode pd > gpurun_out/ncu37.log 2>&1
