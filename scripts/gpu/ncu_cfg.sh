# ncu --set full of one step of a config's libdp kernels (CFG, TAG env), for the small-config analysis
set -x
ncu --set full --clock-control none --import-source on -k 'regex:fd_|gram|solve|precode' -s 4 -c 4 -o gpurun_out/${TAG}_cfg${CFG} python bench.py --config ${CFG} --steps 2 --warmup 2 --profile-run > /dev/null 2>&1
ls -la gpurun_out/${TAG}_cfg${CFG}.ncu-rep
