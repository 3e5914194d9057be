# ncu --set full of the FD kernel (one launch after warm-up) of the current build
ncu --set full --clock-control none --import-source on -k regex:fd_tc -s 2 -c 1 -o gpurun_out/${TAG:-fd} python bench.py --mode fd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ls -la gpurun_out/${TAG:-fd}.ncu-rep
