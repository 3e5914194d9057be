# ncu --set full of the FD kernel with source: SASS-level and CUDA-source-level per-line stall samples
set -x
ncu --set full --clock-control none --import-source on -k regex:fd_tc -s 2 -c 1 -o gpurun_out/fdsrc python bench.py --mode fd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ncu -i gpurun_out/fdsrc.ncu-rep --page source --csv > gpurun_out/fdsrc.sass.csv 2>gpurun_out/fdsrc.err1
ncu -i gpurun_out/fdsrc.ncu-rep --page source --csv --print-source cuda > gpurun_out/fdsrc.cuda.csv 2>gpurun_out/fdsrc.err2
ncu -i gpurun_out/fdsrc.ncu-rep --page raw --csv > gpurun_out/fdsrc.raw.csv 2>/dev/null
ls -la gpurun_out/fdsrc*
