# ncu --set full of the SIMT FD kernel at cfg3 / cfg2 (one launch after warm-up) with source
set -x
for c in 3 2; do
ncu --set full --clock-control none --import-source on -k regex:fd_fused -s 2 -c 1 -o gpurun_out/fdc$c python bench.py --config $c --mode fd --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ncu -i gpurun_out/fdc$c.ncu-rep --page source --csv > gpurun_out/fdc$c.sass.csv 2>/dev/null
ncu -i gpurun_out/fdc$c.ncu-rep --page raw --csv > gpurun_out/fdc$c.raw.csv 2>/dev/null
done
ls -la gpurun_out/fdc*
