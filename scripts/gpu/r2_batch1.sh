set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/ffma2_probe.cu -o /tmp/ffma2 && /tmp/ffma2 > gpurun_out/r2_ffma2.txt 2>&1
python bench.py > gpurun_out/r2_b4.json 2> gpurun_out/r2_b4.err
python bench.py --fp64 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/r2_b4_fp64.json 2> gpurun_out/r2_b4_fp64.err
python bench.py --K 7 --no-cpu-baseline > gpurun_out/r2_b4_K7.json 2> gpurun_out/r2_b4_K7.err
for c in 2 3 fig2a fig2b fig2c fig2d fig2e; do python bench.py --config $c --no-e2e > gpurun_out/r2_b_$c.json 2> gpurun_out/r2_b_$c.err; done
python bench.py --impl reference > gpurun_out/r2_b4_ref.json 2> gpurun_out/r2_b4_ref.err
python bench.py --oracle-seconds > gpurun_out/r2_oracle_seconds.json 2>&1
nproc > gpurun_out/r2_nproc.txt; lscpu >> gpurun_out/r2_nproc.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --profile-run > /dev/null 2>&1
ls -la gpurun_out | tail -30
