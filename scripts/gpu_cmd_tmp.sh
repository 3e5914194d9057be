mkdir -p gpurun_out
for n in 3 4 6 8; do
DP_HOST_CHUNKS=$n timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$n.txt 2>&1
done
