# FD L2 prefetch distance of the next CTAs' tiles (DP_FD_PF x num_sms CTAs ahead; 0 = off)
set -x
run() { timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 "${@:2}" > gpurun_out/$1.json 2>&1; }
for pf in 3 0 1 2 6; do DP_FD_PF=$pf run pf_$pf --mode fd; done
DP_FD_PF=3 run pf_3b --mode fd
