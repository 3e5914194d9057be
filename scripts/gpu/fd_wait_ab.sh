# FD kernel many-waiter mbarrier waits: parked try_wait (default) vs nanosleep back-off vs plain polling
set -x
run() { timeout 300 python bench.py --mode fd --steps 300 --no-cpu-baseline --no-e2e --no-apply --latency-frames 50 > gpurun_out/$1.json 2>&1; }
for i in 1 2; do
DP_LIB_PATH=$PWD/ab_libs/libdp_park.so run fdw_park_$i
DP_LIB_PATH=$PWD/ab_libs/libdp_sleep.so run fdw_sleep_$i
DP_LIB_PATH=$PWD/ab_libs/libdp_spin.so run fdw_spin_$i
done
