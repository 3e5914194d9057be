for pad in 0 20000 40000; do
  DP_FD_SMEM_PAD=$pad timeout 120 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --mode fd | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pad $pad', round(d['ms_per_step']*1e3,1), {k:round(v['ms_avg']*1e3,1) for k,v in d['roofline']['kernels'].items()})"
done
