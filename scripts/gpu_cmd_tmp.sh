mkdir -p gpurun_out
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/torchrun1.txt 2>&1
echo "rc=$?" >> gpurun_out/torchrun1.txt
