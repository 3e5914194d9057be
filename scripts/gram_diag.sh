#!/bin/bash
# PD Gram / precode kernel ablation: build libdp variants with -DDP_GRAM_DIAG=1/2/3 and
# -DDP_PC2_DIAG=1/2/3 (no UMMAs; also no residual math; also no epilogue work) into diag/ and time the PD frame with each through DP_LIB_PATH.
#   here:        bash scripts/gram_diag.sh build
#   on the GPU:  bash scripts/gram_diag.sh run     (writes gpurun_out/diag_<v>.txt)
set -e
cd "$(dirname "$0")/.."
if [ "$1" = build ]; then
  mkdir -p diag
  NCCL=$(python -c "import nvidia.nccl, os; print(os.path.dirname(nvidia.nccl.__file__))" 2>/dev/null || python -c "import os, nvidia; print(os.path.join(list(nvidia.__path__)[0], 'nccl'))")
  for v in 1 2 3; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden -DDP_BUILD -DDP_GRAM_DIAG=$v -DDP_PC2_DIAG=$v -I include -I paper_1804_10987_b200/csrc \
      -I "$NCCL/include" paper_1804_10987_b200/csrc/dp_api.cu -o diag/libdp_diag$v.so -L "$NCCL/lib" -l:libnccl.so.2 \
      -Xlinker -rpath,"$NCCL/lib" &
  done
  wait
else
  mkdir -p gpurun_out
  for v in 0 1 2 3; do
    if [ $v = 0 ]; then L=""; else L="DP_LIB_PATH=$PWD/diag/libdp_diag$v.so"; fi
    env $L timeout -s KILL 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e --mode pd > gpurun_out/diag_$v.txt 2>&1
  done
fi
