nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -I paper_1804_10987_b200/csrc scripts/kmaj32_probe.cu -o scripts/libkprobe.so -lcuda && python scripts/kmaj32_probe.py
