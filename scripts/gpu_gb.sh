nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gb tools/gather_bench.cu -lcuda && timeout 120 /tmp/gb
