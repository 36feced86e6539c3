nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_bench tools/fp64_bench.cu && /tmp/fp64_bench
