nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gridsync tools/gridsync_bench.cu && timeout 120 /tmp/gridsync | tee gpurun_out/gridsync.json
