nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulkred_probe tools/bulkred_probe.cu && timeout 120 /tmp/bulkred_probe
