nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_slot tools/tma_slot_probe.cu -lcuda && timeout 120 /tmp/tma_slot
