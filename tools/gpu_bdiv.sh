bash tools/gpu_ab.sh 4096 4096 4096 3000 2000
