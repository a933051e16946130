timeout 900 python -m pytest tests/test_gpu_sdsn.py -x -q -k "onchip or full_size or deterministic or parity" 2>&1 | tail -1
bash tools/gpu_ab.sh 4096 4096 3000 2000 1024 500
