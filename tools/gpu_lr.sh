for rep in 1 2; do timeout 600 bash tools/ab.sh python tools/k4r_call.py 4096 2>&1; done
bash tools/gpu_ab.sh 4096 4096
