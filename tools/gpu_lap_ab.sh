timeout 1200 python -m pytest tests/test_gpu_kernels.py -x -q -k "lap" 2>&1 | tail -2
for rep in 1 2; do timeout 900 bash tools/ab.sh python tools/lap_c4_time.py 2>&1 | grep -v "^$"; done
