timeout 1500 bash tools/ab.sh python tools/lap_c4_time.py 2>&1 | grep -v "^$"
