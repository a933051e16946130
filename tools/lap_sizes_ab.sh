for a in "2000 twoperm" "2000 flat" "6000 twoperm" "8192 twoperm"; do python tools/lap_big_time.py $a; done; python tools/lap_c4_time.py
