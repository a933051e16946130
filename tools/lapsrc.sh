python tools/lap_c4_time.py > gpurun_out/lap_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:lap_cluster -s 1 -c 1 -o gpurun_out/prof_lapsrc python tools/lap_c4_time.py > gpurun_out/ncu_lapsrc.log 2>&1
ncu -i gpurun_out/prof_lapsrc.ncu-rep --page source --csv --print-source sass > gpurun_out/lap_source.csv 2>/dev/null
rm -f gpurun_out/prof_lapsrc.ncu-rep
cat gpurun_out/lap_plain.log
