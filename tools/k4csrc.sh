python tools/sdsn_one.py 500 fp64 > gpurun_out/k4c_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:sdsn_cluster -s 2 -c 1 -o gpurun_out/prof_k4c python tools/sdsn_one.py 500 fp64 > gpurun_out/ncu_k4c.log 2>&1
ncu -i gpurun_out/prof_k4c.ncu-rep --page source --csv --print-source sass > gpurun_out/k4c_source2.csv 2>/dev/null
rm -f gpurun_out/prof_k4c.ncu-rep
cat gpurun_out/k4c_plain.log
