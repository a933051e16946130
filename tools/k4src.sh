#!/bin/bash
# Dev (on the GPU box): ncu source-level capture of the streaming SDSN kernel K4 at n / precision,
# summarised by tools/sass_stalls.py.  Usage: bash tools/k4src.sh <n> <fp32|fp64> [passes] [tag]
n=$1; prec=$2; k=${3:-200}; tag=${4:-k4}
python tools/sdsn_one.py $n $prec $k > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sdsn_kernel -s 2 -c 1 -o gpurun_out/prof_${tag} python tools/sdsn_one.py $n $prec $k > gpurun_out/ncu_${tag}.log 2>&1
ncu -i gpurun_out/prof_${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_source.csv 2>/dev/null
ncu -i gpurun_out/prof_${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
rm -f gpurun_out/prof_${tag}.ncu-rep
python tools/sass_stalls.py gpurun_out/${tag}_source.csv 60 0.4 > gpurun_out/${tag}_stalls.txt
cat gpurun_out/${tag}_plain.log
