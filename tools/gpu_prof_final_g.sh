# ncu --set full of the top two kernels of the final tree (K4r, LAP) + csv pages
OUT=gpurun_out; TAG=r02g
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra-precisions"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdsn_res -s 3 -c 1 -o $OUT/prof_sdsn_$TAG $CMD > $OUT/ncu_sdsn_$TAG.log 2>&1; echo "sdsn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lap_ -c 1 -o $OUT/prof_lap_$TAG $CMD > $OUT/ncu_lap_$TAG.log 2>&1; echo "lap rc=$?"
for k in sdsn lap; do
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page details --csv > $OUT/ncu_prof_${k}_${TAG}_details.csv 2>/dev/null
  ncu -i $OUT/prof_${k}_$TAG.ncu-rep --page raw --csv > $OUT/ncu_prof_${k}_${TAG}_raw.csv 2>/dev/null
done
ls -la $OUT | grep $TAG
