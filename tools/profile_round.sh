#!/bin/bash
# Usage (on the GPU box, via gpurun): bash tools/profile_round.sh <tag>
# 1) default bench (the reported number)  2) short bench plain run, then under ncu:
#    launch list (gpu__time_duration) and one --set full capture each of the SDSN and GEMM kernels.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_${TAG}.json 2> $OUT/bench_${TAG}.err; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra-precisions"
timeout 600 $CMD > $OUT/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $OUT/launches_${TAG}.csv $CMD > $OUT/ncu_launch_${TAG}.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdsn -s 3 -c 1 -o $OUT/prof_sdsn_${TAG} $CMD > $OUT/ncu_sdsn_${TAG}.log 2>&1; echo "ncu sdsn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 4 -c 2 -o $OUT/prof_gemm_${TAG} $CMD > $OUT/ncu_gemm_${TAG}.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lap_ -c 1 -o $OUT/prof_lap_${TAG} $CMD > $OUT/ncu_lap_${TAG}.log 2>&1; echo "ncu lap rc=$?"
ls -la $OUT
