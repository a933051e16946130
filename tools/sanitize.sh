#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the libfram kernels, one small case per run
# (tools/sanitize_cases.py).  Usage: bash tools/sanitize.sh <outdir>
out=${1:-gpurun_out/sanitize}
mkdir -p $out
CS=/usr/local/cuda/bin/compute-sanitizer
for c in k4c:20 k4c:500 k4c32:64 k4r:500 k4r:4096 k4:4096 k7:500 k7c:4096 k8:64 gemm:256 k4s:256 fram:300; do
  name=${c/:/_}; args=${c/:/ }
  for tool in memcheck racecheck synccheck; do
    timeout -s KILL 600 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_cases.py $args \
      > $out/${tool}_$name.log 2>&1
    echo "$tool $name rc=$? $(grep -m1 -E 'ERROR SUMMARY|RACECHECK SUMMARY' $out/${tool}_$name.log)"
  done
done
