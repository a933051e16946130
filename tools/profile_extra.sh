#!/bin/bash
# Usage (on the GPU box, via gpurun): bash tools/profile_extra.sh <tag>
# ncu --set full captures of the kernels outside the C4 bf16 step: the streaming SDSN (K4) in FP64 at
# n = 4096 (the --precision fp64 bench) and FP32 at n = 16384, the row-sharded pass kernel (K4s) at
# n = 16384, and the n = 16384 cluster LAP.  Each command first runs plain (exit 0) before ncu.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
run() {   # name, kernel regex, skip count, command...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 600 "$@" > $OUT/plain_${name}_${TAG}.log 2>&1 || { echo "$name plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 \
    -o $OUT/prof_${name}_${TAG} "$@" > $OUT/ncu_${name}_${TAG}.log 2>&1; echo "ncu $name rc=$?"
}
run sdsn_fp64 sdsn_kernel 1 python tools/sdsn_stream_timing.py 4096 fp64
run sdsn_fp32_16k sdsn_kernel 1 python tools/sdsn_bench.py 16384 fp32
run sdsn_sh sh_pass 60 python tools/sh_sdsn_time.py 16384
run lap_16k lap_cluster 1 python tools/lap_big_time.py 16384 twoperm
ls -la $OUT
