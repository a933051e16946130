#!/bin/bash
# Dev A/B: link a variant of libfram.so into tools/ab/<name>.so with one source recompiled under
# extra nvcc flags (the other objects come from the package build).  Usage:
#   bash tools/build_variant.sh <name> <source.cu>[,<source2.cu>...] [-DFOO=1 ...]
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/.."
python -c "from paper_2508_00887_b200 import build as b; b.build()" >/dev/null
B=paper_2508_00887_b200/build
mkdir -p /tmp/fram_variant tools/ab
rm -f /tmp/fram_variant/*.o
for one in ${src//,/ }; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -Iinclude -Ipaper_2508_00887_b200/csrc \
    --expt-relaxed-constexpr "$@" -c paper_2508_00887_b200/csrc/$one -o /tmp/fram_variant/$(basename $one .cu).o
done
objs=""
for o in $B/*.o; do
  if [ -f /tmp/fram_variant/$(basename $o) ]; then objs="$objs /tmp/fram_variant/$(basename $o)"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/ab/$name.so $objs -ldl -lpthread
echo "built tools/ab/$name.so"
