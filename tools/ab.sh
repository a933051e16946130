#!/bin/bash
# Dev A/B: run a command with each tools/ab/*.so swapped in for the package's libfram.so, then the
# current build; restores the current build.  Usage: bash tools/ab.sh <command...>
set -u
LIB=paper_2508_00887_b200/libfram.so
cp $LIB /tmp/ab_current.so
for so in tools/ab/*.so /tmp/ab_current.so; do
  cp "$so" $LIB
  echo "== $(basename $so)"
  "$@"
done
cp /tmp/ab_current.so $LIB
