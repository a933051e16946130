# dev: A/B every tools/ab/*.so against the current build (args: sizes)
for n in "$@"; do timeout 600 bash tools/ab.sh python tools/sdsn_bench.py $n fp32 2>&1; done
