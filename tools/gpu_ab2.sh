# dev: A/B every tools/ab/*.so against the current build; args: "n prec" pairs
while [ $# -gt 1 ]; do timeout 600 bash tools/ab.sh python tools/sdsn_bench.py $1 $2 2>&1; shift 2; done
