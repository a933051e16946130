echo "NCCL_DEBUG=${NCCL_DEBUG:-unset}"
echo "---- c5 stdout lines:"; timeout 900 python bench.py --workload c5 --steps 1 --warmup 1 --max-outer 2 2>/dev/null | wc -l
echo "---- c4 default stdout:"; timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; ls=sys.stdin.read().splitlines(); print(len(ls), 'lines'); d=json.loads(ls[-1]); print(d['value'], d['e2e']['value'])"
