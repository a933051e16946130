timeout 1200 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -3
for rep in 1 2 3; do
timeout 1200 bash tools/ab.sh bash -c "python bench.py --workload c3 --precision tf32 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c \"import json,sys; d=json.loads(sys.stdin.read()); print('tf32', round(d['value']), d['unit'], round(d['ms_per_step'],2), 'ms', {k: d[k] for k in d if 'acc' in k})\""
done
