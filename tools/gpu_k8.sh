timeout 1200 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -3
for prec in tf32 fp64 bf16; do
timeout 1200 bash tools/ab.sh bash -c "python bench.py --workload c3 --precision $prec --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c \"import json,sys; d=json.loads(sys.stdin.read()); print('$prec', round(d['value']), d['unit'], round(d['ms_per_step'],2), 'ms', d.get('accuracy', d.get('inlier_accuracy')))\""
done
