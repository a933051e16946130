for rep in 1 2; do for prec in bf16 fp64 tf32; do
timeout 1200 bash tools/ab.sh bash -c "python bench.py --workload c3 --precision $prec --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c \"import json,sys; d=json.loads(sys.stdin.read()); print('$prec', round(d['value']), d['unit'], round(d['ms_per_step'],2), 'ms')\""
done; done
