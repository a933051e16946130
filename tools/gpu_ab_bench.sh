# dev: A/B every tools/ab/*.so against the current build on the C4 bench (device-resident number + LAP)
for rep in 1 2; do
timeout 1200 bash tools/ab.sh bash -c 'python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extra-precisions | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d[\"value\"],2), \"it/s\", round(d[\"ms_per_step\"],1), \"ms  lap\", round(d[\"lap_ms_per_step\"],2), \"ms  k4r\", round(d[\"roofline\"][\"us_per_pass\"],3))"'
done
