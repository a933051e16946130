# final validation of a tree on one GPU: full -m gpu suite, smoke, default bench, launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_final12.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_final12.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final12.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final12.log
timeout 900 python bench.py > gpurun_out/bench_final12.json 2> gpurun_out/bench_final12.err; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extra-precisions"
timeout 600 $CMD > gpurun_out/plain_final12.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_final12.csv $CMD > gpurun_out/ncu_launch_final12.log 2>&1; echo "launch list rc=$?"
