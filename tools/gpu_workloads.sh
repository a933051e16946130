timeout 900 python bench.py --workload ubc --steps 3 --warmup 3 > gpurun_out/ubc_final8.json 2> gpurun_out/ubc_final8.err; echo "ubc rc=$?"
for p in tf32 fp64; do timeout 900 python bench.py --workload c3 --precision $p --steps 3 --warmup 3 > gpurun_out/c3_final8_$p.json 2> gpurun_out/c3_final8_$p.err; echo "c3 $p rc=$?"; done
timeout 1500 python bench.py --workload c5 --steps 1 --warmup 1 > gpurun_out/c5_final8.json 2> gpurun_out/c5_final8.err; echo "c5 rc=$?"
