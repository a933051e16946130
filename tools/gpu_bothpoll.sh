cp paper_2508_00887_b200/libfram.so /tmp/cur.so; cp tools/ab/bothpoll.so paper_2508_00887_b200/libfram.so
timeout 900 python -m pytest tests/test_gpu_sdsn.py -x -q -k "onchip or full_size or deterministic" 2>&1 | tail -1
cp /tmp/cur.so paper_2508_00887_b200/libfram.so
bash tools/gpu_ab.sh 4096 4096 4096 3000 2048 1024
