for n in 20 64 128 256 500 600; do python tools/sdsn_one.py $n fp64 400; done; python tools/sdsn_one.py 128 fp32 400
