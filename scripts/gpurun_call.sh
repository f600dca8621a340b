mkdir -p gpurun_out
python scripts/bench_layer.py 64 10 stn_
echo t2; python scripts/ab_lib.py paper_1904_12228_b200/ab_t2.so 64 10 stn_
