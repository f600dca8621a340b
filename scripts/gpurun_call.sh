mkdir -p gpurun_out
python scripts/bench_layer.py 64 10 stn_bwd
for t in b2a b2b; do echo $t; python scripts/ab_lib.py paper_1904_12228_b200/ab_$t.so 64 10 stn_bwd; done
