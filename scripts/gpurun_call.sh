# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
mkdir -p gpurun_out
python scripts/bench_layer.py 64 10 stn_bwd
for t in c4a c4b c3d; do echo $t; python scripts/ab_lib.py paper_1904_12228_b200/ab_$t.so 64 10 stn_bwd; done
python scripts/bench_paper.py stn
