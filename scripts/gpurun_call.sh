mkdir -p gpurun_out
for i in 1 2; do python scripts/bench_f3.py f3; done
