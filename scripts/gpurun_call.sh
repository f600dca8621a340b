timeout 600 python -m pytest tests -m gpu -x -q -k "bslice" > gpurun_out/pytest_bs.log 2>&1; echo pytest=$?
for v in tiled staged; do echo "== $v"; RSGRAD_BSLICE_BWD=$v python scripts/bench_layer.py 16 5 bslice_bwd; done > gpurun_out/bs_ab.txt 2>&1
cat gpurun_out/bs_ab.txt; tail -3 gpurun_out/pytest_bs.log
bash scripts/gpurun_prof.sh bss bslice_bwd_staged 4
rm -f gpurun_out/*.ncu-rep
