# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -x -k "bslice" > gpurun_out/pytest_bs.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_bs.log
for i in 1 2 3; do
echo "== smem-prefetch"; python scripts/bench_layer.py 16 5 bslice_bwd
echo "== old"; python scripts/ab_lib.py abtmp/lib_old.so 16 5 bslice_bwd
done
