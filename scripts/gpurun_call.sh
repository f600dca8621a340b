# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -x -k "warp" > gpurun_out/pytest_w.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_w.log
for i in 1 2; do
echo "== v2"; python scripts/bench_layer.py 16 5 warp_bwd
echo "== scalar"; python scripts/ab_lib.py abtmp/lib_nov2.so 16 5 warp_bwd
done
