# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pt_all.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2_pt_all.log
for nb in 16 64; do
echo "== auto $nb"; python scripts/bench_layer.py $nb 10 warp_bwd
done
