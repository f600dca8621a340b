# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "warp" > gpurun_out/r2_pt_warp.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_pt_warp.log
for nb in 16 64; do
echo "== auto $nb"; python scripts/bench_layer.py $nb 10 warp
echo "== minb4 $nb"; python scripts/ab_lib.py abtmp/lib_minb4.so $nb 10 warp_bwd
echo "== r8 $nb"; RSGRAD_WARP_R=8 python scripts/bench_layer.py $nb 10 warp_bwd
echo "== direct $nb"; RSGRAD_WARP_BWD=direct python scripts/bench_layer.py $nb 10 warp_bwd
done
