# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "bslice" 2>&1 | tail -1
for i in 1 2; do
echo "== warp scan"; python scripts/bench_paper.py bslice; python scripts/bench_layer.py 64 5 bslice_bwd
echo "== serial scan"; RSGRAD_LIB=abtmp/lib_serialscan.so python scripts/bench_paper.py bslice; python scripts/ab_lib.py abtmp/lib_serialscan.so 64 5 bslice_bwd
done
