# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "stn or smoke or host or abi" > gpurun_out/r2_pt_stn.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pt_stn.log
python scripts/bench_layer.py 16 10 stn_bwd
python scripts/bench_layer.py 64 10 stn_bwd
python scripts/bench_paper.py
