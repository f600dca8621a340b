# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -x -k "stn or sweep or warp_tiled or host_pointer" > gpurun_out/pytest_stn.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_stn.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python scripts/sanitize_all.py 2>&1 | tail -1
python scripts/bench_layer.py 64 3 stn
