# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
timeout 900 python -m pytest tests -m gpu -q -x -k "warp or sweep or host_pointer or null" > gpurun_out/pytest_w.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_w.log
python scripts/bench_layer.py 64 3 warp
