# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bslice" > gpurun_out/pytest_bs.log 2>&1; tail -3 gpurun_out/pytest_bs.log
