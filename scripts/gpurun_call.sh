# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
PROF_COUNT=2 timeout 600 bash scripts/gpurun_prof.sh lean stn_bwd_lean 8
PROF_COUNT=2 timeout 600 bash scripts/gpurun_prof.sh bsb bslice_bwd_tiled 8
head -5 gpurun_out/lean.md gpurun_out/bsb.md
