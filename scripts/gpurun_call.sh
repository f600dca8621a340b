# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
RSGRAD_LIB=abtmp/lib_splat8.so PROF_COUNT=1 PROF_CMD="python scripts/bench_layer.py 8 1 stn_bwd" bash scripts/gpurun_prof.sh r2_splat "stn_bwd_splat" 8
