# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
MET=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_summary; print(ncu_summary.EXTRA_METRICS)")
python scripts/prof_a11.py 8 7 > gpurun_out/r2_a11_times.jsonl
python scripts/prof_a11.py 64 5 > gpurun_out/r2_a11_times64.jsonl
for i in 0 1 2; do
  ncu --metrics $MET,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k "regex:stn_|warp_|bslice_|det_" python scripts/prof_a11.py 8 1 $i > gpurun_out/r2_a11_v$i.csv 2>/dev/null
done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stn" 2>&1 | tail -1
