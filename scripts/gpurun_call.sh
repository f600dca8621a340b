timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 5 --kernel-regex-exclude kns=stn_out_tile --kernel-regex-exclude kns=stn_bwd_lean python scripts/sanitize_all.py > gpurun_out/racecheck2.txt 2>&1; echo racecheck=$?; grep -E "RACECHECK SUMMARY" gpurun_out/racecheck2.txt; grep -o "rs::<unnamed>::[a-z_0-9]*" gpurun_out/racecheck2.txt | sort | uniq -c | head
timeout 900 python -m pytest tests -m gpu -q -x -k "bslice" > gpurun_out/pytest_bs.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_bs.log
python scripts/bench_layer.py 16 5 bslice_bwd
