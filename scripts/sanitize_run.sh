# compute-sanitizer over every entry point (scripts/sanitize_all.py): memcheck, synccheck,
# initcheck on the product build; racecheck on the RS_RACECHECK_SYNC=1 build (mbarrier
# hand-offs also expressed as bar.sync).  Logs -> gpurun_out/r2_san_*.log
CS=compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 python scripts/sanitize_all.py > gpurun_out/r2_san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/r2_san_$tool.log
done
RSGRAD_LIB=abtmp/lib_racecheck.so timeout 2400 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_all.py > gpurun_out/r2_san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/r2_san_racecheck.log
