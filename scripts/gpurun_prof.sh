# usage: bash scripts/gpurun_prof.sh TAG KERNEL_REGEX NB [ENV=VAL ...]
# ncu --set full of the matching kernels of one bench_layer pass (NB samples), then
# the summary table, per-line and per-SASS hot spots, written to gpurun_out/ (the
# .ncu-rep itself is removed when large so the merge back stays small)
# (PROF_CMD overrides the profiled command, e.g. "python scripts/bench_next.py")
TAG=$1; KR=$2; NB=$3; shift 3
CMD=${PROF_CMD:-python scripts/bench_layer.py $NB 1}
MET=$(python -c "import sys; sys.path.insert(0,'scripts'); import ncu_summary; print(ncu_summary.EXTRA_METRICS)")
env "$@" ncu --set full --metrics $MET --import-source on --clock-control none -k "regex:$KR" -c ${PROF_COUNT:-4} -f -o gpurun_out/$TAG \
    $CMD > gpurun_out/$TAG.log 2>&1
python scripts/ncu_summary.py gpurun_out/$TAG.ncu-rep gpurun_out/$TAG.md >> gpurun_out/$TAG.log 2>&1
for k in $(ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys,re
r=list(csv.reader(sys.stdin)); i=r[0].index('Kernel Name')
print(' '.join(sorted({re.sub(r'[(<].*','',x[i]).split('::')[-1] for x in r[2:]})))"); do
  ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda,sass -k "regex:$k" > /tmp/src_$k.csv 2>/dev/null
  echo "=== $k" >> gpurun_out/$TAG.hot.txt
  python scripts/src_hot.py /tmp/src_$k.csv 60 >> gpurun_out/$TAG.hot.txt 2>&1
  ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass -k "regex:$k" > /tmp/sass_$k.csv 2>/dev/null
  python scripts/sass_hot.py /tmp/sass_$k.csv >> gpurun_out/$TAG.hot.txt 2>&1
done
sz=$(stat -c %s gpurun_out/$TAG.ncu-rep); [ "$sz" -gt 20000000 ] && rm gpurun_out/$TAG.ncu-rep
true
