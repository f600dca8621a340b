timeout 900 python -m pytest tests -m gpu -q -x -k "stn" > gpurun_out/pytest_stn.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_stn.log
for i in 1 2; do
echo "== bank rows"; python scripts/bench_layer.py 16 5 stn
echo "== no bank rows"; python scripts/ab_lib.py abtmp/lib_nobank.so 16 5 stn
done > gpurun_out/bank_ab.txt 2>&1; cat gpurun_out/bank_ab.txt
bash scripts/gpurun_prof.sh stnbank "stn_out_tile" 4
rm -f gpurun_out/*.ncu-rep
cut -c1-400 gpurun_out/stnbank.md
