# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
for i in 1 2; do
echo "== base"; python scripts/bench_layer.py 16 5 stn
for v in fi16 fi48 f8k; do echo "== $v"; python scripts/ab_lib.py abtmp/lib_$v.so 16 5 stn; done
done
