{
echo "== base"; python scripts/bench_layer.py 16 5 stn
for v in ot512b1 ot512b2 ot384fi24 ot384fi48; do echo "== $v"; python scripts/ab_lib.py abtmp/lib_$v.so 16 5 stn; done
echo "== base"; python scripts/bench_layer.py 16 5 stn
} > gpurun_out/sweep2.txt 2>&1; cat gpurun_out/sweep2.txt
