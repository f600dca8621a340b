# scratch: the command list of the most recent gpurun call (see DESIGN.md 9a for the reproducible commands)
for i in 1 2 3; do
echo "== lastblock"; python scripts/bench_layer.py 64 10 stn_bwd
echo "== separate"; python scripts/ab_lib.py abtmp/lib_sepfin.so 64 10 stn_bwd
done
echo "== lastblock K2"; python scripts/bench_paper.py stn
echo "== separate K2"; RSGRAD_LIB=abtmp/lib_sepfin.so python scripts/bench_paper.py stn
