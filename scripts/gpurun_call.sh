timeout 900 python -m pytest tests -m gpu -q -x -k "bslice" > gpurun_out/pytest_bs.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_bs.log
for i in 1 2; do
echo "== dyn smem, minb2"; python scripts/bench_layer.py 16 5 bslice_bwd
echo "== dyn smem, minb3"; python scripts/ab_lib.py abtmp/lib_b3.so 16 5 bslice_bwd
echo "== old"; python scripts/ab_lib.py abtmp/lib_old.so 16 5 bslice_bwd
done
