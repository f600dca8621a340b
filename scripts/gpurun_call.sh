timeout 900 python -m pytest tests -m gpu -q -x -k "warp or bicubic" > gpurun_out/pytest_w.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_w.log
for i in 1 2; do
echo "== new"; python scripts/bench_layer.py 16 5 warp
echo "== old"; python scripts/ab_lib.py abtmp/lib_old.so 16 5 warp
done
