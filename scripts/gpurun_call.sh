timeout 600 python -m pytest tests -m gpu -x -q -k "conv" > gpurun_out/pytest_conv.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_conv.log
python scripts/bench_next.py > gpurun_out/next.json 2>&1; cat gpurun_out/next.json
