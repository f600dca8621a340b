timeout 900 python -m pytest tests -m gpu -q -x -k "bicubic or stn3d or variants" > gpurun_out/pytest_f3.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_f3.log
