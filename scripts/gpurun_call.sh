timeout 900 python -m pytest tests -m gpu -q -k "lanczos or bicubic or variants" > gpurun_out/pytest_lz.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_lz.log
