set -x
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
