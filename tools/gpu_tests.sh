# pytest -m gpu on the box, log under gpurun_out/
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/pytest_gpu.log
