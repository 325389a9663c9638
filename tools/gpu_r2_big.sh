# Round-2: big-DAG (k1_big) parity, then the whole GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_big.py -x -q > gpurun_out/r2big_pytest.log 2>&1; echo "big pytest rc $?"
tail -30 gpurun_out/r2big_pytest.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2big_pytest_all.log 2>&1; echo "all pytest rc $?"
tail -15 gpurun_out/r2big_pytest_all.log
