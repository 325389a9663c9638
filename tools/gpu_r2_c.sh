# round 2, batch C: the C++ drivers against the reference, the C++ API bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_drivers.py tests/test_cpp_api.py tests/test_division_api.py -x -q > gpurun_out/c_pytest.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/c_pytest.log
timeout 300 paper_2602_20826_b200/_lib/api_bench 1000000 300 > gpurun_out/c_api_bench.json 2> gpurun_out/c_api_bench.err; echo "api rc $?"
cat gpurun_out/c_api_bench.json
