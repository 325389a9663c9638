# round 2, batch D: the latency path (k1_small) under the full gpu suite + C++ API latency
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/d_pytest.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/d_pytest.log | cut -c1-400
timeout 300 paper_2602_20826_b200/_lib/api_bench 1000000 1000 > gpurun_out/d_api_bench.json 2> gpurun_out/d_api_bench.err; echo "api rc $?"
cat gpurun_out/d_api_bench.json; tail -3 gpurun_out/d_api_bench.err
timeout 300 oracle/_ref/ref_api_bench 100000 1000 > gpurun_out/d_ref_api_bench.json; cat gpurun_out/d_ref_api_bench.json
