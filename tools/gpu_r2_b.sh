# round 2, batch B: gpu tests after the detail-arena change, C++ API bench (both sides), 2-rank shared-GPU bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/b_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/b_pytest.log
timeout 300 paper_2602_20826_b200/_lib/api_bench 1000000 300 > gpurun_out/b_api_bench.json 2> gpurun_out/b_api_bench.err; echo "api rc $?"
cat gpurun_out/b_api_bench.json; tail -3 gpurun_out/b_api_bench.err
timeout 300 oracle/_ref/ref_api_bench 100000 300 > gpurun_out/b_ref_api_bench.json 2>&1; echo "refapi rc $?"
cat gpurun_out/b_ref_api_bench.json
DS_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-makespan > gpurun_out/b_bench2.json 2> gpurun_out/b_bench2.err; echo "bench2 rc $?"
tail -5 gpurun_out/b_bench2.err | cut -c1-300
