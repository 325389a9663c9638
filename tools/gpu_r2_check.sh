set -x
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/g1_pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-makespan > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc $?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g1_ref.json 2>&1; echo "ref rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_front|k1_mid|k1_back_lane' -s 9 -c 3 -o gpurun_out/g1_k1 python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/g1_ncu.log 2>&1; echo "ncu rc $?"
