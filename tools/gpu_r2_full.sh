# Round-2 full GPU pass: gpu tests, bench (both arms), launch list, ncu full of the K1 kernels.
set -x
mkdir -p gpurun_out
nvidia-smi -L
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,ecc.errors.uncorrected.volatile.total --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r2_pytest.log
START=$(date +%s); timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc $? in $(( $(date +%s) - START )) s"
tail -3 gpurun_out/r2_bench.err
START=$(date +%s); timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc $? in $(( $(date +%s) - START )) s"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/r2_launch_bench.log 2>&1; echo "ncu-launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_fast|k1_back_lane|k1_wsort|k1_front|k1_mid' -s 12 -c 6 -o gpurun_out/r2_k1 -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/r2_ncu.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/r2_ncu.log
