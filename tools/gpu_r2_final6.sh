# Round-2 final evidence after the k1_fast closure change: GPU tests, full bench
# (both arms), launch list, ncu full capture of the K1 kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2k_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r2k_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "smoke rc $?"
START=$(date +%s); timeout 1500 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "bench rc $? in $(( $(date +%s) - START )) s"
tail -3 gpurun_out/r2k_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2k_ref.json 2> gpurun_out/r2k_ref.err; echo "ref rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2k_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/r2k_launch_bench.log 2>&1; echo "ncu-launch rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_fast|k1_back_lane|k1_wsort|k1_front|k1_mid' -s 12 -c 6 -o gpurun_out/r2k_k1 -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/r2k_ncu.log 2>&1; echo "ncu rc $?"
