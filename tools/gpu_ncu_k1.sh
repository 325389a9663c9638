mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_fast|k1_back_lane|k1_wsort' -s 9 -c 3 -o gpurun_out/k1fast -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/ncu_k1fast.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/ncu_k1fast.log
