# Source-level ncu capture of one k1_back_lane launch (session pass, 1M C5 DAGs).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_back_lane' -s 3 -c 1 -o gpurun_out/k1back -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/ncu_k1back.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/ncu_k1back.log
