# Source-level ncu capture of one k1_fast<32> and one k1_fast<64> launch.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_fast' -s 6 -c 2 -o gpurun_out/k1fast -f python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan > gpurun_out/ncu_k1fast.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/ncu_k1fast.log
