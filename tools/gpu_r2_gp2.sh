mkdir -p gpurun_out
START=$(date +%s); timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/gp2_bench.json 2> gpurun_out/gp2_bench.err; echo "bench rc $? in $(( $(date +%s) - START )) s"
tail -3 gpurun_out/gp2_bench.err
bash tools/gpu_ncu_back.sh
