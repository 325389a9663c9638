mkdir -p gpurun_out
START=$(date +%s); timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bq.json 2> gpurun_out/bq.err; echo "bench rc $? in $(( $(date +%s) - START )) s"
tail -3 gpurun_out/bq.err
tail -c 3000 gpurun_out/bq.json
