# Re-entry check: GPU tests + a short bench on the rebuilt tree.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rv_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/rv_pytest.log
START=$(date +%s); timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rv_bench.json 2> gpurun_out/rv_bench.err; echo "bench rc $? in $(( $(date +%s) - START )) s"
tail -3 gpurun_out/rv_bench.err
