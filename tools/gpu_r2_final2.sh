# Round-2 final evidence (graph-priority executor): GPU tests, full bench (both arms).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r2g_pytest.log
START=$(date +%s); timeout 1500 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc $? in $(( $(date +%s) - START )) s"
tail -3 gpurun_out/r2g_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2g_ref.json 2> gpurun_out/r2g_ref.err; echo "ref rc $?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc $?"
