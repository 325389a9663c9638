# round 2, batch F: compact hand-off for k1_fast<32> DAGs — K1 parity tests + a short bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_k1.py tests/test_gpu_fuzz.py tests/test_cpp_api.py tests/test_division_api.py -q -x > gpurun_out/f_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/f_pytest.log | cut -c1-400
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-makespan > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc $?"
python - <<'PY'
import json;d=json.loads(open('gpurun_out/f_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['roofline']['pass']['kernels_ms']))
PY
