# round 2, batch E: full gpu suite + a short bench (k1_fast<64> bit-serial phases, latency path)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/e_pytest.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/e_pytest.log | cut -c1-400
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-makespan > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/e_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['roofline']['pass']['kernels_ms']))"
