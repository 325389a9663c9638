# round 2, batch G: walk-key layouts for k1_back_lane (DS_WALK_KEY 0/1/2), parity on each
set -x
mkdir -p gpurun_out
for k in 0 1 2; do
DS_WALK_KEY=$k timeout 600 python -m pytest tests/test_gpu_k1.py -q -x -k "golden or seeded or full_size" > gpurun_out/g_pytest_$k.log 2>&1; echo "pytest $k rc $?"
DS_WALK_KEY=$k timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-makespan --e2e-steps 1 > gpurun_out/g_bench_$k.json 2> gpurun_out/g_bench_$k.err; echo "bench $k rc $?"
python - <<PY
import json;d=json.loads(open('gpurun_out/g_bench_$k.json').read().strip().splitlines()[-1]); print($k, d['value'], json.dumps(d['roofline']['pass']['kernels_ms']))
PY
done
