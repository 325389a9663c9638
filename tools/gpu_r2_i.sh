# round 2, batch I: triangular wire form — parity tests + bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_k1.py tests/test_abi.py -q -x > gpurun_out/i_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/i_pytest.log | cut -c1-400
for w in tri 16; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-makespan --e2e-steps 10 --wire $w > gpurun_out/i_bench_$w.json 2> gpurun_out/i_bench_$w.err; echo "bench $w rc $?"
python - <<PY
import json;d=json.loads(open('gpurun_out/i_bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['h2d_bytes_per_step'], d['e2e']['matches_device_leg'])
PY
done
for c in 3 4 6; do
DS_CHUNKS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-makespan --e2e-steps 10 > gpurun_out/i_bench_c$c.json 2>/dev/null
python - <<PY
import json;d=json.loads(open('gpurun_out/i_bench_c$c.json').read().strip().splitlines()[-1]); print('chunks $c', d['e2e']['value'], d['e2e']['ms_per_step'])
PY
done
