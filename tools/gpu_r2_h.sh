# round 2, batch H: e2e chunking (DS_CHUNKS) and stream count (DS_STREAMS)
set -x
mkdir -p gpurun_out
for c in 3 4 5 6 8; do
DS_CHUNKS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-makespan --e2e-steps 10 > gpurun_out/h_bench_$c.json 2> gpurun_out/h_bench_$c.err
python - <<PY
import json;d=json.loads(open('gpurun_out/h_bench_$c.json').read().strip().splitlines()[-1]); print('chunks', $c, d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])
PY
done
for c in 4 6; do
DS_STREAMS=4 DS_CHUNKS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-makespan --e2e-steps 10 > gpurun_out/h_bench_s4_$c.json 2> /dev/null
python - <<PY
import json;d=json.loads(open('gpurun_out/h_bench_s4_$c.json').read().strip().splitlines()[-1]); print('streams4 chunks', $c, d['e2e']['value'], d['e2e']['ms_per_step'])
PY
done
