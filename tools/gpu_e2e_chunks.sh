# e2e (ds_analyze_batch_tri, 1M C5 DAGs) under chunk / back-stream settings, after the K1 speed-ups.
mkdir -p gpurun_out
for s in "DS_NONE=0" "DS_CHUNKS=3" "DS_CHUNKS=4" "DS_CHUNKS=6" "DS_CHUNKS=8" "DS_PIPE_BACKS=3" "DS_CHUNKS=4 DS_PIPE_BACKS=3" "DS_NONE=1"; do
  env $s timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline --no-makespan > gpurun_out/ec.json 2> gpurun_out/ec.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ec.json').read().strip().splitlines()[-1]); print('$s', round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_leg'])"
done
