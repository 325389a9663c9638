# e2e chunk timelines (DS_E2E_TRACE) for the wire forms and chunk counts.
mkdir -p gpurun_out
for w in 16 tri; do for c in 3 5 8; do
  echo "== wire $w chunks $c"
  DS_E2E_TRACE=1 DS_CHUNKS=$c timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline --no-makespan --wire $w > gpurun_out/e2e_${w}_${c}.json 2> gpurun_out/e2e_${w}_${c}.err
  tail -$((c+1)) gpurun_out/e2e_${w}_${c}.err
  python -c "import json;d=json.load(open('gpurun_out/e2e_${w}_${c}.json'));print('value',round(d['value']/1e6,1),'e2e',round(d['e2e']['value']/1e6,1), d['e2e']['ms_per_step'])"
done; done
