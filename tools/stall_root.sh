# Platform-stall root cause probe: heartbeat on every SM for 20 s while
# sampling the GPU's compute processes, clocks and event reasons.
mkdir -p gpurun_out
( for i in $(seq 1 100); do date +%s.%N; nvidia-smi --query-compute-apps=pid,process_name,used_memory --format=csv,noheader; nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.active,power.draw,temperature.gpu --format=csv,noheader; sleep 0.2; done ) > gpurun_out/stall_smi.log 2>&1 &
SMI=$!
tools/heartbeat 20 148 200 > gpurun_out/stall_hb.json 2>&1
kill $SMI 2>/dev/null
ps -eo pid,comm,args --sort=-pcpu | head -25 > gpurun_out/stall_ps.log
nvidia-smi -q -d PERFORMANCE,CLOCK,ECC > gpurun_out/stall_q.log 2>&1
python - <<'PY'
import json
d=json.load(open('gpurun_out/stall_hb.json'))
g=d['gaps']
print('gaps', d['n_gaps'])
# cluster gaps by start time (ms)
ev={}
for t,us,cta in g:
    k=round(t,0)
    ev.setdefault(k,[]).append((us,cta))
for k in sorted(ev)[:30]:
    v=ev[k]; print(k, len(v), 'ctas', 'max_us', max(x[0] for x in v))
PY
head -20 gpurun_out/stall_ps.log
grep -v "^[0-9.]*$" gpurun_out/stall_smi.log | sort | uniq -c | sort -rn | head
