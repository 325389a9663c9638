# Platform stalls with and without an nvidia-smi poller beside the heartbeat
mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json, sys
d=json.load(open(sys.argv[1])); ev={}
for t,us,cta in d['gaps']: ev.setdefault(round(t/2)*2,[]).append(us)
full=[(k,len(v),max(v)) for k,v in sorted(ev.items()) if len(v)>=100]
print(sys.argv[1], 'events(all SMs):', len(full), 'per s:', round(len(full)/d['secs'],2), 'max_us:', max([x[2] for x in full] or [0]), 'first:', [x[0] for x in full][:8])
PY
}
tools/heartbeat 20 148 200 > gpurun_out/hb_quiet1.json; summ gpurun_out/hb_quiet1.json
( while true; do nvidia-smi --query-gpu=clocks.sm --format=csv,noheader > /dev/null; sleep 0.05; done ) &
P=$!
tools/heartbeat 20 148 200 > gpurun_out/hb_smi20hz.json; summ gpurun_out/hb_smi20hz.json
kill $P
tools/heartbeat 20 148 200 > gpurun_out/hb_quiet2.json; summ gpurun_out/hb_quiet2.json
dmesg 2>/dev/null | tail -20
cat /proc/interrupts | grep -i nv | head
