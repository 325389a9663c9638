# e2e with prioritised chunk streams: wire x chunks, priorities on/off.
mkdir -p gpurun_out
run() {  # wire chunks prio
  DS_E2E_TRACE=1 DS_CHUNKS=$2 DS_STREAM_PRIO=$3 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline --no-makespan --wire $1 > gpurun_out/e2e3_$1_$2_$3.json 2> gpurun_out/e2e3_$1_$2_$3.err
  echo "== wire $1 chunks $2 prio $3: $(python -c "import json;d=json.load(open('gpurun_out/e2e3_$1_$2_$3.json'));print('e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3))")"
  tail -$2 gpurun_out/e2e3_$1_$2_$3.err
}
for w in tri 16; do for c in 4 5 6 8; do run $w $c 1; done; run $w 5 0; done
