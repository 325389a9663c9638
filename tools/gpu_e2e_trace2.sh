# e2e: stream-slot count x chunk count (tri and 16-bit wire forms).
mkdir -p gpurun_out
run() {  # wire chunks streams
  DS_E2E_TRACE=1 DS_CHUNKS=$2 DS_STREAMS=$3 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline --no-makespan --wire $1 > gpurun_out/e2e2_$1_$2_$3.json 2> gpurun_out/e2e2_$1_$2_$3.err
  echo "== wire $1 chunks $2 streams $3: $(python -c "import json;d=json.load(open('gpurun_out/e2e2_$1_$2_$3.json'));print('e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3))")"
  tail -$2 gpurun_out/e2e2_$1_$2_$3.err
}
run tri 5 5; run tri 8 8; run tri 6 6; run tri 4 4; run 16 5 5; run 16 8 8; run wide 8 8
