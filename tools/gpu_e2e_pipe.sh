# e2e host pipeline: parity test, then wire x chunks sweep (pipe on/off).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_k1.py -q -x -k "pipeline or full_size or compact16 or session" > gpurun_out/pipe_pytest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pipe_pytest.log
run() {  # wire chunks pipe
  DS_E2E_TRACE=1 DS_CHUNKS=$2 DS_PIPE=$3 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline --no-makespan --wire $1 > gpurun_out/pipe_$1_$2_$3.json 2> gpurun_out/pipe_$1_$2_$3.err
  echo "== wire $1 chunks $2 pipe $3: $(python -c "import json;d=json.load(open('gpurun_out/pipe_$1_$2_$3.json'));print('e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_leg'])")"
  tail -$2 gpurun_out/pipe_$1_$2_$3.err
}
for w in tri 16; do for c in 4 6 8 12; do run $w $c 1; done; done
run wide 8 1
