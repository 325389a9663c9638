# Pipeline with two alternating back streams (DS_PIPE_BACK2): parity + e2e.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1.py -q -x -k "tri or pipeline or full_size" > gpurun_out/b2_pytest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/b2_pytest.log
run() {  # tag wire chunks env...
  tag=$1; w=$2; c=$3; shift 3
  env DS_CHUNKS=$c "$@" timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline --no-makespan --wire $w > gpurun_out/b2_$tag.json 2> gpurun_out/b2_$tag.err
  echo "== $tag wire $w chunks $c $*: $(python -c "import json;d=json.load(open('gpurun_out/b2_$tag.json'));print('e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_leg'])")"
}
for c in 4 5 6; do run t$c tri $c; done
for c in 5 6 8; do run b3_$c tri $c DS_PIPE_BACKS=3; done
run s5 16 5
DS_E2E_TRACE=1 DS_CHUNKS=5 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan 2>&1 >/dev/null | tail -6
