# e2e host pipeline knobs: split front/back streams, stream priorities.
mkdir -p gpurun_out
run() {  # tag wire chunks env...
  tag=$1; w=$2; c=$3; shift 3
  env DS_E2E_TRACE=1 DS_CHUNKS=$c "$@" timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --no-cpu-baseline --no-makespan --wire $w > gpurun_out/p2_$tag.json 2> gpurun_out/p2_$tag.err
  echo "== $tag wire $w chunks $c $*: $(python -c "import json;d=json.load(open('gpurun_out/p2_$tag.json'));print('e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_leg'])")"
  tail -$c gpurun_out/p2_$tag.err
}
run a tri 4 DS_PIPE_SPLIT=0
run b tri 4 DS_STREAM_PRIO=0
run c tri 4 DS_PIPE_SPLIT=0 DS_STREAM_PRIO=0
run d tri 1
run e 16 1
run f wide 1
run g tri 2
run h tri 2 DS_PIPE_SPLIT=0
