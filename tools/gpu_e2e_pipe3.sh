# e2e host pipeline without tracing: wire x chunks x priorities.
mkdir -p gpurun_out
run() {  # tag wire chunks env...
  tag=$1; w=$2; c=$3; shift 3
  env DS_CHUNKS=$c "$@" timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline --no-makespan --wire $w > gpurun_out/p3_$tag.json 2> gpurun_out/p3_$tag.err
  echo "== $tag wire $w chunks $c $*: $(python -c "import json;d=json.load(open('gpurun_out/p3_$tag.json'));print('e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_leg'])")"
}
for c in 3 4 5 6 8; do run t$c tri $c; run tp$c tri $c DS_STREAM_PRIO=0; done
for c in 4 5 6; do run s$c 16 $c; run sn$c 16 $c DS_PIPE=0; done
run tn5 tri 5 DS_PIPE=0
