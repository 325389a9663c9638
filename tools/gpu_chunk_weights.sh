# e2e (triangular form) under non-uniform chunk sizes (DS_CHUNK_WEIGHTS).
run() {
  env DS_CHUNK_WEIGHTS=$1 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 10 --no-cpu-baseline --no-makespan --wire tri > gpurun_out/cw.json 2> gpurun_out/cw.err
  echo "== weights $1: $(python -c "import json;d=json.load(open('gpurun_out/cw.json'));print('e2e',round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3), d['e2e']['matches_device_leg'])")"
}
mkdir -p gpurun_out
for w in 1,1,1,1,1 2,2,2,2,1 3,3,3,3,2,1 1,2,2,2,2,1 4,4,4,4,2,1,1 2,3,3,3,2 1,2,3,3,2,1; do run $w; done
