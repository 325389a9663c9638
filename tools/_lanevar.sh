cp paper_2602_20826_b200/_lib/libdagsched_b200.so /tmp/orig.so
for v in mb8 mb10 mb12; do
  for c in 0 6 4 3 2; do
  cp lanevar/$v/libdagsched_b200.so paper_2602_20826_b200/_lib/libdagsched_b200.so
  DS_K1_LANE_CTAS_PER_SM=$c timeout 300 python bench.py --no-makespan --no-cpu-baseline --e2e-steps 1 --steps 10 > gpurun_out/bench_v.json 2>&1
  echo $v cps=$c $(tail -1 gpurun_out/bench_v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['pass']['kernels_ms'].get('k1_back_lane'), d['dags_ok'])")
  done
done
cp /tmp/orig.so paper_2602_20826_b200/_lib/libdagsched_b200.so
