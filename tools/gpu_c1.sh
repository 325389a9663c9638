# C1 latency: api_bench (small corpus), kernel durations of k1_small under ncu.
mkdir -p gpurun_out
./paper_2602_20826_b200/_lib/api_bench 1000 500 > gpurun_out/c1_api.json; cat gpurun_out/c1_api.json
./oracle/_ref/ref_api_bench 1000 500
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none -k regex:k1_small -c 40 --csv ./paper_2602_20826_b200/_lib/api_bench 1000 20 > gpurun_out/c1_ncu.csv 2>&1; tail -8 gpurun_out/c1_ncu.csv
