# Lane-walk task order: time (A/B, results checksummed) and k1_back_lane DRAM bytes.
mkdir -p gpurun_out
python tools/k1_env_ab.py DS_K1_WIDE_FIRST=0 DS_K1_WIDE_FIRST=1 2>&1 | grep -E "==|n 1000000" | sed 's/k1_analyse_retry.*//'
for wf in 0 1; do
  DS_K1_WIDE_FIRST=$wf timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k1_back_lane -s 3 -c 1 --csv python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-makespan 2>/dev/null \
    | grep -E "dram__bytes|gpu__time" | awk -F'","' -v wf=$wf '{print "wide_first=" wf, $(NF-2), $(NF)}'
done
