mkdir -p gpurun_out
timeout 60 tools/heartbeat 10 4 50 > gpurun_out/hb_alone.json 2>&1; echo "hb rc $?"
nvidia-smi --query-compute-apps=pid,process_name,used_memory --format=csv > gpurun_out/apps.txt 2>&1
nvidia-smi -q -d COMPUTE,PERFORMANCE > gpurun_out/smi_q.txt 2>&1
timeout 900 python tools/exec_study.py --replays 100 > gpurun_out/exec_study.log 2>&1; echo "study rc $?"
tail -20 gpurun_out/exec_study.log
