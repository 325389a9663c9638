mkdir -p gpurun_out
timeout 900 python tools/exec_study.py --replays 200 --dags c1,c3,c4_0,c4_1,c4_2,c2:8 --windows c4_0 > gpurun_out/exec_study2.log 2>&1; echo "study rc $?"
tail -3 gpurun_out/exec_study2.log
PYTEST_ARGS="-k executor" bash tools/gpu_tests.sh
