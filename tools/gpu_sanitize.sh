# compute-sanitizer memcheck / racecheck over the newer device paths (big-DAG
# size classes, triangular lazy widening, K6 HBM slots, the dynamic engine).
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
CS="compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20"
timeout 1500 $CS python -m pytest tests/test_gpu_big.py -q -x -k "mixed or limit or small_host" > gpurun_out/san_big.log 2>&1; echo "memcheck big rc $?"; tail -4 gpurun_out/san_big.log
timeout 1500 $CS python -m pytest tests/test_gpu_k1.py -q -x -k "triangular" > gpurun_out/san_tri.log 2>&1; echo "memcheck tri rc $?"; tail -4 gpurun_out/san_tri.log
timeout 1500 $CS python -m pytest tests/test_gpu_simulator.py -q -x -k "big" > gpurun_out/san_k6.log 2>&1; echo "memcheck k6 rc $?"; tail -4 gpurun_out/san_k6.log
timeout 1500 $CS python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/san_exec.log 2>&1; echo "memcheck executor rc $?"; tail -4 gpurun_out/san_exec.log
