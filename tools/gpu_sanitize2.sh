# compute-sanitizer follow-up: executor memcheck without the bandwidth sanity
# test (instrumentation makes it slow by design), racecheck / synccheck on the
# shared-memory warp-state kernels (big-DAG classes, triangular fast path).
mkdir -p gpurun_out
CS="compute-sanitizer --error-exitcode 9 --print-limit 20"
timeout 1500 $CS --tool memcheck python -m pytest tests/test_gpu_executor.py -q -x -k "not bench_sane" > gpurun_out/san2_exec.log 2>&1; echo "memcheck executor rc $?"; tail -3 gpurun_out/san2_exec.log
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_big.py -q -x -k "limit or small_host" > gpurun_out/san2_race_big.log 2>&1; echo "racecheck big rc $?"; tail -3 gpurun_out/san2_race_big.log
timeout 1500 $CS --tool racecheck python -m pytest tests/test_gpu_k1.py -q -x -k "triangular_wire_form_invalid or fixtures_bounds" > gpurun_out/san2_race_k1.log 2>&1; echo "racecheck k1 rc $?"; tail -3 gpurun_out/san2_race_k1.log
timeout 1500 $CS --tool synccheck python -m pytest tests/test_gpu_k1.py -q -x -k "triangular_wire_form_invalid or fixtures_bounds" > gpurun_out/san2_sync_k1.log 2>&1; echo "synccheck k1 rc $?"; tail -3 gpurun_out/san2_sync_k1.log
