mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1.py tests/test_gpu_fuzz.py tests/test_division_api.py tests/test_cpp_api.py tests/test_abi.py -x -q > gpurun_out/pt_k1.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pt_k1.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-makespan > gpurun_out/bk1.json 2> gpurun_out/bk1.err; echo "bench rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bk1.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], json.dumps(d['roofline']['pass']['kernels_ms']))"
timeout 600 python tools/stall_probe2.py --hb-secs 30 --replays 40000 > gpurun_out/stall2.log 2>&1; echo "stall rc $?"; tail -12 gpurun_out/stall2.log | cut -c1-600
