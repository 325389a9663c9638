# e2e chunk timeline of the final pipeline (triangular form, 5 chunks, two back streams).
DS_E2E_TRACE=1 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-makespan 2>&1 >/dev/null | tail -7
python tools/chunk_eff_probe.py 2>&1 | tail -7
