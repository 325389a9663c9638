# e2e host-side timeline: enqueue end and synchronise time next to the chunk events.
DS_E2E_TRACE=1 DS_CHUNKS=4 timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline --no-makespan --wire tri 2>&1 >/dev/null | tail -12
