# compute-sanitizer over the reworked k1_fast (ancestors-or-self closure,
# shared-atomic group masks in k1_fast<64>): memcheck and racecheck.
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_k1.py -q -x -k "seeded_corpora or triangular_wire_form_matches_wide or paper_benchmark" > gpurun_out/san3_$tool.log 2>&1
  echo "$tool rc $?"; tail -3 gpurun_out/san3_$tool.log
done
