# compute-sanitizer over the smoke decision and a few parity tests (under gpurun)
cd "$(dirname "$0")/.."
O=gpurun_out/san; mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$tool.log 2>&1
  echo "smoke $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|smoke ok' $O/smoke_$tool.log | tr '\n' ' ')"
done
for tool in memcheck synccheck initcheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q -x -m gpu \
    "tests/test_gpu_parity.py::test_random_trees_gpu_equals_oracle[3]" \
    "tests/test_prefetch_round.py::test_prefetch_round_equals_reference_loop[5]" \
    "tests/test_delta.py" "tests/test_defer.py" > $O/tests_$tool.log 2>&1
  echo "tests $tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $O/tests_$tool.log | tail -2 | tr '\n' ' ')"
done
